// cgbn_reduce.cuh — reduction kernels: flat, team, cluster-team (k_reduce_ct), channels_last rows
// Part of the single translation unit cgbn.cu (included there, in order).

#pragma once

namespace {

// flat reduction (see header). A CTA's slice covers consecutive channels c0, c0+1, ...
// (segments). Segments are processed in batches of up to kMaxSegF: first every
// segment's data is reduced to one CTA partial (warp shuffle, thread 0 folds the
// kWarps values in order), then the tails of all segments of the batch run in
// parallel — thread k publishes segment k's partial in slot (b + c) and takes the
// channel's arrival ticket (or finishes the channel directly when this CTA covers it
// alone), and warp k (mod kWarps) of the last CTA to arrive folds the slots b0+c..b1+c
// in index order and finishes the channel. Running the tails in parallel keeps the
// L2 round trips of one segment from delaying the loads of the next.
constexpr int kMaxSegF = 16;

template <class Op>
__global__ void __launch_bounds__(kThreads, 3)
k_reduce_flat(Geom g, Op op, double* __restrict__ out, double2* __restrict__ ws,
              unsigned* __restrict__ tickets) {
  pdl_wait();  // inputs may come from the previous kernel (PDL launch)
  pdl_trigger();
  __shared__ double sa[kWarps], sb[kWarps];
  __shared__ double s_S1[kMaxSegF], s_S2[kMaxSegF];
  __shared__ typename Op::Init s_init[kMaxSegF];
  __shared__ int s_last[kMaxSegF];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint64_t u_beg = cta_begin(g, blockIdx.x), u_end = cta_begin(g, blockIdx.x + 1);
  if (u_beg >= u_end) return;
  const uint32_t c_first = (uint32_t)(u_beg / g.Lv), c_last = (uint32_t)((u_end - 1) / g.Lv);
  for (uint32_t cb = c_first; cb <= c_last; cb += kMaxSegF) {
    const int nseg = (int)min((uint32_t)kMaxSegF, c_last - cb + 1);
    for (int k = 0; k < nseg; ++k) {
      const uint32_t c = cb + k;
      const uint64_t cbase = (uint64_t)c * g.Lv;
      const uint32_t j0 = (uint32_t)(max(u_beg, cbase) - cbase);
      const uint32_t j1 = (uint32_t)(min(u_end, cbase + g.Lv) - cbase);
      op.init(g, c);
      double S1, S2;
      reduce_range(g, c, j0 + threadIdx.x, j1, kThreads, op, S1, S2);
      S1 = warp_sum(S1);
      S2 = warp_sum(S2);
      if (l == 0) { sa[w] = S1; sb[w] = S2; }
      __syncthreads();
      if (threadIdx.x == 0) {
        S1 = sa[0]; S2 = sb[0];
#pragma unroll
        for (int i = 1; i < kWarps; ++i) { S1 += sa[i]; S2 += sb[i]; }
        s_S1[k] = S1;
        s_S2[k] = S2;
        s_init[k] = op.get_init();
      }
      __syncthreads();
    }
    // tails of the batch, one thread per segment
    if (threadIdx.x < nseg) {
      const int k = threadIdx.x;
      const uint32_t c = cb + k;
      const uint64_t cbase = (uint64_t)c * g.Lv;
      const uint32_t b0 = cta_of(g, cbase), b1 = cta_of(g, cbase + g.Lv - 1);
      int last = 0;
      if (b0 == b1) {
        Op o = op;
        o.set_init(s_init[k]);
        o.finish(g, c, s_S1[k], s_S2[k], out, o.prefetch(c));
      } else {
        ws[(size_t)blockIdx.x + c] = make_double2(s_S1[k], s_S2[k]);
        __threadfence();
        last = atomicAdd(&tickets[c], 1u) == b1 - b0;
      }
      s_last[k] = last;
    }
    __syncthreads();
    // folds: warp w takes segments w, w + kWarps, ... completed by this CTA
    for (int k = w; k < nseg; k += kWarps) {
      if (!s_last[k]) continue;
      const uint32_t c = cb + k;
      const uint64_t cbase = (uint64_t)c * g.Lv;
      const uint32_t b0 = cta_of(g, cbase), b1 = cta_of(g, cbase + g.Lv - 1);
      __threadfence();
      const uint32_t cnt = b1 - b0 + 1;
      double x1 = 0.0, x2 = 0.0;
      for (uint32_t i = l; i < cnt; i += 32) {
        const double2 t = __ldcg(&ws[(size_t)b0 + c + i]);
        x1 += t.x;
        x2 += t.y;
      }
      x1 = warp_sum(x1);
      x2 = warp_sum(x2);
      if (l == 0) {
        Op o = op;
        o.set_init(s_init[k]);
        o.finish(g, c, x1, x2, out);
        tickets[c] = 0u;  // leave the workspace reusable
      }
    }
    __syncthreads();  // smem is reused by the next batch
  }
}

// team reduction: 2^tpc_log2 threads per channel, 256/tpc channels per tile.
template <class Op>
__global__ void __launch_bounds__(kThreads, 3)
k_reduce_team(Geom g, Op op, double* __restrict__ out) {
  pdl_wait();  // inputs may come from the previous kernel (PDL launch)
  pdl_trigger();
  __shared__ double sa[kWarps], sb[kWarps];
  const uint32_t tpc = 1u << g.tpc_log2;
  const uint32_t cpt = kThreads >> g.tpc_log2;
  const uint32_t q = threadIdx.x & (tpc - 1);
  const uint32_t team = threadIdx.x >> g.tpc_log2;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t tiles = (g.C + cpt - 1) / cpt;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t c = tile * cpt + team;
    double S1 = 0.0, S2 = 0.0;
    typename Op::Pre pre;
    if (q == 0 && c < g.C) pre = op.prefetch(c);  // overlaps the data loads below
    if (c < g.C) {
      op.init(g, c);
      reduce_range(g, c, q, g.Lv, tpc, op, S1, S2);
    }
    S1 = warp_sum(S1);
    S2 = warp_sum(S2);
    if (tpc == 32) {
      if (l == 0 && c < g.C) op.finish(g, c, S1, S2, out, pre);
    } else {
      if (l == 0) { sa[w] = S1; sb[w] = S2; }
      __syncthreads();
      if (q == 0 && c < g.C) {
        const int wpt = (int)(tpc >> 5);
        for (int i = 1; i < wpt; ++i) { S1 += sa[w + i]; S2 += sb[w + i]; }
        op.finish(g, c, S1, S2, out, pre);
      }
      __syncthreads();
    }
  }
}

// cluster-team reduction (NCHW default). Cluster q of KC CTAs (runtime cluster size,
// 1..8) owns channels q*nch .. q*nch+nch-1 with nch = 256 >> TL. In every CTA of the
// cluster, team i (2^TL threads) streams CTA rank r's share [r*Lv/KC, (r+1)*Lv/KC) of
// channel q*nch+i with no block barrier: warp partials go to shared memory, one
// __syncthreads folds each team's warps in ascending order, one cluster barrier, then
// rank (i % KC) folds the KC CTA partials of channel i over DSMEM in rank order and
// finishes the channel. Compared with k_reduce_flat this removes the slot/ticket round
// trips through L2 (tools/flatlab.cu: 3-4 us per launch at ResNet mid shapes) and the
// per-segment block barriers. Clusters loop over q when C needs more CTAs than fit.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(v));
  return v;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(v));
  return v;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ double2 ld_dsmem(const double2* p, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}

template <class Op, int TL>
__global__ void __launch_bounds__(kThreads, CGBN_CT_MINB)
k_reduce_ct(Geom g, Op op, double* __restrict__ out) {
  pdl_wait();  // inputs may come from the previous kernel (PDL launch)
  pdl_trigger();
  constexpr uint32_t tpc = 1u << TL;
  constexpr uint32_t nch = kThreads >> TL;
  constexpr uint32_t wpt = tpc / 32;
  __shared__ double2 wpart[kWarps];
  __shared__ double2 cpart[nch];
  __shared__ typename Op::Pre spre[nch];
  const uint32_t KC = cluster_size(), r = cluster_rank();
  const uint32_t team = threadIdx.x >> TL, tq = threadIdx.x & (tpc - 1);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  // rank r's share of every channel stream: a balanced split in 32-bit arithmetic
  const uint32_t base = g.Lv / KC, rem = g.Lv - base * KC;
  const uint32_t j0 = r * base + min(r, rem);
  const uint32_t j1 = j0 + base + (r < rem ? 1u : 0u);
  const uint32_t nq = (g.C + nch - 1) / nch;
  for (uint32_t q = blockIdx.x / KC; q < nq; q += gridDim.x / KC) {
    const uint32_t c = q * nch + team;
    const bool live = c < g.C;
    const bool fin = live && tq == 0 && team % KC == r;
    Op o = op;
    if (fin) o.prefetch_async(c, &spre[team]);  // lands while the data streams
    double S1 = 0.0, S2 = 0.0;
    if (live) {
      o.init(g, c);
      reduce_range(g, c, j0 + tq, j1, tpc, o, S1, S2);
    }
    S1 = warp_sum(S1);
    S2 = warp_sum(S2);
    if (l == 0) wpart[w] = make_double2(S1, S2);
    if (fin) cp_async_wait_all();
    __syncthreads();
    if (tq == 0) {
      double2 t = wpart[team * wpt];
#pragma unroll
      for (uint32_t k = 1; k < wpt; ++k) {
        t.x += wpart[team * wpt + k].x;
        t.y += wpart[team * wpt + k].y;
      }
      cpart[team] = t;
    }
    if (KC > 1) cluster_barrier(); else __syncthreads();
    if (fin) {
      double a = 0.0, b = 0.0;
      for (uint32_t k = 0; k < KC; ++k) {
        const double2 t = ld_dsmem(&cpart[team], k);
        a += t.x;
        b += t.y;
      }
      o.finish(g, c, a, b, out, spre[team]);
    }
    // wpart/cpart are reused by the next q; peers may still be reading cpart over DSMEM
    if (KC > 1) cluster_barrier(); else __syncthreads();
  }
}

// ----------------------------------------------------------------------------------
// Row reductions for channels_last (NHWC) and 2-D (N, C) activations: M = N*H*W rows of
// C contiguous floats (C % 4 == 0). Thread = one float4 of 4 adjacent channels; the
// threads of a CTA cover a channel slice of CS4 float4 (<= 256) and rpp = 256 / CS4 rows
// per pass, so every warp load is a contiguous 512-byte row segment. A CTA reduces a
// block of rows; its per-channel partials are folded over the rpp thread rows in shared
// memory (ascending) and stored in slots[c * nb + row block]; k_fold_rows then folds
// the nb row blocks of each channel with one warp (fixed lane order + shuffle tree) and
// runs the channel finisher of the matching NCHW op. Deterministic, no atomics.

struct NGeom {
  uint32_t M;        // rows
  uint32_t C, C4;    // channels, float4 per row
  uint32_t CS4;      // float4 per channel slice (<= 256)
  uint32_t rpp;      // rows per pass = 256 / CS4
  uint32_t nslices;  // ceil(C4 / CS4)
  uint32_t nb;       // row blocks per slice
};

// fp32 rows per round (statistics / backward reduction without ReLU): 4 / 2 with two
// rounds in flight measured better than 8 / 4 one at a time (channels_last fp32 step
// 2.507 -> 2.467 ms, no spills; tools/gpu/rows_ab.sh, profiles/r2_rows_ab/)
#ifndef CGBN_ROWS_U32
#define CGBN_ROWS_U32 4
#endif
#ifndef CGBN_ROWS_BU32
#define CGBN_ROWS_BU32 2
#endif
#ifndef CGBN_ROWS_U16
#define CGBN_ROWS_U16 8  // 16-bit rows per round, statistics / backward (A/B knobs)
#endif
#ifndef CGBN_ROWS_BU16
#define CGBN_ROWS_BU16 4
#endif

// Forward statistics over rows: the shift K of every channel is the NCHW op's (row 0).
template <class T, bool PUSH = false>
struct StatsRows {
  static constexpr int kU = sizeof(T) == 4 ? CGBN_ROWS_U32 : CGBN_ROWS_U16;
  static constexpr int kIn = 1;
  static constexpr bool kPipe = true;  // two rounds in flight when they fit (k_reduce_rows)
  StatsOp<T, 1, PUSH> base;
  Geom gg;
  struct State { double K[4]; };
  struct Regs { Vec<T, 4> v; };
  __device__ __forceinline__ void init(uint32_t c4, State& s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      StatsOp<T, 1, PUSH> o = base;
      o.init(gg, 4 * c4 + j);
      s.K[j] = o.K;
    }
  }
  __device__ __forceinline__ void load(size_t u, Regs& r) const { r.v.load(base.x + 4 * u); }
  __device__ __forceinline__ void acc(const State& s, const Regs& r, double (&a)[4],
                                      double (&b)[4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double d = (double)r.v.get(j) - s.K[j];
      a[j] += d;
      b[j] = __fma_rn(d, d, b[j]);
    }
  }
  // A thread's U rows of one round. 16-bit activations: per channel, fp32 partials over
  // the round's rows, one fp64 add each (StatsOp::acc explains the error bound).
  template <int U>
  __device__ __forceinline__ void acc_round(const State& s, const Regs (&v)[U], uint32_t r,
                                            uint32_t r1, uint32_t rpp, double (&a)[4],
                                            double (&b)[4]) const {
    if constexpr (sizeof(T) == 2) {
      if (base.ksum == nullptr) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float Kf = (float)s.K[j];
          float sj = 0.f, qj = 0.f;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (r + u * rpp < r1) {
              const float d = v[u].v.get(j) - Kf;
              sj += d;
              qj = __fmaf_rn(d, d, qj);
            }
          a[j] += (double)sj;
          b[j] += (double)qj;
        }
        return;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u * rpp < r1) acc(s, v[u], a, b);
  }
};

// Backward sums over rows: [sum g, sum g*(x - mean)] with the forward's ReLU mask.
template <class T, bool RELU, bool PUSH = false>
struct BwdRows {
  static constexpr int kU = sizeof(T) == 4 ? CGBN_ROWS_BU32 : CGBN_ROWS_BU16;
  static constexpr int kIn = 2;
  static constexpr bool kPipe = !RELU;  // (the ReLU mask's state would spill)
  BwdOp<T, 1, RELU, PUSH> base;
  Geom gg;
  struct State { double mean[4], P[4], Q[4]; };
  struct Regs { Vec<T, 4> g, x; };
  __device__ __forceinline__ void init(uint32_t c4, State& s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      BwdOp<T, 1, RELU, PUSH> o = base;
      o.init(gg, 4 * c4 + j);
      s.mean[j] = o.mean;
      s.P[j] = RELU ? o.P : 0.0;
      s.Q[j] = RELU ? o.Q : 0.0;
    }
  }
  __device__ __forceinline__ void load(size_t u, Regs& r) const {
    r.g.load(base.dy + 4 * u);
    r.x.load(base.x + 4 * u);
  }
  __device__ __forceinline__ void acc(const State& s, const Regs& r, double (&a)[4],
                                      double (&b)[4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double gk = (double)r.g.get(j);
      const float xj = r.x.get(j);
      if (RELU && !(bn_out(s.P[j], s.Q[j], xj) > 0.0)) gk = 0.0;
      a[j] += gk;
      b[j] = __fma_rn(gk, (double)xj - s.mean[j], b[j]);
    }
  }
  // 16-bit activations without ReLU: per channel, sum g in an fp32 partial over the
  // round's rows, one fp64 add; sum g*(x - mean) in fp64 per element (BwdOp::acc).
  template <int U>
  __device__ __forceinline__ void acc_round(const State& s, const Regs (&v)[U], uint32_t r,
                                            uint32_t r1, uint32_t rpp, double (&a)[4],
                                            double (&b)[4]) const {
    if constexpr (sizeof(T) == 2 && !RELU) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float sj = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (r + u * rpp < r1) {
            const float gk = v[u].g.get(j);
            sj += gk;
            b[j] = __fma_rn((double)gk, (double)v[u].x.get(j) - s.mean[j], b[j]);
          }
        a[j] += (double)sj;
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u * rpp < r1) acc(s, v[u], a, b);
  }
};

template <class NOp>
__global__ void __launch_bounds__(kThreads, 3)
k_reduce_rows(NGeom g, NOp op, double2* __restrict__ slots) {
  pdl_wait();
  pdl_trigger();
  __shared__ double2 sm[4][kThreads];
  const uint32_t slice = blockIdx.x % g.nslices, rb = blockIdx.x / g.nslices;
  const uint32_t k = threadIdx.x % g.CS4, ro = threadIdx.x / g.CS4;
  const uint32_t c4 = slice * g.CS4 + k;
  const bool active = ro < g.rpp && c4 < g.C4;
  const uint32_t r0 = (uint32_t)((uint64_t)rb * g.M / g.nb);
  const uint32_t r1 = (uint32_t)((uint64_t)(rb + 1) * g.M / g.nb);
  double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
    typename NOp::State s;
    op.init(c4, s);
    constexpr int U = NOp::kU;
    // Two rounds in flight when a round's registers fit in 64 bytes (16-bit data; fp32
    // with 4 / 2 rows per round): round r + 1's loads are issued before round r is
    // reduced (a round at a time left each CTA waiting out one memory latency per round).
    constexpr bool kTwo = NOp::kPipe && sizeof(typename NOp::Regs) * U <= 64;
    typename NOp::Regs va[U], vb[kTwo ? U : 1];
    auto load_round = [&](uint32_t r, typename NOp::Regs (&v)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t rr = r + u * g.rpp;
        if (rr < r1) op.load((size_t)rr * g.C4 + c4, v[u]);
      }
    };
    const uint32_t step = U * g.rpp;
    if constexpr (kTwo) {
      uint32_t r = r0 + ro;
      if (r < r1) load_round(r, va);
      while (r < r1) {
        if (r + step < r1) load_round(r + step, vb);
        op.template acc_round<U>(s, va, r, r1, g.rpp, a, b);
        r += step;
        if (r >= r1) break;
        if (r + step < r1) load_round(r + step, va);
        op.template acc_round<U>(s, vb, r, r1, g.rpp, a, b);
        r += step;
      }
    } else {
      for (uint32_t r = r0 + ro; r < r1; r += step) {
        load_round(r, va);
        op.template acc_round<U>(s, va, r, r1, g.rpp, a, b);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) sm[j][threadIdx.x] = make_double2(a[j], b[j]);
  __syncthreads();
  if (ro == 0 && c4 < g.C4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2 t = sm[j][k];
      for (uint32_t q = 1; q < g.rpp; ++q) {
        const double2 v = sm[j][q * g.CS4 + k];
        t.x += v.x;
        t.y += v.y;
      }
      slots[(size_t)(4 * c4 + j) * g.nb + rb] = t;
    }
  }
}

// One warp per channel: fold the nb row-block partials (lane-strided, then the fixed
// shuffle tree) and finish the channel with the NCHW op's finisher.
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_fold_rows(Geom g, Op op, const double2* __restrict__ slots, uint32_t nb,
            double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const uint32_t c = (blockIdx.x * kThreads + threadIdx.x) >> 5, l = threadIdx.x & 31;
  if (c >= g.C) return;
  double a = 0.0, b = 0.0;
  const double2* p = slots + (size_t)c * nb;
  // all of a lane's slot loads are issued before the first add (a rolled loop waited
  // out one L2 round trip per slot); the adds keep the ascending per-lane order
  constexpr int FU = 8;
  for (uint32_t i0 = l; i0 < nb; i0 += 32 * FU) {
    double2 t[FU];
#pragma unroll
    for (int u = 0; u < FU; ++u)
      if (i0 + 32 * u < nb) t[u] = __ldcg(p + i0 + 32 * u);
#pragma unroll
    for (int u = 0; u < FU; ++u)
      if (i0 + 32 * u < nb) {
        a += t[u].x;
        b += t[u].y;
      }
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (l == 0) {
    Op o = op;
    o.init(g, c);
    o.finish(g, c, a, b, out);
  }
}

}  // namespace
