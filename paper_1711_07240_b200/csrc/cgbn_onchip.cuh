// cgbn_onchip.cuh — single-launch, on-chip BN passes for a single-rank group (sm_100a).
// Part of the single translation unit cgbn.cu (included there, in order).
//
// One BN direction is a per-channel reduction followed by an elementwise pass over the
// same data. When a layer's activations fit in the GPU's shared memory, both run in ONE
// kernel and the data crosses HBM once:
//
//   forward  (batchnorm.py:115-144): read x (4 B/elem) + write y (4)           = 8  B/elem
//   backward (batchnorm.py:188-210): read dy, x (8) + write dx (4)              = 12 B/elem
//
// instead of the split path's 12 and 20 (the elementwise pass re-reads x / dy). There is
// no grid-wide synchronisation: a thread-block cluster of KC CTAs owns `nch` whole
// channels, so a channel's statistics never leave the cluster.
//
// Decomposition (NCHW). Cluster q owns channels [q*nch, q*nch + nch); CTA rank r of the
// cluster owns images [n0_r, n1_r) of them (a balanced split of N). For image n those
// nch planes are ONE contiguous run of nch*HW elements at ((n*C + c0)*HW), so a CTA's
// data is (n1_r - n0_r) runs:
//   1. two warps issue a 1-D bulk copy (cp.async.bulk, mbarrier complete_tx) of every
//      run's 16-byte-aligned cover into shared memory -- the CTA's whole slice is in
//      flight at once, independent of registers;
//   2. once every run has landed (one mbarrier per run), a team of warps per channel
//      reduces the channel's planes out of shared memory (fp64 per element: forward
//      d = x - K with the rank's first element K, backward g and g*(x - mean) with the
//      recomputed ReLU mask);
//   3. warp partials -> one CTA partial per channel in shared memory; cluster barrier;
//      every CTA folds the KC CTA partials of each of its channels over DSMEM in rank
//      order (the same order everywhere, so every CTA derives bitwise-identical
//      coefficients) and runs the channel finisher of the split path
//      (finalize_fwd_channel / finalize_bwd_channel: running statistics, saved
//      statistics, dgamma / dbeta, written by CTA rank c % KC only);
//   4. the elementwise pass reads x (dy) from shared memory and writes y (dx) in memory
//      order over each run with 16-byte stores (scalar at run edges).
// The closing cluster barrier is split (arrive after the DSMEM reads, wait at exit), so
// the peers' last reads overlap the write phase.
//
// Deterministic (fixed thread -> element mapping and fold orders), no atomics. The
// host planner (cgbn_host.cuh onchip_plan) picks (nch, KC) so that every CTA is resident
// in one wave; layers that do not fit take the split kernels.
#pragma once

namespace {
namespace bulk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> this CTA's shared memory (16-byte aligned, multiple of 16 bytes),
// completing `bytes` of transaction count on `bar`
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace bulk
}  // namespace

namespace {
namespace onchip {

constexpr int kThreadsO = 512;
constexpr int kWarpsO = kThreadsO / 32;
constexpr int kMaxImg = 64;  // runs (images) per CTA: one mbarrier each

struct OGeom {
  uint32_t N, C, HW;
  uint32_t nch;         // channels per cluster
  uint32_t KC;          // CTAs per cluster (images split over the ranks)
  uint32_t run_stride;  // shared-memory bytes per run per input (16-aligned, >= cover)
  uint32_t nq;          // write-phase 16-byte chunks per run (aligned: exact; else cover slots)
  uint32_t wpc_log2;    // log2(warps per channel team)
  uint32_t HWv;         // reduction units per plane (HW / VE)
  uint32_t HWu;         // 16-byte chunks per plane (aligned path)
  FastDiv dhwv;         // / HWv
  FastDiv dhw;          // / HW
  FastDiv dhwu;         // / HWu
  FastDiv dnq;          // / nq
  double count;         // N*HW: this rank's elements per channel
};

// Shared-memory header (before the per-channel arrays and the data runs).
constexpr uint32_t kGroups = 4;  // copy groups: the reduction of group g overlaps the copies of g+1..

struct alignas(16) Head {
  uint64_t bar[kGroups];       // one mbarrier per copy group (arrivals = its runs)
  double2 wpart[kWarpsO];
  uint32_t gend[kGroups];      // first run of the next group
  uint8_t lead[kMaxImg];       // elements between a run's 16-byte-aligned cover and its start
};

// Relaxed arrive: it only has to follow this CTA's DSMEM reads of the peers' partials
// (their values are in registers by then), so it needs no release fence -- the .release
// form compiles to MEMBAR.ALL.GPU, which waits for the finisher's global stores.
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Per-channel arrays after the header (16-byte aligned each).
template <bool BWD>
struct ChanArrays {
  double2* part;  // this CTA's partial per channel (read by the peers over DSMEM)
  double* K;      // forward: shift; backward: mean
  double2* c01;   // forward (P, Q); backward (A, B)
  double2* c2;    // backward (Cc, -)
  double2* pq;    // backward ReLU mask (P, Q)
  typename std::conditional<BWD, BwdChan, FwdChan>::type* pre;  // finisher inputs
};

template <bool BWD>
__host__ __device__ inline size_t chan_bytes(uint32_t nch) {
  using Pre = typename std::conditional<BWD, BwdChan, FwdChan>::type;
  return (size_t)nch * (16 + 8 + 16 * (BWD ? 3 : 1) + ((sizeof(Pre) + 15) / 16) * 16) + 16;
}

template <bool BWD>
__device__ __forceinline__ ChanArrays<BWD> chan_arrays(unsigned char* base, uint32_t nch) {
  using Pre = typename std::conditional<BWD, BwdChan, FwdChan>::type;
  ChanArrays<BWD> a;
  size_t o = 0;
  a.part = reinterpret_cast<double2*>(base + o);
  o += (size_t)nch * 16;
  a.c01 = reinterpret_cast<double2*>(base + o);
  o += (size_t)nch * 16;
  a.c2 = reinterpret_cast<double2*>(base + o);
  a.pq = a.c2 + (BWD ? nch : 0);
  o += BWD ? (size_t)nch * 32 : 0;
  a.pre = reinterpret_cast<Pre*>(base + o);
  o += (size_t)nch * ((sizeof(Pre) + 15) / 16) * 16;
  a.K = reinterpret_cast<double*>(base + o);
  return a;
}

// Vector of VE elements from shared memory (VE * sizeof(T) <= 16 bytes, aligned).
template <class T, int VE>
__device__ __forceinline__ void lds_vec(uint32_t addr, float (&v)[VE]) {
  constexpr int B = VE * (int)sizeof(T);
  uint32_t w[4];
  if constexpr (B == 16) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(addr));
  } else if constexpr (B == 8) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(addr));
  } else if constexpr (B == 4) {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(addr));
  } else {
    unsigned short h;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(addr));
    w[0] = h;
  }
#pragma unroll
  for (int k = 0; k < VE; ++k) {
    if constexpr (sizeof(T) == 4) v[k] = __uint_as_float(w[k]);
    else v[k] = h2f<T>((unsigned short)(w[k >> 1] >> (16 * (k & 1))));
  }
}

struct Args {
  const void* x;
  const void* dy;   // backward
  void* out;        // y or dx
  FwdFinal F;       // forward finisher (P/Q null: coefficients stay in shared memory)
  BwdFinal B;       // backward finisher (A..Q null)
  // Statistics only (the rank partial of a multi-rank group, for the exchange): the
  // channel finishers write [mean | M2 | count] (forward) or [sum g | sum g*(x-mean)]
  // (backward) to `partial`, or push it into the fused exchange's regions (push.G > 0),
  // and there is no elementwise pass. Every path that reduces an on-chip-eligible layer
  // uses this kernel, so a rank's statistics are bitwise the same whichever way the
  // group exchanges them.
  double* partial;
  p2p::Push push;
  unsigned long long* trace;  // debug (tools/onchip_trace.py): per-CTA phase timestamps
};

// Debug phase stamps: globaltimer at phase boundaries of CTA b in trace[b * 16 + s]
// (8..11: each copy group landed), trace[b * 16 + 15] = the SM id. Off (null) in every
// production launch.
__device__ __forceinline__ void stamp(const Args& a, int s) {
  if (a.trace && threadIdx.x == 0) {
    a.trace[blockIdx.x * 16 + s] = p2p::now_ns();
    if (s == 0) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      a.trace[blockIdx.x * 16 + 15] = sm;
    }
  }
}

// A channel's rank partial: to `partial` (the layout of the split reductions' kPartial
// finishers), or pushed into row `rank` of every region of the fused exchange, the last
// of the C finishers publishing the rank's flag (p2p::push_done).
__device__ __forceinline__ void partial_out(const Args& a, uint32_t C, uint32_t c, double v0,
                                            double v1, bool with_count, double n) {
  if (a.push.G > 0) {
    const p2p::Push& P = a.push;
    const unsigned long long e = p2p::push_epoch(P);
#pragma unroll
    for (int q = 0; q < p2p::kMaxPush; ++q) {
      if (q >= P.G) break;
      double* dst = p2p::recv_ptr(P.base[q], P.G, P.max_len, (int)(e & 1ull), P.rank);
      dst[c] = v0;
      dst[C + c] = v1;
      if (with_count && c == 0) dst[2 * C] = n;
    }
    p2p::push_done(P, e);
    return;
  }
  a.partial[c] = v0;
  a.partial[C + c] = v1;
  if (with_count && c == 0) a.partial[2 * C] = n;
}

// Balanced image range of CTA rank r.
__device__ __forceinline__ void img_range(const OGeom& g, uint32_t r, uint32_t& n0,
                                          uint32_t& n1) {
  const uint32_t base = g.N / g.KC, rem = g.N - base * g.KC;
  n0 = r * base + min(r, rem);
  n1 = n0 + base + (r < rem ? 1u : 0u);
}

// Accumulate one VE-element unit: forward (d = x - K): a += d, b += d*d; backward
// (g = ReLU-masked dy): a += g, b += g*(x - mean).
// MASKED: `mask` selects the unit's elements that belong to the plane (odd planes are
// read as masked 16-byte covers, as the split reductions' masked vector modes do).
template <class T, int VE, bool BWD, bool RELU, bool MASKED>
__device__ __forceinline__ void acc_unit(uint32_t ax, uint32_t ag, uint32_t mask, double K,
                                         double P, double Q, double& a, double& b) {
  float xv[VE];
  lds_vec<T, VE>(ax, xv);
  if constexpr (!BWD && sizeof(T) == 2) {
    // 16-bit activations, as the split statistics kernels: K (a 16-bit value) and x are
    // exact in fp32, the unit's differences and squares are summed in fp32 and added once
    const float Kf = (float)K;
    float s = 0.f, q = 0.f;
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      if (MASKED && !((mask >> e) & 1u)) continue;
      const float d = xv[e] - Kf;
      s += d;
      q = __fmaf_rn(d, d, q);
    }
    a += (double)s;
    b += (double)q;
  } else if constexpr (!BWD) {
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      if (MASKED && !((mask >> e) & 1u)) continue;
      const double d = (double)xv[e] - K;
      a += d;
      b = __fma_rn(d, d, b);
    }
  } else if constexpr (sizeof(T) == 2 && !RELU) {
    // 16-bit backward: sum g in an fp32 partial of the unit; g*(x - mean) in fp64 per
    // element (BwdOp::acc explains why)
    float gv[VE];
    lds_vec<T, VE>(ag, gv);
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      if (MASKED && !((mask >> e) & 1u)) continue;
      s += gv[e];
      b = __fma_rn((double)gv[e], (double)xv[e] - K, b);
    }
    a += (double)s;
  } else {
    float gv[VE];
    lds_vec<T, VE>(ag, gv);
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      if (MASKED && !((mask >> e) & 1u)) continue;
      double gk = (double)gv[e];
      if (RELU && !(bn_out(P, Q, xv[e]) > 0.0)) gk = 0.0;
      a += gk;
      b = __fma_rn(gk, (double)xv[e] - K, b);
    }
  }
}

// Element mask of masked unit o of a plane whose first element sits `s0` elements into
// its first 16-byte chunk.
template <int UE>
__device__ __forceinline__ uint32_t unit_mask(uint32_t o, uint32_t s0, uint32_t HW) {
  const int lo = (int)s0 - (int)(o * UE);  // plane start relative to the unit
  const int hi = lo + (int)HW;
  uint32_t m = 0u;
#pragma unroll
  for (int e = 0; e < UE; ++e) m |= (e >= lo && e < hi) ? (1u << e) : 0u;
  return m;
}

// VE == 16 / sizeof(T) ("aligned"): every run is 16-byte aligned and a 16-byte chunk
// never crosses a plane (HW % VE == 0). VE == 1 ("odd planes"): runs carry a lead; the
// reduction reads each plane as masked 16-byte covers and the write pass gives a chunk
// the coefficients of the (at most two) channels it spans.
template <class T, int VE, bool BWD, bool RELU>
__global__ void __launch_bounds__(kThreadsO, 2)
k_onchip(OGeom g, Args a) {
  constexpr uint32_t es = sizeof(T);
  constexpr int UE = 16 / (int)es;  // elements per 16-byte chunk
  constexpr bool ALIGNED = VE == UE;
  constexpr uint32_t NIN = BWD ? 2 : 1;
  // 16-bit activations without ReLU, aligned planes: the write pass in fp32 from fp32
  // records the finisher leaves in c01 / c2 (the split kernels' k_ew_affine / k_ew_dx
  // fp32 form, cgbn_ew.cuh: no fp64 conversion per element)
  constexpr bool kF32W = sizeof(T) == 2 && !RELU && ALIGNED;
  extern __shared__ __align__(16) unsigned char smem[];
  Head& H = *reinterpret_cast<Head*>(smem);
  const uint32_t KC = g.KC;
  const uint32_t r = KC > 1 ? cluster_rank() : 0u;
  const uint32_t cbase = (blockIdx.x / KC) * g.nch;
  const uint32_t nch = min(g.nch, g.C - cbase);  // channels of this cluster
  uint32_t n0, n1;
  img_range(g, r, n0, n1);
  const uint32_t nk = n1 - n0;
  ChanArrays<BWD> ca = chan_arrays<BWD>(smem + sizeof(Head), g.nch);
  const uint32_t data =
      (uint32_t)__cvta_generic_to_shared(smem) +
      (uint32_t)(((sizeof(Head) + chan_bytes<BWD>(g.nch) + 15) / 16) * 16);
  const uint32_t kstride = NIN * g.run_stride;  // bytes per image slot (dy | x)
  const uint32_t xoff = (NIN - 1) * g.run_stride;
  const uint32_t run_elems = nch * g.HW;
  const T* xg = static_cast<const T*>(a.x);
  T* og = static_cast<T*>(a.out);
  // element index of run k's first element in the tensor
  auto run_start = [&](uint32_t k) -> size_t {
    return ((size_t)(n0 + k) * g.C + cbase) * g.HW;
  };

  // copy groups: run k belongs to group k * ng / nk; group g's mbarrier expects one
  // arrival (with its bytes) per run
  const uint32_t ng = min(nk, kGroups);
  auto grp = [&](uint32_t k) -> uint32_t { return (k * ng) / nk; };
  stamp(a, 0);
  if (threadIdx.x == 0) {
    for (uint32_t q = 0; q < ng; ++q) {
      const uint32_t k0 = (q * nk + ng - 1) / ng, k1 = ((q + 1) * nk + ng - 1) / ng;
      bulk::mbar_init(&H.bar[q], k1 - k0);
      H.gend[q] = k1;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!ALIGNED)  // each run's lead (elements before its first in its 16-byte cover)
    for (uint32_t k = threadIdx.x; k < nk; k += kThreadsO)
      H.lead[k] = (uint8_t)(((run_start(k) * es) & 15u) / es);
  __syncthreads();
  pdl_wait();  // x / dy (and the finisher inputs) may come from the previous kernel
  pdl_trigger();
  stamp(a, 1);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    // ---- 1. lane 0 of warp w: runs w, w + 16, ...: expect the run's bytes, then issue
    // its bulk copies (a bulk copy is a uniform-datapath instruction, so the lanes of one
    // warp would issue theirs one after another: ~90 cycles each)
    for (uint32_t k = (uint32_t)w; k < nk; k += kWarpsO) {
      const size_t gs = run_start(k);
      const size_t b0 = (gs * es) & ~(size_t)15;
      const size_t b1 = ((gs + run_elems) * es + 15) & ~(size_t)15;
      const uint32_t bytes = (uint32_t)(b1 - b0);
      unsigned char* dst = smem + (data - (uint32_t)__cvta_generic_to_shared(smem)) +
                           (size_t)k * kstride;
      uint64_t* bar = &H.bar[grp(k)];
      bulk::mbar_expect_tx(bar, bytes * NIN);
      if (BWD) bulk::g2s(dst, static_cast<const unsigned char*>(a.dy) + b0, bytes, bar);
      bulk::g2s(dst + xoff, reinterpret_cast<const unsigned char*>(xg) + b0, bytes, bar);
    }
    stamp(a, 2);
  } else {
    // lanes 1..31: the finisher's per-channel inputs, landing while the data streams
    // (read after the barriers that close the reduction)
    // with cp.async: no register waits, so the warp reconverges at once
    if (a.partial == nullptr && a.push.G == 0)
      for (uint32_t i = (uint32_t)w * 31 + (l - 1); i < nch; i += kWarpsO * 31) {
        if constexpr (!BWD) load_fwd_chan_async(a.F, cbase + i, &ca.pre[i]);
        else load_bwd_chan_async(a.B, cbase + i, &ca.pre[i]);
      }
  }
  stamp(a, 3);

  // ---- 2. per-channel reduction out of shared memory (two units in flight per thread)
  {
    const uint32_t wpc = 1u << g.wpc_log2;
    const uint32_t nteams = kWarpsO >> g.wpc_log2;
    const uint32_t team = (uint32_t)w >> g.wpc_log2;
    const uint32_t tq = ((uint32_t)w & (wpc - 1)) * 32 + l;
    const uint32_t tstride = wpc * 32;
    const uint32_t total = nk * g.HWv;
    const uint32_t sq = g.dhwv.div(tstride), sr = tstride - sq * g.HWv;
    for (uint32_t i = team; i < g.nch; i += nteams) {
      double s1a = 0.0, s2a = 0.0, s1b = 0.0, s2b = 0.0;
      double K = 0.0;  // forward: this CTA's shift; backward: the forward mean
      if (i < nch) {
        double P = 0.0, Q = 0.0;
        if constexpr (BWD) {
          const uint32_t c = cbase + i;
          K = a.B.saved[c];
          if (RELU)
            affine_coeffs(K, a.B.saved[2 * g.C + c], (double)a.B.gamma[c], (double)a.B.beta[c],
                          P, Q);
          if (RELU && tq == 0) ca.pq[i] = make_double2(P, Q);  // for the dx pass
        }
        uint32_t k = g.dhwv.div(tq), o = tq - k * g.HWv;
        // aligned: unit o is VE elements at plane offset o * VE; odd planes: unit o is the
        // o-th 16-byte chunk of the plane's aligned cover (mask: the plane's elements)
        auto addr = [&](uint32_t kk, uint32_t oo, uint32_t& mask) -> uint32_t {
          if constexpr (ALIGNED) {
            mask = 0xffu;
            return data + kk * kstride + xoff + (i * g.HW + oo * VE) * es;
          } else {
            const uint32_t st = (uint32_t)H.lead[kk] + i * g.HW;  // plane start (elements)
            const uint32_t s0 = st & (UE - 1);
            mask = unit_mask<UE>(oo, s0, g.HW);
            return data + kk * kstride + xoff + ((st - s0) + oo * UE) * es;
          }
        };
        auto step = [&](uint32_t& kk, uint32_t& oo) {
          oo += sr;
          kk += sq;
          if (oo >= g.HWv) { oo -= g.HWv; ++kk; }
        };
        // the copy groups this thread has waited for: [0, gw); next group starts at run gk
        uint32_t gw = 0, gk = 0;
        for (uint32_t j = tq; j < total; j += 2 * tstride) {
          uint32_t k2 = k, o2 = o;
          step(k2, o2);
          const bool two = j + tstride < total;
          const uint32_t kl = two ? k2 : k;  // the later run of the two units
          while (kl >= gk) {
            bulk::mbar_wait(&H.bar[gw], 0);
            stamp(a, 8 + (int)gw);  // debug: thread 0 sees copy group gw landed
            gk = H.gend[gw];
            if (!BWD && gw == 0) {
              // forward shift: this CTA's first element of the channel (run 0, group 0);
              // the CTA partials are merged with Chan's update, so K may differ per CTA
              float kv[1];
              lds_vec<T, 1>(data + xoff + ((ALIGNED ? 0u : (uint32_t)H.lead[0]) + i * g.HW) * es,
                            kv);
              K = (double)kv[0];
            }
            ++gw;
          }
          constexpr int UV = ALIGNED ? VE : UE;
          uint32_t ma, mb = 0u;
          const uint32_t ua = addr(k, o, ma);
          if (ALIGNED || ma)
            acc_unit<T, UV, BWD, RELU, !ALIGNED>(ua, ua - xoff, ma, K, P, Q, s1a, s2a);
          if (two) {
            const uint32_t ub = addr(k2, o2, mb);
            if (ALIGNED || mb)
              acc_unit<T, UV, BWD, RELU, !ALIGNED>(ub, ub - xoff, mb, K, P, Q, s1b, s2b);
          }
          k = k2;
          o = o2;
          step(k, o);
        }
      }
      const double S1 = warp_sum(s1a + s1b);
      const double S2 = warp_sum(s2a + s2b);
      // forward: a thread that had no unit never read K; the team's thread 0 always has
      // one (tq = 0 < total), and it finishes the partial
      auto partial = [&](double a1, double a2) -> double2 {
        if constexpr (BWD) return make_double2(a1, a2);
        const double nr = (double)nk * g.HW;  // this CTA's count (mean_r, M2_r)
        return make_double2(K + a1 / nr, fmax(a2 - a1 * (a1 / nr), 0.0));
      };
      if (wpc == 1) {
        if (l == 0 && i < nch) ca.part[i] = partial(S1, S2);
      } else {
        if (l == 0) H.wpart[w] = make_double2(S1, S2);
        // the team's warps meet in shared memory; the team's first warp folds the wpc
        // warp partials with the fixed shuffle tree (lane u holds warp u's partial)
        asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(tstride) : "memory");
        if (tq < 32) {
          double2 t = make_double2(0.0, 0.0);
          if ((uint32_t)l < wpc) t = H.wpart[w + l];
          t.x = warp_sum(t.x);
          t.y = warp_sum(t.y);
          if (l == 0 && i < nch) ca.part[i] = partial(t.x, t.y);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(tstride) : "memory");
      }
    }
  }
  cp_async_wait_all();  // this thread's finisher inputs (phase 1)
  if (KC > 1) cluster_barrier();
  else __syncthreads();
  stamp(a, 4);

  // ---- 3. fold the KC CTA partials (rank order) and finish every channel
  for (uint32_t i = threadIdx.x; i < nch; i += kThreadsO) {
    const uint32_t c = cbase + i;
    const bool write = (i % KC) == r;
    const bool stats_only = a.partial != nullptr || a.push.G > 0;
    if constexpr (!BWD) {
      // Chan's pairwise merge of the KC CTA partials (n_u, mean_u, M2_u), rank order
      const double2 t0 = KC > 1 ? ld_dsmem(&ca.part[i], 0) : ca.part[i];
      double n, mean = t0.x, M2 = t0.y;
      {
        uint32_t u0, u1;
        img_range(g, 0, u0, u1);
        n = (double)(u1 - u0) * g.HW;
      }
      for (uint32_t u = 1; u < KC; ++u) {
        const double2 t = ld_dsmem(&ca.part[i], u);
        uint32_t u0, u1;
        img_range(g, u, u0, u1);
        const double nb = (double)(u1 - u0) * g.HW, nn = n + nb;
        const double delta = t.x - mean;
        mean = mean + delta * (nb / nn);
        M2 = M2 + t.y + delta * delta * (n * nb / nn);
        n = nn;
      }
      if (stats_only) {
        if (write) partial_out(a, g.C, c, mean, M2, true, n);
        continue;
      }
      double P, Q;
      finalize_fwd_channel(a.F, c, n, mean, M2, write, ca.pre[i], P, Q);
      if constexpr (kF32W) {  // the fp32 write below: {P, mean_hi, mean_lo, beta}
        const float mh = (float)mean;
        reinterpret_cast<float4*>(ca.c01)[i] =
            make_float4((float)P, mh, (float)(mean - (double)mh), ca.pre[i].beta);
      } else {
        ca.c01[i] = make_double2(P, Q);
      }
    } else {
      double S1 = 0.0, S2 = 0.0;
      for (uint32_t u = 0; u < KC; ++u) {
        const double2 t = KC > 1 ? ld_dsmem(&ca.part[i], u) : ca.part[i];
        S1 += t.x;
        S2 += t.y;
      }
      if (stats_only) {
        if (write) partial_out(a, g.C, c, S1, S2, false, 0.0);
        continue;
      }
      const DxCoef k = finalize_bwd_channel(a.B, c, S1, S2, write, ca.pre[i]);
      if constexpr (kF32W) {  // {A, B, C3 = Cc + B mean, mean_hi}, {mean_lo}
        const double mean = ca.pre[i].mean;
        const float mh = (float)mean;
        reinterpret_cast<float4*>(ca.c01)[i] =
            make_float4((float)k.A, (float)k.B, (float)(k.Cc + k.B * mean), mh);
        reinterpret_cast<float4*>(ca.c2)[i] =
            make_float4((float)(mean - (double)mh), 0.f, 0.f, 0.f);
      } else {
        ca.c01[i] = make_double2(k.A, k.B);
        ca.c2[i] = make_double2(k.Cc, 0.0);
      }
    }
  }
  if (KC > 1) cluster_arrive_relaxed();  // done reading the peers' partials
  __syncthreads();
  stamp(a, 5);

  // ---- 4. elementwise pass from shared memory, memory order over each run
  if (a.partial != nullptr || a.push.G > 0) {
    // statistics only: no elementwise pass
  } else if constexpr (ALIGNED) {
    // 16-byte chunks; a chunk lies in one plane: one coefficient lookup per chunk
    const uint32_t total = nk * g.nq;
    for (uint32_t j = threadIdx.x; j < total; j += kThreadsO) {
      const uint32_t k = g.dnq.div(j), qq = j - k * g.nq;
      const uint32_t i = g.dhwu.div(qq);
      const uint32_t sx = data + k * kstride + xoff + qq * 16;
      float xv[UE];
      lds_vec<T, UE>(sx, xv);
      if constexpr (kF32W) {
        float of[UE];
        const float4 t = reinterpret_cast<const float4*>(ca.c01)[i];
        if constexpr (!BWD) {
#pragma unroll
          for (int e = 0; e < UE; ++e) of[e] = fmaf(t.x, (xv[e] - t.y) - t.z, t.w);
        } else {
          float gv[UE];
          lds_vec<T, UE>(sx - xoff, gv);
          const float ml = reinterpret_cast<const float4*>(ca.c2)[i].x;
#pragma unroll
          for (int e = 0; e < UE; ++e)
            of[e] = fmaf(t.x, gv[e], fmaf(t.y, (xv[e] - t.w) - ml, t.z));
        }
        stvf<T, UE>(og + run_start(k) + (size_t)qq * UE, of);
        continue;
      }
      double o[UE];
      if constexpr (!BWD) {
        const double2 pq = ca.c01[i];
#pragma unroll
        for (int e = 0; e < UE; ++e) {
          double t = __fma_rn(pq.x, (double)xv[e], pq.y);
          if (RELU) t = t > 0.0 ? t : 0.0;
          o[e] = t;
        }
      } else {
        float gv[UE];
        lds_vec<T, UE>(sx - xoff, gv);
        const double2 ab = ca.c01[i];
        const double cc = ca.c2[i].x;
        double2 pq = make_double2(0.0, 0.0);
        if (RELU) pq = ca.pq[i];
#pragma unroll
        for (int e = 0; e < UE; ++e) {
          double gk = (double)gv[e];
          if (RELU && !(bn_out(pq.x, pq.y, xv[e]) > 0.0)) gk = 0.0;
          o[e] = __fma_rn(ab.x, gk, __fma_rn(ab.y, (double)xv[e], cc));
        }
      }
      stv<T, UE>(og + run_start(k) + (size_t)qq * UE, o);
    }
  } else {
    // runs with a lead: walk the 16-byte chunks of each cover, channel per element
    const uint32_t total = nk * g.nq;
    for (uint32_t j = threadIdx.x; j < total; j += kThreadsO) {
      const uint32_t k = g.dnq.div(j), qq = j - k * g.nq;
      const uint32_t lead = H.lead[k];
      if (qq * UE >= lead + run_elems) continue;  // past the run's cover
      const uint32_t sx = data + k * kstride + xoff + qq * 16;
      float xv[UE], gv[UE];
      lds_vec<T, UE>(sx, xv);
      if (BWD) lds_vec<T, UE>(sx - xoff, gv);
      // element e of the chunk is run element qq*UE + e - lead; a chunk spans at most two
      // channels (HW >= 4 > UE / 2 ... planes are at least UE / 2 elements: host check):
      // channel i for e < cut, i + 1 from there on
      const int r0 = (int)(qq * UE) - (int)lead;
      const uint32_t rel = r0 > 0 ? (uint32_t)r0 : 0u;
      const uint32_t i = g.dhw.div(rel);
      const int cut = (int)((i + 1) * g.HW) - r0;  // first e in channel i + 1
      const uint32_t i1 = min(i + 1, nch - 1);
      const double2 c0a = ca.c01[i], c0b = ca.c01[i1];
      double2 c2a = make_double2(0.0, 0.0), c2b = c2a, pqa = c2a, pqb = c2a;
      if (BWD) { c2a = ca.c2[i]; c2b = ca.c2[i1]; }
      if (BWD && RELU) { pqa = ca.pq[i]; pqb = ca.pq[i1]; }
      double o[UE];
      uint32_t inmask = 0;
#pragma unroll
      for (int e = 0; e < UE; ++e) {
        const int re = r0 + e;
        if (re >= 0 && re < (int)run_elems) inmask |= 1u << e;
        const bool hi = e >= cut;
        const double2 c01 = hi ? c0b : c0a;
        double t;
        if constexpr (!BWD) {
          t = __fma_rn(c01.x, (double)xv[e], c01.y);
          if (RELU) t = t > 0.0 ? t : 0.0;
        } else {
          const double2 pq = hi ? pqb : pqa;
          double gk = (double)gv[e];
          if (RELU && !(bn_out(pq.x, pq.y, xv[e]) > 0.0)) gk = 0.0;
          t = __fma_rn(c01.x, gk, __fma_rn(c01.y, (double)xv[e], (hi ? c2b : c2a).x));
        }
        o[e] = t;
      }
      T* dst = og + run_start(k) + r0;  // the chunk's first element (may precede the run)
      if (inmask == (1u << UE) - 1u) {
        stv<T, UE>(dst, o);
      } else {
#pragma unroll
        for (int e = 0; e < UE; ++e)
          if ((inmask >> e) & 1u) st1(dst + e, o[e]);
      }
    }
  }
  if (a.trace) {
    __syncthreads();
    stamp(a, 6);
  }
  if (KC > 1) cluster_wait();  // peers may still read this CTA's partials until here
}

}  // namespace onchip
}  // namespace
