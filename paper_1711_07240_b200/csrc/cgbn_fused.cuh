// cgbn_fused.cuh — single-launch, on-chip-resident CGBN forward / backward (sm_100a).
//
// For activations that fit in the GPU's shared memory (one 512-thread CTA per SM,
// ~200 KB each: ~7.4M fp32 elements forward, ~3.7M backward where dy and x are both
// held) the two passes of each BN direction are fused into one cooperative kernel:
//
//   1. all 512 threads issue 16-byte cp.async copies of this CTA's slice of the
//      channel-major stream into shared memory (~200 KB per SM requested at once; 1-D
//      TMA bulk copies were measured slower here because ResNet planes are as small as
//      784 B), tracked by kQuarters mbarriers so the reduction starts on the first
//      quarter;
//   2. all 16 warps reduce each channel segment of the slice out of shared memory
//      (fp64 per element) and publish one partial per (CTA, channel) in workspace slot
//      (b + c);
//   3. software grid barrier (co-residency guaranteed by the cooperative launch);
//   4. every CTA folds the slots of its channels in index order — the same fixed order
//      on every CTA, so the statistics are bitwise identical wherever they are used —
//      and derives the per-channel coefficients (the first CTA of a channel also writes
//      the saved statistics / running stats / dgamma, dbeta);
//   5. the elementwise pass reads x (and dy) from shared memory and writes y (dx).
//
// x (and dy) therefore cross HBM once: forward traffic 8 B/elem instead of 12,
// backward 12 B/elem instead of 20, and one launch per direction instead of two.
// Eligibility (host): NCHW, HW % 4 == 0 (16-byte plane pieces), 16-byte aligned
// pointers, slice <= capacity, <= kMaxSeg channel segments per CTA. Single rank group
// (G == 1): multi-rank groups use the split kernels around the exchange.
#pragma once

namespace fused {

constexpr int kThreadsF = 512;
constexpr int kWarpsF = kThreadsF / 32;
constexpr int kQuarters = 4;
constexpr int kMaxSeg = 48;
constexpr size_t kDataBytes = 200 * 1024;
constexpr size_t kSmemBytes = kDataBytes;

struct FGeom {
  uint32_t C, HW;
  uint32_t L;     // floats per channel stream (N*HW)
  uint32_t grid;  // CTAs (== co-resident)
  uint64_t T4;    // C*L/4
  FastDiv dhw;
  double count;   // N*HW
};

__device__ __forceinline__ uint64_t fslice(const FGeom& g, uint32_t b) {
  return ((uint64_t)b * g.T4 / g.grid) * 4;
}
__device__ __forceinline__ uint32_t fcta_of(const FGeom& g, uint64_t f) {
  return (uint32_t)((((f >> 2) + 1) * (uint64_t)g.grid - 1) / g.T4);
}
__device__ __forceinline__ size_t foff(const FGeom& g, uint32_t c, uint32_t w) {
  const uint32_t n = g.dhw.div(w);
  return ((size_t)n * g.C + c) * g.HW + (w - n * g.HW);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Sense-reversing software grid barrier over the co-resident grid. bar[0] counts
// arrivals (reset by the last arriver), bar[1] is the generation. The spin is bounded
// (5 s): a grid that can never complete the barrier flags bar[2] and falls through
// instead of hanging the device.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const uint64_t t0 = globaltimer_ns();
      while (*vgen == gen) {
        __nanosleep(32);
        if (globaltimer_ns() - t0 > 5000000000ull) {
          atomicOr(bar + 2, 1u);
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct SegInfo {
  uint32_t c, w0, w1;  // channel, stream range [w0, w1) of channel c
  uint32_t s0;         // offset of the segment in the CTA's smem slice (floats)
};

// Segments of this CTA's slice [f0, f1). Returns the count (<= kMaxSeg guaranteed by
// the host).
__device__ __forceinline__ int slice_segments(const FGeom& g, uint64_t f0, uint64_t f1,
                                              SegInfo* segs) {
  int ns = 0;
  for (uint64_t f = f0; f < f1;) {
    const uint32_t c = (uint32_t)(f / g.L);
    const uint64_t cbase = (uint64_t)c * g.L;
    const uint64_t e = min(f1, cbase + g.L);
    segs[ns] = SegInfo{c, (uint32_t)(f - cbase), (uint32_t)(e - cbase), (uint32_t)(f - f0)};
    ++ns;
    f = e;
  }
  return ns;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tma::smem_u32(dst)), "l"(src)
               : "memory");
}
// The mbarrier's arrival completes when all of this thread's prior cp.async are done.
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tma::smem_u32(bar))
               : "memory");
}

// Every thread copies the float4s i = t, t + kThreadsF, ... of each quarter of the slice
// (cp.async, 16 B each, L2 only) and then arrives on that quarter's mbarrier (count =
// kThreadsF): ~200 KB per SM are requested at once and the reduction of quarter q can
// start as soon as quarter q has landed. NIN streams are packed one after the other
// (stream k at smem + k*cap floats).
template <int NIN>
__device__ __forceinline__ void issue_slice(const FGeom& g, const SegInfo* segs, int ns,
                                           const uint32_t* qb, uint64_t* qbar, uint32_t total,
                                           float* smem, uint32_t cap, const float* in0,
                                           const float* in1) {
  int si = 0;
  for (int q = 0; q < kQuarters; ++q) {
    const uint32_t qe = (q + 1 < kQuarters) ? qb[q + 1] : total;
    for (uint32_t p = qb[q] + 4 * threadIdx.x; p < qe; p += 4 * kThreadsF) {
      while (si + 1 < ns && segs[si + 1].s0 <= p) ++si;
      const SegInfo& sg = segs[si];
      const size_t off = foff(g, sg.c, sg.w0 + (p - sg.s0));
      cp_async16(smem + p, in0 + off);
      if (NIN == 2) cp_async16(smem + cap + p, in1 + off);
    }
    cp_async_arrive(&qbar[q]);
  }
}

// Wait for every quarter overlapping slice range [a, b).
__device__ __forceinline__ void wait_range(const uint32_t* qb, uint64_t* qbar, uint32_t a,
                                           uint32_t b, uint32_t total) {
  for (int q = 0; q < kQuarters; ++q) {
    const uint32_t qs = qb[q], qe = (q + 1 < kQuarters) ? qb[q + 1] : total;
    if (qe > qs && qs < b && qe > a) tma::mbar_wait(&qbar[q], 0);
  }
}

__device__ __forceinline__ void block_sum2_f(double& a, double& b, double* sa, double* sb) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  a = warp_sum(a);
  b = warp_sum(b);
  if (l == 0) { sa[w] = a; sb[w] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = sa[0]; b = sb[0];
#pragma unroll
    for (int i = 1; i < kWarpsF; ++i) { a += sa[i]; b += sb[i]; }
  }
  __syncthreads();
}

// Common prologue: slice, segments, quarter boundaries, barriers, TMA issue.
template <int NIN>
struct SliceCtx {
  uint64_t f0, f1;
  uint32_t total;  // floats in the slice
  int ns;
};

template <int NIN>
__device__ __forceinline__ SliceCtx<NIN> load_slice(const FGeom& g, SegInfo* segs, uint32_t* qb,
                                                    uint64_t* qbar, int* s_ns, float* smem,
                                                    uint32_t cap, const float* in0,
                                                    const float* in1) {
  SliceCtx<NIN> sc;
  sc.f0 = fslice(g, blockIdx.x);
  sc.f1 = fslice(g, blockIdx.x + 1);
  sc.total = (uint32_t)(sc.f1 - sc.f0);
  if (threadIdx.x == 0) {
    *s_ns = slice_segments(g, sc.f0, sc.f1, segs);
    const uint32_t t4 = sc.total >> 2;
    for (int q = 0; q < kQuarters; ++q) qb[q] = (uint32_t)(((uint64_t)t4 * q / kQuarters) * 4);
    for (int q = 0; q < kQuarters; ++q) tma::mbar_init(&qbar[q], kThreadsF);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  sc.ns = *s_ns;
  issue_slice<NIN>(g, segs, sc.ns, qb, qbar, sc.total, smem, cap, in0, in1);
  return sc;
}

template <bool RELU>
__global__ void __launch_bounds__(kThreadsF, 1)
k_fused_fwd(FGeom g, const float* __restrict__ x, float* __restrict__ y, FwdFinal F,
            double2* __restrict__ slots, unsigned* __restrict__ bar) {
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t qbar[kQuarters];
  __shared__ uint32_t qb[kQuarters];
  __shared__ SegInfo segs[kMaxSeg];
  __shared__ double sa[kWarpsF], sb[kWarpsF];
  __shared__ double segK[kMaxSeg], segP[kMaxSeg], segQ[kMaxSeg];
  __shared__ FwdChan segV[kMaxSeg];
  __shared__ int s_ns;
  const uint32_t cap = (uint32_t)(kDataBytes / 4);
  const SliceCtx<1> sc = load_slice<1>(g, segs, qb, qbar, &s_ns, smem, cap, x, x);
  // prefetch every per-channel input the statistics and the finisher need while the
  // slice is in flight
  if (threadIdx.x < sc.ns) {
    const uint32_t c = segs[threadIdx.x].c;
    segK[threadIdx.x] = (double)__ldg(x + (size_t)c * g.HW);
    segV[threadIdx.x] = load_fwd_chan(F, c);
  }
  __syncthreads();

  // 2. per-segment statistics (shift K = first element of the channel on this rank)
  for (int si = 0; si < sc.ns; ++si) {
    const SegInfo sg = segs[si];
    const double K = segK[si];
    const uint32_t len = sg.w1 - sg.w0;
    wait_range(qb, qbar, sg.s0, sg.s0 + len, sc.total);
    const float4* p = reinterpret_cast<const float4*>(smem + sg.s0);
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const uint32_t n4 = len >> 2;
    uint32_t q = threadIdx.x;
    for (; q + kThreadsF < n4; q += 2 * kThreadsF) {
      const float4 u = p[q], v = p[q + kThreadsF];
      const double d0 = (double)u.x - K, d1 = (double)u.y - K, d2 = (double)u.z - K, d3 = (double)u.w - K;
      const double e0 = (double)v.x - K, e1 = (double)v.y - K, e2 = (double)v.z - K, e3 = (double)v.w - K;
      a0 += (d0 + d1) + (d2 + d3);
      a1 += (e0 + e1) + (e2 + e3);
      b0 = __fma_rn(d0, d0, b0); b0 = __fma_rn(d1, d1, b0);
      b0 = __fma_rn(d2, d2, b0); b0 = __fma_rn(d3, d3, b0);
      b1 = __fma_rn(e0, e0, b1); b1 = __fma_rn(e1, e1, b1);
      b1 = __fma_rn(e2, e2, b1); b1 = __fma_rn(e3, e3, b1);
    }
    if (q < n4) {
      const float4 u = p[q];
      const double d0 = (double)u.x - K, d1 = (double)u.y - K, d2 = (double)u.z - K, d3 = (double)u.w - K;
      a0 += (d0 + d1) + (d2 + d3);
      b0 = __fma_rn(d0, d0, b0); b0 = __fma_rn(d1, d1, b0);
      b0 = __fma_rn(d2, d2, b0); b0 = __fma_rn(d3, d3, b0);
    }
    double S1 = a0 + a1, S2 = b0 + b1;
    block_sum2_f(S1, S2, sa, sb);
    if (threadIdx.x == 0) slots[(size_t)blockIdx.x + sg.c] = make_double2(S1, S2);
  }

  // 3. all partials of all CTAs are published
  grid_sync(bar, g.grid);

  // 4. fold (fixed slot order) + finalise + coefficients; first CTA of a channel writes
  if (threadIdx.x < sc.ns) {
    const int si = threadIdx.x;
    const SegInfo sg = segs[si];
    const uint64_t cbase = (uint64_t)sg.c * g.L;
    const uint32_t b0 = fcta_of(g, cbase), b1 = fcta_of(g, cbase + g.L - 4);
    double S1 = 0.0, S2 = 0.0;
    for (uint32_t b = b0; b <= b1; ++b) {
      const double2 t = __ldcg(&slots[(size_t)b + sg.c]);
      S1 += t.x;
      S2 += t.y;
    }
    const double n = g.count;
    const double K = segK[si];
    const double mean = K + S1 / n;
    const double M2 = fmax(S2 - S1 * (S1 / n), 0.0);
    double P, Q;
    finalize_fwd_channel(F, sg.c, n, mean, M2, b0 == blockIdx.x, segV[si], P, Q);
    segP[si] = P;
    segQ[si] = Q;
  }
  __syncthreads();

  // 5. y from shared memory
  for (int si = 0; si < sc.ns; ++si) {
    const SegInfo sg = segs[si];
    const double P = segP[si], Q = segQ[si];
    const float4* p = reinterpret_cast<const float4*>(smem + sg.s0);
    const uint32_t n4 = (sg.w1 - sg.w0) >> 2;
    for (uint32_t q = threadIdx.x; q < n4; q += kThreadsF) {
      const float4 v = p[q];
      float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double t = bn_out(P, Q, o[e]);
        if (RELU) t = t > 0.0 ? t : 0.0;
        o[e] = (float)t;
      }
      *reinterpret_cast<float4*>(y + foff(g, sg.c, sg.w0 + 4 * q)) =
          make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

template <bool RELU>
__global__ void __launch_bounds__(kThreadsF, 1)
k_fused_bwd(FGeom g, const float* __restrict__ dy, const float* __restrict__ x,
            float* __restrict__ dx, BwdFinal F, double2* __restrict__ slots,
            unsigned* __restrict__ bar) {
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t qbar[kQuarters];
  __shared__ uint32_t qb[kQuarters];
  __shared__ SegInfo segs[kMaxSeg];
  __shared__ double sa[kWarpsF], sb[kWarpsF];
  __shared__ double segA[kMaxSeg], segB[kMaxSeg], segC[kMaxSeg], segP[kMaxSeg], segQ[kMaxSeg];
  __shared__ BwdChan segV[kMaxSeg];
  __shared__ int s_ns;
  const uint32_t cap = (uint32_t)(kDataBytes / 8);
  const SliceCtx<2> sc = load_slice<2>(g, segs, qb, qbar, &s_ns, smem, cap, dy, x);
  if (threadIdx.x < sc.ns) {
    const uint32_t c = segs[threadIdx.x].c;
    const BwdChan v = load_bwd_chan(F, c);
    segV[threadIdx.x] = v;
    double P = 0.0, Q = 0.0;
    if (RELU) affine_coeffs(v.mean, v.inv_std, (double)v.gamma, (double)v.beta, P, Q);
    segP[threadIdx.x] = P;
    segQ[threadIdx.x] = Q;
  }
  __syncthreads();
  const uint32_t C = g.C;
  const float* gs = smem;        // dy
  const float* xs = smem + cap;  // x

  for (int si = 0; si < sc.ns; ++si) {
    const SegInfo sg = segs[si];
    const double mean = segV[si].mean;
    const double P = segP[si], Q = segQ[si];
    const uint32_t len = sg.w1 - sg.w0;
    wait_range(qb, qbar, sg.s0, sg.s0 + len, sc.total);
    const float4* pg = reinterpret_cast<const float4*>(gs + sg.s0);
    const float4* px = reinterpret_cast<const float4*>(xs + sg.s0);
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const uint32_t n4 = len >> 2;
    for (uint32_t q = threadIdx.x; q < n4; q += kThreadsF) {
      const float4 gv = pg[q], xv = px[q];
      const float gi[4] = {gv.x, gv.y, gv.z, gv.w};
      const float xi[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double gk = (double)gi[e];
        if (RELU && !(bn_out(P, Q, xi[e]) > 0.0)) gk = 0.0;
        if (e & 1) {
          a1 += gk;
          b1 = __fma_rn(gk, (double)xi[e] - mean, b1);
        } else {
          a0 += gk;
          b0 = __fma_rn(gk, (double)xi[e] - mean, b0);
        }
      }
    }
    double S1 = a0 + a1, S2 = b0 + b1;
    block_sum2_f(S1, S2, sa, sb);
    if (threadIdx.x == 0) slots[(size_t)blockIdx.x + sg.c] = make_double2(S1, S2);
  }

  grid_sync(bar, g.grid);

  if (threadIdx.x < sc.ns) {
    const int si = threadIdx.x;
    const SegInfo sg = segs[si];
    const uint32_t c = sg.c;
    const uint64_t cbase = (uint64_t)c * g.L;
    const uint32_t b0 = fcta_of(g, cbase), b1 = fcta_of(g, cbase + g.L - 4);
    double sdy = 0.0, sdyx = 0.0;
    for (uint32_t b = b0; b <= b1; ++b) {
      const double2 t = __ldcg(&slots[(size_t)b + c]);
      sdy += t.x;
      sdyx += t.y;
    }
    const DxCoef k = finalize_bwd_channel(F, c, sdy, sdyx, b0 == blockIdx.x, segV[si]);
    segA[si] = k.A;
    segB[si] = k.B;
    segC[si] = k.Cc;
    segP[si] = k.P;
    segQ[si] = k.Q;
  }
  __syncthreads();

  for (int si = 0; si < sc.ns; ++si) {
    const SegInfo sg = segs[si];
    const double Ak = segA[si], Bk = segB[si], Ck = segC[si], P = segP[si], Q = segQ[si];
    const float4* pg = reinterpret_cast<const float4*>(gs + sg.s0);
    const float4* px = reinterpret_cast<const float4*>(xs + sg.s0);
    const uint32_t n4 = (sg.w1 - sg.w0) >> 2;
    for (uint32_t q = threadIdx.x; q < n4; q += kThreadsF) {
      const float4 gv = pg[q], xv = px[q];
      const float gi[4] = {gv.x, gv.y, gv.z, gv.w};
      const float xi[4] = {xv.x, xv.y, xv.z, xv.w};
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double gk = (double)gi[e];
        if (RELU && !(bn_out(P, Q, xi[e]) > 0.0)) gk = 0.0;
        o[e] = (float)__fma_rn(Ak, gk, __fma_rn(Bk, (double)xi[e], Ck));
      }
      *reinterpret_cast<float4*>(dx + foff(g, sg.c, sg.w0 + 4 * q)) =
          make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

}  // namespace fused
