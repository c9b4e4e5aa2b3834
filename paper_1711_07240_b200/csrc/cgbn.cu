// cgbn.cu — sm_100a kernels and the C ABI (include/cgbn.h) of the CGBN hot path.
//
// The path is HBM-bandwidth bound (no contraction; tensor cores do not apply), so every
// kernel is a streaming pass over the activation with 128-bit coalesced loads, several
// independent loads in flight per thread (predicated unrolled rounds: loads first,
// then arithmetic), and a deterministic reduction tree.
//
// A channel's "stream" is the concatenation of its N planes (NCHW: N runs of HW floats,
// C*HW apart), Lv vector units long. Two work decompositions, chosen per shape:
//
//  * flat (Lv > kTeamMaxLv): persistent grid of at most (#SMs x resident CTAs/SM). The
//    channel-major stream of T = C*Lv units is split into equal contiguous CTA slices;
//    a slice may cover the tail of one channel, whole channels and the head of another
//    ("segments"). A channel covered by CTAs b0..b1 gets one partial per CTA in
//    workspace slot (b + c); the last CTA to arrive (arrival ticket) folds slots
//    b0+c..b1+c in index order.
//  * team (Lv <= kTeamMaxLv, small spatial extent): a power-of-two team of tpc threads
//    (32..256) owns one whole channel; a CTA holds 256/tpc teams and loops over channel
//    tiles. No cross-CTA combine at all.
//
// All reductions accumulate in fp64 per element and fold in a fixed order, so results
// are bitwise run-to-run reproducible without float atomics.
//
// Reference being replaced (file:line under /root/reference/pkg/src/bigbatch):
//   channel_sum / sequential_sum_rows      tensor.py:121-153   -> reduce kernels, StatsOp
//   _train_forward post-reduction + affine batchnorm.py:121-143 -> affine kernels, kTrain
//   bn_update_running                      batchnorm.py:239-252 (fused into kTrain prologue)
//   _backward_core sums                    batchnorm.py:198-201 -> reduce kernels, BwdOp
//   _backward_core dx                      batchnorm.py:203-209 -> dx kernels
//   allreduce_sum root fold                collectives.py:293-295 (ascending-rank fold,
//                                          done by every consumer kernel's prologue)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "cgbn.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kTeamMaxLv = 2048;   // channels up to this many units use team kernels
constexpr int64_t kMinElemsPerCta = 2048;
constexpr int kMaxCtasPerSm = 8;        // 2048 threads / 256
constexpr size_t kTicketBytes = 65536 * sizeof(unsigned);  // fixed: independent of C

// ----------------------------------------------------------------------------------
// Errors

thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
  return CGBN_OK;
}

// ----------------------------------------------------------------------------------
// Geometry

// Unsigned division by a runtime-constant divisor for n < 2^31 (Granlund-Montgomery):
// q = (umulhi(n, m) + n) >> l with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1.
struct FastDiv {
  uint32_t m, l;
  void init(uint32_t d) {
    uint32_t ll = 0;
    while ((1ull << ll) < d) ++ll;
    l = ll;
    m = (uint32_t)(((1ull << 32) * ((1ull << ll) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
};

// Element offset of vector unit j of channel c: (c*HWv + j + (j / HWv) * gap) * VEC with
// gap = (C-1)*HWv. NCHW: HWv = HW/VEC. NHWC and 2-D (N, C): HWv = 1, VEC = 1.
struct Geom {
  uint32_t C;
  uint32_t Lv;        // vector units per channel stream (N*HW/VEC)
  uint32_t HWv;       // vector units per plane
  uint32_t grid;      // CTAs of this launch
  uint32_t tpc_log2;  // team kernels: log2(threads per channel)
  uint64_t T;         // C * Lv
  uint64_t gap;       // (C-1)*HWv
  FastDiv dhw;
  double count;       // elements per channel on this rank (N*HW)
};

__device__ __forceinline__ size_t voff(const Geom& g, uint32_t c, uint32_t j) {
  return (size_t)c * g.HWv + j + (size_t)g.dhw.div(j) * g.gap;
}

// flat: CTA b owns stream units [cta_begin(b), cta_begin(b+1)).
__device__ __forceinline__ uint64_t cta_begin(const Geom& g, uint32_t b) {
  return (uint64_t)b * g.T / g.grid;
}
// The CTA whose slice contains unit u: the largest b with cta_begin(b) <= u.
__device__ __forceinline__ uint32_t cta_of(const Geom& g, uint64_t u) {
  return (uint32_t)(((u + 1) * (uint64_t)g.grid - 1) / g.T);
}

struct Seg {
  uint32_t c, j0, j1;
};

template <class F>
__device__ __forceinline__ void for_each_segment(const Geom& g, F&& f) {
  const uint64_t u_end = cta_begin(g, blockIdx.x + 1);
  for (uint64_t u = cta_begin(g, blockIdx.x); u < u_end;) {
    const uint32_t c = (uint32_t)(u / g.Lv);
    const uint64_t cbase = (uint64_t)c * g.Lv;
    const uint64_t s_end = min(u_end, cbase + g.Lv);
    f(Seg{c, (uint32_t)(u - cbase), (uint32_t)(s_end - cbase)});
    u = s_end;
  }
}

struct Parts {
  const double* p[CGBN_MAX_GROUP];
  int G;
};

// ----------------------------------------------------------------------------------
// Vector load / store

template <int VEC>
__device__ __forceinline__ void ldv(const float* __restrict__ p, float (&v)[VEC]) {
  if constexpr (VEC == 4) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (VEC == 2) {
    float2 t = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = __ldg(p);
  }
}

template <int VEC>
__device__ __forceinline__ void stv(float* __restrict__ p, const float (&v)[VEC]) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

// Loads in flight per thread per round: ~128 B for one input stream, ~128 B total for
// two (NIN = number of input streams).
template <int VEC, int NIN = 1>
constexpr int unroll_for() { return (NIN == 1 || VEC == 1) ? 8 : 4; }

// Visit units j = start, start+stride, ... < end of channel c in rounds of U: the U
// (predicated) loads of a round are issued before any of them is used. The body gets
// the unit index and recomputes its offset (cheaper than holding U 64-bit offsets).
template <int U, class Op, class Body>
__device__ __forceinline__ void strided_rounds(const Geom& g, uint32_t c, uint32_t start,
                                               uint32_t end, uint32_t stride, const Op& op,
                                               Body&& body) {
  for (uint32_t i = start; i < end; i += U * stride) {
    typename Op::Regs r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j < end) op.load(voff(g, c, j), r[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j < end) body(u, j, r[u]);
    }
  }
}

// ----------------------------------------------------------------------------------
// Shared per-channel arithmetic (fp64). The same inline functions are used by the
// forward and the backward so that the ReLU mask recomputed in the backward is
// bitwise the forward's.

// Chan et al. pairwise merge of (n, mean, M2) partials, folded in ascending rank order.
__device__ __forceinline__ void merge_fwd_partials(const Parts& P, uint32_t c, uint32_t C,
                                                   double& n, double& mean, double& M2) {
  n = P.p[0][2 * C];
  mean = P.p[0][c];
  M2 = P.p[0][C + c];
  for (int r = 1; r < P.G; ++r) {
    const double nb = P.p[r][2 * C], mb = P.p[r][c], Mb = P.p[r][C + c];
    const double nn = n + nb;
    const double delta = mb - mean;
    mean = mean + delta * (nb / nn);
    M2 = M2 + Mb + delta * delta * (n * nb / nn);
    n = nn;
  }
}

// y = P*x + Q with P = gamma*inv_std, Q = beta - mean*P.
__device__ __forceinline__ void affine_coeffs(double mean, double inv_std, double gamma,
                                              double beta, double& P, double& Q) {
  P = gamma * inv_std;
  Q = __fma_rn(-mean, P, beta);
}

__device__ __forceinline__ double bn_out(double P, double Q, float x) {
  return __fma_rn(P, (double)x, Q);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------------------------
// Reduction ops: per-channel sums of two quantities, fp64 per element.

// Forward statistics: sums of d = x - K (K = first element of the channel on this rank,
// the same for every CTA of the channel; d is exact in fp64) -> (mean, M2, count).
template <int VEC>
struct StatsOp {
  static constexpr int kVec = VEC;
  static constexpr int kIn = 1;
  const float* __restrict__ x;
  double K;
  bool shift;
  int mode;                   // 0: forward partial [mean | M2 | count]; 1: raw [sum | sum_sq]
  double* __restrict__ out2;  // mode 1: sum_sq destination (may be null)
  struct Regs { float v[VEC]; };
  __device__ __forceinline__ void init(const Geom& g, uint32_t c) {
    K = shift ? (double)__ldg(x + (size_t)c * g.HWv * VEC) : 0.0;
  }
  __device__ __forceinline__ void load(size_t off, Regs& r) const { ldv<VEC>(x + off * VEC, r.v); }
  __device__ __forceinline__ void acc(const Regs& r, double& a, double& b) const {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const double d = (double)r.v[k] - K;
      a += d;
      b = __fma_rn(d, d, b);
    }
  }
  __device__ __forceinline__ void finish(const Geom& g, uint32_t c, double S1, double S2,
                                         double* __restrict__ out) const {
    const double n = g.count;
    if (mode == 0) {
      const double mean = K + S1 / n;
      const double M2 = fmax(S2 - S1 * (S1 / n), 0.0);
      out[c] = mean;
      out[g.C + c] = M2;
      if (c == 0) out[2 * g.C] = n;
    } else {
      out[c] = S1;
      if (out2) out2[c] = S2;
    }
  }
};

// Backward: g = dy (ReLU-masked when the forward fused a ReLU); fp64 sums of g and
// g*(x - mean).
template <int VEC, bool RELU>
struct BwdOp {
  static constexpr int kVec = VEC;
  static constexpr int kIn = 2;
  const float* __restrict__ dy;
  const float* __restrict__ x;
  const double* __restrict__ saved;
  const float* __restrict__ gamma;
  const float* __restrict__ beta;
  double mean, P, Q;
  struct Regs { float g[VEC]; float x[VEC]; };
  __device__ __forceinline__ void init(const Geom& g, uint32_t c) {
    mean = saved[c];
    const double inv_std = saved[2 * g.C + c];
    if (RELU) affine_coeffs(mean, inv_std, (double)gamma[c], (double)beta[c], P, Q);
  }
  __device__ __forceinline__ void load(size_t off, Regs& r) const {
    ldv<VEC>(dy + off * VEC, r.g);
    ldv<VEC>(x + off * VEC, r.x);
  }
  __device__ __forceinline__ void acc(const Regs& r, double& a, double& b) const {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      double gk = (double)r.g[k];
      if (RELU && !(bn_out(P, Q, r.x[k]) > 0.0)) gk = 0.0;
      a += gk;
      b = __fma_rn(gk, (double)r.x[k] - mean, b);
    }
  }
  __device__ __forceinline__ void finish(const Geom& g, uint32_t c, double S1, double S2,
                                         double* __restrict__ out) const {
    out[c] = S1;
    out[g.C + c] = S2;
  }
};

// Accumulate the strided range in fp64 (two interleaved accumulator pairs).
template <class Op>
__device__ __forceinline__ void reduce_range(const Geom& g, uint32_t c, uint32_t start,
                                             uint32_t end, uint32_t stride, const Op& op,
                                             double& S1, double& S2) {
  constexpr int U = unroll_for<Op::kVec, Op::kIn>();
  double a[2] = {0.0, 0.0}, b[2] = {0.0, 0.0};
  strided_rounds<U>(g, c, start, end, stride, op,
                    [&](int u, uint32_t, const typename Op::Regs& r) {
                      op.acc(r, a[u & 1], b[u & 1]);
                    });
  S1 = a[0] + a[1];
  S2 = b[0] + b[1];
}

// flat reduction (see header): one CTA partial per segment (warp shuffle, then thread 0
// folds the kWarps values in order), cross-CTA fold by the last CTA to arrive.
template <class Op>
__global__ void __launch_bounds__(kThreads, 3)
k_reduce_flat(Geom g, Op op, double* __restrict__ out, double2* __restrict__ ws,
              unsigned* __restrict__ tickets) {
  __shared__ double sa[kWarps], sb[kWarps];
  __shared__ int s_last;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for_each_segment(g, [&](const Seg& sg) {
    const uint32_t c = sg.c;
    op.init(g, c);
    double S1, S2;
    reduce_range(g, c, sg.j0 + threadIdx.x, sg.j1, kThreads, op, S1, S2);
    S1 = warp_sum(S1);
    S2 = warp_sum(S2);
    if (l == 0) { sa[w] = S1; sb[w] = S2; }
    __syncthreads();
    const uint64_t cbase = (uint64_t)c * g.Lv;
    const uint32_t b0 = cta_of(g, cbase), b1 = cta_of(g, cbase + g.Lv - 1);
    if (threadIdx.x == 0) {
      S1 = sa[0]; S2 = sb[0];
#pragma unroll
      for (int i = 1; i < kWarps; ++i) { S1 += sa[i]; S2 += sb[i]; }
      int last = 0;
      if (b0 == b1) {
        op.finish(g, c, S1, S2, out);
      } else {
        ws[(size_t)blockIdx.x + c] = make_double2(S1, S2);
        __threadfence();
        last = atomicAdd(&tickets[c], 1u) == b1 - b0;
      }
      s_last = last;
    }
    __syncthreads();
    if (s_last && w == 0) {
      __threadfence();
      const uint32_t cnt = b1 - b0 + 1;
      double x1 = 0.0, x2 = 0.0;
      for (uint32_t k = l; k < cnt; k += 32) {
        const double2 t = __ldcg(&ws[(size_t)b0 + c + k]);
        x1 += t.x;
        x2 += t.y;
      }
      x1 = warp_sum(x1);
      x2 = warp_sum(x2);
      if (l == 0) {
        op.finish(g, c, x1, x2, out);
        tickets[c] = 0u;  // leave the workspace reusable
      }
    }
    __syncthreads();  // sa/sb/s_last are reused by the next segment
  });
}

// team reduction: 2^tpc_log2 threads per channel, 256/tpc channels per tile.
template <class Op>
__global__ void __launch_bounds__(kThreads, 3)
k_reduce_team(Geom g, Op op, double* __restrict__ out) {
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
    if (c < g.C) {
      op.init(g, c);
      reduce_range(g, c, q, g.Lv, tpc, op, S1, S2);
    }
    S1 = warp_sum(S1);
    S2 = warp_sum(S2);
    if (tpc == 32) {
      if (l == 0 && c < g.C) op.finish(g, c, S1, S2, out);
    } else {
      if (l == 0) { sa[w] = S1; sb[w] = S2; }
      __syncthreads();
      if (q == 0 && c < g.C) {
        const int wpt = (int)(tpc >> 5);
        for (int i = 1; i < wpt; ++i) { S1 += sa[w + i]; S2 += sb[w + i]; }
        op.finish(g, c, S1, S2, out);
      }
      __syncthreads();
    }
  }
}

// ----------------------------------------------------------------------------------
// Elementwise per-channel affine y = P[c]*x + Q[c] (fp64 coefficients and arithmetic,
// one rounding to fp32 at the end), with the per-channel coefficient prologue chosen
// by MODE.

enum AffineMode { kTrain = 0, kEval = 1, kAffine = 2, kXhat = 3 };

struct AffineArgs {
  const float* x;
  float* y;
  Parts parts;
  const float* gamma;
  const float* beta;
  const float* rmean_in;
  const float* rvar_in;
  float* rmean;
  float* rvar;
  double* saved;
  const double* scale;
  const double* shift;
  double eps, momentum;
  unsigned* status;
};

// `first`: the caller is the unique writer of channel c's saved statistics and
// running-stat update.
template <int MODE>
__device__ __forceinline__ void affine_prologue(const Geom& g, const AffineArgs& A, uint32_t c,
                                                bool first, double& P, double& Q) {
  if constexpr (MODE == kTrain) {
    double n, mean, M2;
    merge_fwd_partials(A.parts, c, g.C, n, mean, M2);
    const double var = fmax(M2 / n, 0.0);
    const double inv_std = 1.0 / sqrt(var + A.eps);
    affine_coeffs(mean, inv_std, (double)A.gamma[c], (double)A.beta[c], P, Q);
    if (first) {
      const uint32_t C = g.C;
      A.saved[c] = mean;
      A.saved[C + c] = var;
      A.saved[2 * C + c] = inv_std;
      if (c == 0) A.saved[3 * C] = n;
      unsigned bad = 0;
      if (!isfinite(mean) || !isfinite(var)) bad |= CGBN_STATUS_NONFINITE;
      if (n < 2.0) bad |= CGBN_STATUS_SMALL_COUNT;
      if (bad) {
        if (A.status) atomicOr(A.status, bad);
      } else if (A.rmean) {
        // bn_update_running (batchnorm.py:239-252): unbiased m/(m-1) on the variance.
        const double rho = A.momentum;
        const double unbiased = var * (n / (n - 1.0));
        A.rmean[c] = (float)((1.0 - rho) * (double)A.rmean[c] + rho * mean);
        A.rvar[c] = (float)((1.0 - rho) * (double)A.rvar[c] + rho * unbiased);
      }
    }
  } else if constexpr (MODE == kEval) {
    const double inv_std = 1.0 / sqrt((double)A.rvar_in[c] + A.eps);
    affine_coeffs((double)A.rmean_in[c], inv_std, (double)A.gamma[c], (double)A.beta[c], P, Q);
  } else if constexpr (MODE == kAffine) {
    P = A.scale[c];
    Q = A.shift[c];
  } else {  // kXhat
    affine_coeffs(A.saved[c], A.saved[2 * g.C + c], 1.0, 0.0, P, Q);
  }
}

template <int VEC>
struct LoadX {
  static constexpr int kVec = VEC;
  const float* __restrict__ x;
  struct Regs { float v[VEC]; };
  __device__ __forceinline__ void load(size_t off, Regs& r) const { ldv<VEC>(x + off * VEC, r.v); }
};

template <int VEC, bool RELU>
__device__ __forceinline__ void affine_range(const Geom& g, const AffineArgs& A, uint32_t c,
                                             uint32_t start, uint32_t end, uint32_t stride,
                                             double P, double Q) {
  constexpr int U = unroll_for<VEC, 2>();  // keeps data for the store: budget as 2 streams
  LoadX<VEC> op{A.x};
  float* __restrict__ y = A.y;
  strided_rounds<U>(g, c, start, end, stride, op,
                    [&](int, uint32_t j, const typename LoadX<VEC>::Regs& r) {
                      float v[VEC];
#pragma unroll
                      for (int k = 0; k < VEC; ++k) {
                        double t = bn_out(P, Q, r.v[k]);
                        if (RELU) t = t > 0.0 ? t : 0.0;
                        v[k] = (float)t;
                      }
                      stv<VEC>(y + voff(g, c, j) * VEC, v);
                    });
}

template <int VEC, int MODE, bool RELU>
__global__ void __launch_bounds__(kThreads, 3) k_affine_flat(Geom g, AffineArgs A) {
  __shared__ double sP, sQ;
  for_each_segment(g, [&](const Seg& sg) {
    if (threadIdx.x == 0) {
      double P, Q;
      affine_prologue<MODE>(g, A, sg.c, sg.j0 == 0, P, Q);
      sP = P;
      sQ = Q;
    }
    __syncthreads();
    affine_range<VEC, RELU>(g, A, sg.c, sg.j0 + threadIdx.x, sg.j1, kThreads, sP, sQ);
    __syncthreads();  // sP/sQ are rewritten by the next segment's prologue
  });
}

template <int VEC, int MODE, bool RELU>
__global__ void __launch_bounds__(kThreads, 3) k_affine_team(Geom g, AffineArgs A) {
  const uint32_t tpc = 1u << g.tpc_log2;
  const uint32_t cpt = kThreads >> g.tpc_log2;
  const uint32_t q = threadIdx.x & (tpc - 1);
  const uint32_t team = threadIdx.x >> g.tpc_log2;
  const uint32_t l = threadIdx.x & 31;
  const uint32_t tiles = (g.C + cpt - 1) / cpt;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t c = tile * cpt + team;
    if (c >= g.C) continue;  // whole warps (tpc >= 32) skip together
    double P = 0.0, Q = 0.0;
    if (l == 0) affine_prologue<MODE>(g, A, c, q == 0, P, Q);  // per warp; writer: q == 0
    P = __shfl_sync(0xffffffffu, P, 0);
    Q = __shfl_sync(0xffffffffu, Q, 0);
    affine_range<VEC, RELU>(g, A, c, q, g.Lv, tpc, P, Q);
  }
}

// ----------------------------------------------------------------------------------
// Backward dx: prologue folds the G backward partials (ascending rank order), then
// dx = A*g + B*x + Cc with A = gamma/sqrt(var+eps), B = -A*inv_std*dgamma/m,
// Cc = -A*dbeta/m - B*mean  (== gamma/sqrt(var+eps)*(g - dbeta/m - x_hat*dgamma/m)).

struct DxArgs {
  const float* dy;
  const float* x;
  float* dx;
  Parts parts;
  const double* saved;
  const float* gamma;
  const float* beta;
  float* dgamma;
  float* dbeta;
  unsigned* status;
  double eps;
};

struct DxCoef {
  double A, B, Cc, P, Q;
};

template <bool RELU>
__device__ __forceinline__ DxCoef dx_prologue(const Geom& g, const DxArgs& D, uint32_t c,
                                              bool first) {
  const uint32_t C = g.C;
  double sdy = D.parts.p[0][c], sdyx = D.parts.p[0][C + c];
  for (int r = 1; r < D.parts.G; ++r) {
    sdy += D.parts.p[r][c];
    sdyx += D.parts.p[r][C + c];
  }
  const double mean = D.saved[c];
  const double inv_std = D.saved[2 * C + c];
  const double m = D.saved[3 * C];
  const double dbeta = sdy;
  const double dgamma = sdyx * inv_std;
  const double gam = (double)D.gamma[c];
  DxCoef k;
  // batchnorm.py:205: gamma / sqrt(var + eps) with the backward state's eps (x_hat
  // itself keeps the forward's inv_std, as the reference's cached x_hat does).
  k.A = gam / sqrt(D.saved[C + c] + D.eps);
  k.B = -k.A * inv_std * (dgamma / m);
  k.Cc = -k.A * (dbeta / m) - k.B * mean;
  k.P = k.Q = 0.0;
  if (RELU) affine_coeffs(mean, inv_std, gam, (double)D.beta[c], k.P, k.Q);
  if (first) {
    if (D.dgamma) D.dgamma[c] = (float)dgamma;
    if (D.dbeta) D.dbeta[c] = (float)dbeta;
    if (D.status && (!isfinite(dbeta) || !isfinite(dgamma)))
      atomicOr(D.status, CGBN_STATUS_NONFINITE);
  }
  return k;
}

template <int VEC>
struct LoadGX {
  static constexpr int kVec = VEC;
  const float* __restrict__ dy;
  const float* __restrict__ x;
  struct Regs { float g[VEC]; float x[VEC]; };
  __device__ __forceinline__ void load(size_t off, Regs& r) const {
    ldv<VEC>(dy + off * VEC, r.g);
    ldv<VEC>(x + off * VEC, r.x);
  }
};

template <int VEC, bool RELU>
__device__ __forceinline__ void dx_range(const Geom& g, const DxArgs& D, uint32_t c,
                                         uint32_t start, uint32_t end, uint32_t stride,
                                         const DxCoef& k) {
  constexpr int U = unroll_for<VEC, 2>();
  LoadGX<VEC> op{D.dy, D.x};
  float* __restrict__ dx = D.dx;
  strided_rounds<U>(g, c, start, end, stride, op,
                    [&](int, uint32_t j, const typename LoadGX<VEC>::Regs& r) {
                      float v[VEC];
#pragma unroll
                      for (int e = 0; e < VEC; ++e) {
                        double gk = (double)r.g[e];
                        if (RELU && !(bn_out(k.P, k.Q, r.x[e]) > 0.0)) gk = 0.0;
                        v[e] = (float)__fma_rn(k.A, gk, __fma_rn(k.B, (double)r.x[e], k.Cc));
                      }
                      stv<VEC>(dx + voff(g, c, j) * VEC, v);
                    });
}

template <int VEC, bool RELU>
__global__ void __launch_bounds__(kThreads, 3) k_dx_flat(Geom g, DxArgs D) {
  __shared__ DxCoef sk;
  for_each_segment(g, [&](const Seg& sg) {
    if (threadIdx.x == 0) sk = dx_prologue<RELU>(g, D, sg.c, sg.j0 == 0);
    __syncthreads();
    const DxCoef k = sk;
    dx_range<VEC, RELU>(g, D, sg.c, sg.j0 + threadIdx.x, sg.j1, kThreads, k);
    __syncthreads();  // sk is rewritten by the next segment's prologue
  });
}

template <int VEC, bool RELU>
__global__ void __launch_bounds__(kThreads, 3) k_dx_team(Geom g, DxArgs D) {
  const uint32_t tpc = 1u << g.tpc_log2;
  const uint32_t cpt = kThreads >> g.tpc_log2;
  const uint32_t q = threadIdx.x & (tpc - 1);
  const uint32_t team = threadIdx.x >> g.tpc_log2;
  const uint32_t l = threadIdx.x & 31;
  const uint32_t tiles = (g.C + cpt - 1) / cpt;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t c = tile * cpt + team;
    if (c >= g.C) continue;
    DxCoef k{0.0, 0.0, 0.0, 0.0, 0.0};
    if (l == 0) k = dx_prologue<RELU>(g, D, c, q == 0);
    k.A = __shfl_sync(0xffffffffu, k.A, 0);
    k.B = __shfl_sync(0xffffffffu, k.B, 0);
    k.Cc = __shfl_sync(0xffffffffu, k.Cc, 0);
    if (RELU) {
      k.P = __shfl_sync(0xffffffffu, k.P, 0);
      k.Q = __shfl_sync(0xffffffffu, k.Q, 0);
    }
    dx_range<VEC, RELU>(g, D, c, q, g.Lv, tpc, k);
  }
}

// ----------------------------------------------------------------------------------
// Ascending-rank fold of G vectors (the reference's allreduce_sum arithmetic).

template <typename T>
__global__ void k_fold_sum(Parts P, int64_t n, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = reinterpret_cast<const T*>(P.p[0])[i];
    for (int r = 1; r < P.G; ++r) acc = acc + reinterpret_cast<const T*>(P.p[r])[i];
    out[i] = acc;
  }
}

}  // namespace

#include "cgbn_tma.cuh"

namespace {

// ----------------------------------------------------------------------------------
// Host-side planning

int num_sms_cached() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Workspace: fixed-size ticket array (max C), then (C + max grid) double2 slots.
size_t ws_bytes_for(int64_t C, int sms) {
  return kTicketBytes + ((size_t)C + (size_t)sms * kMaxCtasPerSm) * sizeof(double2);
}

// Per-(kernel, device) caches. Keyed by the kernel's address: kernels of one signature
// share a function-pointer type, so a per-template static would alias them.
std::mutex g_cache_mu;
std::map<std::pair<const void*, int>, int> g_occ_cache;
std::map<std::pair<const void*, int>, bool> g_smem_done;

// Resident CTAs of `kernel` on the whole device.
template <class K>
int64_t resident_ctas(K kernel) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_occ_cache.find(key);
    if (it != g_occ_cache.end()) occ = it->second;
  }
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0) != cudaSuccess ||
        occ <= 0)
      occ = 1;
    if (occ > kMaxCtasPerSm) occ = kMaxCtasPerSm;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_occ_cache[key] = occ;
  }
  return (int64_t)num_sms_cached() * occ;
}

struct Plan {
  int vec;
  bool team;
  bool tma;  // NCHW, HW % 4 == 0, 16-byte aligned: TMA bulk-copy kernels
  Geom g;
  tma::TGeom tg;
  int64_t elems;
};

// CGBN_PATH=tma selects the TMA streaming kernels for eligible shapes (A/B measurement);
// the register kernels are the default (measured faster on every ResNet-50 shape).
int path_override() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CGBN_PATH");
    v = (e && !strcmp(e, "tma")) ? 1 : (e && !strcmp(e, "reg")) ? 2 : 0;
  }
  return v;
}

int validate_shape(int64_t N, int64_t C, int64_t HW, int layout) {
  if (N < 1 || C < 1 || HW < 1)
    return set_error(CGBN_ERR_INVALID, "extents must be positive, got N=%lld C=%lld HW=%lld",
                     (long long)N, (long long)C, (long long)HW);
  if (layout != CGBN_LAYOUT_NCHW && layout != CGBN_LAYOUT_NHWC)
    return set_error(CGBN_ERR_INVALID, "unknown layout %d", layout);
  if (C > 65535) return set_error(CGBN_ERR_INVALID, "C=%lld exceeds 65535", (long long)C);
  if (N * HW >= (1ll << 31))
    return set_error(CGBN_ERR_INVALID, "per-channel count N*HW=%lld must be < 2^31",
                     (long long)(N * HW));
  return CGBN_OK;
}

// `ptrs` are every activation pointer the kernel touches; the vector width is the
// widest one that divides the plane length and the alignment of all of them.
int make_plan(int64_t N, int64_t C, int64_t HW, int layout, const void* const* ptrs, int nptr,
              Plan* out) {
  int rc = validate_shape(N, C, HW, layout);
  if (rc) return rc;
  int64_t planeN = N, planeHW = HW;
  if (layout == CGBN_LAYOUT_NHWC) { planeN = N * HW; planeHW = 1; }
  uintptr_t align = 0;
  for (int k = 0; k < nptr; ++k) align |= (uintptr_t)ptrs[k];
  int vec = 1;
  if (planeHW % 4 == 0 && (align % 16) == 0) vec = 4;
  else if (planeHW % 2 == 0 && (align % 8) == 0) vec = 2;
  Geom g;
  g.C = (uint32_t)C;
  g.HWv = (uint32_t)(planeHW / vec);
  g.Lv = (uint32_t)(planeN * g.HWv);
  g.gap = (uint64_t)(C - 1) * g.HWv;
  g.dhw.init(g.HWv);
  g.count = (double)(N * HW);
  g.T = (uint64_t)C * g.Lv;
  g.grid = 1;
  // team size: smallest power of two in [32, 256] giving <= ~8 units per thread
  uint32_t tl = 5;
  while (tl < 8 && (((uint64_t)g.Lv + (1ull << tl) - 1) >> tl) > 8) ++tl;
  g.tpc_log2 = tl;
  out->vec = vec;
  out->team = g.Lv <= kTeamMaxLv;
  out->g = g;
  out->elems = N * C * HW;
  out->tma = layout == CGBN_LAYOUT_NCHW && HW % 4 == 0 && (align % 16) == 0 &&
             path_override() == 1;
  tma::TGeom& tg = out->tg;
  tg.C = (uint32_t)C;
  tg.HW = (uint32_t)HW;
  tg.L = (uint32_t)(N * HW);
  tg.T4 = (uint64_t)C * tg.L / 4;
  tg.dhw.init((uint32_t)HW);
  tg.count = (double)(N * HW);
  int64_t tgrid = ceil_div((int64_t)tg.T4, 1024);
  if (tgrid > num_sms_cached()) tgrid = num_sms_cached();
  tg.grid = (uint32_t)(tgrid < 1 ? 1 : tgrid);
  return CGBN_OK;
}

int fill_parts(Parts* P, const double* const* partials, int G) {
  if (G < 1 || G > CGBN_MAX_GROUP)
    return set_error(CGBN_ERR_INVALID, "group size %d outside [1, %d]", G, CGBN_MAX_GROUP);
  if (!partials) return set_error(CGBN_ERR_INVALID, "partials array is NULL");
  for (int r = 0; r < G; ++r) {
    if (!partials[r]) return set_error(CGBN_ERR_INVALID, "partials[%d] is NULL", r);
    P->p[r] = partials[r];
  }
  for (int r = G; r < CGBN_MAX_GROUP; ++r) P->p[r] = nullptr;
  P->G = G;
  return CGBN_OK;
}

// flat grid: resident CTAs, but no more than one CTA per kMinElemsPerCta elements.
template <class K>
unsigned flat_grid(K kernel, const Plan& pl) {
  int64_t grid = resident_ctas(kernel);
  const int64_t want = ceil_div(pl.elems, kMinElemsPerCta);
  if (want < grid) grid = want;
  return (unsigned)(grid < 1 ? 1 : grid);
}

// team grid: one CTA per channel tile, capped at the resident CTAs.
template <class K>
unsigned team_grid(K kernel, const Plan& pl) {
  const int64_t cpt = kThreads >> pl.g.tpc_log2;
  int64_t grid = ceil_div(pl.g.C, cpt);
  const int64_t res = resident_ctas(kernel);
  if (grid > res) grid = res;
  return (unsigned)(grid < 1 ? 1 : grid);
}

// One-time opt-in to the large dynamic shared memory of a TMA kernel (per device).
template <class K>
void tma_prepare(K kernel, size_t smem_bytes = tma::kSmemBytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_smem_done.count(key)) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  g_smem_done[key] = true;
}

int ws_parts(const Plan& pl, void* ws, size_t ws_bytes, unsigned** tickets, double2** slots) {
  const size_t need = ws_bytes_for(pl.g.C, num_sms_cached());
  if (!ws || ws_bytes < need)
    return set_error(CGBN_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need,
                     ws_bytes);
  *tickets = reinterpret_cast<unsigned*>(ws);
  *slots = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + kTicketBytes);
  return CGBN_OK;
}

template <class TOp>
int launch_tma_reduce(const Plan& pl, const TOp& op, double* out, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  unsigned* tickets;
  double2* slots;
  int rc = ws_parts(pl, ws, ws_bytes, &tickets, &slots);
  if (rc) return rc;
  tma_prepare(tma::k_tma_reduce<TOp>);
  tma::k_tma_reduce<TOp><<<pl.tg.grid, tma::kThreadsTma, tma::kSmemBytes, st>>>(
      pl.tg, op, out, slots, tickets);
  return CGBN_OK;
}

template <class Op>
int launch_reduce(const Plan& pl, const Op& op, double* out, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  Geom g = pl.g;
  if (pl.team) {
    g.grid = team_grid(k_reduce_team<Op>, pl);
    k_reduce_team<Op><<<g.grid, kThreads, 0, st>>>(g, op, out);
    return CGBN_OK;
  }
  const size_t need = ws_bytes_for(pl.g.C, num_sms_cached());
  if (!ws || ws_bytes < need)
    return set_error(CGBN_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need,
                     ws_bytes);
  unsigned* tickets = reinterpret_cast<unsigned*>(ws);
  double2* slots = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + kTicketBytes);
  g.grid = flat_grid(k_reduce_flat<Op>, pl);
  k_reduce_flat<Op><<<g.grid, kThreads, 0, st>>>(g, op, out, slots, tickets);
  return CGBN_OK;
}

template <int VEC>
int run_stats(const Plan& pl, const float* x, bool shift, int mode, double* out, double* out2,
              void* ws, size_t wsb, cudaStream_t st) {
  if (VEC == 4 && pl.tma && shift && mode == 0) {
    tma::TmaStats op;
    op.x = x;
    op.K = 0.0;
    return launch_tma_reduce(pl, op, out, ws, wsb, st);
  }
  StatsOp<VEC> op;
  op.x = x;
  op.K = 0.0;
  op.shift = shift;
  op.mode = mode;
  op.out2 = out2;
  return launch_reduce(pl, op, out, ws, wsb, st);
}

template <int VEC, bool RELU>
int run_bwd_reduce(const Plan& pl, const float* dy, const float* x, const double* saved,
                   const float* gamma, const float* beta, double* out, void* ws, size_t wsb,
                   cudaStream_t st) {
  if (VEC == 4 && pl.tma) {
    tma::TmaBwd<RELU> op;
    op.dy = dy;
    op.x = x;
    op.saved = saved;
    op.gamma = gamma;
    op.beta = beta;
    op.mean = op.P = op.Q = 0.0;
    return launch_tma_reduce(pl, op, out, ws, wsb, st);
  }
  BwdOp<VEC, RELU> op;
  op.dy = dy;
  op.x = x;
  op.saved = saved;
  op.gamma = gamma;
  op.beta = beta;
  op.mean = op.P = op.Q = 0.0;
  return launch_reduce(pl, op, out, ws, wsb, st);
}

template <int VEC, int MODE, bool RELU>
void launch_affine_v(const Plan& pl, const AffineArgs& A, cudaStream_t st) {
  Geom g = pl.g;
  if (VEC == 4 && pl.tma) {
    tma_prepare(tma::k_tma_affine<MODE, RELU>);
    tma::k_tma_affine<MODE, RELU><<<pl.tg.grid, tma::kThreadsTma, tma::kSmemBytes, st>>>(pl.tg, A);
    return;
  }
  if (pl.team) {
    g.grid = team_grid(k_affine_team<VEC, MODE, RELU>, pl);
    k_affine_team<VEC, MODE, RELU><<<g.grid, kThreads, 0, st>>>(g, A);
  } else {
    g.grid = flat_grid(k_affine_flat<VEC, MODE, RELU>, pl);
    k_affine_flat<VEC, MODE, RELU><<<g.grid, kThreads, 0, st>>>(g, A);
  }
}

template <int MODE>
void launch_affine(const Plan& pl, const AffineArgs& A, bool relu, cudaStream_t st) {
  if (relu) {
    switch (pl.vec) {
      case 4: launch_affine_v<4, MODE, true>(pl, A, st); break;
      case 2: launch_affine_v<2, MODE, true>(pl, A, st); break;
      default: launch_affine_v<1, MODE, true>(pl, A, st); break;
    }
  } else {
    switch (pl.vec) {
      case 4: launch_affine_v<4, MODE, false>(pl, A, st); break;
      case 2: launch_affine_v<2, MODE, false>(pl, A, st); break;
      default: launch_affine_v<1, MODE, false>(pl, A, st); break;
    }
  }
}

template <int VEC, bool RELU>
void launch_dx_v(const Plan& pl, const DxArgs& D, cudaStream_t st) {
  Geom g = pl.g;
  if (VEC == 4 && pl.tma) {
    tma_prepare(tma::k_tma_dx<RELU>);
    tma::k_tma_dx<RELU><<<pl.tg.grid, tma::kThreadsTma, tma::kSmemBytes, st>>>(pl.tg, D);
    return;
  }
  if (pl.team) {
    g.grid = team_grid(k_dx_team<VEC, RELU>, pl);
    k_dx_team<VEC, RELU><<<g.grid, kThreads, 0, st>>>(g, D);
  } else {
    g.grid = flat_grid(k_dx_flat<VEC, RELU>, pl);
    k_dx_flat<VEC, RELU><<<g.grid, kThreads, 0, st>>>(g, D);
  }
}

AffineArgs empty_affine_args() {
  AffineArgs A;
  A.x = nullptr; A.y = nullptr;
  A.parts.G = 0;
  for (int r = 0; r < CGBN_MAX_GROUP; ++r) A.parts.p[r] = nullptr;
  A.gamma = A.beta = A.rmean_in = A.rvar_in = nullptr;
  A.rmean = A.rvar = nullptr;
  A.saved = nullptr;
  A.scale = A.shift = nullptr;
  A.eps = 0.0; A.momentum = 0.0;
  A.status = nullptr;
  return A;
}

#define CGBN_REQUIRE(cond, ...) \
  do { if (!(cond)) return set_error(CGBN_ERR_INVALID, __VA_ARGS__); } while (0)

}  // namespace

// ==================================================================================
// C ABI

extern "C" {

int cgbn_abi_version(void) { return CGBN_ABI_VERSION; }

#define CGBN_STR2(x) #x
#define CGBN_STR(x) CGBN_STR2(x)
const char* cgbn_build_info(void) {
  return "cgbn sm_100a; nvcc " CGBN_STR(__CUDACC_VER_MAJOR__) "." CGBN_STR(__CUDACC_VER_MINOR__)
         "; kThreads=256; flat+team kernels";
}

const char* cgbn_last_error(void) { return g_last_error.c_str(); }

int cgbn_num_sms(void) { return num_sms_cached(); }

size_t cgbn_workspace_bytes(int64_t N, int64_t C, int64_t HW, int layout) {
  if (validate_shape(N, C, HW, layout)) return 0;
  return ws_bytes_for(C, num_sms_cached());
}

int cgbn_fwd_stats(const float* x, int64_t N, int64_t C, int64_t HW, int layout,
                   double* partial, void* ws, size_t ws_bytes, void* stream) {
  CGBN_REQUIRE(x && partial, "cgbn_fwd_stats: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 1, &pl);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (pl.vec) {
    case 4: rc = run_stats<4>(pl, x, true, 0, partial, nullptr, ws, ws_bytes, st); break;
    case 2: rc = run_stats<2>(pl, x, true, 0, partial, nullptr, ws, ws_bytes, st); break;
    default: rc = run_stats<1>(pl, x, true, 0, partial, nullptr, ws, ws_bytes, st); break;
  }
  if (rc) return rc;
  return check_launch("cgbn_fwd_stats");
}

int cgbn_channel_sum(const float* x, int64_t N, int64_t C, int64_t HW, int layout,
                     double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream) {
  CGBN_REQUIRE(x && sum, "cgbn_channel_sum: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 1, &pl);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (pl.vec) {
    case 4: rc = run_stats<4>(pl, x, false, 1, sum, sum_sq, ws, ws_bytes, st); break;
    case 2: rc = run_stats<2>(pl, x, false, 1, sum, sum_sq, ws, ws_bytes, st); break;
    default: rc = run_stats<1>(pl, x, false, 1, sum, sum_sq, ws, ws_bytes, st); break;
  }
  if (rc) return rc;
  return check_launch("cgbn_channel_sum");
}

int cgbn_fwd_normalize(const float* x, int64_t N, int64_t C, int64_t HW, int layout,
                       const double* const* partials, int G, const float* gamma,
                       const float* beta, double eps, double momentum, float* running_mean,
                       float* running_var, double* saved, int relu, float* y, unsigned* status,
                       void* stream) {
  CGBN_REQUIRE(x && y && gamma && beta && saved, "cgbn_fwd_normalize: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(momentum >= 0.0 && momentum <= 1.0, "momentum must lie in [0, 1], got %g",
               momentum);
  CGBN_REQUIRE((running_mean == nullptr) == (running_var == nullptr),
               "running_mean and running_var must both be set or both be NULL");
  const void* ptrs[] = {x, y};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 2, &pl);
  if (rc) return rc;
  AffineArgs A = empty_affine_args();
  rc = fill_parts(&A.parts, partials, G);
  if (rc) return rc;
  A.x = x; A.y = y;
  A.gamma = gamma; A.beta = beta;
  A.rmean = running_mean; A.rvar = running_var;
  A.saved = saved;
  A.eps = eps; A.momentum = momentum;
  A.status = status;
  launch_affine<kTrain>(pl, A, relu != 0, reinterpret_cast<cudaStream_t>(stream));
  return check_launch("cgbn_fwd_normalize");
}

int cgbn_fwd_eval(const float* x, int64_t N, int64_t C, int64_t HW, int layout,
                  const float* gamma, const float* beta, const float* running_mean,
                  const float* running_var, double eps, int relu, float* y, void* stream) {
  CGBN_REQUIRE(x && y && gamma && beta && running_mean && running_var,
               "cgbn_fwd_eval: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  const void* ptrs[] = {x, y};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 2, &pl);
  if (rc) return rc;
  AffineArgs A = empty_affine_args();
  A.x = x; A.y = y;
  A.gamma = gamma; A.beta = beta;
  A.rmean_in = running_mean; A.rvar_in = running_var;
  A.eps = eps;
  launch_affine<kEval>(pl, A, relu != 0, reinterpret_cast<cudaStream_t>(stream));
  return check_launch("cgbn_fwd_eval");
}

int cgbn_xhat(const float* x, int64_t N, int64_t C, int64_t HW, int layout,
              const double* saved, float* xhat, void* stream) {
  CGBN_REQUIRE(x && saved && xhat, "cgbn_xhat: NULL pointer");
  const void* ptrs[] = {x, xhat};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 2, &pl);
  if (rc) return rc;
  AffineArgs A = empty_affine_args();
  A.x = x; A.y = xhat;
  A.saved = const_cast<double*>(saved);
  launch_affine<kXhat>(pl, A, false, reinterpret_cast<cudaStream_t>(stream));
  return check_launch("cgbn_xhat");
}

int cgbn_channel_affine(const float* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* scale, const double* shift, float* out, void* stream) {
  CGBN_REQUIRE(x && scale && shift && out, "cgbn_channel_affine: NULL pointer");
  const void* ptrs[] = {x, out};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 2, &pl);
  if (rc) return rc;
  AffineArgs A = empty_affine_args();
  A.x = x; A.y = out;
  A.scale = scale; A.shift = shift;
  launch_affine<kAffine>(pl, A, false, reinterpret_cast<cudaStream_t>(stream));
  return check_launch("cgbn_channel_affine");
}

int cgbn_bwd_reduce(const float* dy, const float* x, int64_t N, int64_t C, int64_t HW,
                    int layout, const double* saved, const float* gamma, const float* beta,
                    int relu, double* partial, void* ws, size_t ws_bytes, void* stream) {
  CGBN_REQUIRE(dy && x && saved && partial, "cgbn_bwd_reduce: NULL pointer");
  CGBN_REQUIRE(!relu || (gamma && beta), "cgbn_bwd_reduce: relu needs gamma and beta");
  const void* ptrs[] = {dy, x};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 2, &pl);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (relu) {
    switch (pl.vec) {
      case 4: rc = run_bwd_reduce<4, true>(pl, dy, x, saved, gamma, beta, partial, ws, ws_bytes, st); break;
      case 2: rc = run_bwd_reduce<2, true>(pl, dy, x, saved, gamma, beta, partial, ws, ws_bytes, st); break;
      default: rc = run_bwd_reduce<1, true>(pl, dy, x, saved, gamma, beta, partial, ws, ws_bytes, st); break;
    }
  } else {
    switch (pl.vec) {
      case 4: rc = run_bwd_reduce<4, false>(pl, dy, x, saved, gamma, beta, partial, ws, ws_bytes, st); break;
      case 2: rc = run_bwd_reduce<2, false>(pl, dy, x, saved, gamma, beta, partial, ws, ws_bytes, st); break;
      default: rc = run_bwd_reduce<1, false>(pl, dy, x, saved, gamma, beta, partial, ws, ws_bytes, st); break;
    }
  }
  if (rc) return rc;
  return check_launch("cgbn_bwd_reduce");
}

int cgbn_bwd_dx(const float* dy, const float* x, int64_t N, int64_t C, int64_t HW, int layout,
                const double* const* partials, int G, const double* saved, const float* gamma,
                const float* beta, double eps, int relu, float* dx, float* dgamma,
                float* dbeta, unsigned* status, void* stream) {
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_dx: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_dx: relu needs beta");
  const void* ptrs[] = {dy, x, dx};
  Plan pl;
  int rc = make_plan(N, C, HW, layout, ptrs, 3, &pl);
  if (rc) return rc;
  DxArgs D;
  rc = fill_parts(&D.parts, partials, G);
  if (rc) return rc;
  D.dy = dy; D.x = x; D.dx = dx;
  D.saved = saved; D.gamma = gamma; D.beta = beta;
  D.dgamma = dgamma; D.dbeta = dbeta; D.status = status;
  D.eps = eps;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (relu) {
    switch (pl.vec) {
      case 4: launch_dx_v<4, true>(pl, D, st); break;
      case 2: launch_dx_v<2, true>(pl, D, st); break;
      default: launch_dx_v<1, true>(pl, D, st); break;
    }
  } else {
    switch (pl.vec) {
      case 4: launch_dx_v<4, false>(pl, D, st); break;
      case 2: launch_dx_v<2, false>(pl, D, st); break;
      default: launch_dx_v<1, false>(pl, D, st); break;
    }
  }
  return check_launch("cgbn_bwd_dx");
}

int cgbn_fold_sum(const void* const* vectors, int G, int64_t n, int dtype, void* out,
                  void* stream) {
  CGBN_REQUIRE(vectors && out, "cgbn_fold_sum: NULL pointer");
  CGBN_REQUIRE(n >= 1, "cgbn_fold_sum: n must be >= 1");
  CGBN_REQUIRE(dtype == CGBN_DTYPE_F32 || dtype == CGBN_DTYPE_F64, "unknown dtype %d", dtype);
  Parts P;
  int rc = fill_parts(&P, reinterpret_cast<const double* const*>(vectors), G);
  if (rc) return rc;
  const int threads = 256;
  int64_t blocks = ceil_div(n, threads);
  if (blocks > (int64_t)num_sms_cached() * 8) blocks = (int64_t)num_sms_cached() * 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == CGBN_DTYPE_F64)
    k_fold_sum<double><<<(unsigned)blocks, threads, 0, st>>>(P, n, reinterpret_cast<double*>(out));
  else
    k_fold_sum<float><<<(unsigned)blocks, threads, 0, st>>>(P, n, reinterpret_cast<float*>(out));
  return check_launch("cgbn_fold_sum");
}

}  // extern "C"
