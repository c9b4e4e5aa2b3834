// cgbn.cu — sm_100a kernels and the C ABI (include/cgbn.h) of the CGBN hot path.
//
// The path is HBM-bandwidth bound (no contraction; tensor cores do not apply), so every
// kernel is a streaming pass over the activation with 128-bit coalesced loads, several
// loads in flight per thread, and a deterministic reduction tree. Work decomposition:
// a channel's "stream" is the concatenation of its N planes (NCHW: N runs of HW
// contiguous floats, stride C*HW apart); each channel stream is cut into S chunks and
// CTA (s, c) owns chunk s of channel c. Reductions fold per-thread -> warp shuffle ->
// CTA (fixed order) -> per-channel fixed-order fold of the S CTA partials by the last
// CTA to arrive (arrival ticket), so results are bitwise run-to-run reproducible and
// need no float atomics.
//
// Reference being replaced (file:line under /root/reference/pkg/src/bigbatch):
//   channel_sum / sequential_sum_rows      tensor.py:121-153   -> k_reduce<StatsOp>
//   _train_forward post-reduction + affine batchnorm.py:121-143 -> k_affine<TRAIN>
//   bn_update_running                      batchnorm.py:239-252 (fused into k_affine)
//   _backward_core sums                    batchnorm.py:198-201 -> k_reduce<BwdOp>
//   _backward_core dx                      batchnorm.py:203-209 -> k_bwd_dx
//   allreduce_sum root fold                collectives.py:293-295 (ascending-rank fold,
//                                          done by every consumer kernel's prologue)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "cgbn.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

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

// All sizes in "vector units" of VEC floats. Element offset of vector j of channel c:
//   (c*HWv + j + (j / HWv) * gap) * VEC          with gap = (C-1)*HWv.
// NCHW: HWv = HW/VEC.  NHWC and 2-D (N, C): one "plane" per row, HWv = 1, VEC = 1.
struct Geom {
  uint32_t C;
  uint32_t Lv;     // vector units per channel stream (N*HW/VEC)
  uint32_t HWv;    // vector units per plane
  uint32_t S;      // CTAs per channel
  uint32_t chunk;  // vector units per CTA
  uint64_t gap;    // (C-1)*HWv
  FastDiv dhw;
  double count;    // elements per channel on this rank (N*HW)
};

__device__ __forceinline__ size_t voff(const Geom& g, uint32_t c, uint32_t j) {
  return (size_t)c * g.HWv + j + (size_t)g.dhw.div(j) * g.gap;
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

// ----------------------------------------------------------------------------------
// Deterministic CTA reduction of two fp64 accumulators (result valid in thread 0).

__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double sa[kWarps], sb[kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sa[w] = a; sb[w] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = sa[0]; b = sb[0];
#pragma unroll
    for (int i = 1; i < kWarps; ++i) { a += sa[i]; b += sb[i]; }
  }
}

// ----------------------------------------------------------------------------------
// Reduction ops (per-channel two-accumulator sums over one or two streams)

// Forward statistics: shifted sums of d = x - K (K = first element of the channel on
// this rank, identical for every CTA of the channel) -> (mean, M2, count).
template <int VEC>
struct StatsOp {
  const float* __restrict__ x;
  double K;
  struct Regs { float v[VEC]; };
  __device__ __forceinline__ void init(const Geom& g, uint32_t c) {
    K = shift ? (double)__ldg(x + (size_t)c * g.HWv * VEC) : 0.0;
  }
  __device__ __forceinline__ void load(size_t off, Regs& r) const { ldv<VEC>(x + off * VEC, r.v); }
  // d = x - K is exact in fp64 (both operands are fp32 values).
  __device__ __forceinline__ void acc(const Regs& r, double& a, double& b) const {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const double d = (double)r.v[k] - K;
      a += d;
      b = __fma_rn(d, d, b);
    }
  }
  bool shift;
  // mode 0: forward partial [mean | M2 | count]; mode 1: raw sums [sum | sum_sq]
  int mode;
  double* __restrict__ out2;  // mode 1: sum_sq destination (may be null)
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

// Backward: g = dy (ReLU-masked when the forward fused a ReLU), fp64 sums of g and
// g*(x - mean).
template <int VEC, bool RELU>
struct BwdOp {
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

template <int VEC>
constexpr int unroll_for() { return VEC == 4 ? 4 : 8; }

// Grid (S, C). Each thread issues U independent vector loads per iteration and
// accumulates every element in fp64 (the reference's f64 statistics need ~1e-8
// absolute accuracy on y near 0 under its rel_err floor of 1e-3).
template <int VEC, class Op>
__global__ void __launch_bounds__(kThreads)
k_reduce(Geom g, Op op, double* __restrict__ out, double2* __restrict__ ws,
         unsigned* __restrict__ tickets) {
  constexpr int U = unroll_for<VEC>();
  const uint32_t c = blockIdx.y, s = blockIdx.x;
  const uint32_t i0 = s * g.chunk;
  const uint32_t i1 = min(i0 + g.chunk, g.Lv);
  op.init(g, c);

  // fp64 accumulation per element (the fp32 difference x - shift is rounded once);
  // U independent accumulator pairs keep the DADD/DFMA chains short.
  double a[U], b[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { a[u] = 0.0; b[u] = 0.0; }
  uint32_t i = i0 + threadIdx.x;
  for (; i + (U - 1) * kThreads < i1; i += U * kThreads) {
    typename Op::Regs r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) op.load(voff(g, c, i + u * kThreads), r[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) op.acc(r[u], a[u], b[u]);
  }
  for (; i < i1; i += kThreads) {
    typename Op::Regs r;
    op.load(voff(g, c, i), r);
    op.acc(r, a[0], b[0]);
  }
  double S1 = a[0], S2 = b[0];
#pragma unroll
  for (int u = 1; u < U; ++u) { S1 += a[u]; S2 += b[u]; }
  block_sum2(S1, S2);

  if (g.S == 1) {
    if (threadIdx.x == 0) op.finish(g, c, S1, S2, out);
    return;
  }
  // Cross-CTA: publish this CTA's partial, take a ticket; the last CTA of the channel
  // folds the S partials in index order (deterministic regardless of arrival order).
  __shared__ unsigned s_ticket;
  if (threadIdx.x == 0) {
    ws[(size_t)c * g.S + s] = make_double2(S1, S2);
    __threadfence();
    s_ticket = atomicAdd(&tickets[c], 1u);
  }
  __syncthreads();
  if (s_ticket != g.S - 1) return;
  if (threadIdx.x < 32) {
    __threadfence();
    const int l = threadIdx.x;
    double a = 0.0, b = 0.0;
    for (uint32_t k = l; k < g.S; k += 32) {
      const double2 t = __ldcg(&ws[(size_t)c * g.S + k]);
      a += t.x;
      b += t.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
    if (l == 0) {
      op.finish(g, c, a, b, out);
      tickets[c] = 0u;  // leave the workspace reusable
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

template <int MODE>
__device__ __forceinline__ void affine_prologue(const Geom& g, const AffineArgs& A, uint32_t c,
                                                uint32_t s, double& P, double& Q) {
  if constexpr (MODE == kTrain) {
    double n, mean, M2;
    merge_fwd_partials(A.parts, c, g.C, n, mean, M2);
    const double var = fmax(M2 / n, 0.0);
    const double inv_std = 1.0 / sqrt(var + A.eps);
    affine_coeffs(mean, inv_std, (double)A.gamma[c], (double)A.beta[c], P, Q);
    if (s == 0) {
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

template <int VEC, int MODE, bool RELU>
__global__ void __launch_bounds__(kThreads) k_affine(Geom g, AffineArgs A) {
  constexpr int U = unroll_for<VEC>();
  const uint32_t c = blockIdx.y, s = blockIdx.x;
  __shared__ double sP, sQ;
  if (threadIdx.x == 0) {
    double P, Q;
    affine_prologue<MODE>(g, A, c, s, P, Q);
    sP = P;
    sQ = Q;
  }
  __syncthreads();
  const double P = sP, Q = sQ;
  const uint32_t i0 = s * g.chunk;
  const uint32_t i1 = min(i0 + g.chunk, g.Lv);
  const float* __restrict__ x = A.x;
  float* __restrict__ y = A.y;

  uint32_t i = i0 + threadIdx.x;
  for (; i + (U - 1) * kThreads < i1; i += U * kThreads) {
    float v[U][VEC];
    size_t off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      off[u] = voff(g, c, i + u * kThreads) * VEC;
      ldv<VEC>(x + off[u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        double t = bn_out(P, Q, v[u][k]);
        if (RELU) t = t > 0.0 ? t : 0.0;
        v[u][k] = (float)t;
      }
      stv<VEC>(y + off[u], v[u]);
    }
  }
  for (; i < i1; i += kThreads) {
    float v[VEC];
    const size_t off = voff(g, c, i) * VEC;
    ldv<VEC>(x + off, v);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      double t = bn_out(P, Q, v[k]);
      if (RELU) t = t > 0.0 ? t : 0.0;
      v[k] = (float)t;
    }
    stv<VEC>(y + off, v);
  }
}

// ----------------------------------------------------------------------------------
// Backward dx: prologue folds the G backward partials (ascending rank order), then
// dx = A*g + B*x + Cc with A = gamma/sqrt(var+eps), B = -A*inv_std*dgamma/m,
// Cc = -A*dbeta/m - B*mean  (== gamma*inv_std*(g - dbeta/m - x_hat*dgamma/m)).

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

template <int VEC, bool RELU>
__global__ void __launch_bounds__(kThreads) k_bwd_dx(Geom g, DxArgs D) {
  constexpr int U = unroll_for<VEC>();
  const uint32_t c = blockIdx.y, s = blockIdx.x;
  const uint32_t C = g.C;
  __shared__ double sA, sB, sC, sP, sQ;
  if (threadIdx.x == 0) {
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
    // batchnorm.py:205: gamma / sqrt(var + eps) with the backward state's eps (x_hat
    // itself keeps the forward's inv_std, as the reference's cached x_hat does).
    const double A = gam / sqrt(D.saved[C + c] + D.eps);
    const double B = -A * inv_std * (dgamma / m);
    const double Cc = -A * (dbeta / m) - B * mean;
    sA = A; sB = B; sC = Cc;
    if (RELU) {
      double P, Q;
      affine_coeffs(mean, inv_std, gam, (double)D.beta[c], P, Q);
      sP = P; sQ = Q;
    }
    if (s == 0) {
      if (D.dgamma) D.dgamma[c] = (float)dgamma;
      if (D.dbeta) D.dbeta[c] = (float)dbeta;
      if (D.status && (!isfinite(dbeta) || !isfinite(dgamma)))
        atomicOr(D.status, CGBN_STATUS_NONFINITE);
    }
  }
  __syncthreads();
  const double A = sA, B = sB, Cc = sC;
  double P = 0.0, Q = 0.0;
  if (RELU) { P = sP; Q = sQ; }
  const uint32_t i0 = s * g.chunk;
  const uint32_t i1 = min(i0 + g.chunk, g.Lv);

  uint32_t i = i0 + threadIdx.x;
  for (; i + (U - 1) * kThreads < i1; i += U * kThreads) {
    float gv[U][VEC], xv[U][VEC];
    size_t off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      off[u] = voff(g, c, i + u * kThreads) * VEC;
      ldv<VEC>(D.dy + off[u], gv[u]);
      ldv<VEC>(D.x + off[u], xv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        double gk = (double)gv[u][k];
        if (RELU && !(bn_out(P, Q, xv[u][k]) > 0.0)) gk = 0.0;
        gv[u][k] = (float)__fma_rn(A, gk, __fma_rn(B, (double)xv[u][k], Cc));
      }
      stv<VEC>(D.dx + off[u], gv[u]);
    }
  }
  for (; i < i1; i += kThreads) {
    float gv[VEC], xv[VEC];
    const size_t off = voff(g, c, i) * VEC;
    ldv<VEC>(D.dy + off, gv);
    ldv<VEC>(D.x + off, xv);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      double gk = (double)gv[k];
      if (RELU && !(bn_out(P, Q, xv[k]) > 0.0)) gk = 0.0;
      gv[k] = (float)__fma_rn(A, gk, __fma_rn(B, (double)xv[k], Cc));
    }
    stv<VEC>(D.dx + off, gv);
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

// Splits per channel, independent of vector width (the workspace size must not depend
// on pointer alignment). Target: ~8 resident 256-thread CTAs per SM worth of CTAs, and
// at least ~16 elements per thread per CTA.
int64_t splits_for(int64_t N, int64_t C, int64_t HW, int layout, int sms) {
  (void)layout;
  const int64_t L = N * HW;
  const int64_t target = (int64_t)sms * 8;
  int64_t S = ceil_div(target, C);
  const int64_t smax = ceil_div(L, (int64_t)kThreads * 16);
  if (S > smax) S = smax;
  if (S > 4096) S = 4096;
  if (S < 1) S = 1;
  return S;
}

size_t ws_bytes_for(int64_t C, int64_t S) {
  const size_t tick = ((size_t)C * sizeof(unsigned) + 255) / 256 * 256;
  return tick + (S > 1 ? (size_t)C * (size_t)S * sizeof(double2) : 0);
}

struct Plan {
  int vec;
  Geom g;
  dim3 grid;
};

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
  const int sms = num_sms_cached();
  const int64_t S0 = splits_for(N, C, HW, layout, sms);
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
  int64_t chunk = ceil_div(g.Lv, S0);
  const int64_t S = ceil_div(g.Lv, chunk);
  g.chunk = (uint32_t)chunk;
  g.S = (uint32_t)S;
  out->vec = vec;
  out->g = g;
  out->grid = dim3((unsigned)S, (unsigned)C, 1);
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

template <class Op>
int launch_reduce_op(const Plan& pl, Op op, double* out, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  const size_t need = ws_bytes_for(pl.g.C, pl.g.S);
  if (pl.g.S > 1 && (!ws || ws_bytes < need))
    return set_error(CGBN_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need,
                     ws_bytes);
  unsigned* tickets = reinterpret_cast<unsigned*>(ws);
  double2* parts = reinterpret_cast<double2*>(
      reinterpret_cast<char*>(ws) + (((size_t)pl.g.C * sizeof(unsigned) + 255) / 256 * 256));
  constexpr int VEC = Op::kVec;
  k_reduce<VEC, Op><<<pl.grid, kThreads, 0, st>>>(pl.g, op, out, parts, tickets);
  return CGBN_OK;
}

template <int VEC>
struct StatsOpV : StatsOp<VEC> { static constexpr int kVec = VEC; };
template <int VEC, bool RELU>
struct BwdOpV : BwdOp<VEC, RELU> { static constexpr int kVec = VEC; };

template <int VEC>
int run_stats(const Plan& pl, const float* x, bool shift, int mode, double* out, double* out2,
              void* ws, size_t wsb, cudaStream_t st) {
  StatsOpV<VEC> op;
  op.x = x;
  op.K = 0.0;
  op.shift = shift;
  op.mode = mode;
  op.out2 = out2;
  return launch_reduce_op(pl, op, out, ws, wsb, st);
}

template <int VEC, bool RELU>
int run_bwd_reduce(const Plan& pl, const float* dy, const float* x, const double* saved,
                   const float* gamma, const float* beta, double* out, void* ws, size_t wsb,
                   cudaStream_t st) {
  BwdOpV<VEC, RELU> op;
  op.dy = dy;
  op.x = x;
  op.saved = saved;
  op.gamma = gamma;
  op.beta = beta;
  op.mean = op.P = op.Q = 0.0;
  return launch_reduce_op(pl, op, out, ws, wsb, st);
}

template <int MODE, bool RELU>
void launch_affine(const Plan& pl, const AffineArgs& A, cudaStream_t st) {
  switch (pl.vec) {
    case 4: k_affine<4, MODE, RELU><<<pl.grid, kThreads, 0, st>>>(pl.g, A); break;
    case 2: k_affine<2, MODE, RELU><<<pl.grid, kThreads, 0, st>>>(pl.g, A); break;
    default: k_affine<1, MODE, RELU><<<pl.grid, kThreads, 0, st>>>(pl.g, A); break;
  }
}

template <int MODE>
void launch_affine_relu(const Plan& pl, const AffineArgs& A, bool relu, cudaStream_t st) {
  if (relu) launch_affine<MODE, true>(pl, A, st);
  else launch_affine<MODE, false>(pl, A, st);
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
         "; kThreads=256";
}

const char* cgbn_last_error(void) { return g_last_error.c_str(); }

int cgbn_num_sms(void) { return num_sms_cached(); }

size_t cgbn_workspace_bytes(int64_t N, int64_t C, int64_t HW, int layout) {
  if (validate_shape(N, C, HW, layout)) return 0;
  return ws_bytes_for(C, splits_for(N, C, HW, layout, num_sms_cached()));
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
  launch_affine_relu<kTrain>(pl, A, relu != 0, reinterpret_cast<cudaStream_t>(stream));
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
  launch_affine_relu<kEval>(pl, A, relu != 0, reinterpret_cast<cudaStream_t>(stream));
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
  launch_affine_relu<kXhat>(pl, A, false, reinterpret_cast<cudaStream_t>(stream));
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
  launch_affine_relu<kAffine>(pl, A, false, reinterpret_cast<cudaStream_t>(stream));
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
      case 4: k_bwd_dx<4, true><<<pl.grid, kThreads, 0, st>>>(pl.g, D); break;
      case 2: k_bwd_dx<2, true><<<pl.grid, kThreads, 0, st>>>(pl.g, D); break;
      default: k_bwd_dx<1, true><<<pl.grid, kThreads, 0, st>>>(pl.g, D); break;
    }
  } else {
    switch (pl.vec) {
      case 4: k_bwd_dx<4, false><<<pl.grid, kThreads, 0, st>>>(pl.g, D); break;
      case 2: k_bwd_dx<2, false><<<pl.grid, kThreads, 0, st>>>(pl.g, D); break;
      default: k_bwd_dx<1, false><<<pl.grid, kThreads, 0, st>>>(pl.g, D); break;
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
