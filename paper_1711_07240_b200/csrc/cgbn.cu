// cgbn.cu — sm_100a kernels and the C ABI (include/cgbn.h) of the CGBN hot path.
//
// The path is HBM-bandwidth bound (no contraction; tensor cores do not apply). Each BN
// direction is a per-channel reduction followed by an elementwise pass:
//
//  * reduction kernels (statistics; backward sums) stream a channel's "stream" -- its N
//    planes of HW elements, C*HW apart in NCHW -- with 16-byte loads (4 fp32 or 8
//    bf16 / fp16 values; masked covers for odd planes), several independent loads in
//    flight per thread, an incremental address cursor, and fp64 accumulation per element.
//    Work decompositions, chosen per shape:
//      cluster-team (k_reduce_ct, NCHW default): a thread-block cluster of KC CTAs owns
//        whole channels; in each CTA a team of 2^TL threads streams its rank's share of
//        one channel, warp partials meet in shared memory and the KC CTA partials are
//        folded over DSMEM in rank order (tools/flatlab.cu measured the decomposition);
//      rows (k_reduce_rows + k_fold_rows, NHWC and (N, C)): threads own 4 adjacent
//        channels and walk rows with contiguous loads; row-block partials are folded
//        one warp per channel;
//      flat / team: fallbacks (channel counts too small for clusters to fill the GPU;
//        NHWC with C % 4 != 0).
//    The thread that completes a channel also *finishes* it: for a single-rank group
//    (G == 1) it computes mean/var/inv_std (resp. dgamma/dbeta), updates the running
//    statistics and writes the channel's affine coefficients into a table in the
//    workspace; for G > 1 it writes the rank partial that the group exchanges, and a
//    small finalize kernel folds the G partials (ascending rank order) into the same
//    table after the exchange.
//  * elementwise kernels (normalise, dx) are a memory-order grid-stride sweep over the
//    whole tensor in 16-byte units (coalesced for every layout), run from the end of the
//    tensor for L2 reuse, looking up each element's channel coefficients in the table.
//  * every kernel uses programmatic dependent launch (pdl_wait / pdl_trigger).
//
// Every reduction folds in a fixed order, so results are bitwise run-to-run
// reproducible without float atomics, and all ranks of a group compute identical
// statistics from the identical gathered partials.
//
// Reference being replaced (file:line under /root/reference/pkg/src/bigbatch):
//   channel_sum / sequential_sum_rows      tensor.py:121-153   -> reduce kernels, StatsOp
//   _train_forward finalise                batchnorm.py:121-138 -> finalize_fwd_channel
//   channel_affine (x_hat, y)              batchnorm.py:139-140, tensor.py:156-170 -> k_ew_affine
//   bn_update_running                      batchnorm.py:239-252 (in finalize_fwd_channel)
//   _backward_core sums                    batchnorm.py:198-201 -> reduce kernels, BwdOp
//   _backward_core dgamma/dbeta, dx        batchnorm.py:203-209 -> finalize_bwd_channel, k_ew_dx
//   allreduce_sum root fold                collectives.py:293-295 (ascending-rank fold in
//                                          k_finalize_* / merge_fwd_partials)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <utility>

#include "cgbn.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kTeamMaxLv = 2048;  // channels up to this many units use team kernels
constexpr int64_t kMinElemsPerCta = 2048;
constexpr int kMaxCtasPerSm = 8;  // 2048 threads / 256
// Workspace head: 65536 per-channel tickets (fixed size: independent of C), then 64
// words of grid-barrier state for the fused cooperative kernels.
constexpr size_t kTicketWords = 65536;
constexpr size_t kTicketBytes = (kTicketWords + 64) * sizeof(unsigned);

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

// Unsigned 32-bit division by a runtime-constant divisor, valid for every n < 2^32
// (Hacker's Delight round-up method): t = umulhi(n, m), q = (t + ((n - t) >> s1)) >> s2
// with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1, s1 = min(l, 1), s2 = l - s1.
struct FastDiv {
  uint32_t m, s1, s2;
  void init(uint32_t d) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    s1 = l < 1 ? l : 1;
    s2 = l - s1;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> s1)) >> s2;
  }
};

// Reduction-kernel geometry. Element offset of vector unit j of channel c:
// (c*HWv + j + (j / HWv) * gap) * VEC with gap = (C-1)*HWv. NCHW: HWv = HW/VEC.
// NHWC and 2-D (N, C): HWv = 1, VEC = 1.
// VM (vector mode) 1, 2, 4: exact vectors of VM floats (HW % VM == 0); VM 5 = "masked
// float4": planes whose length is not a multiple of 4 (ResNet 7x7, FPN 25x42 / 13x21) are
// read as the aligned float4 cover of each plane (ceil(HW/4) + 1 units per plane) with a
// per-element mask, so odd planes also stream with 128-bit loads.
struct Geom {
  uint32_t C;
  uint32_t Lv;        // vector units per channel stream (N*HWv)
  uint32_t HWv;       // vector units per plane
  uint32_t grid;      // CTAs of this launch
  uint32_t tpc_log2;  // team kernels: log2(threads per channel)
  uint32_t HW;        // floats per plane (1 for NHWC / 2-D)
  uint64_t T;         // C * Lv
  uint64_t gap;       // (C-1)*HWv
  FastDiv dhw;        // division by HWv
  double count;       // elements per channel on this rank (N*HW)
};

// Vector modes (elements per load unit): 1, 2, 4, 8 exact; 5 = masked 4-element cover
// (fp32), 9 = masked 8-element cover (bf16 / fp16). A unit is at most 16 bytes.
constexpr int vec_of(int vm) { return vm == 5 ? 4 : vm == 9 ? 8 : vm; }
constexpr bool masked_vm(int vm) { return vm == 5 || vm == 9; }

// Unit cursor: the position of one thread in a channel stream, advanced by a fixed
// stride without a division per unit. P = (n*C + c)*HWv is the vector-unit index of the
// start of plane (n, c), o the unit within the plane, ps = (n*C + c)*HW the plane start
// in floats (masked mode). All fit in 32 bits (N*C*HW < 2^32). tools/flatlab.cu measured
// the per-unit FastDiv + 64-bit multiply addressing at 1.2-2 us per launch on ResNet
// mid shapes.
struct Cursor {
  uint32_t P, o, ps;
};

struct Step {
  uint32_t q, r;  // stride = q*HWv + r
};

__device__ __forceinline__ Cursor cursor_at(const Geom& g, uint32_t c, uint32_t j) {
  const uint32_t n = g.dhw.div(j);
  const uint32_t nc = n * g.C + c;
  return Cursor{nc * g.HWv, j - n * g.HWv, nc * g.HW};
}

__device__ __forceinline__ Step step_of(const Geom& g, uint32_t stride) {
  const uint32_t q = g.dhw.div(stride);
  return Step{q, stride - q * g.HWv};
}

__device__ __forceinline__ void advance(const Geom& g, Cursor& k, const Step& s) {
  const uint32_t CHWv = g.C * g.HWv, CHW = g.C * g.HW;
  k.o += s.r;
  k.P += s.q * CHWv;
  k.ps += s.q * CHW;
  if (k.o >= g.HWv) {
    k.o -= g.HWv;
    k.P += CHWv;
    k.ps += CHW;
  }
}

// Address (in floats) and element mask of the unit under the cursor.
template <int VM>
__device__ __forceinline__ uint32_t unit_addr(const Geom& g, const Cursor& k, uint32_t& mask) {
  constexpr uint32_t V = vec_of(VM);
  if constexpr (!masked_vm(VM)) {
    mask = (1u << V) - 1u;
    return (k.P + k.o) * V;
  } else {
    const uint32_t base = (k.ps & ~(V - 1u)) + V * k.o;
    const int lo = (int)(k.ps - base);            // plane start relative to the unit
    const int hi = lo + (int)g.HW;                // plane end relative to the unit
    mask = 0u;
#pragma unroll
    for (int e = 0; e < (int)V; ++e) mask |= (e >= lo && e < hi) ? (1u << e) : 0u;
    return base;
  }
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
// Vector load / store of activation elements (fp32, bf16 or fp16 storage; every kernel
// computes in fp64 and rounds once on output).

template <class T>
__device__ __forceinline__ float h2f(unsigned short h);
template <>
__device__ __forceinline__ float h2f<__nv_bfloat16>(unsigned short h) {
  return __bfloat162float(__ushort_as_bfloat16(h));
}
template <>
__device__ __forceinline__ float h2f<__half>(unsigned short h) {
  return __half2float(__ushort_as_half(h));
}

// one element, as float
template <class T>
__device__ __forceinline__ float ld1(const T* __restrict__ p) {
  if constexpr (sizeof(T) == 4) return __ldg(reinterpret_cast<const float*>(p));
  else return h2f<T>(__ldg(reinterpret_cast<const unsigned short*>(p)));
}

// fp64 -> storage, rounded once
template <class T>
__device__ __forceinline__ uint32_t rnd(double v) {
  if constexpr (sizeof(T) == 4) return __float_as_uint((float)v);
  else if constexpr (std::is_same<T, __nv_bfloat16>::value)
    return __bfloat16_as_ushort(__double2bfloat16(v));
  else return __half_as_ushort(__double2half(v));
}

template <class T>
__device__ __forceinline__ void st1(T* p, double v) {
  if constexpr (sizeof(T) == 4) *reinterpret_cast<float*>(p) = (float)v;
  else *reinterpret_cast<unsigned short*>(p) = (unsigned short)rnd<T>(v);
}

// V elements of T held as raw 32-bit words (the registers of one vector load).
template <class T, int V>
struct Vec {
  static constexpr int kBytes = V * (int)sizeof(T);
  static constexpr int kWords = kBytes >= 4 ? kBytes / 4 : 1;
  uint32_t w[kWords];
  __device__ __forceinline__ void load(const T* __restrict__ p) {
    if constexpr (kBytes == 16) {
      const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    } else if constexpr (kBytes == 8) {
      const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = t.x; w[1] = t.y;
    } else if constexpr (kBytes == 4) {
      w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
    } else {
      w[0] = __ldg(reinterpret_cast<const unsigned short*>(p));
    }
  }
  __device__ __forceinline__ float get(int k) const {
    if constexpr (sizeof(T) == 4) return __uint_as_float(w[k]);
    else return h2f<T>((unsigned short)(w[k >> 1] >> (16 * (k & 1))));
  }
};

// Round V fp64 values to T and store them as one vector.
template <class T, int V>
__device__ __forceinline__ void stv(T* __restrict__ p, const double (&t)[V]) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (V == 4) {
      *reinterpret_cast<float4*>(p) = make_float4((float)t[0], (float)t[1], (float)t[2], (float)t[3]);
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) reinterpret_cast<float*>(p)[k] = (float)t[k];
    }
  } else {
    static_assert(V % 2 == 0, "16-bit stores pack pairs");
    uint32_t w[V / 2];
#pragma unroll
    for (int k = 0; k < V / 2; ++k) w[k] = rnd<T>(t[2 * k]) | (rnd<T>(t[2 * k + 1]) << 16);
    if constexpr (V == 8) *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    else if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    else *reinterpret_cast<uint32_t*>(p) = w[0];
  }
}

// Loads in flight per thread per round: ~128 B for one input stream, ~128 B total for
// two (NIN = number of input streams).
#ifndef CGBN_RED_U1
#define CGBN_RED_U1 8  // loads in flight per thread per round, one input stream
#endif
#ifndef CGBN_RED_U2
#define CGBN_RED_U2 4  // units per round with two input streams (dy, x)
#endif
#ifndef CGBN_CT_MINB
#define CGBN_CT_MINB 4  // k_reduce_ct CTAs per SM (register bound)
#endif
template <int VM, int NIN = 1>
constexpr int unroll_for() { return (NIN == 1 || VM == 1) ? CGBN_RED_U1 : CGBN_RED_U2; }

// Visit units j = start, start+stride, ... < end of channel c in rounds of U: the U
// (predicated) loads of a round are issued before any of them is used.
template <int U, class Op, class Body>
__device__ __forceinline__ void strided_rounds(const Geom& g, uint32_t c, uint32_t start,
                                               uint32_t end, uint32_t stride, const Op& op,
                                               Body&& body) {
  if (start >= end) return;
  Cursor k = cursor_at(g, c, start);
  const Step s = step_of(g, stride);
  for (uint32_t i = start; i < end; i += U * stride) {
    typename Op::Regs r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j < end) op.load(g, k, r[u]);
      advance(g, k, s);  // after U steps: the next round's first unit
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j < end) body(u, j, r[u]);
    }
  }
}

// ----------------------------------------------------------------------------------
// Shared per-channel arithmetic (fp64). The same inline functions produce the forward
// coefficients and the ReLU mask the backward recomputes, so the mask is bitwise the
// forward's.

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

// Programmatic dependent launch (CGBN_NO_PDL=1 disables it). Every kernel waits
// (griddepcontrol.wait) before reading what the previous kernel may have produced and
// then lets the next one launch. The elementwise kernels prefetch their first round of
// x / dy before waiting: they always follow one of our reduction / finalize kernels,
// which passed its own wait, so x / dy are complete; only the coefficients are not.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Asynchronous global -> shared copies (no register staging): the finisher's per-channel
// inputs are fetched while the data streams and waited for only at the end.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ----------------------------------------------------------------------------------
// Channel finishers: the group statistics of one channel -> everything downstream.

// Forward: outputs of one channel once its group (n, mean, M2) is known
// (batchnorm.py:121-141): biased var, inv_std = 1/sqrt(var+eps), coefficient table
// P/Q, saved statistics for the backward, running-stat update with the unbiased
// m/(m-1) correction (batchnorm.py:239-252) and the device status word.
struct FwdFinal {
  const float* gamma;
  const float* beta;
  double eps, momentum;
  float* rmean;  // may be null (no running update)
  float* rvar;
  double* saved;  // [mean C | var C | inv_std C | m]
  double* P;      // coefficient table (null when the caller keeps the coefficients)
  double* Q;
  unsigned* status;
  uint32_t C;
};

// Per-channel inputs of the forward finisher (prefetchable).
struct FwdChan {
  float gamma, beta, rmean, rvar;
};

__device__ __forceinline__ FwdChan load_fwd_chan(const FwdFinal& F, uint32_t c) {
  FwdChan v;
  v.gamma = F.gamma[c];
  v.beta = F.beta[c];
  v.rmean = F.rmean ? F.rmean[c] : 0.f;
  v.rvar = F.rvar ? F.rvar[c] : 0.f;
  return v;
}

__device__ __forceinline__ void load_fwd_chan_async(const FwdFinal& F, uint32_t c, FwdChan* d) {
  cp_async4(&d->gamma, F.gamma + c);
  cp_async4(&d->beta, F.beta + c);
  if (F.rmean) {
    cp_async4(&d->rmean, F.rmean + c);
    cp_async4(&d->rvar, F.rvar + c);
  } else {
    d->rmean = d->rvar = 0.f;
  }
}

__device__ __forceinline__ void finalize_fwd_channel_var(const FwdFinal& F, uint32_t c, double n,
                                                         double mean, double var, bool write,
                                                         const FwdChan& v, double& P, double& Q) {
  const double inv_std = 1.0 / sqrt(var + F.eps);
  affine_coeffs(mean, inv_std, (double)v.gamma, (double)v.beta, P, Q);
  if (F.P) { F.P[c] = P; F.Q[c] = Q; }
  if (!write) return;
  const uint32_t C = F.C;
  F.saved[c] = mean;
  F.saved[C + c] = var;
  F.saved[2 * C + c] = inv_std;
  if (c == 0) F.saved[3 * C] = n;
  unsigned bad = 0;
  if (!isfinite(mean) || !isfinite(var)) bad |= CGBN_STATUS_NONFINITE;
  if (n < 2.0) bad |= CGBN_STATUS_SMALL_COUNT;
  if (bad) {
    if (F.status) atomicOr(F.status, bad);
  } else if (F.rmean) {
    const double rho = F.momentum;
    const double unbiased = var * (n / (n - 1.0));
    F.rmean[c] = (float)((1.0 - rho) * (double)v.rmean + rho * mean);
    F.rvar[c] = (float)((1.0 - rho) * (double)v.rvar + rho * unbiased);
  }
}

__device__ __forceinline__ void finalize_fwd_channel(const FwdFinal& F, uint32_t c, double n,
                                                     double mean, double M2, bool write,
                                                     const FwdChan& v, double& P, double& Q) {
  finalize_fwd_channel_var(F, c, n, mean, fmax(M2 / n, 0.0), write, v, P, Q);
}

__device__ __forceinline__ void finalize_fwd_channel(const FwdFinal& F, uint32_t c, double n,
                                                     double mean, double M2, bool write,
                                                     double& P, double& Q) {
  finalize_fwd_channel(F, c, n, mean, M2, write, load_fwd_chan(F, c), P, Q);
}

// Backward: group sums [sum g, sum g*(x-mean)] of one channel -> dbeta, dgamma
// (group sums, identical on every rank: batchnorm.py:203) and the dx coefficient table
// dx = A*g + B*x + Cc with A = gamma/sqrt(var+eps) (the backward state's eps,
// batchnorm.py:205), B = -A*inv_std*dgamma/m, Cc = -A*dbeta/m - B*mean, plus the
// forward's affine P/Q for the ReLU mask.
struct BwdFinal {
  const double* saved;
  const float* gamma;
  const float* beta;
  double eps;
  int relu;
  double* A;  // coefficient table (null when the caller keeps the coefficients)
  double* B;
  double* Cc;
  double* P;
  double* Q;
  float* dgamma;  // may be null
  float* dbeta;
  unsigned* status;
  uint32_t C;
};

struct DxCoef {
  double A, B, Cc, P, Q;
};

// Per-channel inputs of the backward finisher (prefetchable).
struct BwdChan {
  double mean, var, inv_std, m;
  float gamma, beta;
};

__device__ __forceinline__ BwdChan load_bwd_chan(const BwdFinal& F, uint32_t c) {
  const uint32_t C = F.C;
  BwdChan v;
  v.mean = F.saved[c];
  v.var = F.saved[C + c];
  v.inv_std = F.saved[2 * C + c];
  v.m = F.saved[3 * C];
  v.gamma = F.gamma[c];
  v.beta = F.relu ? F.beta[c] : 0.f;
  return v;
}

__device__ __forceinline__ void load_bwd_chan_async(const BwdFinal& F, uint32_t c, BwdChan* d) {
  const uint32_t C = F.C;
  cp_async8(&d->mean, F.saved + c);
  cp_async8(&d->var, F.saved + C + c);
  cp_async8(&d->inv_std, F.saved + 2 * C + c);
  cp_async8(&d->m, F.saved + 3 * C);
  cp_async4(&d->gamma, F.gamma + c);
  if (F.relu) cp_async4(&d->beta, F.beta + c);
  else d->beta = 0.f;
}

__device__ __forceinline__ DxCoef finalize_bwd_channel(const BwdFinal& F, uint32_t c, double sdy,
                                                       double sdyx, bool write,
                                                       const BwdChan& v) {
  const double mean = v.mean;
  const double inv_std = v.inv_std;
  const double m = v.m;
  const double dbeta = sdy;
  const double dgamma = sdyx * inv_std;
  const double gam = (double)v.gamma;
  DxCoef k;
  k.A = gam / sqrt(v.var + F.eps);
  k.B = -k.A * inv_std * (dgamma / m);
  k.Cc = -k.A * (dbeta / m) - k.B * mean;
  k.P = k.Q = 0.0;
  if (F.relu) affine_coeffs(mean, inv_std, gam, (double)v.beta, k.P, k.Q);
  if (F.A) {
    F.A[c] = k.A;
    F.B[c] = k.B;
    F.Cc[c] = k.Cc;
    F.P[c] = k.P;
    F.Q[c] = k.Q;
  }
  if (write) {
    if (F.dgamma) F.dgamma[c] = (float)dgamma;
    if (F.dbeta) F.dbeta[c] = (float)dbeta;
    if (F.status && (!isfinite(dbeta) || !isfinite(dgamma)))
      atomicOr(F.status, CGBN_STATUS_NONFINITE);
  }
  return k;
}

__device__ __forceinline__ DxCoef finalize_bwd_channel(const BwdFinal& F, uint32_t c, double sdy,
                                                       double sdyx, bool write) {
  return finalize_bwd_channel(F, c, sdy, sdyx, write, load_bwd_chan(F, c));
}

// ----------------------------------------------------------------------------------
// Reduction ops: per-channel fp64 sums of two quantities.

enum FinishMode { kPartial = 0, kRawSums = 1, kLocalFinal = 2, kSumSq = 3 };

// Forward statistics: sums of d = x - K (K = first element of the channel on this rank,
// the same for every CTA of the channel; d is exact in fp64) -> (mean, M2, count).
template <class T, int VM>
struct StatsOp {
  static constexpr int kVec = VM;
  static constexpr int VEC = vec_of(VM);
  static constexpr int kIn = 1;
  using Elem = T;
  const T* __restrict__ x;
  double K;
  bool shift;
  const double* __restrict__ ksum;    // kSumSq: shift by the group mean ksum[c] / *kcount
  const double* __restrict__ kcount;
  int mode;                   // FinishMode
  double* __restrict__ out2;  // kRawSums: sum_sq destination (may be null)
  FwdFinal F;                 // kLocalFinal
  struct Regs { Vec<T, VEC> v; uint32_t m; };
  struct Init { double K; };
  __device__ __forceinline__ void init(const Geom& g, uint32_t c) {
    if (ksum) K = ksum[c] / kcount[0];
    else K = shift ? (double)ld1(x + (size_t)c * g.HW) : 0.0;
  }
  __device__ __forceinline__ Init get_init() const { return Init{K}; }
  __device__ __forceinline__ void set_init(const Init& i) { K = i.K; }
  // per-channel finisher inputs, loaded early to overlap the data stream
  using Pre = FwdChan;
  __device__ __forceinline__ Pre prefetch(uint32_t c) const {
    return mode == kLocalFinal ? load_fwd_chan(F, c) : FwdChan{0.f, 0.f, 0.f, 0.f};
  }
  __device__ __forceinline__ void prefetch_async(uint32_t c, Pre* d) const {
    if (mode == kLocalFinal) load_fwd_chan_async(F, c, d);
  }
  __device__ __forceinline__ void load(const Geom& g, const Cursor& k, Regs& r) const {
    const uint32_t off = unit_addr<VM>(g, k, r.m);
    if (!masked_vm(VM) || r.m) r.v.load(x + off);
  }
  __device__ __forceinline__ void acc(const Regs& r, double& a, double& b) const {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      if (masked_vm(VM) && !((r.m >> k) & 1u)) continue;
      const double d = (double)r.v.get(k) - K;
      a += d;
      b = __fma_rn(d, d, b);
    }
  }
  __device__ __forceinline__ void finish(const Geom& g, uint32_t c, double S1, double S2,
                                         double* __restrict__ out) const {
    finish(g, c, S1, S2, out, prefetch(c));
  }
  __device__ __forceinline__ void finish(const Geom& g, uint32_t c, double S1, double S2,
                                         double* __restrict__ out, const Pre& pre) const {
    const double n = g.count;
    if (mode == kRawSums) {
      out[c] = S1;
      if (out2) out2[c] = S2;
      return;
    }
    if (mode == kSumSq) {  // sum of (x - group mean)^2 (reference two-pass, batchnorm.py:128-129)
      out[c] = S2;
      return;
    }
    const double mean = K + S1 / n;
    const double M2 = fmax(S2 - S1 * (S1 / n), 0.0);
    if (mode == kPartial) {
      out[c] = mean;
      out[g.C + c] = M2;
      if (c == 0) out[2 * g.C] = n;
    } else {
      double P, Q;
      finalize_fwd_channel(F, c, n, mean, M2, true, pre, P, Q);
    }
  }
};

// Backward: g = dy (ReLU-masked when the forward fused a ReLU); fp64 sums of g and
// g*(x - mean).
template <class T, int VM, bool RELU>
struct BwdOp {
  static constexpr int kVec = VM;
  static constexpr int VEC = vec_of(VM);
  static constexpr int kIn = 2;
  using Elem = T;
  const T* __restrict__ dy;
  const T* __restrict__ x;
  const double* __restrict__ saved;
  const float* __restrict__ gamma;
  const float* __restrict__ beta;
  double mean, P, Q;
  int mode;    // kPartial or kLocalFinal
  BwdFinal F;  // kLocalFinal
  struct Regs { Vec<T, VEC> g, x; uint32_t m; };
  struct Init { double mean; };  // finish() needs no per-channel state
  __device__ __forceinline__ void init(const Geom& g, uint32_t c) {
    mean = saved[c];
    const double inv_std = saved[2 * g.C + c];
    if (RELU) affine_coeffs(mean, inv_std, (double)gamma[c], (double)beta[c], P, Q);
  }
  __device__ __forceinline__ Init get_init() const { return Init{mean}; }
  __device__ __forceinline__ void set_init(const Init& i) { mean = i.mean; }
  using Pre = BwdChan;
  __device__ __forceinline__ void prefetch_async(uint32_t c, Pre* d) const {
    if (mode == kLocalFinal) load_bwd_chan_async(F, c, d);
  }
  __device__ __forceinline__ Pre prefetch(uint32_t c) const {
    if (mode == kLocalFinal) return load_bwd_chan(F, c);
    BwdChan v;
    v.mean = v.var = v.inv_std = v.m = 0.0;
    v.gamma = v.beta = 0.f;
    return v;
  }
  __device__ __forceinline__ void load(const Geom& g, const Cursor& k, Regs& r) const {
    const uint32_t off = unit_addr<VM>(g, k, r.m);
    if (!masked_vm(VM) || r.m) {
      r.g.load(dy + off);
      r.x.load(x + off);
    }
  }
  __device__ __forceinline__ void acc(const Regs& r, double& a, double& b) const {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      if (masked_vm(VM) && !((r.m >> k) & 1u)) continue;
      double gk = (double)r.g.get(k);
      const float xk = r.x.get(k);
      if (RELU && !(bn_out(P, Q, xk) > 0.0)) gk = 0.0;
      a += gk;
      b = __fma_rn(gk, (double)xk - mean, b);
    }
  }
  __device__ __forceinline__ void finish(const Geom& g, uint32_t c, double S1, double S2,
                                         double* __restrict__ out) const {
    finish(g, c, S1, S2, out, prefetch(c));
  }
  __device__ __forceinline__ void finish(const Geom& g, uint32_t c, double S1, double S2,
                                         double* __restrict__ out, const Pre& pre) const {
    if (mode == kPartial) {
      out[c] = S1;
      out[g.C + c] = S2;
    } else {
      finalize_bwd_channel(F, c, S1, S2, true, pre);
    }
  }
};

// Accumulate the strided range in fp64 (two interleaved accumulator pairs).
template <class Op>
__device__ __forceinline__ void reduce_range(const Geom& g, uint32_t c, uint32_t start,
                                             uint32_t end, uint32_t stride, const Op& op,
                                             double& S1, double& S2) {
  constexpr int U = unroll_for<Op::kVec, Op::kIn>();
  constexpr int NA = Op::kIn == 1 ? 2 : 1;  // accumulator pairs (registers vs. DADD chains)
  double a[2] = {0.0, 0.0}, b[2] = {0.0, 0.0};
  strided_rounds<U>(g, c, start, end, stride, op,
                    [&](int u, uint32_t, const typename Op::Regs& r) {
                      op.acc(r, a[u % NA], b[u % NA]);
                    });
  S1 = a[0] + a[1];
  S2 = b[0] + b[1];
}

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

// Forward statistics over rows: the shift K of every channel is the NCHW op's (row 0).
template <class T>
struct StatsRows {
  static constexpr int kU = 8;
  static constexpr int kIn = 1;
  StatsOp<T, 1> base;
  Geom gg;
  struct State { double K[4]; };
  struct Regs { Vec<T, 4> v; };
  __device__ __forceinline__ void init(uint32_t c4, State& s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      StatsOp<T, 1> o = base;
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
};

// Backward sums over rows: [sum g, sum g*(x - mean)] with the forward's ReLU mask.
template <class T, bool RELU>
struct BwdRows {
  static constexpr int kU = 4;
  static constexpr int kIn = 2;
  BwdOp<T, 1, RELU> base;
  Geom gg;
  struct State { double mean[4], P[4], Q[4]; };
  struct Regs { Vec<T, 4> g, x; };
  __device__ __forceinline__ void init(uint32_t c4, State& s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      BwdOp<T, 1, RELU> o = base;
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
    for (uint32_t r = r0 + ro; r < r1; r += U * g.rpp) {
      typename NOp::Regs v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t rr = r + u * g.rpp;
        if (rr < r1) op.load((size_t)rr * g.C4 + c4, v[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r + u * g.rpp < r1) op.acc(s, v[u], a, b);
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
  for (uint32_t i = l; i < nb; i += 32) {
    const double2 t = __ldcg(p + i);
    a += t.x;
    b += t.y;
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (l == 0) {
    Op o = op;
    o.init(g, c);
    o.finish(g, c, a, b, out);
  }
}

// ----------------------------------------------------------------------------------
// Finalize kernels (one thread per channel): group partials -> coefficient tables.

__global__ void k_finalize_fwd(Parts parts, FwdFinal F) {
  pdl_wait();  // inputs may come from the previous kernel (PDL launch)
  pdl_trigger();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= F.C) return;
  double n, mean, M2, P, Q;
  merge_fwd_partials(parts, c, F.C, n, mean, M2);
  finalize_fwd_channel(F, c, n, mean, M2, true, P, Q);
}

__global__ void k_finalize_bwd(Parts parts, BwdFinal F) {
  pdl_wait();  // inputs may come from the previous kernel (PDL launch)
  pdl_trigger();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= F.C) return;
  const uint32_t C = F.C;
  double sdy = parts.p[0][c], sdyx = parts.p[0][C + c];
  for (int r = 1; r < parts.G; ++r) {  // ascending rank fold (collectives.py:293-295)
    sdy += parts.p[r][c];
    sdyx += parts.p[r][C + c];
  }
  finalize_bwd_channel(F, c, sdy, sdyx, true);
}

// Eval (batchnorm.py:158-166) and x_hat coefficient tables.
// Reference-literal statistics (batchnorm.py:119-132): group sums [sum | sq | m] ->
// mean = sum/m, var = sq/m (two-pass: sq = sum (x - mean)^2) or max(sq/m - mean^2, 0)
// (one-pass: sq = sum x^2), then the forward finisher.
__global__ void k_finalize_sums(const double* __restrict__ sum, const double* __restrict__ sq,
                                const double* __restrict__ count, int centered, FwdFinal F) {
  pdl_wait();
  pdl_trigger();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= F.C) return;
  const double m = count[0];
  const double mean = sum[c] / m;
  const double var = centered ? sq[c] / m : fmax(sq[c] / m - mean * mean, 0.0);
  double P, Q;
  finalize_fwd_channel_var(F, c, m, mean, var, true, load_fwd_chan(F, c), P, Q);
}

__global__ void k_coef_eval(const float* gamma, const float* beta, const float* rmean,
                            const float* rvar, double eps, double* P, double* Q, uint32_t C) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double inv_std = 1.0 / sqrt((double)rvar[c] + eps);
  affine_coeffs((double)rmean[c], inv_std, (double)gamma[c], (double)beta[c], P[c], Q[c]);
}

__global__ void k_coef_xhat(const double* saved, double* P, double* Q, uint32_t C) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  affine_coeffs(saved[c], saved[2 * C + c], 1.0, 0.0, P[c], Q[c]);
}

// ----------------------------------------------------------------------------------
// Memory-order elementwise kernels: grid-stride over the whole tensor in float4 units.
// Channel of element e: NCHW (e / HW) % C, NHWC and 2-D e % C. CM (channel mode):
// 0 = NCHW with HW % 4 == 0 (one channel per float4), 1 = NCHW per element,
// 2 = NHWC / 2-D per element.

struct EwGeom {
  uint32_t C, HW;
  uint32_t n4;    // E / UE: 16-byte units (UE = 4 fp32 or 8 bf16 / fp16 elements)
  uint32_t tail;  // E % UE
  FastDiv dhw, dc;
  uint32_t rev;   // 1: sweep from the end of the tensor (LRU-friendly after a reduction)
};

__device__ __forceinline__ uint32_t ew_unit(const EwGeom& g, uint32_t j) {
  return g.rev ? g.n4 - 1 - j : j;
}

// Channel of element e. CM 0: NCHW with HW % UE == 0 (one channel per unit); 1: NCHW any
// HW; 2: NHWC / 2-D; 3: NHWC / 2-D with C % UE == 0 (unit = UE consecutive channels).
template <int CM>
__device__ __forceinline__ uint32_t chan_of(const EwGeom& g, uint32_t e) {
  if (CM >= 2) return e - g.dc.div(e) * g.C;
  const uint32_t p = g.dhw.div(e);
  return p - g.dc.div(p) * g.C;
}

// Channels of the 4 elements starting at element e (e % 4 == 0).
template <int CM>
__device__ __forceinline__ void chan4(const EwGeom& g, uint32_t e, uint32_t (&c)[4]) {
  if constexpr (CM == 3) {
    c[0] = e - g.dc.div(e) * g.C;
    c[1] = c[0] + 1;
    c[2] = c[0] + 2;
    c[3] = c[0] + 3;
  } else if constexpr (CM == 0) {
    c[0] = c[1] = c[2] = c[3] = chan_of<0>(g, e);
  } else if constexpr (CM == 1) {
    // odd planes: one division for the chunk, then walk across plane boundaries
    const uint32_t p = g.dhw.div(e);
    uint32_t r = e - p * g.HW;
    uint32_t ch = p - g.dc.div(p) * g.C;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      c[k] = ch;
      if (++r == g.HW) {
        r = 0;
        ch = ch + 1 == g.C ? 0 : ch + 1;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = chan_of<CM>(g, e + k);
  }
}

template <int CM>
__device__ __forceinline__ void ew_coef(const double* __restrict__ T, const uint32_t (&c)[4],
                                        double (&t)[4]) {
  if constexpr (CM == 3) {  // 32-byte aligned: c[0] % 4 == 0 and the table is 16-aligned
    const double2 a = __ldg(reinterpret_cast<const double2*>(T + c[0]));
    const double2 b = __ldg(reinterpret_cast<const double2*>(T + c[0] + 2));
    t[0] = a.x; t[1] = a.y; t[2] = b.x; t[3] = b.y;
  } else if constexpr (CM == 0) {
    t[0] = t[1] = t[2] = t[3] = __ldg(T + c[0]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = __ldg(T + c[k]);
  }
}

#ifndef CGBN_EWU
#define CGBN_EWU 2
#endif
constexpr int kEwU = CGBN_EWU;  // 16-byte units per elementwise thread (one round): 2 measured best of 1/2/4/8 (ResNet-50 79.3% -> 82.0% of HBM vs 4)

template <class T>
constexpr int ew_ue() { return 16 / (int)sizeof(T); }

template <class T, bool RELU, int CM>
__global__ void __launch_bounds__(kThreads)
k_ew_affine(EwGeom g, const T* __restrict__ x, T* __restrict__ y,
            const double* __restrict__ P, const double* __restrict__ Q) {
  constexpr int UE = ew_ue<T>();
  pdl_trigger();  // the next reduction may launch and wait
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  Vec<T, UE> v[kEwU];
  auto load = [&](uint32_t i0) {
#pragma unroll
    for (int u = 0; u < kEwU; ++u)
      if (i0 + u * stride < g.n4) v[u].load(x + (size_t)UE * ew_unit(g, i0 + u * stride));
  };
  load(i);    // x is not written by the kernel we may overlap with
  pdl_wait();  // the coefficient table is
  for (; i < g.n4; i += kEwU * stride) {
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const uint32_t j = i + u * stride;
      if (j >= g.n4) continue;
      const uint32_t jm = ew_unit(g, j);
      double o[UE];
#pragma unroll
      for (int h = 0; h < UE; h += 4) {
        uint32_t c[4];
        chan4<CM>(g, UE * jm + h, c);
        double p[4], q[4];
        ew_coef<CM>(P, c, p);
        ew_coef<CM>(Q, c, q);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double t = __fma_rn(p[k], (double)v[u].get(h + k), q[k]);
          if (RELU) t = t > 0.0 ? t : 0.0;
          o[h + k] = t;
        }
      }
      stv<T, UE>(y + (size_t)UE * jm, o);
    }
    load(i + kEwU * stride);
  }
  if (blockIdx.x == 0 && threadIdx.x < g.tail) {
    const uint32_t e = UE * g.n4 + threadIdx.x;
    const uint32_t c = CM >= 2 ? chan_of<2>(g, e) : chan_of<1>(g, e);
    double t = __fma_rn(P[c], (double)ld1(x + e), Q[c]);
    if (RELU) t = t > 0.0 ? t : 0.0;
    st1(y + e, t);
  }
}

template <class T, bool RELU, int CM>
__global__ void __launch_bounds__(kThreads)
k_ew_dx(EwGeom g, const T* __restrict__ dy, const T* __restrict__ x, T* __restrict__ dx,
        const double* __restrict__ A, const double* __restrict__ B,
        const double* __restrict__ Cc, const double* __restrict__ P,
        const double* __restrict__ Q) {
  constexpr int UE = ew_ue<T>();
  pdl_trigger();  // the next reduction may launch and wait
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  Vec<T, UE> gv[kEwU], xv[kEwU];
  auto load = [&](uint32_t i0) {
#pragma unroll
    for (int u = 0; u < kEwU; ++u)
      if (i0 + u * stride < g.n4) {
        const size_t off = (size_t)UE * ew_unit(g, i0 + u * stride);
        gv[u].load(dy + off);
        xv[u].load(x + off);
      }
  };
  load(i);    // dy and x are not written by the kernel we may overlap with
  pdl_wait();  // the coefficient tables are
  for (; i < g.n4; i += kEwU * stride) {
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const uint32_t j = i + u * stride;
      if (j >= g.n4) continue;
      const uint32_t jm = ew_unit(g, j);
      double o[UE];
#pragma unroll
      for (int h = 0; h < UE; h += 4) {
        uint32_t c[4];
        chan4<CM>(g, UE * jm + h, c);
        double a[4], b[4], cc[4], p[4] = {0.0, 0.0, 0.0, 0.0}, q[4] = {0.0, 0.0, 0.0, 0.0};
        ew_coef<CM>(A, c, a);
        ew_coef<CM>(B, c, b);
        ew_coef<CM>(Cc, c, cc);
        if (RELU) {
          ew_coef<CM>(P, c, p);
          ew_coef<CM>(Q, c, q);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double gk = (double)gv[u].get(h + k);
          const float xk = xv[u].get(h + k);
          if (RELU && !(bn_out(p[k], q[k], xk) > 0.0)) gk = 0.0;
          o[h + k] = __fma_rn(a[k], gk, __fma_rn(b[k], (double)xk, cc[k]));
        }
      }
      stv<T, UE>(dx + (size_t)UE * jm, o);
    }
    load(i + kEwU * stride);
  }
  if (blockIdx.x == 0 && threadIdx.x < g.tail) {
    const uint32_t e = UE * g.n4 + threadIdx.x;
    const uint32_t c = CM >= 2 ? chan_of<2>(g, e) : chan_of<1>(g, e);
    double gk = (double)ld1(dy + e);
    const float xe = ld1(x + e);
    if (RELU && !(bn_out(P[c], Q[c], xe) > 0.0)) gk = 0.0;
    st1(dx + e, __fma_rn(A[c], gk, __fma_rn(B[c], (double)xe, Cc[c])));
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
#include "cgbn_fused.cuh"
#include "cgbn_p2p.cuh"

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

// Workspace: tickets + barrier words | (C + max grid) double2 per-CTA partial slots |
// coefficient table (5 x C doubles: P, Q, A, B, Cc).
// Row reductions (NHWC / 2-D, C % 4 == 0): rows per block >= 32 keeps the partial
// slots (nb * C double2) under 1/8 of the activation bytes.
bool rows_layout(int64_t C, int64_t HW, int layout) {
  return (layout == CGBN_LAYOUT_NHWC || HW == 1) && C % 4 == 0 && !getenv("CGBN_NO_ROWS");
}

NGeom rows_geom(int64_t N, int64_t C, int64_t HW, int64_t ctas) {
  NGeom g;
  g.M = (uint32_t)(N * HW);
  g.C = (uint32_t)C;
  g.C4 = (uint32_t)(C / 4);
  g.CS4 = g.C4 < (uint32_t)kThreads ? g.C4 : (uint32_t)kThreads;
  g.rpp = (uint32_t)kThreads / g.CS4;
  g.nslices = (g.C4 + g.CS4 - 1) / g.CS4;
  int64_t nb = ceil_div(ctas, (int64_t)g.nslices);
  const int64_t cap = (int64_t)g.M / 32;
  if (nb > cap) nb = cap;
  if (nb > (int64_t)g.M) nb = g.M;
  g.nb = (uint32_t)(nb < 1 ? 1 : nb);
  return g;
}

size_t slots_bytes(int64_t N, int64_t C, int64_t HW, int layout, int sms) {
  size_t n = (size_t)C + (size_t)sms * kMaxCtasPerSm;
  if (rows_layout(C, HW, layout)) {
    const NGeom g = rows_geom(N, C, HW, (int64_t)sms * kMaxCtasPerSm);
    const size_t r = (size_t)g.nb * (size_t)C;
    if (r > n) n = r;
  }
  return n * sizeof(double2);
}
size_t ws_bytes_for(int64_t N, int64_t C, int64_t HW, int layout, int sms) {
  return kTicketBytes + slots_bytes(N, C, HW, layout, sms) + 5 * (size_t)C * sizeof(double);
}

struct WsView {
  unsigned* tickets;
  unsigned* bar;
  double2* slots;
  double* P;
  double* Q;
  double* A;
  double* B;
  double* Cc;
};

int ws_view(void* ws, size_t ws_bytes, int64_t N, int64_t C, int64_t HW, int layout,
            WsView* v) {
  const int sms = num_sms_cached();
  const size_t need = ws_bytes_for(N, C, HW, layout, sms);
  if (!ws || ws_bytes < need)
    return set_error(CGBN_ERR_INVALID, "workspace too small: need %zu bytes, got %zu", need,
                     ws_bytes);
  if (reinterpret_cast<uintptr_t>(ws) % 16)
    return set_error(CGBN_ERR_INVALID, "workspace must be 16-byte aligned");
  char* b = reinterpret_cast<char*>(ws);
  v->tickets = reinterpret_cast<unsigned*>(b);
  v->bar = v->tickets + kTicketWords;
  v->slots = reinterpret_cast<double2*>(b + kTicketBytes);
  double* coef =
      reinterpret_cast<double*>(b + kTicketBytes + slots_bytes(N, C, HW, layout, sms));
  v->P = coef;
  v->Q = coef + C;
  v->A = coef + 2 * C;
  v->B = coef + 3 * C;
  v->Cc = coef + 4 * C;
  return CGBN_OK;
}

// Per-(kernel, device) caches. Keyed by the kernel's address: kernels of one signature
// share a function-pointer type, so a per-template static would alias them.
std::mutex g_cache_mu;
std::map<std::pair<const void*, int>, int> g_occ_cache;
std::map<std::pair<const void*, int>, bool> g_smem_done;

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

template <class K>
void smem_optin(K kernel, size_t smem_bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_smem_done.count(key)) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  g_smem_done[key] = true;
}

// CGBN_PATH=tma selects the TMA streaming statistics reductions (A/B measurement);
// CGBN_PATH=reg disables every TMA / cp.async variant.
int path_override() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CGBN_PATH");
    v = (e && !strcmp(e, "tma")) ? 1 : (e && !strcmp(e, "reg")) ? 2 : 0;
  }
  return v;
}

// The ABI's `layout` argument carries the activation dtype in bits 4..7
// (CGBN_ACT_F32 / CGBN_ACT_BF16 / CGBN_ACT_F16, include/cgbn.h).
int split_fmt(int* layout, int* act) {
  const int f = *layout;
  *act = (f >> 4) & 0xF;
  *layout = f & 0xF;
  if (f & ~0xFF) return set_error(CGBN_ERR_INVALID, "unknown layout/format bits 0x%x", f);
  if (*act > 2) return set_error(CGBN_ERR_INVALID, "unknown activation dtype %d", *act);
  return CGBN_OK;
}

int act_bytes(int act) { return act == 0 ? 4 : 2; }

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
  if (N * C * HW >= (1ll << 32))
    return set_error(CGBN_ERR_INVALID, "tensor of %lld elements exceeds 2^32",
                     (long long)(N * C * HW));
  return CGBN_OK;
}

struct Plan {
  int act;  // activation dtype (0 fp32, 1 bf16, 2 fp16)
  int vec;
  bool rows;  // NHWC / 2-D with C % 4 == 0: row reduction (k_reduce_rows + k_fold_rows)
  bool team;
  bool ct;   // NCHW: cluster-team reduction (k_reduce_ct) when it fills the GPU
  bool tma;  // NCHW, HW % 4 == 0, 16-byte aligned, CGBN_PATH=tma
  Geom g;
  tma::TGeom tg;
  int64_t elems;
};

// Reduction plan. `ptrs` are every activation pointer the kernel touches; the vector
// width is the widest one that divides the plane length and the alignment of all.
int make_plan(int64_t N, int64_t C, int64_t HW, int layout, int act, const void* const* ptrs,
              int nptr, Plan* out) {
  int rc = validate_shape(N, C, HW, layout);
  if (rc) return rc;
  int64_t planeN = N, planeHW = HW;
  if (layout == CGBN_LAYOUT_NHWC) { planeN = N * HW; planeHW = 1; }
  uintptr_t align = 0;
  for (int k = 0; k < nptr; ++k) align |= (uintptr_t)ptrs[k];
  const int es = act_bytes(act);
  const int64_t vmax = 16 / es;  // elements per 16-byte unit
  const int64_t E = N * C * HW;
  int vec = 1;
  if (planeHW % vmax == 0 && (align % 16) == 0) vec = (int)vmax;
  else if (es == 2 && planeHW % 4 == 0 && (align % 8) == 0)
    vec = 4;  // exact 8-byte units: faster than masked 16-byte covers (bf16 14x14 stats 4.4 -> 3.3 us)
  else if (layout == CGBN_LAYOUT_NCHW && HW >= 16 && (align % 16) == 0 && E % vmax == 0 &&
           E + 2 * vmax < (1ll << 32) && !getenv("CGBN_NO_MASKED"))
    vec = es == 4 ? 5 : 9;  // masked 16-byte cover of odd planes (never leaves the tensor)
  else if (es == 2 && planeHW % 4 == 0 && (align % 8) == 0) vec = 4;
  else if (planeHW % 2 == 0 && (align % (2 * es)) == 0) vec = 2;
  const int V = vec_of(vec);
  Geom g;
  g.C = (uint32_t)C;
  g.HW = (uint32_t)planeHW;
  g.HWv = (uint32_t)(masked_vm(vec) ? (planeHW + V - 1) / V + 1 : planeHW / vec);
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
  out->act = act;
  out->vec = vec;
  out->team = g.Lv <= kTeamMaxLv;
  out->ct = layout == CGBN_LAYOUT_NCHW && !getenv("CGBN_NO_CT");
  out->rows = rows_layout(C, HW, layout) && (align % 16) == 0;
  out->g = g;
  out->elems = N * C * HW;
  out->tma = act == 0 && layout == CGBN_LAYOUT_NCHW && HW % 4 == 0 && (align % 16) == 0 &&
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

template <class K>
unsigned flat_grid(K kernel, const Plan& pl) {
  int64_t grid = resident_ctas(kernel);
  const int64_t want = ceil_div(pl.elems, kMinElemsPerCta);
  if (want < grid) grid = want;
  return (unsigned)(grid < 1 ? 1 : grid);
}

template <class K>
unsigned team_grid(K kernel, const Plan& pl) {
  const int64_t cpt = kThreads >> pl.g.tpc_log2;
  int64_t grid = ceil_div(pl.g.C, cpt);
  const int64_t res = resident_ctas(kernel);
  if (grid > res) grid = res;
  return (unsigned)(grid < 1 ? 1 : grid);
}

// Launch with programmatic dependent launch allowed (see pdl_trigger / pdl_wait).
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("CGBN_NO_PDL") ? 0 : 1;
  return v == 1;
}

template <class K, class... Args>
void launch_pdl(K kernel, unsigned grid, bool pdl, cudaStream_t st, Args... args) {
  if (!pdl || !pdl_enabled()) {
    kernel<<<grid, kThreads, 0, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Clusters of `kc` CTAs of `kernel` that can be co-resident (cached; 0 if unsupported).
std::map<std::tuple<const void*, int, int>, int> g_cluster_cache;

template <class K>
int64_t cluster_capacity(K kernel, uint32_t kc) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, (int)kc);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cluster_cache.find(key);
    if (it != g_cluster_cache.end()) return (int64_t)it->second * kc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kc * 64);
  cfg.blockDim = dim3(kThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cluster_cache[key] = n;
  return (int64_t)n * kc;
}

struct CtCfg {
  int tl;
  uint32_t kc, grid;
};

// Cluster-team configuration, from the lab sweep (tools/flatlab.cu "sweep", B200,
// ResNet-50 shapes). Cluster sizes are powers of two; U = vector loads of each input a
// thread keeps in flight per round.
//  - latency-bound (the whole stream fits in one round of the resident slots): the
//    fewest CTAs whose threads need a single round, unclustered first (a cluster costs
//    ~1 us of barrier + DSMEM at these sizes);
//  - bandwidth-bound: the largest grid that fits in one wave (bytes in flight), then the
//    smaller cluster, then the larger team.
// Returns false when nothing fills a quarter of the slots (tiny C: the flat kernel
// spreads one channel over more CTAs than a cluster holds).
template <class Op>
int64_t ct_cluster_cap(int tl, uint32_t kc) {
  switch (tl) {
    case 8: return cluster_capacity(k_reduce_ct<Op, 8>, kc);
    case 7: return cluster_capacity(k_reduce_ct<Op, 7>, kc);
    case 6: return cluster_capacity(k_reduce_ct<Op, 6>, kc);
    default: return cluster_capacity(k_reduce_ct<Op, 5>, kc);
  }
}

template <class Op>
bool choose_ct(const Plan& pl, CtCfg* cfg) {
  constexpr int64_t U = unroll_for<Op::kVec, Op::kIn>();
  const int64_t slots = resident_ctas(k_reduce_ct<Op, 8>);
  const int64_t C = pl.g.C, Lv = pl.g.Lv;
  bool latency_bound = C * Lv <= slots * kThreads * U;
  int64_t best_n = 0;
  double best = 1e30;
again:
  for (uint32_t kc = 1; kc <= 8; kc *= 2) {
    for (int tl = 8; tl >= 5; --tl) {
      const int64_t tpc = 1 << tl;
      if (kc > 1 && Lv / kc < tpc) continue;  // every thread keeps >= 1 unit
      const int64_t n = ceil_div(C, (int64_t)kThreads >> tl) * kc;
      if (n > slots) continue;
      const int64_t units = ceil_div(Lv, (int64_t)kc * tpc);
      double score;
      if (latency_bound) {
        if (units > U) continue;
        score = (kc > 1 ? 1e6 : 0.0) + (double)n;  // unclustered, then fewest CTAs
      } else {
        score = -(double)n * 16.0 + kc;  // most CTAs, then smallest cluster
      }
      if (score >= best) continue;
      if (kc > 1 && n > ct_cluster_cap<Op>(tl, kc)) continue;
      best = score;
      best_n = n;
      cfg->tl = tl;
      cfg->kc = kc;
      cfg->grid = (uint32_t)n;
    }
  }
  if (latency_bound && best_n == 0) {
    latency_bound = false;  // no single-round configuration: rank by fill instead
    goto again;
  }
  if (const char* f = getenv("CGBN_CT_FORCE")) {  // "tl,kc" (experiments only)
    int tl = 0, kc = 0;
    if (sscanf(f, "%d,%d", &tl, &kc) == 2 && tl >= 5 && tl <= 8 && kc >= 1 && kc <= 8) {
      cfg->tl = tl;
      cfg->kc = (uint32_t)kc;
      cfg->grid = (uint32_t)(ceil_div(C, (int64_t)kThreads >> tl) * kc);
      best_n = cfg->grid;
    }
  }
  if (getenv("CGBN_DEBUG_PLAN"))
    fprintf(stderr, "[cgbn] ct C=%lld Lv=%lld in=%d slots=%lld %s -> tl=%d kc=%u grid=%lld\n",
            (long long)C, (long long)Lv, Op::kIn, (long long)slots,
            latency_bound ? "latency" : "bandwidth", best_n ? cfg->tl : -1, best_n ? cfg->kc : 0,
            (long long)best_n);
  if (best_n == 0 && ceil_div(C, kThreads >> 5) > slots) {
    // very wide layers: 8 channels per CTA, CTAs loop over channel groups
    cfg->tl = 5;
    cfg->kc = 1;
    cfg->grid = (uint32_t)slots;
    return true;
  }
  return best_n * 4 >= slots;
}

template <class Op, int TL>
int launch_ct(Geom g, const Op& op, double* out, uint32_t kc, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (kc > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = kc;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_reduce_ct<Op, TL>, g, op, out);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cluster reduction launch failed: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

template <class Op>
int launch_reduce(const Plan& pl, const Op& op, double* out, const WsView& w, cudaStream_t st) {
  Geom g = pl.g;
  CtCfg cc;
  if (pl.ct && choose_ct<Op>(pl, &cc)) {
    g.grid = cc.grid;
    switch (cc.tl) {
      case 8: return launch_ct<Op, 8>(g, op, out, cc.kc, st);
      case 7: return launch_ct<Op, 7>(g, op, out, cc.kc, st);
      case 6: return launch_ct<Op, 6>(g, op, out, cc.kc, st);
      default: return launch_ct<Op, 5>(g, op, out, cc.kc, st);
    }
  }
  if (pl.team) {
    g.grid = team_grid(k_reduce_team<Op>, pl);
    launch_pdl(k_reduce_team<Op>, g.grid, true, st, g, op, out);
  } else {
    g.grid = flat_grid(k_reduce_flat<Op>, pl);
    launch_pdl(k_reduce_flat<Op>, g.grid, true, st, g, op, out, w.slots, w.tickets);
  }
  return CGBN_OK;
}

template <class TOp>
int launch_tma_reduce(const Plan& pl, const TOp& op, double* out, const WsView& w,
                      cudaStream_t st) {
  smem_optin(tma::k_tma_reduce<TOp>, tma::kSmemBytes);
  tma::k_tma_reduce<TOp><<<pl.tg.grid, tma::kThreadsTma, tma::kSmemBytes, st>>>(
      pl.tg, op, out, w.slots, w.tickets);
  return CGBN_OK;
}

// Row reduction (NHWC / 2-D): k_reduce_rows -> k_fold_rows (finisher of `op`).
template <class NOp, class Op>
int launch_rows(const Plan& pl, const NOp& nop, const Op& op, double* out, const WsView& w,
                cudaStream_t st) {
  const int64_t N = 1, HW = pl.g.count;  // rows = N*HW of the original geometry
  const NGeom ng = rows_geom(N, pl.g.C, HW, resident_ctas(k_reduce_rows<NOp>));
  const unsigned grid = ng.nslices * ng.nb;
  launch_pdl(k_reduce_rows<NOp>, grid, true, st, ng, nop, w.slots);
  Geom g = pl.g;
  const unsigned fgrid = (unsigned)ceil_div((int64_t)pl.g.C * 32, kThreads);
  launch_pdl(k_fold_rows<Op>, fgrid, true, st, g, op, (const double2*)w.slots, ng.nb, out);
  return CGBN_OK;
}

// Forward statistics in mode kPartial / kRawSums / kLocalFinal / kSumSq.
template <class T, int VEC>
int run_stats(const Plan& pl, const void* xv, bool shift, int mode, double* out, double* out2,
              const FwdFinal* F, const WsView& w, cudaStream_t st, const double* ksum,
              const double* kcount) {
  const T* x = static_cast<const T*>(xv);
  if constexpr (std::is_same<T, float>::value && VEC == 4) {
    if (pl.tma && shift && mode == kPartial) {
      tma::TmaStats op;
      op.x = x;
      op.K = 0.0;
      return launch_tma_reduce(pl, op, out, w, st);
    }
  }
  StatsOp<T, VEC> op;
  op.x = x;
  op.K = 0.0;
  op.shift = shift;
  op.ksum = ksum;
  op.kcount = kcount;
  op.mode = mode;
  op.out2 = out2;
  if (F) op.F = *F;
  if constexpr (VEC == 1) {
    if (pl.rows) {
      StatsRows<T> nop;
      nop.base = op;
      nop.gg = pl.g;
      return launch_rows(pl, nop, op, out, w, st);
    }
  }
  return launch_reduce(pl, op, out, w, st);
}

template <class T, int VEC, bool RELU>
int run_bwd_reduce(const Plan& pl, const void* dyv, const void* xv, const double* saved,
                   const float* gamma, const float* beta, int mode, double* out,
                   const BwdFinal* F, const WsView& w, cudaStream_t st) {
  const T* dy = static_cast<const T*>(dyv);
  const T* x = static_cast<const T*>(xv);
  if constexpr (std::is_same<T, float>::value && VEC == 4) {
    if (pl.tma && mode == kPartial) {
      tma::TmaBwd<RELU> op;
      op.dy = dy;
      op.x = x;
      op.saved = saved;
      op.gamma = gamma;
      op.beta = beta;
      op.mean = op.P = op.Q = 0.0;
      return launch_tma_reduce(pl, op, out, w, st);
    }
  }
  BwdOp<T, VEC, RELU> op;
  op.dy = dy;
  op.x = x;
  op.saved = saved;
  op.gamma = gamma;
  op.beta = beta;
  op.mean = op.P = op.Q = 0.0;
  op.mode = mode;
  if (F) op.F = *F;
  if constexpr (VEC == 1) {
    if (pl.rows) {
      BwdRows<T, RELU> nop;
      nop.base = op;
      nop.gg = pl.g;
      return launch_rows(pl, nop, op, out, w, st);
    }
  }
  return launch_reduce(pl, op, out, w, st);
}

// fp32: vector modes 1, 2, 4, 5 (masked float4); bf16 / fp16: 1, 2, 4, 8, 9 (masked 8).
template <class T>
int dispatch_stats_t(const Plan& pl, const void* x, bool shift, int mode, double* out,
                     double* out2, const FwdFinal* F, const WsView& w, cudaStream_t st,
                     const double* ksum, const double* kcount) {
  if constexpr (sizeof(T) == 4) {
    switch (pl.vec) {
      case 5: return run_stats<T, 5>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 4: return run_stats<T, 4>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 2: return run_stats<T, 2>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      default: return run_stats<T, 1>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
    }
  } else {
    switch (pl.vec) {
      case 9: return run_stats<T, 9>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 8: return run_stats<T, 8>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 4: return run_stats<T, 4>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      case 2: return run_stats<T, 2>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
      default: return run_stats<T, 1>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
    }
  }
}

int dispatch_stats(const Plan& pl, const void* x, bool shift, int mode, double* out,
                   double* out2, const FwdFinal* F, const WsView& w, cudaStream_t st,
                   const double* ksum = nullptr, const double* kcount = nullptr) {
  switch (pl.act) {
    case 1:
      return dispatch_stats_t<__nv_bfloat16>(pl, x, shift, mode, out, out2, F, w, st, ksum,
                                             kcount);
    case 2:
      return dispatch_stats_t<__half>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
    default:
      return dispatch_stats_t<float>(pl, x, shift, mode, out, out2, F, w, st, ksum, kcount);
  }
}

template <class T, bool RELU>
int dispatch_bwd_t(const Plan& pl, const void* dy, const void* x, const double* saved,
                   const float* gamma, const float* beta, int mode, double* out,
                   const BwdFinal* F, const WsView& w, cudaStream_t st) {
  if constexpr (sizeof(T) == 4) {
    switch (pl.vec) {
      case 5: return run_bwd_reduce<T, 5, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 4: return run_bwd_reduce<T, 4, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 2: return run_bwd_reduce<T, 2, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      default:
        return run_bwd_reduce<T, 1, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
    }
  } else {
    switch (pl.vec) {
      case 9: return run_bwd_reduce<T, 9, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 8: return run_bwd_reduce<T, 8, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 4: return run_bwd_reduce<T, 4, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      case 2: return run_bwd_reduce<T, 2, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
      default:
        return run_bwd_reduce<T, 1, RELU>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
    }
  }
}

template <class T>
int dispatch_bwd_r(const Plan& pl, const void* dy, const void* x, const double* saved,
                   const float* gamma, const float* beta, bool relu, int mode, double* out,
                   const BwdFinal* F, const WsView& w, cudaStream_t st) {
  return relu ? dispatch_bwd_t<T, true>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st)
              : dispatch_bwd_t<T, false>(pl, dy, x, saved, gamma, beta, mode, out, F, w, st);
}

int dispatch_bwd_reduce(const Plan& pl, const void* dy, const void* x, const double* saved,
                        const float* gamma, const float* beta, bool relu, int mode, double* out,
                        const BwdFinal* F, const WsView& w, cudaStream_t st) {
  switch (pl.act) {
    case 1:
      return dispatch_bwd_r<__nv_bfloat16>(pl, dy, x, saved, gamma, beta, relu, mode, out, F, w,
                                           st);
    case 2:
      return dispatch_bwd_r<__half>(pl, dy, x, saved, gamma, beta, relu, mode, out, F, w, st);
    default:
      return dispatch_bwd_r<float>(pl, dy, x, saved, gamma, beta, relu, mode, out, F, w, st);
  }
}

// ---- elementwise

struct EwPlan {
  EwGeom g;
  int cm;
  int act;
};

int make_ew(int64_t N, int64_t C, int64_t HW, int layout, int act, const void* const* ptrs,
            int nptr, EwPlan* out) {
  int rc = validate_shape(N, C, HW, layout);
  if (rc) return rc;
  uintptr_t align = 0;
  for (int k = 0; k < nptr; ++k) align |= (uintptr_t)ptrs[k];
  if (align % 16)
    return set_error(CGBN_ERR_INVALID, "activation pointers must be 16-byte aligned");
  const uint64_t E = (uint64_t)N * C * HW;
  const uint32_t UE = 16 / act_bytes(act);  // elements per 16-byte unit
  EwGeom& g = out->g;
  g.C = (uint32_t)C;
  g.HW = (uint32_t)HW;
  g.n4 = (uint32_t)(E / UE);
  g.tail = (uint32_t)(E % UE);
  g.dhw.init((uint32_t)HW);
  g.dc.init((uint32_t)C);
  // Sweep from the end of the tensor: the preceding channel-major reduction read the
  // high-n planes of every channel last, so they are the likeliest L2 hits (measured
  // +1.5% on the ResNet-50 step, up to 7% on the 100 MB layers; CGBN_EW_FORWARD=1 off).
  g.rev = getenv("CGBN_EW_FORWARD") ? 0u : 1u;
  // channel modes work on 4-element chunks of a unit: CM 0 / 3 need HW % 4 / C % 4 only
  (void)UE;
  if (layout == CGBN_LAYOUT_NHWC || HW == 1) out->cm = (C % 4 == 0) ? 3 : 2;
  else out->cm = (HW % 4 == 0) ? 0 : 1;
  out->act = act;
  return CGBN_OK;
}

// One round of kEwU units per thread, not a persistent grid: a copy-like kernel streams
// faster with many short-lived CTAs than with one resident wave that loops (ResNet-50
// step +3%, 100 MB layers 4-6 us faster; CGBN_EW_PERSISTENT=1 restores the resident
// grid for A/B).
template <class K>
unsigned ew_grid(K kernel, const EwPlan& ep) {
  int64_t grid = ceil_div((int64_t)ep.g.n4 + 1, kThreads * kEwU);
  static const bool persistent = getenv("CGBN_EW_PERSISTENT") != nullptr;
  if (persistent) {
    const int64_t res = resident_ctas(kernel);
    if (grid > res) grid = res;
  }
  return (unsigned)(grid < 1 ? 1 : grid);
}

// pdl: the kernel before this launch on `st` is one of ours that does not write x
// (a reduction, finalize or coefficient kernel), so x may be prefetched before the
// dependency wait.
template <class T, bool RELU, int CM>
void launch_ew_affine_t(const EwPlan& ep, const void* x, void* y, const double* P,
                        const double* Q, bool pdl, cudaStream_t st) {
  launch_pdl(k_ew_affine<T, RELU, CM>, ew_grid(k_ew_affine<T, RELU, CM>, ep), pdl, st, ep.g,
             static_cast<const T*>(x), static_cast<T*>(y), P, Q);
}

template <class T, bool RELU>
void launch_ew_affine_r(const EwPlan& ep, int cm, const void* x, void* y, const double* P,
                        const double* Q, bool pdl, cudaStream_t st) {
  if (cm == 0) launch_ew_affine_t<T, RELU, 0>(ep, x, y, P, Q, pdl, st);
  else if (cm == 1) launch_ew_affine_t<T, RELU, 1>(ep, x, y, P, Q, pdl, st);
  else if (cm == 2) launch_ew_affine_t<T, RELU, 2>(ep, x, y, P, Q, pdl, st);
  else launch_ew_affine_t<T, RELU, 3>(ep, x, y, P, Q, pdl, st);
}

template <class T>
void launch_ew_affine_d(const EwPlan& ep, int cm, bool relu, const void* x, void* y,
                        const double* P, const double* Q, bool pdl, cudaStream_t st) {
  if (relu) launch_ew_affine_r<T, true>(ep, cm, x, y, P, Q, pdl, st);
  else launch_ew_affine_r<T, false>(ep, cm, x, y, P, Q, pdl, st);
}

void launch_ew_affine(const EwPlan& ep, bool relu, const void* x, void* y, const double* P,
                      const double* Q, cudaStream_t st, bool pdl = true) {
  int cm = ep.cm;
  if (cm == 3 && (((uintptr_t)P | (uintptr_t)Q) % 16) != 0) cm = 2;  // caller's tables
  if (ep.act == 1) launch_ew_affine_d<__nv_bfloat16>(ep, cm, relu, x, y, P, Q, pdl, st);
  else if (ep.act == 2) launch_ew_affine_d<__half>(ep, cm, relu, x, y, P, Q, pdl, st);
  else launch_ew_affine_d<float>(ep, cm, relu, x, y, P, Q, pdl, st);
}

template <class T, bool RELU, int CM>
void launch_ew_dx_t(const EwPlan& ep, const void* dy, const void* x, void* dx, const WsView& w,
                    cudaStream_t st) {
  launch_pdl(k_ew_dx<T, RELU, CM>, ew_grid(k_ew_dx<T, RELU, CM>, ep), true, st, ep.g,
             static_cast<const T*>(dy), static_cast<const T*>(x), static_cast<T*>(dx),
             (const double*)w.A, (const double*)w.B, (const double*)w.Cc, (const double*)w.P,
             (const double*)w.Q);
}

template <class T, bool RELU>
void launch_ew_dx_r(const EwPlan& ep, const void* dy, const void* x, void* dx, const WsView& w,
                    cudaStream_t st) {
  if (ep.cm == 0) launch_ew_dx_t<T, RELU, 0>(ep, dy, x, dx, w, st);
  else if (ep.cm == 1) launch_ew_dx_t<T, RELU, 1>(ep, dy, x, dx, w, st);
  else if (ep.cm == 2) launch_ew_dx_t<T, RELU, 2>(ep, dy, x, dx, w, st);
  else launch_ew_dx_t<T, RELU, 3>(ep, dy, x, dx, w, st);
}

template <class T>
void launch_ew_dx_d(const EwPlan& ep, bool relu, const void* dy, const void* x, void* dx,
                    const WsView& w, cudaStream_t st) {
  if (relu) launch_ew_dx_r<T, true>(ep, dy, x, dx, w, st);
  else launch_ew_dx_r<T, false>(ep, dy, x, dx, w, st);
}

void launch_ew_dx(const EwPlan& ep, bool relu, const void* dy, const void* x, void* dx,
                  const WsView& w, cudaStream_t st) {
  if (ep.act == 1) launch_ew_dx_d<__nv_bfloat16>(ep, relu, dy, x, dx, w, st);
  else if (ep.act == 2) launch_ew_dx_d<__half>(ep, relu, dy, x, dx, w, st);
  else launch_ew_dx_d<float>(ep, relu, dy, x, dx, w, st);
}

unsigned chan_blocks(int64_t C) { return (unsigned)ceil_div(C, 256); }

FwdFinal make_fwd_final(int64_t C, const float* gamma, const float* beta, double eps,
                        double momentum, float* rm, float* rv, double* saved, unsigned* status,
                        const WsView& w) {
  FwdFinal F;
  F.gamma = gamma; F.beta = beta;
  F.eps = eps; F.momentum = momentum;
  F.rmean = rm; F.rvar = rv;
  F.saved = saved;
  F.P = w.P; F.Q = w.Q;
  F.status = status;
  F.C = (uint32_t)C;
  return F;
}

BwdFinal make_bwd_final(int64_t C, const double* saved, const float* gamma, const float* beta,
                        double eps, bool relu, float* dgamma, float* dbeta, unsigned* status,
                        const WsView& w) {
  BwdFinal F;
  F.saved = saved; F.gamma = gamma; F.beta = beta;
  F.eps = eps;
  F.relu = relu ? 1 : 0;
  F.A = w.A; F.B = w.B; F.Cc = w.Cc; F.P = w.P; F.Q = w.Q;
  F.dgamma = dgamma; F.dbeta = dbeta;
  F.status = status;
  F.C = (uint32_t)C;
  return F;
}

// ---- fused cooperative kernels (cgbn_fused.cuh)

bool fused_plan(int64_t N, int64_t C, int64_t HW, int layout, uintptr_t align, int nin,
                fused::FGeom* fg) {
  if (path_override() == 2 || getenv("CGBN_NO_FUSED")) return false;
  if (layout != CGBN_LAYOUT_NCHW || HW % 4 != 0 || (align % 16) != 0) return false;
  if (validate_shape(N, C, HW, layout) != CGBN_OK) return false;
  const int64_t L = N * HW;
  const int64_t T4 = C * L / 4;
  int64_t grid = ceil_div(T4, 64);
  if (grid > num_sms_cached()) grid = num_sms_cached();
  if (grid < 1) grid = 1;
  const int64_t max_slice = ceil_div(T4, grid) * 4;
  const int64_t cap = (int64_t)(fused::kDataBytes / (4 * nin));
  if (max_slice > cap) return false;
  if (max_slice / L + 2 > fused::kMaxSeg) return false;
  fg->C = (uint32_t)C;
  fg->HW = (uint32_t)HW;
  fg->L = (uint32_t)L;
  fg->grid = (uint32_t)grid;
  fg->T4 = (uint64_t)T4;
  fg->dhw.init((uint32_t)HW);
  fg->count = (double)L;
  return true;
}

// Cooperative grids must never interleave on one device (their grid barriers could
// deadlock): launches from different streams of one process are chained through a
// per-device event. Skipped under stream capture, where a graph replays in order.
std::mutex g_coop_mu;
cudaEvent_t g_coop_last[64] = {nullptr};

template <class K, class... Args>
int launch_cooperative(K kernel, unsigned grid, size_t smem, cudaStream_t st, Args... args) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  const bool chain = cap == cudaStreamCaptureStatusNone && dev >= 0 && dev < 64;
  std::unique_lock<std::mutex> lk(g_coop_mu, std::defer_lock);
  if (chain) {
    lk.lock();
    if (!g_coop_last[dev]) cudaEventCreateWithFlags(&g_coop_last[dev], cudaEventDisableTiming);
    cudaStreamWaitEvent(st, g_coop_last[dev], 0);
  }
  smem_optin(kernel, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(fused::kThreadsF);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (chain) cudaEventRecord(g_coop_last[dev], st);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cooperative launch failed: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

#define CGBN_REQUIRE(cond, ...) \
  do { if (!(cond)) return set_error(CGBN_ERR_INVALID, __VA_ARGS__); } while (0)

#define CGBN_TRY(expr) \
  do { int rc_ = (expr); if (rc_) return rc_; } while (0)

int check_fwd_args(const void* x, const void* y, const float* gamma, const float* beta,
                   const double* saved, double eps, double momentum, const float* running_mean,
                   const float* running_var) {
  CGBN_REQUIRE(x && y && gamma && beta && saved, "forward: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(momentum >= 0.0 && momentum <= 1.0, "momentum must lie in [0, 1], got %g",
               momentum);
  CGBN_REQUIRE((running_mean == nullptr) == (running_var == nullptr),
               "running_mean and running_var must both be set or both be NULL");
  return CGBN_OK;
}

}  // namespace

// ==================================================================================
// C ABI

extern "C" {

int cgbn_abi_version(void) { return CGBN_ABI_VERSION; }

#define CGBN_STR2(x) #x
#define CGBN_STR(x) CGBN_STR2(x)
const char* cgbn_build_info(void) {
  return "cgbn sm_100a; nvcc " CGBN_STR(__CUDACC_VER_MAJOR__) "." CGBN_STR(__CUDACC_VER_MINOR__)
         "; cluster-team / row reductions (fp64) + memory-order elementwise, PDL; fp32 / bf16 / "
         "fp16 activations; fused cooperative and TMA variants opt-in";
}

const char* cgbn_last_error(void) { return g_last_error.c_str(); }

int cgbn_num_sms(void) { return num_sms_cached(); }

size_t cgbn_workspace_bytes(int64_t N, int64_t C, int64_t HW, int layout) {
  int act = 0;
  if (split_fmt(&layout, &act)) return 0;
  if (validate_shape(N, C, HW, layout)) return 0;
  return ws_bytes_for(N, C, HW, layout, num_sms_cached());
}

int cgbn_fwd_stats(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   double* partial, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && partial, "cgbn_fwd_stats: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CGBN_TRY(dispatch_stats(pl, x, true, kPartial, partial, nullptr, nullptr, w, st));
  return check_launch("cgbn_fwd_stats");
}

int cgbn_channel_sum(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                     double* sum, double* sum_sq, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && sum, "cgbn_channel_sum: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  pl.tma = false;
  CGBN_TRY(dispatch_stats(pl, x, false, kRawSums, sum, sum_sq, nullptr, w, st));
  return check_launch("cgbn_channel_sum");
}

int cgbn_centered_sumsq(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* sum, const double* count, double* out, void* ws,
                        size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && sum && count && out, "cgbn_centered_sumsq: NULL pointer");
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  pl.tma = false;
  CGBN_TRY(dispatch_stats(pl, x, false, kSumSq, out, nullptr, nullptr, w, st, sum, count));
  return check_launch("cgbn_centered_sumsq");
}

int cgbn_fwd_normalize_sums(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                            const double* sum, const double* sq, const double* count,
                            int centered, const float* gamma, const float* beta, double eps,
                            double momentum, float* running_mean, float* running_var,
                            double* saved, int relu, void* y, unsigned* status, void* ws,
                            size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  CGBN_REQUIRE(sum && sq && count, "cgbn_fwd_normalize_sums: NULL pointer");
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  launch_pdl(k_finalize_sums, chan_blocks(C), true, st, sum, sq, count, centered ? 1 : 0, F);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st);
  return check_launch("cgbn_fwd_normalize_sums");
}

int cgbn_fwd_normalize(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                       const double* const* partials, int G, const float* gamma,
                       const float* beta, double eps, double momentum, float* running_mean,
                       float* running_var, double* saved, int relu, void* y, unsigned* status,
                       void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  Parts parts;
  CGBN_TRY(fill_parts(&parts, partials, G));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  launch_pdl(k_finalize_fwd, chan_blocks(C), true, st, parts, F);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st);
  return check_launch("cgbn_fwd_normalize");
}

int cgbn_fwd_train_local(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                         const float* gamma, const float* beta, double eps, double momentum,
                         float* running_mean, float* running_var, double* saved, int relu,
                         void* y, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  const void* ptrs[] = {x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 1, &pl));
  const void* eptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, eptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  pl.tma = false;  // the TMA reductions only emit partials
  CGBN_TRY(dispatch_stats(pl, x, true, kLocalFinal, nullptr, nullptr, &F, w, st));
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st);
  return check_launch("cgbn_fwd_train_local");
}

int cgbn_fwd_eval(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                  const float* gamma, const float* beta, const float* running_mean,
                  const float* running_var, double eps, int relu, void* y, void* ws,
                  size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && y && gamma && beta && running_mean && running_var,
               "cgbn_fwd_eval: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  const void* ptrs[] = {x, y};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_coef_eval<<<chan_blocks(C), 256, 0, st>>>(gamma, beta, running_mean, running_var, eps, w.P,
                                              w.Q, (uint32_t)C);
  launch_ew_affine(ep, relu != 0, x, y, w.P, w.Q, st);
  return check_launch("cgbn_fwd_eval");
}

int cgbn_xhat(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
              const double* saved, void* xhat, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && saved && xhat, "cgbn_xhat: NULL pointer");
  const void* ptrs[] = {x, xhat};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_coef_xhat<<<chan_blocks(C), 256, 0, st>>>(saved, w.P, w.Q, (uint32_t)C);
  launch_ew_affine(ep, false, x, xhat, w.P, w.Q, st);
  return check_launch("cgbn_xhat");
}

int cgbn_channel_affine(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                        const double* scale, const double* shift, void* out, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(x && scale && shift && out, "cgbn_channel_affine: NULL pointer");
  const void* ptrs[] = {x, out};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 2, &ep));
  // no PDL: the previous kernel on the stream may be the caller's producer of x
  launch_ew_affine(ep, false, x, out, scale, shift, reinterpret_cast<cudaStream_t>(stream), false);
  return check_launch("cgbn_channel_affine");
}

int cgbn_bwd_reduce(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                    int layout, const double* saved, const float* gamma, const float* beta,
                    int relu, double* partial, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && partial, "cgbn_bwd_reduce: NULL pointer");
  CGBN_REQUIRE(!relu || (gamma && beta), "cgbn_bwd_reduce: relu needs gamma and beta");
  const void* ptrs[] = {dy, x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 2, &pl));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CGBN_TRY(dispatch_bwd_reduce(pl, dy, x, saved, gamma, beta, relu != 0, kPartial, partial,
                               nullptr, w, st));
  return check_launch("cgbn_bwd_reduce");
}

int cgbn_bwd_dx(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                const double* const* partials, int G, const double* saved, const float* gamma,
                const float* beta, double eps, int relu, void* dx, float* dgamma,
                float* dbeta, unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_dx: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_dx: relu needs beta");
  const void* ptrs[] = {dy, x, dx};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, ptrs, 3, &ep));
  Parts parts;
  CGBN_TRY(fill_parts(&parts, partials, G));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const BwdFinal F =
      make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  launch_pdl(k_finalize_bwd, chan_blocks(C), true, st, parts, F);
  launch_ew_dx(ep, relu != 0, dy, x, dx, w, st);
  return check_launch("cgbn_bwd_dx");
}

int cgbn_bwd_local(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW,
                   int layout, const double* saved, const float* gamma, const float* beta,
                   double eps, int relu, void* dx, float* dgamma, float* dbeta,
                   unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_local: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_local: relu needs beta");
  const void* ptrs[] = {dy, x};
  Plan pl;
  CGBN_TRY(make_plan(N, C, HW, layout, act, ptrs, 2, &pl));
  const void* eptrs[] = {dy, x, dx};
  EwPlan ep;
  CGBN_TRY(make_ew(N, C, HW, layout, act, eptrs, 3, &ep));
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const BwdFinal F =
      make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  pl.tma = false;
  CGBN_TRY(dispatch_bwd_reduce(pl, dy, x, saved, gamma, beta, relu != 0, kLocalFinal, nullptr,
                               &F, w, st));
  launch_ew_dx(ep, relu != 0, dy, x, dx, w, st);
  return check_launch("cgbn_bwd_local");
}

int cgbn_fused_supported(int64_t N, int64_t C, int64_t HW, int layout, int backward) {
  int act = 0;
  if (split_fmt(&layout, &act) || act != 0) return 0;  // fp32 only
  fused::FGeom fg;
  return fused_plan(N, C, HW, layout, 0, backward ? 2 : 1, &fg) ? 1 : 0;
}

int cgbn_fwd_fused(const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   const float* gamma, const float* beta, double eps, double momentum,
                   float* running_mean, float* running_var, double* saved, int relu, void* y,
                   unsigned* status, void* ws, size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  if (act != 0) return set_error(CGBN_ERR_UNSUPPORTED, "%s: fp32 activations only", "cgbn_fwd_fused");
  CGBN_TRY(check_fwd_args(x, y, gamma, beta, saved, eps, momentum, running_mean, running_var));
  CGBN_TRY(validate_shape(N, C, HW, layout));
  fused::FGeom fg;
  if (!fused_plan(N, C, HW, layout, (uintptr_t)x | (uintptr_t)y, 1, &fg))
    return set_error(CGBN_ERR_UNSUPPORTED, "cgbn_fwd_fused: shape/layout not eligible");
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  FwdFinal F =
      make_fwd_final(C, gamma, beta, eps, momentum, running_mean, running_var, saved, status, w);
  F.P = F.Q = nullptr;  // the fused kernel keeps its coefficients in shared memory
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const float* xf = static_cast<const float*>(x);
  float* yf = static_cast<float*>(y);
  CGBN_TRY(relu ? launch_cooperative(fused::k_fused_fwd<true>, fg.grid, fused::kSmemBytes, st, fg,
                                     xf, yf, F, w.slots, w.bar)
                : launch_cooperative(fused::k_fused_fwd<false>, fg.grid, fused::kSmemBytes, st,
                                     fg, xf, yf, F, w.slots, w.bar));
  return check_launch("cgbn_fwd_fused");
}

int cgbn_bwd_fused(const void* dy, const void* x, int64_t N, int64_t C, int64_t HW, int layout,
                   const double* saved, const float* gamma, const float* beta, double eps,
                   int relu, void* dx, float* dgamma, float* dbeta, unsigned* status, void* ws,
                   size_t ws_bytes, void* stream) {
  int act = 0;
  CGBN_TRY(split_fmt(&layout, &act));
  if (act != 0) return set_error(CGBN_ERR_UNSUPPORTED, "%s: fp32 activations only", "cgbn_bwd_fused");
  CGBN_REQUIRE(dy && x && saved && gamma && dx, "cgbn_bwd_fused: NULL pointer");
  CGBN_REQUIRE(eps > 0.0, "eps must be positive, got %g", eps);
  CGBN_REQUIRE(!relu || beta, "cgbn_bwd_fused: relu needs beta");
  CGBN_TRY(validate_shape(N, C, HW, layout));
  fused::FGeom fg;
  if (!fused_plan(N, C, HW, layout, (uintptr_t)dy | (uintptr_t)x | (uintptr_t)dx, 2, &fg))
    return set_error(CGBN_ERR_UNSUPPORTED, "cgbn_bwd_fused: shape/layout not eligible");
  WsView w;
  CGBN_TRY(ws_view(ws, ws_bytes, N, C, HW, layout, &w));
  BwdFinal F = make_bwd_final(C, saved, gamma, beta, eps, relu != 0, dgamma, dbeta, status, w);
  F.A = F.B = F.Cc = F.P = F.Q = nullptr;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const float* dyf = static_cast<const float*>(dy);
  const float* xf = static_cast<const float*>(x);
  float* dxf = static_cast<float*>(dx);
  CGBN_TRY(relu ? launch_cooperative(fused::k_fused_bwd<true>, fg.grid, fused::kSmemBytes, st, fg,
                                     dyf, xf, dxf, F, w.slots, w.bar)
                : launch_cooperative(fused::k_fused_bwd<false>, fg.grid, fused::kSmemBytes, st,
                                     fg, dyf, xf, dxf, F, w.slots, w.bar));
  return check_launch("cgbn_bwd_fused");
}

size_t cgbn_p2p_region_bytes(int G, int64_t max_len) {
  if (G < 1 || G > CGBN_MAX_GROUP || max_len < 1) return 0;
  return p2p::region_bytes(G, max_len);
}

int cgbn_p2p_alloc(size_t bytes, void** region, void* ipc_handle) {
  CGBN_REQUIRE(region && ipc_handle && bytes > 0, "cgbn_p2p_alloc: bad argument");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_alloc: cudaMalloc: %s", cudaGetErrorString(e));
  e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess)
    e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(ipc_handle), p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_alloc: %s", cudaGetErrorString(e));
  }
  *region = p;
  return CGBN_OK;
}

int cgbn_p2p_open(const void* ipc_handle, void** region) {
  CGBN_REQUIRE(region && ipc_handle, "cgbn_p2p_open: NULL pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(region, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_open: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

int cgbn_p2p_close(void* region) {
  const cudaError_t e = cudaIpcCloseMemHandle(region);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_close: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

int cgbn_p2p_free(void* region) {
  const cudaError_t e = cudaFree(region);
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_free: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

namespace {
int fill_peers(p2p::Peers* P, void* const* regions, int G) {
  if (G < 1 || G > p2p::kMaxPeers)
    return set_error(CGBN_ERR_INVALID, "group size %d outside [1, %d]", G, p2p::kMaxPeers);
  if (!regions) return set_error(CGBN_ERR_INVALID, "regions array is NULL");
  for (int q = 0; q < G; ++q) {
    if (!regions[q]) return set_error(CGBN_ERR_INVALID, "regions[%d] is NULL", q);
    P->base[q] = static_cast<char*>(regions[q]);
  }
  for (int q = G; q < p2p::kMaxPeers; ++q) P->base[q] = nullptr;
  return CGBN_OK;
}
}  // namespace

int cgbn_p2p_exchange(const double* vec, int64_t n, int rank, int G, void* const* regions,
                      int64_t max_len, double* out, unsigned* status, double timeout_s,
                      void* stream) {
  CGBN_REQUIRE(vec && out, "cgbn_p2p_exchange: NULL pointer");
  CGBN_REQUIRE(n >= 1 && n <= max_len, "cgbn_p2p_exchange: n=%lld outside [1, %lld]",
               (long long)n, (long long)max_len);
  CGBN_REQUIRE(rank >= 0 && rank < G, "cgbn_p2p_exchange: rank %d outside [0, %d)", rank, G);
  CGBN_REQUIRE(timeout_s > 0.0, "cgbn_p2p_exchange: timeout must be positive");
  p2p::Peers peers;
  CGBN_TRY(fill_peers(&peers, regions, G));
  launch_pdl(p2p::k_p2p_exchange, 1u, true, reinterpret_cast<cudaStream_t>(stream), vec, n, rank,
             G, peers, max_len, out, status, (uint64_t)(timeout_s * 1e9));
  return check_launch("cgbn_p2p_exchange");
}

int cgbn_p2p_emulate(const double* vecs, int64_t n, int G, void* const* regions, int64_t max_len,
                     double* outs, unsigned* status, double timeout_s, int skip, void* stream) {
  CGBN_REQUIRE(vecs && outs, "cgbn_p2p_emulate: NULL pointer");
  CGBN_REQUIRE(n >= 1 && n <= max_len, "cgbn_p2p_emulate: n outside [1, max_len]");
  CGBN_REQUIRE(timeout_s > 0.0, "cgbn_p2p_emulate: timeout must be positive");
  p2p::Peers peers;
  CGBN_TRY(fill_peers(&peers, regions, G));
  // cooperative launch: the G rank-CTAs are guaranteed co-resident while they wait on
  // each other (the single-GPU stand-in for G processes)
  const uint64_t tns = (uint64_t)(timeout_s * 1e9);
  void* args[] = {(void*)&vecs, (void*)&n,      (void*)&G,      (void*)&peers, (void*)&max_len,
                  (void*)&outs, (void*)&status, (void*)&tns,    (void*)&skip};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)p2p::k_p2p_emulate, dim3(G),
                                                    dim3(p2p::kThreadsP2P), args, 0,
                                                    reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_error(CGBN_ERR_CUDA, "cgbn_p2p_emulate: %s", cudaGetErrorString(e));
  return check_launch("cgbn_p2p_emulate");
}

int cgbn_fold_sum(const void* const* vectors, int G, int64_t n, int dtype, void* out,
                  void* stream) {
  CGBN_REQUIRE(vectors && out, "cgbn_fold_sum: NULL pointer");
  CGBN_REQUIRE(n >= 1, "cgbn_fold_sum: n must be >= 1");
  CGBN_REQUIRE(dtype == CGBN_DTYPE_F32 || dtype == CGBN_DTYPE_F64, "unknown dtype %d", dtype);
  Parts P;
  CGBN_TRY(fill_parts(&P, reinterpret_cast<const double* const*>(vectors), G));
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
