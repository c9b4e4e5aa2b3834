// cgbn_ops.cuh — per-channel fp64 arithmetic, PDL and cp.async helpers, channel finishers, reduction ops
// Part of the single translation unit cgbn.cu (included there, in order).

#pragma once

namespace {

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
  float4* T1;     // fp32 record {P, mean_hi, mean_lo, beta} for 16-bit activations (or null)
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
  if (F.T1) {  // y = P (x - mean) + beta in fp32, the mean as a float pair (no cancellation)
    const float mh = (float)mean;
    F.T1[c] = make_float4((float)P, mh, (float)(mean - (double)mh), v.beta);
  }
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
  float4* T1;     // fp32 records for 16-bit activations (or null): {A, B, C3, 0} with
  float2* T2;     // dx = A g + B (x - mean) + C3 and the mean as a float pair {hi, lo}
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
  if (F.T1) {
    const float mh = (float)mean;
    F.T1[c] = make_float4((float)k.A, (float)k.B, (float)(k.Cc + k.B * mean), 0.f);
    F.T2[c] = make_float2(mh, (float)(mean - (double)mh));
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
// The fused-exchange push (cgbn_*_p2p) as a compile-time option of the reduction Ops, so
// the kernels of every other path keep their parameters and registers (a runtime member
// cost 7-12% on the statistics / backward reductions).
template <bool PUSH>
struct PushSlot {};
template <>
struct PushSlot<true> {
  p2p::Push push;
};

template <class T, int VM, bool PUSH = false>
struct StatsOp : PushSlot<PUSH> {
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
    if constexpr (sizeof(T) == 2 && VEC >= 4) {
      // 16-bit activations: the unit's VEC differences and squares are summed in fp32,
      // then added once to the fp64 accumulators (a quarter of the fp64 conversions and
      // adds). K is the channel's first element or 0 here, so d = x - K is exact in fp32
      // whenever x and K lie within 2^15 of each other, and the partial carries at most
      // VEC - 1 fp32 roundings (~5e-7 relative). kSumSq shifts by the fp64 group mean
      // and keeps the fp64 path.
      if (ksum == nullptr) {
        const float Kf = (float)K;
        float s = 0.f, q = 0.f;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          if (masked_vm(VM) && !((r.m >> k) & 1u)) continue;
          const float d = r.v.get(k) - Kf;
          s += d;
          q = __fmaf_rn(d, d, q);
        }
        a += (double)s;
        b += (double)q;
        return;
      }
    }
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
    if constexpr (PUSH) {
      if (mode == kPartial) {
        // fused exchange: this channel straight into row `rank` of every rank's region
        const p2p::Push& push = this->push;
        const unsigned long long e = p2p::push_epoch(push);
#pragma unroll
        for (int q = 0; q < p2p::kMaxPush; ++q) {
          if (q >= push.G) break;
          double* dst =
              p2p::recv_ptr(push.base[q], push.G, push.max_len, (int)(e & 1ull), push.rank);
          dst[c] = mean;
          dst[g.C + c] = M2;
          if (c == 0) dst[2 * g.C] = n;
        }
        p2p::push_done(push, e);
        return;
      }
    }
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
template <class T, int VM, bool RELU, bool PUSH = false>
struct BwdOp : PushSlot<PUSH> {
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
    if constexpr (sizeof(T) == 2 && VEC >= 4 && !RELU) {
      // 16-bit activations: sum g in an fp32 partial of the unit's VEC terms (bf16 / fp16
      // values add exactly or nearly so), one fp64 add; sum g*(x - mean) per element in
      // fp64 as for fp32 activations. (An fp32 partial of g*(x - mean) left ~1e-6
      // absolute error on dgamma, 5e-4 relative on near-zero channels of [32,2048,7,7].)
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        if (masked_vm(VM) && !((r.m >> k) & 1u)) continue;
        const float gk = r.g.get(k);
        s += gk;
        b = __fma_rn((double)gk, (double)r.x.get(k) - mean, b);
      }
      a += (double)s;
      return;
    }
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
    if constexpr (PUSH) {
      if (mode == kPartial) {
        const p2p::Push& push = this->push;
        const unsigned long long e = p2p::push_epoch(push);
#pragma unroll
        for (int q = 0; q < p2p::kMaxPush; ++q) {
          if (q >= push.G) break;
          double* dst =
              p2p::recv_ptr(push.base[q], push.G, push.max_len, (int)(e & 1ull), push.rank);
          dst[c] = S1;
          dst[g.C + c] = S2;
        }
        p2p::push_done(push, e);
        return;
      }
    }
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

}  // namespace
