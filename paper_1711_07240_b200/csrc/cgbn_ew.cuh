// cgbn_ew.cuh — finalize / coefficient kernels, memory-order elementwise kernels, ascending fold
// Part of the single translation unit cgbn.cu (included there, in order).

#pragma once

namespace {

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

// The same after a fused exchange: every block waits for the group's flags of the current
// epoch in its own region, then folds the G rows (ascending rank order) read there.
// A timed-out exchange yields NaN statistics: the finisher then flags the channel
// non-finite and leaves the running statistics alone, and y / dx come out NaN, instead of
// silently using a missing rank's rows from an older exchange.
__global__ void k_finalize_fwd_p2p(p2p::Pull pull, FwdFinal F) {
  pdl_wait();
  bool timed_out;
  const unsigned long long e = p2p::pull_wait(pull, timed_out);
  pdl_trigger();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= F.C) return;
  Parts parts;
  parts.G = pull.G;
  for (int r = 0; r < pull.G; ++r)
    parts.p[r] = p2p::recv_ptr(pull.own, pull.G, pull.max_len, (int)(e & 1ull), r);
  double n, mean, M2, P, Q;
  merge_fwd_partials(parts, c, F.C, n, mean, M2);
  if (timed_out) n = mean = M2 = __longlong_as_double(0x7ff8000000000000ll);
  finalize_fwd_channel(F, c, n, mean, M2, true, P, Q);
}

__global__ void k_finalize_bwd_p2p(p2p::Pull pull, BwdFinal F) {
  pdl_wait();
  bool timed_out;
  const unsigned long long e = p2p::pull_wait(pull, timed_out);
  pdl_trigger();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= F.C) return;
  const uint32_t C = F.C;
  const int par = (int)(e & 1ull);
  const double* r0 = p2p::recv_ptr(pull.own, pull.G, pull.max_len, par, 0);
  double sdy = r0[c], sdyx = r0[C + c];
  for (int r = 1; r < pull.G; ++r) {  // ascending rank fold (collectives.py:293-295)
    const double* rr = p2p::recv_ptr(pull.own, pull.G, pull.max_len, par, r);
    sdy += rr[c];
    sdyx += rr[C + c];
  }
  if (timed_out) sdy = sdyx = __longlong_as_double(0x7ff8000000000000ll);
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
  uint32_t reuse; // CM 3, fp32: a thread's units share their 4 channels (UE*stride % C == 0)
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

// Coefficients of the UE channels of a channels_last unit starting at channel-aligned
// element e (CM 3: c % 4 == 0), 4 at a time.
template <int UE>
__device__ __forceinline__ void ew_coef_unit(const EwGeom& g, const double* __restrict__ T,
                                             uint32_t e, double* t) {
#pragma unroll
  for (int h = 0; h < UE; h += 4) {
    uint32_t c[4];
    chan4<3>(g, e + h, c);
    double q[4];
    ew_coef<3>(T, c, q);
#pragma unroll
    for (int k = 0; k < 4; ++k) t[h + k] = q[k];
  }
}

#ifndef CGBN_EWU
#define CGBN_EWU 2
#endif
constexpr int kEwU = CGBN_EWU;  // 16-byte units per elementwise thread (one round): 2 measured best of 1/2/4/8 (ResNet-50 79.3% -> 82.0% of HBM vs 4)

template <class T>
constexpr int ew_ue() { return 16 / (int)sizeof(T); }

// fp32 records of the 16-bit passes (cgbn_ops.cuh FwdFinal / BwdFinal T1, T2) for the UE
// channels of a channels_last unit at element e (CM 3), or one channel's record.
template <int UE, class R>
__device__ __forceinline__ void ew_rec_unit(const EwGeom& g, const R* __restrict__ T, uint32_t e,
                                            R (&r)[UE]) {
  const uint32_t c0 = e - g.dc.div(e) * g.C;
#pragma unroll
  for (int k = 0; k < UE; ++k) r[k] = __ldg(T + c0 + k);
}

// The 16-bit activations' normalise without ReLU, in fp32 (the output keeps 8 / 11
// significant bits): y = P ((x - mean_hi) - mean_lo) + beta. x is exact in fp32, the mean
// a float pair, so the difference keeps ~2^-23 relative error whatever |mean| / std, and
// y ~2^-22 — against the output's 2^-8 (bf16) / 2^-11 (fp16) rounding. No fp64 conversion
// (these bound the fp64 path: XU pipe 66% busy, tools/gpu/ncu_bf16.sh).
template <class T, int CM, int U>
__device__ __forceinline__ void ew_affine_f32(const EwGeom& g, const T* __restrict__ x,
                                              T* __restrict__ y, const float4* __restrict__ T1) {
  constexpr int UE = ew_ue<T>();
  pdl_trigger();
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  Vec<T, UE> v[U];
  auto load = [&](uint32_t i0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < g.n4) v[u].load(x + (size_t)UE * ew_unit(g, i0 + u * stride));
  };
  load(i);
  pdl_wait();
  constexpr bool kReuse = CM == 3;
  float4 tr[kReuse ? UE : 1];
  if constexpr (kReuse) {
    if (g.reuse && i < g.n4) ew_rec_unit<UE>(g, T1, UE * ew_unit(g, i), tr);
  }
  for (; i < g.n4; i += U * stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j >= g.n4) continue;
      const uint32_t jm = ew_unit(g, j);
      float o[UE];
      if constexpr (CM == 0) {  // one channel per unit
        const float4 t = __ldg(T1 + chan_of<0>(g, UE * jm));
#pragma unroll
        for (int k = 0; k < UE; ++k) o[k] = fmaf(t.x, (v[u].get(k) - t.y) - t.z, t.w);
      } else {
#pragma unroll
        for (int h = 0; h < UE; h += 4) {
          float4 t[4];
          if (kReuse && g.reuse) {
#pragma unroll
            for (int k = 0; k < 4; ++k) t[k] = tr[kReuse ? h + k : 0];
          } else {
            uint32_t c[4];
            chan4<CM>(g, UE * jm + h, c);
#pragma unroll
            for (int k = 0; k < 4; ++k) t[k] = __ldg(T1 + c[k]);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o[h + k] = fmaf(t[k].x, (v[u].get(h + k) - t[k].y) - t[k].z, t[k].w);
        }
      }
      stvf<T, UE>(y + (size_t)UE * jm, o);
    }
    load(i + U * stride);
  }
  if (blockIdx.x == 0 && threadIdx.x < g.tail) {
    const uint32_t e = UE * g.n4 + threadIdx.x;
    const uint32_t c = CM >= 2 ? chan_of<2>(g, e) : chan_of<1>(g, e);
    const float4 t = __ldg(T1 + c);
    st1(y + e, (double)fmaf(t.x, (ld1(x + e) - t.y) - t.z, t.w));
  }
}

template <class T, bool RELU, int CM, int U>
__global__ void __launch_bounds__(kThreads)
k_ew_affine(EwGeom g, const T* __restrict__ x, T* __restrict__ y,
            const double* __restrict__ P, const double* __restrict__ Q,
            const float4* __restrict__ T1) {
  // (NCHW only: with channels_last units of 8 channels the per-channel records cost more
  // than the conversions they save — step 2.16 -> 2.50 ms, profiles/r2_negative)
  if constexpr (sizeof(T) == 2 && !RELU && CM <= 1) {
    if (T1 != nullptr) {  // training forward: the finisher wrote the fp32 records
      ew_affine_f32<T, CM, U>(g, x, y, T1);
      return;
    }
  }
  constexpr int UE = ew_ue<T>();
  pdl_trigger();  // the next reduction may launch and wait
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  Vec<T, UE> v[U];
  auto load = [&](uint32_t i0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < g.n4) v[u].load(x + (size_t)UE * ew_unit(g, i0 + u * stride));
  };
  load(i);    // x is not written by the kernel we may overlap with
  pdl_wait();  // the coefficient table is
  // channels_last: when every unit of the thread covers the same UE channels, their
  // coefficients are loaded once (fp64 tables would otherwise cost 16 B per element)
  constexpr bool kReuse = CM == 3;
  double pr[UE], qr[UE];
  if (kReuse && g.reuse && i < g.n4) {
    ew_coef_unit<UE>(g, P, UE * ew_unit(g, i), pr);
    ew_coef_unit<UE>(g, Q, UE * ew_unit(g, i), qr);
  }
  for (; i < g.n4; i += U * stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j >= g.n4) continue;
      const uint32_t jm = ew_unit(g, j);
      double o[UE];
#pragma unroll
      for (int h = 0; h < UE; h += 4) {
        double p[4], q[4];
        if (kReuse && g.reuse) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            p[k] = pr[h + k];
            q[k] = qr[h + k];
          }
        } else {
          uint32_t c[4];
          chan4<CM>(g, UE * jm + h, c);
          ew_coef<CM>(P, c, p);
          ew_coef<CM>(Q, c, q);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double t = __fma_rn(p[k], (double)v[u].get(h + k), q[k]);
          if (RELU) t = t > 0.0 ? t : 0.0;
          o[h + k] = t;
        }
      }
      stv<T, UE>(y + (size_t)UE * jm, o);
    }
    load(i + U * stride);
  }
  if (blockIdx.x == 0 && threadIdx.x < g.tail) {
    const uint32_t e = UE * g.n4 + threadIdx.x;
    const uint32_t c = CM >= 2 ? chan_of<2>(g, e) : chan_of<1>(g, e);
    double t = __fma_rn(P[c], (double)ld1(x + e), Q[c]);
    if (RELU) t = t > 0.0 ? t : 0.0;
    st1(y + e, t);
  }
}

// The 16-bit activations' dx without ReLU, in fp32: dx = A g + B ((x - mean_hi) - mean_lo)
// + C3 with C3 = Cc + B mean (= -A dbeta / m), the same error argument as ew_affine_f32.
template <class T, int CM, int U>
__device__ __forceinline__ void ew_dx_f32(const EwGeom& g, const T* __restrict__ dy,
                                          const T* __restrict__ x, T* __restrict__ dx,
                                          const float4* __restrict__ T1,
                                          const float2* __restrict__ T2) {
  constexpr int UE = ew_ue<T>();
  pdl_trigger();
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  Vec<T, UE> gv[U], xv[U];
  auto load = [&](uint32_t i0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < g.n4) {
        const size_t off = (size_t)UE * ew_unit(g, i0 + u * stride);
        gv[u].load(dy + off);
        xv[u].load(x + off);
      }
  };
  load(i);
  pdl_wait();
  constexpr bool kReuse = CM == 3;
  float4 tr[kReuse ? UE : 1];
  float2 mr[kReuse ? UE : 1];
  if constexpr (kReuse) {
    if (g.reuse && i < g.n4) {
      ew_rec_unit<UE>(g, T1, UE * ew_unit(g, i), tr);
      ew_rec_unit<UE>(g, T2, UE * ew_unit(g, i), mr);
    }
  }
  for (; i < g.n4; i += U * stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j >= g.n4) continue;
      const uint32_t jm = ew_unit(g, j);
      float o[UE];
      if constexpr (CM == 0) {
        const uint32_t c = chan_of<0>(g, UE * jm);
        const float4 t = __ldg(T1 + c);
        const float2 m = __ldg(T2 + c);
#pragma unroll
        for (int k = 0; k < UE; ++k)
          o[k] = fmaf(t.x, gv[u].get(k), fmaf(t.y, (xv[u].get(k) - m.x) - m.y, t.z));
      } else {
#pragma unroll
        for (int h = 0; h < UE; h += 4) {
          float4 t[4];
          float2 m[4];
          if (kReuse && g.reuse) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              t[k] = tr[kReuse ? h + k : 0];
              m[k] = mr[kReuse ? h + k : 0];
            }
          } else {
            uint32_t c[4];
            chan4<CM>(g, UE * jm + h, c);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              t[k] = __ldg(T1 + c[k]);
              m[k] = __ldg(T2 + c[k]);
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o[h + k] = fmaf(t[k].x, gv[u].get(h + k),
                            fmaf(t[k].y, (xv[u].get(h + k) - m[k].x) - m[k].y, t[k].z));
        }
      }
      stvf<T, UE>(dx + (size_t)UE * jm, o);
    }
    load(i + U * stride);
  }
  if (blockIdx.x == 0 && threadIdx.x < g.tail) {
    const uint32_t e = UE * g.n4 + threadIdx.x;
    const uint32_t c = CM >= 2 ? chan_of<2>(g, e) : chan_of<1>(g, e);
    const float4 t = __ldg(T1 + c);
    const float2 m = __ldg(T2 + c);
    st1(dx + e, (double)fmaf(t.x, ld1(dy + e), fmaf(t.y, (ld1(x + e) - m.x) - m.y, t.z)));
  }
}

template <class T, bool RELU, int CM, int U>
__global__ void __launch_bounds__(kThreads)
k_ew_dx(EwGeom g, const T* __restrict__ dy, const T* __restrict__ x, T* __restrict__ dx,
        const double* __restrict__ A, const double* __restrict__ B,
        const double* __restrict__ Cc, const double* __restrict__ P,
        const double* __restrict__ Q, const float4* __restrict__ T1,
        const float2* __restrict__ T2) {
  if constexpr (sizeof(T) == 2 && !RELU && CM <= 1) {  // (NCHW only, as k_ew_affine)
    if (T1 != nullptr) {  // the backward finisher wrote the fp32 records
      ew_dx_f32<T, CM, U>(g, dy, x, dx, T1, T2);
      return;
    }
  }
  constexpr int UE = ew_ue<T>();
  pdl_trigger();  // the next reduction may launch and wait
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  Vec<T, UE> gv[U], xv[U];
  auto load = [&](uint32_t i0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < g.n4) {
        const size_t off = (size_t)UE * ew_unit(g, i0 + u * stride);
        gv[u].load(dy + off);
        xv[u].load(x + off);
      }
  };
  load(i);    // dy and x are not written by the kernel we may overlap with
  pdl_wait();  // the coefficient tables are
  constexpr bool kReuse = CM == 3;  // see k_ew_affine
  double ar[UE], br[UE], cr[UE], pr[UE], qr[UE];
  if (kReuse && g.reuse && i < g.n4) {
    const uint32_t e0 = UE * ew_unit(g, i);
    ew_coef_unit<UE>(g, A, e0, ar);
    ew_coef_unit<UE>(g, B, e0, br);
    ew_coef_unit<UE>(g, Cc, e0, cr);
    if (RELU) {
      ew_coef_unit<UE>(g, P, e0, pr);
      ew_coef_unit<UE>(g, Q, e0, qr);
    }
  }
  for (; i < g.n4; i += U * stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * stride;
      if (j >= g.n4) continue;
      const uint32_t jm = ew_unit(g, j);
      double o[UE];
#pragma unroll
      for (int h = 0; h < UE; h += 4) {
        double a[4], b[4], cc[4], p[4] = {0.0, 0.0, 0.0, 0.0}, q[4] = {0.0, 0.0, 0.0, 0.0};
        if (kReuse && g.reuse) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            a[k] = ar[h + k];
            b[k] = br[h + k];
            cc[k] = cr[h + k];
            if (RELU) {
              p[k] = pr[h + k];
              q[k] = qr[h + k];
            }
          }
        } else {
          uint32_t c[4];
          chan4<CM>(g, UE * jm + h, c);
          ew_coef<CM>(A, c, a);
          ew_coef<CM>(B, c, b);
          ew_coef<CM>(Cc, c, cc);
          if (RELU) {
            ew_coef<CM>(P, c, p);
            ew_coef<CM>(Q, c, q);
          }
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
    load(i + U * stride);
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
