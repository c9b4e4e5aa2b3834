// flatlab.cu — decomposes the per-launch cost of the channel-major flat reduction
// (k_reduce_flat in csrc/cgbn.cu) at ResNet-50 shapes, in CUDA graphs of back-to-back
// launches over rotating buffers (> L2):
//   V0  memory-order fp64 stats over the whole tensor (the streaming ideal)
//   V1  channel-major CTA slices, one stream per CTA (addressing cost only)
//   V2  V1 + per-channel segments (K load, block reduce per segment)
//   V3  V2 + cross-CTA tail (slot + ticket, last CTA folds and finishes)
//   V4  V3 with software-pipelined rounds (next round's loads issued before the
//       current round is accumulated)
//   V5  V3 with 2 CTAs of 512 threads... (grid variants via argv)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/bin/flatlab tools/flatlab.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int kT = 256, kW = kT / 32;

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

struct G {
  uint32_t C, Lv, HWv, grid, HW;
  uint64_t T, gap;
  FastDiv dhw;
  double count;
};

__device__ __forceinline__ size_t voff(const G& g, uint32_t c, uint32_t j) {
  return (size_t)c * g.HWv + j + (size_t)g.dhw.div(j) * g.gap;
}
__device__ __forceinline__ uint64_t cta_begin(const G& g, uint32_t b) {
  return (uint64_t)b * g.T / g.grid;
}
__device__ __forceinline__ uint32_t cta_of(const G& g, uint64_t u) {
  return (uint32_t)(((u + 1) * (uint64_t)g.grid - 1) / g.T);
}
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void acc4(const float4& v, double K, double& a, double& b) {
  const double d0 = (double)v.x - K, d1 = (double)v.y - K, d2 = (double)v.z - K,
               d3 = (double)v.w - K;
  a += (d0 + d1) + (d2 + d3);
  b = fma(d0, d0, b); b = fma(d1, d1, b); b = fma(d2, d2, b); b = fma(d3, d3, b);
}

// V0: memory order
__global__ void __launch_bounds__(kT) v0(const float4* __restrict__ x, size_t n4, double* out) {
  double a = 0, b = 0;
  const size_t stride = (size_t)gridDim.x * kT;
  for (size_t i = (size_t)blockIdx.x * kT + threadIdx.x; i < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i + u * stride < n4) v[u] = __ldg(&x[i + u * stride]);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i + u * stride < n4) acc4(v[u], 1.0, a, b);
  }
  if (a + b == 12345.0) out[0] = a;
}

// U-unrolled strided range of channel c, optional software pipelining.
template <bool PIPE>
__device__ __forceinline__ void range(const G& g, const float* __restrict__ x, uint32_t c,
                                      uint32_t j, uint32_t end, double K, double& a,
                                      double& b) {
  constexpr int U = 8;
  if (!PIPE) {
    for (; j < end; j += U * kT) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j + u * kT < end) v[u] = __ldg(reinterpret_cast<const float4*>(x) + voff(g, c, j + u * kT));
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j + u * kT < end) acc4(v[u], K, a, b);
    }
  } else {
    constexpr int H = U / 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4 p[H], q[H];
#pragma unroll
    for (int u = 0; u < H; ++u)
      if (j + u * kT < end) p[u] = __ldg(x4 + voff(g, c, j + u * kT));
    for (; j < end; j += 2 * H * kT) {
      const uint32_t j1 = j + H * kT, j2 = j + 2 * H * kT;
#pragma unroll
      for (int u = 0; u < H; ++u)
        if (j1 + u * kT < end) q[u] = __ldg(x4 + voff(g, c, j1 + u * kT));
#pragma unroll
      for (int u = 0; u < H; ++u)
        if (j + u * kT < end) acc4(p[u], K, a, b);
#pragma unroll
      for (int u = 0; u < H; ++u)
        if (j2 + u * kT < end) p[u] = __ldg(x4 + voff(g, c, j2 + u * kT));
#pragma unroll
      for (int u = 0; u < H; ++u)
        if (j1 + u * kT < end) acc4(q[u], K, a, b);
    }
  }
}

// V1: slice as one stream (ignores channel boundaries for accumulation, keeps addressing)
__global__ void __launch_bounds__(kT, 3) v1(G g, const float* __restrict__ x, double* out) {
  const uint64_t ub = cta_begin(g, blockIdx.x), ue = cta_begin(g, blockIdx.x + 1);
  double a = 0, b = 0;
  for (uint64_t u = ub; u < ue;) {
    const uint32_t c = (uint32_t)(u / g.Lv);
    const uint64_t cb = (uint64_t)c * g.Lv;
    const uint64_t se = min(ue, cb + g.Lv);
    range<false>(g, x, c, (uint32_t)(u - cb) + threadIdx.x, (uint32_t)(se - cb), 1.0, a, b);
    u = se;
  }
  if (a + b == 12345.0) out[0] = a;
}

// V2/V3/V4
template <bool TAIL, bool PIPE>
__global__ void __launch_bounds__(kT, 3) vseg(G g, const float* __restrict__ x, double* out,
                                              double2* ws, unsigned* tickets) {
  __shared__ double sa[kW], sb[kW];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint64_t ub = cta_begin(g, blockIdx.x), ue = cta_begin(g, blockIdx.x + 1);
  for (uint64_t u = ub; u < ue;) {
    const uint32_t c = (uint32_t)(u / g.Lv);
    const uint64_t cb = (uint64_t)c * g.Lv;
    const uint64_t se = min(ue, cb + g.Lv);
    const double K = (double)__ldg(x + (size_t)c * g.HW);
    double a = 0, b = 0;
    range<PIPE>(g, x, c, (uint32_t)(u - cb) + threadIdx.x, (uint32_t)(se - cb), K, a, b);
    a = wsum(a);
    b = wsum(b);
    if (l == 0) { sa[w] = a; sb[w] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
      a = sa[0]; b = sb[0];
      for (int i = 1; i < kW; ++i) { a += sa[i]; b += sb[i]; }
      if (!TAIL) {
        if (a + b == 12345.0) out[c] = a;
      } else {
        const uint32_t b0 = cta_of(g, cb), b1 = cta_of(g, cb + g.Lv - 1);
        bool last = true;
        if (b0 != b1) {
          ws[(size_t)blockIdx.x + c] = make_double2(a, b);
          __threadfence();
          last = atomicAdd(&tickets[c], 1u) == b1 - b0;
          if (last) {
            __threadfence();
            a = 0; b = 0;
            for (uint32_t i = b0; i <= b1; ++i) {
              const double2 t = __ldcg(&ws[(size_t)i + c]);
              a += t.x; b += t.y;
            }
            tickets[c] = 0;
          }
        }
        if (last) {
          const double n = g.count;
          out[c] = K + a / n;
          out[g.C + c] = fmax(b - a * (a / n), 0.0);
        }
      }
    }
    __syncthreads();
    u = se;
  }
}

// V7: clusters of KC CTAs own whole channels (cluster q: channels q, q+Q, ...); each CTA
// reduces 1/KC of every such channel with no block barrier per channel (warp partials to
// smem), then one cluster barrier and a DSMEM fold in rank order.
constexpr int kMaxCh = 32;
template <int KC, int MINB, int DS = 1>
__global__ void __cluster_dims__(KC, 1, 1) __launch_bounds__(kT, MINB) vclu(G g, const float* __restrict__ x, double* out,
                                                 uint32_t Q) {
  __shared__ double2 wpart[kMaxCh][kW];
  __shared__ double2 cpart[kMaxCh];
  __shared__ double sK[kMaxCh];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t r = cl.block_rank();
  const uint32_t q = blockIdx.x / KC;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t nch = q < g.C ? (g.C - q + Q - 1) / Q : 0;
  const uint32_t j0 = (uint32_t)((uint64_t)r * g.Lv / KC), j1 = (uint32_t)((uint64_t)(r + 1) * g.Lv / KC);
  for (uint32_t i = 0; i < nch; ++i) {
    const uint32_t c = q + i * Q;
    const double K = (double)__ldg(x + (size_t)c * g.HW);
    if (threadIdx.x == 0) sK[i] = K;
    double a = 0, b = 0;
    range<false>(g, x, c, j0 + threadIdx.x, j1, K, a, b);
    a = wsum(a);
    b = wsum(b);
    if (l == 0) wpart[i][w] = make_double2(a, b);
  }
  __syncthreads();
  if (threadIdx.x < nch) {
    double2 t = wpart[threadIdx.x][0];
    for (int k = 1; k < kW; ++k) { t.x += wpart[threadIdx.x][k].x; t.y += wpart[threadIdx.x][k].y; }
    cpart[threadIdx.x] = t;
  }
  cl.sync();
  const uint32_t i = threadIdx.x;
  if (i < nch && i % KC == r) {
    double a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const double2* p = DS ? cl.map_shared_rank(&cpart[i], k) : &cpart[i];
      const double2 t = *p;
      a += t.x; b += t.y;
    }
    const uint32_t c = q + i * Q;
    const double n = g.count, K = sK[i];
    out[c] = K + a / n;
    out[g.C + c] = fmax(b - a * (a / n), 0.0);
  }
  cl.sync();
}

// V8: cluster-team. Cluster q (KC CTAs, runtime cluster size) owns channels
// q*nch .. q*nch+nch-1; inside each CTA a team of 256/nch threads streams its channel's
// 1/KC share; warp partials -> one block barrier -> DSMEM fold in rank order.
__device__ __forceinline__ void range_s(const G& g, const float* __restrict__ x, uint32_t c,
                                       uint32_t j, uint32_t end, uint32_t stride, double K,
                                       double& a, double& b) {
  constexpr int U = 8;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (; j < end; j += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u * stride < end) v[u] = __ldg(x4 + voff(g, c, j + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u * stride < end) acc4(v[u], K, a, b);
  }
}

template <int MINB, int TLC = -1, bool F32 = false, int TAILMODE = 0>
__global__ void __launch_bounds__(kT, MINB) vct(G g, const float* __restrict__ x, double* out,
                                                uint32_t nch_log2_rt) {
  const uint32_t nch_log2 = TLC >= 0 ? 8 - TLC : nch_log2_rt;
  __shared__ double2 wpart[kW];
  __shared__ double2 cpart[8];
  __shared__ double sK[8];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t KC = cl.num_blocks(), r = cl.block_rank();
  const uint32_t q = blockIdx.x / KC;
  const uint32_t tl = 8 - nch_log2, tpc = 1u << tl;
  const uint32_t team = threadIdx.x >> tl, tq = threadIdx.x & (tpc - 1);
  const uint32_t c = (q << nch_log2) + team;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint32_t j0 = (uint32_t)((uint64_t)r * g.Lv / KC), j1 = (uint32_t)((uint64_t)(r + 1) * g.Lv / KC);
  double a = 0, b = 0;
  if (TAILMODE == 3 && c < g.C) {
    // same unit count, linear addresses: channel c's share as one contiguous run
    const float4* x4 = reinterpret_cast<const float4*>(x) + (size_t)c * g.Lv;
    for (uint32_t j = j0 + tq; j < j1; j += 8 * tpc) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u * tpc < j1) v[u] = __ldg(x4 + j + u * tpc);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u * tpc < j1) acc4(v[u], 1.0, a, b);
    }
    if (a + b == 12345.0) out[blockIdx.x] = a;
    return;
  }
  if (TAILMODE == 4 && c < g.C) {
    // channel-major addresses computed incrementally (no division per unit)
    const float4* x4 = reinterpret_cast<const float4*>(x) + (size_t)c * g.HWv;
    const uint64_t pstride = (uint64_t)g.C * g.HWv;
    uint32_t j = j0 + tq;
    uint32_t n = g.dhw.div(j), o = j - n * g.HWv;
    const uint32_t sq = (8 * tpc) / g.HWv, sr = (8 * tpc) % g.HWv;
    const uint32_t tq1 = tpc / g.HWv, tr1 = tpc % g.HWv;
    for (; j < j1; j += 8 * tpc) {
      float4 v[8];
      uint32_t nn = n, oo = o;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j + u * tpc < j1) v[u] = __ldg(x4 + nn * pstride + oo);
        nn += tq1; oo += tr1;
        if (oo >= g.HWv) { oo -= g.HWv; ++nn; }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u * tpc < j1) acc4(v[u], 1.0, a, b);
      n += sq; o += sr;
      if (o >= g.HWv) { o -= g.HWv; ++n; }
    }
    if (a + b == 12345.0) out[blockIdx.x] = a;
    return;
  }
  if (TAILMODE == 5 && c < g.C) {
    const double K = (double)__ldg(x + (size_t)c * g.HW);
    if (tq == 0) sK[team] = K;
    range<true>(g, x, c, j0 + tq, j1, K, a, b);  // pipelined, stride kT
  } else if (c < g.C) {
    const double K = (double)__ldg(x + (size_t)c * g.HW);
    if (tq == 0) sK[team] = K;
    if (F32) {
      float fa = 0.f, fb = 0.f;
      const float4* x4 = reinterpret_cast<const float4*>(x);
      const float Kf = (float)K;
      for (uint32_t j = j0 + tq; j < j1; j += 8 * tpc) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j + u * tpc < j1) v[u] = __ldg(x4 + voff(g, c, j + u * tpc));
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j + u * tpc < j1) {
            const float d0 = v[u].x - Kf, d1 = v[u].y - Kf, d2 = v[u].z - Kf, d3 = v[u].w - Kf;
            fa += (d0 + d1) + (d2 + d3);
            fb = fmaf(d0, d0, fb); fb = fmaf(d1, d1, fb); fb = fmaf(d2, d2, fb); fb = fmaf(d3, d3, fb);
          }
      }
      a = fa; b = fb;
    } else {
      range_s(g, x, c, j0 + tq, j1, tpc, K, a, b);
    }
  }
  if (TAILMODE == 1) {  // no reduction at all: just keep the values alive
    if (a + b == 12345.0) out[blockIdx.x] = a;
    return;
  }
  a = wsum(a);
  b = wsum(b);
  if (l == 0) wpart[w] = make_double2(a, b);
  __syncthreads();
  if (TAILMODE == 2) {  // block reduce only, per-CTA partial to global, no cluster step
    if (threadIdx.x == 0) out[blockIdx.x] = wpart[0].x + wpart[1].x;
    return;
  }
  if (tq == 0 && c < g.C) {
    const int w0 = (int)(team << tl) >> 5, nw = (int)tpc >> 5;
    double2 t = wpart[w0];
    for (int k = 1; k < nw; ++k) { t.x += wpart[w0 + k].x; t.y += wpart[w0 + k].y; }
    cpart[team] = t;
  }
  if (KC > 1) cl.sync(); else __syncthreads();
  if (threadIdx.x < (1u << nch_log2)) {
    const uint32_t i = threadIdx.x, ci = (q << nch_log2) + i;
    if (ci < g.C && i % KC == r) {
      double A = 0, B = 0;
      for (uint32_t k = 0; k < KC; ++k) {
        const double2 t = *cl.map_shared_rank(&cpart[i], k);
        A += t.x; B += t.y;
      }
      const double n = g.count, K = sK[i];
      out[ci] = K + A / n;
      out[g.C + ci] = fmax(B - A * (A / n), 0.0);
    }
  }
  if (KC > 1) cl.sync();
}

template <int MINB, bool F32 = false, int TM = 0>
void launch_vct(const G& g, const float* x, double* out, uint32_t KC, uint32_t nl,
                cudaStream_t st, bool ct = false) {
  const uint32_t nch = 1u << nl;
  const uint32_t Q = (g.C + nch - 1) / nch;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Q * KC);
  cfg.blockDim = dim3(kT);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = KC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (!ct) { cudaLaunchKernelEx(&cfg, vct<MINB, -1, F32>, g, x, out, nl); return; }
  switch (nl) {
    case 0: cudaLaunchKernelEx(&cfg, vct<MINB, 8, F32, TM>, g, x, out, nl); break;
    case 1: cudaLaunchKernelEx(&cfg, vct<MINB, 7, F32, TM>, g, x, out, nl); break;
    case 2: cudaLaunchKernelEx(&cfg, vct<MINB, 6, F32, TM>, g, x, out, nl); break;
    default: cudaLaunchKernelEx(&cfg, vct<MINB, 5, F32, TM>, g, x, out, nl); break;
  }
}

// V9: non-persistent flat reduction. CTA b reduces the units [b*CU, (b+1)*CU) of the
// channel-major stream in one round (incremental addresses), per channel segment:
// slot (b + c) + arrival ticket; the last CTA of a channel folds its slots (lane-parallel
// loads, fixed order) and finishes it.
template <int UPT>
__global__ void __launch_bounds__(kT) v9(G g, const float* __restrict__ x, double* out,
                                           double2* ws, unsigned* tickets) {
  constexpr uint32_t CU = kT * UPT;
  __shared__ double sa[kW], sb[kW];
  __shared__ int s_last;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const uint64_t ub = (uint64_t)blockIdx.x * CU, ue = min(g.T, ub + CU);
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (uint64_t u = ub; u < ue;) {
    const uint32_t c = (uint32_t)(u / g.Lv);
    const uint64_t cb = (uint64_t)c * g.Lv;
    const uint64_t se = min(ue, cb + g.Lv);
    const double K = (double)__ldg(x + (size_t)c * g.HW);
    double a = 0, b = 0;
    const uint32_t j0 = (uint32_t)(u - cb), j1 = (uint32_t)(se - cb);
    float4 v[UPT];
#pragma unroll
    for (int k = 0; k < UPT; ++k) {
      const uint32_t j = j0 + threadIdx.x + k * kT;
      if (j < j1) v[k] = __ldg(x4 + voff(g, c, j));
    }
#pragma unroll
    for (int k = 0; k < UPT; ++k)
      if (j0 + threadIdx.x + k * kT < j1) acc4(v[k], K, a, b);
    a = wsum(a);
    b = wsum(b);
    if (l == 0) { sa[w] = a; sb[w] = b; }
    __syncthreads();
    const uint32_t b0 = (uint32_t)(cb / CU), b1 = (uint32_t)((cb + g.Lv - 1) / CU);
    if (threadIdx.x == 0) {
      a = sa[0]; b = sb[0];
      for (int i = 1; i < kW; ++i) { a += sa[i]; b += sb[i]; }
      int last = 1;
      if (b0 != b1) {
        ws[(size_t)blockIdx.x + c] = make_double2(a, b);
        __threadfence();
        last = atomicAdd(&tickets[c], 1u) == b1 - b0;
      } else {
        out[c] = K + a / g.count;
        out[g.C + c] = fmax(b - a * (a / g.count), 0.0);
        last = 0;
      }
      s_last = last;
    }
    __syncthreads();
    if (s_last && w == 0) {
      __threadfence();
      double x1 = 0, x2 = 0;
      for (uint32_t i = b0 + l; i <= b1; i += 32) {
        const double2 t = __ldcg(&ws[(size_t)i + c]);
        x1 += t.x; x2 += t.y;
      }
      x1 = wsum(x1); x2 = wsum(x2);
      if (l == 0) {
        out[c] = K + x1 / g.count;
        out[g.C + c] = fmax(x2 - x1 * (x1 / g.count), 0.0);
        tickets[c] = 0;
      }
    }
    __syncthreads();
    u = se;
  }
}

// V10: cluster-team streaming with a per-thread cp.async ring in shared memory (S stages
// of U units): loads stay in flight continuously instead of draining per round. No tail
// (compare with V8t4). Incremental channel-major addresses.
template <int TLC, int U, int S>
__global__ void __launch_bounds__(kT) v10(G g, const float* __restrict__ x, double* out) {
  extern __shared__ float4 ring[];  // [S][U][kT]
  constexpr uint32_t tpc = 1u << TLC;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t KC = cl.num_blocks(), r = cl.block_rank();
  const uint32_t q = blockIdx.x / KC;
  const uint32_t nl = 8 - TLC;
  const uint32_t team = threadIdx.x >> TLC, tq = threadIdx.x & (tpc - 1);
  const uint32_t c = (q << nl) + team;
  const uint32_t j0 = (uint32_t)((uint64_t)r * g.Lv / KC), j1 = (uint32_t)((uint64_t)(r + 1) * g.Lv / KC);
  double a = 0, b = 0;
  if (c < g.C) {
    const float4* x4 = reinterpret_cast<const float4*>(x) + (size_t)c * g.HWv;
    const uint64_t pstride = (uint64_t)g.C * g.HWv;
    // cursor
    uint32_t jj = j0 + tq;
    uint32_t n = g.dhw.div(jj), o = jj - n * g.HWv;
    const uint32_t sq = tpc / g.HWv, sr = tpc % g.HWv;
    auto issue = [&](int stage, uint32_t jstart) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (jstart + u * tpc < j1) {
          const float4* src = x4 + n * pstride + o;
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ring[(stage * U + u) * kT + threadIdx.x]);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
        n += sq; o += sr;
        if (o >= g.HWv) { o -= g.HWv; ++n; }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const uint32_t step = U * tpc;
    uint32_t jissue = j0 + tq;
#pragma unroll
    for (int s0 = 0; s0 < S - 1; ++s0) { issue(s0, jissue); jissue += step; }
    int stage = 0;
    for (uint32_t jc = j0 + tq; jc < j1; jc += step) {
      issue((stage + S - 1) % S, jissue);
      jissue += step;
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (jc + u * tpc < j1) acc4(ring[(stage * U + u) * kT + threadIdx.x], 1.0, a, b);
      stage = (stage + 1) % S;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  if (a + b == 12345.0) out[blockIdx.x] = a;
}

template <int U, int S>
void launch_v10(const G& g, const float* x, double* out, uint32_t KC, uint32_t nl, cudaStream_t st) {
  const uint32_t nch = 1u << nl;
  const uint32_t Q = (g.C + nch - 1) / nch;
  const size_t smem = (size_t)S * U * kT * sizeof(float4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Q * KC);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = KC; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (nl) {
    case 0: cudaFuncSetAttribute(v10<8, U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaLaunchKernelEx(&cfg, v10<8, U, S>, g, x, out); break;
    case 1: cudaFuncSetAttribute(v10<7, U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaLaunchKernelEx(&cfg, v10<7, U, S>, g, x, out); break;
    case 2: cudaFuncSetAttribute(v10<6, U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaLaunchKernelEx(&cfg, v10<6, U, S>, g, x, out); break;
    default: cudaFuncSetAttribute(v10<5, U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
             cudaLaunchKernelEx(&cfg, v10<5, U, S>, g, x, out); break;
  }
}

int main(int argc, char** argv) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct S { int N, C, H; };
  std::vector<S> shapes = {{32, 64, 56}, {32, 256, 56}, {32, 128, 28}, {32, 512, 28}, {32, 1024, 14}, {32, 256, 28}, {32, 256, 14}, {32, 512, 14}};
  const size_t maxe = (size_t)32 * 256 * 56 * 56;
  const int rot = 10;
  float* x;
  cudaMalloc(&x, maxe * 4 * rot);
  cudaMemset(x, 0, maxe * 4 * rot);
  double *out, *wsd;
  unsigned* tk;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&wsd, 1 << 26);
  cudaMalloc(&tk, 1 << 18);
  cudaMemset(tk, 0, 1 << 18);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaFuncSetAttribute(vclu<16, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int mult = argc > 1 ? atoi(argv[1]) : 3;
  const bool check = argc > 2 && strcmp(argv[2], "sweep") != 0 && strcmp(argv[2], "grid") != 0;
  const bool sweep = argc > 2 && strcmp(argv[2], "sweep") == 0;
  const char* only = argc > 3 ? argv[3] : nullptr;
  for (auto s : shapes) {
    const size_t E = (size_t)s.N * s.C * s.H * s.H;
    G g;
    g.C = s.C; g.HW = s.H * s.H; g.HWv = g.HW / 4; g.Lv = s.N * g.HWv;
    g.T = (uint64_t)g.C * g.Lv; g.gap = (uint64_t)(g.C - 1) * g.HWv; g.dhw.init(g.HWv);
    g.count = (double)s.N * g.HW;
    g.grid = sms * mult;
    if (g.T < (uint64_t)g.grid * kT) g.grid = (uint32_t)((g.T + kT - 1) / kT);
    auto timeit = [&](const char* name, auto launch) {
      if (only && !strstr(name, only)) return;
      for (int r = 0; r < 3; ++r) launch(x + (size_t)(r % rot) * maxe);
      if (cudaError_t e = cudaDeviceSynchronize(); e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        cudaGetLastError();
        return;
      }
      if (check) { printf("%s ok\n", name); return; }
      cudaGraph_t gr;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < 20; ++r) launch(x + (size_t)(r % rot) * maxe);
      cudaStreamEndCapture(st, &gr);
      cudaGraphInstantiate(&ge, gr, 0);
      cudaGraphLaunch(ge, st);
      cudaStreamSynchronize(st);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / 100;
      printf("[%d,%d,%d,%d] %-28s %7.2f us %7.1f GB/s\n", s.N, s.C, s.H, s.H, name, us,
             E * 4 / (us * 1e-6) / 1e9);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(gr);
    };
    if (argc > 2 && strcmp(argv[2], "grid") == 0) {
      for (int gcount : {sms * 4, 512, sms * 3, 384, sms * 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "V0 memory order grid=%d", gcount);
        timeit(nm, [&](const float* p) {
          v0<<<gcount, kT, 0, st>>>(reinterpret_cast<const float4*>(p), E / 4, out);
        });
      }
      continue;
    }
    if (sweep) {
      timeit("V0 memory order", [&](const float* p) {
        v0<<<sms * 4, kT, 0, st>>>(reinterpret_cast<const float4*>(p), E / 4, out);
      });
      for (uint32_t nl = 0; nl <= 3; ++nl)
        for (uint32_t kc = 1; kc <= 8; kc *= 2) {
          const uint32_t n = ((g.C + (1u << nl) - 1) >> nl) * kc;
          if (n > (uint32_t)sms * 4 || n < 64) continue;
          char nm[64];
          snprintf(nm, sizeof nm, "V8c nch=%u KC=%u ctas=%u", 1u << nl, kc, n);
          timeit(nm, [&](const float* p) { launch_vct<4>(g, p, out, kc, nl, st, true); });
        }
      continue;
    }
    timeit("V0 memory order", [&](const float* p) {
      v0<<<sms * 4, kT, 0, st>>>(reinterpret_cast<const float4*>(p), E / 4, out);
    });
    timeit("V1 slices, addressing", [&](const float* p) { v1<<<g.grid, kT, 0, st>>>(g, p, out); });
    timeit("V2 + segments/K", [&](const float* p) {
      vseg<false, false><<<g.grid, kT, 0, st>>>(g, p, out, (double2*)wsd, tk);
    });
    timeit("V3 + tail (current)", [&](const float* p) {
      vseg<true, false><<<g.grid, kT, 0, st>>>(g, p, out, (double2*)wsd, tk);
    });
    timeit("V4 + pipelined rounds", [&](const float* p) {
      vseg<true, true><<<g.grid, kT, 0, st>>>(g, p, out, (double2*)wsd, tk);
    });
    {
      G g2 = g;
      g2.grid = (uint32_t)((g.T + 8 * kT - 1) / (8 * kT));
      timeit("V5 tail, 1 round per CTA", [&](const float* p) {
        vseg<true, false><<<g2.grid, kT, 0, st>>>(g2, p, out, (double2*)wsd, tk);
      });
      g2.grid = (uint32_t)((g.T + 4 * kT - 1) / (4 * kT));
      timeit("V6 tail, 4 units per thread", [&](const float* p) {
        vseg<true, false><<<g2.grid, kT, 0, st>>>(g2, p, out, (double2*)wsd, tk);
      });
      auto qof = [&](int slots, int kc) {
        uint32_t qmax = slots / kc;
        uint32_t per = (g.C + qmax - 1) / qmax;
        return (g.C + per - 1) / per;
      };
      {
        uint32_t Q = qof(sms * 3, 8);
        timeit("V7 cluster8 mb3", [&](const float* p) { vclu<8, 3><<<Q * 8, kT, 0, st>>>(g, p, out, Q); });
        timeit("V7x cluster8 local", [&](const float* p) { vclu<8, 3, 0><<<Q * 8, kT, 0, st>>>(g, p, out, Q); });
        Q = qof(sms * 4, 8);
        timeit("V7 cluster8 mb4", [&](const float* p) { vclu<8, 4><<<Q * 8, kT, 0, st>>>(g, p, out, Q); });
        Q = qof(sms * 4, 4);
        timeit("V7 cluster4 mb4", [&](const float* p) { vclu<4, 4><<<Q * 4, kT, 0, st>>>(g, p, out, Q); });
        Q = qof(sms * 4, 16);
        for (int mb : {3, 4}) {
          const uint32_t slots = sms * mb;
          uint32_t bestK = 1, bestL = 0, bestN = 0;
          for (uint32_t nl = 0; nl <= 3; ++nl)
            for (uint32_t kc = 1; kc <= 8; ++kc) {
              const uint32_t n = ((g.C + (1u << nl) - 1) >> nl) * kc;
              if (n <= slots && n > bestN) { bestN = n; bestK = kc; bestL = nl; }
            }
          char nm[64];
          snprintf(nm, sizeof nm, "V8 ct mb%d KC=%u nch=%u", mb, bestK, 1u << bestL);
          if (mb == 3) continue;
          timeit(nm, [&](const float* p) { launch_vct<4>(g, p, out, bestK, bestL, st); });
          timeit("V8c compile-time tpc", [&](const float* p) { launch_vct<4>(g, p, out, bestK, bestL, st, true); });
          timeit("V8f compile-time tpc, fp32 acc", [&](const float* p) { launch_vct<4, true>(g, p, out, bestK, bestL, st, true); });
          timeit("V8t1 no reduction tail", [&](const float* p) { launch_vct<4, false, 1>(g, p, out, bestK, bestL, st, true); });
          timeit("V8t2 block reduce only", [&](const float* p) { launch_vct<4, false, 2>(g, p, out, bestK, bestL, st, true); });
          if (bestL == 0) timeit("V8p pipelined (nch=1)", [&](const float* p) { launch_vct<4, false, 5>(g, p, out, bestK, bestL, st, true); });
          timeit("V8t3 linear addresses", [&](const float* p) { launch_vct<4, false, 3>(g, p, out, bestK, bestL, st, true); });
          timeit("V10 cp.async ring U4 S3", [&](const float* p) { launch_v10<4, 3>(g, p, out, bestK, bestL, st); });
          timeit("V10 cp.async ring U4 S4", [&](const float* p) { launch_v10<4, 4>(g, p, out, bestK, bestL, st); });
          timeit("V10 cp.async ring U2 S6", [&](const float* p) { launch_v10<2, 6>(g, p, out, bestK, bestL, st); });
          timeit("V10 cp.async ring U8 S2", [&](const float* p) { launch_v10<8, 2>(g, p, out, bestK, bestL, st); });
          {
            const uint32_t g4 = (uint32_t)((g.T + kT * 4 - 1) / (kT * 4));
            timeit("V9 nonpersistent flat UPT4", [&](const float* p) { v9<4><<<g4, kT, 0, st>>>(g, p, out, (double2*)wsd, tk); });
            const uint32_t g8 = (uint32_t)((g.T + kT * 8 - 1) / (kT * 8));
            timeit("V9 nonpersistent flat UPT8", [&](const float* p) { v9<8><<<g8, kT, 0, st>>>(g, p, out, (double2*)wsd, tk); });
            const uint32_t g2 = (uint32_t)((g.T + kT * 2 - 1) / (kT * 2));
            timeit("V9 nonpersistent flat UPT2", [&](const float* p) { v9<2><<<g2, kT, 0, st>>>(g, p, out, (double2*)wsd, tk); });
          }
          timeit("V8t4 incremental addresses", [&](const float* p) { launch_vct<4, false, 4>(g, p, out, bestK, bestL, st, true); });
        }
        timeit("V7 cluster16 mb4", [&](const float* p) { vclu<16, 4><<<Q * 16, kT, 0, st>>>(g, p, out, Q); });
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
