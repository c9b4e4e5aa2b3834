// cgbn_tma.cuh — TMA bulk-copy streaming kernels for the CGBN hot path (sm_100a).
//
// Opt-in (CGBN_PATH=tma) statistics reductions for NCHW activations whose plane length
// HW is a multiple of 4 floats (every plane piece is then 16-byte aligned, as
// cp.async.bulk requires). Measured against the register kernels on every ResNet-50 /
// FPN shape they were 5-10% slower on large planes and up to 2.5x slower on 14x14
// planes (one producer lane issuing hundreds of 784-byte bulk copies), so the register
// kernels are the default; kept for A/B measurement. One persistent CTA per SM: warp kConsumerWarps is the producer — one elected lane walks the CTA's slice
// of the channel-major float stream and issues 1-D bulk copies
//   cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes
// of plane pieces into a kStages-deep shared-memory ring (full/empty mbarrier pairs);
// the kConsumerWarps consumer warps reduce or transform each stage out of shared memory.
// With ~190 KB per SM in flight the HBM pipe stays full independent of register
// pressure, and small tensors are fetched in one prefetch wave.
//
// A chunk (one ring stage) never crosses a channel: the stream slice [f0, f1) of CTA b
// is cut at channel boundaries and at kChunk floats; a chunk may hold several plane
// pieces (planes of one channel are C*HW apart in memory), each its own bulk copy.
// Cross-CTA statistics use the same slot (b + c) / arrival-ticket fold as the
// register kernels in cgbn.cu, so the result is deterministic.
#pragma once

namespace tma {

constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreadsTma = kConsumers + 32;
constexpr int kStages = 6;
constexpr uint32_t kStageBytes = 32768;  // per stage, split over the input streams
constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 2 * kStages * sizeof(uint64_t) + 128;

struct TGeom {
  uint32_t C, HW;
  uint32_t L;      // floats per channel stream (N*HW)
  uint32_t grid;
  uint64_t T4;     // C*L/4 (slices are cut in 4-float units)
  FastDiv dhw;     // division by HW
  double count;    // N*HW
};

__device__ __forceinline__ uint64_t tslice_begin(const TGeom& g, uint32_t b) {
  return ((uint64_t)b * g.T4 / g.grid) * 4;
}
// CTA whose slice contains float position f (f multiple of 4).
__device__ __forceinline__ uint32_t tcta_of(const TGeom& g, uint64_t f) {
  return (uint32_t)((((f >> 2) + 1) * (uint64_t)g.grid - 1) / g.T4);
}
// element offset of float w of channel c's stream (w % 4 == 0 keeps float4 in a plane)
__device__ __forceinline__ size_t toff(const TGeom& g, uint32_t c, uint32_t w) {
  const uint32_t n = g.dhw.div(w);
  return ((size_t)n * g.C + c) * g.HW + (w - n * g.HW);
}

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

struct Chunk {
  uint32_t c, w, nf;  // channel, first float of the chunk in the channel stream, floats
};

// Deterministic chunk walk of this CTA's slice (producer and consumers run the same one).
struct ChunkWalk {
  uint64_t f, f1;
  uint32_t cap;  // floats per chunk per stream
  __device__ __forceinline__ bool next(const TGeom& g, Chunk& ch) {
    if (f >= f1) return false;
    const uint32_t c = (uint32_t)(f / g.L);
    const uint64_t cbase = (uint64_t)c * g.L;
    const uint32_t w = (uint32_t)(f - cbase);
    const uint64_t cend = min(f1, cbase + g.L);
    const uint32_t nf = (uint32_t)min((uint64_t)cap, cend - f);
    ch = Chunk{c, w, nf};
    f += nf;
    return true;
  }
};

template <int NIN>
struct Ring {
  float* buf;  // kStages x NIN x cap floats
  uint64_t* full;
  uint64_t* empty;
  uint32_t cap;
  __device__ __forceinline__ float* stage(int s, int in) const {
    return buf + ((size_t)s * NIN + in) * cap;
  }
};

template <int NIN>
__device__ __forceinline__ Ring<NIN> ring_setup(unsigned char* smem) {
  Ring<NIN> R;
  R.cap = kStageBytes / (4 * NIN);
  R.buf = reinterpret_cast<float*>(smem);
  R.full = reinterpret_cast<uint64_t*>(smem + (size_t)kStages * kStageBytes);
  R.empty = R.full + kStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  return R;
}

// Producer: one lane streams every chunk of the slice into the ring.
template <int NIN>
__device__ __forceinline__ void produce(const TGeom& g, const Ring<NIN>& R,
                                        const float* __restrict__ in0,
                                        const float* __restrict__ in1) {
  ChunkWalk walk{tslice_begin(g, blockIdx.x), tslice_begin(g, blockIdx.x + 1), R.cap};
  Chunk ch;
  uint32_t k = 0;
  while (walk.next(g, ch)) {
    const int s = (int)(k % kStages);
    const uint32_t r = k / kStages;
    if (r > 0) mbar_wait(&R.empty[s], (r - 1) & 1);
    mbar_expect_tx(&R.full[s], ch.nf * 4u * NIN);
    uint32_t p = 0, w = ch.w;
    while (p < ch.nf) {
      const uint32_t n = g.dhw.div(w);
      const uint32_t h = w - n * g.HW;
      const uint32_t len = min(ch.nf - p, g.HW - h);
      const size_t off = ((size_t)n * g.C + ch.c) * g.HW + h;
      bulk_g2s(R.stage(s, 0) + p, in0 + off, len * 4u, &R.full[s]);
      if (NIN == 2) bulk_g2s(R.stage(s, 1) + p, in1 + off, len * 4u, &R.full[s]);
      p += len;
      w += len;
    }
    ++k;
  }
}

// ---------------------------------------------------------------------------------
// Reductions (forward statistics, backward sums) over the ring.

template <class Op>
__device__ __forceinline__ void tma_finish_channel(const TGeom& g, Op& op, uint32_t c, double S1,
                                                   double S2, double* __restrict__ out,
                                                   double2* __restrict__ ws,
                                                   unsigned* __restrict__ tickets, double* sa,
                                                   double* sb, int* s_last) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  S1 = warp_sum(S1);
  S2 = warp_sum(S2);
  if (l == 0) { sa[w] = S1; sb[w] = S2; }
  consumer_sync();
  const uint64_t cbase = (uint64_t)c * g.L;
  const uint32_t b0 = tcta_of(g, cbase), b1 = tcta_of(g, cbase + g.L - 4);
  if (threadIdx.x == 0) {
    S1 = sa[0]; S2 = sb[0];
#pragma unroll
    for (int i = 1; i < kConsumerWarps; ++i) { S1 += sa[i]; S2 += sb[i]; }
    int last = 0;
    if (b0 == b1) {
      op.finish_stats(g.C, g.count, c, S1, S2, out);
    } else {
      ws[(size_t)blockIdx.x + c] = make_double2(S1, S2);
      __threadfence();
      last = atomicAdd(&tickets[c], 1u) == b1 - b0;
    }
    *s_last = last;
  }
  consumer_sync();
  if (*s_last && w == 0) {
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
      op.finish_stats(g.C, g.count, c, x1, x2, out);
      tickets[c] = 0u;
    }
  }
  consumer_sync();  // sa/sb/s_last reuse
}

// Op interface (TMA flavour): kIn, init_channel(g, c), acc4(const float4* in[kIn], a, b),
// finish_stats(C, count, c, S1, S2, out).
template <class Op>
__global__ void __launch_bounds__(kThreadsTma, 1)
k_tma_reduce(TGeom g, Op op, double* __restrict__ out, double2* __restrict__ ws,
             unsigned* __restrict__ tickets) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double sa[kConsumerWarps], sb[kConsumerWarps];
  __shared__ int s_last;
  constexpr int NIN = Op::kIn;
  const Ring<NIN> R = ring_setup<NIN>(smem);
  if (threadIdx.x >= kConsumers) {
    if (threadIdx.x == kConsumers) produce<NIN>(g, R, op.in0(), op.in1());
    return;
  }
  ChunkWalk walk{tslice_begin(g, blockIdx.x), tslice_begin(g, blockIdx.x + 1), R.cap};
  Chunk ch;
  uint32_t k = 0;
  uint32_t cur = 0xffffffffu;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  while (walk.next(g, ch)) {
    if (ch.c != cur) {
      if (cur != 0xffffffffu)
        tma_finish_channel(g, op, cur, a0 + a1, b0 + b1, out, ws, tickets, sa, sb, &s_last);
      a0 = a1 = b0 = b1 = 0.0;
      cur = ch.c;
      op.init_channel(g.C, g.HW, cur);
    }
    const int s = (int)(k % kStages);
    mbar_wait(&R.full[s], (k / kStages) & 1);
    const float4* p0 = reinterpret_cast<const float4*>(R.stage(s, 0));
    const float4* p1 = reinterpret_cast<const float4*>(R.stage(s, NIN - 1));
    const uint32_t n4 = ch.nf >> 2;
    uint32_t q = threadIdx.x;
    for (; q + kConsumers < n4; q += 2 * kConsumers) {
      op.acc4(p0[q], p1[q], a0, b0);
      op.acc4(p0[q + kConsumers], p1[q + kConsumers], a1, b1);
    }
    if (q < n4) op.acc4(p0[q], p1[q], a0, b0);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&R.empty[s]);
    ++k;
  }
  if (cur != 0xffffffffu)
    tma_finish_channel(g, op, cur, a0 + a1, b0 + b1, out, ws, tickets, sa, sb, &s_last);
}

struct TmaStats {
  static constexpr int kIn = 1;
  const float* __restrict__ x;
  double K;
  __device__ const float* in0() const { return x; }
  __device__ const float* in1() const { return x; }
  __device__ __forceinline__ void init_channel(uint32_t C, uint32_t HW, uint32_t c) {
    (void)C;
    K = (double)__ldg(x + (size_t)c * HW);  // first element of channel c (n = 0, hw = 0)
  }
  __device__ __forceinline__ void acc4(const float4& v, const float4&, double& a,
                                       double& b) const {
    const double d0 = (double)v.x - K, d1 = (double)v.y - K;
    const double d2 = (double)v.z - K, d3 = (double)v.w - K;
    a += (d0 + d1) + (d2 + d3);
    b = __fma_rn(d0, d0, b);
    b = __fma_rn(d1, d1, b);
    b = __fma_rn(d2, d2, b);
    b = __fma_rn(d3, d3, b);
  }
  __device__ __forceinline__ void finish_stats(uint32_t C, double n, uint32_t c, double S1,
                                               double S2, double* __restrict__ out) const {
    const double mean = K + S1 / n;
    const double M2 = fmax(S2 - S1 * (S1 / n), 0.0);
    out[c] = mean;
    out[C + c] = M2;
    if (c == 0) out[2 * C] = n;
  }
};

template <bool RELU>
struct TmaBwd {
  static constexpr int kIn = 2;
  const float* __restrict__ dy;
  const float* __restrict__ x;
  const double* __restrict__ saved;
  const float* __restrict__ gamma;
  const float* __restrict__ beta;
  double mean, P, Q;
  __device__ const float* in0() const { return dy; }
  __device__ const float* in1() const { return x; }
  __device__ __forceinline__ void init_channel(uint32_t C, uint32_t HW, uint32_t c) {
    (void)HW;
    mean = saved[c];
    if (RELU) affine_coeffs(mean, saved[2 * C + c], (double)gamma[c], (double)beta[c], P, Q);
  }
  __device__ __forceinline__ void one(float gf, float xf, double& a, double& b) const {
    double gk = (double)gf;
    if (RELU && !(bn_out(P, Q, xf) > 0.0)) gk = 0.0;
    a += gk;
    b = __fma_rn(gk, (double)xf - mean, b);
  }
  __device__ __forceinline__ void acc4(const float4& gv, const float4& xv, double& a,
                                       double& b) const {
    one(gv.x, xv.x, a, b);
    one(gv.y, xv.y, a, b);
    one(gv.z, xv.z, a, b);
    one(gv.w, xv.w, a, b);
  }
  __device__ __forceinline__ void finish_stats(uint32_t C, double, uint32_t c, double S1,
                                               double S2, double* __restrict__ out) const {
    out[c] = S1;
    out[C + c] = S2;
  }
};

}  // namespace tma
