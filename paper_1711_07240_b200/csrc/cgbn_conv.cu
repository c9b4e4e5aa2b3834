// cgbn_conv.cu — producer fusion: a 1x1 convolution on the tcgen05
// tensor cores whose epilogue emits the BN forward partial of its own output, so the
// statistics pass of the BN forward never re-reads the activation (fwd 12 -> 8 B/elem).
//
// The reference's producer is the conv layer that feeds every BN in its model
// (/root/reference/pkg/src/bigbatch/model.py:235-242: out = cols @ W^T + b, an im2col
// GEMM), followed by sync_bn_forward / bn_forward_local (model.py:247-258), whose first
// step is channel_sum over that output (batchnorm.py:118, tensor.py:143-153). Here the
// GEMM is the pointwise (1x1) case, z[n][co][p] = sum_ci W[co][ci] * x[n][ci][p] + b[co],
// NCHW, bf16 operands, fp32 accumulation in TMEM, z stored as fp32 or bf16, and the
// epilogue reduces each output channel of its tile to (mean, centred M2) of the values
// *as stored* — the partial cgbn_fwd_stats would have computed from z.
//
// Kernel anatomy (one CTA per 128-channel x 128-pixel output tile of one image, 128
// threads, 2 CTAs per SM so one tile's epilogue overlaps the other's loads):
//   warp 0 / lane 0   TMA producer: W tile [128 co][64 ci] (K-major, 128B swizzle) and
//                     x tile [64 ci][128 px] (two 64-pixel boxes, MN-major, 128B swizzle)
//                     into an S-stage ring, mbarrier complete_tx;
//   warp 1 / lane 0   MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128 N=128 K=16,
//                     accumulator in 128 TMEM columns; tcgen05.commit frees ring slots
//                     and finally signals the epilogue;
//   warps 0-3         epilogue: tcgen05.ld 32x32b (thread t owns TMEM lane t = output
//                     channel m0+t, so each thread reduces its own channel with no
//                     cross-thread traffic), + bias, round to the output type, stage
//                     128-byte rows in 128B-swizzled shared memory and TMA-store them
//                     (clipping the pixel / channel tails); a second TMEM sweep forms the
//                     tile's centred M2 around the tile mean.
// Tile partials (mean, M2) go to a tile-major slot array; k_conv_fold merges the tiles
// of each channel with Chan's update in a fixed order into this rank's forward partial
// [mean (C) | M2 (C) | count] (include/cgbn.h), which the unchanged exchange and
// cgbn_fwd_normalize consume.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "cgbn.h"

// Error reporting shared with cgbn.cu (its thread-local cgbn_last_error message).
int cgbn_internal_set_error(int code, const char* msg);

namespace {

constexpr int BM = 128;       // output channels per tile (TMEM lanes)
constexpr int BN = 128;       // pixels per tile (TMEM columns)
constexpr int BK = 64;        // input channels per ring stage (128 B of bf16)
constexpr int kConvThreads = 128;
constexpr uint32_t kTileA = BM * BK * 2;      // 16 KB
constexpr uint32_t kTileB = BK * BN * 2;      // 16 KB (two 64-pixel boxes of 8 KB)
constexpr uint32_t kStage = kTileA + kTileB;  // 32 KB
constexpr uint32_t kStageOut = BM * 128;      // one 128-byte row per channel: 16 KB

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return cgbn_internal_set_error(code, buf);
}

// ------------------------------------------------------------------------------------
// PTX wrappers (sm_100a)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CGBN_MBW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CGBN_MBW_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tm),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor (tcgen05): start >> 4 in [0,14), leading byte offset
// >> 4 in [16,30), stride byte offset >> 4 in [32,46), version 1 at [46,48), layout type
// at [61,64) (2 = 128-byte swizzle).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, A K-major, B MN-major, N, M.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

template <class OutT>
struct OutTraits;
template <>
struct OutTraits<float> {
  static constexpr int kCols = 32;  // columns per 128-byte staged row
  __device__ static float round(float v) { return v; }
};
template <>
struct OutTraits<__nv_bfloat16> {
  static constexpr int kCols = 64;
  __device__ static float round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
};

struct ConvArgs {
  const float* bias;  // may be null
  double2* slots;     // [tiles per channel][Cout] (mean, M2); null = no statistics
  int Cout, HW, tilesP, mtiles, kblocks;
};

// One output tile. S = ring stages.
template <int S, class OutT>
__global__ void __launch_bounds__(kConvThreads, 2)
    k_conv1x1(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
              const __grid_constant__ CUtensorMap tmZ, const ConvArgs a) {
  constexpr int kCols = OutTraits<OutT>::kCols;
  constexpr int kChunks = BN / kCols;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* ring = smem;                        // S x [A 16 KB | B 16 KB]
  uint8_t* stage_out = smem + S * kStage;      // 2 x 16 KB (double-buffered TMA store)
  uint64_t* full = (uint64_t*)(stage_out + 2 * kStageOut);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bid = blockIdx.x;
  const int mt = bid % a.mtiles;
  const int rest = bid / a.mtiles;
  const int pt = rest % a.tilesP;
  const int img = rest / a.tilesP;
  const int m0 = mt * BM, p0 = pt * BN;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmZ) : "memory");
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // x may be produced by the kernel before us (programmatic dependent launch).
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0 && lane == 0) {
    // TMA producer
    for (int kb = 0; kb < a.kblocks; ++kb) {
      const int s = kb % S;
      if (kb >= S) mbar_wait(&empty[s], ((kb / S) & 1) ^ 1);
      uint8_t* A = ring + s * kStage;
      uint8_t* B = A + kTileA;
      mbar_expect_tx(&full[s], kStage);
      tma_load_2d(A, &tmW, &full[s], kb * BK, m0);
      tma_load_3d(B, &tmX, &full[s], p0, kb * BK, img);
      tma_load_3d(B + kTileB / 2, &tmX, &full[s], p0 + 64, kb * BK, img);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    for (int kb = 0; kb < a.kblocks; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      tc_fence_after();
      const uint32_t A = smem_u32(ring + s * kStage);
      const uint32_t B = A + kTileA;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        // A: K-major rows of 128 B, 8-row atoms 1024 B apart; K step = 32 B in the row.
        // B: MN-major, 64-pixel halves 8 KB apart (LBO), 8-channel groups 1 KB apart
        //    (SBO); K step = 16 rows = 2 KB.
        const uint64_t ad = sdesc(A + k * 32, 16, 1024);
        const uint64_t bd = sdesc(B + k * 2048, kTileB / 2, 1024);
        mma_bf16(tmem, ad, bd, kIdesc, (kb | k) != 0);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(done);
  }
  __syncwarp();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---------------- epilogue: thread t <-> TMEM lane t <-> channel m0 + t
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const int c = m0 + row;
  const bool cvalid = c < a.Cout;
  const float bias = (a.bias != nullptr && cvalid) ? a.bias[c] : 0.f;
  const int nvalid = min(BN, a.HW - p0);
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  double sum = 0.0;
  for (int j = 0; j < kChunks; ++j) {
    uint32_t packed[32];
#pragma unroll
    for (int h = 0; h < kCols / 32; ++h) {
      float v[32];
      tmem_ld32(trow + j * kCols + h * 32, v);
      // fp64 per element (as the BN statistics kernels): fp32 partial sums lose ~1e-6
      // of a channel mean far from zero, which the reference's 1e-3 floor exposes in y
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float r = OutTraits<OutT>::round(v[i] + bias);
        v[i] = r;
        s4[i & 3] += (j * kCols + h * 32 + i < nvalid) ? (double)r : 0.0;
      }
      sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
      if constexpr (sizeof(OutT) == 4) {
#pragma unroll
        for (int i = 0; i < 32; ++i) packed[i] = __float_as_uint(v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
          packed[h * 16 + i] = *reinterpret_cast<uint32_t*>(&b2);
        }
      }
    }
    // stage this thread's 128-byte row (128B swizzle: 16-byte chunk q -> q ^ (row & 7))
    uint8_t* buf = stage_out + (j & 1) * kStageOut;
    if (j >= 2) {
      if (threadIdx.x == 0) bulk_wait_read1();
      epi_bar();
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint4 u = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
      *reinterpret_cast<uint4*>(buf + row * 128 + ((q ^ (row & 7)) << 4)) = u;
    }
    fence_proxy_async();
    epi_bar();
    if (threadIdx.x == 0) {
      if (p0 + j * kCols < a.HW) tma_store_3d(&tmZ, buf, p0 + j * kCols, m0, img);
      bulk_commit();  // (an empty group past the pixel tail keeps the group count uniform)
    }
  }

  if (a.slots != nullptr) {
    // second TMEM sweep: centred M2 of the stored values around the tile mean
    const double mean = sum / (double)nvalid;
    double q4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < BN / 32; ++j) {
      if (j * 32 >= nvalid) break;
      float v[32];
      tmem_ld32(trow + j * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const double d =
            (j * 32 + i < nvalid) ? (double)OutTraits<OutT>::round(v[i] + bias) - mean : 0.0;
        q4[i & 3] = fma(d, d, q4[i & 3]);
      }
    }
    const double m2 = (q4[0] + q4[1]) + (q4[2] + q4[3]);
    if (cvalid) {
      const int t = img * a.tilesP + pt;
      a.slots[(size_t)t * a.Cout + c] = make_double2(mean, m2);
    }
  }

  if (threadIdx.x == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, BN);
}

// Merge the per-tile (mean, M2) partials of each channel (Chan's update, fixed order:
// warp w folds tiles w, w + 8, ...; the 8 warp partials are then folded in warp order)
// into the rank's forward partial [mean (C) | M2 (C) | count]. Block = 32 channels x 8
// warps; a warp reads 32 consecutive channels of one tile (512 contiguous bytes).
__global__ void __launch_bounds__(256) k_conv_fold(const double2* __restrict__ slots, int Cout,
                                                   int HW, int tilesP, int tiles,
                                                   double* __restrict__ partial) {
  __shared__ double sn[8][32], smean[8][32], sm2[8][32];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double n = 0.0, mean = 0.0, M2 = 0.0;
  if (c < Cout) {
    for (int t = w; t < tiles; t += 8) {
      const double2 p = slots[(size_t)t * Cout + c];
      const int pt = t % tilesP;
      const double nb = (double)min(BN, HW - pt * BN);
      const double nn = n + nb;
      const double delta = p.x - mean;
      mean = mean + delta * (nb / nn);
      M2 = M2 + p.y + delta * delta * (n * nb / nn);
      n = nn;
    }
  }
  sn[w][lane] = n;
  smean[w][lane] = mean;
  sm2[w][lane] = M2;
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (w == 0 && c < Cout) {
    n = sn[0][lane];
    mean = smean[0][lane];
    M2 = sm2[0][lane];
    for (int r = 1; r < 8; ++r) {
      const double nb = sn[r][lane];
      if (nb == 0.0) continue;
      const double nn = n + nb;
      const double delta = smean[r][lane] - mean;
      mean = mean + delta * (nb / nn);
      M2 = M2 + sm2[r][lane] + delta * delta * (n * nb / nn);
      n = nn;
    }
    partial[c] = mean;
    partial[Cout + c] = M2;
    if (c == 0) partial[2 * Cout] = n;
  }
}

// ------------------------------------------------------------------------------------
// Host side

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

// rank-r tensor map with 128-byte swizzle; dims / strides innermost first (strides in
// bytes, for dims 1..r-1).
int make_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
             const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(CGBN_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, dt, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CGBN_ERR_INVALID, "tensor map encoding failed (CUresult %d)", (int)r);
  return CGBN_OK;
}

constexpr int kStages = 2;

size_t conv_smem_bytes() { return 1024 + kStages * kStage + 2 * kStageOut + 8 * (2 * kStages + 1) + 16; }

template <class OutT>
int launch_conv(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                int64_t Cout, int64_t HW, void* z, double2* slots, cudaStream_t st) {
  CUtensorMap tmW, tmX, tmZ;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)Cin, (cuuint64_t)Cout};
    const cuuint64_t strides[1] = {(cuuint64_t)Cin * 2};
    const cuuint32_t box[2] = {BK, BM};
    if (int rc = make_map(&tmW, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box)) return rc;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)HW, (cuuint64_t)Cin, (cuuint64_t)N};
    const cuuint64_t strides[2] = {(cuuint64_t)HW * 2, (cuuint64_t)(Cin * HW * 2)};
    const cuuint32_t box[3] = {64, BK, 1};
    if (int rc = make_map(&tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x, dims, strides, box)) return rc;
  }
  {
    constexpr int sz = sizeof(OutT);
    const cuuint64_t dims[3] = {(cuuint64_t)HW, (cuuint64_t)Cout, (cuuint64_t)N};
    const cuuint64_t strides[2] = {(cuuint64_t)HW * sz, (cuuint64_t)(Cout * HW * sz)};
    const cuuint32_t box[3] = {(cuuint32_t)OutTraits<OutT>::kCols, BM, 1};
    const CUtensorMapDataType dt =
        sz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    if (int rc = make_map(&tmZ, dt, 3, z, dims, strides, box)) return rc;
  }
  ConvArgs a;
  a.bias = bias;
  a.slots = slots;
  a.Cout = (int)Cout;
  a.HW = (int)HW;
  a.tilesP = (int)((HW + BN - 1) / BN);
  a.mtiles = (int)((Cout + BM - 1) / BM);
  a.kblocks = (int)((Cin + BK - 1) / BK);
  const size_t smem = conv_smem_bytes();
  auto kern = k_conv1x1<kStages, OutT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long grid = (long long)a.mtiles * a.tilesP * N;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kConvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = getenv("CGBN_NO_PDL") ? 0 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmW, tmX, tmZ, a);
  if (e != cudaSuccess) return fail(CGBN_ERR_CUDA, "conv1x1 launch failed: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

int validate(const void* x, const void* w, const void* z, int64_t N, int64_t Cin, int64_t Cout,
             int64_t HW, int out_dtype) {
  if (!x || !w || !z) return fail(CGBN_ERR_INVALID, "conv1x1: null tensor pointer");
  if (N <= 0 || Cin <= 0 || Cout <= 0 || HW <= 0)
    return fail(CGBN_ERR_INVALID, "conv1x1: extents must be positive");
  if (out_dtype != CGBN_ACT_F32 && out_dtype != CGBN_ACT_BF16)
    return fail(CGBN_ERR_INVALID, "conv1x1: output dtype must be CGBN_ACT_F32 or CGBN_ACT_BF16");
  if (HW % 8 != 0)
    return fail(CGBN_ERR_UNSUPPORTED, "conv1x1: H*W=%lld must be a multiple of 8 (TMA row stride)",
                (long long)HW);
  if (Cin % 8 != 0)
    return fail(CGBN_ERR_UNSUPPORTED, "conv1x1: Cin=%lld must be a multiple of 8", (long long)Cin);
  if (Cout > 65535 || N > 65535 || HW * N > (1ll << 31))
    return fail(CGBN_ERR_INVALID, "conv1x1: extents too large");
  if (((uintptr_t)x | (uintptr_t)w | (uintptr_t)z) & 15)
    return fail(CGBN_ERR_INVALID, "conv1x1: pointers must be 16-byte aligned");
  return CGBN_OK;
}

int tiles_per_channel(int64_t N, int64_t HW) { return (int)(N * ((HW + BN - 1) / BN)); }

}  // namespace

extern "C" {

size_t cgbn_conv1x1_ws_bytes(int64_t N, int64_t Cout, int64_t HW) {
  if (N <= 0 || Cout <= 0 || HW <= 0) return 0;
  return (size_t)tiles_per_channel(N, HW) * (size_t)Cout * sizeof(double2);
}

int cgbn_conv1x1(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                 int64_t Cout, int64_t HW, int out_dtype, void* z, void* stream) {
  if (int rc = validate(x, w, z, N, Cin, Cout, HW, out_dtype)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = out_dtype == CGBN_ACT_F32
               ? launch_conv<float>(x, w, bias, N, Cin, Cout, HW, z, nullptr, st)
               : launch_conv<__nv_bfloat16>(x, w, bias, N, Cin, Cout, HW, z, nullptr, st);
  return rc;
}

int cgbn_conv1x1_stats(const void* x, const void* w, const float* bias, int64_t N, int64_t Cin,
                       int64_t Cout, int64_t HW, int out_dtype, void* z, double* partial,
                       void* ws, size_t ws_bytes, void* stream) {
  if (int rc = validate(x, w, z, N, Cin, Cout, HW, out_dtype)) return rc;
  if (!partial) return fail(CGBN_ERR_INVALID, "conv1x1_stats: partial is NULL");
  const size_t need = cgbn_conv1x1_ws_bytes(N, Cout, HW);
  if (!ws || ws_bytes < need)
    return fail(CGBN_ERR_INVALID, "conv1x1_stats: workspace too small (need %lld, got %lld)",
                (long long)need, (long long)ws_bytes);
  if ((uintptr_t)ws & 15) return fail(CGBN_ERR_INVALID, "conv1x1_stats: workspace must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  double2* slots = (double2*)ws;
  int rc = out_dtype == CGBN_ACT_F32
               ? launch_conv<float>(x, w, bias, N, Cin, Cout, HW, z, slots, st)
               : launch_conv<__nv_bfloat16>(x, w, bias, N, Cin, Cout, HW, z, slots, st);
  if (rc) return rc;
  const int tilesP = (int)((HW + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((Cout + 31) / 32));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = getenv("CGBN_NO_PDL") ? 0 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_conv_fold, (const double2*)slots, (int)Cout, (int)HW,
                                     tilesP, tiles_per_channel(N, HW), partial);
  if (e != cudaSuccess) return fail(CGBN_ERR_CUDA, "conv fold launch failed: %s", cudaGetErrorString(e));
  return CGBN_OK;
}

}  // extern "C"
