// im2col TMA fill throughput per SM (B200), the 3x3 producer conv's mainloop bound: one CTA
// per SM, one thread issues per ring stage one tiled W box (128 x 64 bf16, 16 KB) and the
// stage's x pixels as im2col boxes of `box` pixels (64 channels each, 128B swizzle), walking
// taps / k-blocks / pixel tiles as the conv does; another thread releases each stage as soon
// as it lands (no MMA). x is [32][H][W][C] NHWC bf16, L2-resident after the first pass (as
// in the conv). Reports bytes per SM clock for pixel-tile widths and box sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o im2colbench im2colbench.cu && ./im2colbench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1)
    k_fill(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
           int stages, int pix, int box, int iters, int H, int W, int C, int N, int Cout,
           int producers, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t stage_bytes = 16384u + (uint32_t)pix * 128u;
  uint64_t* full = (uint64_t*)(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  const int kblocks = C / 64, HW = H * W, M = N * HW;
  const int tiles = M / pix;
  const int pw = threadIdx.x >> 5;  // producer warps 0 and 2 (lane 0) alternate stages
  if ((threadIdx.x & 31) == 0 && (pw == 0 || (pw == 2 && producers == 2))) {
    int tile = blockIdx.x % tiles, tap = 0, kb = 0;
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (producers == 2 && (it & 1) != (pw == 2 ? 1 : 0)) {  // the other producer's stage
        if (++kb == kblocks) {
          kb = 0;
          if (++tap == 9) {
            tap = 0;
            tile += gridDim.x;
            if (tile >= tiles) tile -= tiles;
          }
        }
        continue;
      }
      if (it >= stages) {
        const uint32_t par = ((it / stages) & 1) ^ 1;
        asm volatile("{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
      }
      uint8_t* A = smem + s * stage_bytes;
      uint8_t* B = A + 16384;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(A)),
          "l"(&tmW), "r"(su32(&full[s])), "r"(kb * 64), "r"(0), "r"(tap)
          : "memory");
      const int ty = tap / 3, tx = tap - ty * 3;
      for (int j = 0; j < pix / box; ++j) {
        const int px = tile * pix + j * box;
        const int n = px / HW, rem = px - n * HW, ho = rem / W, wo = rem - ho * W;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(su32(B + j * box * 128)),
            "l"(&tmX), "r"(su32(&full[s])), "r"(kb * 64), "r"(wo - 1), "r"(ho - 1), "r"(n),
            "h"((uint16_t)tx), "h"((uint16_t)ty)
            : "memory");
      }
      if (++kb == kblocks) {
        kb = 0;
        if (++tap == 9) {
          tap = 0;
          tile += gridDim.x;
          if (tile >= tiles) tile -= tiles;
        }
      }
    }
  } else if (threadIdx.x == 32) {  // consumer
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      const uint32_t par = (it / stages) & 1;
      asm volatile("{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n}" ::"r"(su32(&full[s])), "r"(par) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

int main() {
  void *p1 = nullptr, *p2 = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p1, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p2, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p1;
  EncodeIm2colFn enc2 = (EncodeIm2colFn)p2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 256 * sizeof(unsigned long long));
  // (H, W, C): the ResNet-50 stride-1 3x3 layers
  const int shapes[][3] = {{56, 56, 64}, {28, 28, 128}, {14, 14, 256}, {7, 7, 512}};
  const int cfg[][3] = {{128, 128, 6}, {128, 64, 6}, {128, 32, 6}, {256, 256, 4}, {256, 128, 4},
                        {256, 64, 4}};
  for (int producers = 1; producers <= 2; ++producers)
  for (auto& sh : shapes) {
    const int H = sh[0], W = sh[1], C = sh[2], N = 32, Cout = 128;
    void *x, *w;
    const size_t xb = (size_t)N * H * W * C * 2, wb = (size_t)Cout * 9 * C * 2;
    cudaMalloc(&x, xb);
    cudaMalloc(&w, wb);
    cudaMemset(x, 0, xb);
    cudaMemset(w, 0, wb);
    CUtensorMap tmW;
    {
      const cuuint64_t d[3] = {(cuuint64_t)C, (cuuint64_t)Cout, 9};
      const cuuint64_t st[2] = {(cuuint64_t)9 * C * 2, (cuuint64_t)C * 2};
      const cuuint32_t b[3] = {64, 128, 1};
      const cuuint32_t es[3] = {1, 1, 1};
      if (enc(&tmW, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("w encode failed\n");
        return 1;
      }
    }
    for (auto& c : cfg) {
      const int pix = c[0], box = c[1], stages = c[2];
      if ((N * H * W) % pix || stages % producers) continue;
      CUtensorMap tmX;
      const cuuint64_t d[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
      const cuuint64_t st[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
      const int lo[2] = {-1, -1}, hi[2] = {-1, -1};
      const cuuint32_t es[4] = {1, 1, 1, 1};
      if (enc2(&tmX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, d, st, lo, hi, 64, (cuuint32_t)box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("x encode failed\n");
        return 1;
      }
      const size_t smem = 1024 + (size_t)stages * (16384 + pix * 128) + 16 * stages;
      cudaFuncSetAttribute(k_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 2000;
      for (int rep = 0; rep < 2; ++rep)
        k_fill<<<sms, 128, smem>>>(tmW, tmX, stages, pix, box, iters, H, W, C, N, Cout, producers, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[256];
      cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < sms; ++i) avg += h[i];
      avg /= sms;
      const double bytes = (double)iters * (16384 + pix * 128);
      printf("{\"producers\": %d, \"H\": %d, \"C\": %d, \"pix\": %d, \"box\": %d, \"stages\": %d, \"bytes_per_clk_sm\": %.1f, \"clk_per_stage\": %.0f}\n",
             producers, H, C, pix, box, stages, bytes / avg, avg / iters);
    }
    cudaFree(x);
    cudaFree(w);
  }
  return 0;
}
