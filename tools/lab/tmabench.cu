// TMA fill throughput per SM (B200), the producer-conv mainloop's suspected bound: one CTA
// per SM, one thread issues 2-D tiled TMA loads (128-byte rows, 128B swizzle) into an
// S-stage ring, another thread releases each stage as soon as it lands (no MMA). Reports
// bytes per SM clock for box heights / boxes per stage / ring depths, from an
// L2-resident 32 MB tensor (the conv's operands are re-read from L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmabench tmabench.cu -lcuda && ./tmabench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1)
    k_fill(const __grid_constant__ CUtensorMap tm, int stages, int boxes, int rows, int iters,
           int nrows_total, int producers, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t stage_bytes = (uint32_t)boxes * rows * 128;
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
  const int pw = threadIdx.x >> 5;  // producer warps 0 and 2 (lane 0) split the iterations
  if ((threadIdx.x & 31) == 0 && (pw == 0 || (pw == 2 && producers == 2))) {  // producer
    for (int it = pw == 0 ? 0 : 1; it < iters; it += producers) {
      const int s = it % stages;
      if (it >= stages) {
        const uint32_t par = ((it / stages) & 1) ^ 1;
        asm volatile("{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes) : "memory");
      for (int b = 0; b < boxes; ++b) {
        // (a power-of-two mask: a 64-bit modulo here cost ~250 clocks per box)
        const int row0 = (int)(((uint32_t)(blockIdx.x * 997 + it * boxes + b) * (uint32_t)rows) &
                               (uint32_t)(nrows_total - 1));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su32(smem + s * stage_bytes + b * rows * 128)),
            "l"(&tm), "r"(su32(&full[s])), "r"(0), "r"(row0)
            : "memory");
      }
    }
  } else if (threadIdx.x == 32) {  // consumer: release each stage when it lands
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

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const int nrows = 262144;  // x 128 B = 32 MB
  void* buf;
  cudaMalloc(&buf, (size_t)nrows * 128);
  cudaMemset(buf, 1, (size_t)nrows * 128);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int cfg[][3] = {{4, 2, 128}, {6, 2, 128}, {8, 2, 128}, {6, 1, 256}, {6, 4, 64},
                        {4, 3, 128}, {3, 2, 256}, {12, 1, 128}, {6, 2, 64}, {2, 2, 128},
                        {1, 2, 128}, {12, 2, 64}};
  for (int producers = 1; producers <= 2; ++producers)
  for (auto& c : cfg) {
    const int stages = c[0], boxes = c[1], rows = c[2];
    if (stages % producers) continue;
    CUtensorMap tm;
    const cuuint64_t dims[2] = {64, (cuuint64_t)nrows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {64, (cuuint32_t)rows};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const size_t smem = 1024 + (size_t)stages * boxes * rows * 128 + 16 * stages;
    cudaFuncSetAttribute(k_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep)
      k_fill<<<sms, 128, smem>>>(tm, stages, boxes, rows, iters, nrows, producers, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mx = 0, avg = 0;
    for (int i = 0; i < sms; ++i) { mx = h[i] > mx ? h[i] : mx; avg += h[i]; }
    avg /= sms;
    const double bytes = (double)iters * boxes * rows * 128;
    printf("{\"producers\": %d, \"stages\": %d, \"boxes\": %d, \"rows\": %d, \"stage_kb\": %d, \"bytes_per_clk_sm\": %.1f, \"chip_tb_s_at_1.92ghz\": %.2f}\n",
           producers, stages, boxes, rows, boxes * rows * 128 / 1024, bytes / avg, bytes / avg * sms * 1.92e9 / 1e12);
  }
  return 0;
}
