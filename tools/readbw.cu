// readbw.cu — B200 streaming-bandwidth microbenchmark used to set the realistic ceiling
// for the CGBN kernels: read-only fp64 statistics vs copy, and the effect of the access
// order (GPU-wide grid-stride sweep vs one contiguous slice per CTA) at ResNet sizes.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/readbw tools/readbw.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

// ORDER 0: grid-stride (unit i -> CTA (i/256) % grid); 1: contiguous slice per CTA.
// MODE 1: fp64 sum + sum of squares; 2: copy.
template <int U, int MODE, int ORDER>
__global__ void __launch_bounds__(256) k(const float4* __restrict__ x, float4* __restrict__ y,
                                         size_t n4, double* out) {
  double a = 0.0, b = 0.0;
  size_t i, end, stride;
  if (ORDER == 0) {
    stride = (size_t)gridDim.x * blockDim.x;
    i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    end = n4;
  } else {
    const size_t per = (n4 + gridDim.x - 1) / gridDim.x;
    i = blockIdx.x * per + threadIdx.x;
    end = min(n4, (blockIdx.x + 1) * per);
    stride = blockDim.x;
  }
  for (; i < end; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < end) v[u] = __ldg(&x[i + u * stride]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * stride >= end) continue;
      if (MODE == 1) {
        const double d0 = (double)v[u].x - 1.0, d1 = (double)v[u].y - 1.0;
        const double d2 = (double)v[u].z - 1.0, d3 = (double)v[u].w - 1.0;
        a += (d0 + d1) + (d2 + d3);
        b = fma(d0, d0, b); b = fma(d1, d1, b); b = fma(d2, d2, b); b = fma(d3, d3, b);
      }
      if (MODE == 2) y[i + u * stride] = v[u];
    }
  }
  if (a + b == 12345.0) out[0] = a + b;
}

template <int U, int MODE, int ORDER>
void run(const char* name, const float4* x, float4* y, size_t n4, double* out, int grid,
         size_t rot) {
  // rotate over `rot` disjoint buffers so every launch streams from HBM
  for (int w = 0; w < 3; ++w) k<U, MODE, ORDER><<<grid, 256>>>(x, y, n4, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it = 30;
  cudaEventRecord(e0);
  for (int r = 0; r < it; ++r)
    k<U, MODE, ORDER><<<grid, 256>>>(x + (r % rot) * n4, y + (r % rot) * n4, n4, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)n4 * 16 * (MODE == 2 ? 2 : 1);
  printf("%-22s %-6s U=%2d grid=%5d %7.1f MB %8.1f GB/s (%.1f us)\n", name,
         ORDER ? "slice" : "stride", U, grid, n4 * 16 / 1e6, bytes / (ms / it * 1e-3) / 1e9,
         ms / it * 1e3);
}

int main() {
  const size_t total4 = (size_t)1 << 27;  // 2 GiB of float4 per buffer
  float4 *x, *y;
  double* out;
  cudaMalloc(&x, total4 * 16);
  cudaMalloc(&y, total4 * 16);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, total4 * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (size_t mb : {1024, 103, 51, 26, 13, 6}) {
    const size_t n4 = mb * 1000000 / 16;
    const size_t rot = total4 / n4 > 16 ? 16 : total4 / n4;
    for (int g : {sms * 3, sms * 4, sms * 8}) {
      run<8, 1, 0>("fp64 stats", x, y, n4, out, g, rot);
      run<8, 1, 1>("fp64 stats", x, y, n4, out, g, rot);
    }
    run<4, 2, 0>("copy", x, y, n4, out, sms * 4, rot);
    run<4, 2, 1>("copy", x, y, n4, out, sms * 4, rot);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
