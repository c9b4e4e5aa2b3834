// orderbw.cu — does the channel-major plane order of a per-channel reduction cost DRAM
// bandwidth vs a linear memory sweep? Reads an NCHW fp32 tensor (fp64 accumulate) in
// (a) memory order (grid-stride float4), (b) channel-major: CTA team per channel walking
// its N planes, (c) plane order: each CTA takes consecutive planes in memory order and
// emits one partial per plane. Timed inside a CUDA graph of 40 launches over rotating
// buffers. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/orderbw tools/orderbw.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void mem_order(const float4* __restrict__ x, size_t n4, double* out) {
  double a = 0, b = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i + u * stride < n4) v[u] = __ldg(&x[i + u * stride]);
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i + u * stride < n4) {
      const double d = (double)v[u].x + v[u].y + v[u].z + v[u].w;
      a += d; b = fma(d, d, b);
    }
  }
  if (a + b == 1234.5) out[0] = a;
}

// one CTA per channel tile (tpc threads per channel), units = float4 of the channel's planes
__global__ void chan_order(const float4* __restrict__ x, int N, int C, int HW4, double* out) {
  const int c = blockIdx.x;
  const int L = N * HW4;
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < L; i += 8 * blockDim.x) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = i + u * blockDim.x;
      if (j < L) { const int n = j / HW4, r = j - n * HW4; v[u] = __ldg(&x[((size_t)n * C + c) * HW4 + r]); }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i + u * blockDim.x < L) {
      const double d = (double)v[u].x + v[u].y + v[u].z + v[u].w;
      a += d; b = fma(d, d, b);
    }
  }
  if (a + b == 1234.5) out[c] = a;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total4 = (size_t)1 << 26;
  float4* x; double* out;
  cudaMalloc(&x, total4 * 16); cudaMalloc(&out, 1 << 20); cudaMemset(x, 0, total4 * 16);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct S { int N, C, H; } shapes[] = {{32,128,28},{32,64,56},{32,256,14},{32,1024,14},{32,256,56}};
  for (auto s : shapes) {
    const int HW4 = s.H * s.H / 4;
    const size_t n4 = (size_t)s.N * s.C * HW4;
    const int rot = (int)(total4 / n4 > 16 ? 16 : total4 / n4);
    for (int mode = 0; mode < 2; ++mode) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 40; ++i) {
        const float4* p = x + (i % rot) * n4;
        if (mode == 0) mem_order<<<sms * 4, 256, 0, st>>>(p, n4, out);
        else chan_order<<<s.C, 256, 0, st>>>(p, s.N, s.C, HW4, out);
      }
      cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
      cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / 40;
      printf("[%d,%d,%d,%d] %-6s %7.2f us %7.1f GB/s\n", s.N, s.C, s.H, s.H,
             mode ? "chan" : "memory", us, n4 * 16 / (us * 1e3));
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
