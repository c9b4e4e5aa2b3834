// launchlat.cu — per-launch overhead of short streaming kernels on B200: plain stream
// launches vs CUDA graph vs programmatic dependent launch (PDL) inside a graph.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/launchlat tools/launchlat.cu
#include <cuda_runtime.h>
#include <cstdio>

template <bool PDL>
__global__ void __launch_bounds__(256) rd(const float4* __restrict__ x, size_t n4, double* out) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  double a = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i + u * stride < n4) v[u] = __ldg(&x[i + u * stride]);
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i + u * stride < n4) a += (double)v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  if (a == 12345.0) out[0] = a;
}

int main() {
  float4* x; double* out;
  const size_t total4 = (size_t)1 << 26;
  cudaMalloc(&x, total4 * 16); cudaMalloc(&out, 8); cudaMemset(x, 0, total4 * 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (size_t mb : {1, 6, 26, 103}) {
    const size_t n4 = mb * 1000000 / 16;
    const int rot = (int)(total4 / n4 > 8 ? 8 : total4 / n4);
    const int nk = 64;
    unsigned grid = sms * 4;
    auto launch = [&](int i, bool pdl) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      if (pdl) cudaLaunchKernelEx(&cfg, rd<true>, (const float4*)(x + (i % rot) * n4), n4, out);
      else cudaLaunchKernelEx(&cfg, rd<false>, (const float4*)(x + (i % rot) * n4), n4, out);
    };
    for (int mode = 0; mode < 3; ++mode) {  // 0 stream, 1 graph, 2 graph+PDL
      cudaGraphExec_t ge = nullptr;
      if (mode > 0) {
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < nk; ++i) launch(i, mode == 2);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
      } else {
        for (int i = 0; i < nk; ++i) launch(i, false);
      }
      cudaStreamSynchronize(st);
      cudaEventRecord(e0, st);
      for (int r = 0; r < 5; ++r) {
        if (mode > 0) cudaGraphLaunch(ge, st);
        else for (int i = 0; i < nk; ++i) launch(i, false);
      }
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / (5 * nk);
      printf("%4zu MB %-12s %7.2f us/kernel  %7.1f GB/s\n", mb,
             mode == 0 ? "stream" : mode == 1 ? "graph" : "graph+PDL", us, n4 * 16 / (us * 1e3));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
