// Throughput of the instructions the BN kernels' fp64 arithmetic leans on (B200):
// F2F.F64.F32, F2F.F32.F64, DADD, DFMA, FFMA, LDS.128. Each kernel runs a long dependent-
// free stream of one instruction kind over many warps; ops/clk/SM = ops / (time * clk * SMs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o convbench convbench.cu && ./convbench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_f2f64(const float* in, double* out) {
  float a = in[threadIdx.x], b = a + 1.f, c = a + 2.f, d = a + 3.f;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < ITERS; ++i) {
    s0 = (double)a; s1 = (double)b; s2 = (double)c; s3 = (double)d;  // 4 F2F, no DADD
    a = __int_as_float(__double2loint(s0) ^ 1); b = __int_as_float(__double2hiint(s1));
    c = __int_as_float(__double2hiint(s2) + 1); d = __int_as_float(__double2hiint(s3) + 2);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

__global__ void k_dadd(const float* in, double* out) {
  double a = in[threadIdx.x], b = a + 1, c = a + 2, d = a + 3, e = 1e-9;
  for (int i = 0; i < ITERS; ++i) { a += e; b += e; c += e; d += e; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_ffma(const float* in, double* out) {
  float a = in[threadIdx.x], b = a + 1, c = a + 2, d = a + 3, e = 1.0001f;
  for (int i = 0; i < ITERS; ++i) { a = fmaf(a, e, 1e-9f); b = fmaf(b, e, 1e-9f); c = fmaf(c, e, 1e-9f); d = fmaf(d, e, 1e-9f); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_f2f32(const float* in, double* out) {
  double a = in[threadIdx.x], b = a + 1, c = a + 2, d = a + 3;
  float s = 0;
  for (int i = 0; i < ITERS; ++i) {
    float fa = (float)a, fb = (float)b, fc = (float)c, fd = (float)d;  // 4 F2F.F32.F64
    a = __hiloint2double(__float_as_int(fa), 1); b = __hiloint2double(__float_as_int(fb), 2);
    c = __hiloint2double(__float_as_int(fc), 3); d = __hiloint2double(__float_as_int(fd), 4);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + s;
}

__global__ void k_lds(const float* in, double* out) {
  __shared__ float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(in[0], 1, 2, 3);
  __syncthreads();
  float acc = 0;
  int j = threadIdx.x;
  for (int i = 0; i < ITERS; ++i) {
    float4 v = buf[(j + i) & 1023];
    acc += v.x;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class K>
void run(const char* name, K k, int opsPerIter, const float* in, double* out, int sms) {
  const int blocks = sms * 4, threads = 512;
  k<<<blocks, threads>>>(in, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(in, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = (double)blocks * threads * ITERS * opsPerIter;
  double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("{\"op\": \"%s\", \"ms\": %.3f, \"ops_per_clk_per_sm\": %.1f}\n", name, ms, per_clk_sm);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* in; double* out;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, (size_t)sms * 4 * 512 * 8);
  run("F2F.F64.F32", k_f2f64, 4, in, out, sms);
  run("F2F.F32.F64", k_f2f32, 4, in, out, sms);
  run("DADD", k_dadd, 4, in, out, sms);
  run("FFMA", k_ffma, 4, in, out, sms);
  run("LDS.128 (1 per iter, elements x4)", k_lds, 1, in, out, sms);
  return 0;
}
