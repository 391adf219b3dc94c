// Microbenchmark: MUFU ex2 throughput, f32 vs bf16x2 vs f16x2 (elements / clock / SM).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
__global__ void k_f32(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bf16x2(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) { __nv_bfloat162 v = __floats2bfloat162_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *(uint32_t*)&v; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) { __nv_bfloat162 v = *(__nv_bfloat162*)&a[i]; s += __low2float(v) + __high2float(v); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f16x2(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) { __half2 v = __floats2half2_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *(uint32_t*)&v; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) { __half2 v = *(__half2*)&a[i]; s += __low2float(v) + __high2float(v); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, blocks = sms * 4, thr = 512;
  for (int rep = 0; rep < 2; ++rep) {
    for (int kind = 0; kind < 3; ++kind) {
      cudaEventRecord(a);
      if (kind == 0) k_f32<<<blocks, thr>>>(out, iters);
      if (kind == 1) k_bf16x2<<<blocks, thr>>>(out, iters);
      if (kind == 2) k_f16x2<<<blocks, thr>>>(out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double elems = (double)blocks * thr * iters * 8 * (kind ? 2 : 1);
      double per_clk_sm = elems / (ms * 1e-3) / sms / (clk * 1e3);
      if (rep) printf("%s: %.3f ms, %.1f elements/clk/SM (at the nominal %d MHz)\n",
                      kind == 0 ? "ex2.f32" : kind == 1 ? "ex2.bf16x2" : "ex2.f16x2", ms, per_clk_sm, clk / 1000);
    }
  }
  return 0;
}
