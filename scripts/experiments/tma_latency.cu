// Calibration: latency of cp.async.bulk (global -> shared, mbarrier completion) on B200,
// one load at a time vs `depth` loads in flight per CTA, 1 CTA vs all SMs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void k(const char* src, size_t span, int bytes, int depth, int iters, unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint64_t rng = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  unsigned long long tot = 0, n = 0;
  uint64_t t0[8];
  uint32_t ph[8] = {0};
  auto issue = [&](int i) {
    rng = rng * 6364136223846793005ull + 1442695040888963407ull;
    size_t off = ((rng >> 20) % (span / bytes)) * (size_t)bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(bytes));
    t0[i] = gt();
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(sm + (size_t)i * bytes)), "l"(src + off), "r"(bytes), "r"(sa(&bar[i])) : "memory");
  };
  for (int i = 0; i < depth; ++i) issue(i);
  for (int it = 0; it < iters; ++it) {
    const int i = it % depth;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa(&bar[i])), "r"(ph[i]));
    ph[i] ^= 1;
    const uint64_t t1 = gt();
    if (it >= depth) { tot += t1 - t0[i]; ++n; }
    issue(i);
  }
  out[2 * blockIdx.x] = tot; out[2 * blockIdx.x + 1] = n;
}
int main() {
  size_t span = (size_t)4 << 30;
  char* src; cudaMalloc(&src, span); cudaMemset(src, 1, span);
  unsigned long long* out; cudaMalloc(&out, 2 * 1024 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int ctas, bytes, depth; size_t span; };
  C cs[] = {{1, 32768, 1, span}, {1, 32768, 1, 1 << 20}, {1, 8192, 1, span}, {1, 32768, 4, span},
            {sms, 32768, 1, span}, {sms, 32768, 5, span}, {sms, 8192, 5, span}, {sms, 32768, 5, 64 << 20}};
  for (auto c : cs) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k<<<c.ctas, 32, c.bytes * c.depth>>>(src, c.span, c.bytes, c.depth, iters, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2 * 1024]; cudaMemcpy(h, out, 16 * c.ctas, cudaMemcpyDeviceToHost);
    double tot = 0, n = 0; for (int i = 0; i < c.ctas; ++i) { tot += h[2 * i]; n += h[2 * i + 1]; }
    printf("ctas %3d bytes %6d depth %d span %6zu MB: latency %.2f us, throughput %.2f TB/s (%s)\n", c.ctas, c.bytes,
           c.depth, c.span >> 20, tot / n / 1e3, (double)c.ctas * iters * c.bytes / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
}
