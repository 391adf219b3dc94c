// Calibration: TMA 2-D tensor loads shaped like the attention K chunks (boxes of 64
// rows x 128 B from a [rows][hd = 128] bf16 pool, SWIZZLE_128B), `nbox` boxes per
// chunk, `depth` chunks in flight per CTA, all SMs: per-chunk latency + throughput.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void k(const __grid_constant__ CUtensorMap map, const char* src, long rows, int nbox, int depth, int iters,
                  int seq, int bulk1d, int opbytes, unsigned long long* out) {
  extern __shared__ __align__(1024) char sm_raw[];
  char* sm = (char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint64_t rng = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  unsigned long long tot = 0, n = 0;
  uint64_t t0[8];
  uint32_t ph[8] = {0};
  long cursor = (long)blockIdx.x * 4096;
  auto issue = [&](int i) {
    long r0;
    if (seq) { r0 = cursor % (rows - 128); cursor += 128; }
    else { rng = rng * 6364136223846793005ull + 1442695040888963407ull; r0 = (long)((rng >> 20) % (uint64_t)(rows / 256 - 2)) * 128; }
    if (bulk1d) {   // nbox contiguous ops of opbytes from row r0
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(nbox * opbytes));
      t0[i] = gt();
      for (int b = 0; b < nbox; ++b)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(sm + ((size_t)i * nbox + b) * opbytes)), "l"(src + r0 * 256 + (size_t)b * opbytes),
                     "r"(opbytes), "r"(sa(&bar[i])) : "memory");
      return;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(nbox * 8192));
    t0[i] = gt();
    for (int b = 0; b < nbox; ++b) {
      const int c0 = (b & 1) * 64, c1 = (int)(r0 + (b >> 1) * 64);
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(sm + ((size_t)i * nbox + b) * 8192)), "l"(&map), "r"(c0), "r"(c1), "r"(sa(&bar[i])) : "memory");
    }
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
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const long rows = 8l << 20;   // 8 M rows x 256 B = 2 GiB
  void* src; cudaMalloc(&src, rows * 256); cudaMemset(src, 1, rows * 256);
  unsigned long long* out; cudaMalloc(&out, 2 * 1024 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  EncFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t d[2] = {128, (cuuint64_t)rows}, st[1] = {256};
  cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int ctas, nbox, depth, bulk1d, opbytes; long span_rows; };
  const long l2rows = (48l << 20) / 256;
  C cs[] = {
    {1, 4, 3, 0, 8192, rows}, {1, 4, 3, 1, 8192, rows}, {1, 1, 3, 1, 32768, rows},
    {1, 4, 3, 0, 8192, l2rows}, {1, 4, 3, 1, 8192, l2rows}, {1, 1, 3, 1, 32768, l2rows}, {1, 2, 3, 1, 16384, l2rows},
    {1, 4, 5, 0, 8192, l2rows}, {1, 1, 5, 1, 32768, l2rows},
    {sms, 4, 3, 0, 8192, l2rows}, {sms, 4, 3, 1, 8192, l2rows}, {sms, 1, 3, 1, 32768, l2rows}, {sms, 2, 3, 1, 16384, l2rows},
    {sms, 4, 5, 0, 8192, l2rows}, {sms, 1, 5, 1, 32768, l2rows},
    {sms, 4, 5, 0, 8192, rows}, {sms, 1, 5, 1, 32768, rows}};
  for (auto c : cs) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 300;
    cudaEventRecord(a);
    k<<<c.ctas, 32, 1024 + c.nbox * c.depth * c.opbytes>>>(map, (const char*)src, c.span_rows, c.nbox, c.depth, iters, 0,
                                                         c.bulk1d, c.opbytes, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2 * 1024]; cudaMemcpy(h, out, 16 * c.ctas, cudaMemcpyDeviceToHost);
    double tot = 0, n = 0; for (int i = 0; i < c.ctas; ++i) { tot += h[2 * i]; n += h[2 * i + 1]; }
    const double chunk = (double)c.nbox * c.opbytes;
    printf("ctas %3d %s %d x %5d B depth %d %s: in flight %4.0f KB, latency %.2f us, %.1f GB/s per SM, %.2f TB/s (%s)\n",
           c.ctas, c.bulk1d ? "bulk1d" : "tma2d ", c.nbox, c.opbytes, c.depth, c.span_rows == rows ? "HBM" : "L2 ",
           chunk * c.depth / 1024, tot / n / 1e3, (double)iters * chunk / (ms * 1e-3) / 1e9,
           (double)c.ctas * iters * chunk / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}
