// common.cuh -- shared device helpers of the sm_100a kernels (product side).
#pragma once

// gate/up weight rows are interleaved in groups of GU_GROUP rows (gate rows of
// features [16g, 16g+16), then their up rows): the layout the fused SwiGLU
// epilogues, swiglu_kernel and interleave_gu_kernel share
constexpr int GU_GROUP = 16;
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <stdint.h>

#define HSD_DEV __device__ __forceinline__

typedef __nv_bfloat16 bf16;

// silu(g) * u with the fast exponential / division (the bf16 SwiGLU epilogues;
// __fdividef(g, inf) = 0 gives silu(-large) = 0)
HSD_DEV float silu_mul_fast(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

enum DType { DT_F32 = 0, DT_BF16 = 1, DT_I32 = 2, DT_U64 = 3 };

// ---------------------------------------------------------------- conversion
HSD_DEV float to_f32(float x) { return x; }
HSD_DEV float to_f32(bf16 x) { return __bfloat162float(x); }
template <typename T> HSD_DEV T from_f32(float x);
template <> HSD_DEV float from_f32<float>(float x) { return x; }
template <> HSD_DEV bf16 from_f32<bf16>(float x) { return __float2bfloat16_rn(x); }

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. (SC'11). Product-side implementation; checked against the
// Random123 known-answer vectors in tests/test_gpu_*.py.
struct u32x4 { uint32_t x, y, z, w; };

HSD_DEV u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    u32x4 n;
    n.x = hi1 ^ c.y ^ k0; n.y = lo1; n.z = hi0 ^ c.w ^ k1; n.w = lo0;
    c = n;
  }
  return c;
}
HSD_DEV uint32_t lane_of(const u32x4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
// sampling uniform in (0,1): ((x>>9)+0.5)*2^-23. k = x>>9 < 2^23, so k + 0.5 has at
// most 24 significant bits and every step is exact in fp32: u in [2^-24, 1 - 2^-24],
// never 0 or 1 (a 24-bit k + 0.5 would round to 2^24 at k = 2^24-1, i.e. u = 1 and
// an infinite Gumbel score)
HSD_DEV float unit_open(uint32_t x) { return ((float)(x >> 9) + 0.5f) * 1.1920928955078125e-07f; }

#define TAG_ACCEPT 0x5EED0001u
#define TAG_GUMBEL 0x5EED0002u
#define TAG_PLANT 0x5EED0003u

// ---------------------------------------------------------------- reductions
HSD_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
HSD_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// block-wide sum with a fixed (deterministic) reduction tree; `red` >= 32 floats
HSD_DEV float block_sum(float v, float* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = (threadIdx.x < (unsigned)nw) ? red[threadIdx.x] : 0.f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  float r = red[0];
  __syncthreads();
  return r;
}
HSD_DEV float block_max(float v, float* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = (threadIdx.x < (unsigned)nw) ? red[threadIdx.x] : -INFINITY;
  if (w == 0) t = warp_max(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  float r = red[0];
  __syncthreads();
  return r;
}

// (value desc, index asc) "better" comparison used by argmax / top-k (R8)
HSD_DEV bool better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}
// warp argmax over (value, index) pairs with the tie rule above
HSD_DEV void warp_argmax(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(ov, oi, v, i)) { v = ov; i = oi; }
  }
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel may start
// while its predecessor is still running. Every kernel therefore executes
// pdl_wait() (griddepcontrol.wait: all prerequisite grids complete, memory
// visible) before touching data produced upstream, and pdl_trigger() to let
// its own dependents start their prologue early.
HSD_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
HSD_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- L2 weight prefetch
// Kernels that leave HBM idle (row kernels, attention, K-TREE) carry the byte range
// of weights a LATER GEMM will stream; thread 0 of every CTA issues its share as
// cp.async.bulk.prefetch.L2 (fire and forget, no completion tracking) before the
// PDL wait -- weights are never written after init. The engine sets g_l2pf right
// before a launch; the launcher consumes it (take_l2pf) into the kernel argument.
struct L2Pf {
  const char* p;
  unsigned long long bytes;
  int late;   // 1: issue after the PDL wait (only inside the idle window), 0: before it
};
extern L2Pf g_l2pf;
inline L2Pf take_l2pf() {
  L2Pf r = g_l2pf;
  g_l2pf = L2Pf{nullptr, 0ull, 0};
  return r;
}
HSD_DEV void l2pf_issue(const L2Pf& pf, int late = 0) {
  if (pf.bytes == 0 || pf.late != late || threadIdx.x != 0 || threadIdx.y != 0) return;
  const unsigned long long nb = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
  const unsigned long long b = blockIdx.x + (unsigned long long)gridDim.x * (blockIdx.y + (unsigned long long)gridDim.y * blockIdx.z);
  const unsigned long long per = (((pf.bytes + nb - 1) / nb) + 4095ull) & ~4095ull;
  const unsigned long long lo = b * per, hi = lo + per < pf.bytes ? lo + per : pf.bytes;
  for (unsigned long long o = lo; o < hi; o += 65536ull) {
    const unsigned sz = (unsigned)((hi - o) < 65536ull ? (hi - o) : 65536ull) & ~15u;
    if (sz) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf.p + o), "r"(sz) : "memory");
  }
}

// ---------------------------------------------------------------- kernel stamps
// hsd_kstamp: the engine hands the NEXT GEMM launch a stamp slot (like L2Pf);
// kernels fold per-CTA %globaltimer entry / exit times into [slot][id] arrays.
constexpr int KST_SLOTS = 64;     // replays kept (step counter mod 64)
constexpr int KST_MAXID = 512;    // stamped launches per step
struct KStamp {
  unsigned long long* buf;        // [2][KST_SLOTS][KST_MAXID]: entry minima, then exit maxima
  int id;
  const int* step;                // device step counter (slot = step mod KST_SLOTS)
};
extern KStamp g_kstamp;
inline KStamp take_kstamp() {
  KStamp r = g_kstamp;
  g_kstamp = KStamp{nullptr, 0, nullptr};
  return r;
}
// entry = the first return from griddepcontrol.wait (call from thread 0 only, right
// after its pdl_wait); exit = the last CTA's exit (thread 0 at the very end)
HSD_DEV void kst_enter(const KStamp& k) {
  if (k.buf == nullptr || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMin(k.buf + (size_t)((*k.step) & (KST_SLOTS - 1)) * KST_MAXID + k.id, t);
}
HSD_DEV void kst_exit(const KStamp& k) {
  if (k.buf == nullptr || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMax(k.buf + (size_t)KST_SLOTS * KST_MAXID + (size_t)((*k.step) & (KST_SLOTS - 1)) * KST_MAXID + k.id, t);
}

extern bool g_hsd_pdl;   // engine.cu; HSD_PDL=0 disables (A/B testing)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_hsd_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// launch_k with a runtime thread-block cluster size along x (grid.x % cluster_x == 0)
template <typename... KArgs, typename... Args>
inline void launch_k_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_hsd_pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- error word
#define DEV_ERR_BAD_TREE 1
#define DEV_ERR_BAD_TOKEN 2
#define DEV_ERR_OVERFLOW 4
