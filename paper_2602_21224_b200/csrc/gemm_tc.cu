// gemm_tc.cu -- tcgen05 bf16 GEMM for sm_100a: C[M,N] (+)= A[M,K] W[N,K]^T.
//
// Swap-AB: the WEIGHT matrix W[N,K] is the 128-row UMMA "A" operand (M_mma = 128
// output features per tile) and the token rows A[M,K] are the UMMA "B" operand
// (N_mma = token tile, 16..256). Decode/verify GEMMs have few tokens (6..260)
// and are bound by streaming the weights once from HBM, so:
//  - TMA (cp.async.bulk.tensor, 128B swizzle) streams 128x64 weight tiles and
//    Ntok x 64 token tiles into a deep shared-memory ring (mbarrier full/empty);
//  - one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128,
//    N=Ntile, K=16) with the fp32 accumulator in TMEM (two accumulator buffers);
//  - 4 epilogue warps tcgen05.ld the accumulator (lane = output feature,
//    column = token) and reduce into C with coalesced fp32 red.add;
//  - stream-K: the (tile, k-block) units are split evenly over one CTA per SM,
//    so every SM streams the same number of weight bytes whatever the shape.
// Tokens / features / K beyond the tensor bounds are zero-filled by TMA.
#include <cuda.h>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include "gemm_tc.cuh"
#include "tc_ptx.cuh"

namespace {
using namespace tc;
constexpr int BM = 128;          // weight rows per tile (UMMA M)
constexpr int BK = 64;           // K per stage (one 128-byte swizzle atom of bf16)
constexpr int NTHREADS = 192;    // warp0 TMA, warp1 MMA, warps 2..5 epilogue
constexpr int A_BYTES = BM * BK * 2;

struct TcParams {
  int M, N, K, ldc;
  int n_tiles_n, n_tiles_t, n_kb;
  long units;
  int ntile;                      // tokens per tile, multiple of 16, <= 256
  int stages;
  uint32_t idesc;
  uint32_t tmem_cols;
  int vec4;                       // C rows 16-byte aligned (ldc % 4 == 0, C aligned)
  float* C;
};

__global__ void __launch_bounds__(NTHREADS, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned carve-up: [stages x A][stages x B][barriers]
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int b_bytes = P.ntile * BK * 2;
  uint8_t* sA = base;
  uint8_t* sB = base + (size_t)P.stages * A_BYTES;
  uint64_t* bars = (uint64_t*)(sB + (size_t)P.stages * b_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + P.stages;
  uint64_t* tfull = bars + 2 * P.stages;       // [2]
  uint64_t* tempty = bars + 2 * P.stages + 2;  // [2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * P.stages + 4);
  float* epi_smem = (float*)(bars + 2 * P.stages + 6);    // 4 warps x [16 tokens][36]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long u0 = (long)blockIdx.x * P.units / gridDim.x;
  const long u1 = (long)(blockIdx.x + 1) * P.units / gridDim.x;

  if (threadIdx.x == 32) {
    for (int s = 0; s < P.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      // PDL: the weight tiles of the first ring stages do not depend on the
      // previous kernel -- stream them before griddepcontrol.wait, so the ring
      // fills while the predecessor drains; token tiles only after the wait.
      const long npre = (u1 - u0) < P.stages ? (u1 - u0) : P.stages;
      for (long i = 0; i < npre; ++i) {
        const long u = u0 + i;
        const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
        mbar_expect_tx(&full[i], A_BYTES + b_bytes);
        tma_load_2d(&tmW, &full[i], sA + (size_t)i * A_BYTES, kb * BK, (t / P.n_tiles_t) * BM, pw);
      }
      pdl_wait();
      for (long i = 0; i < npre; ++i) {
        const long u = u0 + i;
        const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
        tma_load_2d(&tmX, &full[i], sB + (size_t)i * b_bytes, kb * BK, (t % P.n_tiles_t) * P.ntile, px);
      }
      int stage = (int)(npre % P.stages);
      uint32_t phase = npre == P.stages ? 1u : 0u;
      for (long u = u0 + npre; u < u1; ++u) {
        const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
        const int tn = t / P.n_tiles_t, tt = t % P.n_tiles_t;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], A_BYTES + b_bytes);
        tma_load_2d(&tmW, &full[stage], sA + (size_t)stage * A_BYTES, kb * BK, tn * BM, pw);
        tma_load_2d(&tmX, &full[stage], sB + (size_t)stage * b_bytes, kb * BK, tt * P.ntile, px);
        if (++stage == P.stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    pdl_wait();
    if (lane == 0) {
      int stage = 0, buf = 0;
      uint32_t phase = 0, aphase = 0;
      for (long u = u0; u < u1; ++u) {
        const int kb = (int)(u % P.n_kb);
        const bool first = (u == u0) || kb == 0;
        const bool last = (u == u1 - 1) || kb == P.n_kb - 1;
        if (first) {
          mbar_wait(&tempty[buf], aphase ^ 1);
          fence_after();
        }
        mbar_wait(&full[stage], phase);
        fence_after();
        const uint64_t ad = desc_sw128(sA + (size_t)stage * A_BYTES);
        const uint64_t bd = desc_sw128(sB + (size_t)stage * b_bytes);
        const uint32_t dt = tmem + (uint32_t)(buf * P.ntile);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          mma_bf16(dt, ad + 2 * kk, bd + 2 * kk, P.idesc, (first && kk == 0) ? 0u : 1u);
        mma_commit(&empty[stage]);
        if (last) {
          mma_commit(&tfull[buf]);
          buf ^= 1;
          if (buf == 0) aphase ^= 1;
        }
        if (++stage == P.stages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue: 4 warps = 128 TMEM lanes (lane quarter = warp % 4)
    pdl_wait();
    const int q = warp & 3;
    int buf = 0;
    uint32_t aphase = 0;
    long u = u0;
    while (u < u1) {
      const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
      long seg_end = u + (P.n_kb - kb);
      if (seg_end > u1) seg_end = u1;
      const int tn = t / P.n_tiles_t, tt = t % P.n_tiles_t;
      mbar_wait(&tfull[buf], aphase);
      fence_after();
      // TMEM -> registers (thread = output feature, 16 tokens) -> shared-memory
      // transpose -> each thread adds 4 consecutive features of one token with a
      // single 16-byte red.global.add.v4.f32 (4x fewer L2 atomics than scalar).
      const int row0 = tn * BM + q * 32;
      float* tp = epi_smem + (warp - 2) * (16 * 36);
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * P.ntile);
      for (int c0 = 0; c0 < P.ntile; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + c0, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) tp[j * 36 + lane] = __uint_as_float(r[j]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int f = lane + 32 * i, tk = f >> 3, r4 = (f & 7) * 4;
          const int tok = tt * P.ntile + c0 + tk, row = row0 + r4;
          if (tok < P.M && row < P.N) {
            const float4 v = *(const float4*)(tp + tk * 36 + r4);
            float* dst = &P.C[(size_t)tok * P.ldc + row];
            if (row + 3 < P.N && P.vec4) {
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                           "f"(v.w)
                           : "memory");
            } else {
              atomicAdd(dst, v.x);
              if (row + 1 < P.N) atomicAdd(dst + 1, v.y);
              if (row + 2 < P.N) atomicAdd(dst + 2, v.z);
              if (row + 3 < P.N) atomicAdd(dst + 3, v.w);
            }
          }
        }
        __syncwarp();
      }
      fence_before();
      mbar_arrive(&tempty[buf]);
      buf ^= 1;
      if (buf == 0) aphase ^= 1;
      u = seg_end;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
}

// ------------------------------------------------------------------ host side
}  // namespace

// ---- TMA descriptor helpers shared with attention_tc.cu (declared in tc_ptx.cuh)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

bool tma_available() { return encode_fn() != nullptr; }

bool tma_map_bf16(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_elems,
                  const uint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; }
  for (int i = 0; i + 1 < rank; ++i) s[i] = strides_elems[i] * 2;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), d, s, b, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool make_map(CUtensorMap* m, const void* ptr, int rows, int cols, int ld, int box_rows) {
  uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  uint64_t strides[1] = {(uint64_t)ld};
  uint32_t box[2] = {(uint32_t)BK, (uint32_t)box_rows};
  return tma_map_bf16(m, ptr, 2, dims, strides, box);
}

bool gemm_tc_supported(int M, int N, int K, int lda, int ldw) {
  return M >= 1 && N >= 1 && K >= 16 && K % 8 == 0 && lda % 8 == 0 && ldw % 8 == 0 && encode_fn() != nullptr;
}

int gemm_tc_bf16(const bf16* A, int lda, const bf16* W, int ldw, float* C, int ldc, int M, int N, int K,
                 bool accumulate, cudaStream_t st, bool c_zeroed) {
  int launched = 0;
  if (!accumulate && !c_zeroed) {
    cudaMemset2DAsync(C, (size_t)ldc * 4, 0, (size_t)N * 4, M, st);
  }
  TcParams P;
  P.M = M; P.N = N; P.K = K; P.ldc = ldc; P.C = C;
  // token tile: all tokens in one tile when they fit (weights streamed once)
  int n_tok_tiles = (M + 255) / 256;
  int nt = (M + n_tok_tiles - 1) / n_tok_tiles;
  nt = (nt + 15) / 16 * 16;
  if (nt < 16) nt = 16;
  P.ntile = nt;
  P.n_tiles_t = (M + nt - 1) / nt;
  P.n_tiles_n = (N + BM - 1) / BM;
  P.n_kb = (K + BK - 1) / BK;
  P.units = (long)P.n_tiles_n * P.n_tiles_t * P.n_kb;
  const int b_bytes = nt * BK * 2;
  // ring size: several CTAs per SM (default 2) so one CTA's prologue / epilogue
  // overlaps another's streaming, and PDL-launched successors can become
  // resident while this kernel drains.
  static const int ring_kb = [] { const char* e = getenv("HSD_GEMM_RING_KB"); return e ? atoi(e) : 100; }();
  static const int per_sm = [] { const char* e = getenv("HSD_GEMM_CTAS_PER_SM"); return e ? atoi(e) : 2; }();
  int stages = (ring_kb * 1024) / (A_BYTES + b_bytes);
  if (stages > 16) stages = 16;
  if (stages < 2) stages = 2;
  P.stages = stages;
  P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nt >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * nt)) cols <<= 1;
  P.tmem_cols = cols;
  CUtensorMap mw, mx;
  if (!make_map(&mw, W, N, K, ldw, BM) || !make_map(&mx, A, M, K, lda, nt)) return launched;
  P.vec4 = (ldc % 4 == 0) && (((uintptr_t)C & 15) == 0);
  size_t smem = 1024 + (size_t)stages * (A_BYTES + b_bytes) + (2 * stages + 6) * 8 + 4 * 16 * 36 * 4 + 16;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = true;
  }
  const long max_ctas = (long)num_sms() * per_sm;
  long grid = P.units < max_ctas ? P.units : max_ctas;
  launch_k(gemm_tc_kernel, dim3((unsigned)grid), dim3(NTHREADS), smem, st, mw, mx, P);
  launched += 1;
  return launched;
}
