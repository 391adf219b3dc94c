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
#include <cstring>
#include <mutex>
#include <unordered_map>
#include "gemm_tc.cuh"
#include "tc_ptx.cuh"

unsigned long long* g_gemm_trace = nullptr;   // HSD_GEMM_TRACE: last launch's phase stamps

namespace {
using namespace tc;
constexpr int BM = 128;          // weight rows per tile (UMMA M)
constexpr int BK = 64;           // K per stage (one 128-byte swizzle atom of bf16)
constexpr int NTHREADS = 192;    // warp0 TMA, warp1 MMA, warps 2..5 epilogue
constexpr int NTHREADS2 = 320;   // pair kernel: warps 2..5 and 6..9 = two epilogue groups
constexpr int A_BYTES = BM * BK * 2;
constexpr int EPI_LD = BM + 4;   // epilogue stage row stride (floats)
enum { EPI_ATOMIC = 0, EPI_STORE = 1, EPI_ADD = 2, EPI_SWIGLU = 3, EPI_QKV = 4 };

struct TcParams {
  int M, N, K, ldc;
  int n_tiles_n, n_tiles_t, n_kb;
  long units;
  int ntile;                      // tokens per tile, multiple of 16, <= 256
  int stages;
  uint32_t idesc;
  uint32_t tmem_cols;
  int vec4;                       // C rows 16-byte aligned (ldc % 4 == 0, C aligned)
  int dp;                         // 1: data-parallel (a CTA owns whole tiles), 0: stream-K
  int wt;                         // pair kernel: 256-row weight tiles per super tile (1 or 2)
  int nbuf;                       // pair kernel: accumulator buffers in TMEM (1 or 2)
  int exp;                        // HSD_GEMM_EXP experiment bits (pair kernel): 1 skip stores, 2 red.add residual
  int epi;                        // GemmEpi
  float* C;
  bf16* H;                        // EPI_SWIGLU output [M, N/2] bf16
  int ldh;
  unsigned long long* trace;      // debug phase trace (HSD_GEMM_TRACE) or null
  QkvEpi qe;                      // EPI_QKV (pair kernel)
  int tma_out;                    // pair kernel: STORE / ADD / SWIGLU outputs leave by TMA store / reduce-add
  int pre;                        // pair kernel: weight halves of the first stages before griddepcontrol.wait
  int pf_ahead;                   // pair kernel: L2 prefetch distance (units) of the weight stream, 0 = off
  KStamp kst;                     // per-launch %globaltimer stamps (hsd_kstamp) or kst.buf == null
};
HSD_DEV uint64_t gtime_g() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// launch duration inside graph replays: every CTA's thread 0 folds its entry time
// (atomicMin) and exit time (atomicMax) into the slot (step mod KST_SLOTS, launch id)
// entry = the first return from griddepcontrol.wait in the CTA (inputs ready); the
// pre-wait weight prefetch overlaps the predecessor and is not counted
HSD_DEV void kstamp_wait(const KStamp& k) {
  // one thread per CTA (thread 0 = the TMA producer's lane): every waiting thread
  // hitting one address serialised ~50k atomics per launch in L2
  if (k.buf == nullptr || threadIdx.x != 0) return;
  const size_t e = (size_t)((*k.step) & (KST_SLOTS - 1)) * KST_MAXID + k.id;
  atomicMin(k.buf + e, (unsigned long long)gtime_g());
}
HSD_DEV void kstamp(const KStamp& k, bool end) {
  if (k.buf == nullptr || threadIdx.x != 0) return;
  const size_t e = (size_t)((*k.step) & (KST_SLOTS - 1)) * KST_MAXID + k.id;
  const unsigned long long t = gtime_g();
  if (end) atomicMax(k.buf + (size_t)KST_SLOTS * KST_MAXID + e, t);
  else atomicMin(k.buf + e, t);
}
// CTA 0 records slots 0..15, the last CTA slots 16..31: start, pre-PDL weight
// loads issued, PDL released, first / last stage landed (MMA), epilogue start /
// end, CTA end
#define GTRACE(i) do { if (P.trace && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) \
    P.trace[(blockIdx.x == 0 ? 0 : 16) + (i)] = gtime_g(); } while (0)

// The idx-th (tile, k-block) unit of this CTA. Stream-K: a contiguous range of
// units; data-parallel: whole tiles blockIdx.x, blockIdx.x + grid, ...
struct Sched {
  long u0, count;
  int dp, n_kb;
  HSD_DEV long unit(long i) const {
    if (!dp) return u0 + i;
    return ((long)blockIdx.x + (i / n_kb) * (long)gridDim.x) * n_kb + i % n_kb;
  }
};

HSD_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
HSD_DEV void epi_bar_g(int g) { asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory"); }

__global__ void __launch_bounds__(NTHREADS, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ CUtensorMap tmO, TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned carve-up: [stages x A][stages x B][barriers][epilogue stage]
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
  float* stage_buf = (float*)(bars + 2 * P.stages + 6);   // [16 tokens][EPI_LD] fp32
  // P.tma_out (stream-K partials): dense [2 buffers][16 tokens][128] fp32 stages, 1024-aligned,
  // each chunk leaves by one TMA bulk reduce-add
  float* const dstage = (float*)(((uintptr_t)(bars + 2 * P.stages + 6) + 1023) & ~(uintptr_t)1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GTRACE(0);
  Sched sc;
  sc.dp = P.dp;
  sc.n_kb = P.n_kb;
  if (P.dp) {
    const long n_tiles = (long)P.n_tiles_n * P.n_tiles_t;
    const long mine = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    sc.u0 = 0;
    sc.count = mine * P.n_kb;
  } else {
    sc.u0 = (long)blockIdx.x * P.units / gridDim.x;
    sc.count = (long)(blockIdx.x + 1) * P.units / gridDim.x - sc.u0;
  }

  // Thread 0 initialises the barriers and, before the CTA-wide barrier, issues
  // the first ring stages' WEIGHT loads (no kernel writes the weights, so they
  // may precede griddepcontrol.wait): the TMA latency overlaps warp 2's TMEM
  // allocation and the predecessor's drain. Token tiles only after the wait.
  const long npre = sc.count < P.stages ? sc.count : P.stages;
  uint64_t pw = 0, px = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    pw = policy_evict_first();
    px = policy_evict_last();
    GTRACE(9);
    for (long i = 0; i < npre; ++i) {
      const long u = sc.unit(i);
      const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
      mbar_expect_tx(&full[i], A_BYTES + b_bytes);
      tma_load_2d(&tmW, &full[i], sA + (size_t)i * A_BYTES, kb * BK, (t / P.n_tiles_t) * BM, pw);
      if (i == 0) GTRACE(11);
    }
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
  if (threadIdx.x == 0) GTRACE(8);
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      GTRACE(1);
      pdl_wait();
    kstamp_wait(P.kst);
      GTRACE(2);
      for (long i = 0; i < npre; ++i) {
        const long u = sc.unit(i);
        const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
        tma_load_2d(&tmX, &full[i], sB + (size_t)i * b_bytes, kb * BK, (t % P.n_tiles_t) * P.ntile, px);
      }
      int stage = (int)(npre % P.stages);
      uint32_t phase = npre == P.stages ? 1u : 0u;
      for (long i = npre; i < sc.count; ++i) {
        const long u = sc.unit(i);
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
    kstamp_wait(P.kst);
    if (lane == 0) {
      int stage = 0, buf = 0;
      uint32_t phase = 0, aphase = 0;
      for (long i = 0; i < sc.count; ++i) {
        const int kb = (int)(sc.unit(i) % P.n_kb);
        const bool first = (i == 0) || kb == 0;
        const bool last = (i == sc.count - 1) || kb == P.n_kb - 1;
        if (first) {
          mbar_wait(&tempty[buf], aphase ^ 1);
          fence_after();
        }
        mbar_wait(&full[stage], phase);
        fence_after();
        if (i == 0) GTRACE(3);
        if (i == sc.count - 1) GTRACE(4);
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
    // Per 16-token chunk: TMEM -> registers (thread = output feature) -> a
    // [16 tokens][128 features] fp32 stage in shared memory -> the 128 threads
    // emit token-major 16-byte vectors: red.add.v4 (stream-K partial sums),
    // st.v4 (data-parallel), ld+add+st (data-parallel residual), or SwiGLU of
    // the interleaved gate/up rows into bf16 (data-parallel).
    pdl_wait();
    kstamp_wait(P.kst);
    const int q = warp & 3, et = threadIdx.x - 64;      // 0..127
    int buf = 0, ck = 0;
    uint32_t aphase = 0;
    long i = 0;
    while (i < sc.count) {
      const long u = sc.unit(i);
      const int t = (int)(u / P.n_kb), kb = (int)(u % P.n_kb);
      long seg = P.n_kb - kb;
      if (i + seg > sc.count) seg = sc.count - i;
      const int tn = t / P.n_tiles_t, tt = t % P.n_tiles_t;
      mbar_wait(&tfull[buf], aphase);
      fence_after();
      if (threadIdx.x == 64) GTRACE(5);
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * P.ntile);
      for (int c0 = 0; c0 < P.ntile; c0 += 16, ++ck) {
        uint32_t r[16];
        tmem_ld16(taddr + c0, r);
        if (P.tma_out) {
          // stream-K partial: [16 tokens][128 features] dense stage -> one TMA reduce-add
          // into the zero-kept fp32 scratch (the issuing thread waits until the previous
          // chunk's bulk op has read its buffer, before the second barrier)
          float* sb = dstage + (size_t)(ck & 1) * 16 * BM;
#pragma unroll
          for (int j = 0; j < 16; ++j) sb[j * BM + q * 32 + lane] = __uint_as_float(r[j]);
          fence_proxy_async();
          epi_bar();
          if (et == 0) {
            tma_reduce_add_2d(&tmO, sb, tn * BM, tt * P.ntile + c0);
            bulk_commit();
            bulk_wait_read<1>();
          }
          epi_bar();
          continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) stage_buf[j * EPI_LD + q * 32 + lane] = __uint_as_float(r[j]);
        epi_bar();
        if (P.epi == EPI_SWIGLU) {
          // rows [32g, 32g+16) of the tile are the gate rows of features 16g.., the
          // next 16 rows their up rows (GU_GROUP interleave)
          const int tk = et >> 3, f8 = (et & 7) * 8;
          const int tok = tt * P.ntile + c0 + tk, f0 = tn * (BM / 2) + f8;
          if (tok < P.M && f0 < P.N / 2) {
            const float* g = stage_buf + tk * EPI_LD + 2 * GU_GROUP * (f8 / GU_GROUP) + f8 % GU_GROUP;
            const float* uu = g + GU_GROUP;
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a0 = g[2 * e], a1 = g[2 * e + 1];
              const __nv_bfloat162 hv = __floats2bfloat162_rn(a0 / (1.0f + expf(-a0)) * uu[2 * e],
                                                              a1 / (1.0f + expf(-a1)) * uu[2 * e + 1]);
              w[e] = *(const uint32_t*)&hv;
            }
            *(uint4*)(P.H + (size_t)tok * P.ldh + f0) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        } else {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int slot = et + 128 * v, tk = slot >> 5, r4 = (slot & 31) * 4;
            const int tok = tt * P.ntile + c0 + tk, row = tn * BM + r4;
            if (tok >= P.M || row >= P.N) continue;
            const float4 val = *(const float4*)(stage_buf + tk * EPI_LD + r4);
            float* dst = &P.C[(size_t)tok * P.ldc + row];
            if (row + 3 < P.N && P.vec4) {
              if (P.epi == EPI_ATOMIC) {
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(val.x), "f"(val.y),
                             "f"(val.z), "f"(val.w)
                             : "memory");
              } else if (P.epi == EPI_ADD) {
                float4 o = *(const float4*)dst;
                o.x += val.x; o.y += val.y; o.z += val.z; o.w += val.w;
                *(float4*)dst = o;
              } else {
                *(float4*)dst = val;
              }
            } else {
              const float vv[4] = {val.x, val.y, val.z, val.w};
              for (int e = 0; e < 4 && row + e < P.N; ++e) {
                if (P.epi == EPI_ATOMIC) atomicAdd(dst + e, vv[e]);
                else if (P.epi == EPI_ADD) dst[e] += vv[e];
                else dst[e] = vv[e];
              }
            }
          }
        }
        epi_bar();
      }
      if (threadIdx.x == 64) GTRACE(6);
      fence_before();
      mbar_arrive(&tempty[buf]);
      buf ^= 1;
      if (buf == 0) aphase ^= 1;
      i += seg;
    }
    if (P.tma_out && et == 0) bulk_wait<0>();   // every bulk reduce of this CTA complete
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) GTRACE(7);
  kstamp(P.kst, true);
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
}

// ------------------------------------------------------------------ CTA-pair kernel
// Data-parallel GEMM on a CTA pair (cluster of 2 on one TPC): one tile = 256
// weight rows x ntile tokens, computed by tcgen05.mma.cta_group::2 (M = 256)
// issued by the leader (rank 0). CTA r stages weight rows [r*128, +128) and
// tokens [r*ntile/2, +ntile/2) of every k-block (the UMMA 2x1SM operand split),
// so each SM ingests (128 + ntile/2) x 64 x 2 bytes per k-block instead of
// (128 + ntile) x 64 x 2 -- the single-CTA kernel's limit at large M. Each CTA's
// TMEM holds its 128 rows of the accumulator; the epilogue is the data-parallel
// one of gemm_tc_kernel on that 128-row half.
// Super tiles (P.wt = 2): 512 weight rows x ntile tokens -- the token stage is
// staged once and feeds two M = 256 MMAs (accumulators side by side in TMEM, one
// buffer when 2 x 2 x ntile > 512 columns). At c3 the kernel is bound by L2 -> SM
// operand traffic (~9.8 TB/s chip-wide, ncu l1tex__m_xbar2l1tex_read_bytes), and a
// 512 x 240 tile moves (512 + 240) / (2 (256 + 240)) = 0.76 of the bytes per flop.
// WT is a template parameter: a runtime super-tile loop in the MMA issuer / TMA
// producer cost ~20 % on every c3 shape (QKV 93 -> 112 us).
template <int WT>
__global__ void __launch_bounds__(NTHREADS2, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    const __grid_constant__ CUtensorMap tmO, TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int half_nt = P.ntile / 2;
  const int bh = half_nt * BK * 2;                     // this CTA's token half per stage
  constexpr int wt = WT;
  const int nbuf = P.nbuf;
  const int a_bytes = wt * A_BYTES;                    // this CTA's weight rows per stage
  uint8_t* sA = base;
  uint8_t* sB = base + (size_t)P.stages * a_bytes;
  uint64_t* bars = (uint64_t*)(sB + (size_t)P.stages * bh);
  uint64_t* full = bars;                       // [stages] (the leader's count both CTAs' bytes)
  uint64_t* empty = bars + P.stages;           // [stages]
  uint64_t* tfull = bars + 2 * P.stages;       // [2]
  uint64_t* tempty = bars + 2 * P.stages + 2;  // [2] (leader: one arrival per CTA)
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * P.stages + 4);
  // epilogue region (1024-aligned): 2 groups x [16 tokens][EPI_LD] fp32 padded stages
  // (SwiGLU / QKV / thread-store paths); with P.tma_out the same bytes hold dense
  // stages [2 groups][2 buffers][16][128] fp32 for TMA stores (STORE / ADD), and
  // SwiGLU's bf16 outputs [2 groups][2 buffers][16][64] (128-byte swizzle) sit at +24 KB
  uint8_t* const epi_mem = (uint8_t*)(((uintptr_t)(bars + 2 * P.stages + 6) + 1023) & ~(uintptr_t)1023);
  float* stage_buf = (float*)epi_mem;
  __shared__ int tmeta[2][16][3];   // EPI_QKV: per group, the chunk's tokens' (pos, K offset, V offset)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)(blockIdx.x & 1);
  const bool leader = rank == 0;
  const long pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int n_tm = (P.N + 2 * BM * wt - 1) / (2 * BM * wt);
  const long n_tiles = (long)n_tm * P.n_tiles_t;
  const long my_tiles = pair < n_tiles ? (n_tiles - 1 - pair) / n_pairs + 1 : 0;
  const long count = my_tiles * P.n_kb;
  auto tile_of = [&](long i) { return pair + (i / P.n_kb) * n_pairs; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }   // 2 CTAs x 2 groups
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  const uint32_t full0 = mapa_u32(&full[0], 0);        // the leader's full barriers
  const uint32_t tempty0 = mapa_u32(&tempty[0], 0);    // the leader's accumulator-empty barriers

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: each stages its operand halves)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      // Weights are never written by a kernel, so the weight halves of the first ring
      // stages are issued BEFORE griddepcontrol.wait (they overlap the predecessor's
      // tail); their token halves follow the wait. P.pre = 0 disables it.
      const long npre = P.pre ? (count < P.stages ? count : P.stages) : 0;
      auto load_w = [&](long i, int stg) {
        const long t = tile_of(i);
        const int kb = (int)(i % P.n_kb), tm = (int)(t / P.n_tiles_t);
        for (int w = 0; w < wt; ++w)
          tma_load_2d_2sm(&tmW, full0 + 8u * stg, sA + (size_t)stg * a_bytes + w * A_BYTES, kb * BK,
                          (2 * (tm * wt + w) + rank) * BM, pw);
      };
      auto load_x = [&](long i, int stg) {
        const long t = tile_of(i);
        const int kb = (int)(i % P.n_kb), tt = (int)(t % P.n_tiles_t);
        tma_load_2d_2sm(&tmX, full0 + 8u * stg, sB + (size_t)stg * bh, kb * BK, tt * P.ntile + rank * half_nt, px);
      };
      // (experiment HSD_GEMM_PF_AHEAD = d: an L2 prefetch of unit i + d's weight boxes
      // is issued with unit i's loads -- the weight stream's DRAM latency off the ring)
      auto prefetch_w = [&](long i) {
        if (P.pf_ahead <= 0 || i >= count) return;
        const long t = tile_of(i);
        const int kb = (int)(i % P.n_kb), tm = (int)(t / P.n_tiles_t);
        for (int w = 0; w < wt; ++w)
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&tmW), "r"(kb * BK),
                       "r"((2 * (tm * wt + w) + rank) * BM)
                       : "memory");
      };
      for (long i = 0; i < npre; ++i) {   // ring stages are free at start
        if (leader) mbar_expect_tx(&full[i], 2u * (a_bytes + bh));
        load_w(i, (int)i);
      }
      for (long i = 0; i < (P.pf_ahead > 0 ? P.pf_ahead : 0); ++i) prefetch_w(npre + i);
      pdl_wait();
    kstamp_wait(P.kst);
      for (long i = 0; i < npre; ++i) load_x(i, (int)i);
      int stage = (int)(npre % P.stages);
      uint32_t phase = npre == P.stages ? 1u : 0u;
      for (long i = npre; i < count; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (leader) mbar_expect_tx(&full[stage], 2u * (a_bytes + bh));
        load_w(i, stage);
        load_x(i, stage);
        prefetch_w(i + P.pf_ahead);
        if (++stage == P.stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the leader's lane 0 issues for the pair
    pdl_wait();
    kstamp_wait(P.kst);
    if (leader && lane == 0) {
      int stage = 0, buf = 0;
      uint32_t phase = 0, aphase = 0;
      for (long i = 0; i < count; ++i) {
        const int kb = (int)(i % P.n_kb);
        const bool first = kb == 0, last = kb == P.n_kb - 1;
        if (first) {
          mbar_wait(&tempty[buf], aphase ^ 1);
          fence_after();
        }
        mbar_wait(&full[stage], phase);
        fence_after();
        const uint64_t bd = desc_sw128(sB + (size_t)stage * bh);
        for (int w = 0; w < wt; ++w) {
          const uint64_t ad = desc_sw128(sA + (size_t)stage * a_bytes + w * A_BYTES);
          const uint32_t dt = tmem + (uint32_t)((buf * wt + w) * P.ntile);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_bf16_2sm(dt, ad + 2 * kk, bd + 2 * kk, P.idesc, (first && kk == 0) ? 0u : 1u);
        }
        mma_commit_2sm(&empty[stage], 3);
        if (last) {
          mma_commit_2sm(&tfull[buf], 3);
          if (++buf == nbuf) { buf = 0; aphase ^= 1; }
        }
        if (++stage == P.stages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue: this CTA's 128 accumulator rows (output features).
    // Two groups of 4 warps take alternate 16-token chunks (each group's warps
    // cover the 4 TMEM lane quarters), each with its own staging buffer and named
    // barrier, so one group's TMEM loads / barriers overlap the other's stores:
    // with one accumulator buffer (super tiles) the epilogue is not hidden behind
    // the next tile's MMAs, and a single group ran at ~12 GB/s per SM.
    pdl_wait();
    kstamp_wait(P.kst);
    const int q = warp & 3, grp = (warp - 2) >> 2, et = threadIdx.x - 64 - 128 * grp;
    float* const stage_g = stage_buf + grp * 16 * EPI_LD;
    int ck = 0;                                   // this group's chunk counter (TMA-store buffer parity)
    int buf = 0;
    uint32_t aphase = 0;
    for (long ti = 0; ti < my_tiles; ++ti) {
      const long t = pair + ti * n_pairs;
      const int tm = (int)(t / P.n_tiles_t), tt = (int)(t % P.n_tiles_t);
      mbar_wait(&tfull[buf], aphase);
      fence_after();
      // (timing experiment HSD_GEMM_EXP bit 4: no epilogue at all -- MMA / operand time only)
      for (int w = 0; w < ((P.exp & 4) ? 0 : wt); ++w) {
      const int tn = 2 * (tm * wt + w) + rank;        // this CTA's 128-row weight tile
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((buf * wt + w) * P.ntile);
      for (int c0 = 16 * grp; c0 < P.ntile; c0 += 32, ++ck) {
        uint32_t r[16];
        tmem_ld16(taddr + c0, r);
        if (P.tma_out && (P.epi == EPI_STORE || P.epi == EPI_ADD)) {
          // [16 tokens][128 features] dense fp32 stage -> one TMA store (or reduce-add
          // into the residual stream) of the box at (feature tn*128, token row);
          // rows past M are clipped by the TMA unit. The issuing thread waits until
          // the store of the chunk before has read its buffer, before barrier B
          float* sb = (float*)epi_mem + (size_t)(grp * 2 + (ck & 1)) * 16 * BM;
#pragma unroll
          for (int j = 0; j < 16; ++j) sb[j * BM + q * 32 + lane] = __uint_as_float(r[j]);
          fence_proxy_async();
          epi_bar_g(grp);
          if (et == 0) {
            if (!(P.exp & 1)) {
              if (P.epi == EPI_ADD) tma_reduce_add_2d(&tmO, sb, tn * BM, tt * P.ntile + c0);
              else tma_store_2d(&tmO, sb, tn * BM, tt * P.ntile + c0);
              bulk_commit();
            }
            bulk_wait_read<1>();
          }
          epi_bar_g(grp);
          continue;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) stage_g[j * EPI_LD + q * 32 + lane] = __uint_as_float(r[j]);
        if (P.epi == EPI_QKV && et < 16) {
          // the chunk's per-token cache offsets (elements, kv head 0, dim 0): pos, K row, V slot
          const QkvEpi& e = P.qe;
          const int tok = tt * P.ntile + c0 + et;
          int pos = -1, ko = 0, vo = -1;
          if (tok < P.M && (pos = e.pos[tok]) >= 0) {
            const int kp = e.kvpos[tok];
            const int page = e.block_table[(size_t)e.req[tok] * e.pages_per_req + kp / e.page_size];
            const int slot = kp % e.page_size, blk = e.page_size * e.hd;
            ko = ((page * 2) * e.Hkv) * blk + slot * e.hd;
            vo = ((page * 2 + 1) * e.Hkv) * blk + slot;
          }
          tmeta[grp][et][0] = pos; tmeta[grp][et][1] = ko; tmeta[grp][et][2] = vo;
        }
        epi_bar_g(grp);
        if (P.epi == EPI_QKV) {
          // fused RoPE / q / KV writes (qkv_rope_kv's work): the staged chunk holds all
          // 128 features (whole heads) of 16 tokens, so a dimension's rotation partner
          // d +- hd/2 is in the same stage row. q / K: a thread takes 16 consecutive
          // dims of one token (thread -> (token et % 16, dims): conflict-free stage
          // reads; two 16-byte stores). V (transposed cache, [d][slot]): a thread takes
          // one dim of the 16 tokens, writing runs of consecutive slots as 8 / 4 / 2
          // byte vectors; the chunk's per-token cache offsets were computed once
          // (tmeta) before the stage barrier.
          const QkvEpi& e = P.qe;
          const int hd = e.hd, half = hd >> 1;
          const int h0 = tn * BM / hd;                  // first head of the tile
          if (!(P.exp & 1) && h0 < e.Hq + e.Hkv) {
            const int tk = et & 15, f16 = (et >> 4) * 16;
            const int tok = tt * P.ntile + c0 + tk;
            const int h = h0 + f16 / hd, d0 = f16 % hd;
            if (tok < P.M) {
              const int pos = tmeta[grp][tk][0];
              const float* src = stage_g + tk * EPI_LD + f16;
              const float* prt = src + (d0 < half ? half : -half);
              uint32_t o[8];
              if (pos >= 0) {
                const int j0 = d0 & (half - 1);
                const float4* co = (const float4*)(e.rc + (size_t)pos * half + j0);
                const float4* si = (const float4*)(e.rs + (size_t)pos * half + j0);
                const float sg = d0 < half ? -1.f : 1.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float4 x = ((const float4*)src)[i], y = ((const float4*)prt)[i], c4 = co[i], s4 = si[i];
                  const __nv_bfloat162 a0 = __floats2bfloat162_rn(x.x * c4.x + sg * y.x * s4.x, x.y * c4.y + sg * y.y * s4.y);
                  const __nv_bfloat162 a1 = __floats2bfloat162_rn(x.z * c4.z + sg * y.z * s4.z, x.w * c4.w + sg * y.w * s4.w);
                  o[2 * i] = *(const uint32_t*)&a0;
                  o[2 * i + 1] = *(const uint32_t*)&a1;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = 0u;
              }
              bf16* dst = nullptr;
              if (h < e.Hq) dst = e.q_out + ((size_t)tok * e.Hq + h) * hd + d0;
              else if (pos >= 0)
                dst = (bf16*)e.kv_base + (size_t)tmeta[grp][tk][1] + (size_t)(h - e.Hq) * e.page_size * hd + d0;
              if (dst) {
                ((uint4*)dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
                ((uint4*)dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
              }
            }
          } else if (!(P.exp & 1) && h0 < e.Hq + 2 * e.Hkv) {
            // V heads: thread = one feature (head, dim) of the tile, 16 tokens
            const int h = h0 + et / hd, d = et % hd;
            bf16* vb = (bf16*)e.kv_base + (size_t)(h - e.Hq - e.Hkv) * e.page_size * hd + (size_t)d * e.page_size;
            const int nj = min(16, P.M - (tt * P.ntile + c0));
            int j = 0;
            while (j < nj) {
              const int vo = tmeta[grp][j][2];
              if (vo < 0) { ++j; continue; }
              const float x0 = stage_g[j * EPI_LD + et];
              // run of consecutive cache slots starting at j (same page), up to 4
              int run = 1;
              while (run < 4 && j + run < nj && tmeta[grp][j + run][2] == vo + run) ++run;
              if (run == 4 && (vo & 3) == 0) {
                const __nv_bfloat162 a0 = __floats2bfloat162_rn(x0, stage_g[(j + 1) * EPI_LD + et]);
                const __nv_bfloat162 a1 = __floats2bfloat162_rn(stage_g[(j + 2) * EPI_LD + et], stage_g[(j + 3) * EPI_LD + et]);
                *(uint2*)(vb + vo) = make_uint2(*(const uint32_t*)&a0, *(const uint32_t*)&a1);
                j += 4;
              } else if (run >= 2 && (vo & 1) == 0) {
                *(__nv_bfloat162*)(vb + vo) = __floats2bfloat162_rn(x0, stage_g[(j + 1) * EPI_LD + et]);
                j += 2;
              } else {
                vb[vo] = __float2bfloat16_rn(x0);
                ++j;
              }
            }
          }
        } else if (P.epi == EPI_SWIGLU) {
          // rows [32g, 32g+16) of the tile: gate rows of features 16g.., then their up rows.
          // Thread -> (token et % 16, 8 features): the 8 threads of a 16-byte load phase
          // read 8 different token rows (EPI_LD = 132: 4 banks apart), conflict-free
          // (HSD_GEMM_EXP bit 8, experiment: thread -> (token et / 8, 8 features), each warp
          // store 4 whole 128-byte lines, 4-way bank conflicts on the stage reads)
          const int tk = (P.exp & 8) ? et >> 3 : et & 15, f8 = (P.exp & 8) ? (et & 7) * 8 : (et >> 4) * 8;
          const int tok = tt * P.ntile + c0 + tk, f0 = tn * (BM / 2) + f8;
          if (tok < P.M && f0 < P.N / 2 && !(P.exp & 1)) {
            const float* g = stage_g + tk * EPI_LD + 2 * GU_GROUP * (f8 / GU_GROUP) + f8 % GU_GROUP;
            const float4 g0 = *(const float4*)g, g1 = *(const float4*)(g + 4);
            const float4 u0 = *(const float4*)(g + GU_GROUP), u1 = *(const float4*)(g + GU_GROUP + 4);
            const __nv_bfloat162 h0 = __floats2bfloat162_rn(silu_mul_fast(g0.x, u0.x), silu_mul_fast(g0.y, u0.y));
            const __nv_bfloat162 h1 = __floats2bfloat162_rn(silu_mul_fast(g0.z, u0.z), silu_mul_fast(g0.w, u0.w));
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(silu_mul_fast(g1.x, u1.x), silu_mul_fast(g1.y, u1.y));
            const __nv_bfloat162 h3 = __floats2bfloat162_rn(silu_mul_fast(g1.z, u1.z), silu_mul_fast(g1.w, u1.w));
            const uint4 hv = make_uint4(*(const uint32_t*)&h0, *(const uint32_t*)&h1, *(const uint32_t*)&h2,
                                        *(const uint32_t*)&h3);
            if (P.tma_out)   // [16][64] bf16 box, 128-byte swizzle: 16-byte unit f8/8 of row tk at unit ^ (tk & 7)
              *(uint4*)(epi_mem + 24576 + (grp * 2 + (ck & 1)) * 2048 + tk * 128 + (((f8 >> 3) ^ (tk & 7)) << 4)) = hv;
            else
              *(uint4*)(P.H + (size_t)tok * P.ldh + f0) = hv;
          }
          if (P.tma_out) {
            fence_proxy_async();
            epi_bar_g(grp);
            if (et == 0) {
              if (!(P.exp & 1)) {
                tma_store_2d(&tmO, epi_mem + 24576 + (grp * 2 + (ck & 1)) * 2048, tn * (BM / 2), tt * P.ntile + c0);
                bulk_commit();
              }
              bulk_wait_read<1>();
            }
          }
        } else {
          // residual add: all 4 residual vectors of this thread are loaded before the
          // first store (the stores may alias them for the compiler, which otherwise
          // serialised one global round trip per vector: c3 O projection 102 us)
          float4 res[4];
          // residual add as one fp32 red.add per element (the tile is this CTA's
          // alone, so C + v is rounded exactly once, as a load / add / store would)
          const bool red = !(P.exp & 2);
          if (P.exp & 1) { epi_bar_g(grp); continue; }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int slot = et + 128 * v, tk = slot >> 5, r4 = (slot & 31) * 4;
            const int tok = tt * P.ntile + c0 + tk, row = tn * BM + r4;
            res[v] = (P.epi == EPI_ADD && !red && P.vec4 && tok < P.M && row + 3 < P.N)
                         ? *(const float4*)&P.C[(size_t)tok * P.ldc + row]
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int slot = et + 128 * v, tk = slot >> 5, r4 = (slot & 31) * 4;
            const int tok = tt * P.ntile + c0 + tk, row = tn * BM + r4;
            if (tok >= P.M || row >= P.N) continue;
            const float4 val = *(const float4*)(stage_g + tk * EPI_LD + r4);
            float* dst = &P.C[(size_t)tok * P.ldc + row];
            if (row + 3 < P.N && P.vec4) {
              if (red && P.epi == EPI_ADD)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(val.x), "f"(val.y),
                             "f"(val.z), "f"(val.w)
                             : "memory");
              else
                *(float4*)dst = make_float4(res[v].x + val.x, res[v].y + val.y, res[v].z + val.z, res[v].w + val.w);
            } else {
              const float vv[4] = {val.x, val.y, val.z, val.w};
              for (int e = 0; e < 4 && row + e < P.N; ++e) dst[e] = (P.epi == EPI_ADD ? dst[e] : 0.f) + vv[e];
            }
          }
        }
        epi_bar_g(grp);
      }
      }
      // this group has read its chunks of the accumulator: one arrival on the leader
      fence_before();
      if (et == 0) mbar_arrive_cluster(tempty0 + 8u * buf);
      if (++buf == nbuf) { buf = 0; aphase ^= 1; }
    }
    if (P.tma_out && et == 0) bulk_wait<0>();   // every TMA store of this group complete
  }
  fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  fence_after();
  kstamp(P.kst, true);
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
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

// output maps for the pair kernel's TMA stores: fp32 C rows (box 128 features x 16
// tokens, no swizzle) or bf16 SwiGLU rows (box 64 x 16, 128-byte swizzle)
static bool make_out_map(CUtensorMap* m, const void* ptr, int rows, int cols, int ld, bool f32) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || ((uintptr_t)ptr & 15) || (ld * (f32 ? 4 : 2)) % 16) return false;
  cuuint64_t d[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, st[1] = {(cuuint64_t)ld * (f32 ? 4 : 2)};
  cuuint32_t b[2] = {(cuuint32_t)(f32 ? BM : BM / 2), 16u}, es[2] = {1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), d,
            st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, f32 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

static void tc_tiles(int M, int& nt, int& n_tok_tiles, int cap = 0) {
  static const int max_nt_env = [] { const char* e = getenv("HSD_GEMM_MAX_NT"); return e ? atoi(e) : 256; }();
  const int max_nt = cap > 0 ? cap : max_nt_env;
  n_tok_tiles = (M + max_nt - 1) / max_nt;
  nt = (M + n_tok_tiles - 1) / n_tok_tiles;
  nt = (nt + 15) / 16 * 16;
  if (nt < 16) nt = 16;
}

// Data-parallel only with >= 4 output tiles per SM (c3's gate/up and verify
// head): below that, whole-tile ownership leaves SMs idle or unbalanced while
// the weights stream, and stream-K's partial-sum atomics are cheap.
//
// Below that, the CTA-pair kernel (256-row weight tiles, num_sms/2 pairs) still
// owns whole tiles efficiently when its pair-tile count spans >= 1.5 waves and
// fills >= 85 % of the last one (c2 prefill M = 1024: 0.86; 16.5 -> 15.1 ms): c3's QKV (216 pair tiles = 2.92 waves), O and
// down (144 = 1.95 waves) at M = 2080. Batch-1 / small-M shapes (c2, c5 b = 2,
// the draft GEMMs) stay stream-K. HSD_GEMM_DP_WAVE=0 restores the 4-tiles rule.
bool gemm_tc_dp(int M, int N, int K, bool accumulate) {
  int nt, ntt;
  tc_tiles(M, nt, ntt);
  if ((long)((N + BM - 1) / BM) * ntt >= 4L * num_sms()) return true;
  static const bool wave_rule = [] {
    const char* e = getenv("HSD_GEMM_DP_WAVE");
    const char* p = getenv("HSD_GEMM_2SM");
    return !(e && atoi(e) == 0) && !(p && atoi(p) == 0);
  }();
  const long pairs = num_sms() / 2;
  if (!wave_rule || pairs < 1) return false;
  // (K / accumulate are not used by the rule: c3's O projection -- residual add,
  // K = 4096 -- ran at 684 TFLOP/s on pairs vs 876 stream-K in an isolated ncu
  // capture, but keeping it stream-K in the step measured no gain)
  (void)K;
  (void)accumulate;
  const long ptiles = (long)((N + 2 * BM - 1) / (2 * BM)) * ntt;
  const long full = ptiles / pairs, rem = ptiles % pairs;
  const double waves = (double)ptiles / (double)pairs;
  const double eff = waves / (double)(full + (rem ? 1 : 0));
  static const double min_eff = [] { const char* e = getenv("HSD_GEMM_DP_EFF"); return e ? atof(e) : 0.85; }();
  return waves >= 1.5 && eff >= min_eff;
}

// Tiling of the pair kernel: super-tile width wt (256-row weight tiles per tile)
// and token tile nt. The per-pair L2 -> SM operand bytes of a tile are
// (256 wt + nt) K 2 and the busiest pair runs ceil(tiles / pairs) tiles, so pick
// the (wt, nt) with the smallest ceil(tiles / pairs) (256 wt + nt) -- with a 5 %
// handicap on wt = 2 when it leaves one accumulator buffer (the epilogue then no
// longer overlaps the next tile's MMAs). Candidates: the default token tile
// (tc_tiles) and, opt-in, a narrower one (HSD_GEMM_NT_ALT, e.g. 176). c3 (74
// pairs): QKV (N 6144) -> wt 1, nt 240 (3 x 496); with nt 176 allowed -> wt 2,
// nt 176 (2 x 688), 87 vs 100 us with a plain-store epilogue, but no gain in the
// step, where QKV runs the fused RoPE / KV epilogue and wt 2 leaves it one
// accumulator buffer; O / down -> wt 2 (1 x 752); gate/up -> wt 2 (7 x 752).
// HSD_GEMM_WT=1|2 forces the width.
static void pair_tiling(int M, int N, int& wt_out, int& nt_out, int& ntt_out, bool heavy_epi = false) {
  static const int env = [] { const char* e = getenv("HSD_GEMM_WT"); return e ? atoi(e) : 0; }();
  // the fused QKV epilogue (RoPE + scattered cache writes) is too long to leave
  // un-overlapped: with it, only double-buffered (wt = 1) tilings are considered
  // (c3 prefill QKV, M = 4096: 254 us on wt = 2 / one accumulator buffer).
  // HSD_GEMM_QKV_WT2=1 lifts the restriction.
  static const bool qkv_wt2 = [] { const char* e = getenv("HSD_GEMM_QKV_WT2"); return e && atoi(e) == 1; }();
  static const int nt_alt = [] { const char* e = getenv("HSD_GEMM_NT_ALT"); return e ? atoi(e) : 0; }();
  const long pairs = num_sms() / 2;
  double best = 1e300;
  int cands[2] = {0, nt_alt}, nt0 = -1;
  for (int ci = 0; ci < 2; ++ci) {
    if (ci == 1 && nt_alt < 16) continue;
    int nt, ntt;
    tc_tiles(M, nt, ntt, cands[ci]);
    if (ci == 0) nt0 = nt;
    else if (nt >= nt0) continue;                    // the narrower token tile only
    for (int wt = 1; wt <= 2; ++wt) {
      if (env == 1 || env == 2) { if (wt != env) continue; }
      else if (heavy_epi && !qkv_wt2 && wt == 2 && 2 * 2 * nt > 512) continue;
      const long tiles = (long)((N + 2 * BM * wt - 1) / (2 * BM * wt)) * ntt;
      double c = (double)((tiles + pairs - 1) / pairs) * (256.0 * wt + nt);
      if (wt == 2 && 4 * nt > 512) c *= 1.05;
      if (c < best) { best = c; wt_out = wt; nt_out = nt; ntt_out = ntt; }
    }
  }
}

static int gemm_tc2_launch(const bf16* A, int lda, const bf16* W, int ldw, float* C, int ldc, int M, int N, int K,
                           int epi, bf16* H, int ldh, cudaStream_t st, KStamp ks, const QkvEpi* qe = nullptr) {
  TcParams P{};   // (value-initialised: every field not set below is 0)
  if (qe) P.qe = *qe;
  P.M = M; P.N = N; P.K = K; P.ldc = ldc; P.C = C; P.H = H; P.ldh = ldh; P.epi = epi; P.dp = 1;
  P.trace = nullptr;
  P.kst = ks;
  int nt = 0, ntt = 0, wt = 1;
  pair_tiling(M, N, wt, nt, ntt, epi == EPI_QKV);
  P.ntile = nt;
  P.n_tiles_t = ntt;
  P.n_tiles_n = (N + BM - 1) / BM;
  P.n_kb = (K + BK - 1) / BK;
  P.units = 0;
  P.wt = wt;
  {
    const char* e = getenv("HSD_GEMM_EXP");
    P.exp = e ? atoi(e) : 0;
  }
  const int bh = (nt / 2) * BK * 2;
  static const int pre_env = [] { const char* e = getenv("HSD_GEMM_PRE"); return e ? atoi(e) : 1; }();
  static const int pf_env = [] { const char* e = getenv("HSD_GEMM_PF_AHEAD"); return e ? atoi(e) : 0; }();
  P.pre = pre_env;
  P.pf_ahead = pf_env;
  // outputs by TMA store / reduce-add (HSD_GEMM_TMA_OUT=0: thread stores from the
  // padded stage): the epilogue then only stages chunks and issues one bulk copy each
  // (default 2: STORE / ADD only -- SwiGLU's bf16 output by TMA measured neutral to
  // slightly slower: c3 gate/up 352 vs 348 us, step 38.4 vs 37.7 ms; 1: SwiGLU too)
  static const int tma_out_on = [] { const char* e = getenv("HSD_GEMM_TMA_OUT"); return e ? atoi(e) : 2; }();
  CUtensorMap mo;
  memset(&mo, 0, sizeof(mo));
  P.tma_out = 0;
  if (tma_out_on && (epi == EPI_STORE || epi == EPI_ADD) && C)
    P.tma_out = make_out_map(&mo, C, M, N, ldc, true) ? 1 : 0;
  else if (tma_out_on == 1 && epi == EPI_SWIGLU && H)
    P.tma_out = make_out_map(&mo, H, M, N / 2, ldh, false) ? 1 : 0;
  // ring: the 226 KB less the epilogue region (+ its 1024-byte alignment) and barriers
  const size_t epi_bytes = P.tma_out ? 32768 : 2 * 16 * EPI_LD * 4;
  int stages = (int)((226 * 1024 - 2048 - epi_bytes - 512) / (P.wt * A_BYTES + bh));
  if (stages > 16) stages = 16;
  P.stages = stages;
  P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nt >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
  P.nbuf = 2 * P.wt * nt <= 512 ? 2 : 1;
  uint32_t cols = 32;
  while (cols < (uint32_t)(P.nbuf * P.wt * nt)) cols <<= 1;
  P.tmem_cols = cols;
  CUtensorMap mw, mx;
  if (!make_map(&mw, W, N, K, ldw, BM) || !make_map(&mx, A, M, K, lda, nt / 2)) return 0;
  P.vec4 = (ldc % 4 == 0) && (((uintptr_t)C & 15) == 0);
  const size_t smem = 1024 + (size_t)stages * (P.wt * A_BYTES + bh) + (2 * stages + 6) * 8 + 1024 + epi_bytes;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(gemm_tc2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);   // (+ static tmeta)
    cudaFuncSetAttribute(gemm_tc2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    attr_done = true;
  }
  const long pairs = (long)((N + 2 * BM * P.wt - 1) / (2 * BM * P.wt)) * ntt;
  const long max_pairs = num_sms() / 2;
  const long grid = 2 * (pairs < max_pairs ? pairs : max_pairs);
  if (P.wt == 2) launch_k_cluster(gemm_tc2_kernel<2>, dim3((unsigned)grid), dim3(NTHREADS2), smem, st, 2, mw, mx, mo, P);
  else launch_k_cluster(gemm_tc2_kernel<1>, dim3((unsigned)grid), dim3(NTHREADS2), smem, st, 2, mw, mx, mo, P);
  return 1;
}

static int gemm_tc_launch(const bf16* A, int lda, const bf16* W, int ldw, float* C, int ldc, int M, int N, int K,
                          int epi, int dp, bf16* H, int ldh, cudaStream_t st, bool allow_pair = true) {
  TcParams P{};   // (value-initialised: every field not set below is 0)
  P.M = M; P.N = N; P.K = K; P.ldc = ldc; P.C = C; P.H = H; P.ldh = ldh; P.epi = epi; P.dp = dp;
  P.wt = 1; P.nbuf = 2; P.exp = 0;
  P.kst = take_kstamp();
  // data-parallel shapes (large M: c3/c4/c5 verify) run on CTA pairs (2-SM UMMA)
  static const bool pair_on = [] { const char* e = getenv("HSD_GEMM_2SM"); return !(e && atoi(e) == 0); }();
  if (dp && allow_pair && pair_on && num_sms() >= 2) return gemm_tc2_launch(A, lda, W, ldw, C, ldc, M, N, K, epi, H, ldh, st, P.kst);
  static unsigned long long* trace = [] {
    unsigned long long* t = nullptr;
    if (getenv("HSD_GEMM_TRACE")) { cudaMalloc(&t, 32 * 8); cudaMemset(t, 0, 32 * 8); }
    return t;
  }();
  P.trace = trace;
  g_gemm_trace = trace;
  int nt, ntt;
  tc_tiles(M, nt, ntt);
  P.ntile = nt;
  P.n_tiles_t = ntt;
  P.n_tiles_n = (N + BM - 1) / BM;
  P.n_kb = (K + BK - 1) / BK;
  P.units = (long)P.n_tiles_n * P.n_tiles_t * P.n_kb;
  const int b_bytes = nt * BK * 2;
  // ring size: several CTAs per SM (default 2) so one CTA's prologue / epilogue
  // overlaps another's streaming, and PDL-launched successors can become
  // resident while this kernel drains.
  static const int ring_kb = [] { const char* e = getenv("HSD_GEMM_RING_KB"); return e ? atoi(e) : 100; }();
  static const int per_sm = [] { const char* e = getenv("HSD_GEMM_CTAS_PER_SM"); return e ? atoi(e) : 2; }();
  // at least 3 stages in flight: wide token tiles (compute-bound shapes) get a
  // bigger ring and one CTA per SM instead of two shallow ones
  int ring = ring_kb * 1024, cps = per_sm;
  static const int min_stages = [] { const char* e = getenv("HSD_GEMM_MIN_STAGES"); return e ? atoi(e) : 3; }();
  if (ring / (A_BYTES + b_bytes) < min_stages) { ring = 200 * 1024; cps = 1; }
  int stages = ring / (A_BYTES + b_bytes);
  if (stages > 16) stages = 16;
  if (stages < 2) stages = 2;
  P.stages = stages;
  P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nt >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * nt)) cols <<= 1;
  P.tmem_cols = cols;
  CUtensorMap mw, mx;
  if (!make_map(&mw, W, N, K, ldw, BM) || !make_map(&mx, A, M, K, lda, nt)) return 0;
  P.vec4 = (ldc % 4 == 0) && (((uintptr_t)C & 15) == 0);
  // stream-K partials by TMA bulk reduce-add (HSD_GEMM_TMA_SK=0: red.add.v4 from the threads)
  static const int tma_sk = [] { const char* e = getenv("HSD_GEMM_TMA_SK"); return e ? atoi(e) : 1; }();
  CUtensorMap mo;
  memset(&mo, 0, sizeof(mo));
  P.tma_out = (tma_sk && epi == EPI_ATOMIC && C && make_out_map(&mo, C, M, N, ldc, true)) ? 1 : 0;
  size_t smem = 1024 + (size_t)stages * (A_BYTES + b_bytes) + (2 * stages + 6) * 8 + 16 * EPI_LD * 4 + 16;
  if (P.tma_out) smem = 1024 + (size_t)stages * (A_BYTES + b_bytes) + (2 * stages + 6) * 8 + 1024 + 2 * 16 * BM * 4;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = true;
  }
  const long max_ctas = (long)num_sms() * cps;
  const long work = dp ? (long)P.n_tiles_n * P.n_tiles_t : P.units;
  const long grid = work < max_ctas ? work : max_ctas;
  launch_k(gemm_tc_kernel, dim3((unsigned)grid), dim3(NTHREADS), smem, st, mw, mx, mo, P);
  return 1;
}

int gemm_tc_bf16(const bf16* A, int lda, const bf16* W, int ldw, float* C, int ldc, int M, int N, int K,
                 bool accumulate, cudaStream_t st, bool c_zeroed) {
  // data-parallel (whole tiles per CTA, plain stores / residual adds) when the
  // output has at least one tile per SM; else stream-K with red.add partials
  const int dp = gemm_tc_dp(M, N, K, accumulate) ? 1 : 0;
  if (!dp && !accumulate && !c_zeroed) cudaMemset2DAsync(C, (size_t)ldc * 4, 0, (size_t)N * 4, M, st);
  const int epi = dp ? (accumulate ? EPI_ADD : EPI_STORE) : EPI_ATOMIC;
  return gemm_tc_launch(A, lda, W, ldw, C, ldc, M, N, K, epi, dp, nullptr, 0, st);
}

// Decode-size gate/up (one token tile, >= one 128-row weight tile per SM: c2's
// 172 tiles at M <= 256) CAN run data-parallel on single CTAs with SwiGLU in the
// epilogue (whole tiles per CTA in one wave, no stream-K partials, no separate
// SwiGLU launch) -- measured slower on c2 (step 4.73 -> 5.19 ms: one CTA cannot
// pull a 1.4 MB weight tile at its share of HBM bandwidth), so it is opt-in
// (HSD_GEMM_SWIGLU_1CTA=1) for experiments.
static bool swiglu_1cta(int M, int N) {
  static const bool on = [] { const char* e = getenv("HSD_GEMM_SWIGLU_1CTA"); return e && atoi(e) == 1; }();
  int nt, ntt;
  tc_tiles(M, nt, ntt);
  const long tiles = (long)((N + BM - 1) / BM) * ntt;
  return on && ntt == 1 && tiles >= num_sms() && tiles <= 2L * num_sms();
}

bool gemm_tc_swiglu_ok(int M, int N, int K) {
  if (N % BM) return false;
  return gemm_tc_dp(M, N, K, false) || swiglu_1cta(M, N);
}

int gemm_tc_swiglu_bf16(const bf16* A, int lda, const bf16* W, int ldw, bf16* H, int ldh, int M, int N, int K,
                        cudaStream_t st) {
  if (N % BM) return 0;
  if (gemm_tc_dp(M, N, K, false)) return gemm_tc_launch(A, lda, W, ldw, nullptr, 0, M, N, K, EPI_SWIGLU, 1, H, ldh, st);
  if (swiglu_1cta(M, N))
    return gemm_tc_launch(A, lda, W, ldw, nullptr, 0, M, N, K, EPI_SWIGLU, 1, H, ldh, st, /*allow_pair=*/false);
  return 0;
}

// QKV GEMM with RoPE / bf16 q / paged K, V writes fused into the CTA-pair epilogue
// (verify pass at data-parallel shapes: c3 / c4 / c5). Needs whole heads per
// 128-row weight tile and the pair kernel.
bool gemm_tc_qkv_ok(int M, int N, int K, int hd, int Hq, int Hkv) {
  static const bool on = [] { const char* e = getenv("HSD_GEMM_QKV_EPI"); return !(e && atoi(e) == 0); }();
  static const bool pair_on = [] { const char* e = getenv("HSD_GEMM_2SM"); return !(e && atoi(e) == 0); }();
  // every 128-row weight tile holds heads of one kind only (q, k or v)
  // (hd = 128 only: the shapes the full-size parity tests cover -- c3 / c4 / c5 verify and prefill)
  return on && pair_on && num_sms() >= 2 && hd == 128 && (Hq * hd) % BM == 0 && (Hkv * hd) % BM == 0 &&
         N == (Hq + 2 * Hkv) * hd && gemm_tc_dp(M, N, K, false);
}

int gemm_tc_qkv_bf16(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K, const QkvEpi& e,
                     cudaStream_t st) {
  if (!gemm_tc_qkv_ok(M, N, K, e.hd, e.Hq, e.Hkv)) return 0;
  return gemm_tc2_launch(A, lda, W, ldw, nullptr, 0, M, N, K, EPI_QKV, nullptr, 0, st, take_kstamp(), &e);
}
