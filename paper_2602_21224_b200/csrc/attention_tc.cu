// attention_tc.cu -- tree-masked attention on tcgen05 tensor cores (bf16, hd 64/128,
// page_size 64): the verify / draft attention of PAPER.md:95 (tree-shaped
// attention) over the paged KV cache, flash-decoding style with split-KV.
//
// One CTA = (key split, kv head h, request x q-tile of 128 (row, head) pairs).
//  warp 0      : TMA producer -- the q tile once (3-D map: hd x G heads x rows),
//                then per 128-key chunk (2 pages via the block table) K [128 x hd]
//                into a 3-stage K ring (freed by the S MMA);
//  warp 2      : TMA producer of V^T [hd x 128] into a 2-stage V ring (freed by the
//                P V MMA). Two producers, so a K load never queues behind a V load
//                that waits for a P V MMA (one producer serialised them: S_{j+1} was
//                issued only after K_{j+1} landed behind V_j, the load latency
//                exposed every chunk). Chunks wholly below the rows this pass
//                writes load before griddepcontrol.wait.
//  warp 1      : MMA issuer -- S_j = Q K_j^T (M=128, N=128, K=hd) into one of two
//                TMEM score buffers, S_{j+1} issued before P_j is ready; then
//                O += P_j V_j (M=128, N=hd, K=128) with P_j read from TMEM (the
//                bf16 P_j overwrites the first 64 columns of S_j's buffer).
//                The V^T tile carries 16 extra constant rows (a row of ones, then
//                zeros), so the same MMA also accumulates l = sum_k P_jk in O's
//                column hd: the row sum of exactly the bf16 P the MMA consumed,
//                with no per-key additions in the softmax warps.
//  warps 2..   : softmax -- TMEM lane t = one (row, head) is owned by SW warps
//                (same lane quarter), each taking 128 / SW of the chunk's keys:
//                a visibility mask (committed range | tree-ancestor bits, see
//                attention.cu) per 32 keys, scores exponentiated as
//                ex2(s * log2e/sqrt(hd) - m) in one FFMA + ex2.approx, the pair
//                exchanging its row max through shared memory. The running max is
//                raised lazily (only when a chunk exceeds it by > 8 in log2 units),
//                so the O rescale -- the one step that must wait for P_{j-1} V --
//                is rare; P_j is written with tcgen05.st and never waits for the
//                previous PV MMA.
// Splits > 1 write (o, m, l) partials and a merge kernel combines them.
#include <cooperative_groups.h>
#include "kernels.cuh"
#include "tc_ptx.cuh"
namespace cg = cooperative_groups;

unsigned long long* g_attn_trace = nullptr;   // debug phase trace (HSD_ATTN_TRACE)

namespace {
using namespace tc;
// softmax warps per TMEM lane quarter (SW): each owns CHUNK / SW keys of a chunk;
// the CTA has 64 + 128 * SW threads (TMA warp, MMA warp, 4 * SW softmax warps)
// the CTA has 96 + 128 * SW threads: warp 0 TMA (Q, K), warp 1 MMA, warp 2 TMA (V),
// then 4 * SW softmax warps (warp w reads TMEM lane quarter w % 4)
template <int SW> constexpr int nthreads() { return 96 + 128 * SW; }
constexpr int SM0 = 96;        // first softmax thread
constexpr int PAGE = 64;
constexpr int CHUNK = 128;     // keys per softmax iteration = 2 pages
constexpr int QROWS = 128;

// Debug phase trace (HSD_ATTN_TRACE env -> P.trace != null): CTA (0,0,0) records
// %globaltimer at phase boundaries, softmax thread 64 (lane row 64) and MMA lane.
HSD_DEV uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
struct AttnParams {
  int M, R, Hq, G, hd, n_qtiles, max_keys, keys_per_split, direct;
  int dyn;                     // 1: key splits divide the CTA's VISIBLE chunks (device-side), not max_keys
  int exp_flags;               // timing experiments only (HSD_ATTN_EXP, results wrong): 1 = drop the last q-tile
  int cluster;                 // 1: the S key-split CTAs form a cluster and reduce over DSMEM
  RowMeta m;
  KVLayer kv;
  const bf16* q;               // [M][Hq][hd] (read directly when the q tile lives in TMEM)
  bf16* out;
  float* ws;
  uint32_t idesc_s, idesc_o;
  unsigned long long* trace;   // [64] timestamps or null
  L2Pf pf;                     // weights of a later GEMM to prefetch into L2 (common.cuh)
  KStamp kst;                  // per-launch stamps (hsd_kstamp) or kst.buf == null
};
// compiled in only with -DHSD_ATTN_TRACE_ON (the %globaltimer reads cost issue slots in the loop)
#ifdef HSD_ATTN_TRACE_ON
#define TRACE(i) do { if (P.trace && blockIdx.x < 2 && blockIdx.y == 0 && blockIdx.z == 0) P.trace[(i) + 128 * blockIdx.x] = gtime(); } while (0)
#else
#define TRACE(i) do { } while (0)
#endif
constexpr int VEXTRA = 16;     // constant V^T rows per page: row hd = ones (-> l in O column hd), then zeros

// bits [a, b) of a 32-bit word (a, b clamped to [0, 32])
HSD_DEV uint32_t range32(int a, int b) {
  a = max(0, min(32, a));
  b = max(0, min(32, b));
  if (b <= a) return 0u;
  const uint32_t hi = b == 32 ? 0xffffffffu : ((1u << b) - 1u);
  return hi & ~((1u << a) - 1u);
}
// bits d0 .. d0+31 of the 256-bit ancestor mask (0 outside [0, 256))
HSD_DEV uint32_t anc32(const uint64_t (&a)[4], int d0) {
  if (d0 >= 256 || d0 <= -32) return 0u;
  int sh = 0;
  if (d0 < 0) { sh = -d0; d0 = 0; }
  const int w = d0 >> 6, o = d0 & 63;
  uint64_t lo = 0, hi = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {       // static indexing keeps the mask in registers
    if (i == w) lo = a[i];
    if (i == w + 1) hi = a[i];
  }
  const uint64_t v = o == 0 ? lo : ((lo >> o) | (hi << (64 - o)));
  return ((uint32_t)v) << sh;
}
HSD_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
HSD_DEV void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {   // caller issues tcgen05.wait::ld
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
HSD_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
HSD_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// the SW softmax warps of lane quarter q (named barrier 1 + q)
template <int SW>
HSD_DEV void quad_sync(int q) { asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * SW) : "memory"); }

// PAIR: two CTAs of a cluster (cta_group::2, one TPC) run the q-tiles 2c and 2c+1
// of a (request, kv head) as ONE M = 256 tile: S = Q K^T takes B (the 128-key K
// chunk) as two 64-key halves, one page per CTA, and O += P V takes B (V^T, N =
// hd + 16 rows) as two row halves -- every SM stages HALF of each K / V chunk, so
// the per-SM K / V stream (the limit of the single-CTA kernel: TMA latency ~3.5
// us under load through a 3-stage ring) halves, and the
// rings get 4 stages. The leader's lane 0 issues every MMA for the pair; S / P / O
// stay per CTA (each CTA's TMEM holds its 128 rows), so the softmax is unchanged.
template <int SW, bool PAIR>
__global__ void __launch_bounds__(nthreads<SW>(), 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmV2,
                        AttnParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // single CTA: Q lives in TMEM (A operand of S = Q K^T read from TMEM, like P for P V),
  // so its 32 KB of shared memory go to a 4th K stage -- the K ring's depth over the
  // ~3.5 us TMA latency under load sets the chunk period (K landing gated every S)
  constexpr bool QTM = !PAIR;
  constexpr int KSTAGES = 4;                // K ring: a stage frees when its S MMA completes
  constexpr int VSTAGES = PAIR ? 4 : 2;     // V ring: a stage frees when its P V MMA completes
  constexpr int KROWS = PAIR ? PAGE : CHUNK;   // keys of each chunk this CTA stages
  const int hd = P.hd, natom = hd / 64;
  const int q_bytes = QROWS * hd * 2;          // natom atoms of [128 rows x 128 B]
  const int k_bytes = KROWS * hd * 2;          // natom atoms of [KROWS keys x 128 B]
  const int vrows = PAIR ? (hd + VEXTRA) / 2 : hd + VEXTRA;   // V^T rows (of N = hd + 16) staged here
  const int v_page = vrows * 128;              // one page's atom column: [vrows x 128 B]
  const int v_bytes = 2 * v_page;              // 2 atom columns (pages)
  // pair: the cluster is (2, 1, 1) -- x = 2 * split + rank -- and z walks the pairs of q-tiles
  const int crank = PAIR ? (int)(blockIdx.x & 1) : 0;
  const bool leader = crank == 0;
  uint8_t* sQ = base;
  uint8_t* sK = sQ + (QTM ? 0 : q_bytes);
  uint8_t* sV = sK + KSTAGES * k_bytes;
  uint64_t* bars = (uint64_t*)(sV + VSTAGES * v_bytes);   // P lives in TMEM over its S buffer
  uint64_t* kfull = bars;                 // [KSTAGES] (pair: the leader's counts both CTAs' bytes)
  uint64_t* kempty = kfull + KSTAGES;     // [KSTAGES]
  uint64_t* vfull = kempty + KSTAGES;     // [VSTAGES]
  uint64_t* vempty = vfull + VSTAGES;     // [VSTAGES]
  uint64_t* qbar = vempty + VSTAGES;
  uint64_t* sfull = qbar + 1;            // [2]
  uint64_t* pfull = sfull + 2;           // [2]
  uint64_t* pvdone = pfull + 2;          // one phase per P_j V_j MMA
  uint64_t* odone = pvdone + 1;          // after the last P V MMA
  uint32_t* tmem_slot = (uint32_t*)(odone + 1);
  __shared__ int tile_lo, tile_hi, safe_hi;
  constexpr int NTHREADS = nthreads<SW>();
  constexpr int KPW = CHUNK / SW;          // keys per softmax warp per chunk (64 or 32)
  constexpr int NSM = 128 * SW;            // softmax threads
  __shared__ float red_max[2][SW][QROWS];   // [chunk parity][key part][row]
  __shared__ float fin_m[QROWS], fin_l[QROWS];   // cluster mode: this split's (m, l) per tile row
  __shared__ float wts[QROWS][8];                // cluster mode: merge weight of each split, per row

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, h = blockIdx.y;
  const int nsplit = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int nz = PAIR ? P.n_qtiles / 2 : P.n_qtiles;   // grid z entries per (request, kv head)
  const int grp = blockIdx.z / nz;
  const int qt = PAIR ? 2 * (int)(blockIdx.z % nz) + crank : (int)(blockIdx.z % nz);
  const RowMeta& m = P.m;
  const int req = m.req[grp * P.R];
  if (!PAIR && (P.exp_flags & 1) && P.n_qtiles > 1 && qt == P.n_qtiles - 1) return;

  if (threadIdx.x == 0) { tile_lo = 0x7fffffff; tile_hi = 0; safe_hi = 0x7fffffff; TRACE(0); }
  if (threadIdx.x == 32) {
    for (int s = 0; s < KSTAGES; ++s) { mbar_init(&kfull[s], 1); mbar_init(&kempty[s], 1); }
    for (int s = 0; s < VSTAGES; ++s) { mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1); }
    mbar_init(qbar, QTM ? NSM / 32 : 1);   // (Q in TMEM: one arrive per softmax warp)
    // one arrive per softmax warp (pair: the leader's counts both CTAs' warps)
    for (int b = 0; b < 2; ++b) { mbar_init(&sfull[b], 1); mbar_init(&pfull[b], (PAIR ? 2 : 1) * NSM / 32); }
    mbar_init(pvdone, 1);
    mbar_init(odone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the constant rows of every V stage / page: V^T row hd = bf16 1.0, rows hd+1.. = 0
  // (TMA writes the dimension rows only; the ones row has swizzle phase 0 and is
  // uniform anyway). Pair: the follower holds them, at local rows hd - vrows ..
  const int c0row = PAIR ? (crank == 1 ? hd - vrows : vrows) : hd;
  const int n_const = vrows - c0row;
  for (int i = threadIdx.x; i < VSTAGES * 2 * n_const * 32; i += blockDim.x) {
    const int w = i & 31, r = (i >> 5) % n_const, sp = (i >> 5) / n_const;
    ((uint32_t*)(sV + (size_t)sp * v_page + (size_t)(c0row + r) * 128))[w] = r == 0 ? 0x3F803F80u : 0u;
  }
  fence_proxy_async();
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if constexpr (PAIR) {   // the partner's barriers initialised before any load or MMA targets them
    fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    fence_after();
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0) TRACE(1);
  // Programmatic dependent launch: only q and the K/V rows this pass's qkv_rope_kv
  // writes (every request row's own position) come from the kernel right before
  // this one. Every kernel upstream of that one has completed when this grid
  // starts (qkv_rope_kv triggers only after its own griddepcontrol.wait), so the
  // row metadata and all keys below the request's smallest row position (the
  // committed cache, earlier draft passes) are final: they are read -- and their
  // first chunks TMA-loaded -- before the producer's griddepcontrol.wait.
  pdl_trigger();   // dependents wait for this grid's completion before reading it
  // softmax threads: this lane's (row, head) and its key bounds
  const int q4 = warp & 3;
  const int lane_row = q4 * 32 + lane;                // tile row-head index owned by this thread
  int row = -1, head = 0, klo = 0, khi = 0, slot = -1, tb = 0;
  uint64_t anc[4] = {0, 0, 0, 0};
  bool valid = false, writable = false;   // writable: an output row of this request
  if (warp >= 3) {
    const int rh = qt * QROWS + lane_row;
    const int rl = rh / P.G, g = rh % P.G;
    row = grp * P.R + rl;
    head = h * P.G + g;
    writable = rl < P.R && row < P.M;
    valid = writable && m.pos[row] >= 0;
    if (valid) {
      klo = m.klo[row]; khi = m.khi[row]; slot = m.slot[row];
      int lo = klo, hi = khi;
      if (slot >= 0) {
        tb = m.tbase[req];
        for (int w = 0; w < m.anc_words && w < 4; ++w)
          anc[w] = m.anc[((size_t)req * m.t_max + slot) * m.anc_words + w];
        lo = min(lo, tb);
        hi = max(hi, tb + slot + 1);
      }
      if (hi > lo) { atomicMin(&tile_lo, lo); atomicMax(&tile_hi, hi); }
    }
    int pmin = 0x7fffffff;
    for (int r = threadIdx.x - SM0; r < P.R; r += NSM) {
      const int rr = grp * P.R + r;
      const int pr = rr < P.M ? m.pos[rr] : -1;
      if (pr >= 0) {
        pmin = min(pmin, pr);
        if (PAIR) {   // both CTAs of a pair stream the key range of the whole group
          int lo2 = m.klo[rr], hi2 = m.khi[rr];
          const int sl = m.slot[rr];
          if (sl >= 0) { const int t2 = m.tbase[req]; lo2 = min(lo2, t2); hi2 = max(hi2, t2 + sl + 1); }
          if (hi2 > lo2) { atomicMin(&tile_lo, lo2); atomicMax(&tile_hi, hi2); }
        }
      }
    }
    if (pmin != 0x7fffffff) atomicMin(&safe_hi, pmin);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // key range of this split: with P.dyn the S splits divide the chunks this tile
  // actually sees ([tile_lo, tile_hi), known only on the device) evenly, so a
  // context far below the capacity max_keys does not leave splits idle while
  // others take several chunks; identical in every split CTA of the tile
  int k_begin, k_end;
  if (P.dyn) {
    const int c0 = tile_lo / CHUNK, c1 = (tile_hi + CHUNK - 1) / CHUNK;
    const int cps = c1 > c0 ? (c1 - c0 + nsplit - 1) / nsplit : 0;
    k_begin = (c0 + split * cps) * CHUNK;
    k_end = k_begin + cps * CHUNK;
  } else {
    k_begin = split * P.keys_per_split;
    k_end = min(P.max_keys, k_begin + P.keys_per_split);
  }
  const int lo = max(k_begin, tile_lo), hi = min(k_end, tile_hi);
  const int c_first = lo / CHUNK;
  const int n_chunks = hi > lo ? (hi + CHUNK - 1) / CHUNK - c_first : 0;
  const uint32_t tS = tmem;              // 2 x 128 columns (double-buffered scores)
  const uint32_t tO = tmem + 256;        // hd + 16 columns (l in column hd)
  const uint32_t tQ = tmem + 256 + 144;  // (QTM) the q tile: hd / 2 columns, 2 bf16 per column

  if (warp == 0) {
    if (lane == 0 && n_chunks == 0) { l2pf_issue(P.pf); l2pf_issue(P.pf, 1); }
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
      // K/V rows: read once per tile; with several q-tiles per (request, kv head) the
      // sibling tiles' CTAs (co-scheduled, 8 CTAs apart) re-read them from L2
      const uint64_t pol = P.n_qtiles > 1 ? policy_evict_normal() : policy_evict_first();
      const uint64_t polq = policy_evict_last();
      const int row0 = grp * P.R + qt * (QROWS / P.G);
      auto page_of = [&](int j, int pg) {
        return P.kv.block_table[(size_t)req * P.kv.pages_per_req + 2 * (c_first + j) + pg];
      };
      const uint32_t kfull0 = PAIR ? mapa_u32(&kfull[0], 0) : 0u;
      auto load_k = [&](int j) {
        const int s = j % KSTAGES;
        mbar_wait(&kempty[s], ((j / KSTAGES) & 1) ^ 1);
        if (j < 16) TRACE(96 + j);               // K_j load issued
        if constexpr (PAIR) {   // this CTA's page of the chunk (N half), bytes on the leader's barrier
          if (leader) mbar_expect_tx(&kfull[s], 2 * k_bytes);
          const int krow = ((page_of(j, crank) * 2 + 0) * P.kv.kv_heads + h) * PAGE;
          for (int a = 0; a < natom; ++a)
            tma_load_2d_2sm(&tmK, kfull0 + 8u * s, sK + (size_t)s * k_bytes + a * (KROWS * 128), a * 64, krow, pol);
        } else {
          mbar_expect_tx(&kfull[s], k_bytes);
          for (int pg = 0; pg < 2; ++pg) {
            const int krow = ((page_of(j, pg) * 2 + 0) * P.kv.kv_heads + h) * PAGE;
            for (int a = 0; a < natom; ++a)
              tma_load_2d(&tmK, &kfull[s], sK + (size_t)s * k_bytes + a * (CHUNK * 128) + pg * (PAGE * 128), a * 64,
                          krow, pol);
          }
        }
      };
      auto safe = [&](int j) { return (c_first + j + 1) * CHUNK <= safe_hi; };
      int kj = 0;
      while (kj < n_chunks && kj < KSTAGES && safe(kj)) load_k(kj++);
      pdl_wait();
      kst_enter(P.kst);
      if (P.pf.late) l2pf_issue(P.pf, 1);   // (the late variant goes ahead of q)
      if (threadIdx.x == 0) TRACE(2);
      if constexpr (QTM) {
        // (the softmax warps load q into TMEM)
      } else if constexpr (PAIR) {
        if (leader) mbar_expect_tx(qbar, 2 * q_bytes);
        for (int a = 0; a < natom; ++a)
          tma_load_3d_2sm(&tmQ, mapa_u32(qbar, 0), sQ + a * (QROWS * 128), a * 64, h * P.G, row0, polq);
      } else {
        mbar_expect_tx(qbar, q_bytes);
        for (int a = 0; a < natom; ++a)
          tma_load_3d(&tmQ, qbar, sQ + a * (QROWS * 128), a * 64, h * P.G, row0, polq);
      }
      while (kj < n_chunks) load_k(kj++);
      l2pf_issue(P.pf);   // after this CTA's last K load: the bulk prefetch queues behind it in TMA
    }
  } else if (warp == 2) {
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const uint64_t pol = P.n_qtiles > 1 ? policy_evict_normal() : policy_evict_first();
      const uint32_t vfull0 = PAIR ? mapa_u32(&vfull[0], 0) : 0u;
      auto load_v = [&](int j) {
        const int s = j % VSTAGES;
        mbar_wait(&vempty[s], ((j / VSTAGES) & 1) ^ 1);
        if (!PAIR && (P.exp_flags & 2)) { mbar_arrive(&vfull[s]); return; }   // timing experiment: no V traffic
        if (!PAIR || leader) mbar_expect_tx(&vfull[s], 2 * hd * 128);   // (pair: both CTAs' rows)
        for (int pg = 0; pg < 2; ++pg) {
          const int page = P.kv.block_table[(size_t)req * P.kv.pages_per_req + 2 * (c_first + j) + pg];
          const int vrow = ((page * 2 + 1) * P.kv.kv_heads + h) * hd;
          if constexpr (PAIR)   // this CTA's dimension rows: [0, vrows) / [vrows, hd)
            tma_load_2d_2sm(crank ? &tmV2 : &tmV, vfull0 + 8u * s, sV + (size_t)s * v_bytes + pg * v_page, 0,
                            vrow + (crank ? vrows : 0), pol);
          else
            tma_load_2d(&tmV, &vfull[s], sV + (size_t)s * v_bytes + pg * v_page, 0, vrow, pol);
        }
      };
      int vj = 0;
      while (vj < n_chunks && vj < VSTAGES && (c_first + vj + 1) * CHUNK <= safe_hi) load_v(vj++);
      pdl_wait();
      while (vj < n_chunks) load_v(vj++);
    }
  } else if (warp == 1) {
    if (lane == 0 && n_chunks > 0 && leader) {   // (pair: the leader issues for both CTAs)
      mbar_wait(qbar, 0);
      TRACE(3);
      auto commit = [&](uint64_t* bar) {
        if constexpr (PAIR) mma_commit_2sm(bar, 3);
        else mma_commit(bar);
      };
      auto issue_s = [&](int j) {
        const int s = j % KSTAGES;
        mbar_wait(&kfull[s], (j / KSTAGES) & 1);
        fence_after();
        if (j < 16) TRACE(112 + j);              // K_j landed (seen by the MMA warp)
        const uint32_t d = tS + (uint32_t)((j & 1) * CHUNK);
        for (int kk = 0; kk < hd / 16; ++kk) {
          const int a = kk >> 2, off = kk & 3;
          const uint64_t bd = desc_sw128(sK + (size_t)s * k_bytes + a * (KROWS * 128)) + 2 * off;
          if constexpr (QTM) {
            mma_bf16_ts(d, tQ + (uint32_t)(kk * 8), bd, P.idesc_s, kk > 0 ? 1u : 0u);
          } else {
            const uint64_t ad = desc_sw128(sQ + a * (QROWS * 128)) + 2 * off;
            if constexpr (PAIR) mma_bf16_2sm(d, ad, bd, P.idesc_s, kk > 0 ? 1u : 0u);
            else mma_bf16(d, ad, bd, P.idesc_s, kk > 0 ? 1u : 0u);
          }
        }
        commit(&sfull[j & 1]);
        commit(&kempty[s]);
      };
      issue_s(0);
      for (int j = 0; j < n_chunks; ++j) {
        if (j + 1 < n_chunks) issue_s(j + 1);
        if (j < 16) TRACE(64 + 2 * j);           // S_{j+1} issued
        mbar_wait(&pfull[j & 1], (j >> 1) & 1);
        fence_after();
        const int s = j % VSTAGES;
        mbar_wait(&vfull[s], (j / VSTAGES) & 1);
        if (j < 16) TRACE(65 + 2 * j);           // P_j and V_j ready: P V issued
        // O += P_j V_j with P_j (bf16, 2 keys per column) over S_j's TMEM columns;
        // tcgen05.mma executes in issue order, so S_{j+2} (issued later into the
        // same columns) cannot overtake this read
        const uint32_t tP = tS + (uint32_t)((j & 1) * CHUNK);
        for (int kk = 0; kk < CHUNK / 16; ++kk) {
          const int ka = kk >> 2, off = kk & 3;
          const uint64_t vd = desc_sw128(sV + (size_t)s * v_bytes + ka * v_page) + 2 * off;
          if constexpr (PAIR) mma_bf16_ts_2sm(tO, tP + (uint32_t)(kk * 8), vd, P.idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          else mma_bf16_ts(tO, tP + (uint32_t)(kk * 8), vd, P.idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        commit(&vempty[s]);
        commit(pvdone);
      }
      commit(odone);
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int part = (warp - 3) >> 2;                  // which KPW keys of the chunk
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    float mrow = -INFINITY;                            // running row max, log2 domain
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int hcols = hd / SW;                          // this part's O columns
    // a warp whose 32 lane rows are all padding (the last q-tile of a (request, kv
    // head): c3's third tile holds 4 of 128 valid pairs) computes nothing: its P
    // rows are never consumed by a valid O row (rows of P V are independent)
    const bool live = __any_sync(0xffffffffu, valid);
    if constexpr (QTM) {
      // this thread's (row, head) q row, dims [part * hd / SW, (part + 1) * hd / SW), into
      // TMEM columns hd / (2 SW) wide at its lane (bf16 pairs, the A layout of the TS MMA);
      // q is written by the kernel right before this one
      pdl_wait();
      constexpr int QC = 64 / SW;                      // columns per part at hd = 128
      const int qc = hd / (2 * SW);                    // (hd = 64: half of QC)
      uint32_t qw[QC];
      const uint4* src = writable ? (const uint4*)(P.q + ((size_t)row * P.Hq + head) * hd + part * (hd / SW)) : nullptr;
#pragma unroll
      for (int i = 0; i < QC / 4; ++i) {
        const uint4 v = (src && i < qc / 4) ? src[i] : make_uint4(0u, 0u, 0u, 0u);
        qw[4 * i] = v.x; qw[4 * i + 1] = v.y; qw[4 * i + 2] = v.z; qw[4 * i + 3] = v.w;
      }
      if constexpr (QC == 32) {
        if (qc == 32) tmem_st32(tQ + lane_off + (uint32_t)(part * 32), qw);
        else { uint32_t w16[16]; for (int i = 0; i < 16; ++i) w16[i] = qw[i]; tmem_st16(tQ + lane_off + (uint32_t)(part * 16), w16); }
      } else {
        if (qc == 16) tmem_st16(tQ + lane_off + (uint32_t)(part * 16), qw);
        else { uint32_t w8[8]; for (int i = 0; i < 8; ++i) w8[i] = qw[i]; tmem_st8(tQ + lane_off + (uint32_t)(part * 8), w8); }
      }
      tmem_st_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(qbar);
    }
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(&sfull[j & 1], (j >> 1) & 1);   // (also paces the pfull phases)
      fence_after();
      if (live && !(P.exp_flags & 4)) {   // (exp 4: timing experiment without the softmax)
      if (threadIdx.x == SM0 && j < 12) TRACE(8 + 4 * j);
      const int kb = (c_first + j) * CHUNK + part * KPW;       // this part's keys
      uint32_t r0[32], r1[32];
      tmem_ld32_nw(tS + lane_off + (uint32_t)((j & 1) * CHUNK + part * KPW), r0);
      if constexpr (KPW == 64) tmem_ld32_nw(tS + lane_off + (uint32_t)((j & 1) * CHUNK + part * KPW + 32), r1);
      uint32_t vm0 = 0u, vm1 = 0xffffffffu;
      if (valid) {
        vm0 = range32(klo - kb, khi - kb);
        if (slot >= 0) vm0 |= anc32(anc, kb - tb) & range32(0, m.t_max - (kb - tb));
        vm0 &= range32(k_begin - kb, k_end - kb);
        if constexpr (KPW == 64) {
          vm1 = range32(klo - kb - 32, khi - kb - 32);
          if (slot >= 0) vm1 |= anc32(anc, kb + 32 - tb) & range32(0, m.t_max - (kb + 32 - tb));
          vm1 &= range32(k_begin - kb - 32, k_end - kb - 32);
        }
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // raw scores, -inf where invisible (scale_log2 > 0 keeps the order, and is
      // folded into the exponent's FFMA below)
      float s[KPW];
      if (__all_sync(0xffffffffu, (vm0 & vm1) == 0xffffffffu)) {   // whole warp sees all its keys
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(r0[i]);
          if constexpr (KPW == 64) s[32 + i] = __uint_as_float(r1[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = ((vm0 >> i) & 1u) ? __uint_as_float(r0[i]) : -INFINITY;
          if constexpr (KPW == 64) s[32 + i] = ((vm1 >> i) & 1u) ? __uint_as_float(r1[i]) : -INFINITY;
        }
      }
      // 8 independent max chains (a single chain is KPW dependent FMNMX)
      float mxp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mxp[k] = s[k];
#pragma unroll
      for (int i = 8; i < KPW; ++i) mxp[i & 7] = fmaxf(mxp[i & 7], s[i]);
      float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                       fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
      red_max[j & 1][part][lane_row] = mx;
      quad_sync<SW>(q4);
#pragma unroll
      for (int p2 = 0; p2 < SW; ++p2) mx = fmaxf(mx, red_max[j & 1][p2][lane_row]);
      mx *= scale_log2;
      // lazy rescale: keep the running max unless the chunk raises it by more than
      // 2^8 (P <= 256, exact in bf16's exponent range; fp32 O and l absorb it); a
      // row with nothing visible yet has O == 0 exactly, so it just adopts the max
      float alpha = 1.f;
      if (mrow == -INFINITY) {
        mrow = mx;
      } else if (mx > mrow + 8.f) {
        alpha = ex2(mrow - mx);
        mrow = mx;
      }
      const float msub = mrow == -INFINITY ? 0.f : mrow;   // P = 0, never ex2(-inf + inf)
      if (threadIdx.x == SM0 && j < 12) TRACE(9 + 4 * j);
      // P_j (bf16) over this part's KPW/2 columns of S_j (KPW keys, 2 per column);
      // its row sum l is accumulated by the P V MMA itself (O column hd)
      uint32_t pw[32];
#pragma unroll
      for (int i = 0; i < KPW / 2; ++i) {
        const float p0 = ex2(fmaf(s[2 * i], scale_log2, -msub)), p1 = ex2(fmaf(s[2 * i + 1], scale_log2, -msub));
        __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
        pw[i] = *(uint32_t*)&pr;
      }
      if constexpr (KPW == 64) {
        tmem_st32(tS + lane_off + (uint32_t)((j & 1) * CHUNK + part * 32), pw);
      } else {
        uint32_t pw16[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pw16[i] = pw[i];
        tmem_st16(tS + lane_off + (uint32_t)((j & 1) * CHUNK + part * 16), pw16);
      }
      if (__any_sync(0xffffffffu, alpha != 1.f)) {
        // O must hold P_{<j} V exactly once before it is scaled: S_j completing
        // implies P_{j-2} V done, so pvdone is within one phase of j-1
        if (j > 0) {
          mbar_wait(pvdone, (j - 1) & 1);
          fence_after();
        }
        if (threadIdx.x == SM0 && j < 12) TRACE(10 + 4 * j);
        for (int c = 0; c < hcols; c += 16) {
          uint32_t o[16];
          tmem_ld16(tO + lane_off + (uint32_t)(part * hcols + c), o);
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tO + lane_off + (uint32_t)(part * hcols + c), o);
        }
        if (part == 0) {   // the l column (and its 15 zero neighbours)
          uint32_t o[16];
          tmem_ld16(tO + lane_off + (uint32_t)hd, o);
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16(tO + lane_off + (uint32_t)hd, o);
        }
      }
      tmem_st_wait();
      }   // live
      fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && !leader) mbar_arrive_cluster(mapa_u32(&pfull[j & 1], 0));   // the leader issues P V
        else mbar_arrive(&pfull[j & 1]);
      }
      if (threadIdx.x == SM0 && j < 12) TRACE(11 + 4 * j);
    }
    // ------------------------------------------------------------ epilogue
    float ltot = 0.f;   // l = O column hd (the ones row of V^T), 0 for a row that saw nothing
    if (n_chunks > 0) {
      mbar_wait(odone, 0);
      fence_after();
      uint32_t o[16];
      tmem_ld16(tO + lane_off + (uint32_t)hd, o);
      if (valid) ltot = __uint_as_float(o[0]);
    }
    if (threadIdx.x == SM0) { TRACE(4); if (P.trace && blockIdx.x < 2 && blockIdx.y == 0 && blockIdx.z == 0) P.trace[7 + 128 * blockIdx.x] = n_chunks; }
    if (threadIdx.x == SM0) TRACE(56);
    // O half-row (hcols fp32) -> the idle K/V ring (>= 128 rows x hd fp32) ->
    // each warp then writes its 32 rows row by row with coalesced vectors
    float* ostage = (float*)sK;                       // [128 rows][hd + 4]
    const int ost = hd + 4;
    const float inv = (P.direct && ltot > 0.f) ? 1.0f / ltot : 1.0f;
    for (int c = 0; c < hcols; c += 16) {
      uint32_t o[16];
      if (n_chunks > 0) tmem_ld16(tO + lane_off + (uint32_t)(part * hcols + c), o);
      else
        for (int i = 0; i < 16; ++i) o[i] = 0u;
      float* dst = ostage + lane_row * ost + part * hcols + c;
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *(float4*)(dst + i) = ltot > 0.f ? make_float4(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv,
                                                       __uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (P.cluster && part == 0) { fin_m[lane_row] = mrow; fin_l[lane_row] = ltot; }
    asm volatile("bar.sync 5, %0;" ::"r"(NSM) : "memory");   // all softmax warps staged their rows
    if (threadIdx.x == SM0) TRACE(57);
    if (!P.cluster) {
    // the CTA's valid rows of one (kv head, q-tile): all 256 softmax threads write
    // them as coalesced 16-byte vectors; split partials go to ONE contiguous block
    // ws[split][head][row][hd] per (split, head)
    {
      // warp w takes tile rows w*rpi + lane/vpr, stepping 8*rpi; lanes cover hd
      // as float4s; (row, head) of a tile row advance incrementally (no divides)
      const int sw = (threadIdx.x - SM0) >> 5;
      const int n_rh = min(QROWS, P.R * P.G - qt * QROWS);        // valid (row, head) pairs in the tile
      const int vpr = hd / 4, rpi = 32 / vpr;
      const int d4 = (lane % vpr) * 4;
      const int step = 4 * SW * rpi, step_rl = step / P.G, step_g = step % P.G;
      int lr = sw * rpi + lane / vpr;
      int rl2 = (qt * QROWS + lr) / P.G, g2 = (qt * QROWS + lr) % P.G;
      for (; lr < n_rh; lr += step) {
        const int row2 = grp * P.R + rl2, head2 = h * P.G + g2;
        if (row2 < P.M) {
          const float4 x = *(const float4*)(ostage + lr * ost + d4);
          if (P.direct) {
            const __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
            *(uint2*)(P.out + ((size_t)row2 * P.Hq + head2) * hd + d4) =
                make_uint2(*(const uint32_t*)&a, *(const uint32_t*)&b);
          } else {
            *(float4*)(P.ws + (((size_t)split * P.Hq + head2) * P.M + row2) * hd + d4) = x;
          }
        }
        rl2 += step_rl;
        g2 += step_g;
        if (g2 >= P.G) { g2 -= P.G; ++rl2; }
      }
    }
    if (threadIdx.x == SM0) TRACE(58);
    if (!P.direct && writable && part == 0) {
      const size_t base_ml = (size_t)nsplit * P.M * P.Hq * hd;
      const size_t idx = ((size_t)split * P.Hq + head) * P.M + row;
      P.ws[base_ml + 2 * idx] = mrow;      // log2 domain (merge uses exp2)
      P.ws[base_ml + 2 * idx + 1] = ltot;
    }
    }
  }
  if (P.cluster) {
    // split merge inside the cluster: every CTA staged its unnormalised O rows
    // and (m, l) in shared memory; CTA r combines tile rows [r n/S, (r+1) n/S)
    // over the S peers (DSMEM) -- o = sum_s 2^(m_s - M) o_s / sum_s 2^(m_s - M) l_s
    // -- and writes them as bf16. No global partials, no merge kernel.
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int S = gridDim.x, r = (int)cl.block_rank();
    const int n_rh = min(QROWS, P.R * P.G - qt * QROWS);
    const int r0 = r * n_rh / S, r1 = (r + 1) * n_rh / S;
    const int ost = hd + 4;
    if ((int)threadIdx.x < r1 - r0) {
      const int lr = r0 + threadIdx.x;
      float mp[8], lp[8], mm = -INFINITY;
      for (int p = 0; p < S; ++p) {
        mp[p] = *cl.map_shared_rank(&fin_m[lr], p);
        lp[p] = *cl.map_shared_rank(&fin_l[lr], p);
        if (lp[p] > 0.f) mm = fmaxf(mm, mp[p]);
      }
      float l = 0.f;
      for (int p = 0; p < S; ++p) l += lp[p] > 0.f ? lp[p] * ex2(mp[p] - mm) : 0.f;
      const float inv = l > 0.f ? 1.0f / l : 0.f;
      for (int p = 0; p < S; ++p) wts[lr][p] = lp[p] > 0.f ? ex2(mp[p] - mm) * inv : 0.f;
    }
    __syncthreads();
    const float* peer[8];
    for (int p = 0; p < S; ++p) peer[p] = cl.map_shared_rank((const float*)sK, p);
    const int vpr = hd / 4;
    for (int e = threadIdx.x; e < (r1 - r0) * vpr; e += NTHREADS) {
      const int lr = r0 + e / vpr, d4 = (e % vpr) * 4;
      const int rh2 = qt * QROWS + lr, rl2 = rh2 / P.G, g2 = rh2 % P.G, row2 = grp * P.R + rl2;
      if (row2 >= P.M) continue;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = 0; p < S; ++p) {
        const float w = wts[lr][p];
        if (w == 0.f) continue;                 // a split that saw nothing may hold stale rows
        const float4 v = *(const float4*)(peer[p] + lr * ost + d4);
        acc.x += w * v.x; acc.y += w * v.y; acc.z += w * v.z; acc.w += w * v.w;
      }
      const __nv_bfloat162 a = __floats2bfloat162_rn(acc.x, acc.y), b = __floats2bfloat162_rn(acc.z, acc.w);
      *(uint2*)(P.out + ((size_t)row2 * P.Hq + h * P.G + g2) * hd + d4) =
          make_uint2(*(const uint32_t*)&a, *(const uint32_t*)&b);
    }
    cl.sync();   // no CTA leaves while a peer still reads its shared memory
  }
  if (threadIdx.x == 0) TRACE(59);
  if (threadIdx.x == 32) TRACE(60);
  if (threadIdx.x == SM0) TRACE(61);
  if (threadIdx.x == 96) TRACE(62);
  fence_before();
  if constexpr (PAIR)   // neither CTA leaves while the pair's MMAs or arrivals may still touch it
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  fence_after();
  if (threadIdx.x == 0) TRACE(5);
  kst_exit(P.kst);
  if (warp == 2) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---------------------------------------------------------------------------------
// Two q-tiles per CTA (c3 / c4 / c5 verify, every prefill): the per-SM K / V stream
// is the limit of the one-tile kernel -- each SM pulls ~57 GB/s through TMA at most
// (scripts/experiments/tma2d_latency.cu) and every q-tile CTA of a (request, kv head)
// pulls the whole K / V (c3: 3 tiles -> 3x the algorithmic bytes into SMs). Here one
// CTA runs tiles 2c and 2c+1 (M = 256 rows) on every K / V chunk it loads: the S
// and P V MMAs run once per tile on the same shared-memory chunk, the 4 x SW softmax
// warps treat tile A then tile B (the tensor core does tile A's P V and next S while
// the warps work on tile B), so the bytes streamed per (row, head) halve.
// TMEM (512 columns): S_A, S_B (one 128-column buffer each: S_t(j+1) is issued after
// P_t(j) V in the same order, and completes only after it) and O_A, O_B (hd columns).
// Shared memory: q of both tiles, 2-stage K and V rings. l is summed by the softmax
// warps (no ones row: no TMEM column left for it).
template <int SW>
__global__ void __launch_bounds__(nthreads<SW>(), 1)
    attention_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, AttnParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int KSTAGES = 2, VSTAGES = 2;
  const int hd = P.hd, natom = hd / 64;
  const int q_bytes = QROWS * hd * 2;          // one tile: natom atoms of [128 rows x 128 B]
  const int k_bytes = CHUNK * hd * 2;          // natom atoms of [128 keys x 128 B]
  const int v_page = hd * 128;                 // one page's V^T atom column [hd rows x 128 B]
  const int v_bytes = 2 * v_page;
  uint8_t* sQ = base;                          // [2 tiles]
  uint8_t* sK = sQ + 2 * q_bytes;
  uint8_t* sV = sK + KSTAGES * k_bytes;
  uint64_t* bars = (uint64_t*)(sV + VSTAGES * v_bytes);
  uint64_t* kfull = bars;                 // [KSTAGES]
  uint64_t* kempty = kfull + KSTAGES;     // [KSTAGES]
  uint64_t* vfull = kempty + KSTAGES;     // [VSTAGES]
  uint64_t* vempty = vfull + VSTAGES;     // [VSTAGES]
  uint64_t* qbar = vempty + VSTAGES;
  uint64_t* sfull = qbar + 1;             // [tile]
  uint64_t* pfull = sfull + 2;            // [tile]
  uint64_t* odone = pfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(odone + 1);
  constexpr int KPW = CHUNK / SW;          // keys per softmax warp per chunk
  constexpr int NSM = 128 * SW;
  __shared__ int tile_lo, tile_hi, safe_hi, has_b;
  __shared__ float red_max[2][2][SW][QROWS];   // [chunk parity][tile][key part][row]
  __shared__ float red_l[2][SW][QROWS];        // [tile][key part][row]
  __shared__ uint64_t anc_s[2][QROWS][4];      // tree-ancestor bits of every tile row

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, nsplit = gridDim.x, h = blockIdx.y;
  const int nz = (P.n_qtiles + 1) / 2;
  const int grp = blockIdx.z / nz, qt0 = 2 * (int)(blockIdx.z % nz);   // tiles qt0, qt0 + 1
  const RowMeta& m = P.m;
  const int req = m.req[grp * P.R];

  if (threadIdx.x == 0) { tile_lo = 0x7fffffff; tile_hi = 0; safe_hi = 0x7fffffff; has_b = 0; TRACE(0); }
  if (threadIdx.x == 32) {
    for (int s = 0; s < KSTAGES; ++s) { mbar_init(&kfull[s], 1); mbar_init(&kempty[s], 1); }
    for (int s = 0; s < VSTAGES; ++s) { mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1); }
    mbar_init(qbar, 1);
    for (int t = 0; t < 2; ++t) { mbar_init(&sfull[t], 1); mbar_init(&pfull[t], NSM / 32); }
    mbar_init(odone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  // softmax threads: this lane's (row, head) in tile A and in tile B
  const int q4 = warp & 3, lane_row = q4 * 32 + lane;
  int row[2] = {-1, -1}, head[2] = {0, 0}, klo[2] = {0, 0}, khi[2] = {0, 0}, slot[2] = {-1, -1};
  bool valid[2] = {false, false}, writable[2] = {false, false};
  int tb = 0;
  if (warp >= 3) {
    const int part0 = ((warp - 3) >> 2) == 0;
    for (int t = 0; t < 2; ++t) {
      const int rh = (qt0 + t) * QROWS + lane_row;
      const int rl = rh / P.G, g = rh % P.G;
      row[t] = grp * P.R + rl;
      head[t] = h * P.G + g;
      writable[t] = qt0 + t < P.n_qtiles && rl < P.R && row[t] < P.M;
      valid[t] = writable[t] && m.pos[row[t]] >= 0;
      if (valid[t]) {
        klo[t] = m.klo[row[t]]; khi[t] = m.khi[row[t]]; slot[t] = m.slot[row[t]];
        int lo = klo[t], hi = khi[t];
        if (slot[t] >= 0) {
          tb = m.tbase[req];
          if (part0)
            for (int w = 0; w < 4; ++w)
              anc_s[t][lane_row][w] = w < m.anc_words ? m.anc[((size_t)req * m.t_max + slot[t]) * m.anc_words + w] : 0ull;
          lo = min(lo, tb);
          hi = max(hi, tb + slot[t] + 1);
        }
        if (hi > lo) { atomicMin(&tile_lo, lo); atomicMax(&tile_hi, hi); }
        if (t == 1) has_b = 1;
      }
    }
    int pmin = 0x7fffffff;
    for (int r = threadIdx.x - SM0; r < P.R; r += NSM) {
      const int pr = grp * P.R + r < P.M ? m.pos[grp * P.R + r] : -1;
      if (pr >= 0) pmin = min(pmin, pr);
    }
    if (pmin != 0x7fffffff) atomicMin(&safe_hi, pmin);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntile = has_b ? 2 : 1;
  int k_begin, k_end;
  if (P.dyn) {
    const int c0 = tile_lo / CHUNK, c1 = (tile_hi + CHUNK - 1) / CHUNK;
    const int cps = c1 > c0 ? (c1 - c0 + nsplit - 1) / nsplit : 0;
    k_begin = (c0 + split * cps) * CHUNK;
    k_end = k_begin + cps * CHUNK;
  } else {
    k_begin = split * P.keys_per_split;
    k_end = min(P.max_keys, k_begin + P.keys_per_split);
  }
  const int lo = max(k_begin, tile_lo), hi = min(k_end, tile_hi);
  const int c_first = lo / CHUNK;
  const int n_chunks = hi > lo ? (hi + CHUNK - 1) / CHUNK - c_first : 0;
  auto tS = [&](int t) { return tmem + (uint32_t)(t * 128); };          // S_t (P_t over its first 64 columns)
  auto tO = [&](int t) { return tmem + 256u + (uint32_t)(t * 128); };   // O_t: hd columns

  if (warp == 0) {
    if (lane == 0 && n_chunks == 0) { l2pf_issue(P.pf); l2pf_issue(P.pf, 1); }
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
      const uint64_t pol = P.n_qtiles > 2 ? policy_evict_normal() : policy_evict_first();
      const uint64_t polq = policy_evict_last();
      auto load_k = [&](int j) {
        const int s = j % KSTAGES;
        mbar_wait(&kempty[s], ((j / KSTAGES) & 1) ^ 1);
        mbar_expect_tx(&kfull[s], k_bytes);
        for (int pg = 0; pg < 2; ++pg) {
          const int page = P.kv.block_table[(size_t)req * P.kv.pages_per_req + 2 * (c_first + j) + pg];
          const int krow = ((page * 2 + 0) * P.kv.kv_heads + h) * PAGE;
          for (int a = 0; a < natom; ++a)
            tma_load_2d(&tmK, &kfull[s], sK + (size_t)s * k_bytes + a * (CHUNK * 128) + pg * (PAGE * 128), a * 64,
                        krow, pol);
        }
      };
      int kj = 0;
      while (kj < n_chunks && kj < KSTAGES && (c_first + kj + 1) * CHUNK <= safe_hi) load_k(kj++);
      pdl_wait();
      kst_enter(P.kst);
      mbar_expect_tx(qbar, ntile * q_bytes);
      for (int t = 0; t < ntile; ++t) {
        const int row0 = grp * P.R + (qt0 + t) * (QROWS / P.G);
        for (int a = 0; a < natom; ++a)
          tma_load_3d(&tmQ, qbar, sQ + (size_t)t * q_bytes + a * (QROWS * 128), a * 64, h * P.G, row0, polq);
      }
      while (kj < n_chunks) load_k(kj++);
      l2pf_issue(P.pf);
    }
  } else if (warp == 2) {
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const uint64_t pol = P.n_qtiles > 2 ? policy_evict_normal() : policy_evict_first();
      auto load_v = [&](int j) {
        const int s = j % VSTAGES;
        mbar_wait(&vempty[s], ((j / VSTAGES) & 1) ^ 1);
        mbar_expect_tx(&vfull[s], 2 * hd * 128);
        for (int pg = 0; pg < 2; ++pg) {
          const int page = P.kv.block_table[(size_t)req * P.kv.pages_per_req + 2 * (c_first + j) + pg];
          tma_load_2d(&tmV, &vfull[s], sV + (size_t)s * v_bytes + pg * v_page, 0,
                      ((page * 2 + 1) * P.kv.kv_heads + h) * hd, pol);
        }
      };
      int vj = 0;
      while (vj < n_chunks && vj < VSTAGES && (c_first + vj + 1) * CHUNK <= safe_hi) load_v(vj++);
      pdl_wait();
      while (vj < n_chunks) load_v(vj++);
    }
  } else if (warp == 1) {
    if (lane == 0 && n_chunks > 0) {
      mbar_wait(qbar, 0);
      auto issue_s = [&](int t, int j) {   // S_t(j) = Q_t K_j^T
        const int s = j % KSTAGES;
        for (int kk = 0; kk < hd / 16; ++kk) {
          const int a = kk >> 2, off = kk & 3;
          const uint64_t ad = desc_sw128(sQ + (size_t)t * q_bytes + a * (QROWS * 128)) + 2 * off;
          const uint64_t bd = desc_sw128(sK + (size_t)s * k_bytes + a * (CHUNK * 128)) + 2 * off;
          mma_bf16(tS(t), ad, bd, P.idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sfull[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) V_j, P_t from TMEM
        const int s = j % VSTAGES;
        for (int kk = 0; kk < CHUNK / 16; ++kk) {
          const int ka = kk >> 2, off = kk & 3;
          const uint64_t vd = desc_sw128(sV + (size_t)s * v_bytes + ka * v_page) + 2 * off;
          mma_bf16_ts(tO(t), tS(t) + (uint32_t)(kk * 8), vd, P.idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(&kfull[0], 0);
      fence_after();
      for (int t = 0; t < ntile; ++t) issue_s(t, 0);
      mma_commit(&kempty[0]);
      for (int j = 0; j < n_chunks; ++j) {
        const bool more = j + 1 < n_chunks;
        mbar_wait(&vfull[j % VSTAGES], (j / VSTAGES) & 1);
        if (j < 16) TRACE(64 + 2 * j);           // V_j landed
        mbar_wait(&pfull[0], j & 1);
        fence_after();
        issue_pv(0, j);
        if (more) {   // tile A's next scores right behind its P V (S_A overwrites P_A in issue order)
          mbar_wait(&kfull[(j + 1) % KSTAGES], ((j + 1) / KSTAGES) & 1);
          fence_after();
          if (j < 16) TRACE(65 + 2 * j);         // K_{j+1} landed
          issue_s(0, j + 1);
        }
        if (ntile == 2) {
          mbar_wait(&pfull[1], j & 1);
          fence_after();
          issue_pv(1, j);
        }
        mma_commit(&vempty[j % VSTAGES]);
        if (more) {
          if (ntile == 2) issue_s(1, j + 1);
          mma_commit(&kempty[(j + 1) % KSTAGES]);
        }
      }
      mma_commit(odone);
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int part = (warp - 3) >> 2;
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int hcols = hd / SW;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const bool live[2] = {__any_sync(0xffffffffu, valid[0]) != 0, __any_sync(0xffffffffu, valid[1]) != 0};
    for (int j = 0; j < n_chunks; ++j) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (t >= ntile) break;
        mbar_wait(&sfull[t], j & 1);   // also: P_t(j-1) V is done (issued before S_t(j))
        fence_after();
        if (threadIdx.x == SM0 && j < 12) TRACE(8 + 4 * j + 2 * t);       // S_t(j) ready
        if (live[t]) {
          const int kb = (c_first + j) * CHUNK + part * KPW;
          uint32_t r0[32], r1[32];
          tmem_ld32_nw(tS(t) + lane_off + (uint32_t)(part * KPW), r0);
          if constexpr (KPW == 64) tmem_ld32_nw(tS(t) + lane_off + (uint32_t)(part * KPW + 32), r1);
          uint32_t vm0 = 0u, vm1 = 0xffffffffu;
          if (valid[t]) {
            vm0 = range32(klo[t] - kb, khi[t] - kb);
            if (slot[t] >= 0) {
              const uint64_t(&an)[4] = anc_s[t][lane_row];
              uint64_t a4[4] = {an[0], an[1], an[2], an[3]};
              vm0 |= anc32(a4, kb - tb) & range32(0, m.t_max - (kb - tb));
              if constexpr (KPW == 64) vm1 = range32(klo[t] - kb - 32, khi[t] - kb - 32) |
                                             (anc32(a4, kb + 32 - tb) & range32(0, m.t_max - (kb + 32 - tb)));
            } else if constexpr (KPW == 64) {
              vm1 = range32(klo[t] - kb - 32, khi[t] - kb - 32);
            }
            vm0 &= range32(k_begin - kb, k_end - kb);
            if constexpr (KPW == 64) vm1 &= range32(k_begin - kb - 32, k_end - kb - 32);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float s[KPW];
          if (__all_sync(0xffffffffu, (vm0 & vm1) == 0xffffffffu)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              s[i] = __uint_as_float(r0[i]);
              if constexpr (KPW == 64) s[32 + i] = __uint_as_float(r1[i]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              s[i] = ((vm0 >> i) & 1u) ? __uint_as_float(r0[i]) : -INFINITY;
              if constexpr (KPW == 64) s[32 + i] = ((vm1 >> i) & 1u) ? __uint_as_float(r1[i]) : -INFINITY;
            }
          }
          float mxp[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) mxp[k] = s[k];
#pragma unroll
          for (int i = 8; i < KPW; ++i) mxp[i & 7] = fmaxf(mxp[i & 7], s[i]);
          float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                           fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
          red_max[j & 1][t][part][lane_row] = mx;
          quad_sync<SW>(q4);
#pragma unroll
          for (int p2 = 0; p2 < SW; ++p2) mx = fmaxf(mx, red_max[j & 1][t][p2][lane_row]);
          mx *= scale_log2;
          float alpha = 1.f;   // lazy rescale (as in the one-tile kernel)
          if (mrow[t] == -INFINITY) {
            mrow[t] = mx;
          } else if (mx > mrow[t] + 8.f) {
            alpha = ex2(mrow[t] - mx);
            mrow[t] = mx;
          }
          const float msub = mrow[t] == -INFINITY ? 0.f : mrow[t];
          float ps[4] = {0.f, 0.f, 0.f, 0.f};
          uint32_t pw[32];
#pragma unroll
          for (int i = 0; i < KPW / 2; ++i) {
            const float p0 = ex2(fmaf(s[2 * i], scale_log2, -msub)), p1 = ex2(fmaf(s[2 * i + 1], scale_log2, -msub));
            ps[i & 3] += p0 + p1;
            __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
            pw[i] = *(uint32_t*)&pr;
          }
          if constexpr (KPW == 64) {
            tmem_st32(tS(t) + lane_off + (uint32_t)(part * 32), pw);
          } else {
            uint32_t pw16[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pw16[i] = pw[i];
            tmem_st16(tS(t) + lane_off + (uint32_t)(part * 16), pw16);
          }
          if (__any_sync(0xffffffffu, alpha != 1.f)) {   // O_t holds P_t(<j) V: S_t(j) completing implies it
            for (int c = 0; c < hcols; c += 16) {
              uint32_t o[16];
              tmem_ld16(tO(t) + lane_off + (uint32_t)(part * hcols + c), o);
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st16(tO(t) + lane_off + (uint32_t)(part * hcols + c), o);
            }
          }
          lrow[t] = lrow[t] * alpha + ((ps[0] + ps[1]) + (ps[2] + ps[3]));
          tmem_st_wait();
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[t]);
        if (threadIdx.x == SM0 && j < 12) TRACE(9 + 4 * j + 2 * t);       // P_t(j) written
      }
    }
    // ------------------------------------------------------------ epilogue
    if (threadIdx.x == SM0 && P.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) P.trace[7] = n_chunks;
    for (int t = 0; t < 2; ++t) red_l[t][part][lane_row] = lrow[t];
    if (n_chunks > 0) {
      mbar_wait(odone, 0);
      fence_after();
    }
    float* ostage = (float*)sK;                       // [128 rows][hd + 4] (K / V rings idle now)
    const int ost = hd + 4;
    for (int t = 0; t < ntile; ++t) {
      asm volatile("bar.sync 5, %0;" ::"r"(NSM) : "memory");   // red_l written / the previous tile's rows read
      float ltot = 0.f;
#pragma unroll
      for (int p2 = 0; p2 < SW; ++p2) ltot += red_l[t][p2][lane_row];
      if (!valid[t]) ltot = 0.f;
      const float inv = (P.direct && ltot > 0.f) ? 1.0f / ltot : 1.0f;
      for (int c = 0; c < hcols; c += 16) {
        uint32_t o[16];
        if (n_chunks > 0) tmem_ld16(tO(t) + lane_off + (uint32_t)(part * hcols + c), o);
        else
          for (int i = 0; i < 16; ++i) o[i] = 0u;
        float* dst = ostage + lane_row * ost + part * hcols + c;
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *(float4*)(dst + i) = ltot > 0.f ? make_float4(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv,
                                                         __uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      asm volatile("bar.sync 5, %0;" ::"r"(NSM) : "memory");   // all rows of tile t staged
      const int qt = qt0 + t;
      const int sw = (threadIdx.x - SM0) >> 5;
      const int n_rh = min(QROWS, P.R * P.G - qt * QROWS);
      const int vpr = hd / 4, rpi = 32 / vpr;
      const int d4 = (lane % vpr) * 4;
      const int step = 4 * SW * rpi, step_rl = step / P.G, step_g = step % P.G;
      int lr = sw * rpi + lane / vpr;
      int rl2 = (qt * QROWS + lr) / P.G, g2 = (qt * QROWS + lr) % P.G;
      for (; lr < n_rh; lr += step) {
        const int row2 = grp * P.R + rl2, head2 = h * P.G + g2;
        if (row2 < P.M) {
          const float4 x = *(const float4*)(ostage + lr * ost + d4);
          if (P.direct) {
            const __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
            *(uint2*)(P.out + ((size_t)row2 * P.Hq + head2) * hd + d4) =
                make_uint2(*(const uint32_t*)&a, *(const uint32_t*)&b);
          } else {
            *(float4*)(P.ws + (((size_t)split * P.Hq + head2) * P.M + row2) * hd + d4) = x;
          }
        }
        rl2 += step_rl;
        g2 += step_g;
        if (g2 >= P.G) { g2 -= P.G; ++rl2; }
      }
      if (!P.direct && writable[t] && part == 0) {
        const size_t base_ml = (size_t)nsplit * P.M * P.Hq * hd;
        const size_t idx = ((size_t)split * P.Hq + head[t]) * P.M + row[t];
        P.ws[base_ml + 2 * idx] = mrow[t];
        P.ws[base_ml + 2 * idx + 1] = ltot;
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  kst_exit(P.kst);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// split merge: one warp per (row, head), lanes over hd:
// o = sum_s e^{m_s - M} o_s / sum_s e^{m_s - M} l_s
__global__ void attention_merge_bf16_kernel(const float* __restrict__ ws, int S, int M, int Hq, int hd,
                                            bf16* __restrict__ out, L2Pf pf, KStamp kst) {
  l2pf_issue(pf);
  pdl_wait();
  l2pf_issue(pf, 1);
  pdl_trigger();
  // one warp per (row, head); partials are laid out ws[split][head][row][hd]
  const int pair = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (pair >= M * Hq) return;
  const int row = pair / Hq, head = pair % Hq;
  const size_t base = (size_t)S * M * Hq * hd;
  float Mx = -INFINITY;
  for (int s = 0; s < S; ++s) {
    const size_t idx = ((size_t)s * Hq + head) * M + row;
    if (ws[base + 2 * idx + 1] > 0.f) Mx = fmaxf(Mx, ws[base + 2 * idx]);
  }
  float den = 0.f, num[4] = {0.f, 0.f, 0.f, 0.f};
  for (int s = 0; s < S; ++s) {
    const size_t idx = ((size_t)s * Hq + head) * M + row;
    const float l = ws[base + 2 * idx + 1];
    if (l <= 0.f) continue;
    const float w = exp2f(ws[base + 2 * idx] - Mx);   // m is in log2 units
    den = fmaf(w, l, den);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int d = lane + 32 * i;
      if (d < hd) num[i] = fmaf(w, ws[idx * hd + d], num[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) out[(size_t)pair * hd + d] = __float2bfloat16_rn(den > 0.f ? num[i] / den : 0.f);
  }
  kst_exit(kst);   // the split merge ends the attention launch
}
}  // namespace

bool attention_tc_supported(int hd, int page_size, DType dt) {
  return dt == DT_BF16 && page_size == PAGE && (hd == 64 || hd == 128) && tma_available();
}

int launch_attention_tc(const void* q, int M, int R, int n_req, const RowMeta& m, const KVLayer& kv, int Hq,
                        int max_keys, void* out, float* ws, size_t ws_floats, size_t kv_layer_elems,
                        cudaStream_t st) {
  const int hd = kv.head_dim, G = Hq / kv.kv_heads;
  if (QROWS % G) return -1;
  AttnParams P;
  P.pf = take_l2pf();
  P.kst = take_kstamp();
  P.M = M; P.R = R; P.Hq = Hq; P.G = G; P.hd = hd; P.m = m; P.kv = kv;
  P.out = (bf16*)out; P.ws = ws; P.max_keys = max_keys; P.q = (const bf16*)q;
  P.n_qtiles = (R * G + QROWS - 1) / QROWS;
  // CTA pairs (M = 256, cta_group::2) when a (request, kv head) spans >= 2 q-tiles:
  // opt-in (HSD_ATTN_PAIR=1), measured slower on c3 (302 -> 490 us per launch): the
  // follower sees each S through the leader's multicast commit ~0.45 us late and its
  // per-warp remote pfull arrivals (release.cluster) cost ~0.6 us per chunk, so the
  // pair runs at ~2 us per chunk although each SM streams half of it
  static const int pair_env = [] { const char* e = getenv("HSD_ATTN_PAIR"); return e ? atoi(e) : 0; }();
  // two q-tiles per CTA (attention_tc2_kernel) whenever a (request, kv head) spans >= 2
  // q-tiles: c3 / c4 / c5 verify, prefill. HSD_ATTN_TC2=0 keeps one tile per CTA.
  static const int tc2_env = [] { const char* e = getenv("HSD_ATTN_TC2"); return e ? atoi(e) : 0; }();
  const bool tc2 = tc2_env && !pair_env && P.n_qtiles >= 2;
  const bool pair = pair_env && P.n_qtiles >= 2;
  if (pair) P.n_qtiles += P.n_qtiles & 1;
  const int z_per_group = tc2 ? (P.n_qtiles + 1) / 2 : P.n_qtiles;   // CTAs along z per (request, kv head)
  {   // read per launch: scripts/attn_trace.py switches it on for the traced pass only
    const char* e = getenv("HSD_ATTN_EXP");
    P.exp_flags = e ? atoi(e) : 0;
  }
  static bool trace_init = [] {
    if (getenv("HSD_ATTN_TRACE")) cudaMalloc(&g_attn_trace, 256 * 8);
    return true;
  }();
  (void)trace_init;
  P.trace = g_attn_trace;
  P.idesc_s = idesc_bf16(pair ? 256 : 128, CHUNK);
  P.idesc_o = idesc_bf16(pair ? 256 : 128, tc2 ? hd : hd + VEXTRA);   // O columns [0, hd) (+ l in column hd)
  // splits: enough CTAs for ~2 per SM, each split a whole number of pages
  const int base_ctas = n_req * kv.kv_heads * z_per_group;
  const int pages = (max_keys + CHUNK - 1) / CHUNK;     // chunks of 2 pages
  // key splits: the kernel holds ~190 KB of shared memory and all 512 TMEM
  // columns (one CTA per SM) and pays ~3 chunk-times of fixed cost per CTA (PDL
  // wait, Q load, epilogue), so extra splits only pay while the grid is under
  // about one wave: S = round(SMs / base), measured best on c2 (S=4), c3 (S=1,
  // monotone worse above) and c5 batch 2 (S=2) -- DESIGN.md section 7.
  int S = max(1, (2 * num_sms() + base_ctas) / (2 * base_ctas));
  S = min(S, max(1, pages / 2));
  // Latency-bound regime (a few chunks per split CTA, c2): one CTA per SM (all TMEM
  // columns, ~190 KB of shared memory), so a second wave of split CTAs adds a whole
  // CTA latency -- cap S at one wave (c2: S 5 -> 4) and divide the chunks each tile
  // really sees evenly on the device (c2 step 4.95 -> 4.73 ms). With many chunks
  // per split (c5, b = 2: 70 chunks) the per-SM K/V stream is the limit and
  // spreading over every SM wins even past one wave (cap there: 46.1 -> 48.8 ms).
  // HSD_ATTN_DYNSPLIT: 0 off, 1 cap + device ranges (default), 2 cap only.
  static const int dyn = [] { const char* e = getenv("HSD_ATTN_DYNSPLIT"); return e ? atoi(e) : 1; }();
  const bool latency_bound = (pages + S - 1) / S <= 4;
  if (dyn && latency_bound) S = min(S, max(1, num_sms() / base_ctas));
  P.dyn = dyn == 1 && latency_bound;
  static const int s_override = [] { const char* e = getenv("HSD_ATTN_SPLITS"); return e ? atoi(e) : 0; }();
  if (s_override > 0) S = min(s_override, pages);
  // two splits reduce inside a 2-CTA cluster over DSMEM (no workspace, no merge
  // kernel): c5 (b = 2) attention 6.8-7.3 -> 6.5 ms. Wider clusters measured
  // slower (c2, S = 4: step 4.95 -> 5.38 ms) -- a 2-CTA cluster fits one TPC's SM
  // pair, 4+ need GPC-wide co-scheduling against the PDL-overlapped predecessor.
  // HSD_ATTN_CLUSTER_MAX raises the limit (<= 8) for experiments.
  static const int cluster_max = [] {
    const char* e = getenv("HSD_ATTN_CLUSTER_MAX");
    return e ? atoi(e) : 2;
  }();
  P.cluster = (!pair && !tc2 && S >= 2 && S <= cluster_max && S <= 8) ? 1 : 0;
  while (!P.cluster && S > 1 && (size_t)S * M * Hq * (hd + 2) > ws_floats) --S;
  int pps = (pages + S - 1) / S;
  P.keys_per_split = pps * CHUNK;
  if (!P.cluster && !P.dyn) S = (pages + pps - 1) / pps;   // cluster / dynamic modes keep S (empty splits contribute 0)
  P.direct = S == 1;
  // tensor maps: q [M][Hq][hd] viewed (hd, heads, rows) with the head offset in
  // the coordinate; K pool rows of hd; V^T pool rows of page_size.
  CUtensorMap mq, mk, mv, mv2;
  uint64_t dq[3] = {(uint64_t)hd, (uint64_t)Hq, (uint64_t)M};
  uint64_t sq[2] = {(uint64_t)hd, (uint64_t)Hq * hd};
  uint32_t bq[3] = {64, (uint32_t)G, (uint32_t)(QROWS / G)};
  uint64_t dk[2] = {(uint64_t)hd, (uint64_t)(kv_layer_elems / hd)};
  uint64_t sk[1] = {(uint64_t)hd};
  uint32_t bk[2] = {64, (uint32_t)PAGE};
  uint64_t dv[2] = {(uint64_t)PAGE, (uint64_t)(kv_layer_elems / PAGE)};
  uint64_t sv[1] = {(uint64_t)PAGE};
  // pair: the leader stages V^T rows [0, vrows), the follower [vrows, hd) (+ the constant rows)
  const int vrows = pair ? (hd + VEXTRA) / 2 : hd;
  uint32_t bv[2] = {(uint32_t)PAGE, (uint32_t)vrows};
  uint32_t bv2[2] = {(uint32_t)PAGE, (uint32_t)(pair ? hd - vrows : hd)};
  if (!tma_map_bf16(&mq, q, 3, dq, sq, bq) || !tma_map_bf16(&mk, kv.base, 2, dk, sk, bk) ||
      !tma_map_bf16(&mv, kv.base, 2, dv, sv, bv) || !tma_map_bf16(&mv2, kv.base, 2, dv, sv, bv2))
    return -1;
  const int kst = tc2 ? 2 : 4, vst = (pair ? 4 : 2);
  const size_t smem = tc2 ? 1024 + 2 * (size_t)QROWS * hd * 2 + kst * ((size_t)CHUNK * hd * 2) +
                                vst * ((size_t)2 * hd * 128) + (2 * kst + 2 * vst + 8) * 8 + 64
                          : 1024 + (pair ? (size_t)QROWS * hd * 2 : 0) + kst * ((size_t)(pair ? PAGE : CHUNK) * hd * 2) +
                                vst * ((size_t)2 * (pair ? (hd + VEXTRA) / 2 : hd + VEXTRA) * 128) +
                                (2 * kst + 2 * vst + 8) * 8 + 64;
  // softmax warps per lane quarter: 2 (8 softmax warps, 64 keys each) or 4 (16 warps,
  // 32 keys each: shorter per-thread chains, more warps to hide TMEM/barrier latency).
  // Measured: c3 (768 CTAs, many waves) attention 11.6 -> 11.1
  // ms with 4; c2 (<= 1 wave) 1.05 -> 1.08 ms. So 4 when the grid spans > 2 waves.
  // HSD_ATTN_SW=2|4 forces one.
  static const int sw_env = [] { const char* e = getenv("HSD_ATTN_SW"); return e ? atoi(e) : 0; }();
  const int sw = sw_env == 2 || sw_env == 4 ? sw_env : ((size_t)S * base_ctas > 2 * (size_t)num_sms() ? 4 : 2);
  static size_t attr[6] = {0, 0, 0, 0, 0, 0};   // (the kernels also have ~2-18 KB of static shared memory)
  auto launch = [&](auto kern, int nthr, size_t& at) {
    if (smem > at) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      at = smem;
    }
    dim3 grid(pair ? 2 * S : S, kv.kv_heads, n_req * (pair ? P.n_qtiles / 2 : z_per_group));
    if (pair) launch_k_cluster(kern, grid, dim3(nthr), smem, st, 2, mq, mk, mv, mv2, P);
    else if (P.cluster) launch_k_cluster(kern, grid, dim3(nthr), smem, st, S, mq, mk, mv, mv2, P);
    else launch_k(kern, grid, dim3(nthr), smem, st, mq, mk, mv, mv2, P);
    if (getenv("HSD_DEBUG_LAUNCH")) {
      const cudaError_t e = cudaPeekAtLastError();
      fprintf(stderr, "attention_tc launch: grid (%d, %d, %d) threads %d smem %zu pair %d cluster %d S %d M %d R %d G %d: %s\n",
              grid.x, grid.y, grid.z, nthr, smem, (int)pair, P.cluster, S, M, R, G, cudaGetErrorString(e));
    }
    return true;
  };
  auto launch3 = [&](auto kern, int nthr, size_t& at) {   // two-tile kernel: (q, K, V) maps
    if (smem > at) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      at = smem;
    }
    launch_k(kern, dim3(S, kv.kv_heads, n_req * z_per_group), dim3(nthr), smem, st, mq, mk, mv, P);
    return true;
  };
  bool ok;
  if (tc2) ok = sw == 4 ? launch3(attention_tc2_kernel<4>, nthreads<4>(), attr[5])
                        : launch3(attention_tc2_kernel<2>, nthreads<2>(), attr[4]);
  else if (pair) ok = sw == 4 ? launch(attention_tc_kernel<4, true>, nthreads<4>(), attr[3])
                         : launch(attention_tc_kernel<2, true>, nthreads<2>(), attr[2]);
  else ok = sw == 4 ? launch(attention_tc_kernel<4, false>, nthreads<4>(), attr[1])
                    : launch(attention_tc_kernel<2, false>, nthreads<2>(), attr[0]);
  if (!ok) return -1;
  if (P.cluster) return 1;
  int launched = 1;
  if (S > 1) {
    launch_k(attention_merge_bf16_kernel, (M * Hq + 7) / 8, 256, 0, st, ws, S, M, Hq, hd, (bf16*)out,
             take_l2pf(), P.kst);
    launched++;
  }
  return launched;
}
