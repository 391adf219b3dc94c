// attention_tc.cu -- tree-masked attention on tcgen05 tensor cores (bf16, hd 64/128,
// page_size 64): the verify / draft attention of PAPER.md:95 (tree-shaped
// attention) over the paged KV cache, flash-decoding style with split-KV.
//
// One CTA = (key split, kv head h, request x q-tile of 128 (row, head) pairs).
//  warp 0      : TMA producer of K -- per 128-key chunk (2 pages via the block
//                table) K [128 x hd] into a 4-stage K ring (freed by the S MMA);
//  warp 2      : TMA producer of V^T [hd x 128] into a 2-stage V ring (freed by the
//                P V MMA). Two producers, so a K load never queues behind a V load
//                that waits for a P V MMA. Chunks wholly below the rows this pass
//                writes load before griddepcontrol.wait.
//  warp 1      : MMA issuer -- S_j = Q K_j^T (M=128, N=128, K=hd) into one of two
//                TMEM score buffers with q read from TMEM (TS form), S_{j+1} issued
//                before P_j is ready; then O += P_j V_j (M=128, N=hd+16, K=128) with
//                P_j read from TMEM (the bf16 P_j overwrites the first 64 columns of
//                S_j's buffer). The V^T tile carries 16 extra constant rows (a row of
//                ones, then zeros), so the same MMA also accumulates l = sum_k P_jk in
//                O's column hd: the row sum of exactly the bf16 P the MMA consumed.
//  warps 3..   : softmax -- first each thread writes its (row, head) q row into the
//                TMEM q tile (its share of the columns), then per chunk: TMEM lane
//                t = one (row, head) is owned by SW warps (same lane quarter), each
//                taking 128 / SW of the chunk's keys: a visibility mask (committed
//                range | tree-ancestor bits, see attention.cu) per 32 keys, scores
//                exponentiated as ex2(s * log2e/sqrt(hd) - m) in one FFMA +
//                ex2.approx, the SW warps exchanging their row max through shared
//                memory. The running max is raised lazily (only when a chunk exceeds
//                it by > 8 in log2 units), so the O rescale -- the one step that must
//                wait for P_{j-1} V -- is rare; P_j is written with tcgen05.st and
//                never waits for the previous PV MMA. A warp whose 32 rows are all
//                padding skips the chunk (rows of P V are independent).
// TMEM: 2 x 128 score columns, hd + 16 O columns, hd / 2 q columns (512 allocated).
// Splits > 1 write (o, m, l) partials; 2 splits merge over DSMEM in a 2-CTA cluster,
// more by a merge kernel.
//
// Measured alternatives: two q-tiles per CTA and CTA pairs
// (cta_group::2, M = 256) both halve the K / V stream per row but ran slower on c3;
// per 128 x 128 chunk the softmax (~1.1-1.3 us), the tensor core (~1.0 us for S and
// P V) and the per-SM TMA stream (64 KB at <= ~57 GB/s) are already balanced.
#include <cooperative_groups.h>
#include "kernels.cuh"
#include "tc_ptx.cuh"
namespace cg = cooperative_groups;

unsigned long long* g_attn_trace = nullptr;   // debug phase trace (HSD_ATTN_TRACE)

namespace {
using namespace tc;
// softmax warps per TMEM lane quarter (SW): each owns CHUNK / SW keys of a chunk;
// the CTA has 96 + 128 * SW threads: warp 0 TMA (K), warp 1 MMA, warp 2 TMA (V),
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
  int light_last;              // 1: the partly filled last q-tiles run after all full ones (HSD_ATTN_ORDER)
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
// 2^x on the FMA pipe for finite x <= 8 (the lazy running max bounds x): 2^floor(x)
// times a degree-3 minimax polynomial of the fraction (max rel err ~1e-4, below the
// bf16 rounding of P); x clamped at -125 (the result is then ~2^-125, not 0 -- used
// only where every key is visible, so no -inf inputs)
HSD_DEV float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float fi = floorf(x);
  const float f = x - fi;
  const float p = fmaf(fmaf(fmaf(0.0788220f, f, 0.2261575f), f, 0.6951461f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)fi << 23));
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

// NPOLY of each thread's KPW exponentials (fully visible chunks) run on the FMA pipe
// instead of MUFU (16 ex2 / clock / SM bounds the exponent phase)
template <int SW, int NPOLY>
__global__ void __launch_bounds__(nthreads<SW>(), 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // single CTA: Q lives in TMEM (A operand of S = Q K^T read from TMEM, like P for P V),
  // so its 32 KB of shared memory go to a 4th K stage -- the K ring's depth over the
  // ~3.5 us TMA latency under load sets the chunk period (K landing gated every S)
  constexpr int KSTAGES = 4;                // K ring: a stage frees when its S MMA completes
  constexpr int VSTAGES = 2;                // V ring: a stage frees when its P V MMA completes
  const int hd = P.hd, natom = hd / 64;
  const int k_bytes = CHUNK * hd * 2;          // natom atoms of [128 keys x 128 B] (2 pages each)
  const int v_page = (hd + VEXTRA) * 128;      // one page's atom column: [hd + 16 rows x 128 B]
  const int v_bytes = 2 * v_page;              // 2 atom columns (pages)
  uint8_t* sK = base;
  uint8_t* sV = sK + KSTAGES * k_bytes;
  uint64_t* bars = (uint64_t*)(sV + VSTAGES * v_bytes);   // P lives in TMEM over its S buffer
  uint64_t* kfull = bars;                 // [KSTAGES]
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
  const int split = blockIdx.x, nsplit = gridDim.x, h = blockIdx.y;
  // CTA order: (request, q-tile) request-major, or with P.light_last the partly
  // filled last q-tile of every request after all full ones (longest first)
  int grp, qt;
  if (P.light_last) {
    const int nf = P.n_qtiles - 1, nfull = nf * (int)(gridDim.z / P.n_qtiles);
    if ((int)blockIdx.z < nfull) { grp = blockIdx.z / nf; qt = blockIdx.z % nf; }
    else { grp = blockIdx.z - nfull; qt = nf; }
  } else {
    grp = blockIdx.z / P.n_qtiles; qt = blockIdx.z % P.n_qtiles;
  }
  const RowMeta& m = P.m;
  const int req = m.req[grp * P.R];
  if ((P.exp_flags & 1) && P.n_qtiles > 1 && qt == P.n_qtiles - 1) return;

  if (threadIdx.x == 0) { tile_lo = 0x7fffffff; tile_hi = 0; safe_hi = 0x7fffffff; TRACE(0); }
  if (threadIdx.x == 32) {
    for (int s = 0; s < KSTAGES; ++s) { mbar_init(&kfull[s], 1); mbar_init(&kempty[s], 1); }
    for (int s = 0; s < VSTAGES; ++s) { mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1); }
    mbar_init(qbar, NSM / 32);             // q in TMEM: one arrive per softmax warp
    for (int b = 0; b < 2; ++b) { mbar_init(&sfull[b], 1); mbar_init(&pfull[b], NSM / 32); }   // one arrive per softmax warp
    mbar_init(pvdone, 1);
    mbar_init(odone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the constant rows of every V stage / page: V^T row hd = bf16 1.0, rows hd+1.. = 0
  // (TMA writes rows [0, hd) only; row hd has swizzle phase 0 and is uniform anyway)
  for (int i = threadIdx.x; i < VSTAGES * 2 * VEXTRA * 32; i += blockDim.x) {
    const int w = i & 31, r = (i >> 5) % VEXTRA, sp = (i >> 5) / VEXTRA;
    ((uint32_t*)(sV + (size_t)sp * v_page + (size_t)(hd + r) * 128))[w] = r == 0 ? 0x3F803F80u : 0u;
  }
  fence_proxy_async();
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
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
      if (pr >= 0) pmin = min(pmin, pr);
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
  const uint32_t tQ = tmem + 256 + 144;  // the q tile: hd / 2 columns, 2 bf16 per column

  if (warp == 0) {
    if (lane == 0 && n_chunks == 0) { l2pf_issue(P.pf); l2pf_issue(P.pf, 1); }
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
      // K/V rows: read once per tile; with several q-tiles per (request, kv head) the
      // sibling tiles' CTAs (co-scheduled, 8 CTAs apart) re-read them from L2
      const uint64_t pol = P.n_qtiles > 1 ? policy_evict_normal() : policy_evict_first();
      auto load_k = [&](int j) {
        const int s = j % KSTAGES;
        mbar_wait(&kempty[s], ((j / KSTAGES) & 1) ^ 1);
        if (j < 16) TRACE(96 + j);               // K_j load issued
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
      if (P.pf.late) l2pf_issue(P.pf, 1);
      if (threadIdx.x == 0) TRACE(2);
      while (kj < n_chunks) load_k(kj++);
      l2pf_issue(P.pf);   // after this CTA's last K load: the bulk prefetch queues behind it in TMA
    }
  } else if (warp == 2) {
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const uint64_t pol = P.n_qtiles > 1 ? policy_evict_normal() : policy_evict_first();
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
      mbar_wait(qbar, 0);   // q in TMEM (written by the softmax warps)
      fence_after();
      TRACE(3);
      auto issue_s = [&](int j) {   // S_j = Q K_j^T, A (q) from TMEM
        const int s = j % KSTAGES;
        mbar_wait(&kfull[s], (j / KSTAGES) & 1);
        fence_after();
        if (j < 16) TRACE(112 + j);              // K_j landed (seen by the MMA warp)
        const uint32_t d = tS + (uint32_t)((j & 1) * CHUNK);
        for (int kk = 0; kk < hd / 16; ++kk) {
          const int a = kk >> 2, off = kk & 3;
          const uint64_t bd = desc_sw128(sK + (size_t)s * k_bytes + a * (CHUNK * 128)) + 2 * off;
          mma_bf16_ts(d, tQ + (uint32_t)(kk * 8), bd, P.idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sfull[j & 1]);
        mma_commit(&kempty[s]);
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
          mma_bf16_ts(tO, tP + (uint32_t)(kk * 8), vd, P.idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&vempty[s]);
        mma_commit(pvdone);
      }
      mma_commit(odone);
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
    {
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
      const bool allvis = __all_sync(0xffffffffu, (vm0 & vm1) == 0xffffffffu);
      if (allvis) {   // whole warp sees all its keys
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
      if (NPOLY > 0 && allvis) {
#pragma unroll
        for (int i = 0; i < KPW / 2; ++i) {
          const float x0 = fmaf(s[2 * i], scale_log2, -msub), x1 = fmaf(s[2 * i + 1], scale_log2, -msub);
          const bool poly = (i % (KPW / 2 / (NPOLY / 2 > 0 ? NPOLY / 2 : 1))) == 0;   // spread over the row
          const float p0 = poly ? ex2_poly(x0) : ex2(x0), p1 = poly ? ex2_poly(x1) : ex2(x1);
          __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
          pw[i] = *(uint32_t*)&pr;
        }
      } else {
#pragma unroll
        for (int i = 0; i < KPW / 2; ++i) {
          const float p0 = ex2(fmaf(s[2 * i], scale_log2, -msub)), p1 = ex2(fmaf(s[2 * i + 1], scale_log2, -msub));
          __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
          pw[i] = *(uint32_t*)&pr;
        }
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
        mbar_arrive(&pfull[j & 1]);
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
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) TRACE(5);
  kst_exit(P.kst);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}


// ------------------------------------------------------------ dual-tile kernel
// One CTA = (key split, kv head h, request x PAIR of q-tiles {2p, 2p+1}): one K / V
// stream feeds 256 (row, head) pairs, so each SM ingests half the K / V bytes per
// row of the single-tile kernel. Each q-tile keeps the single-tile kernel's
// pipeline -- a double-buffered score tile, so S_X(j+1) is computed while the
// softmax group of tile X turns S_X(j) into P_X(j) -- and the two tiles' groups
// share the MMA warp and the K / V rings.
//  Chunks of 64 keys (one page). TMEM per tile X (256 columns): two score buffers
//  of 64 columns (P as bf16 over a buffer's first 32 columns), O_X [hd]. q tiles
//  in shared memory (SS-form S MMAs), 4-stage K and V^T rings of one page each.
//  The row sum l is accumulated by the softmax warps from the bf16-rounded P the
//  MMA consumes; a lazy rescale waits for P_X(j-1) V (pvdone) like the single-tile
//  kernel.
constexpr int DCHUNK = 64;
constexpr int DST = 4;   // ring stages (K and V each)
template <int SW> constexpr int dual_threads() { return 96 + 2 * 128 * SW; }

template <int SW>
__global__ void __launch_bounds__(dual_threads<SW>(), 1)
    attention_dual_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                          AttnParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int hd = P.hd, natom = hd / 64;
  const int q_bytes = QROWS * hd * 2;           // one q tile: natom atoms [128 rows x 128 B]
  const int k_bytes = DCHUNK * hd * 2;          // natom atoms [64 keys x 128 B]
  const int v_bytes = hd * 128;                 // V^T [hd rows x 64 keys]
  uint8_t* sQ = base;
  uint8_t* sK = sQ + 2 * q_bytes;
  uint8_t* sV = sK + DST * k_bytes;
  uint64_t* bars = (uint64_t*)(sV + DST * v_bytes);
  uint64_t* kfull = bars;                 // [DST]
  uint64_t* kempty = kfull + DST;         // [DST]
  uint64_t* vfull = kempty + DST;         // [DST]
  uint64_t* vempty = vfull + DST;         // [DST]
  uint64_t* qbar = vempty + DST;
  uint64_t* sfull = qbar + 1;             // [tile][buffer]
  uint64_t* pfull = sfull + 4;            // [tile][buffer]
  uint64_t* pvdone = pfull + 4;           // [tile]: one phase per P_X(j) V
  uint64_t* odone = pvdone + 2;
  uint32_t* tmem_slot = (uint32_t*)(odone + 1);
  __shared__ int tile_lo, tile_hi, safe_hi;
  constexpr int NSMG = 128 * SW;                // softmax threads per group
  constexpr int KPW = DCHUNK / SW;              // keys per softmax warp per chunk (32 at SW = 2)
  static_assert(KPW == 32 || KPW == 16, "dual kernel: SW 2 or 4");
  __shared__ float red_max[2][2][SW][QROWS];    // [tile][chunk parity][part][row]
  __shared__ float red_l[2][SW][QROWS];         // epilogue: l per part

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, nsplit = gridDim.x, h = blockIdx.y;
  const int npairs = (P.n_qtiles + 1) / 2;
  const int grp = blockIdx.z / npairs, tp = blockIdx.z % npairs;
  const RowMeta& m = P.m;
  const int req = m.req[grp * P.R];
  const int RG = P.R * P.G;
  const bool hasB = (2 * tp + 1) * QROWS < RG;   // (uniform) tile B holds at least one pair

  if (threadIdx.x == 0) { tile_lo = 0x7fffffff; tile_hi = 0; safe_hi = 0x7fffffff; }
  if (threadIdx.x == 32) {
    for (int s = 0; s < DST; ++s) {
      mbar_init(&kfull[s], 1); mbar_init(&kempty[s], 1);
      mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1);
    }
    mbar_init(qbar, (hasB ? 2 : 1) * NSMG / 32);
    for (int x = 0; x < 4; ++x) { mbar_init(&sfull[x], 1); mbar_init(&pfull[x], NSMG / 32); }
    for (int x = 0; x < 2; ++x) mbar_init(&pvdone[x], 1);
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
  const int X = warp >= 3 ? (warp - 3) / (4 * SW) : 0;
  const bool in_tile = warp >= 3 && (X == 0 || hasB);
  const int q4 = warp & 3;
  const int lane_row = q4 * 32 + lane;
  const int part = warp >= 3 ? ((warp - 3) % (4 * SW)) >> 2 : 0;
  const int qt = 2 * tp + X;
  int row = -1, head = 0, klo = 0, khi = 0, slot = -1, tb = 0;
  uint64_t anc[4] = {0, 0, 0, 0};
  bool valid = false, writable = false;
  if (in_tile) {
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
      if (hi > lo && part == 0) { atomicMin(&tile_lo, lo); atomicMax(&tile_hi, hi); }
    }
  }
  if (warp >= 3) {
    int pmin = 0x7fffffff;
    for (int r = threadIdx.x - SM0; r < P.R; r += 2 * NSMG) {
      const int rr = grp * P.R + r;
      const int pr = rr < P.M ? m.pos[rr] : -1;
      if (pr >= 0) pmin = min(pmin, pr);
    }
    if (pmin != 0x7fffffff) atomicMin(&safe_hi, pmin);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  int k_begin, k_end;
  if (P.dyn) {
    const int c0 = tile_lo / DCHUNK, c1 = (tile_hi + DCHUNK - 1) / DCHUNK;
    const int cps = c1 > c0 ? (c1 - c0 + nsplit - 1) / nsplit : 0;
    k_begin = (c0 + split * cps) * DCHUNK;
    k_end = k_begin + cps * DCHUNK;
  } else {
    k_begin = split * P.keys_per_split;
    k_end = min(P.max_keys, k_begin + P.keys_per_split);
  }
  const int lo = max(k_begin, tile_lo), hi = min(k_end, tile_hi);
  const int c_first = lo / DCHUNK;
  const int n_chunks = hi > lo ? (hi + DCHUNK - 1) / DCHUNK - c_first : 0;
  // TMEM columns of tile x: score buffers at 256 x + {0, 64}, O at 256 x + 128
  auto tS_of = [&](int x, int j) { return tmem + (uint32_t)(256 * x + 64 * (j & 1)); };
  auto tO_of = [&](int x) { return tmem + (uint32_t)(256 * x + 128); };

  if (warp == 0) {
    if (lane == 0 && n_chunks == 0) { l2pf_issue(P.pf); l2pf_issue(P.pf, 1); }
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
      const uint64_t pol = P.n_qtiles > 2 ? policy_evict_normal() : policy_evict_first();
      auto load_k = [&](int j) {
        const int s = j % DST;
        mbar_wait(&kempty[s], ((j / DST) & 1) ^ 1);
        mbar_expect_tx(&kfull[s], k_bytes);
        const int page = P.kv.block_table[(size_t)req * P.kv.pages_per_req + c_first + j];
        const int krow = ((page * 2 + 0) * P.kv.kv_heads + h) * PAGE;
        for (int a = 0; a < natom; ++a)
          tma_load_2d(&tmK, &kfull[s], sK + (size_t)s * k_bytes + a * (DCHUNK * 128), a * 64, krow, pol);
      };
      int kj = 0;
      while (kj < n_chunks && kj < DST && (c_first + kj + 1) * DCHUNK <= safe_hi) load_k(kj++);
      pdl_wait();
      kst_enter(P.kst);
      while (kj < n_chunks) load_k(kj++);
      l2pf_issue(P.pf);
    }
  } else if (warp == 2) {
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const uint64_t pol = P.n_qtiles > 2 ? policy_evict_normal() : policy_evict_first();
      auto load_v = [&](int j) {
        const int s = j % DST;
        mbar_wait(&vempty[s], ((j / DST) & 1) ^ 1);
        mbar_expect_tx(&vfull[s], v_bytes);
        const int page = P.kv.block_table[(size_t)req * P.kv.pages_per_req + c_first + j];
        tma_load_2d(&tmV, &vfull[s], sV + (size_t)s * v_bytes, 0, ((page * 2 + 1) * P.kv.kv_heads + h) * hd, pol);
      };
      int vj = 0;
      while (vj < n_chunks && vj < DST && (c_first + vj + 1) * DCHUNK <= safe_hi) load_v(vj++);
      pdl_wait();
      while (vj < n_chunks) load_v(vj++);
    }
  } else if (warp == 1) {
    if (lane == 0 && n_chunks > 0) {
      mbar_wait(qbar, 0);                       // both q tiles in shared memory
      fence_after();
      const int ntile = hasB ? 2 : 1;
      auto issue_s = [&](int j) {               // S_x(j) = Q_x K_j^T for both tiles
        const int s = j % DST;
        mbar_wait(&kfull[s], (j / DST) & 1);
        fence_after();
        for (int x = 0; x < ntile; ++x) {
          for (int kk = 0; kk < hd / 16; ++kk) {
            const int a = kk >> 2, off = kk & 3;
            const uint64_t ad = desc_sw128(sQ + (size_t)x * q_bytes + a * (QROWS * 128)) + 2 * off;
            const uint64_t bd = desc_sw128(sK + (size_t)s * k_bytes + a * (DCHUNK * 128)) + 2 * off;
            mma_bf16(tS_of(x, j), ad, bd, P.idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&sfull[2 * x + (j & 1)]);
        }
        mma_commit(&kempty[s]);
      };
      issue_s(0);
      for (int j = 0; j < n_chunks; ++j) {
        // S(j+1) into the other score buffer (it held P(j-1), consumed by P(j-1) V,
        // issued earlier: tcgen05.mma executes in issue order)
        if (j + 1 < n_chunks) issue_s(j + 1);
        const int s = j % DST;
        mbar_wait(&vfull[s], (j / DST) & 1);
        fence_after();
        for (int x = 0; x < ntile; ++x) {
          mbar_wait(&pfull[2 * x + (j & 1)], (j >> 1) & 1);
          fence_after();
          for (int kk = 0; kk < DCHUNK / 16; ++kk) {
            const uint64_t vd = desc_sw128(sV + (size_t)s * v_bytes) + 2 * kk;
            mma_bf16_ts(tO_of(x), tS_of(x, j) + (uint32_t)(kk * 8), vd, P.idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&pvdone[x]);
        }
        mma_commit(&vempty[s]);
      }
      mma_commit(odone);
    }
  } else if (in_tile) {
    // ------------------------------------------------------------ softmax group X
    const float scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    float mrow = -INFINITY, lsum = 0.f;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tO = tO_of(X);
    const int hcols = hd / SW;
    const bool live = __any_sync(0xffffffffu, valid);
    {
      // this thread's q row, dims [part hd/SW, (part+1) hd/SW), into the SW128 q tile
      pdl_wait();
      const int d0 = part * hcols;
      const uint4* src = writable ? (const uint4*)(P.q + ((size_t)row * P.Hq + head) * hd + d0) : nullptr;
      uint8_t* qt_base = sQ + (size_t)X * q_bytes;
      for (int c = 0; c < hcols / 8; ++c) {
        const int d = d0 + 8 * c, a = d >> 6, ch = (d & 63) >> 3;
        const uint4 v = src ? src[c] : make_uint4(0u, 0u, 0u, 0u);
        *(uint4*)(qt_base + a * (QROWS * 128) + lane_row * 128 + ((ch ^ (lane_row & 7)) << 4)) = v;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(qbar);
    }
    const int bar_id = 1 + X * 4 + q4;          // the SW warps of this group and lane quarter
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(&sfull[2 * X + (j & 1)], (j >> 1) & 1);
      fence_after();
      const uint32_t tS = tS_of(X, j);
      if (live) {
        const int kb = (c_first + j) * DCHUNK + part * KPW;
        uint32_t r0[32];
        if constexpr (KPW == 32) tmem_ld32_nw(tS + lane_off + (uint32_t)(part * KPW), r0);
        else { uint32_t r16[16]; tmem_ld16_nw(tS + lane_off + (uint32_t)(part * KPW), r16); for (int i = 0; i < 16; ++i) r0[i] = r16[i]; }
        uint32_t vm0 = 0u;
        if (valid) {
          vm0 = range32(klo - kb, khi - kb);
          if (slot >= 0) vm0 |= anc32(anc, kb - tb) & range32(0, m.t_max - (kb - tb));
          vm0 &= range32(k_begin - kb, k_end - kb);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float s[KPW];
#pragma unroll
        for (int i = 0; i < KPW; ++i) s[i] = ((vm0 >> i) & 1u) ? __uint_as_float(r0[i]) : -INFINITY;
        float mxp[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mxp[k] = s[k];
#pragma unroll
        for (int i = 8; i < KPW; ++i) mxp[i & 7] = fmaxf(mxp[i & 7], s[i]);
        float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                         fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        red_max[X][j & 1][part][lane_row] = mx;
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * SW) : "memory");
#pragma unroll
        for (int p2 = 0; p2 < SW; ++p2) mx = fmaxf(mx, red_max[X][j & 1][p2][lane_row]);
        mx *= scale_log2;
        float alpha = 1.f;
        if (mrow == -INFINITY) {
          mrow = mx;
        } else if (mx > mrow + 8.f) {
          alpha = ex2(mrow - mx);
          mrow = mx;
        }
        const float msub = mrow == -INFINITY ? 0.f : mrow;
        uint32_t pw[KPW / 2];
        float ls = 0.f;
#pragma unroll
        for (int i = 0; i < KPW / 2; ++i) {
          const float p0 = ex2(fmaf(s[2 * i], scale_log2, -msub)), p1 = ex2(fmaf(s[2 * i + 1], scale_log2, -msub));
          __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
          const float2 pf = __bfloat1622float2(pr);
          ls += pf.x + pf.y;
          pw[i] = *(uint32_t*)&pr;
        }
        if constexpr (KPW == 32) {
          tmem_st16(tS + lane_off + (uint32_t)(part * 16), pw);
        } else {
          tmem_st8(tS + lane_off + (uint32_t)(part * 8), pw);
        }
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
          // O_X must hold P_X(<j) V exactly once before it is scaled: S_X(j) completing
          // implies P_X(j-2) V done, so pvdone[X] is within one phase of j-1
          if (j > 0) {
            mbar_wait(&pvdone[X], (j - 1) & 1);
            fence_after();
          }
          for (int c = 0; c < hcols; c += 16) {
            uint32_t o[16];
            tmem_ld16(tO + lane_off + (uint32_t)(part * hcols + c), o);
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(tO + lane_off + (uint32_t)(part * hcols + c), o);
          }
        }
        lsum = lsum * alpha + ls;
        tmem_st_wait();
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[2 * X + (j & 1)]);
    }
    // ------------------------------------------------------------ epilogue
    red_l[X][part][lane_row] = lsum;
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * SW) : "memory");
    float ltot = 0.f;
#pragma unroll
    for (int p2 = 0; p2 < SW; ++p2) ltot += red_l[X][p2][lane_row];
    if (!valid) ltot = 0.f;
    if (n_chunks > 0) {
      mbar_wait(odone, 0);
      fence_after();
    }
    const float inv = (P.direct && ltot > 0.f) ? 1.0f / ltot : 1.0f;
    for (int c = 0; c < hcols; c += 16) {
      uint32_t o[16];
      if (n_chunks > 0) tmem_ld16(tO + lane_off + (uint32_t)(part * hcols + c), o);   // (warp-collective)
      else
        for (int i = 0; i < 16; ++i) o[i] = 0u;
      if (writable) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = ltot > 0.f ? __uint_as_float(o[i]) * inv : 0.f;
        const int d = part * hcols + c;
        if (P.direct) {
          uint32_t w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            w[i] = *(const uint32_t*)&b2;
          }
          uint4* dst = (uint4*)(P.out + ((size_t)row * P.Hq + head) * hd + d);
          dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
          dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        } else {
          float4* dst = (float4*)(P.ws + (((size_t)split * P.Hq + head) * P.M + row) * hd + d);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
    }
    if (writable && !P.direct && part == 0) {
      const size_t base_ml = (size_t)nsplit * P.M * P.Hq * hd;
      const size_t idx = ((size_t)split * P.Hq + head) * P.M + row;
      P.ws[base_ml + 2 * idx] = mrow;
      P.ws[base_ml + 2 * idx + 1] = ltot;
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
  {
    static const int order_env = [] { const char* e = getenv("HSD_ATTN_ORDER"); return e ? atoi(e) : 0; }();
    P.light_last = order_env == 1 && P.n_qtiles > 1 && (R * G) % QROWS != 0 && (R * G) % QROWS <= QROWS / 2;
  }
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
  P.idesc_s = idesc_bf16(128, CHUNK);
  P.idesc_o = idesc_bf16(128, hd + VEXTRA);   // O columns [0, hd) + l in column hd
  // splits: enough CTAs for ~2 per SM, each split a whole number of pages
  const int base_ctas = n_req * kv.kv_heads * P.n_qtiles;
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
  // (three quarters of a wave: c2's 9 visible chunks per (kv head, q-tile) split 3 / 3 / 3
  // with S = 3, where S = 4 left one split CTA idle and gave the merge kernel a fourth
  // partial to read -- step 4.78 -> 4.68 ms)
  if (dyn && latency_bound) S = min(S, max(1, (3 * num_sms()) / (4 * base_ctas)));
  P.dyn = dyn == 1 && latency_bound;
  static const int s_override = [] { const char* e = getenv("HSD_ATTN_SPLITS"); return e ? atoi(e) : 0; }();
  if (s_override > 0) S = min(s_override, pages);
  // (experiment: key splits of the one-row draft chain passes only, R = 1)
  static const int s_draft = [] { const char* e = getenv("HSD_ATTN_SPLITS_DRAFT"); return e ? atoi(e) : 0; }();
  if (s_draft > 0 && R == 1) S = min(s_draft, pages);
  // two splits reduce inside a 2-CTA cluster over DSMEM (no workspace, no merge
  // kernel): c5 (b = 2) attention 6.8-7.3 -> 6.5 ms. Wider clusters measured
  // slower (c2, S = 4: step 4.95 -> 5.38 ms) -- a 2-CTA cluster fits one TPC's SM
  // pair, 4+ need GPC-wide co-scheduling against the PDL-overlapped predecessor.
  // HSD_ATTN_CLUSTER_MAX raises the limit (<= 8) for experiments.
  static const int cluster_max = [] {
    const char* e = getenv("HSD_ATTN_CLUSTER_MAX");
    return e ? atoi(e) : 2;
  }();
  P.cluster = (S >= 2 && S <= cluster_max && S <= 8) ? 1 : 0;
  while (!P.cluster && S > 1 && (size_t)S * M * Hq * (hd + 2) > ws_floats) --S;
  int pps = (pages + S - 1) / S;
  P.keys_per_split = pps * CHUNK;
  if (!P.cluster && !P.dyn) S = (pages + pps - 1) / pps;   // cluster / dynamic modes keep S (empty splits contribute 0)
  P.direct = S == 1;
  // tensor maps: K pool rows of hd; V^T pool rows of page_size (q is read by the
  // softmax warps straight into TMEM)
  CUtensorMap mk, mv;
  uint64_t dk[2] = {(uint64_t)hd, (uint64_t)(kv_layer_elems / hd)};
  uint64_t sk[1] = {(uint64_t)hd};
  uint32_t bk[2] = {64, (uint32_t)PAGE};
  uint64_t dv[2] = {(uint64_t)PAGE, (uint64_t)(kv_layer_elems / PAGE)};
  uint64_t sv[1] = {(uint64_t)PAGE};
  uint32_t bv[2] = {(uint32_t)PAGE, (uint32_t)hd};
  if (!tma_map_bf16(&mk, kv.base, 2, dk, sk, bk) || !tma_map_bf16(&mv, kv.base, 2, dv, sv, bv)) return -1;
  // Dual-tile kernel (two q-tiles per CTA, one K / V stream; HSD_ATTN_DUAL=0 disables):
  // when a (request, kv head) has >= 2 q-tiles (c3 / c4 / c5 verify passes)
  static const int dual_env = [] { const char* e = getenv("HSD_ATTN_DUAL"); return e ? atoi(e) : 0; }();
  if (dual_env && P.n_qtiles >= 2 && hd == 128) {
    const int npairs = (P.n_qtiles + 1) / 2;
    const int base2 = n_req * kv.kv_heads * npairs;
    const int dchunks = (max_keys + DCHUNK - 1) / DCHUNK;   // 64-key chunks (pages)
    int S2 = max(1, (2 * num_sms() + base2) / (2 * base2));
    S2 = min(S2, max(1, dchunks / 2));
    if (s_override > 0) S2 = min(s_override, dchunks);
    while (S2 > 1 && (size_t)S2 * M * Hq * (hd + 2) > ws_floats) --S2;
    const bool lb = (dchunks + S2 - 1) / S2 <= 8;
    if (dyn && lb) S2 = min(S2, max(1, num_sms() / base2));
    P.dyn = dyn == 1 && lb;
    const int cps2 = (dchunks + S2 - 1) / S2;
    P.keys_per_split = cps2 * DCHUNK;
    if (!P.dyn) S2 = (dchunks + cps2 - 1) / cps2;
    P.direct = S2 == 1;
    P.cluster = 0;
    P.idesc_s = idesc_bf16(128, DCHUNK);
    P.idesc_o = idesc_bf16(128, hd);
    CUtensorMap mk2, mv2;
    uint64_t dk2[2] = {(uint64_t)hd, (uint64_t)(kv_layer_elems / hd)};
    uint64_t sk2[1] = {(uint64_t)hd};
    uint32_t bk2[2] = {64, (uint32_t)PAGE};
    uint64_t dv2[2] = {(uint64_t)PAGE, (uint64_t)(kv_layer_elems / PAGE)};
    uint64_t sv2[1] = {(uint64_t)PAGE};
    uint32_t bv2[2] = {(uint32_t)PAGE, (uint32_t)hd};
    if (!tma_map_bf16(&mk2, kv.base, 2, dk2, sk2, bk2) || !tma_map_bf16(&mv2, kv.base, 2, dv2, sv2, bv2)) return -1;
    const size_t smem2 = 1024 + 2 * ((size_t)QROWS * hd * 2) + DST * ((size_t)DCHUNK * hd * 2) + DST * ((size_t)hd * 128) +
                         (4 * DST + 16) * 8 + 64;
    static size_t attr2 = 0;
    if (smem2 > attr2) {
      if (cudaFuncSetAttribute(attention_dual_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2) !=
          cudaSuccess) {
        cudaGetLastError();
        return -1;
      }
      attr2 = smem2;
    }
    launch_k(attention_dual_kernel<2>, dim3(S2, kv.kv_heads, n_req * npairs), dim3(dual_threads<2>()), smem2, st, mk2,
             mv2, P);
    if (S2 > 1) {
      launch_k(attention_merge_bf16_kernel, (M * Hq + 7) / 8, 256, 0, st, ws, S2, M, Hq, hd, (bf16*)out, take_l2pf(),
               P.kst);
      return 2;
    }
    return 1;
  }
  const int kst = 4, vst = 2;
  const size_t smem = 1024 + kst * ((size_t)CHUNK * hd * 2) + vst * ((size_t)2 * (hd + VEXTRA) * 128) +
                      (2 * kst + 2 * vst + 8) * 8 + 64;
  // softmax warps per lane quarter: 2 (8 softmax warps, 64 keys each) or 4 (16 warps,
  // 32 keys each: shorter per-thread chains, more warps to hide TMEM/barrier latency).
  // Measured: c3 (768 CTAs, many waves) attention 11.6 -> 11.1
  // ms with 4; c2 (<= 1 wave) 1.05 -> 1.08 ms. So 4 when the grid spans > 2 waves.
  // HSD_ATTN_SW=2|4 forces one.
  static const int sw_env = [] { const char* e = getenv("HSD_ATTN_SW"); return e ? atoi(e) : 0; }();
  const int sw = sw_env == 2 || sw_env == 4 ? sw_env : ((size_t)S * base_ctas > 2 * (size_t)num_sms() ? 4 : 2);
  static size_t attr[4] = {0, 0, 0, 0};   // (the kernel also has ~8-10 KB of static shared memory)
  static const int poly_env = [] { const char* e = getenv("HSD_ATTN_POLY"); return e ? atoi(e) : 0; }();
  auto launch = [&](auto kern, int nthr, size_t& at) {
    if (smem > at) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      at = smem;
    }
    dim3 grid(S, kv.kv_heads, n_req * P.n_qtiles);
    if (P.cluster) launch_k_cluster(kern, grid, dim3(nthr), smem, st, S, mk, mv, P);
    else launch_k(kern, grid, dim3(nthr), smem, st, mk, mv, P);
    return true;
  };
  const bool ok = poly_env == 8
                      ? (sw == 4 ? launch(attention_tc_kernel<4, 8>, nthreads<4>(), attr[3])
                                 : launch(attention_tc_kernel<2, 8>, nthreads<2>(), attr[2]))
                      : (sw == 4 ? launch(attention_tc_kernel<4, 0>, nthreads<4>(), attr[1])
                                 : launch(attention_tc_kernel<2, 0>, nthreads<2>(), attr[0]));
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
