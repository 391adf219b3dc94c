// attention_tc.cu -- tree-masked attention on tcgen05 tensor cores (bf16, hd 64/128,
// page_size 64): the verify / draft attention of PAPER.md:95 (tree-shaped
// attention) over the paged KV cache, flash-decoding style with split-KV.
//
// One CTA = (key split, kv head h, request x q-tile of 128 (row, head) pairs).
//  warp 0      : TMA producer -- the q tile once (3-D map: hd x G heads x rows),
//                then per 64-key page: K [64 keys x hd] and V^T [hd x 64 keys]
//                into a 3-stage shared-memory ring (pages via the block table).
//  warp 1      : MMA issuer -- S_j = Q K_j^T (M=128, N=64, K=hd) into one of two
//                TMEM score buffers, then O += P_j V_j (M=128, N=hd, K=64) into
//                the TMEM output accumulator; S_{j+1} is issued before P_j is
//                ready so softmax of page j overlaps the score MMA of page j+1.
//  warps 2..5  : softmax -- thread t owns TMEM lane t = one (row, head): loads
//                its 64 scores, applies the visibility test (committed range,
//                or tree-ancestor bit, see attention.cu), online max/sum,
//                rescales its O row in TMEM when the max grows, writes P (bf16,
//                128B-swizzled) to shared memory for the PV MMA.
// Splits > 1 write (o, m, l) partials in the SIMT kernel's layout and reuse
// its merge kernel.
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace {
using namespace tc;
constexpr int NTHREADS = 192;
constexpr int PAGE = 64;
constexpr int STAGES = 3;
constexpr int QROWS = 128;

struct AttnParams {
  int M, R, Hq, G, hd, n_qtiles, max_keys, keys_per_split, direct;
  RowMeta m;
  KVLayer kv;
  bf16* out;
  float* ws;
  uint32_t idesc_s, idesc_o;
};

HSD_DEV bool vis(int key, int klo, int khi, int slot, int tb, int t_max, const uint64_t (&a)[4]) {
  if (key >= klo && key < khi) return true;
  if (slot < 0) return false;
  int d = key - tb;
  if (d < 0 || d >= t_max) return false;
  return (a[d >> 6] >> (d & 63)) & 1ull;
}

__global__ void __launch_bounds__(NTHREADS, 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, AttnParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int hd = P.hd, natom = hd / 64;
  const int q_bytes = QROWS * hd * 2;          // natom atoms of [128 rows x 128 B]
  const int k_bytes = PAGE * hd * 2;           // natom atoms of [64 keys x 128 B]
  const int v_bytes = hd * PAGE * 2;           // one atom column of [hd rows x 128 B]
  const int p_bytes = QROWS * PAGE * 2;        // [128 rows x 128 B]
  uint8_t* sQ = base;
  uint8_t* sK = sQ + q_bytes;
  uint8_t* sV = sK + STAGES * k_bytes;
  uint8_t* sP = sV + STAGES * v_bytes;
  uint64_t* bars = (uint64_t*)(sP + 2 * p_bytes);
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = bars + STAGES;       // [STAGES]
  uint64_t* qbar = bars + 2 * STAGES;
  uint64_t* sfull = qbar + 1;            // [2]
  uint64_t* pfull = sfull + 2;           // [2]
  uint64_t* pvdone = pfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(pvdone + 1);
  __shared__ int tile_lo, tile_hi;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, h = blockIdx.y;
  const int grp = blockIdx.z / P.n_qtiles, qt = blockIdx.z % P.n_qtiles;
  const RowMeta& m = P.m;
  const int req = m.req[grp * P.R];
  const int k_begin = split * P.keys_per_split;
  const int k_end = min(P.max_keys, k_begin + P.keys_per_split);

  if (threadIdx.x == 0) { tile_lo = 0x7fffffff; tile_hi = 0; }
  if (threadIdx.x == 32) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(qbar, 1);
    for (int b = 0; b < 2; ++b) { mbar_init(&sfull[b], 1); mbar_init(&pfull[b], 128); }
    mbar_init(pvdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  // softmax threads: this lane's (row, head) and its key bounds
  const int q4 = warp & 3;
  const int lane_row = q4 * 32 + lane;                // tile row-head index owned by this thread
  int row = -1, head = 0, klo = 0, khi = 0, slot = -1, tb = 0;
  uint64_t anc[4] = {0, 0, 0, 0};
  bool valid = false, writable = false;   // writable: an output row of this request
  if (warp >= 2) {
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
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int lo = max(k_begin, tile_lo), hi = min(k_end, tile_hi);
  const int c_first = lo / PAGE;
  const int n_chunks = hi > lo ? (hi + PAGE - 1) / PAGE - c_first : 0;
  const uint32_t tS = tmem;              // 2 x 64 columns
  const uint32_t tO = tmem + 128;        // hd columns

  if (warp == 0) {
    if (lane == 0 && n_chunks > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
      const uint64_t pol = policy_evict_first();
      const uint64_t polq = policy_evict_last();
      const int row0 = grp * P.R + qt * (QROWS / P.G);
      mbar_expect_tx(qbar, q_bytes);
      for (int a = 0; a < natom; ++a)
        tma_load_3d(&tmQ, qbar, sQ + a * (QROWS * 128), a * 64, h * P.G, row0, polq);
      for (int j = 0; j < n_chunks; ++j) {
        const int s = j % STAGES;
        const uint32_t ph = (j / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int page = P.kv.block_table[(size_t)req * P.kv.pages_per_req + c_first + j];
        mbar_expect_tx(&full[s], k_bytes + v_bytes);
        const int krow = ((page * 2 + 0) * P.kv.kv_heads + h) * PAGE;
        for (int a = 0; a < natom; ++a)
          tma_load_2d(&tmK, &full[s], sK + (size_t)s * k_bytes + a * (PAGE * 128), a * 64, krow, pol);
        const int vrow = ((page * 2 + 1) * P.kv.kv_heads + h) * hd;
        tma_load_2d(&tmV, &full[s], sV + (size_t)s * v_bytes, 0, vrow, pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_chunks > 0) {
      mbar_wait(qbar, 0);
      auto issue_s = [&](int j) {
        const int s = j % STAGES;
        mbar_wait(&full[s], (j / STAGES) & 1);
        fence_after();
        const uint32_t d = tS + (uint32_t)((j & 1) * 64);
        for (int kk = 0; kk < hd / 16; ++kk) {
          const int a = kk >> 2, off = kk & 3;
          const uint64_t ad = desc_sw128(sQ + a * (QROWS * 128)) + 2 * off;
          const uint64_t bd = desc_sw128(sK + (size_t)s * k_bytes + a * (PAGE * 128)) + 2 * off;
          mma_bf16(d, ad, bd, P.idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sfull[j & 1]);
      };
      issue_s(0);
      for (int j = 0; j < n_chunks; ++j) {
        if (j + 1 < n_chunks) issue_s(j + 1);
        mbar_wait(&pfull[j & 1], (j >> 1) & 1);
        fence_after();
        const int s = j % STAGES;
        const uint64_t pd0 = desc_sw128(sP + (j & 1) * p_bytes);
        const uint64_t vd0 = desc_sw128(sV + (size_t)s * v_bytes);
        for (int kk = 0; kk < PAGE / 16; ++kk)
          mma_bf16(tO, pd0 + 2 * kk, vd0 + 2 * kk, P.idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
        mma_commit(pvdone);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const float scale = 1.0f / sqrtf((float)hd);
    float mrow = -INFINITY, lrow = 0.f;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    uint8_t* prow_base = sP + lane_row * 128;
    for (int j = 0; j < n_chunks; ++j) {
      mbar_wait(&sfull[j & 1], (j >> 1) & 1);
      fence_after();
      const int key0 = (c_first + j) * PAGE;
      float s[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[16];
        tmem_ld16(tS + lane_off + (uint32_t)((j & 1) * 64 + c * 16), r);
#pragma unroll
        for (int i = 0; i < 16; ++i) s[c * 16 + i] = __uint_as_float(r[i]);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const int key = key0 + i;
        const bool ok = valid && key >= k_begin && key < k_end && vis(key, klo, khi, slot, tb, m.t_max, anc);
        s[i] = ok ? s[i] * scale : -INFINITY;
        mx = fmaxf(mx, s[i]);
      }
      const float mnew = fmaxf(mrow, mx);
      const float alpha = (mrow == -INFINITY) ? (mnew == -INFINITY ? 1.f : 0.f) : expf(mrow - mnew);
      if (j > 0) {
        mbar_wait(pvdone, (j - 1) & 1);   // O (and the P buffer being reused) are free
        fence_after();
        const bool need = alpha != 1.f;
        if (__any_sync(0xffffffffu, need)) {
          for (int c = 0; c < hd; c += 16) {
            uint32_t r[16];
            tmem_ld16(tO + lane_off + (uint32_t)c, r);
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st16(tO + lane_off + (uint32_t)c, r);
          }
          tmem_st_wait();
        }
      }
      float psum = 0.f;
      uint8_t* prow = prow_base + (j & 1) * p_bytes;
#pragma unroll
      for (int c16 = 0; c16 < 8; ++c16) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = s[c16 * 8 + 2 * e] == -INFINITY ? 0.f : expf(s[c16 * 8 + 2 * e] - mnew);
          const float p1 = s[c16 * 8 + 2 * e + 1] == -INFINITY ? 0.f : expf(s[c16 * 8 + 2 * e + 1] - mnew);
          __nv_bfloat162 pr = __floats2bfloat162_rn(p0, p1);
          psum += __low2float(pr) + __high2float(pr);     // l sums exactly what the MMA sees
          w[e] = *(uint32_t*)&pr;
        }
        *(uint4*)(prow + ((c16 ^ (lane_row & 7)) * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      lrow = lrow * alpha + psum;
      mrow = mnew;
      fence_proxy_async();
      fence_before();
      mbar_arrive(&pfull[j & 1]);
    }
    // ------------------------------------------------------------ epilogue
    if (n_chunks > 0) {
      mbar_wait(pvdone, (n_chunks - 1) & 1);
      fence_after();
    }
    for (int c = 0; c < hd; c += 16) {
      uint32_t r[16];
      if (n_chunks > 0) tmem_ld16(tO + lane_off + (uint32_t)c, r);
      else
        for (int i = 0; i < 16; ++i) r[i] = 0u;
      if (writable) {
        if (P.direct) {
          const float inv = lrow > 0.f ? 1.0f / lrow : 0.f;
          bf16* o = P.out + ((size_t)row * P.Hq + head) * hd + c;
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(r[i]) * inv, __uint_as_float(r[i + 1]) * inv);
            *(__nv_bfloat162*)(o + i) = v;
          }
        } else {
          float* o = P.ws + (((size_t)split * P.M + row) * P.Hq + head) * hd + c;
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = lrow > 0.f ? __uint_as_float(r[i]) : 0.f;
        }
      }
    }
    if (!P.direct && writable) {
      const size_t base_ml = (size_t)gridDim.x * P.M * P.Hq * hd;
      const size_t idx = ((size_t)split * P.M + row) * P.Hq + head;
      P.ws[base_ml + 2 * idx] = mrow;
      P.ws[base_ml + 2 * idx + 1] = lrow;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

__global__ void attention_merge_bf16_kernel(const float* __restrict__ ws, int S, int M, int Hq, int hd,
                                            bf16* __restrict__ out) {
  int row = blockIdx.x, head = blockIdx.y;
  size_t base = (size_t)S * M * Hq * hd;
  float Mx = -INFINITY;
  for (int s = 0; s < S; ++s) {
    size_t idx = ((size_t)s * M + row) * Hq + head;
    if (ws[base + 2 * idx + 1] > 0.f) Mx = fmaxf(Mx, ws[base + 2 * idx]);
  }
  for (int d = threadIdx.x; d < hd; d += blockDim.x) {
    float num = 0.f, den = 0.f;
    for (int s = 0; s < S; ++s) {
      size_t idx = ((size_t)s * M + row) * Hq + head;
      float l = ws[base + 2 * idx + 1];
      if (l <= 0.f) continue;
      float w = expf(ws[base + 2 * idx] - Mx);
      num = fmaf(w, ws[idx * hd + d], num);
      den = fmaf(w, l, den);
    }
    out[((size_t)row * Hq + head) * hd + d] = __float2bfloat16_rn(den > 0.f ? num / den : 0.f);
  }
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
  P.M = M; P.R = R; P.Hq = Hq; P.G = G; P.hd = hd; P.m = m; P.kv = kv;
  P.out = (bf16*)out; P.ws = ws; P.max_keys = max_keys;
  P.n_qtiles = (R * G + QROWS - 1) / QROWS;
  P.idesc_s = idesc_bf16(128, PAGE);
  P.idesc_o = idesc_bf16(128, hd);
  // splits: enough CTAs for ~2 per SM, each split a whole number of pages
  const int base_ctas = n_req * kv.kv_heads * P.n_qtiles;
  const int pages = (max_keys + PAGE - 1) / PAGE;
  int S = (2 * num_sms() + base_ctas - 1) / base_ctas;
  if (S > pages) S = pages;
  if (S > 32) S = 32;
  if (S < 1) S = 1;
  while (S > 1 && (size_t)S * M * Hq * (hd + 2) > ws_floats) --S;
  int pps = (pages + S - 1) / S;
  P.keys_per_split = pps * PAGE;
  S = (pages + pps - 1) / pps;
  P.direct = S == 1;
  // tensor maps: q [M][Hq][hd] viewed (hd, heads, rows) with the head offset in
  // the coordinate; K pool rows of hd; V^T pool rows of page_size.
  CUtensorMap mq, mk, mv;
  uint64_t dq[3] = {(uint64_t)hd, (uint64_t)Hq, (uint64_t)M};
  uint64_t sq[2] = {(uint64_t)hd, (uint64_t)Hq * hd};
  uint32_t bq[3] = {64, (uint32_t)G, (uint32_t)(QROWS / G)};
  uint64_t dk[2] = {(uint64_t)hd, (uint64_t)(kv_layer_elems / hd)};
  uint64_t sk[1] = {(uint64_t)hd};
  uint32_t bk[2] = {64, (uint32_t)PAGE};
  uint64_t dv[2] = {(uint64_t)PAGE, (uint64_t)(kv_layer_elems / PAGE)};
  uint64_t sv[1] = {(uint64_t)PAGE};
  uint32_t bv[2] = {(uint32_t)PAGE, (uint32_t)hd};
  if (!tma_map_bf16(&mq, q, 3, dq, sq, bq) || !tma_map_bf16(&mk, kv.base, 2, dk, sk, bk) ||
      !tma_map_bf16(&mv, kv.base, 2, dv, sv, bv))
    return -1;
  const size_t smem = 1024 + (size_t)QROWS * hd * 2 + STAGES * ((size_t)PAGE * hd * 2 * 2) + 2 * (size_t)QROWS * PAGE * 2 +
                      (2 * STAGES + 7) * 8 + 64;
  static size_t attr = 0;   // (the kernel also has ~1 KB of static shared memory)
  if (smem > attr) {
    if (cudaFuncSetAttribute(attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    attr = smem;
  }
  dim3 grid(S, kv.kv_heads, n_req * P.n_qtiles);
  attention_tc_kernel<<<grid, NTHREADS, smem, st>>>(mq, mk, mv, P);
  int launched = 1;
  if (S > 1) {
    attention_merge_bf16_kernel<<<dim3(M, Hq), 128, 0, st>>>(ws, S, M, Hq, hd, (bf16*)out);
    launched++;
  }
  return launched;
}
