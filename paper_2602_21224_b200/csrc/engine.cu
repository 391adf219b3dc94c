// engine.cu -- hsd_ctx and the C ABI of include/hsd.h.
//
// Orchestrates one step of the draft-tree verify-and-reuse loop
// as a fixed sequence of kernel launches on the context stream, sized for the
// padded maxima (b x T_max verify slots, b x (N+1) draft rows) with every
// data-dependent count kept on the device, so a whole step is capturable in one
// CUDA graph and replayed with no host synchronisation.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <string>
#include <vector>
#include <algorithm>
#include <nvtx3/nvToolsExt.h>

#include "../../include/hsd.h"
#include "kernels.cuh"
#include "tree.cuh"
#include "accept.cuh"
#include "gemm_tc.cuh"

// NVTX stage ranges (host side; visible to nsys / ncu --nvtx around eager and staged
// calls and around graph capture -- a replayed graph carries no host ranges)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

int64_t g_hsd_launches = 0;
// Timing ablation (debug only, results become meaningless): HSD_ABLATE is a list
// of kernel classes to SKIP, e.g. "attn,rms,rope,swiglu,gemm,tree,draft".
static const char* g_ablate = getenv("HSD_ABLATE");
static bool ablate(const char* what) { return g_ablate && strstr(g_ablate, what) != nullptr; }
static bool g_attn_tc = [] {
  const char* e = getenv("HSD_ATTN_TC");
  return e == nullptr || atoi(e) != 0;
}();
bool g_hsd_pdl = [] {
  const char* e = getenv("HSD_PDL");
  return e == nullptr || atoi(e) != 0;
}();

namespace {
// prompt rows per prefill forward (HSD_PREFILL_CHUNK, default 4096 = a whole c3
// prompt): at 1024 rows the pair GEMMs' tile count falls under the data-parallel
// wave rule at c3 widths (QKV: 96 pair tiles = 1.3 waves) and runs stream-K
static int prefill_chunk() {
  static const int v = [] { const char* e = getenv("HSD_PREFILL_CHUNK"); return e ? std::max(256, atoi(e)) : 4096; }();
  return v;
}
constexpr int MAXN_TREE = 256;

// ------------------------------------------------------------------ row metadata kernels
struct MetaBuf {
  int32_t *tok, *pos, *kvpos, *req, *klo, *khi, *slot;
  RowMeta view(const int32_t* tbase, const uint64_t* anc, int t_max, int anc_words) const {
    RowMeta m;
    m.tok = tok; m.pos = pos; m.kvpos = kvpos; m.req = req; m.klo = klo; m.khi = khi; m.slot = slot;
    m.tbase = tbase; m.anc = anc; m.t_max = t_max; m.anc_words = anc_words;
    return m;
  }
};

// verify rows r*T + s: slot s of request r's tree at position p + depth, K/V
// stored at p + s; sees the committed cache [0, p) plus its tree ancestors.
__global__ void meta_verify_kernel(MetaBuf mb, int T, const int32_t* t_n, const int32_t* t_tok,
                                   const int32_t* t_depth, const int32_t* p) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x, s = threadIdx.x;
  if (s >= T) return;
  int row = r * T + s;
  bool act = s < t_n[r];
  mb.tok[row] = act ? t_tok[row] : 0;
  mb.pos[row] = act ? p[r] + t_depth[row] : -1;
  mb.kvpos[row] = p[r] + s;
  mb.req[row] = r;
  mb.klo[row] = 0;
  mb.khi[row] = p[r];
  mb.slot[row] = act ? s : -1;
}

// draft prefill rows r*(N+1) + j: pending pair j at position p - n_pend + 1 + j,
// causal over the draft KV positions [1, pos] (reading R1/R2).
__global__ void meta_dprefill_kernel(MetaBuf mb, int R, const int32_t* n_pend, const int32_t* pend_tok,
                                     const int32_t* p, int no_first) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x, j = threadIdx.x;
  if (j >= R) return;
  int row = r * R + j;
  int np = n_pend[r];
  bool act = j < np;
  int pos = p[r] - np + 1 + j;
  mb.tok[row] = act ? pend_tok[row] : 0;
  mb.pos[row] = act ? pos : -1;
  mb.kvpos[row] = act ? pos : 0;
  mb.req[row] = r;
  mb.klo[row] = 1;
  mb.khi[row] = act ? pos + 1 : 0;
  // -2 marks the root pair (the ground-truth token just committed) for the
  // "w/o first token" ablation (R26): draft_concat drops its embedding
  mb.slot[row] = (no_first && act && j == np - 1) ? -2 : -1;
}

// chain step i: row r at position p + i, causal over draft KV [1, p + i]

// row metadata of chain step i for request r (position p + i, keys [1, p + i]): written
// by the kernel that ends the previous chain step (no separate metadata launch)
HSD_DEV void chain_meta(const MetaBuf& mb, int r, int i, const int32_t* p) {
  const int pos = p[r] + i;
  mb.tok[r] = 0; mb.pos[r] = pos; mb.kvpos[r] = pos; mb.req[r] = r;
  mb.klo[r] = 1; mb.khi[r] = pos + 1; mb.slot[r] = -1;
}

// h_1 = draft output at the last pending row -> xw[r] and chain[r][0]; meta of chain step 1
__global__ void gather_last_kernel(const float* x, int R, const int32_t* n_pend, int n, float* xw, float* chain,
                                   int N, MetaBuf mc, const int32_t* p) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x;
  if (threadIdx.x == 0 && N > 1) chain_meta(mc, r, 1, p);
  const float* src = x + ((size_t)r * R + n_pend[r] - 1) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    xw[(size_t)r * n + i] = src[i];
    chain[((size_t)r * N) * n + i] = src[i];
  }
}

// chain row i -> chain[r][i]; meta of chain step i + 1
__global__ void copy_chain_kernel(const float* xw, int n, float* chain, int N, int i, MetaBuf mc, const int32_t* p) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x;
  if (threadIdx.x == 0 && i + 1 < N) chain_meta(mc, r, i + 1, p);
  for (int c = threadIdx.x; c < n; c += blockDim.x) chain[((size_t)r * N + i) * n + c] = xw[(size_t)r * n + c];
}

// first token after prefill: argmax (greedy) or Gumbel sample with step 0, slot 0 (R22);
// then the pending draft pair (H_{P0-1}, t_{P0}) and the request state.
__global__ void first_token_kernel(const float* logits, int V, int mode, float invT, uint32_t seed, int req_g,
                                   int r, const float* Hlast, int n, int P0, int N, float* pend_H,
                                   int32_t* pend_tok, int32_t* n_pend, int32_t* root_tok, int32_t* p,
                                   int32_t* d_first) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int b4 = threadIdx.x; b4 * 4 < V; b4 += blockDim.x) {
    u32x4 c = {(uint32_t)b4, 0u, 0u, (uint32_t)req_g};
    u32x4 rr = philox4x32_10(c, seed, TAG_GUMBEL);
    for (int q = 0; q < 4; ++q) {
      int v = b4 * 4 + q;
      if (v >= V) break;
      float z = mode == 0 ? logits[v] : logits[v] * invT - logf(-logf(unit_open(lane_of(rr, q))));
      if (better(z, v, bv, bi)) { bv = z; bi = v; }
    }
  }
  warp_argmax(bv, bi);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
    warp_argmax(bv, bi);
    if (lane == 0) si[0] = bi;
  }
  __syncthreads();
  int t = si[0];
  for (int i = threadIdx.x; i < n; i += blockDim.x) pend_H[((size_t)r * (N + 1)) * n + i] = Hlast[i];
  if (threadIdx.x == 0) {
    pend_tok[r * (N + 1)] = t;
    for (int j = 1; j <= N; ++j) pend_tok[r * (N + 1) + j] = -1;
    n_pend[r] = 1;
    root_tok[r] = t;
    p[r] = P0;
    if (d_first) d_first[r] = t;
  }
}

__global__ void gather_same_kernel_f32(const float* src, const int32_t* idx, int n, float* dst) {
  int r = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[(size_t)r * n + i] = src[(size_t)idx[r] * n + i];
}
__global__ void gather_same_kernel_bf16(const bf16* src, const int32_t* idx, int n, bf16* dst) {
  int r = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[(size_t)r * n + i] = src[(size_t)idx[r] * n + i];
}
__global__ void f32_to_dt_kernel(const float* src, size_t count, bf16* dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}
}  // namespace

// ====================================================================== context
struct LayerW { void *wqkv, *wo, *wgu, *wd; };

// L2 weight prefetch (common.cuh L2Pf; cap swept on c2: 0 / 32 / 48 / 64 / 96 / 128 / 160 MB ->
// 4.89 / 4.77 / 4.76 / 4.74 / 4.73 / 4.76 / 4.86 ms): kernels that leave HBM idle carry a byte
// range of the weights the NEXT GEMM(s) will stream. HSD_L2PF_MB (default 96, 0 =
// off) caps the range handed to a long idle window (qkv_rope + attention, SwiGLU,
// K-TREE); short windows (an RMSNorm right before its GEMM) get a third of it.
L2Pf g_l2pf = {nullptr, 0ull, 0};
KStamp g_kstamp = {nullptr, 0, nullptr};
// HSD_L2PF_WHERE: bitmask of the windows that prefetch (default 4 = attention only:
// the others measured flat or slower on c2; 1 rmsnorm-1, 2 qkv_rope,
// 4 attention, 8 rmsnorm-2, 16 SwiGLU, 32 K-TREE); HSD_L2PF_LATE=1 issues after the PDL wait
static const int g_l2pf_where = [] { const char* e = getenv("HSD_L2PF_WHERE"); return e ? atoi(e) : 4; }();
static const int g_l2pf_late = [] { const char* e = getenv("HSD_L2PF_LATE"); return e ? atoi(e) : 0; }();
static const size_t g_l2pf_cap = [] {
  const char* e = getenv("HSD_L2PF_MB");
  return (size_t)(e ? atof(e) : 96.0) * (size_t)(1 << 20);
}();
struct PfScope {   // the next launch inside this scope carries [p + off, p + off + min(bytes, cap))
  PfScope(const void* p, size_t total, size_t off, size_t cap, int where) {
    if (g_l2pf_cap == 0 || p == nullptr || off >= total || !(g_l2pf_where & where)) return;
    g_l2pf = L2Pf{(const char*)p + off, (unsigned long long)(std::min(total - off, cap) & ~(size_t)15), g_l2pf_late};
  }
  ~PfScope() { g_l2pf = L2Pf{nullptr, 0ull, 0}; }
};

// Kernel categories for hsd_profile (CUDA events around each launch; eager only).
enum ProfCat { P_GEMM_VERIFY, P_GEMM_DRAFT, P_HEAD_VERIFY, P_HEAD_DRAFT, P_ATTN_VERIFY, P_ATTN_DRAFT, P_TREE,
               P_RESAMPLE, P_WALK, P_COMPACT, P_ROWWISE, P_NCAT };
static const char* kProfNames[P_NCAT] = {"gemm_verify", "gemm_draft", "head_verify", "head_draft",
                                         "attn_verify", "attn_draft", "tree", "resample", "walk", "compact",
                                         "rowwise"};
struct ProfRec { int cat; cudaEvent_t a, b; double bytes, flops; };

struct hsd_ctx {
  hsd_config cfg;
  int pchunk = 1024;                // prompt rows per prefill forward (prefill_chunk())
  int dev = 0;
  cudaStream_t st = nullptr;
  DType dt = DT_F32;
  size_t esz = 4;
  int n, L, Hq, Hkv, hd, f, V, qd, kd, qkvd;
  int N, k, B, Br, r, Vh, d;
  int T, W;          // verify slots, anc words
  int maxb, b = 0;   // capacity, active requests
  bool use_tc = false;
  // weights
  void *embed = nullptr, *head = nullptr, *head_rank = nullptr, *fc = nullptr, *gu_tmp = nullptr;
  std::vector<LayerW> layers;
  LayerW draft{};
  void* table = nullptr;
  float* table_scale = nullptr;   // HSD_FLAG_TABLE_FP8: per-row e4m3 scale [Vh] (R25)
  int32_t *perm_d = nullptr, *rank_d = nullptr;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  int max_pos = 0;
  // KV
  void *kv_t = nullptr, *kv_d = nullptr;
  size_t kv_layer_elems = 0;
  int pages_per_req = 0, page_size = 64;
  int32_t* block_table = nullptr;
  // state
  int32_t *p, *root_tok, *n_pend, *pend_tok, *step;
  int32_t* req_id = nullptr;       // [maxb] global request id per slot (random streams)
  std::vector<int32_t> req_id_h;   // host copy
  // host-side bound on every slot's committed length p: p grows by at most N + 1
  // per step, and a step writes target / draft KV up to p + T - 1, so a step is
  // refused (HSD_ESTATE) once p_hi + T would pass the KV capacity max_pos
  std::vector<int64_t> p_hi;
  float* pend_H;
  int* err;
  int32_t *pt_n, *pt_tok, *pt_par, *pt_depth;
  float* pt_lj;
  int32_t *t_n, *t_tok, *t_par, *t_depth;
  float* t_lj;
  uint64_t* t_anc;
  int32_t *acc_n, *acc_slots, *bonus, *emitted, *n_emitted;
  int32_t* plant = nullptr;
  int plant_stride = 0;
  // workspace
  int Mcap;
  float *x_d, *xw, *Hver, *chain, *big, *draft_logits, *logits, *x_p, *H_prompt, *attn_ws;
  float* big_dp = nullptr;   // QKV output of a data-parallel (storing) GEMM: no re-zeroing needed
  size_t attn_ws_floats;
  void *a, *qb, *ob, *h;   // h: SwiGLU output [Mcap, f] (never aliases the GEMM input a)
  int32_t* argmax;
  MetaBuf mv, md, mc, mp;
  // vocab-sharded lm_head (shard.cu): G column shards, this one = srank
  int shard_mode = HSD_SHARD_NONE, G = 1, srank = 0, shard_rows = 0, shard_wmax = 0;
  int shard_lo[HSD_MAX_SHARDS + 1] = {};
  void* comm = nullptr;
  void* a_all = nullptr;         // [G * rows, n] all-gathered normalised rows (NCCL)
  float* lslice = nullptr;       // [G * rows, w] this shard's logits columns
  float* lrecv = nullptr;        // [G][rows][wmax] draft-logit column slices (all-to-all target)
  float *pv_loc = nullptr, *pv_all = nullptr;     // partial argmax values [G*rows], [G][G*rows]
  // stochastic acceptance over the sharded head (shard.cu): per-row records of this
  // shard's columns [rows_g][rec] and of every shard [G][rows_g][rec]; their merge
  // for this rank's verify rows (lse, tree-token logits, Gumbel top-KG); the tree
  // tokens and request ids of every rank's rows (NCCL: all-gathered each step)
  float *sp_loc = nullptr, *sp_all = nullptr, *sh_lse = nullptr, *sh_tl = nullptr, *sh_gv = nullptr;
  int32_t *sh_gi = nullptr, *tt_all = nullptr, *rid_all = nullptr;
  int32_t *pi_loc = nullptr, *pi_all = nullptr;   // partial argmax token ids
  std::string nccl_err;          // first collective failure (surfaced as HSD_ENCCL)
  // hsd_kstamp: per-launch %globaltimer stamps of the verify GEMMs inside graph replays
  unsigned long long* kst_buf = nullptr;
  bool kst_on = false;
  int kst_n = 0;
  std::vector<double> kst_bytes, kst_flops;
  std::vector<int> kst_cat;
  // host staging for e2e
  int32_t *h_pinned = nullptr;
  // graph
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
  // staged calls (build / verify / accept) replay their own per-stage graphs
  cudaGraphExec_t sgraph[3] = {nullptr, nullptr, nullptr};
  int64_t sgraph_kernels[3] = {0, 0, 0}, sgraph_replays[3] = {0, 0, 0};
  int stage = 0;       // 0 idle, 1 tree built, 2 verified
  int64_t launches0 = 0, graph_replays = 0;
  std::vector<void*> allocs;
  std::string errmsg;
  // profiling
  bool prof_on = false, capturing = false;
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[P_NCAT] = {}, prof_bytes[P_NCAT] = {}, prof_flops[P_NCAT] = {};
  int64_t prof_n[P_NCAT] = {};
  int pass_verify = 0;   // 1 while running the verify pass (GEMM category)
  double attn_bytes = 0; // algorithmic bytes of the next attention launch (profile mode)
};

// Profile mode only (eager, synchronising): per-request positions and tree
// sizes on the host, to state attention's algorithmic bytes per launch:
// every visible K/V row once + the q rows read + the output rows written.
static double attn_bytes_for(hsd_ctx* c, int pass, int chain_i) {
  if (!c->prof_on || c->capturing) return 0;
  std::vector<int32_t> p(c->b), tn(c->b), np(c->b);
  cudaStreamSynchronize(c->st);
  cudaMemcpy(p.data(), c->p, 4 * c->b, cudaMemcpyDeviceToHost);
  cudaMemcpy(tn.data(), c->t_n, 4 * c->b, cudaMemcpyDeviceToHost);
  cudaMemcpy(np.data(), c->n_pend, 4 * c->b, cudaMemcpyDeviceToHost);
  double keys = 0, rows = 0;
  for (int r = 0; r < c->b; ++r) {
    if (pass == 0) { keys += p[r] + tn[r]; rows += tn[r]; }          // verify
    else if (pass == 1) { keys += p[r]; rows += np[r]; }             // draft prefill (positions 1..p)
    else { keys += p[r] + chain_i; rows += 1; }                       // chain step i
  }
  return keys * 2.0 * c->kd * c->esz + rows * 2.0 * c->qd * c->esz;
}

static cudaEvent_t prof_event(hsd_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Prof {
  hsd_ctx* c;
  ProfRec r;
  bool on;
  Prof(hsd_ctx* ctx, int cat, double bytes = 0, double flops = 0) : c(ctx) {
    on = c->prof_on && !c->capturing;
    if (!on) return;
    r.cat = cat; r.bytes = bytes; r.flops = flops;
    r.a = prof_event(c); r.b = prof_event(c);
    cudaEventRecord(r.a, c->st);
  }
  ~Prof() {
    if (!on) return;
    cudaEventRecord(r.b, c->st);
    c->prof_pending.push_back(r);
  }
};

static void prof_collect(hsd_ctx* c) {
  if (c->prof_pending.empty()) return;
  cudaStreamSynchronize(c->st);
  for (auto& r : c->prof_pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->prof_ms[r.cat] += ms;
    c->prof_bytes[r.cat] += r.bytes;
    c->prof_flops[r.cat] += r.flops;
    c->prof_n[r.cat] += 1;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->prof_pending.clear();
}

static hsd_status fail(hsd_ctx* c, hsd_status s, const std::string& m) {
  if (c) c->errmsg = m;
  return s;
}

#define CU(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      return fail(ctx, HSD_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    }                                                                           \
  } while (0)

static void* dalloc(hsd_ctx* c, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  cudaMemsetAsync(p, 0, bytes, c->st);
  c->allocs.push_back(p);
  return p;
}

// hsd_kstamp: while a stamped graph is captured, the next verify GEMM launch gets
// stamp slot id kst_n (its algorithmic bytes / flops recorded for hsd_kstamp_read)
static void kstamp_next(hsd_ctx* c, int cat, double bytes, double flops) {
  if (!c->kst_on || !c->capturing || (cat != P_GEMM_VERIFY && cat != P_ATTN_VERIFY) || c->kst_n >= KST_MAXID)
    return;
  g_kstamp = KStamp{c->kst_buf, c->kst_n++, c->step};
  c->kst_bytes.push_back(bytes);
  c->kst_flops.push_back(flops);
  c->kst_cat.push_back(cat);
}

// GEMM dispatch: C[M,N] (+)= A[M,K] W[N,K]^T. Algorithmic bytes: W once, A once,
// C written once (read too when accumulating).
static void gemm(hsd_ctx* c, const void* A, int lda, const void* Wt, int ldw, float* C, int ldc, int M, int N,
                 int K, bool acc, int cat = -1, bool c_zeroed = false) {
  if (ablate("gemm")) return;
  if (cat < 0) cat = c->pass_verify ? P_GEMM_VERIFY : P_GEMM_DRAFT;
  Prof pf(c, cat, (double)N * K * c->esz + (double)M * K * c->esz + (double)M * N * 4 * (acc ? 2 : 1),
          2.0 * M * N * K);
  // TMA needs 16-byte aligned operand bases; gemm_tc_bf16 returns 0 (nothing launched)
  // when it cannot encode a tensor map -- both fall back to the SIMT kernel
  const bool aligned = (((uintptr_t)A | (uintptr_t)Wt) & 15) == 0;
  int launched = 0;
  if (c->use_tc && c->dt == DT_BF16 && aligned && gemm_tc_supported(M, N, K, lda, ldw)) {
    kstamp_next(c, cat, (double)N * K * c->esz + (double)M * K * c->esz + (double)M * N * 4 * (acc ? 2 : 1),
                2.0 * M * N * K);
    launched = gemm_tc_bf16((const bf16*)A, lda, (const bf16*)Wt, ldw, C, ldc, M, N, K, acc, c->st, c_zeroed);
    g_hsd_launches += launched;
  }
  if (launched == 0) {
    gemm_simt(A, lda, Wt, ldw, c->dt, C, ldc, M, N, K, acc, c->st);
    g_hsd_launches += 1;
  }
}

static KVLayer kv_layer(hsd_ctx* c, void* pool, int layer) {
  KVLayer kv;
  kv.base = (char*)pool + (size_t)layer * c->kv_layer_elems * c->esz;
  kv.block_table = c->block_table;
  kv.pages_per_req = c->pages_per_req;
  kv.page_size = c->page_size;
  kv.kv_heads = c->Hkv;
  kv.head_dim = c->hd;
  return kv;
}

// One Llama decoder layer over M padded rows (R rows per request, n_req requests),
// residual stream x (fp32) updated in place.
static void layer_forward(hsd_ctx* c, const LayerW& w, float* x, int M, int R, int n_req, const RowMeta& m,
                          const KVLayer& kv, int max_keys) {
  const int n = c->n;
  const size_t es = c->esz, b_qkv = (size_t)c->qkvd * n * es, b_o = (size_t)n * c->qd * es,
               b_gu = (size_t)2 * c->f * n * es, b_d = (size_t)n * c->f * es, cap = g_l2pf_cap;
  if (!ablate("rms")) {
    Prof pf(c, P_ROWWISE);
    PfScope l2(w.wqkv, b_qkv, 0, cap / 3, 1);
    launch_rmsnorm(x, M, n, c->cfg.rms_eps, c->a, c->dt, m.pos, c->st);
  }
  // c->big is kept zero outside a GEMM -> consumer window (qkv_rope_kv and
  // swiglu re-zero what they read), so these GEMMs accumulate without a memset
  // a data-parallel QKV GEMM STORES its output (into big_dp), so qkv_rope need not
  // re-zero it; the stream-K one accumulates into the zero-kept scratch big
  const bool qkv_dp = c->use_tc && c->dt == DT_BF16 && gemm_tc_supported(M, c->qkvd, n, n, n) &&
                      gemm_tc_dp(M, c->qkvd, n, false);
  bool qkv_fused = false;
  if (qkv_dp && !ablate("gemm") && !ablate("rope") && c->kv_layer_elems < (size_t)INT32_MAX && gemm_tc_qkv_ok(M, c->qkvd, n, c->hd, c->Hq, c->Hkv)) {
    // CTA-pair QKV GEMM whose epilogue applies RoPE and writes bf16 q and the
    // paged K / V rows itself (no fp32 QKV row, no qkv_rope_kv launch)
    const int cat = c->pass_verify ? P_GEMM_VERIFY : P_GEMM_DRAFT;
    const double by = (double)c->qkvd * n * c->esz + (double)M * n * c->esz + (double)M * c->qkvd * 2,
                 fl = 2.0 * M * c->qkvd * n;
    Prof pf(c, cat, by, fl);
    kstamp_next(c, cat, by, fl);
    QkvEpi e;
    e.pos = m.pos; e.kvpos = m.kvpos; e.req = m.req; e.rc = c->rope_cos; e.rs = c->rope_sin;
    e.q_out = (bf16*)c->qb; e.kv_base = kv.base; e.block_table = kv.block_table;
    e.pages_per_req = kv.pages_per_req; e.page_size = kv.page_size; e.Hq = c->Hq; e.Hkv = c->Hkv; e.hd = c->hd;
    const int k = gemm_tc_qkv_bf16((const bf16*)c->a, n, (const bf16*)w.wqkv, n, M, c->qkvd, n, e, c->st);
    g_hsd_launches += k;
    qkv_fused = k > 0;
  }
  if (!qkv_fused) {
    float* qkv = qkv_dp ? c->big_dp : c->big;
    gemm(c, c->a, n, w.wqkv, n, qkv, c->qkvd, M, c->qkvd, n, false, -1, true);
    if (!ablate("rope")) { Prof pf(c, P_ROWWISE);
      PfScope l2(w.wo, b_o, 0, std::max(cap, b_o), 2);
      launch_qkv_rope_kv(qkv, M, m, c->rope_cos, c->rope_sin, c->Hq, kv, c->qb, c->dt, c->st, !qkv_dp); }
  } else {
    g_hsd_launches -= 1;   // (the rope_kv launch counted below did not happen)
  }
  if (!ablate("attn")) {
    // algorithmic attention bytes: the request's committed K/V rows once (per
    // kv head) + q/out rows; exact per-row key counts are device-side, so the
    // host uses the capacity-free estimate recorded by hsd_profile_read callers.
    Prof pf(c, c->pass_verify ? P_ATTN_VERIFY : P_ATTN_DRAFT, c->attn_bytes);
    int tc_launched = -1;
    PfScope l2(w.wgu, b_gu, 0, cap, 4);
    if (c->use_tc && g_attn_tc && attention_tc_supported(c->hd, c->page_size, c->dt)) {
      kstamp_next(c, c->pass_verify ? P_ATTN_VERIFY : P_ATTN_DRAFT, 0.0, 0.0);
      tc_launched = launch_attention_tc(c->qb, M, R, n_req, m, kv, c->Hq, max_keys, c->ob, c->attn_ws,
                                        c->attn_ws_floats, c->kv_layer_elems, c->st);
      g_kstamp = KStamp{nullptr, 0, nullptr};   // (unconsumed if the tc kernel declined)
    }
    if (tc_launched > 1) g_hsd_launches += tc_launched - 1;   // the split merge
    if (tc_launched < 0)
      launch_attention(c->qb, M, R, n_req, m, kv, c->Hq, c->dt, max_keys, c->ob, c->attn_ws, c->attn_ws_floats,
                       c->st);
  }
  gemm(c, c->ob, c->qd, w.wo, c->qd, x, n, M, n, c->qd, true);
  if (!ablate("rms")) {
    Prof pf(c, P_ROWWISE);
    PfScope l2(w.wgu, b_gu, cap, cap / 3, 8);
    launch_rmsnorm(x, M, n, c->cfg.rms_eps, c->a, c->dt, m.pos, c->st);
  }
  bool fused = false;
  if (c->use_tc && c->dt == DT_BF16 && gemm_tc_supported(M, 2 * c->f, n, n, n) && gemm_tc_swiglu_ok(M, 2 * c->f, n)) {
    // data-parallel gate/up GEMM with SwiGLU in the epilogue, bf16 h straight to c->a
    Prof pf(c, c->pass_verify ? P_GEMM_VERIFY : P_GEMM_DRAFT,
            (double)2 * c->f * n * c->esz + (double)M * n * c->esz + (double)M * c->f * c->esz,
            2.0 * M * 2 * c->f * n);
    kstamp_next(c, c->pass_verify ? P_GEMM_VERIFY : P_GEMM_DRAFT,
                (double)2 * c->f * n * c->esz + (double)M * n * c->esz + (double)M * c->f * c->esz,
                2.0 * M * 2 * c->f * n);
    const int k = gemm_tc_swiglu_bf16((const bf16*)c->a, n, (const bf16*)w.wgu, n, (bf16*)c->h, c->f, M, 2 * c->f,
                                      n, c->st);
    g_hsd_launches += k;
    fused = k > 0;
  }
  if (!fused) {
    gemm(c, c->a, n, w.wgu, n, c->big, 2 * c->f, M, 2 * c->f, n, false, -1, true);
    Prof pf(c, P_ROWWISE);
    PfScope l2(w.wd, b_d, 0, cap, 16);
    if (!ablate("swiglu")) { launch_swiglu(c->big, M, c->f, c->h, c->dt, m.pos, c->st); g_hsd_launches += 1; }
  }
  gemm(c, c->h, c->f, w.wd, c->f, x, n, M, n, c->f, true);
  g_hsd_launches += 4;  // rmsnorm x2, rope_kv, attention (merge and swiglu counted where launched)
}

// ------------------------------------------------------- vocab-sharded lm_head
// shard s owns head columns [lo_s, lo_{s+1}). c->a holds the M
// normalised rows. SIM computes every shard's columns itself; NCCL computes its
// own columns for the all-gathered rows of all G ranks (rank r's rows at r*M).
static void shard_head_verify(hsd_ctx* c, int M) {
  const size_t es = c->esz;
  const int n = c->n, G = c->G, r = c->srank;
  const int* lo = c->shard_lo;
  if (c->cfg.accept_mode == HSD_STOCHASTIC) {
    // per-row records over each shard's columns -> merged lse / tree-token logits /
    // Gumbel top-KG of this rank's rows (shard.cu); the walk never needs full rows
    const int T = c->T;
    const size_t rec = stoch_record_floats(T);
    const uint32_t seed = (uint32_t)c->cfg.seed;
    const float temp = c->cfg.temperature;
    if (c->shard_mode == HSD_SHARD_SIM) {
      for (int s = 0; s < G; ++s) {
        const int w = lo[s + 1] - lo[s];
        gemm(c, c->a, n, (const char*)c->head + (size_t)lo[s] * n * es, n, c->lslice, w, M, w, n, false, P_HEAD_VERIFY);
        { Prof pf(c, P_ROWWISE);
          launch_stoch_part(c->lslice, M, w, w, lo[s], T, c->t_tok, c->req_id, c->step, seed, temp,
                            c->sp_all + (size_t)s * M * rec, c->st); }
      }
      { Prof pf(c, P_ROWWISE);
        launch_stoch_merge(c->sp_all, G, (size_t)M, 0, M, T, c->sh_lse, c->sh_tl, c->sh_gv, c->sh_gi, c->st); }
      g_hsd_launches += G + 1;
      return;
    }
    const int w = lo[r + 1] - lo[r];
    const int b = c->b;
    if (!shard_allgather(c->a, c->a_all, (size_t)M * n * es, c->comm, c->st, c->nccl_err)) return;
    if (!shard_allgather(c->t_tok, c->tt_all, (size_t)b * T * 4, c->comm, c->st, c->nccl_err)) return;
    if (!shard_allgather(c->req_id, c->rid_all, (size_t)b * 4, c->comm, c->st, c->nccl_err)) return;
    gemm(c, c->a_all, n, (const char*)c->head + (size_t)lo[r] * n * es, n, c->lslice, w, G * M, w, n, false,
         P_HEAD_VERIFY);
    { Prof pf(c, P_ROWWISE);
      launch_stoch_part(c->lslice, G * M, w, w, lo[r], T, c->tt_all, c->rid_all, c->step, seed, temp, c->sp_loc,
                        c->st); }
    if (!shard_allgather(c->sp_loc, c->sp_all, (size_t)G * M * rec * 4, c->comm, c->st, c->nccl_err)) return;
    { Prof pf(c, P_ROWWISE);
      launch_stoch_merge(c->sp_all, G, (size_t)G * M, r * M, M, T, c->sh_lse, c->sh_tl, c->sh_gv, c->sh_gi, c->st); }
    g_hsd_launches += 2;
    return;
  }
  if (c->shard_mode == HSD_SHARD_SIM) {
    for (int s = 0; s < G; ++s) {
      const int w = lo[s + 1] - lo[s];
      gemm(c, c->a, n, (const char*)c->head + (size_t)lo[s] * n * es, n, c->lslice, w, M, w, n, false, P_HEAD_VERIFY);
      { Prof pf(c, P_ROWWISE); launch_argmax_part(c->lslice, M, w, w, lo[s], c->pv_all + (size_t)s * M, c->pi_all + (size_t)s * M, c->st); }
    }
    { Prof pf(c, P_ROWWISE); launch_argmax_merge(c->pv_all, c->pi_all, G, M, 0, M, c->mv.pos, c->argmax, c->st); }
    g_hsd_launches += G + 1;
    return;
  }
  const int w = lo[r + 1] - lo[r];
  if (!shard_allgather(c->a, c->a_all, (size_t)M * n * es, c->comm, c->st, c->nccl_err)) return;
  gemm(c, c->a_all, n, (const char*)c->head + (size_t)lo[r] * n * es, n, c->lslice, w, G * M, w, n, false,
       P_HEAD_VERIFY);
  { Prof pf(c, P_ROWWISE); launch_argmax_part(c->lslice, G * M, w, w, lo[r], c->pv_loc, c->pi_loc, c->st); }
  if (!shard_allgather(c->pv_loc, c->pv_all, (size_t)G * M * 4, c->comm, c->st, c->nccl_err)) return;
  if (!shard_allgather(c->pi_loc, c->pi_all, (size_t)G * M * 4, c->comm, c->st, c->nccl_err)) return;
  { Prof pf(c, P_ROWWISE); launch_argmax_merge(c->pv_all, c->pi_all, G, G * M, r * M, M, c->mv.pos, c->argmax, c->st); }
  g_hsd_launches += 2;
}

// draft one-pass logits, sharded: full fp32 rows reassembled for the row owner
static void shard_head_draft(hsd_ctx* c, int R) {
  const size_t es = c->esz;
  const int n = c->n, G = c->G, r = c->srank, wmax = c->shard_wmax;
  const int* lo = c->shard_lo;
  if (c->shard_mode == HSD_SHARD_SIM) {
    for (int s = 0; s < G; ++s) {
      const int w = lo[s + 1] - lo[s];
      gemm(c, c->a, n, (const char*)c->head_rank + (size_t)lo[s] * n * es, n, c->lrecv + (size_t)s * R * wmax, w, R,
           w, n, false, P_HEAD_DRAFT);
    }
  } else {
    const int w = lo[r + 1] - lo[r];
    if (!shard_allgather(c->a, c->a_all, (size_t)R * n * es, c->comm, c->st, c->nccl_err)) return;
    gemm(c, c->a_all, n, (const char*)c->head_rank + (size_t)lo[r] * n * es, n, c->lslice, w, G * R, w, n, false,
         P_HEAD_DRAFT);
    size_t so[HSD_MAX_SHARDS], sb[HSD_MAX_SHARDS], ro[HSD_MAX_SHARDS], rb[HSD_MAX_SHARDS];
    for (int p = 0; p < G; ++p) {
      so[p] = (size_t)p * R * w * 4; sb[p] = (size_t)R * w * 4;
      ro[p] = (size_t)p * R * wmax * 4; rb[p] = (size_t)R * (lo[p + 1] - lo[p]) * 4;
    }
    if (!shard_alltoallv((const char*)c->lslice, so, sb, (char*)c->lrecv, ro, rb, G, c->comm, c->st, c->nccl_err))
      return;
  }
  { Prof pf(c, P_ROWWISE); launch_scatter_cols(c->lrecv, (size_t)R * wmax, R, G, lo, c->draft_logits, c->V, c->st); }
  g_hsd_launches += 1;
}

// ---------------------------------------------------------------------- stages
static void stage_build(hsd_ctx* c) {
  Nvtx nv("hsd S0+S1 draft chain, one-pass logits, Alg. 1 tree");
  const int b = c->b, N = c->N, n = c->n, R = N + 1;
  const int kvmax = c->max_pos;
  // S0 (1): draft prefill of the pending pairs x_j = W_fc [H_{j-1}; E(t_j)] (R1)
  launch_k(meta_dprefill_kernel, b, 32 * ((R + 31) / 32), 0, c->st, c->md, R, c->n_pend, c->pend_tok, c->p,
           (c->cfg.flags & HSD_FLAG_NO_FIRST_TOKEN) ? 1 : 0);
  RowMeta mdv = c->md.view(nullptr, nullptr, 0, 0);
  c->attn_bytes = attn_bytes_for(c, 1, 0);
  launch_draft_concat(c->pend_H, c->md.tok, c->md.pos, c->md.slot, c->embed, c->dt, b * R, n, c->a, c->st);
  gemm(c, c->a, 2 * n, c->fc, 2 * n, c->x_d, n, b * R, n, 2 * n, false);
  layer_forward(c, c->draft, c->x_d, b * R, R, b, mdv, kv_layer(c, c->kv_d, 0), kvmax);
  launch_k(gather_last_kernel, b, 256, 0, c->st, c->x_d, R, c->n_pend, n, c->xw, c->chain, N, c->mc, c->p);
  g_hsd_launches += 3;
  // S0 (2): chain h_{i+1} = TL(h_i) at positions p + i (R2)
  RowMeta mcv = c->mc.view(nullptr, nullptr, 0, 0);
  const bool token_ar = (c->cfg.flags & HSD_FLAG_TOKEN_AR) != 0;
  const size_t ldL = (size_t)N * c->V;   // draft_logits [b, N, V]: request rows N * V apart
  for (int i = 1; i < N; ++i) {
    // (chain step i's row metadata was written by gather_last / the previous copy_chain)
    if (token_ar) {
      // token-level AR draft (EAGLE-style, NEXT-2, R27): the draft's own top-1 token of
      // step i is fed back, x_{i+1} = W_fc [h_i ; E(argmax l_i)] -- one lm_head GEMV,
      // one argmax and one fc GEMM per step instead of the one-pass head below
      launch_rmsnorm(c->xw, b, n, c->cfg.rms_eps, c->a, c->dt, nullptr, c->st);
      gemm(c, c->a, n, c->head_rank, n, c->draft_logits + (size_t)(i - 1) * c->V, (int)ldL, b, c->V, n, false,
           P_HEAD_DRAFT);
      launch_token_ar_input(c->draft_logits + (size_t)(i - 1) * c->V, ldL, c->V, c->perm_d, c->xw, b, n, c->embed,
                            c->dt, c->a, c->st);
      gemm(c, c->a, 2 * n, c->fc, 2 * n, c->xw, n, b, n, 2 * n, false);
      g_hsd_launches += 2;
    }
    c->attn_bytes = attn_bytes_for(c, 2, i);
    layer_forward(c, c->draft, c->xw, b, 1, b, mcv, kv_layer(c, c->kv_d, 0), kvmax);
    launch_k(copy_chain_kernel, b, 256, 0, c->st, c->xw, n, c->chain, N, i, c->mc, c->p);
    g_hsd_launches += 1;
  }
  if (token_ar) {   // the last chain row's logits
    launch_rmsnorm(c->xw, b, n, c->cfg.rms_eps, c->a, c->dt, nullptr, c->st);
    gemm(c, c->a, n, c->head_rank, n, c->draft_logits + (size_t)(N - 1) * c->V, (int)ldL, b, c->V, n, false,
         P_HEAD_DRAFT);
    g_hsd_launches += 1;
  } else {
    // S1a: one-pass logits L = RMSNorm_f(H_chain) W_head^T, rank order
    launch_rmsnorm(c->chain, b * N, n, c->cfg.rms_eps, c->a, c->dt, nullptr, c->st);
    if (c->shard_mode != HSD_SHARD_NONE) shard_head_draft(c, b * N);
    else gemm(c, c->a, n, c->head_rank, n, c->draft_logits, c->V, b * N, c->V, n, false, P_HEAD_DRAFT);
    g_hsd_launches += 1;
  }
  // S1b + S1c: Alg. 1, prune, fuse, linearise (+ planting)
  TreeParams P{};
  P.N = N; P.k = c->k; P.B = c->B; P.Br = c->Br; P.r = c->r; P.V = c->V; P.Vh = c->Vh; P.t_max = c->T;
  P.anc_words = c->W;
  P.fusion = (c->cfg.flags & HSD_FLAG_FUSION) ? 1 : 0;
  P.resample = (c->cfg.flags & HSD_FLAG_RESAMPLE) ? 1 : 0;
  P.zero_table = (c->cfg.flags & HSD_FLAG_ZERO_TABLE) ? 1 : 0;
  P.L = c->draft_logits; P.table = c->table; P.tdt = c->dt; P.tscale = c->table_scale; P.perm = c->perm_d; P.rank_of = c->rank_d;
  P.root_tok = c->root_tok;
  P.pt_n = c->pt_n; P.pt_tok = c->pt_tok; P.pt_par = c->pt_par; P.pt_depth = c->pt_depth; P.pt_lj = c->pt_lj;
  P.t_n = c->t_n; P.t_tok = c->t_tok; P.t_par = c->t_par; P.t_depth = c->t_depth; P.t_lj = c->t_lj;
  P.t_anc = c->t_anc;
  P.p = c->p; P.step = c->step;
  P.plant = (c->cfg.flags & HSD_FLAG_PLANTED) ? c->plant : nullptr;
  P.plant_stride = c->plant_stride;
  for (int i = 0; i < HSD_MAX_PLANT_DEPTH_DEV; ++i) P.plant_rates[i] = c->cfg.plant_rates[i];
  P.seed = (uint32_t)c->cfg.seed; P.req_id = c->req_id; P.err = c->err;
  P.pf = L2Pf{nullptr, 0ull, 0};
  if (g_l2pf_cap && !c->layers.empty()) {   // verify layer 0's QKV weights stream next
    PfScope l2(c->layers[0].wqkv, (size_t)c->qkvd * n * c->esz, 0, g_l2pf_cap, 32);
    P.pf = take_l2pf();
  }
  if (!ablate("tree")) { Prof pf(c, P_TREE); launch_tree(P, TREE_MODE_FRESH, b, c->st); }
  g_hsd_launches += 1;
}

static void stage_verify(hsd_ctx* c) {
  Nvtx nv("hsd S2 target tree verify");
  const int b = c->b, T = c->T, n = c->n, M = b * T;
  launch_k(meta_verify_kernel, b, 32 * ((T + 31) / 32), 0, c->st, c->mv, T, c->t_n, c->t_tok, c->t_depth, c->p);
  RowMeta m = c->mv.view(c->p, c->t_anc, T, c->W);
  launch_embed(c->embed, c->dt, c->mv.tok, c->mv.pos, M, n, c->Hver, c->st);
  g_hsd_launches += 2;
  c->pass_verify = 1;
  c->attn_bytes = attn_bytes_for(c, 0, 0);
  for (int l = 0; l < c->L; ++l) layer_forward(c, c->layers[l], c->Hver, M, T, b, m, kv_layer(c, c->kv_t, l), c->max_pos);
  c->pass_verify = 0;
  launch_rmsnorm(c->Hver, M, n, c->cfg.rms_eps, c->a, c->dt, c->mv.pos, c->st);
  if (c->shard_mode != HSD_SHARD_NONE) {
    shard_head_verify(c, M);
  } else {
    gemm(c, c->a, n, c->head, n, c->logits, c->V, M, c->V, n, false, P_HEAD_VERIFY);
  }
  if (c->cfg.accept_mode == HSD_GREEDY && c->shard_mode == HSD_SHARD_NONE) {   // the stochastic walk reads the logits rows itself
    Prof pf(c, P_ROWWISE);
    launch_argmax_rows(c->logits, M, c->V, c->mv.pos, c->argmax, c->st);
  }
  g_hsd_launches += 2;
}

// S3 + S4 without Alg. 2: walk, KV compaction, commit (append: the dedicated
// verify pass of the re-sampled tree, fusion off -- tokens / pairs follow the
// step's first pass)
static void walk_compact_commit(hsd_ctx* c, int append) {
  const int b = c->b;
  AcceptParams A{};
  A.mode = c->cfg.accept_mode == HSD_STOCHASTIC ? 1 : 0;
  A.append = append;
  A.N = c->N; A.t_max = c->T; A.V = c->V; A.temperature = c->cfg.temperature;
  A.seed = (uint32_t)c->cfg.seed; A.req_id = c->req_id;
  A.t_tok = c->t_tok; A.t_par = c->t_par; A.t_n = c->t_n; A.argmax = c->argmax; A.logits = c->logits;
  A.sh_lse = c->sh_lse; A.sh_tl = c->sh_tl; A.sh_gv = c->sh_gv; A.sh_gi = c->sh_gi;   // (null unless sharded + stochastic)
  A.step = c->step;
  A.acc_n = c->acc_n; A.acc_slots = c->acc_slots; A.bonus = c->bonus; A.emitted = c->emitted;
  A.n_emitted = c->n_emitted;
  { Prof pf(c, P_WALK); launch_walk(A, b, c->st); }
  CompactParams C{};
  C.kv_base = c->kv_t; C.layer_stride = c->kv_layer_elems; C.block_table = c->block_table;
  C.pages_per_req = c->pages_per_req; C.page_size = c->page_size; C.kv_heads = c->Hkv; C.head_dim = c->hd;
  C.N = c->N; C.acc_n = c->acc_n; C.acc_slots = c->acc_slots; C.p = c->p;
  { Prof pf(c, P_COMPACT, 2.0 * b * c->N * c->L * 2 * c->kd * c->esz); launch_compact(C, b, c->L, c->dt, c->st); }
  CommitParams M{};
  M.N = c->N; M.t_max = c->T; M.hidden = c->n; M.Hverify = c->Hver; M.append = append;
  M.acc_n = c->acc_n; M.acc_slots = c->acc_slots; M.emitted = c->emitted; M.bonus = c->bonus;
  M.n_emitted = c->n_emitted;
  M.pend_H = c->pend_H; M.pend_tok = c->pend_tok; M.n_pend = c->n_pend; M.root_tok = c->root_tok; M.p = c->p;
  M.step = c->step;
  launch_commit(M, b, c->st);
  g_hsd_launches += 3;
}

static void stage_accept(hsd_ctx* c, int32_t* d_emitted, int32_t* d_n) {
  Nvtx nv("hsd S3+S4 walk, compaction, Alg. 2");
  const int b = c->b;
  AcceptParams A{};
  A.mode = c->cfg.accept_mode == HSD_STOCHASTIC ? 1 : 0;
  A.N = c->N; A.t_max = c->T; A.V = c->V; A.temperature = c->cfg.temperature;
  A.seed = (uint32_t)c->cfg.seed; A.req_id = c->req_id;
  A.t_tok = c->t_tok; A.t_par = c->t_par; A.t_n = c->t_n; A.argmax = c->argmax; A.logits = c->logits;
  A.sh_lse = c->sh_lse; A.sh_tl = c->sh_tl; A.sh_gv = c->sh_gv; A.sh_gi = c->sh_gi;   // (null unless sharded + stochastic)
  A.step = c->step;
  A.acc_n = c->acc_n; A.acc_slots = c->acc_slots; A.bonus = c->bonus; A.emitted = c->emitted;
  A.n_emitted = c->n_emitted;
  { Prof pf(c, P_WALK); launch_walk(A, b, c->st); }
  CompactParams C{};
  C.kv_base = c->kv_t; C.layer_stride = c->kv_layer_elems; C.block_table = c->block_table;
  C.pages_per_req = c->pages_per_req; C.page_size = c->page_size; C.kv_heads = c->Hkv; C.head_dim = c->hd;
  C.N = c->N; C.acc_n = c->acc_n; C.acc_slots = c->acc_slots; C.p = c->p;
  { Prof pf(c, P_COMPACT, 2.0 * b * c->N * c->L * 2 * c->kd * c->esz); launch_compact(C, b, c->L, c->dt, c->st); }
  // Alg. 2 re-sampling into the pending tree (reads acc_n, bonus, draft logits)
  TreeParams P{};
  P.N = c->N; P.k = c->k; P.B = c->B; P.Br = c->Br; P.r = c->r; P.V = c->V; P.Vh = c->Vh; P.t_max = c->T;
  P.anc_words = c->W;
  P.fusion = (c->cfg.flags & HSD_FLAG_FUSION) ? 1 : 0;
  P.resample = (c->cfg.flags & HSD_FLAG_RESAMPLE) ? 1 : 0;
  P.zero_table = (c->cfg.flags & HSD_FLAG_ZERO_TABLE) ? 1 : 0;
  P.L = c->draft_logits; P.table = c->table; P.tdt = c->dt; P.tscale = c->table_scale; P.perm = c->perm_d; P.rank_of = c->rank_d;
  P.pt_n = c->pt_n; P.pt_tok = c->pt_tok; P.pt_par = c->pt_par; P.pt_depth = c->pt_depth; P.pt_lj = c->pt_lj;
  P.acc_n = c->acc_n; P.bonus = c->bonus; P.err = c->err; P.req_id = c->req_id;
  P.pf = L2Pf{nullptr, 0ull, 0};
  if (g_l2pf_cap) {   // the next step's draft prefill GEMM streams W_fc first
    PfScope l2(c->fc, (size_t)2 * c->n * c->n * c->esz, 0, g_l2pf_cap, 32);
    P.pf = take_l2pf();
  }
  if (!ablate("tree")) { Prof pf(c, P_RESAMPLE); launch_tree(P, TREE_MODE_RESAMPLE, b, c->st); }
  CommitParams M{};
  M.N = c->N; M.t_max = c->T; M.hidden = c->n; M.Hverify = c->Hver;
  M.acc_n = c->acc_n; M.acc_slots = c->acc_slots; M.emitted = c->emitted; M.bonus = c->bonus;
  M.pend_H = c->pend_H; M.pend_tok = c->pend_tok; M.n_pend = c->n_pend; M.root_tok = c->root_tok; M.p = c->p;
  M.step = c->step;
  M.n_emitted = c->n_emitted;
  launch_commit(M, b, c->st);
  g_hsd_launches += 4;
  if ((c->cfg.flags & HSD_FLAG_RESAMPLE) && !(c->cfg.flags & HSD_FLAG_FUSION)) {
    // re-sampling WITHOUT verification fusion (the Fig. 12 ablation): the Alg. 2
    // tree just built, rooted at the new bonus token, is verified by its own target
    // pass in this step; the next step's tree is fresh only
    launch_pending_as_tree(c->pt_n, c->pt_tok, c->pt_par, c->pt_depth, c->pt_lj, c->Br + 1, c->t_n, c->t_tok,
                           c->t_par, c->t_depth, c->t_lj, c->t_anc, c->T, c->W, b, c->st);
    g_hsd_launches += 1;
    stage_verify(c);
    walk_compact_commit(c, 1);
  }
  if (d_emitted) cudaMemcpyAsync(d_emitted, c->emitted, sizeof(int32_t) * b * (c->N + 1), cudaMemcpyDeviceToDevice, c->st);
  if (d_n) cudaMemcpyAsync(d_n, c->n_emitted, sizeof(int32_t) * b, cudaMemcpyDeviceToDevice, c->st);
}

static void drop_graphs(hsd_ctx* c) {
  if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }
  for (int i = 0; i < 3; ++i)
    if (c->sgraph[i]) { cudaGraphExecDestroy(c->sgraph[i]); c->sgraph[i] = nullptr; }
}

// Run one stage of a staged step. With a non-legacy stream and profiling off, the
// stage is captured once into its own CUDA graph and replayed (the same launches,
// same order, as inside hsd_step's graph), so staged latencies match the step's.
static bool g_stage_graphs = [] { const char* e = getenv("HSD_STAGE_GRAPHS"); return !(e && e[0] == '0'); }();
template <typename F>
static hsd_status run_stage(hsd_ctx* ctx, int idx, F&& body) {
  hsd_ctx* c = ctx;
  if (c->prof_on || c->st == nullptr || !g_stage_graphs) {
    body();
    CU(cudaGetLastError());
    if (!c->nccl_err.empty()) return fail(c, HSD_ENCCL, c->nccl_err);
    return HSD_OK;
  }
  if (!c->sgraph[idx]) {
    int64_t before = g_hsd_launches;
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    body();
    c->capturing = false;
    CU(cudaStreamEndCapture(c->st, &g));
    if (!c->nccl_err.empty()) return fail(c, HSD_ENCCL, c->nccl_err);
    c->sgraph_kernels[idx] = g_hsd_launches - before;
    g_hsd_launches = before;
    CU(cudaGraphInstantiate(&c->sgraph[idx], g, 0));
    cudaGraphDestroy(g);
  }
  CU(cudaGraphLaunch(c->sgraph[idx], c->st));
  c->sgraph_replays[idx]++;
  return HSD_OK;
}

// Prefill of ONE request slot r (PAPER.md:184 setting; R1, R22): target causal
// forward over the prompt (KV + H), first token, draft prefill over the prompt's
// (H_{j-1}, t_j) pairs. Touches only slot r's state, so it also admits a new request
// into a live batch (hsd_admit, continuous batching).
static hsd_status prefill_one(hsd_ctx* ctx, int r, const int32_t* pt, int P0, int32_t* d_first, int32_t req_g) {
  hsd_ctx* c = ctx;
  c->req_id_h[r] = req_g;
  c->p_hi[r] = P0;
  CU(cudaMemcpyAsync(c->req_id + r, &c->req_id_h[r], 4, cudaMemcpyHostToDevice, c->st));
  const int n = c->n, N = c->N;
  std::vector<int32_t> tok, pos, kvpos, req, klo, khi, slot;
  // target causal forward over the prompt, chunked
  const int PC = c->pchunk;
  for (int s0 = 0; s0 < P0; s0 += PC) {
    int M = std::min(PC, P0 - s0);
    tok.resize(M); pos.resize(M); kvpos.resize(M); req.resize(M); klo.resize(M); khi.resize(M); slot.resize(M);
    for (int i = 0; i < M; ++i) {
      tok[i] = pt[s0 + i]; pos[i] = s0 + i; kvpos[i] = s0 + i; req[i] = r; klo[i] = 0; khi[i] = s0 + i + 1;
      slot[i] = -1;
    }
    CU(cudaMemcpyAsync(c->mp.tok, tok.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.pos, pos.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.kvpos, kvpos.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.req, req.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.klo, klo.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.khi, khi.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.slot, slot.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    RowMeta m = c->mp.view(nullptr, nullptr, 0, 0);
    // rows of this chunk belong to request r: pass them as one "request" with
    // the block table row r by offsetting the row->request map (req[] = r).
    launch_embed(c->embed, c->dt, c->mp.tok, c->mp.pos, M, n, c->x_p, c->st);
    g_hsd_launches += 1;
    for (int l = 0; l < c->L; ++l)
      layer_forward(c, c->layers[l], c->x_p, M, M, 1, m, kv_layer(c, c->kv_t, l), s0 + M);
    CU(cudaMemcpyAsync(c->H_prompt + (size_t)s0 * n, c->x_p, sizeof(float) * M * n, cudaMemcpyDeviceToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  // logits of the last prompt position -> first token (R22)
  const float* Hlast = c->H_prompt + (size_t)(P0 - 1) * n;
  launch_rmsnorm(Hlast, 1, n, c->cfg.rms_eps, c->a, c->dt, nullptr, c->st);
  gemm(c, c->a, n, c->head, n, c->logits, c->V, 1, c->V, n, false);
  launch_k(first_token_kernel, 1, 512, 0, c->st, c->logits, c->V, c->cfg.accept_mode == HSD_STOCHASTIC ? 1 : 0,
                                           1.0f / c->cfg.temperature, (uint32_t)c->cfg.seed,
                                           req_g, r, Hlast, n, P0, N, c->pend_H, c->pend_tok,
                                           c->n_pend, c->root_tok, c->p, d_first);
  g_hsd_launches += 2;
  // draft prefill over pairs j = 1..P0-1: x_j = W_fc [H_{j-1}; E(t_j)] (R1)
  for (int j0 = 1; j0 < P0; j0 += PC) {
    int M = std::min(PC, P0 - j0);
    tok.resize(M); pos.resize(M); kvpos.resize(M); req.resize(M); klo.resize(M); khi.resize(M); slot.resize(M);
    for (int i = 0; i < M; ++i) {
      int j = j0 + i;
      tok[i] = pt[j]; pos[i] = j; kvpos[i] = j; req[i] = r; klo[i] = 1; khi[i] = j + 1; slot[i] = -1;
    }
    CU(cudaMemcpyAsync(c->mp.tok, tok.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.pos, pos.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.kvpos, kvpos.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.req, req.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.klo, klo.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.khi, khi.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->mp.slot, slot.data(), 4 * M, cudaMemcpyHostToDevice, c->st));
    RowMeta m = c->mp.view(nullptr, nullptr, 0, 0);
    launch_draft_concat(c->H_prompt + (size_t)(j0 - 1) * n, c->mp.tok, c->mp.pos, nullptr, c->embed, c->dt, M, n,
                        c->a, c->st);
    gemm(c, c->a, 2 * n, c->fc, 2 * n, c->x_p, n, M, n, 2 * n, false);
    layer_forward(c, c->draft, c->x_p, M, M, 1, m, kv_layer(c, c->kv_d, 0), j0 + M);
    g_hsd_launches += 1;
    CU(cudaStreamSynchronize(c->st));
  }

  return HSD_OK;
}

// ====================================================================== C ABI
extern "C" {

void hsd_config_defaults(hsd_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->rope_theta = 10000.f; c->rms_eps = 1e-5f;
  c->resample_budget_Br = 4; c->resample_threshold_r = 1;
  c->page_size = 64; c->precision = HSD_BF16; c->accept_mode = HSD_GREEDY; c->temperature = 1.f;
  c->flags = HSD_FLAG_RESAMPLE | HSD_FLAG_FUSION;
  c->max_batch = 1;
}

const char* hsd_last_error(const hsd_ctx* ctx) { return ctx ? ctx->errmsg.c_str() : "null context"; }

hsd_status hsd_nccl_unique_id(uint8_t* out) {
  if (!out) return HSD_EINVAL;
  std::string err;
  if (!shard_nccl_unique_id(out, err)) {
    fprintf(stderr, "hsd_nccl_unique_id: %s\n", err.c_str());
    return HSD_ENCCL;
  }
  return HSD_OK;
}

int64_t hsd_kernel_launches(const hsd_ctx* ctx) {
  if (!ctx) return 0;
  int64_t n = (g_hsd_launches - ctx->launches0) + ctx->graph_replays * ctx->graph_kernels;
  for (int i = 0; i < 3; ++i) n += ctx->sgraph_replays[i] * ctx->sgraph_kernels[i];
  return n;
}

static std::string check_config(const hsd_config* c) {
  if (c->vocab < 2 || c->hidden < 1 || c->layers < 0 || c->q_heads < 1 || c->kv_heads < 1 || c->ffn < 1)
    return "model shape must be positive (vocab >= 2)";
  if (c->q_heads % c->kv_heads) return "q_heads must be a multiple of kv_heads";
  if (c->head_dim < 2 || c->head_dim % 2 || c->head_dim > 128) return "head_dim must be even and <= 128";
  if (c->q_heads * c->head_dim < 1) return "bad heads";
  if (c->steps_N < 1 || c->steps_N > 16) return "steps_N must be in [1, 16] (contract violation: N < 1)";
  if (c->branch_k < 1 || c->branch_k > 8) return "branch_k must be in [1, 8]";
  if (c->branch_k > c->vocab) return "k > |V| (contract violation)";
  if (c->budget_B < 1) return "budget_B must be >= 1 (contract violation: B < 1)";
  if (c->resample_budget_Br < 0 || c->resample_threshold_r < 0) return "B_r and r must be >= 0";
  if (c->resample_budget_Br + 1 > 64) return "B_r + 1 must be <= 64 (pending-tree capacity)";
  long cand = 1 + c->branch_k + (long)(c->steps_N - 1) * c->branch_k * c->branch_k;
  if (cand > MAXN_TREE) return "1 + k + (N-1)k^2 candidate nodes exceed the device tree capacity (256)";
  if (c->budget_B + c->resample_budget_Br + 1 > MAXN_TREE) return "B + B_r + 1 exceeds 256 verify slots";
  if (c->hot_tokens < 0 || c->hot_tokens > c->vocab) return "hot_tokens out of range";
  if (c->hot_tokens > 0 && c->vocab_perm == nullptr) return "hot_tokens > 0 requires vocab_perm";
  if (c->max_batch < 1 || c->max_ctx < 2) return "max_batch >= 1 and max_ctx >= 2 required";
  if (c->page_size < 1) return "page_size >= 1";
  if (c->precision != HSD_FP32_VERIFY && c->precision != HSD_BF16) return "precision must be FP32_VERIFY or BF16";
  if (c->accept_mode != HSD_GREEDY && c->accept_mode != HSD_STOCHASTIC) return "bad accept_mode";
  if (c->accept_mode == HSD_STOCHASTIC && !(c->temperature > 0.f)) return "temperature must be > 0";
  if (c->shard_mode != HSD_SHARD_NONE) {
    if (c->shard_mode != HSD_SHARD_NCCL && c->shard_mode != HSD_SHARD_SIM) return "bad shard_mode";
    if (c->vocab_shards < 1 || c->vocab_shards > HSD_MAX_SHARDS) return "vocab_shards must be in [1, 16]";
    if (c->vocab < 128 * c->vocab_shards) return "vocab_shards > V / 128 (each shard owns >= 128 columns)";
    if (c->shard_mode == HSD_SHARD_SIM && c->shard_rank != 0) return "HSD_SHARD_SIM requires shard_rank 0";
    if (c->shard_rank < 0 || c->shard_rank >= c->vocab_shards) return "shard_rank must be in [0, vocab_shards)";
  }
  return "";
}

hsd_status hsd_init_model(const hsd_config* cfg, int device, void* cuda_stream, hsd_ctx** out) {
  if (!out) return HSD_EINVAL;
  *out = nullptr;
  if (!cfg) return HSD_EINVAL;
  std::string why = check_config(cfg);
  if (!why.empty()) {
    static thread_local std::string last;
    last = why;
    fprintf(stderr, "hsd_init_model: %s\n", why.c_str());
    return HSD_EINVAL;
  }
  if (cfg->shard_mode != HSD_SHARD_NONE && (cfg->flags & HSD_FLAG_TOKEN_AR)) {
    fprintf(stderr, "hsd_init_model: the token-AR draft mode is not combined with the vocab-sharded head\n");
    return HSD_EUNSUP;
  }
  if (cfg->shard_mode != HSD_SHARD_NONE && cfg->accept_mode != HSD_GREEDY &&
      cfg->branch_k + cfg->resample_budget_Br >= HSD_SHARD_KG) {
    // a rejected set (the children of one node, <= k + B_r) must leave a candidate in
    // the merged Gumbel top-KG
    fprintf(stderr, "hsd_init_model: stochastic + vocab shards needs branch_k + B_r < %d\n", HSD_SHARD_KG);
    return HSD_EUNSUP;
  }
  hsd_ctx* ctx = new hsd_ctx();
  ctx->cfg = *cfg;
  ctx->dev = device;
  ctx->launches0 = g_hsd_launches;
  CU(cudaSetDevice(device));
  ctx->st = (cudaStream_t)cuda_stream;
  tree_trace_init();
  hsd_ctx* c = ctx;
  c->dt = cfg->precision == HSD_BF16 ? DT_BF16 : DT_F32;
  c->esz = c->dt == DT_BF16 ? 2 : 4;
  c->use_tc = (cfg->flags & HSD_FLAG_TCGEN05) && c->dt == DT_BF16;
  c->n = cfg->hidden; c->L = cfg->layers; c->Hq = cfg->q_heads; c->Hkv = cfg->kv_heads; c->hd = cfg->head_dim;
  c->f = cfg->ffn; c->V = cfg->vocab; c->qd = c->Hq * c->hd; c->kd = c->Hkv * c->hd; c->qkvd = c->qd + 2 * c->kd;
  c->N = cfg->steps_N; c->k = cfg->branch_k; c->B = cfg->budget_B; c->Br = cfg->resample_budget_Br;
  c->r = cfg->resample_threshold_r;
  c->Vh = cfg->hot_tokens > 0 ? cfg->hot_tokens : c->V;
  c->d = cfg->table_rank > 0 ? cfg->table_rank : std::max(1, c->n / 16);
  c->T = c->B + c->Br + 1;
  c->W = (c->T + 63) / 64;
  c->maxb = cfg->max_batch;
  c->page_size = cfg->page_size;
  const int n = c->n, V = c->V;
  const size_t es = c->esz;
  bool fail_alloc = false;
  auto A = [&](size_t bytes) {
    void* p = dalloc(c, bytes);
    if (!p) fail_alloc = true;
    return p;
  };
  // ---- weights (R23): Philox, tensor ids as in DESIGN.md section 4
  const uint32_t seed = (uint32_t)cfg->seed;
  auto sc = [](int fan_in) { return sqrtf(3.0f / (float)fan_in); };
  c->embed = A((size_t)V * n * es);
  c->head = A((size_t)V * n * es);
  c->fc = A((size_t)n * 2 * n * es);
  if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
  launch_philox_fill(c->embed, c->dt, (size_t)V * n, seed, 1, 1.0f, c->st);
  launch_philox_fill(c->head, c->dt, (size_t)V * n, seed, 2, sc(n), c->st);
  launch_philox_fill(c->fc, c->dt, (size_t)n * 2 * n, seed, 5, sc(2 * n), c->st);
  auto make_layer = [&](uint32_t tid0) {
    LayerW w;
    w.wqkv = A((size_t)c->qkvd * n * es);
    w.wo = A((size_t)n * c->qd * es);
    w.wgu = A((size_t)2 * c->f * n * es);
    w.wd = A((size_t)n * c->f * es);
    if (fail_alloc) return w;
    launch_philox_fill(w.wqkv, c->dt, (size_t)c->qd * n, seed, tid0 + 0, sc(n), c->st);
    launch_philox_fill((char*)w.wqkv + (size_t)c->qd * n * es, c->dt, (size_t)c->kd * n, seed, tid0 + 1, sc(n), c->st);
    launch_philox_fill((char*)w.wqkv + (size_t)(c->qd + c->kd) * n * es, c->dt, (size_t)c->kd * n, seed, tid0 + 2,
                       sc(n), c->st);
    launch_philox_fill(w.wo, c->dt, (size_t)n * c->qd, seed, tid0 + 3, sc(c->qd), c->st);
    // gate (tid+4) then up (tid+5) into a scratch, then interleaved in 16-row
    // groups (see launch_swiglu / gemm_tc_swiglu_bf16)
    launch_philox_fill(c->gu_tmp, c->dt, (size_t)c->f * n, seed, tid0 + 4, sc(n), c->st);
    launch_philox_fill((char*)c->gu_tmp + (size_t)c->f * n * es, c->dt, (size_t)c->f * n, seed, tid0 + 5, sc(n),
                       c->st);
    launch_interleave_gu(c->gu_tmp, c->f, n, w.wgu, c->dt, c->st);
    launch_philox_fill(w.wd, c->dt, (size_t)n * c->f, seed, tid0 + 6, sc(c->f), c->st);
    return w;
  };
  if (c->f % 64) { hsd_destroy(c); fprintf(stderr, "hsd_init_model: ffn must be a multiple of 64\n"); return HSD_EINVAL; }
  c->gu_tmp = A((size_t)2 * c->f * n * es);
  if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
  for (int l = 0; l < c->L; ++l) c->layers.push_back(make_layer(100 + 8 * l));
  c->draft = make_layer(60);
  CU(cudaStreamSynchronize(c->st));
  cudaFree(c->gu_tmp);
  c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), c->gu_tmp));
  c->gu_tmp = nullptr;
  if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
  // ---- vocab permutation (hot set, R5)
  std::vector<int32_t> perm, rank;
  if (cfg->hot_tokens > 0) {
    perm.assign(cfg->vocab_perm, cfg->vocab_perm + V);
    rank.assign(V, -1);
    for (int i = 0; i < V; ++i) {
      if (perm[i] < 0 || perm[i] >= V || rank[perm[i]] >= 0) {
        hsd_destroy(c);
        fprintf(stderr, "hsd_init_model: vocab_perm is not a permutation\n");
        return HSD_EINVAL;
      }
      rank[perm[i]] = i;
    }
    c->perm_d = (int32_t*)A(sizeof(int32_t) * V);
    c->rank_d = (int32_t*)A(sizeof(int32_t) * V);
    if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
    CU(cudaMemcpyAsync(c->perm_d, perm.data(), sizeof(int32_t) * V, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->rank_d, rank.data(), sizeof(int32_t) * V, cudaMemcpyHostToDevice, c->st));
    // draft head rows in rank order, so hot columns of L are contiguous
    c->head_rank = A((size_t)V * n * es);
    if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
    if (c->dt == DT_F32) gather_same_kernel_f32<<<V, 256, 0, c->st>>>((const float*)c->head, c->perm_d, n, (float*)c->head_rank);
    else gather_same_kernel_bf16<<<V, 256, 0, c->st>>>((const bf16*)c->head, c->perm_d, n, (bf16*)c->head_rank);
  } else {
    c->head_rank = c->head;
  }
  // ---- token-info table W_collapsed = W_E W1 W2, row RMSNorm, 2-D hot prune
  {
    const int d = c->d, Vh = c->Vh;
    void* w1 = A((size_t)d * n * es);
    void* w2 = A((size_t)V * d * es);
    float* Esel = (float*)A((size_t)Vh * n * 4);
    float* W1f = (float*)A((size_t)d * n * 4);
    float* W2f = (float*)A((size_t)V * d * 4);
    float* C1 = (float*)A((size_t)Vh * d * 4);
    int chunk = (int)std::max<size_t>(1, std::min<size_t>(Vh, (size_t)(512u << 20) / ((size_t)V * 4)));
    float* C2 = (float*)A((size_t)chunk * V * 4);
    const bool fp8 = (cfg->flags & HSD_FLAG_TABLE_FP8) != 0;
    const size_t tes = fp8 ? 1 : es;               // e4m3 codes + a per-row scale (R25)
    c->table = A((size_t)Vh * Vh * tes);
    if (fp8) c->table_scale = (float*)A((size_t)Vh * 4);
    if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
    launch_philox_fill(w1, c->dt, (size_t)d * n, seed, 3, sc(n), c->st);
    launch_philox_fill(w2, c->dt, (size_t)V * d, seed, 4, sc(d), c->st);
    launch_gather_rows_f32(c->embed, c->dt, c->perm_d, Vh, n, Esel, c->st);
    launch_gather_rows_f32(w1, c->dt, nullptr, d, n, W1f, c->st);
    launch_gather_rows_f32(w2, c->dt, c->perm_d, V, d, W2f, c->st);
    gemm_simt(Esel, n, W1f, n, DT_F32, C1, d, Vh, d, n, false, c->st);
    for (int r0 = 0; r0 < Vh; r0 += chunk) {
      int rows = std::min(chunk, Vh - r0);
      gemm_simt(C1 + (size_t)r0 * d, d, W2f, d, DT_F32, C2, V, rows, V, d, false, c->st);
      if (fp8)
        launch_table_rows_fp8(C2, rows, V, Vh, (char*)c->table + (size_t)r0 * Vh, c->table_scale + r0, c->st);
      else
        launch_table_rows(C2, rows, V, Vh, nullptr, (char*)c->table + (size_t)r0 * Vh * es, c->dt, c->st);
    }
    CU(cudaStreamSynchronize(c->st));
    for (void* p : {w1, w2, (void*)Esel, (void*)W1f, (void*)W2f, (void*)C1, (void*)C2}) {
      cudaFree(p);
      c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), p));
    }
  }
  // ---- RoPE tables (host double precision)
  c->pages_per_req = (cfg->max_ctx + c->T + c->N + 8 + c->page_size - 1) / c->page_size;
  c->pages_per_req += c->pages_per_req & 1;   // even: the tcgen05 attention reads pages in pairs
  c->max_pos = c->pages_per_req * c->page_size;
  {
    int half = c->hd / 2;
    std::vector<float> hc((size_t)c->max_pos * half), hs((size_t)c->max_pos * half);
    for (int pos = 0; pos < c->max_pos; ++pos)
      for (int i = 0; i < half; ++i) {
        double inv = std::pow((double)cfg->rope_theta, -(2.0 * i) / (double)c->hd);
        double ang = (double)pos * inv;
        hc[(size_t)pos * half + i] = (float)std::cos(ang);
        hs[(size_t)pos * half + i] = (float)std::sin(ang);
      }
    c->rope_cos = (float*)A(hc.size() * 4);
    c->rope_sin = (float*)A(hs.size() * 4);
    if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
    CU(cudaMemcpyAsync(c->rope_cos, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice, c->st));
    CU(cudaMemcpyAsync(c->rope_sin, hs.data(), hs.size() * 4, cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  // ---- paged KV pools + identity block table
  {
    const int b = c->maxb;
    c->kv_layer_elems = (size_t)b * c->pages_per_req * 2 * c->Hkv * c->page_size * c->hd;
    c->kv_t = A(c->kv_layer_elems * es * std::max(1, c->L));
    c->kv_d = A(c->kv_layer_elems * es);
    c->block_table = (int32_t*)A(sizeof(int32_t) * b * c->pages_per_req);
    if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
    std::vector<int32_t> bt((size_t)b * c->pages_per_req);
    for (size_t i = 0; i < bt.size(); ++i) bt[i] = (int32_t)i;
    CU(cudaMemcpyAsync(c->block_table, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice, c->st));
  }
  // ---- state + workspace
  {
    const int b = c->maxb, T = c->T, N = c->N, Br1 = c->Br + 1;
    auto I = [&](size_t cnt) { return (int32_t*)A(cnt * 4); };
    auto F = [&](size_t cnt) { return (float*)A(cnt * 4); };
    c->req_id = I(b); c->req_id_h.assign(b, 0); c->p_hi.assign(b, 0);
    c->p = I(b); c->root_tok = I(b); c->n_pend = I(b); c->pend_tok = I((size_t)b * (N + 1)); c->step = I(1);
    c->pend_H = F((size_t)b * (N + 1) * n); c->err = (int*)I(1);
    c->pt_n = I(b); c->pt_tok = I((size_t)b * Br1); c->pt_par = I((size_t)b * Br1); c->pt_depth = I((size_t)b * Br1);
    c->pt_lj = F((size_t)b * Br1);
    c->t_n = I(b); c->t_tok = I((size_t)b * T); c->t_par = I((size_t)b * T); c->t_depth = I((size_t)b * T);
    c->t_lj = F((size_t)b * T); c->t_anc = (uint64_t*)A((size_t)b * T * c->W * 8);
    c->acc_n = I(b); c->acc_slots = I((size_t)b * N); c->bonus = I(b); c->emitted = I((size_t)b * (N + 1));
    c->n_emitted = I(b);
    c->pchunk = std::min(prefill_chunk(), std::max(256, cfg->max_ctx));
    c->Mcap = std::max({b * T, b * (N + 1), c->pchunk});
    const int Mc = c->Mcap;
    const size_t wa = std::max({(size_t)2 * n, (size_t)c->qd, (size_t)c->f});
    c->a = A((size_t)Mc * wa * es);
    c->qb = A((size_t)Mc * c->qd * es);
    c->ob = A((size_t)Mc * c->qd * es);
    c->h = A((size_t)Mc * c->f * es);
    c->big = F((size_t)Mc * std::max(c->qkvd, 2 * c->f));
    c->big_dp = F((size_t)Mc * c->qkvd);
    c->x_d = F((size_t)b * (N + 1) * n);
    c->xw = F((size_t)b * n);
    c->Hver = F((size_t)b * T * n);
    c->chain = F((size_t)b * N * n);
    c->draft_logits = F((size_t)b * N * V);
    c->logits = F((size_t)std::max(b * T, 1) * V);
    c->argmax = I((size_t)b * T);
    c->x_p = F((size_t)c->pchunk * n);
    c->H_prompt = F((size_t)(cfg->max_ctx + 1) * n);
    c->attn_ws_floats = attention_ws_floats(std::max(b * T, b * (N + 1)), c->Hq, c->hd, 16);
    c->attn_ws = F(c->attn_ws_floats);
    auto meta = [&](MetaBuf& m, size_t rows) {
      m.tok = I(rows); m.pos = I(rows); m.kvpos = I(rows); m.req = I(rows); m.klo = I(rows); m.khi = I(rows);
      m.slot = I(rows);
    };
    meta(c->mv, (size_t)b * T);
    meta(c->md, (size_t)b * (N + 1));
    meta(c->mc, (size_t)b);
    meta(c->mp, (size_t)c->pchunk);
    if (cfg->shard_mode != HSD_SHARD_NONE) {
      c->shard_mode = cfg->shard_mode;
      c->G = cfg->vocab_shards;
      c->srank = cfg->shard_rank;
      for (int s = 0; s < c->G; ++s) c->shard_lo[s] = (int)(((long)s * V / c->G) / 128 * 128);
      c->shard_lo[c->G] = V;
      c->shard_wmax = 0;
      for (int s = 0; s < c->G; ++s) c->shard_wmax = std::max(c->shard_wmax, c->shard_lo[s + 1] - c->shard_lo[s]);
      const int rows = std::max(b * T, b * N), G = c->G, wmax = c->shard_wmax;
      c->shard_rows = rows;
      const int grows = c->shard_mode == HSD_SHARD_NCCL ? G * rows : rows;
      c->lslice = F((size_t)grows * wmax);
      c->lrecv = F((size_t)G * rows * wmax);
      c->pv_loc = F((size_t)G * rows); c->pi_loc = I((size_t)G * rows);
      c->pv_all = F((size_t)G * G * rows); c->pi_all = I((size_t)G * G * rows);
      if (c->shard_mode == HSD_SHARD_NCCL) c->a_all = A((size_t)G * rows * n * es);
      if (cfg->accept_mode == HSD_STOCHASTIC) {
        const size_t rec = stoch_record_floats(T), vrows = (size_t)b * T;
        const size_t grow = c->shard_mode == HSD_SHARD_NCCL ? (size_t)G * vrows : vrows;
        c->sp_loc = F(grow * rec);
        c->sp_all = F((size_t)G * grow * rec);
        c->sh_lse = F(vrows);
        c->sh_tl = F(vrows * T);
        c->sh_gv = F(vrows * HSD_SHARD_KG);
        c->sh_gi = I(vrows * HSD_SHARD_KG);
        c->tt_all = I((size_t)G * vrows);
        c->rid_all = I((size_t)G * b);
      }
    }
    if (fail_alloc) { hsd_destroy(c); return HSD_ENOMEM; }
    if (cudaMallocHost(&c->h_pinned, sizeof(int32_t) * (size_t)b * (N + 2)) != cudaSuccess) c->h_pinned = nullptr;
  }
  CU(cudaStreamSynchronize(c->st));
  CU(cudaGetLastError());
  if (c->shard_mode == HSD_SHARD_NCCL) {
    std::string err;
    if (!shard_nccl_init(&c->comm, c->G, cfg->nccl_id, c->srank, err)) {
      fprintf(stderr, "hsd_init_model: %s\n", err.c_str());
      hsd_destroy(c);
      return HSD_ENCCL;
    }
  }
  *out = c;
  return HSD_OK;
}

hsd_status hsd_prefill(hsd_ctx* ctx, int32_t n_req, const int32_t* h_tokens, int32_t stride, const int32_t* h_lens,
                       int32_t* d_first) {
  if (!ctx) return HSD_EINVAL;
  Nvtx nv("hsd prefill");
  hsd_ctx* c = ctx;
  if (n_req < 1 || n_req > c->maxb) return fail(c, HSD_EINVAL, "n_req must be in [1, max_batch]");
  if (!h_tokens || !h_lens || stride < 1) return fail(c, HSD_EINVAL, "null prompt arrays");
  for (int r = 0; r < n_req; ++r) {
    if (h_lens[r] < 2 || h_lens[r] > stride || h_lens[r] > c->cfg.max_ctx)
      return fail(c, HSD_EINVAL, "prompt length must be in [2, min(stride, max_ctx)]");
    for (int i = 0; i < h_lens[r]; ++i)
      if (h_tokens[(size_t)r * stride + i] < 0 || h_tokens[(size_t)r * stride + i] >= c->V)
        return fail(c, HSD_EINVAL, "token outside [0, V) (contract violation)");
  }
  drop_graphs(c);
  c->b = n_req;
  const int n = c->n, N = c->N;
  CU(cudaMemsetAsync(c->step, 0, 4, c->st));
  CU(cudaMemsetAsync(c->step, 0, 4, c->st));
  // step counter starts at 1 for the first speculative step (0 = prefill)
  {
    int one = 1;
    CU(cudaMemcpyAsync(c->step, &one, 4, cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  std::vector<int32_t> ones(c->maxb, 1);
  CU(cudaMemcpyAsync(c->pt_n, ones.data(), 4 * n_req, cudaMemcpyHostToDevice, c->st));
  CU(cudaStreamSynchronize(c->st));
  for (int r = 0; r < n_req; ++r) {
    const hsd_status st = prefill_one(c, r, h_tokens + (size_t)r * stride, h_lens[r], d_first, c->cfg.req_offset + r);
    if (st != HSD_OK) return st;
  }
  CU(cudaStreamSynchronize(c->st));
  CU(cudaGetLastError());
  c->stage = 0;
  return HSD_OK;
}

// capacity contract (include/hsd.h): a step writes KV rows up to p + T - 1 and the
// tree's RoPE positions up to p + N; p itself grows by at most N + 1 per step
static hsd_status check_capacity(hsd_ctx* c) {
  // fusion off: the extra verify of the re-sampled tree starts up to N positions later
  const bool extra = (c->cfg.flags & HSD_FLAG_RESAMPLE) && !(c->cfg.flags & HSD_FLAG_FUSION);
  const int need = c->T + (extra ? c->N + 1 : 0);
  bool tight = false;
  for (int r = 0; r < c->b; ++r) tight |= c->p_hi[r] + need > c->max_pos;
  if (tight) {   // the bound assumes N + 1 tokens per step: refresh it from the device's p
    std::vector<int32_t> p(c->b);
    if (cudaStreamSynchronize(c->st) != cudaSuccess ||
        cudaMemcpy(p.data(), c->p, 4 * c->b, cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(c, HSD_ECUDA, "check_capacity: reading p");
    for (int r = 0; r < c->b; ++r) c->p_hi[r] = p[r];
  }
  for (int r = 0; r < c->b; ++r)
    if (c->p_hi[r] + need > c->max_pos)
      return fail(c, HSD_ESTATE, "context capacity exhausted: slot " + std::to_string(r) + " may hold " +
                                     std::to_string(c->p_hi[r]) + " committed tokens, a step needs " +
                                     std::to_string(c->T) + " more KV rows of " + std::to_string(c->max_pos));
  return HSD_OK;
}

hsd_status hsd_admit(hsd_ctx* ctx, int32_t slot, const int32_t* h_tokens, int32_t len, int32_t req_id,
                     int32_t* d_first) {
  if (!ctx) return HSD_EINVAL;
  hsd_ctx* c = ctx;
  if (c->b < 1) return fail(c, HSD_ESTATE, "hsd_admit before hsd_prefill");
  if (c->stage != 0) return fail(c, HSD_ESTATE, "hsd_admit in the middle of a staged step");
  if (slot < 0 || slot >= c->b) return fail(c, HSD_EINVAL, "slot must be in [0, batch)");
  if (!h_tokens || len < 2 || len > c->cfg.max_ctx) return fail(c, HSD_EINVAL, "prompt length must be in [2, max_ctx]");
  if (c->shard_mode == HSD_SHARD_NCCL) return fail(c, HSD_EUNSUP, "hsd_admit with the NCCL vocab-sharded head");
  for (int i = 0; i < len; ++i)
    if (h_tokens[i] < 0 || h_tokens[i] >= c->V) return fail(c, HSD_EINVAL, "token outside [0, V) (contract violation)");
  const int32_t one = 1;   // no pending re-sampled tree for the new request
  CU(cudaMemcpyAsync(c->pt_n + slot, &one, 4, cudaMemcpyHostToDevice, c->st));
  CU(cudaStreamSynchronize(c->st));
  if (req_id < 0) return fail(c, HSD_EINVAL, "req_id must be >= 0");
  const hsd_status st = prefill_one(c, slot, h_tokens, len, d_first, req_id);
  if (st != HSD_OK) return st;
  CU(cudaStreamSynchronize(c->st));
  CU(cudaGetLastError());
  return HSD_OK;
}

hsd_status hsd_set_block_table(hsd_ctx* ctx, const int32_t* h_table) {
  if (!ctx || !h_table) return fail(ctx, HSD_EINVAL, "null block table");
  hsd_ctx* c = ctx;
  if (c->stage != 0) return fail(c, HSD_ESTATE, "hsd_set_block_table in the middle of a staged step");
  const size_t n = (size_t)c->maxb * c->pages_per_req;
  std::vector<char> seen(n, 0);
  for (size_t i = 0; i < n; ++i) {
    const int32_t pg = h_table[i];
    if (pg < 0 || (size_t)pg >= n || seen[pg]) return fail(c, HSD_EINVAL, "block table is not a permutation of the pages");
    seen[pg] = 1;
  }
  CU(cudaMemcpyAsync(c->block_table, h_table, 4 * n, cudaMemcpyHostToDevice, c->st));
  CU(cudaStreamSynchronize(c->st));
  drop_graphs(c);
  return HSD_OK;
}

hsd_status hsd_set_plant(hsd_ctx* ctx, const int32_t* h_plant, int32_t stride) {
  if (!ctx || !h_plant || stride < 1) return fail(ctx, HSD_EINVAL, "bad plant array");
  hsd_ctx* c = ctx;
  if (c->b < 1) return fail(c, HSD_ESTATE, "hsd_set_plant needs hsd_prefill first");
  if (c->plant) {
    cudaFree(c->plant);
    c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), (void*)c->plant));
  }
  c->plant = (int32_t*)dalloc(c, sizeof(int32_t) * (size_t)c->b * stride);
  if (!c->plant) return fail(c, HSD_ENOMEM, "plant alloc");
  c->plant_stride = stride;
  CU(cudaMemcpyAsync(c->plant, h_plant, sizeof(int32_t) * (size_t)c->b * stride, cudaMemcpyHostToDevice, c->st));
  CU(cudaStreamSynchronize(c->st));
  drop_graphs(c);
  return HSD_OK;
}

static void fill_tree_view(hsd_ctx* c, hsd_tree_view* v) {
  if (!v) return;
  v->tok = c->t_tok; v->par = c->t_par; v->depth = c->t_depth; v->logjoint = c->t_lj; v->n = c->t_n;
  v->anc = c->t_anc; v->batch = c->b; v->t_max = c->T; v->anc_words = c->W;
}
static void fill_verify_view(hsd_ctx* c, hsd_verify_view* v) {
  if (!v) return;
  v->logits = c->shard_mode != HSD_SHARD_NONE ? nullptr : c->logits;   // sharded: no full rows
  v->argmax = c->argmax; v->hidden = c->Hver;
  v->batch = c->b; v->t_max = c->T; v->vocab = c->V; v->hidden_dim = c->n;
}

hsd_status hsd_build_tree(hsd_ctx* ctx, hsd_tree_view* out) {
  if (!ctx) return HSD_EINVAL;
  if (ctx->b < 1) return fail(ctx, HSD_ESTATE, "hsd_build_tree before hsd_prefill");
  { const hsd_status s = check_capacity(ctx); if (s != HSD_OK) return s; }
  { const hsd_status s = run_stage(ctx, 0, [&] { stage_build(ctx); }); if (s != HSD_OK) return s; }
  ctx->stage = 1;
  fill_tree_view(ctx, out);
  return HSD_OK;
}

hsd_status hsd_force_tree(hsd_ctx* ctx, const int32_t* h_tok, const int32_t* h_par, const int32_t* h_depth,
                          const int32_t* h_n) {
  if (!ctx || !h_tok || !h_par || !h_depth || !h_n) return fail(ctx, HSD_EINVAL, "null tree arrays");
  hsd_ctx* c = ctx;
  if (c->stage != 1) return fail(c, HSD_ESTATE, "hsd_force_tree must follow hsd_build_tree");
  const int T = c->T, W = c->W, b = c->b;
  std::vector<uint64_t> anc((size_t)b * T * W, 0);
  for (int r = 0; r < b; ++r) {
    int nn = h_n[r];
    if (nn < 1 || nn > T) return fail(c, HSD_EINVAL, "tree node count out of range");
    for (int s = 0; s < nn; ++s) {
      int pa = h_par[r * T + s];
      if ((s == 0) != (pa < 0) || pa >= s) return fail(c, HSD_EINVAL, "parents must precede children");
      if (h_tok[r * T + s] < 0 || h_tok[r * T + s] >= c->V) return fail(c, HSD_EINVAL, "token outside [0, V)");
      uint64_t* a = &anc[((size_t)r * T + s) * W];
      if (pa >= 0) std::memcpy(a, &anc[((size_t)r * T + pa) * W], W * 8);
      a[s >> 6] |= 1ull << (s & 63);
    }
  }
  CU(cudaMemcpyAsync(c->t_tok, h_tok, 4 * b * T, cudaMemcpyHostToDevice, c->st));
  CU(cudaMemcpyAsync(c->t_par, h_par, 4 * b * T, cudaMemcpyHostToDevice, c->st));
  CU(cudaMemcpyAsync(c->t_depth, h_depth, 4 * b * T, cudaMemcpyHostToDevice, c->st));
  CU(cudaMemcpyAsync(c->t_n, h_n, 4 * b, cudaMemcpyHostToDevice, c->st));
  CU(cudaMemcpyAsync(c->t_anc, anc.data(), 8 * anc.size(), cudaMemcpyHostToDevice, c->st));
  CU(cudaStreamSynchronize(c->st));
  return HSD_OK;
}

hsd_status hsd_verify_tree(hsd_ctx* ctx, hsd_verify_view* out) {
  if (!ctx) return HSD_EINVAL;
  if (ctx->stage != 1) return fail(ctx, HSD_ESTATE, "hsd_verify_tree requires hsd_build_tree");
  { const hsd_status s = run_stage(ctx, 1, [&] { stage_verify(ctx); }); if (s != HSD_OK) return s; }
  ctx->stage = 2;
  fill_verify_view(ctx, out);
  return HSD_OK;
}

hsd_status hsd_accept_and_compact(hsd_ctx* ctx, int32_t* d_emitted, int32_t* d_n_emitted) {
  if (!ctx) return HSD_EINVAL;
  if (ctx->stage != 2) return fail(ctx, HSD_ESTATE, "hsd_accept_and_compact requires hsd_verify_tree");
  { const hsd_status s = run_stage(ctx, 2, [&] { stage_accept(ctx, nullptr, nullptr); }); if (s != HSD_OK) return s; }
  if (d_emitted)
    CU(cudaMemcpyAsync(d_emitted, ctx->emitted, sizeof(int32_t) * ctx->b * (ctx->N + 1), cudaMemcpyDeviceToDevice, ctx->st));
  if (d_n_emitted) CU(cudaMemcpyAsync(d_n_emitted, ctx->n_emitted, sizeof(int32_t) * ctx->b, cudaMemcpyDeviceToDevice, ctx->st));
  for (int r = 0; r < ctx->b; ++r) ctx->p_hi[r] += ctx->N + 1;
  ctx->stage = 0;
  return HSD_OK;
}

hsd_status hsd_step(hsd_ctx* ctx, int32_t* d_emitted, int32_t* d_n_emitted) {
  if (!ctx) return HSD_EINVAL;
  Nvtx nv("hsd step");
  hsd_ctx* c = ctx;
  if (c->b < 1) return fail(c, HSD_ESTATE, "hsd_step before hsd_prefill");
  if (c->stage != 0) return fail(c, HSD_ESTATE, "hsd_step in the middle of a staged step");
  { const hsd_status s = check_capacity(c); if (s != HSD_OK) return s; }
  for (int r = 0; r < c->b; ++r) c->p_hi[r] += c->N + 1;
  if (c->prof_on) {
    // profiled steps run eagerly so every launch is bracketed by CUDA events
    stage_build(c); stage_verify(c); stage_accept(c, d_emitted, d_n_emitted);
    CU(cudaGetLastError());
    if (!c->nccl_err.empty()) return fail(c, HSD_ENCCL, c->nccl_err);
    return HSD_OK;
  }
  if (!c->graph) {
    if (c->st == nullptr) {
      // graphs cannot capture the legacy stream: run eagerly
      stage_build(c); stage_verify(c); stage_accept(c, nullptr, nullptr);
      CU(cudaGetLastError());
      if (!c->nccl_err.empty()) return fail(c, HSD_ENCCL, c->nccl_err);
    } else {
      int64_t before = g_hsd_launches;
      cudaGraph_t g;
      CU(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
      c->capturing = true;
      stage_build(c); stage_verify(c); stage_accept(c, nullptr, nullptr);
      c->capturing = false;
      CU(cudaStreamEndCapture(c->st, &g));
      if (!c->nccl_err.empty()) return fail(c, HSD_ENCCL, c->nccl_err);
      c->graph_kernels = g_hsd_launches - before;
      g_hsd_launches = before;  // counted per replay instead
      CU(cudaGraphInstantiate(&c->graph, g, 0));
      cudaGraphDestroy(g);
    }
  }
  if (c->graph) {
    CU(cudaGraphLaunch(c->graph, c->st));
    c->graph_replays++;
  }
  if (d_emitted) CU(cudaMemcpyAsync(d_emitted, c->emitted, 4 * c->b * (c->N + 1), cudaMemcpyDeviceToDevice, c->st));
  if (d_n_emitted) CU(cudaMemcpyAsync(d_n_emitted, c->n_emitted, 4 * c->b, cudaMemcpyDeviceToDevice, c->st));
  return HSD_OK;
}

hsd_status hsd_step_host(hsd_ctx* ctx, int32_t* h_emitted, int32_t* h_n_emitted) {
  hsd_status s = hsd_step(ctx, nullptr, nullptr);
  if (s != HSD_OK) return s;
  hsd_ctx* c = ctx;
  const int b = c->b, N = c->N;
  if (c->h_pinned) {
    CU(cudaMemcpyAsync(c->h_pinned, c->emitted, 4 * b * (N + 1), cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(c->h_pinned + b * (N + 1), c->n_emitted, 4 * b, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    if (h_emitted) std::memcpy(h_emitted, c->h_pinned, 4 * b * (N + 1));
    if (h_n_emitted) std::memcpy(h_n_emitted, c->h_pinned + b * (N + 1), 4 * b);
  } else {
    if (h_emitted) CU(cudaMemcpyAsync(h_emitted, c->emitted, 4 * b * (N + 1), cudaMemcpyDeviceToHost, c->st));
    if (h_n_emitted) CU(cudaMemcpyAsync(h_n_emitted, c->n_emitted, 4 * b, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
  }
  return HSD_OK;
}

hsd_status hsd_sync(hsd_ctx* ctx) {
  if (!ctx) return HSD_EINVAL;
  CU(cudaStreamSynchronize(ctx->st));
  CU(cudaGetLastError());
  int e = 0;
  CU(cudaMemcpy(&e, ctx->err, 4, cudaMemcpyDeviceToHost));
  if (e) {
    cudaMemset(ctx->err, 0, 4);
    return fail(ctx, HSD_EDEVICE, "device-side violation flag " + std::to_string(e));
  }
  return HSD_OK;
}

hsd_status hsd_get_tensor(hsd_ctx* ctx, const char* name, hsd_tensor* out) {
  if (!ctx || !name || !out) return HSD_EINVAL;
  hsd_ctx* c = ctx;
  const int b = std::max(c->b, 1), T = c->T, N = c->N, n = c->n, Br1 = c->Br + 1;
  const int adt = c->dt == DT_BF16 ? 1 : 0;
  auto set = [&](void* p, int dt, std::initializer_list<int64_t> dims) {
    out->ptr = p; out->dtype = dt; out->ndim = (int)dims.size();
    int i = 0;
    for (auto d : dims) out->dims[i++] = d;
    return HSD_OK;
  };
  std::string s(name);
  if (s == "p") return set(c->p, 2, {b});
  if (s == "root_tok") return set(c->root_tok, 2, {b});
  if (s == "step") return set(c->step, 2, {1});
  if (s == "n_pend") return set(c->n_pend, 2, {b});
  if (s == "pend_tok") return set(c->pend_tok, 2, {b, N + 1});
  if (s == "pend_H") return set(c->pend_H, 0, {b, N + 1, n});
  if (s == "chain") return set(c->chain, 0, {b, N, n});
  if (s == "draft_logits") return set(c->draft_logits, 0, {b, N, c->V});
  if (s == "tree_tok") return set(c->t_tok, 2, {b, T});
  if (s == "tree_par") return set(c->t_par, 2, {b, T});
  if (s == "tree_depth") return set(c->t_depth, 2, {b, T});
  if (s == "tree_lj") return set(c->t_lj, 0, {b, T});
  if (s == "tree_n") return set(c->t_n, 2, {b});
  if (s == "tree_anc") return set(c->t_anc, 3, {b, T, c->W});
  if (s == "pt_n") return set(c->pt_n, 2, {b});
  if (s == "pt_tok") return set(c->pt_tok, 2, {b, Br1});
  if (s == "pt_par") return set(c->pt_par, 2, {b, Br1});
  if (s == "pt_depth") return set(c->pt_depth, 2, {b, Br1});
  if (s == "pt_lj") return set(c->pt_lj, 0, {b, Br1});
  if (s == "verify_logits") return set(c->logits, 0, {b, T, c->V});
  if (s == "shard_lse" && c->sh_lse) return set(c->sh_lse, 0, {b, T});
  if (s == "shard_tl" && c->sh_tl) return set(c->sh_tl, 0, {b, T, T});
  if (s == "shard_gv" && c->sh_gv) return set(c->sh_gv, 0, {b, T, HSD_SHARD_KG});
  if (s == "shard_gi" && c->sh_gi) return set(c->sh_gi, 2, {b, T, HSD_SHARD_KG});
  if (s == "verify_argmax") return set(c->argmax, 2, {b, T});
  if (s == "verify_hidden") return set(c->Hver, 0, {b, T, n});
  if (s == "acc_n") return set(c->acc_n, 2, {b});
  if (s == "acc_slots") return set(c->acc_slots, 2, {b, N});
  if (s == "bonus") return set(c->bonus, 2, {b});
  if (s == "emitted") return set(c->emitted, 2, {b, N + 1});
  if (s == "n_emitted") return set(c->n_emitted, 2, {b});
  if (s == "table") return set(c->table, c->table_scale ? 4 : adt, {c->Vh, c->Vh});
  if (s == "table_scale" && c->table_scale) return set(c->table_scale, 0, {c->Vh});
  if (s == "embed") return set(c->embed, adt, {c->V, n});
  if (s == "head") return set(c->head, adt, {c->V, n});
  if (s == "block_table") return set(c->block_table, 2, {c->maxb, c->pages_per_req});
  if (s == "kv") return set(c->kv_t, adt, {std::max(1, c->L), c->maxb * c->pages_per_req, 2, (int64_t)c->Hkv * c->page_size * c->hd});
  if (s == "kv_draft") return set(c->kv_d, adt, {1, c->maxb * c->pages_per_req, 2, (int64_t)c->Hkv * c->page_size * c->hd});
  extern unsigned long long* g_attn_trace;
  if (s == "attn_trace" && g_attn_trace) return set(g_attn_trace, 3, {256});
  extern unsigned long long* g_tree_trace;
  if (s == "tree_trace" && g_tree_trace) return set(g_tree_trace, 3, {64});
  if (s == "layer0_wqkv" && c->L > 0) return set(c->layers[0].wqkv, adt, {c->qkvd, n});
  // target layer weights by name, e.g. "layer7_wo" ([out, in] row-major, nn.Linear layout;
  // gate/up rows interleaved in GU_GROUP = 16-row groups, see launch_swiglu)
  if (s.rfind("layer", 0) == 0) {
    const size_t us = s.find('_');
    if (us != std::string::npos) {
      const int l = atoi(s.substr(5, us - 5).c_str());
      const std::string part = s.substr(us + 1);
      if (l >= 0 && l < c->L) {
        const LayerW& w = c->layers[l];
        if (part == "wqkv") return set(w.wqkv, adt, {c->qkvd, n});
        if (part == "wo") return set(w.wo, adt, {n, c->qd});
        if (part == "wgu") return set(w.wgu, adt, {2 * (int64_t)c->f, n});
        if (part == "wd") return set(w.wd, adt, {n, c->f});
      }
    }
  }
  return fail(c, HSD_EINVAL, "unknown tensor name " + s);
}

hsd_status hsd_debug_gemm(const void* A, int32_t lda, const void* W, int32_t ldw, float* C, int32_t ldc,
                          int32_t M, int32_t N, int32_t K, int32_t accumulate, int32_t dtype, int32_t use_tc,
                          void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (use_tc == 2) {   // data-parallel gate/up GEMM with fused SwiGLU: C is bf16 H [M, N/2], ld = ldc
    if (dtype != 1 || !gemm_tc_supported(M, N, K, lda, ldw)) return HSD_EUNSUP;
    const int k = gemm_tc_swiglu_bf16((const bf16*)A, lda, (const bf16*)W, ldw, (bf16*)C, ldc, M, N, K, st);
    if (k == 0) return HSD_EUNSUP;
    g_hsd_launches += k;
  } else if (use_tc) {
    if (dtype != 1 || !gemm_tc_supported(M, N, K, lda, ldw)) return HSD_EUNSUP;
    g_hsd_launches += gemm_tc_bf16((const bf16*)A, lda, (const bf16*)W, ldw, C, ldc, M, N, K, accumulate != 0, st);
    extern unsigned long long* g_gemm_trace;
    if (g_gemm_trace) {   // debug (HSD_GEMM_TRACE): phase stamps of this launch, us from CTA 0's start
      unsigned long long t[32];
      cudaStreamSynchronize(st);
      cudaMemcpy(t, g_gemm_trace, sizeof(t), cudaMemcpyDeviceToHost);
      fprintf(stderr, "gemm_trace M=%d N=%d K=%d", M, N, K);
      for (int i = 0; i < 32; ++i)
        if (i % 16 < 12) fprintf(stderr, " %.2f", t[i] ? (double)(long long)(t[i] - t[0]) / 1e3 : -1.0);
      fprintf(stderr, "\n");
    }
  } else {
    gemm_simt(A, lda, W, ldw, dtype == 1 ? DT_BF16 : DT_F32, C, ldc, M, N, K, accumulate != 0, st);
    g_hsd_launches += 1;
  }
  return cudaGetLastError() == cudaSuccess ? HSD_OK : HSD_ECUDA;
}

hsd_status hsd_debug_gumbel(const float* d_logits, int32_t ld, int32_t V, float temperature, uint64_t seed,
                            int32_t req, int32_t step, int32_t n, const int32_t* d_row, const int32_t* d_slot,
                            int32_t* d_out, void* stream) {
  if (!d_logits || !d_row || !d_slot || !d_out || V < 1 || ld < V || n < 0 || !(temperature > 0.f)) return HSD_EINVAL;
  launch_gumbel_debug(d_logits, ld, V, temperature, (uint32_t)seed, req, step, n, d_row, d_slot, d_out,
                      (cudaStream_t)stream);
  g_hsd_launches += 1;
  return cudaGetLastError() == cudaSuccess ? HSD_OK : HSD_ECUDA;
}

hsd_status hsd_profile(hsd_ctx* ctx, int enable) {
  if (!ctx) return HSD_EINVAL;
  prof_collect(ctx);
  if (enable) {
    for (int i = 0; i < P_NCAT; ++i) { ctx->prof_ms[i] = 0; ctx->prof_bytes[i] = 0; ctx->prof_flops[i] = 0; ctx->prof_n[i] = 0; }
  }
  ctx->prof_on = enable != 0;
  return HSD_OK;
}

hsd_status hsd_profile_read(hsd_ctx* ctx, const char* category, double* total_ms, int64_t* launches,
                            double* bytes, double* flops) {
  if (!ctx || !category) return HSD_EINVAL;
  prof_collect(ctx);
  for (int i = 0; i < P_NCAT; ++i) {
    if (std::string(category) == kProfNames[i]) {
      if (total_ms) *total_ms = ctx->prof_ms[i];
      if (launches) *launches = ctx->prof_n[i];
      if (bytes) *bytes = ctx->prof_bytes[i];
      if (flops) *flops = ctx->prof_flops[i];
      return HSD_OK;
    }
  }
  return fail(ctx, HSD_EINVAL, std::string("unknown profile category ") + category);
}

hsd_status hsd_kstamp(hsd_ctx* ctx, int enable) {
  if (!ctx) return HSD_EINVAL;
  hsd_ctx* c = ctx;
  if (c->stage != 0) return fail(c, HSD_ESTATE, "hsd_kstamp in the middle of a staged step");
  const size_t n = (size_t)2 * KST_SLOTS * KST_MAXID;
  if (enable && !c->kst_buf) {
    c->kst_buf = (unsigned long long*)dalloc(c, n * 8);
    if (!c->kst_buf) return fail(c, HSD_ENOMEM, "kstamp buffer");
  }
  if (enable) {
    CU(cudaMemsetAsync(c->kst_buf, 0xff, n / 2 * 8, c->st));            // entry minima
    CU(cudaMemsetAsync(c->kst_buf + n / 2, 0, n / 2 * 8, c->st));       // exit maxima
    CU(cudaStreamSynchronize(c->st));
  }
  c->kst_on = enable != 0;
  c->kst_n = 0;
  c->kst_bytes.clear();
  c->kst_flops.clear();
  c->kst_cat.clear();
  drop_graphs(c);   // the next hsd_step recaptures (with or without stamps)
  return HSD_OK;
}

static hsd_status kstamp_read_cat(hsd_ctx* ctx, int want_cat, double* avg_us, int64_t* samples,
                                  double* bytes_per_launch, double* flops_per_launch) {
  if (!ctx) return HSD_EINVAL;
  hsd_ctx* c = ctx;
  if (!c->kst_buf || c->kst_n == 0) return fail(c, HSD_ESTATE, "hsd_kstamp_read: no stamped replay");
  CU(cudaStreamSynchronize(c->st));
  const size_t n = (size_t)KST_SLOTS * KST_MAXID;
  std::vector<unsigned long long> h(2 * n);
  CU(cudaMemcpy(h.data(), c->kst_buf, 2 * n * 8, cudaMemcpyDeviceToHost));
  double sum = 0.0;
  int64_t cnt = 0;
  for (size_t slot = 0; slot < (size_t)KST_SLOTS; ++slot)
    for (int id = 0; id < c->kst_n; ++id) {
      if (c->kst_cat[id] != want_cat) continue;
      const unsigned long long a = h[slot * KST_MAXID + id], b = h[n + slot * KST_MAXID + id];
      if (a != ~0ull && b != 0ull && b > a) { sum += (double)(b - a); ++cnt; }
    }
  if (getenv("HSD_KST_DUMP")) {   // debug: per-launch durations of the first stamped slot
    for (size_t slot = 0; slot < (size_t)KST_SLOTS; ++slot) {
      if (h[slot * KST_MAXID] == ~0ull) continue;
      fprintf(stderr, "kstamp slot %zu:", slot);
      for (int id = 0; id < c->kst_n && id < 16; ++id) {
        const unsigned long long a = h[slot * KST_MAXID + id], b = h[n + slot * KST_MAXID + id];
        fprintf(stderr, " %d:%.1f(+%.1f)", id, a != ~0ull && b ? (double)(long long)(b - a) / 1e3 : -1.0,
                id > 0 && a != ~0ull ? (double)(long long)(a - h[slot * KST_MAXID + id - 1]) / 1e3 : 0.0);
      }
      fprintf(stderr, "\n");
      break;
    }
  }
  double by = 0.0, fl = 0.0;
  int nid = 0;
  for (int id = 0; id < c->kst_n; ++id)
    if (c->kst_cat[id] == want_cat) { by += c->kst_bytes[id]; fl += c->kst_flops[id]; ++nid; }
  if (avg_us) *avg_us = cnt ? sum / cnt / 1e3 : 0.0;
  if (samples) *samples = cnt;
  if (bytes_per_launch) *bytes_per_launch = nid ? by / nid : 0.0;
  if (flops_per_launch) *flops_per_launch = nid ? fl / nid : 0.0;
  return HSD_OK;
}

hsd_status hsd_kstamp_read(hsd_ctx* ctx, double* avg_us, int64_t* samples, double* bytes_per_launch,
                           double* flops_per_launch) {
  return kstamp_read_cat(ctx, P_GEMM_VERIFY, avg_us, samples, bytes_per_launch, flops_per_launch);
}

hsd_status hsd_kstamp_read_attention(hsd_ctx* ctx, double* avg_us, int64_t* samples) {
  return kstamp_read_cat(ctx, P_ATTN_VERIFY, avg_us, samples, nullptr, nullptr);
}

hsd_status hsd_destroy(hsd_ctx* ctx) {
  if (!ctx) return HSD_EINVAL;
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  else cudaDeviceSynchronize();
  drop_graphs(ctx);
  prof_collect(ctx);
  shard_nccl_destroy(ctx->comm);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  delete ctx;
  return HSD_OK;
}

}  // extern "C"
