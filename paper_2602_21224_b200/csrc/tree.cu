// tree.cu -- K-TREE: token-info tree construction on the device.
//
//  Alg. 1 BuildSubtree: for each step i and each frontier
//    node u: v = l_i + r(u.token) (token-info bias row),
//    lse = logsumexp(v), children = top-k of v with log p = v - lse and
//    logjoint = logjoint(u) + log p; frontier = TopkByJointProb(Q_next, k).
//  Prune to the top-B nodes by joint probability.
//  Verification fusion: union with the pending re-sampled tree.
//  Linearise depth-major + ancestor bitmasks for tree attention.
//  Alg. 2: the same builder rooted at the bonus token over
//    the leftover logit rows.
// Tie rules = DESIGN.md R8. One CTA of 1024 threads per request; every vocab
// pass is a coalesced sweep of the logit row plus the table row with per-thread
// online (max, sum-exp) and a per-thread top-8 list, merged warp-wise.
#include <cooperative_groups.h>
#include "kernels.cuh"
#include "tree.cuh"

namespace cg = cooperative_groups;

namespace {
constexpr int NT = 1024;
constexpr int CL = 8;       // CTAs per request (one thread-block cluster)
constexpr int KMAX = 8;
constexpr int MAXN = 256;
constexpr int MAXW = MAXN / 64;

struct NodesSm {
  int tok[MAXN], par[MAXN], depth[MAXN];
  float lj[MAXN];
  int n;
};

// (v desc, token asc): token = perm[j] (identity when perm == null); an empty
// entry (j < 0) ranks after every real one. Strict order.
HSD_DEV int tok_of(int j, const int32_t* perm) { return j < 0 ? 0x7fffffff : (perm ? perm[j] : j); }
HSD_DEV bool better_j(float v, int j, float w, int i, const int32_t* perm) {
  if (v != w) return v > w;
  return tok_of(j, perm) < tok_of(i, perm);
}
// strict total order across lanes (lane id as the last key)
HSD_DEV bool beats(float v, int j, int l, float w, int i, int m, const int32_t* perm) {
  if (v != w) return v > w;
  int a = tok_of(j, perm), b = tok_of(i, perm);
  if (a != b) return a < b;
  return l < m;
}

struct Top {
  float v[KMAX];
  int j[KMAX];
};

HSD_DEV void top_init(Top& t) {
#pragma unroll
  for (int s = 0; s < KMAX; ++s) { t.v[s] = -INFINITY; t.j[s] = -1; }
}
HSD_DEV void top_insert(Top& t, float v, int j, const int32_t* perm) {
  if (!better_j(v, j, t.v[KMAX - 1], t.j[KMAX - 1], perm)) return;
  t.v[KMAX - 1] = v; t.j[KMAX - 1] = j;
#pragma unroll
  for (int s = KMAX - 1; s > 0; --s) {
    if (better_j(t.v[s], t.j[s], t.v[s - 1], t.j[s - 1], perm)) {
      float tv = t.v[s]; t.v[s] = t.v[s - 1]; t.v[s - 1] = tv;
      int tj = t.j[s]; t.j[s] = t.j[s - 1]; t.j[s - 1] = tj;
    }
  }
}

// Partial result of one CTA's sweep over its vocab slice for one frontier node:
// online (max, sum-exp) and the slice's top-k (v, j) sorted by (v desc, token asc).
struct Partial {
  float m, s;
  float v[KMAX];
  int j[KMAX];
};

// One CTA-wide sweep: v_j = L[j] + bias[j] over j in [lo, hi) (bias only for hot
// columns j < Vh). Thread 0 returns the CTA partial in *out.
template <typename TT>
HSD_DEV void vocab_pass(const float* __restrict__ Lrow, const TT* __restrict__ bias, int lo, int hi, int Vh, int k,
                        const int32_t* perm, Partial* out, float* red_f, int* red_i) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = NT / 32;
  float m = -INFINITY, s = 0.f;
  Top t;
  top_init(t);
  for (int j = lo + threadIdx.x; j < hi; j += NT) {
    float v = Lrow[j];
    if (bias != nullptr && j < Vh) v += to_f32(bias[j]);
    if (v > m) { s = s * expf(m - v) + 1.f; m = v; }
    else s += expf(v - m);
    top_insert(t, v, j, perm);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
    float nm = fmaxf(m, om);
    s = (m == -INFINITY ? 0.f : s * expf(m - nm)) + (om == -INFINITY ? 0.f : os * expf(om - nm));
    m = nm;
  }
  // warp top-k: k rounds of argmax over the lanes' list heads
  int head = 0;
  float wv[KMAX];
  int wj[KMAX];
  for (int r = 0; r < k; ++r) {
    float hv = -INFINITY;
    int hj = -1;
#pragma unroll
    for (int q = 0; q < KMAX; ++q)
      if (q == head) { hv = t.v[q]; hj = t.j[q]; }
    float bv = hv;
    int bj = hj, bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oj = __shfl_xor_sync(0xffffffffu, bj, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (beats(ov, oj, ol, bv, bj, bl, perm)) { bv = ov; bj = oj; bl = ol; }
    }
    wv[r] = bv; wj[r] = bj;
    if (lane == bl) head++;
  }
  __syncthreads();
  if (lane == 0) {
    red_f[w * 2] = m; red_f[w * 2 + 1] = s;
    for (int r = 0; r < k; ++r) { red_f[64 + w * KMAX + r] = wv[r]; red_i[w * KMAX + r] = wj[r]; }
  }
  __syncthreads();
  if (w == 0) {
    float mm = lane < nw ? red_f[lane * 2] : -INFINITY, ss = lane < nw ? red_f[lane * 2 + 1] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float om = __shfl_xor_sync(0xffffffffu, mm, o), os = __shfl_xor_sync(0xffffffffu, ss, o);
      float nm = fmaxf(mm, om);
      ss = (mm == -INFINITY ? 0.f : ss * expf(mm - nm)) + (om == -INFINITY ? 0.f : os * expf(om - nm));
      mm = nm;
    }
    int hd = 0;
    for (int r = 0; r < k; ++r) {
      float hv = (lane < nw && hd < k) ? red_f[64 + lane * KMAX + hd] : -INFINITY;
      int hj = (lane < nw && hd < k) ? red_i[lane * KMAX + hd] : -1;
      float bv = hv;
      int bj = hj, bl = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oj = __shfl_xor_sync(0xffffffffu, bj, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (beats(ov, oj, ol, bv, bj, bl, perm)) { bv = ov; bj = oj; bl = ol; }
      }
      if (lane == 0) { out->v[r] = bv; out->j[r] = bj; }
      if (lane == bl) hd++;
    }
    if (lane == 0) { out->m = mm; out->s = ss; }
  }
  __syncthreads();
}

// Alg. 1 BuildSubtree on a thread-block cluster of CL CTAs: every CTA sweeps its
// vocab slice for every frontier node and stores its Partial in the LEADER's
// shared memory (DSMEM); the leader merges (exact (max, sum-exp) combination and
// top-k over the CL sorted lists), appends the children in frontier order and
// selects the next frontier (TopkByJointProb). Node arrays live in the leader.
struct ClusterSm {
  Partial part[KMAX][CL];
  int Q[KMAX], Qtok[KMAX], nq;
};

HSD_DEV void build_subtree(const TreeParams& P, int req, int row0, int steps, int root_tok, NodesSm& nd,
                           ClusterSm& cs, float* red_f, int* red_i) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  ClusterSm* lead = cluster.map_shared_rank(&cs, 0);
  __shared__ int qtok_local[KMAX], nq_local;
  __shared__ Partial mine;
  if (rank == 0 && threadIdx.x == 0) {
    nd.tok[0] = root_tok; nd.par[0] = -1; nd.depth[0] = 0; nd.lj[0] = 0.f; nd.n = 1;
    cs.Q[0] = 0; cs.Qtok[0] = root_tok; cs.nq = 1;
  }
  cluster.sync();
  const int per = (P.V + CL - 1) / CL;
  const int lo = min(P.V, rank * per), hi = min(P.V, lo + per);
  for (int i = 0; i < steps; ++i) {
    if (threadIdx.x == 0) {
      nq_local = lead->nq;
      for (int q = 0; q < KMAX; ++q) qtok_local[q] = lead->Qtok[q];
    }
    __syncthreads();
    const float* Lrow = P.L + ((size_t)req * P.N + row0 + i) * P.V;
    for (int qi = 0; qi < nq_local; ++qi) {
      const int tok = qtok_local[qi];
      const int rk = P.rank_of ? P.rank_of[tok] : tok;
      const bool has_bias = !P.zero_table && rk < P.Vh;
      if (P.tdt == DT_F32)
        vocab_pass<float>(Lrow, has_bias ? (const float*)P.table + (size_t)rk * P.Vh : nullptr, lo, hi, P.Vh, P.k,
                          P.perm, &mine, red_f, red_i);
      else
        vocab_pass<bf16>(Lrow, has_bias ? (const bf16*)P.table + (size_t)rk * P.Vh : nullptr, lo, hi, P.Vh, P.k,
                         P.perm, &mine, red_f, red_i);
      if (threadIdx.x == 0) lead->part[qi][rank] = mine;
      __syncthreads();
    }
    cluster.sync();
    if (rank == 0) {
      const int start = nd.n;
      // one thread per frontier node: merge the CL partials, append k children
      if (threadIdx.x < cs.nq) {
        const int qi = threadIdx.x, u = cs.Q[qi];
        float M = -INFINITY;
        for (int c = 0; c < CL; ++c) M = fmaxf(M, cs.part[qi][c].m);
        float S = 0.f;
        for (int c = 0; c < CL; ++c)
          if (cs.part[qi][c].m != -INFINITY) S += cs.part[qi][c].s * expf(cs.part[qi][c].m - M);
        const float lse = M + logf(S);
        int hd[CL];
        for (int c = 0; c < CL; ++c) hd[c] = 0;
        for (int r = 0; r < P.k; ++r) {
          int bc = -1;
          for (int c = 0; c < CL; ++c) {
            if (hd[c] >= P.k) continue;
            const float v = cs.part[qi][c].v[hd[c]];
            const int j = cs.part[qi][c].j[hd[c]];
            if (j < 0) continue;
            if (bc < 0 || better_j(v, j, cs.part[qi][bc].v[hd[bc]], cs.part[qi][bc].j[hd[bc]], P.perm)) bc = c;
          }
          const int n = start + qi * P.k + r;
          const float v = cs.part[qi][bc].v[hd[bc]];
          const int j = cs.part[qi][bc].j[hd[bc]];
          hd[bc]++;
          nd.tok[n] = P.perm ? P.perm[j] : j;
          nd.par[n] = u;
          nd.depth[n] = nd.depth[u] + 1;
          nd.lj[n] = nd.lj[u] + (v - lse);
        }
      }
      __syncthreads();
      // TopkByJointProb(Q_next, k): joint desc, token asc, parent creation index asc
      if (threadIdx.x == 0) {
        const int cnt_new = cs.nq * P.k;
        nd.n = start + cnt_new;
        int cnt = 0;
        bool used[KMAX * KMAX];
        for (int c = 0; c < cnt_new; ++c) used[c] = false;
        for (int r = 0; r < P.k && r < cnt_new; ++r) {
          int best = -1;
          for (int c = start; c < nd.n; ++c) {
            if (used[c - start]) continue;
            if (best < 0 || nd.lj[c] > nd.lj[best] ||
                (nd.lj[c] == nd.lj[best] &&
                 (nd.tok[c] < nd.tok[best] || (nd.tok[c] == nd.tok[best] && nd.par[c] < nd.par[best]))))
              best = c;
          }
          used[best - start] = true;
          cs.Q[cnt] = best;
          cs.Qtok[cnt] = nd.tok[best];
          cnt++;
        }
        cs.nq = cnt;
      }
      __syncthreads();
    }
    cluster.sync();
  }
}

// keep the top-`keep` non-root nodes (joint desc, depth asc, token asc, parent asc),
// compacted in creation order.
HSD_DEV void prune_nodes(NodesSm& nd, int keep, NodesSm& tmp) {
  __shared__ int flag[MAXN], newidx[MAXN];
  int n = nd.n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int f = 1;
    if (i > 0) {
      int c = 0;
      for (int j = 1; j < n; ++j) {
        bool less = nd.lj[j] > nd.lj[i] ||
                    (nd.lj[j] == nd.lj[i] &&
                     (nd.depth[j] < nd.depth[i] ||
                      (nd.depth[j] == nd.depth[i] &&
                       (nd.tok[j] < nd.tok[i] || (nd.tok[j] == nd.tok[i] && nd.par[j] < nd.par[i])))));
        c += less;
      }
      f = c < keep;
    }
    flag[i] = f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int i = 0; i < n; ++i) { newidx[i] = flag[i] ? c : -1; c += flag[i]; }
    tmp.n = c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!flag[i]) continue;
    int t = newidx[i];
    tmp.tok[t] = nd.tok[i];
    tmp.par[t] = nd.par[i] >= 0 ? newidx[nd.par[i]] : -1;
    tmp.depth[t] = nd.depth[i];
    tmp.lj[t] = nd.lj[i];
  }
  __syncthreads();
  int n2 = tmp.n;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    nd.tok[i] = tmp.tok[i]; nd.par[i] = tmp.par[i]; nd.depth[i] = tmp.depth[i]; nd.lj[i] = tmp.lj[i];
  }
  if (threadIdx.x == 0) nd.n = n2;
  __syncthreads();
}

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT) tree_kernel(TreeParams P, int mode) {
  pdl_wait();
  pdl_trigger();
  __shared__ NodesSm nd, tmp;
  __shared__ ClusterSm cs;
  __shared__ float red_f[64 + 32 * KMAX];
  __shared__ int red_i[32 * KMAX];
  __shared__ int slot_of[MAXN], maxdepth;
  __shared__ uint64_t anc[MAXN][MAXW];
  const int req = blockIdx.x / CL;
  const bool leader = cg::this_cluster().block_rank() == 0;
  const int Br1 = P.Br + 1;

  if (mode == TREE_MODE_RESAMPLE) {
    // Alg. 2: if N_remain = N - m - 1 > r build from the bonus over rows m+1..N-1
    int m = P.acc_n[req];
    int bonus = P.bonus[req];
    int n_remain = P.N - m - 1;
    if (P.resample && n_remain > P.r && n_remain > 0) {
      build_subtree(P, req, m + 1, n_remain, bonus, nd, cs, red_f, red_i);
      if (!leader) return;
      prune_nodes(nd, P.Br, tmp);
    } else {
      if (!leader) return;
      if (threadIdx.x == 0) {
        nd.tok[0] = bonus; nd.par[0] = -1; nd.depth[0] = 0; nd.lj[0] = 0.f; nd.n = 1;
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < Br1; i += blockDim.x) {
      bool ok = i < nd.n;
      P.pt_tok[req * Br1 + i] = ok ? nd.tok[i] : -1;
      P.pt_par[req * Br1 + i] = ok ? nd.par[i] : -1;
      P.pt_depth[req * Br1 + i] = ok ? nd.depth[i] : -1;
      P.pt_lj[req * Br1 + i] = ok ? nd.lj[i] : -INFINITY;
    }
    if (threadIdx.x == 0) P.pt_n[req] = nd.n;
    return;
  }

  // ---- fresh tree: Alg. 1 over all N rows from the root (last committed token)
  const int root = P.root_tok[req];
  build_subtree(P, req, 0, P.N, root, nd, cs, red_f, red_i);
  if (!leader) return;
  prune_nodes(nd, P.B, tmp);
  // ---- verification fusion with the pending re-sampled tree
  int pn = P.pt_n[req];
  if (P.fusion && pn > 1) {
    if (threadIdx.x == 0) {
      int map[MAXN];
      if (P.pt_tok[req * Br1] != root) atomicOr(P.err, DEV_ERR_BAD_TREE);
      map[0] = 0;
      for (int j = 1; j < pn && j < MAXN; ++j) {
        int ptok = P.pt_tok[req * Br1 + j];
        int fpar = map[P.pt_par[req * Br1 + j]];
        float plj = P.pt_lj[req * Br1 + j];
        int hit = -1;
        for (int i = 1; i < nd.n; ++i)
          if (nd.par[i] == fpar && nd.tok[i] == ptok) { hit = i; break; }
        if (hit >= 0) {
          if (plj > nd.lj[hit]) nd.lj[hit] = plj;
          map[j] = hit;
        } else if (nd.n < MAXN) {
          int n = nd.n;
          nd.tok[n] = ptok; nd.par[n] = fpar; nd.depth[n] = nd.depth[fpar] + 1; nd.lj[n] = plj;
          map[j] = n;
          nd.n = n + 1;
        }
      }
    }
    __syncthreads();
    prune_nodes(nd, P.B + P.Br, tmp);
  }
  // ---- linearise: BFS, siblings by (joint desc, token asc); level by level
  const int n = nd.n;
  if (threadIdx.x == 0) {
    int md = 0;
    for (int i = 0; i < n; ++i) md = max(md, nd.depth[i]);
    maxdepth = md;
    slot_of[0] = 0;
    for (int w = 0; w < MAXW; ++w) anc[0][w] = 0ull;
    anc[0][0] = 1ull;
  }
  __syncthreads();
  int offset = 1;
  for (int d = 1; d <= maxdepth; ++d) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (nd.depth[i] != d) continue;
      int c = 0;
      int pi = slot_of[nd.par[i]];
      for (int j = 0; j < n; ++j) {
        if (nd.depth[j] != d) continue;
        int pj = slot_of[nd.par[j]];
        bool less = pj < pi || (pj == pi && (nd.lj[j] > nd.lj[i] || (nd.lj[j] == nd.lj[i] && nd.tok[j] < nd.tok[i])));
        c += less;
      }
      slot_of[i] = offset + c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (nd.depth[i] != d) continue;
      int s = slot_of[i], ps = slot_of[nd.par[i]];
      for (int w = 0; w < MAXW; ++w) anc[s][w] = anc[ps][w];
      anc[s][s >> 6] |= 1ull << (s & 63);
    }
    int cnt = 0;
    for (int i = 0; i < n; ++i) cnt += nd.depth[i] == d;
    offset += cnt;
    __syncthreads();
  }
  // ---- write the linearised tree
  const int T = P.t_max;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int s = slot_of[i];
    P.t_tok[req * T + s] = nd.tok[i];
    P.t_par[req * T + s] = nd.par[i] >= 0 ? slot_of[nd.par[i]] : -1;
    P.t_depth[req * T + s] = nd.depth[i];
    P.t_lj[req * T + s] = nd.lj[i];
  }
  for (int s = n + threadIdx.x; s < T; s += blockDim.x) {
    P.t_tok[req * T + s] = 0; P.t_par[req * T + s] = -1; P.t_depth[req * T + s] = -1;
    P.t_lj[req * T + s] = -INFINITY;
  }
  for (int i = threadIdx.x; i < T * P.anc_words; i += blockDim.x) {
    int s = i / P.anc_words, w = i % P.anc_words;
    P.t_anc[(size_t)req * T * P.anc_words + i] = (s < n && w < MAXW) ? anc[s][w] : 0ull;
  }
  if (threadIdx.x == 0) P.t_n[req] = n;
  __syncthreads();
  // ---- planted-continuation perf mode (reading R24), after linearisation
  if (P.plant != nullptr && threadIdx.x == 0) {
    int p = P.p[req];
    int step = *P.step;
    int cur = 0;
    for (int d = 1; d <= P.N && d <= HSD_MAX_PLANT_DEPTH_DEV; ++d) {
      int first = -1, hit = -1;
      if (p + d >= P.plant_stride) break;
      int want = P.plant[(size_t)req * P.plant_stride + p + d];
      for (int s = 1; s < n; ++s) {
        if (P.t_par[req * T + s] != cur) continue;
        if (first < 0) first = s;
        if (P.t_tok[req * T + s] == want && hit < 0) hit = s;
      }
      if (first < 0) break;
      u32x4 c = {(uint32_t)d, (uint32_t)step, (uint32_t)(P.req_offset + req), 0u};
      u32x4 r = philox4x32_10(c, P.seed, TAG_PLANT);
      if (!(unit_open(r.x) < P.plant_rates[d - 1])) break;
      cur = hit >= 0 ? hit : first;
      P.t_tok[req * T + cur] = want;
    }
  }
}
}  // namespace

void launch_tree(const TreeParams& P, int mode, int n_req, cudaStream_t st) {
  if (n_req <= 0) return;
  launch_k(tree_kernel, n_req * CL, NT, 0, st, P, mode);
}
