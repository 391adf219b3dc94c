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

#define perm_of(P) ((P).perm)
// per-thread top-KC list, sorted by (value desc, token asc); KC = k exactly, so
// the admission test is against the k-th best and insertion bubbles k-1 steps
template <int KC>
struct Top {
  float v[KC];
  int j[KC];
};

template <int KC>
HSD_DEV void top_init(Top<KC>& t) {
#pragma unroll
  for (int s = 0; s < KC; ++s) { t.v[s] = -INFINITY; t.j[s] = -1; }
}
template <int KC>
HSD_DEV void top_insert(Top<KC>& t, float v, int j, const int32_t* perm) {
  if (!better_j(v, j, t.v[KC - 1], t.j[KC - 1], perm)) return;
  t.v[KC - 1] = v; t.j[KC - 1] = j;
#pragma unroll
  for (int s = KC - 1; s > 0; --s) {
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

// Alg. 1 BuildSubtree on a thread-block cluster of CL CTAs (one request).
// Every round (one step i of Alg. 1):
//  1. each CTA sweeps its 1/CL vocab slice for ALL frontier nodes at once: the
//     32 warps are split into one group per frontier node; a thread keeps an
//     online (max, sum-exp) and a top-8 of l_i + r(node.token);
//  2. warp merges, then the group's leader warp merges its warps' lists into the
//     (node, CTA) Partial and BROADCASTS it into every CTA's shared memory
//     (DSMEM, double-buffered by round parity);
//  3. one cluster barrier; then every CTA merges the CL partials of every node
//     (exact (max, sum-exp) combination, top-k by rank), appends the children in
//     frontier order and runs TopkByJointProb -- redundantly and identically, so
//     no second barrier is needed to publish the frontier.
struct ClusterSm {
  Partial part[2][KMAX][CL];
  int Q[KMAX], Qtok[KMAX], nq;
};

HSD_DEV void merge_lists_lanes(int nlists, const float* lv, const int* lj, int k, const int32_t* perm, float* ov,
                               int* oj) {
  // warp-collective: lane l < nlists owns sorted list l (KMAX entries, stride KMAX)
  const int lane = threadIdx.x & 31;
  int hd = 0;
  for (int r = 0; r < k; ++r) {
    float bv = (lane < nlists && hd < k) ? lv[lane * KMAX + hd] : -INFINITY;
    int bj = (lane < nlists && hd < k) ? lj[lane * KMAX + hd] : -1, bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ovv = __shfl_xor_sync(0xffffffffu, bv, o);
      const int ojj = __shfl_xor_sync(0xffffffffu, bj, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (beats(ovv, ojj, ol, bv, bj, bl, perm)) { bv = ovv; bj = ojj; bl = ol; }
    }
    if (lane == 0) { ov[r] = bv; oj[r] = bj; }
    if (lane == bl) hd++;
  }
}

template <int KT>
HSD_DEV void build_subtree(const TreeParams& P, int req, int row0, int steps, int root_tok, NodesSm& nd,
                           ClusterSm& cs) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ float wv[32 * KMAX], wm[32], ws[32];
  __shared__ int wj[32 * KMAX];
  if (threadIdx.x == 0) {
    nd.tok[0] = root_tok; nd.par[0] = -1; nd.depth[0] = 0; nd.lj[0] = 0.f; nd.n = 1;
    cs.Q[0] = 0; cs.Qtok[0] = root_tok; cs.nq = 1;
  }
  cluster.sync();   // every CTA of the cluster is running before any DSMEM store
  const int per = (P.V + CL - 1) / CL;
  const int lo = min(P.V, rank * per), hi = min(P.V, lo + per);
  const int K = P.k;
  for (int i = 0; i < steps; ++i) {
    const int par = i & 1;
    const int nq = cs.nq;
    const int wpn = 32 / nq;                       // warps per frontier node
    const int qi = w / wpn, wg = w % wpn;          // this warp's node and index in its group
    const float* Lrow = P.L + ((size_t)req * P.N + row0 + i) * P.V;
    // ---- 1. sweep
    float m = -INFINITY, sacc = 0.f;
    Top<KT> t;
    top_init(t);
    if (qi < nq) {
      const int tok = cs.Qtok[qi];
      const int rk = P.rank_of ? P.rank_of[tok] : tok;
      const bool has_bias = !P.zero_table && rk < P.Vh;
      const int gthreads = wpn * 32, gt = wg * 32 + lane;
      constexpr int U = 4;
      for (int base = lo + gt; base < hi; base += gthreads * U) {
        float lv[U], bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = base + u * gthreads;
          lv[u] = j < hi ? Lrow[j] : 0.f;
          float b = 0.f;
          if (has_bias && j < hi && j < P.Vh) {
            const size_t ix = (size_t)rk * P.Vh + j;
            if (P.tscale) {
              const __half_raw hr = __nv_cvt_fp8_to_halfraw(((const __nv_fp8_storage_t*)P.table)[ix], __NV_E4M3);
              b = __half2float(__half(hr)) * P.tscale[rk];
            } else {
              b = P.tdt == DT_F32 ? ((const float*)P.table)[ix] : to_f32(((const bf16*)P.table)[ix]);
            }
          }
          bv[u] = b;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = base + u * gthreads;
          if (j >= hi) break;
          const float v = lv[u] + bv[u];
          if (v > m) { sacc = sacc * expf(m - v) + 1.f; m = v; }
          else sacc += expf(v - m);
          top_insert(t, v, j, perm_of(P));
        }
      }
    }
    // ---- 2a. warp merge: (max, sum) butterfly and top-k of the lanes' lists
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sacc, o);
      const float nm = fmaxf(m, om);
      sacc = (m == -INFINITY ? 0.f : sacc * expf(m - nm)) + (om == -INFINITY ? 0.f : os * expf(om - nm));
      m = nm;
    }
    {
      int head = 0;
      for (int r = 0; r < K; ++r) {
        float hv = -INFINITY;
        int hj = -1;
#pragma unroll
        for (int q = 0; q < KT; ++q)
          if (q == head) { hv = t.v[q]; hj = t.j[q]; }
        float bv = hv;
        int bj = hj, bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
          if (beats(ov, oj, ol, bv, bj, bl, perm_of(P))) { bv = ov; bj = oj; bl = ol; }
        }
        if (lane == 0) { wv[w * KMAX + r] = bv; wj[w * KMAX + r] = bj; }
        if (lane == bl) head++;
      }
      if (lane == 0) { wm[w] = m; ws[w] = sacc; }
    }
    __syncthreads();
    // ---- 2b. group leader warps: merge the group's warps, broadcast the Partial
    if (qi < nq && wg == 0) {
      const int w0 = qi * wpn;
      float mm = lane < wpn ? wm[w0 + lane] : -INFINITY, ss = lane < wpn ? ws[w0 + lane] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, mm, o), os = __shfl_xor_sync(0xffffffffu, ss, o);
        const float nm = fmaxf(mm, om);
        ss = (mm == -INFINITY ? 0.f : ss * expf(mm - nm)) + (om == -INFINITY ? 0.f : os * expf(om - nm));
        mm = nm;
      }
      __shared__ Partial grp[KMAX];
      merge_lists_lanes(wpn, wv + w0 * KMAX, wj + w0 * KMAX, K, perm_of(P), grp[qi].v, grp[qi].j);
      if (lane == 0) { grp[qi].m = mm; grp[qi].s = ss; }
      __syncwarp();
      if (lane < CL) {                           // lane c writes this partial into CTA c
        Partial* dst = cluster.map_shared_rank(&cs.part[par][qi][rank], lane);
        *dst = grp[qi];
      }
    }
    cluster.sync();
    // ---- 3. every CTA: merge the CL partials, children, TopkByJointProb
    const int start = nd.n;
    for (int tt = threadIdx.x; tt < nq * CL * KMAX; tt += blockDim.x) {
      const int q = tt / (CL * KMAX), c = (tt / KMAX) % CL, e = tt % KMAX;
      if (e >= K) continue;
      const Partial& pc = cs.part[par][q][c];
      const float v = pc.v[e];
      const int j = pc.j[e];
      if (j < 0) continue;
      int rnk = 0;
      for (int c2 = 0; c2 < CL; ++c2)
        for (int e2 = 0; e2 < K; ++e2) {
          const int j2 = cs.part[par][q][c2].j[e2];
          if (j2 >= 0 && better_j(cs.part[par][q][c2].v[e2], j2, v, j, perm_of(P))) ++rnk;
        }
      if (rnk < K) {
        float M = -INFINITY, S = 0.f;
        for (int c2 = 0; c2 < CL; ++c2) M = fmaxf(M, cs.part[par][q][c2].m);
        for (int c2 = 0; c2 < CL; ++c2)
          if (cs.part[par][q][c2].m != -INFINITY) S += cs.part[par][q][c2].s * expf(cs.part[par][q][c2].m - M);
        const float lse = M + logf(S);
        const int u = cs.Q[q], n = start + q * K + rnk;
        nd.tok[n] = P.perm ? P.perm[j] : j;
        nd.par[n] = u;
        nd.depth[n] = nd.depth[u] + 1;
        nd.lj[n] = nd.lj[u] + (v - lse);
      }
    }
    __syncthreads();
    const int cnt_new = nq * K;
    __shared__ int newQ[KMAX];
    for (int c = threadIdx.x; c < cnt_new; c += blockDim.x) {
      const int a = start + c;
      int rnk = 0;
      for (int b = start; b < start + cnt_new; ++b) {
        const bool bb = nd.lj[b] > nd.lj[a] ||
                        (nd.lj[b] == nd.lj[a] &&
                         (nd.tok[b] < nd.tok[a] || (nd.tok[b] == nd.tok[a] && nd.par[b] < nd.par[a])));
        rnk += bb;
      }
      if (rnk < K) newQ[rnk] = a;
    }
    __syncthreads();
    if (threadIdx.x < KMAX) {
      const int q = threadIdx.x;
      if (q < K && q < cnt_new) { cs.Q[q] = newQ[q]; cs.Qtok[q] = nd.tok[newQ[q]]; }
      if (q == 0) { nd.n = start + cnt_new; cs.nq = K < cnt_new ? K : cnt_new; }
    }
    __syncthreads();
  }
}

// keep the top-`keep` non-root nodes (joint desc, depth asc, token asc, parent asc),
// compacted in creation order.
HSD_DEV void prune_nodes(NodesSm& nd, int keep, NodesSm& tmp) {
  __shared__ int flag[MAXN], newidx[MAXN], wsum[MAXN / 32];
  const int n = nd.n;
  // rank of node i among non-root nodes: 4 threads per node, each a quarter of j
  for (int t = threadIdx.x; t < 4 * MAXN; t += blockDim.x) {
    const int i = t >> 2, part = t & 3;
    int c = 0;
    if (i > 0 && i < n) {
      const float li = nd.lj[i];
      const int di = nd.depth[i], ti = nd.tok[i], pi = nd.par[i];
      for (int j = 1 + part; j < n; j += 4) {
        const float lj = nd.lj[j];
        c += lj > li || (lj == li && (nd.depth[j] < di ||
                                      (nd.depth[j] == di && (nd.tok[j] < ti || (nd.tok[j] == ti && nd.par[j] < pi)))));
      }
    }
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    if (part == 0 && i < MAXN) flag[i] = (i < n) && (i == 0 || c < keep);
  }
  __syncthreads();
  // exclusive prefix sum of flags (creation order preserved)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < MAXN) {
    const unsigned b = __ballot_sync(0xffffffffu, flag[threadIdx.x]);
    if (lane == 0) wsum[w] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x < MAXN) {
    const unsigned b = __ballot_sync(0xffffffffu, flag[threadIdx.x]);
    int off = 0;
    for (int q = 0; q < w; ++q) off += wsum[q];
    newidx[threadIdx.x] = flag[threadIdx.x] ? off + __popc(b & ((1u << lane) - 1u)) : -1;
    if (threadIdx.x == MAXN - 1) tmp.n = off + __popc(b);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!flag[i]) continue;
    const int t = newidx[i];
    tmp.tok[t] = nd.tok[i];
    tmp.par[t] = nd.par[i] >= 0 ? newidx[nd.par[i]] : -1;
    tmp.depth[t] = nd.depth[i];
    tmp.lj[t] = nd.lj[i];
  }
  __syncthreads();
  const int n2 = tmp.n;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    nd.tok[i] = tmp.tok[i]; nd.par[i] = tmp.par[i]; nd.depth[i] = tmp.depth[i]; nd.lj[i] = tmp.lj[i];
  }
  if (threadIdx.x == 0) nd.n = n2;
  __syncthreads();
}

template <int KT>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT) tree_kernel(TreeParams P, int mode) {
  l2pf_issue(P.pf);
  pdl_wait();
  l2pf_issue(P.pf, 1);
  pdl_trigger();
  __shared__ NodesSm nd, tmp;
  __shared__ ClusterSm cs;
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
      build_subtree<KT>(P, req, m + 1, n_remain, bonus, nd, cs);
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
  build_subtree<KT>(P, req, 0, P.N, root, nd, cs);
  if (!leader) return;
  prune_nodes(nd, P.B, tmp);
  // ---- verification fusion with the pending re-sampled tree
  int pn = P.pt_n[req];
  if (P.fusion && pn > 1) {
    if (threadIdx.x < 32) {            // warp 0: pending nodes in creation order, lanes search
      const int lane = threadIdx.x;
      int map[HSD_MAX_BR1];
      if (lane == 0 && P.pt_tok[req * Br1] != root) atomicOr(P.err, DEV_ERR_BAD_TREE);
      map[0] = 0;
      for (int j = 1; j < pn && j < HSD_MAX_BR1; ++j) {
        const int ptok = P.pt_tok[req * Br1 + j];
        const int fpar = map[P.pt_par[req * Br1 + j]];
        const float plj = P.pt_lj[req * Br1 + j];
        const int nn = nd.n;
        int hit = 0x7fffffff;
        for (int i = 1 + lane; i < nn; i += 32)
          if (nd.par[i] == fpar && nd.tok[i] == ptok) hit = min(hit, i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hit = min(hit, __shfl_xor_sync(0xffffffffu, hit, o));
        if (hit != 0x7fffffff) {
          if (lane == 0 && plj > nd.lj[hit]) nd.lj[hit] = plj;
          map[j] = hit;
        } else {
          if (lane == 0 && nn < MAXN) {
            nd.tok[nn] = ptok; nd.par[nn] = fpar; nd.depth[nn] = nd.depth[fpar] + 1; nd.lj[nn] = plj;
            nd.n = nn + 1;
          }
          map[j] = nn < MAXN ? nn : 0;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    prune_nodes(nd, P.B + P.Br, tmp);
  }
  // ---- linearise: BFS, siblings by (joint desc, token asc); nodes bucketed by
  //      depth, each ranked only among its own depth's bucket
  const int n = nd.n;
  __shared__ int dcnt[HSD_MAX_PLANT_DEPTH_DEV + 2], doff[HSD_MAX_PLANT_DEPTH_DEV + 2], bucket[MAXN];
  if (threadIdx.x < HSD_MAX_PLANT_DEPTH_DEV + 2) dcnt[threadIdx.x] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&dcnt[nd.depth[i]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0, md = 0;
    for (int d = 0; d < HSD_MAX_PLANT_DEPTH_DEV + 2; ++d) {
      doff[d] = acc;
      acc += dcnt[d];
      if (dcnt[d]) md = d;
      dcnt[d] = 0;
    }
    maxdepth = md;
    slot_of[0] = 0;
    for (int w = 0; w < MAXW; ++w) anc[0][w] = 0ull;
    anc[0][0] = 1ull;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int d = nd.depth[i];
    bucket[doff[d] + atomicAdd(&dcnt[d], 1)] = i;
  }
  __syncthreads();
  for (int d = 1; d <= maxdepth; ++d) {
    const int b0 = doff[d], nb = dcnt[d];
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const int i = bucket[b0 + t];
      const int pi = slot_of[nd.par[i]];
      int c = 0;
      for (int u = 0; u < nb; ++u) {
        const int j = bucket[b0 + u];
        const int pj = slot_of[nd.par[j]];
        c += pj < pi || (pj == pi && (nd.lj[j] > nd.lj[i] || (nd.lj[j] == nd.lj[i] && nd.tok[j] < nd.tok[i])));
      }
      slot_of[i] = b0 + c;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const int i = bucket[b0 + t];
      const int sl = slot_of[i], ps = slot_of[nd.par[i]];
      for (int w = 0; w < MAXW; ++w) anc[sl][w] = anc[ps][w];
      anc[sl][sl >> 6] |= 1ull << (sl & 63);
    }
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
  switch (P.k) {
    case 1: launch_k(tree_kernel<1>, n_req * CL, NT, 0, st, P, mode); break;
    case 2: launch_k(tree_kernel<2>, n_req * CL, NT, 0, st, P, mode); break;
    case 3: launch_k(tree_kernel<3>, n_req * CL, NT, 0, st, P, mode); break;
    case 4: launch_k(tree_kernel<4>, n_req * CL, NT, 0, st, P, mode); break;
    case 5: launch_k(tree_kernel<5>, n_req * CL, NT, 0, st, P, mode); break;
    case 6: launch_k(tree_kernel<6>, n_req * CL, NT, 0, st, P, mode); break;
    case 7: launch_k(tree_kernel<7>, n_req * CL, NT, 0, st, P, mode); break;
    default: launch_k(tree_kernel<8>, n_req * CL, NT, 0, st, P, mode); break;
  }
}
