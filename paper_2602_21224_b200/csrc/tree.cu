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

unsigned long long* g_tree_trace = nullptr;   // debug phase trace (HSD_TREE_TRACE)

namespace {
constexpr int NT = 1024;
// Debug phase trace: thread 0 of request 0's leader CTA stamps %globaltimer
#define TTRACE(i)                                                                                   \
  do {                                                                                              \
    if (P.trace && threadIdx.x == 0 && blockIdx.x == 0) {                                           \
      uint64_t t_;                                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                        \
      P.trace[(i)] = t_;                                                                            \
    }                                                                                               \
  } while (0)
// CTAs per request (one thread-block cluster): 8, or 4 when the batch has more
// requests than 8-CTA clusters fit at once (one 1024-thread CTA per SM: c3's 32
// requests ran as 3 waves of 15 clusters; 4-CTA clusters take them in one wave)
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
HSD_DEV float ex2f_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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
template <int CL>
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

template <int KT, int CL>
HSD_DEV void build_subtree(const TreeParams& P, int req, int row0, int steps, int root_tok, NodesSm& nd,
                           ClusterSm<CL>& cs) {
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
    // ---- 1. sweep. Each thread keeps an online (max, sum-exp); each WARP keeps
    //      one top-k list distributed over lanes 0..k-1 (sorted, R8 order). A
    //      batch of 32 candidates (one per lane) is tested against the warp's
    //      k-th best with one ballot; only the (few) winners are inserted, one
    //      warp-wide shift each. (Per-thread lists inserted ~half of all
    //      elements at ~16 elements per thread -- the sweep was issue-bound on
    //      the insertion bubble, HSD_TREE_TRACE + ncu source counters.)
    float m = -INFINITY, sacc = 0.f;
    float ev = -INFINITY;   // lane < K: this lane's entry of the warp's top-k
    int ej = -1;
    if (qi < nq) {
      const int tok = cs.Qtok[qi];
      const int rk = P.rank_of ? P.rank_of[tok] : tok;
      const bool has_bias = !P.zero_table && rk < P.Vh;
      const int gthreads = wpn * 32;
      float tv = -INFINITY;   // the warp's current k-th best (v, j)
      int tj = -1;
      bool seeded = false;    // warp-uniform: the list holds the first batch's top-k
      constexpr int U = 4;
      for (int wbase = lo + wg * 32; wbase < hi; wbase += gthreads * U) {   // warp-uniform trip count
        float lv[U], bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = wbase + lane + u * gthreads;
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
        // branch-free online (max, sum-exp) per batch of U: one rescale of the
        // running sum per batch, exponentials as ex2.approx of log2e-scaled differences
        float v[U], mb = m;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = wbase + lane + u * gthreads;
          v[u] = j < hi ? lv[u] + bv[u] : -INFINITY;
          mb = fmaxf(mb, v[u]);
        }
        constexpr float LOG2E = 1.4426950408889634f;
        float add = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) add += ex2f_approx((v[u] - mb) * LOG2E);   // -inf -> 0
        sacc = (m == -INFINITY ? 0.f : sacc * ex2f_approx((m - mb) * LOG2E)) + add;
        m = mb;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = wbase + lane + u * gthreads;
          if (!seeded) {
            // the warp's list is still empty (first batch of the round): every lane
            // would be a candidate, so seed it with a warp bitonic sort of the
            // batch (R8 order, empty slots last) instead of 32 serial insertions
            float sv = j < hi ? v[u] : -INFINITY;
            int sj = j < hi ? j : -1;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
              for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, sv, jj);
                const int oj = __shfl_xor_sync(0xffffffffu, sj, jj);
                const bool want_better = ((lane & jj) == 0) == ((lane & kk) == 0);
                const bool other_better = better_j(ov, oj, sv, sj, perm_of(P));
                if (want_better == other_better) { sv = ov; sj = oj; }
              }
            }
            if (lane < K) { ev = sv; ej = sj; }
            tv = __shfl_sync(0xffffffffu, sv, K - 1);
            tj = __shfl_sync(0xffffffffu, sj, K - 1);
            seeded = true;
            continue;
          }
          unsigned cand = __ballot_sync(0xffffffffu, j < hi && better_j(v[u], j, tv, tj, perm_of(P)));
          while (cand) {
            const int src = __ffs(cand) - 1;
            cand &= cand - 1;
            const float xv = __shfl_sync(0xffffffffu, v[u], src);
            const int xj = __shfl_sync(0xffffffffu, j, src);
            if (!better_j(xv, xj, tv, tj, perm_of(P))) continue;    // the k-th best rose meanwhile
            const int pos = __popc(__ballot_sync(0xffffffffu, lane < K && better_j(ev, ej, xv, xj, perm_of(P))));
            const float upv = __shfl_up_sync(0xffffffffu, ev, 1);
            const int upj = __shfl_up_sync(0xffffffffu, ej, 1);
            if (lane < K) {
              if (lane == pos) { ev = xv; ej = xj; }
              else if (lane > pos) { ev = upv; ej = upj; }
            }
            tv = __shfl_sync(0xffffffffu, ev, K - 1);
            tj = __shfl_sync(0xffffffffu, ej, K - 1);
          }
        }
      }
    }
    TTRACE(2 + 4 * i);
    // ---- 2a. warp merge: (max, sum) butterfly; the top-k is already warp-wide
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sacc, o);
      const float nm = fmaxf(m, om);
      sacc = (m == -INFINITY ? 0.f : sacc * expf(m - nm)) + (om == -INFINITY ? 0.f : os * expf(om - nm));
      m = nm;
    }
    {
      if (lane < K) { wv[w * KMAX + lane] = ev; wj[w * KMAX + lane] = ej; }
      if (lane == 0) { wm[w] = m; ws[w] = sacc; }
    }
    __syncthreads();
    TTRACE(3 + 4 * i);
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
    TTRACE(4 + 4 * i);
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
    TTRACE(5 + 4 * i);
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

template <int KT, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT) tree_kernel(TreeParams P, int mode) {
  TTRACE(0);
  l2pf_issue(P.pf);
  pdl_wait();
  TTRACE(1);
  l2pf_issue(P.pf, 1);
  pdl_trigger();
  __shared__ NodesSm nd, tmp;
  __shared__ ClusterSm<CL> cs;
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
      build_subtree<KT, CL>(P, req, m + 1, n_remain, bonus, nd, cs);
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
  build_subtree<KT, CL>(P, req, 0, P.N, root, nd, cs);
  if (!leader) return;
  TTRACE(40);
  prune_nodes(nd, P.B, tmp);
  TTRACE(41);
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
    TTRACE(42);
    prune_nodes(nd, P.B + P.Br, tmp);
  }
  TTRACE(43);
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
  TTRACE(44);
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
      u32x4 c = {(uint32_t)d, (uint32_t)step, (uint32_t)P.req_id[req], 0u};
      u32x4 r = philox4x32_10(c, P.seed, TAG_PLANT);
      if (!(unit_open(r.x) < P.plant_rates[d - 1])) break;
      cur = hit >= 0 ? hit : first;
      P.t_tok[req * T + cur] = want;
    }
  }
}
}  // namespace

// called by hsd_init_model (outside any graph capture)
void tree_trace_init() {
  if (getenv("HSD_TREE_TRACE") && !g_tree_trace) cudaMalloc(&g_tree_trace, 64 * 8);
}

int num_sms();   // gemm_tc.cu (cached device SM count)

void launch_tree(const TreeParams& P0, int mode, int n_req, cudaStream_t st) {
  if (n_req <= 0) return;
  TreeParams P = P0;
  P.trace = mode == TREE_MODE_FRESH ? g_tree_trace : nullptr;   // (never mutate the kernel's P: a local copy)
  static const int cl_env = [] { const char* e = getenv("HSD_TREE_CL"); return e ? atoi(e) : 0; }();
  const int cl = cl_env == 4 || cl_env == 8 ? cl_env : (n_req * 8 > num_sms() ? 4 : 8);
  auto go = [&](auto kern, int c) { launch_k(kern, n_req * c, NT, 0, st, P, mode); };
#define HSD_TREE_CASE(KK)                                              \
  case KK:                                                             \
    if (cl == 4) go(tree_kernel<KK, 4>, 4); else go(tree_kernel<KK, 8>, 8); \
    break;
  switch (P.k) {
    HSD_TREE_CASE(1)
    HSD_TREE_CASE(2)
    HSD_TREE_CASE(3)
    HSD_TREE_CASE(4)
    HSD_TREE_CASE(5)
    HSD_TREE_CASE(6)
    HSD_TREE_CASE(7)
    default:
      if (cl == 4) go(tree_kernel<8, 4>, 4); else go(tree_kernel<8, 8>, 8);
      break;
#undef HSD_TREE_CASE
  }
}
