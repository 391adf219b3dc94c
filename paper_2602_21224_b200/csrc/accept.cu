// accept.cu -- S3 acceptance walk and S4 compaction / state update.
//
// Greedy (PAPER.md:378, :449 T = 0): from the root slot follow the child whose
//   token equals the target argmax at the current slot; the bonus token is the
//   argmax where the walk stops.
// Stochastic (reading R13): children in slot order are accepted with
//   p(c) / (1 - sum_rejected p) against a Philox uniform u(req, step, slot,
//   rank); if all are rejected the bonus is a Gumbel-max sample from the
//   residual (V minus the rejected tokens); at a leaf the bonus ~ p.
// Compaction: KV[p + j] <- KV[p + s_j] for the accepted slots s_j (s_j >= j); each
//   thread loads all its source elements before storing (in-place hazard).
#include "kernels.cuh"
#include "accept.cuh"

namespace {
constexpr int WT = 1024;

// lse of x/T over V (CTA-wide, deterministic)
HSD_DEV float row_lse(const float* x, int V, float invT, float* red) {
  float m = -INFINITY, s = 0.f;
  constexpr int U = 8;   // U independent loads in flight per thread
  for (int base = threadIdx.x; base < V; base += blockDim.x * U) {
    float xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = base + u * blockDim.x;
      xv[u] = j < V ? x[j] : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float v = xv[u] * invT;
      if (v == -INFINITY) continue;
      if (v > m) { s = s * expf(m - v) + 1.f; m = v; }
      else s += expf(v - m);
    }
  }
  float M = block_max(m, red);
  s = (m == -INFINITY) ? 0.f : s * expf(m - M);
  s = block_sum(s, red);
  return M + logf(s);
}

// Gumbel-max over v not in `excl` (n_excl entries): argmax_v x_v/T - log(-log U_v)
HSD_DEV int gumbel_argmax(const float* x, int V, float invT, uint32_t seed, uint32_t req, uint32_t step,
                          uint32_t slot, const int* excl, int n_excl, float* redf, int* redi) {
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int b4 = threadIdx.x; b4 * 4 < V; b4 += blockDim.x) {
    u32x4 c = {(uint32_t)b4, slot, step, req};
    u32x4 r = philox4x32_10(c, seed, TAG_GUMBEL);
    float xv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) xv[q] = b4 * 4 + q < V ? x[b4 * 4 + q] : 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int v = b4 * 4 + q;
      if (v >= V) break;
      bool ex = false;
      for (int e = 0; e < n_excl; ++e) ex |= (excl[e] == v);
      if (ex) continue;
      float u = unit_open(lane_of(r, q));
      float z = xv[q] * invT - logf(-logf(u));
      if (better(z, v, bv, bi)) { bv = z; bi = v; }
    }
  }
  warp_argmax(bv, bi);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) { redf[w] = bv; redi[w] = bi; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    bv = lane < nw ? redf[lane] : -INFINITY;
    bi = lane < nw ? redi[lane] : 0x7fffffff;
    warp_argmax(bv, bi);
    if (lane == 0) redi[0] = bi;
  }
  __syncthreads();
  int res = redi[0];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(WT) walk_kernel(AcceptParams P) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32];
  __shared__ int redi[32];
  __shared__ int acc[32], m_sh, bonus_sh, cur_sh, done_sh, excl[64], n_excl;
  const int req = blockIdx.x, T = P.t_max;
  const int* tok = P.t_tok + req * T;
  const int* par = P.t_par + req * T;
  const int n = P.t_n[req];
  if (P.append && n == 0) {   // no re-sampled tree to verify for this request
    if (threadIdx.x == 0) P.acc_n[req] = -1;
    return;
  }
  // append: tokens follow the step's first pass; at most N + 1 emitted per step
  const int n0 = P.append ? P.n_emitted[req] : 0, cap = P.N - n0;
  if (threadIdx.x == 0) { m_sh = 0; cur_sh = 0; done_sh = 0; }
  __syncthreads();
  if (P.mode == 0) {
    if (threadIdx.x == 0) {
      int cur = 0, m = 0;
      while (true) {
        int a = P.argmax[req * T + cur];
        int nxt = -1;
        for (int s = cur + 1; s < n; ++s)
          if (par[s] == cur && tok[s] == a) { nxt = s; break; }
        if (nxt < 0 || m >= cap) { bonus_sh = a; break; }
        acc[m++] = nxt;
        cur = nxt;
      }
      m_sh = m;
    }
    __syncthreads();
  } else {
    const float invT = 1.0f / P.temperature;
    const uint32_t rq = (uint32_t)P.req_id[req], st = (uint32_t)(*P.step);
    const bool sh = P.sh_lse != nullptr;
    while (true) {
      int cur = cur_sh;
      const size_t row = (size_t)req * T + cur;
      const float* x = sh ? nullptr : P.logits + row * P.V;
      const float lse = sh ? P.sh_lse[row] : row_lse(x, P.V, invT, red);
      if (threadIdx.x == 0) {
        n_excl = 0;
        float S = 0.f;
        int took = -1, rank = 0;
        for (int s = cur + 1; s < n && took < 0; ++s) {
          if (par[s] != cur) continue;
          int t = tok[s];
          float pc = expf((sh ? P.sh_tl[row * T + s] : x[t]) * invT - lse);
          u32x4 c = {(uint32_t)cur, (uint32_t)rank, st, rq};
          float u = unit_open(philox4x32_10(c, P.seed, TAG_ACCEPT).x);
          float denom = 1.f - S;
          float pres = denom > 0.f ? pc / denom : 0.f;
          if (u < pres) took = s;
          else { if (n_excl < 64) excl[n_excl++] = t; S += pc; }
          ++rank;
        }
        if (took >= 0 && m_sh < cap) { acc[m_sh++] = took; cur_sh = took; }
        else done_sh = 1;
      }
      __syncthreads();
      if (done_sh) {
        int b = -1;
        if (sh) {   // the best merged Gumbel candidate that was not rejected (same scores, same order)
          if (threadIdx.x == 0) {
            for (int k = 0; k < HSD_SHARD_KG && b < 0; ++k) {
              const int v = P.sh_gi[row * HSD_SHARD_KG + k];
              bool ex = false;
              for (int e = 0; e < n_excl; ++e) ex |= excl[e] == v;
              if (!ex) b = v;
            }
            if (b < 0) b = P.sh_gi[row * HSD_SHARD_KG];   // (unreachable: n_excl < KG is checked at init)
            bonus_sh = b;
          }
        } else {
          b = gumbel_argmax(x, P.V, invT, P.seed, rq, st, (uint32_t)cur, excl, n_excl, red, redi);
        }
        if (threadIdx.x == 0 && !sh) bonus_sh = b;
        break;
      }
    }
    __syncthreads();
  }
  // outputs
  const int m = m_sh;
  for (int j = n0 + threadIdx.x; j <= P.N; j += blockDim.x) {
    int v = -1;
    if (j - n0 < m) v = tok[acc[j - n0]];
    else if (j - n0 == m) v = bonus_sh;
    P.emitted[req * (P.N + 1) + j] = v;
  }
  for (int j = threadIdx.x; j < P.N; j += blockDim.x) P.acc_slots[req * P.N + j] = j < m ? acc[j] : -1;
  if (threadIdx.x == 0) {
    P.acc_n[req] = m;
    P.bonus[req] = bonus_sh;
    P.n_emitted[req] = n0 + m + 1;
  }
}

// KV compaction (S4, "accepted-path KV is kept"): the accepted slots'
// rows p + s_j move to the committed rows p + 1 + j. Grid (b, layers, 2*Hkv), one
// (kind, kv head) block of the paged cache per CTA. Every source row is read into
// registers before any row is stored (in place: a source p + s_j may be the
// destination of a later j'). K pages are [slot][hd]: a row is hd contiguous
// elements, moved as 16-byte vectors (bf16: 16 threads per hd-128 row). V pages
// are V^T [hd][slot]: one element per (d, j), the m destinations of a d-row
// being consecutive positions.
template <typename T>
__global__ void __launch_bounds__(256) compact_kernel(CompactParams P) {
  pdl_wait();
  pdl_trigger();
  const int req = blockIdx.x, layer = blockIdx.y, kh = blockIdx.z;
  const int kind = kh / P.kv_heads, h = kh % P.kv_heads;
  const int m = min(P.acc_n[req], 16);
  if (m <= 0) return;   // (-1: request skipped by the extra verify pass)
  const int p = P.p[req], hd = P.head_dim, ps = P.page_size;
  const int32_t* bt = P.block_table + (size_t)req * P.pages_per_req;
  const int32_t* sl = P.acc_slots + req * P.N;
  T* base = (T*)P.kv_base + (size_t)layer * P.layer_stride;
  // one pass, so every load precedes every store: m <= 16 rows, hd <= 128 give at
  // most 16 x 128 / VW vector items (K) or 16 x 128 scalar items (V, or K with hd
  // not a multiple of VW) -- within 256 threads x PER
  constexpr int VW = 16 / sizeof(T);            // elements per 16-byte vector
  constexpr int PER = 8;
  if (kind == 0 && hd % VW == 0) {
    const int vpr = hd / VW, items = m * vpr;     // (row j, vector) items
    uint4 v[PER / 2];
#pragma unroll
    for (int k = 0; k < PER / 2; ++k) {
      const int i = k * blockDim.x + threadIdx.x;
      if (i < items) {
        const int j = i / vpr, c = (i % vpr) * VW, key = p + sl[j];
        v[k] = *(const uint4*)(base + kv_offset(bt[key / ps], 0, P.kv_heads, h, ps, hd, key % ps, c));
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER / 2; ++k) {
      const int i = k * blockDim.x + threadIdx.x;
      if (i < items) {
        const int j = i / vpr, c = (i % vpr) * VW, key = p + 1 + j;
        *(uint4*)(base + kv_offset(bt[key / ps], 0, P.kv_heads, h, ps, hd, key % ps, c)) = v[k];
      }
    }
  } else {
    const int items = m * hd;                     // (d, j) items, j fastest: a d-row's stores are consecutive
    T v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = k * blockDim.x + threadIdx.x;
      if (i < items) {
        const int d = i / m, j = i % m, key = p + sl[j];
        v[k] = base[kv_offset(bt[key / ps], kind, P.kv_heads, h, ps, hd, key % ps, d)];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = k * blockDim.x + threadIdx.x;
      if (i < items) {
        const int d = i / m, j = i % m, key = p + 1 + j;
        base[kv_offset(bt[key / ps], kind, P.kv_heads, h, ps, hd, key % ps, d)] = v[k];
      }
    }
  }
}

// state update: pending draft pairs, root, position, step counter
__global__ void commit_kernel(CommitParams P) {
  pdl_wait();
  pdl_trigger();
  const int req = blockIdx.x;
  const int m = P.acc_n[req];
  const int n = P.hidden;
  if (threadIdx.x == 0 && req == 0) atomicAdd(P.step, 1);   // one random-stream step per verify pass
  if (m < 0) return;                                        // skipped by the extra verify pass
  // this pass's tokens start at e0 of the step's emitted row; its pairs at o0 of the pending pairs
  const int e0 = P.n_emitted[req] - (m + 1), o0 = P.append ? P.n_pend[req] : 0;
  for (int j = 0; j <= m; ++j) {
    int slot = j == 0 ? 0 : P.acc_slots[req * P.N + j - 1];
    const float* src = P.Hverify + ((size_t)req * P.t_max + slot) * n;
    float* dst = P.pend_H + ((size_t)req * (P.N + 1) + o0 + j) * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();   // every thread has read n_pend before thread 0 updates it
  if (threadIdx.x == 0) {
    for (int j = o0; j <= P.N; ++j)
      P.pend_tok[req * (P.N + 1) + j] = j - o0 <= m ? P.emitted[req * (P.N + 1) + e0 + j - o0] : -1;
    P.n_pend[req] = o0 + m + 1;
    P.root_tok[req] = P.bonus[req];
    P.p[req] += m + 1;
  }
}
// the Alg. 2 pending tree as a verify tree (one thread per request; <= 64 nodes)
__global__ void pending_as_tree_kernel(const int32_t* pt_n, const int32_t* pt_tok, const int32_t* pt_par,
                                       const int32_t* pt_depth, const float* pt_lj, int br1, int32_t* t_n,
                                       int32_t* t_tok, int32_t* t_par, int32_t* t_depth, float* t_lj,
                                       uint64_t* t_anc, int t_max, int anc_words) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (threadIdx.x != 0) return;
  const int n = min(pt_n[r], br1);
  if (n <= 1) { t_n[r] = 0; return; }
  const int32_t* tk = pt_tok + r * br1;
  const int32_t* pa = pt_par + r * br1;
  const float* lj = pt_lj + r * br1;
  int order[64], slot_of[64];
  int len = 1, head = 0;
  order[0] = 0; slot_of[0] = 0;
  while (head < len) {   // BFS; the children of u by (lj desc, token asc, creation order)
    const int u = order[head++];
    int start = len;
    for (int c = 1; c < n; ++c)
      if (pa[c] == u) order[len++] = c;
    for (int i = start + 1; i < len; ++i) {   // insertion sort of the new children
      const int c = order[i];
      int j = i - 1;
      while (j >= start && (lj[order[j]] < lj[c] || (lj[order[j]] == lj[c] && tk[order[j]] > tk[c]))) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = c;
    }
    for (int i = start; i < len; ++i) slot_of[order[i]] = i;
  }
  for (int s = 0; s < len; ++s) {
    const int i = order[s];
    const int ps = s == 0 ? -1 : slot_of[pa[i]];
    t_tok[r * t_max + s] = tk[i];
    t_par[r * t_max + s] = ps;
    t_depth[r * t_max + s] = pt_depth[r * br1 + i];
    t_lj[r * t_max + s] = lj[i];
    uint64_t* a = t_anc + ((size_t)r * t_max + s) * anc_words;
    for (int w = 0; w < anc_words; ++w) a[w] = ps >= 0 ? t_anc[((size_t)r * t_max + ps) * anc_words + w] : 0ull;
    a[s >> 6] |= 1ull << (s & 63);
  }
  t_n[r] = len;
}

// test hook (hsd_debug_gumbel): pair i = one Gumbel-max draw over logits row row[i]
// with the walk's own device function and Philox stream (seed, req, step, slot[i])
__global__ void __launch_bounds__(WT) gumbel_debug_kernel(const float* logits, int ld, int V, float invT, uint32_t seed,
                                                          uint32_t req, uint32_t step, const int32_t* row,
                                                          const int32_t* slot, int32_t* out) {
  __shared__ float red[32];
  __shared__ int redi[32];
  const int i = blockIdx.x;
  const int b = gumbel_argmax(logits + (size_t)row[i] * ld, V, invT, seed, req, step, (uint32_t)slot[i], nullptr, 0,
                              red, redi);
  if (threadIdx.x == 0) out[i] = b;
}
}  // namespace

void launch_gumbel_debug(const float* logits, int ld, int V, float temperature, uint32_t seed, int req, int step,
                         int n, const int32_t* row, const int32_t* slot, int32_t* out, cudaStream_t st) {
  if (n > 0)
    gumbel_debug_kernel<<<n, WT, 0, st>>>(logits, ld, V, 1.0f / temperature, seed, (uint32_t)req, (uint32_t)step, row,
                                          slot, out);
}

void launch_pending_as_tree(const int32_t* pt_n, const int32_t* pt_tok, const int32_t* pt_par,
                            const int32_t* pt_depth, const float* pt_lj, int br1, int32_t* t_n, int32_t* t_tok,
                            int32_t* t_par, int32_t* t_depth, float* t_lj, uint64_t* t_anc, int t_max, int anc_words,
                            int n_req, cudaStream_t st) {
  if (n_req > 0)
    launch_k(pending_as_tree_kernel, n_req, 32, 0, st, pt_n, pt_tok, pt_par, pt_depth, pt_lj, br1, t_n, t_tok, t_par,
             t_depth, t_lj, t_anc, t_max, anc_words);
}

void launch_walk(const AcceptParams& P, int n_req, cudaStream_t st) {
  if (n_req > 0) launch_k(walk_kernel, n_req, WT, 0, st, P);
}
void launch_compact(const CompactParams& P, int n_req, int layers, DType dt, cudaStream_t st) {
  if (n_req <= 0) return;
  dim3 grid(n_req, layers, 2 * P.kv_heads);
  if (dt == DT_F32) launch_k(compact_kernel<float>, grid, 256, 0, st, P);
  else launch_k(compact_kernel<bf16>, grid, 256, 0, st, P);
}
void launch_commit(const CommitParams& P, int n_req, cudaStream_t st) {
  if (n_req > 0) launch_k(commit_kernel, n_req, 256, 0, st, P);
}
