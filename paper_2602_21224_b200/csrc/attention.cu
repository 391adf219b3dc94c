// attention.cu -- tree-masked attention over the paged KV cache (PAPER.md:95
// "tree-shaped attention", :582 SpecInfer tree masks), split-KV online softmax.
//
// Query row r (one token: a tree slot, a draft row or a prefill row) of request
// q sees key position k iff
//     klo[r] <= k < khi[r]                                  (committed cache / causal)
//  or slot[r] >= 0 and 0 <= k - tbase[q] < t_max and bit (k - tbase[q]) of
//     anc[q, slot[r]] is set                                (its tree ancestors and itself)
// One CTA = (key split, kv head, request x q-tile of QT (row, head) pairs of the
// GQA group). K/V sub-chunks of CH keys are staged in shared memory (fp32) and
// every warp owns (row, head) pairs: lanes split the keys for QK^T and the head
// dimension for PV. Splits > 1 write (o, m, l) partials merged by a second
// kernel with the exact log-sum-exp rule.
#include "kernels.cuh"

namespace {
constexpr int CH = 64;     // keys per shared-memory sub-chunk
constexpr int QT = 32;     // (row, head) pairs per CTA
constexpr int NW = 8;      // warps per CTA
constexpr int MAXHD = 128;

template <typename T>
HSD_DEV T kv_elem(const KVLayer& kv, int req, int key, int kind, int h, int d) {
  int page = kv.block_table[(size_t)req * kv.pages_per_req + key / kv.page_size];
  return ((const T*)kv.base)[kv_offset(page, kind, kv.kv_heads, h, kv.page_size, kv.head_dim, key % kv.page_size, d)];
}

HSD_DEV bool visible(const RowMeta& m, int row, int req, int key) {
  if (key >= m.klo[row] && key < m.khi[row]) return true;
  int s = m.slot[row];
  if (s < 0) return false;
  int d = key - m.tbase[req];
  if (d < 0 || d >= m.t_max) return false;
  uint64_t w = m.anc[((size_t)req * m.t_max + s) * m.anc_words + (d >> 6)];
  return (w >> (d & 63)) & 1ull;
}

template <typename T>
__global__ void __launch_bounds__(NW * 32) attention_kernel(const T* __restrict__ q, int M, int R, RowMeta m,
                                                            KVLayer kv, int Hq, int max_keys, int keys_per_split,
                                                            int n_qtiles, T* __restrict__ out,
                                                            float* __restrict__ ws) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float smem[];
  const int hd = kv.head_dim, Hkv = kv.kv_heads, G = Hq / Hkv;
  float* Ks = smem;                       // [CH][hd+1]
  float* Vs = Ks + CH * (hd + 1);         // [CH][hd]
  float* Qs = Vs + CH * hd;               // [QT][hd]
  float* Os = Qs + QT * hd;               // [QT][hd]
  float* Ms = Os + QT * hd;               // [QT]
  float* Ls = Ms + QT;                    // [QT]
  float* Ps = Ls + QT;                    // [NW][CH]
  __shared__ int tile_lo, tile_hi;

  const int split = blockIdx.x, h = blockIdx.y;
  const int grp = blockIdx.z / n_qtiles, qt = blockIdx.z % n_qtiles;   // rows [grp*R, grp*R+R)
  const int req = m.req[grp * R];                                      // their request (KV / tree)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float scale = 1.0f / sqrtf((float)hd);
  const int k_begin = split * keys_per_split;
  const int k_end = min(max_keys, k_begin + keys_per_split);

  // load the q tile, init state, compute the tile's key bounds
  if (threadIdx.x == 0) { tile_lo = 0x7fffffff; tile_hi = 0; }
  __syncthreads();
  for (int i = threadIdx.x; i < QT * hd; i += blockDim.x) {
    int t = i / hd, d = i % hd, rh = qt * QT + t;
    int rl = rh / G, g = rh % G, row = grp * R + rl;
    float v = 0.f;
    if (rl < R && m.pos[row] >= 0) v = to_f32(q[((size_t)row * Hq + h * G + g) * hd + d]);
    Qs[i] = v;
    Os[i] = 0.f;
  }
  if (threadIdx.x < QT) {
    int rh = qt * QT + threadIdx.x, rl = rh / G, row = grp * R + rl;
    Ms[threadIdx.x] = -INFINITY;
    Ls[threadIdx.x] = 0.f;
    if (rl < R && m.pos[row] >= 0) {
      int lo = m.klo[row], hi = m.khi[row];
      if (m.slot[row] >= 0) {
        lo = min(lo, m.tbase[req]);
        hi = max(hi, m.tbase[req] + m.slot[row] + 1);
      }
      if (hi > lo) { atomicMin(&tile_lo, lo); atomicMax(&tile_hi, hi); }
    }
  }
  __syncthreads();
  const int lo = max(k_begin, tile_lo), hi = min(k_end, tile_hi);

  for (int c0 = lo - (lo % CH); c0 < hi; c0 += CH) {
    __syncthreads();
    for (int i = threadIdx.x; i < CH * hd; i += blockDim.x) {
      int kk = i / hd, d = i % hd, key = c0 + kk;
      float kvk = 0.f, kvv = 0.f;
      if (key < max_keys) {
        kvk = to_f32(kv_elem<T>(kv, req, key, 0, h, d));
        kvv = to_f32(kv_elem<T>(kv, req, key, 1, h, d));
      }
      Ks[kk * (hd + 1) + d] = kvk;
      Vs[kk * hd + d] = kvv;
    }
    __syncthreads();
    for (int t = warp; t < QT; t += NW) {
      int rh = qt * QT + t, rl = rh / G, row = grp * R + rl;
      if (rl >= R || m.pos[row] < 0) continue;
      float s[CH / 32];
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < CH / 32; ++j) {
        int kk = lane + 32 * j, key = c0 + kk;
        float v = -INFINITY;
        if (key >= k_begin && key < k_end && visible(m, row, req, key)) {
          float acc = 0.f;
          const float* kr = Ks + kk * (hd + 1);
          const float* qr = Qs + t * hd;
          for (int d = 0; d < hd; ++d) acc = fmaf(qr[d], kr[d], acc);
          v = acc * scale;
        }
        s[j] = v;
        mx = fmaxf(mx, v);
      }
      mx = warp_max(mx);
      if (mx == -INFINITY) continue;
      float m_old = Ms[t];
      float m_new = fmaxf(m_old, mx);
      float alpha = (m_old == -INFINITY) ? 0.f : expf(m_old - m_new);
      float psum = 0.f;
#pragma unroll
      for (int j = 0; j < CH / 32; ++j) {
        float p = (s[j] == -INFINITY) ? 0.f : expf(s[j] - m_new);
        Ps[warp * CH + lane + 32 * j] = p;
        psum += p;
      }
      psum = warp_sum(psum);
      __syncwarp();
      for (int d = lane; d < hd; d += 32) {
        float o = Os[t * hd + d] * alpha;
        for (int kk = 0; kk < CH; ++kk) o = fmaf(Ps[warp * CH + kk], Vs[kk * hd + d], o);
        Os[t * hd + d] = o;
      }
      __syncwarp();
      if (lane == 0) { Ms[t] = m_new; Ls[t] = Ls[t] * alpha + psum; }
      __syncwarp();
    }
  }
  __syncthreads();
  // epilogue
  const bool direct = (gridDim.x == 1);
  for (int i = threadIdx.x; i < QT * hd; i += blockDim.x) {
    int t = i / hd, d = i % hd, rh = qt * QT + t;
    int rl = rh / G, g = rh % G, row = grp * R + rl;
    if (rl >= R) continue;
    int head = h * G + g;
    float l = Ls[t];
    if (direct) {
      out[((size_t)row * Hq + head) * hd + d] = from_f32<T>(l > 0.f ? Os[i] / l : 0.f);
    } else {
      ws[(((size_t)split * M + row) * Hq + head) * hd + d] = Os[i];
    }
  }
  if (!direct && threadIdx.x < QT) {
    int t = threadIdx.x, rh = qt * QT + t, rl = rh / G, g = rh % G, row = grp * R + rl;
    if (rl < R) {
      size_t base = (size_t)gridDim.x * M * Hq * hd;
      size_t idx = ((size_t)split * M + row) * Hq + h * G + g;
      ws[base + 2 * idx] = Ms[t];
      ws[base + 2 * idx + 1] = Ls[t];
    }
  }
}

// merge split partials: o = sum_s e^{m_s - M} o_s / sum_s e^{m_s - M} l_s
template <typename T>
__global__ void attention_merge_kernel(const float* __restrict__ ws, int S, int M, int Hq, int hd,
                                       T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
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
    out[((size_t)row * Hq + head) * hd + d] = from_f32<T>(den > 0.f ? num / den : 0.f);
  }
}
}  // namespace

static int pick_splits(int base_ctas, int max_keys) {
  int max_s = (max_keys + CH - 1) / CH;
  int s = (2 * 148 + base_ctas - 1) / base_ctas;
  if (s > max_s) s = max_s;
  if (s > 32) s = 32;
  if (s < 1) s = 1;
  return s;
}

size_t attention_ws_floats(int M, int Hq, int hd, int max_splits) {
  return (size_t)max_splits * M * Hq * (hd + 2);
}

void launch_attention(const void* q, int M, int R, int n_req, const RowMeta& m, const KVLayer& kv, int Hq,
                      DType dt, int max_keys, void* out, float* ws, size_t ws_floats, cudaStream_t st) {
  if (M <= 0) return;
  const int G = Hq / kv.kv_heads, hd = kv.head_dim;
  const int n_qtiles = (R * G + QT - 1) / QT;
  const int base = n_req * kv.kv_heads * n_qtiles;
  int S = pick_splits(base, max_keys);
  while (S > 1 && attention_ws_floats(M, Hq, hd, S) > ws_floats) --S;
  int kps = (max_keys + S - 1) / S;
  kps = (kps + CH - 1) / CH * CH;
  S = (max_keys + kps - 1) / kps;
  size_t smem = (size_t)(CH * (hd + 1) + CH * hd + 2 * QT * hd + 2 * QT + NW * CH) * sizeof(float);
  dim3 grid(S, kv.kv_heads, n_req * n_qtiles);
  if (dt == DT_F32) {
    cudaFuncSetAttribute(attention_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(attention_kernel<float>, grid, NW * 32, smem, st, (const float*)q, M, R, m, kv, Hq, max_keys, kps,
                                                         n_qtiles, (float*)out, ws);
    if (S > 1) launch_k(attention_merge_kernel<float>, dim3(M, Hq), 128, 0, st, ws, S, M, Hq, hd, (float*)out);
  } else {
    cudaFuncSetAttribute(attention_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(attention_kernel<bf16>, grid, NW * 32, smem, st, (const bf16*)q, M, R, m, kv, Hq, max_keys, kps,
                                                        n_qtiles, (bf16*)out, ws);
    if (S > 1) launch_k(attention_merge_kernel<bf16>, dim3(M, Hq), 128, 0, st, ws, S, M, Hq, hd, (bf16*)out);
  }
}
