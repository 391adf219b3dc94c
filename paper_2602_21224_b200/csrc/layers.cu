// layers.cu -- row-wise kernels of the Llama decoder used by draft, verify and
// prefill passes: RMSNorm, embedding gather, RoPE + paged KV write, SwiGLU,
// argmax, draft-input concat (reading R1).
//
// All are bandwidth-trivial at decode sizes (tens of rows), so they are written
// for latency: 128-bit vector accesses, every load of a thread issued before
// use, and grids that put (row, column-chunk) work items on many SMs.
#include <algorithm>
#include "kernels.cuh"

namespace {
template <typename T> struct Vec4;
template <> struct Vec4<float> {
  static HSD_DEV void store(float* p, float a, float b, float c, float d) { *(float4*)p = make_float4(a, b, c, d); }
};
template <> struct Vec4<bf16> {
  static HSD_DEV void store(bf16* p, float a, float b, float c, float d) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
    uint2 u;
    u.x = *(uint32_t*)&lo;
    u.y = *(uint32_t*)&hi;
    *(uint2*)p = u;
  }
};
}  // namespace

// ------------------------------------------------------------------ RMSNorm
// out[r] = x[r] / sqrt(mean(x[r]^2) + eps) (gain 1). Inactive rows -> 0.
// One CTA per row; n % 4 == 0; up to 8 float4 per thread kept in registers.
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x, int n, float eps,
                                                      T* __restrict__ out, const int32_t* __restrict__ pos,
                                                      L2Pf pf) {
  l2pf_issue(pf);
  pdl_wait();
  l2pf_issue(pf, 1);
  pdl_trigger();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const float4* xr = (const float4*)(x + (size_t)r * n);
  T* o = out + (size_t)r * n;
  const bool active = pos == nullptr || pos[r] >= 0;
  const int n4 = n >> 2;
  float4 v[8];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int i = threadIdx.x + j * blockDim.x;
    v[j] = (i < n4 && active) ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
  for (int i = threadIdx.x + 8 * blockDim.x; i < n4; i += blockDim.x) {   // n > 8192 tail
    float4 t = active ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
  }
  s = block_sum(s, red);
  const float inv = active ? 1.0f / sqrtf(s / (float)n + eps) : 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int i = threadIdx.x + j * blockDim.x;
    if (i < n4) Vec4<T>::store(o + 4 * i, v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv);
  }
  for (int i = threadIdx.x + 8 * blockDim.x; i < n4; i += blockDim.x) {
    float4 t = active ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    Vec4<T>::store(o + 4 * i, t.x * inv, t.y * inv, t.z * inv, t.w * inv);
  }
}

void launch_rmsnorm(const float* x, int M, int n, float eps, void* out, DType dt, const int32_t* pos,
                    cudaStream_t st) {
  const L2Pf pf = take_l2pf();
  if (M <= 0) return;
  if (dt == DT_F32) launch_k(rmsnorm_kernel<float>, M, 256, 0, st, x, n, eps, (float*)out, pos, pf);
  else launch_k(rmsnorm_kernel<bf16>, M, 256, 0, st, x, n, eps, (bf16*)out, pos, pf);
}

// ------------------------------------------------------------------ embedding
template <typename T>
__global__ void embed_kernel(const T* __restrict__ E, const int32_t* __restrict__ tok,
                             const int32_t* __restrict__ pos, int n, float* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x;
  float* xr = x + (size_t)r * n;
  const bool active = !(pos && pos[r] < 0);
  const T* e = E + (size_t)(active ? tok[r] : 0) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) xr[i] = active ? to_f32(e[i]) : 0.f;
}

void launch_embed(const void* E, DType dt, const int32_t* tok, const int32_t* pos, int M, int n, float* x,
                  cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32) launch_k(embed_kernel<float>, M, 256, 0, st, (const float*)E, tok, pos, n, x);
  else launch_k(embed_kernel<bf16>, M, 256, 0, st, (const bf16*)E, tok, pos, n, x);
}

// ------------------------------------------------------------------ RoPE + KV write
// qkv row layout: [q (Hq*hd) | k (Hkv*hd) | v (Hkv*hd)], fp32 from the GEMM.
// Llama rotate_half convention: x' = x*cos + rotate_half(x)*sin with angle
// pos * theta^(-2i/hd); cos/sin tables precomputed on the host in double.
// grid (M, Hq + 2*Hkv): one CTA per (row, head); K/V go to the paged cache
// (V transposed, see KVLayer).
// One CTA per row: thread t handles rotation pairs (head, j) strided over the
// row's q and k heads, then the v head dims; the fp32 scratch row is re-zeroed
// after the CTA has read it (so the next tcgen05 GEMM into it needs no memset).
int num_sms();   // gemm_tc.cu (cached device SM count)
constexpr int ROPE_PARTS = 8;     // max q/k CTAs per row (fewer when M is large, see the launcher)
constexpr int VROWS = 32;         // rows per V-transpose CTA

// V rows -> the transposed cache V^T [hd][page_size] per (page, kv head): a CTA
// takes a 32-row x 32-dim tile of one kv head, reads it along hd (lane = dim,
// 128-byte rows; all 8 loads of a thread issued before its zeroing stores) into
// shared memory and writes it along the rows (lane = row), so consecutive
// lanes hit consecutive slots -- contiguous for a tree / prompt chunk, whose
// rows sit at consecutive cache positions.
// 4 consecutive elements (8-byte aligned for bf16, 16-byte for fp32)
template <typename T> HSD_DEV void store4(T* d, float4 v);
template <> HSD_DEV void store4<float>(float* d, float4 v) { *(float4*)d = v; }
template <> HSD_DEV void store4<bf16>(bf16* d, float4 v) {
  const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  *(uint2*)d = make_uint2(*(const uint32_t*)&a, *(const uint32_t*)&b);
}

template <typename T>
__device__ void v_transpose_block(float* __restrict__ qkv, const RowMeta& m, int M, int Hq, const KVLayer& kv,
                                  int vb, int zero) {
  const int hd = kv.head_dim, Hkv = kv.kv_heads, ld = (Hq + 2 * Hkv) * hd;
  const int nd = (hd + 31) / 32;
  const int dc = vb % nd, h = (vb / nd) % Hkv, r0 = (vb / nd / Hkv) * VROWS;
  __shared__ float tile[VROWS][33];
  __shared__ int pg[VROWS], sl[VROWS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;   // 4 warps
  const int nr = min(VROWS, M - r0), d = dc * 32 + lane;
  if (threadIdx.x < VROWS) {
    const int r = r0 + threadIdx.x;
    int page = -1, slot = 0;
    if (threadIdx.x < nr && m.pos[r] >= 0) {
      const int kp = m.kvpos[r];
      page = kv.block_table[(size_t)m.req[r] * kv.pages_per_req + kp / kv.page_size];
      slot = kp % kv.page_size;
    }
    pg[threadIdx.x] = page;
    sl[threadIdx.x] = slot;
  }
  float v[VROWS / 4];
  float* src = qkv + (size_t)r0 * ld + (Hq + Hkv) * hd + h * hd + d;
#pragma unroll
  for (int k = 0; k < VROWS / 4; ++k) {
    const int rr = w + 4 * k;
    v[k] = (rr < nr && d < hd) ? src[(size_t)rr * ld] : 0.f;
  }
#pragma unroll
  for (int k = 0; k < VROWS / 4; ++k) {
    const int rr = w + 4 * k;
    if (zero && rr < nr && d < hd) src[(size_t)rr * ld] = 0.f;    // re-zero the GEMM scratch (see below)
    tile[rr][lane] = v[k];
  }
  __syncthreads();
  T* base = (T*)kv.base;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dd = dc * 32 + w + 4 * k;           // lane = row
    if (lane < nr && pg[lane] >= 0 && dd < hd)
      base[kv_offset(pg[lane], 1, Hkv, h, kv.page_size, hd, sl[lane], dd)] = from_f32<T>(tile[lane][w + 4 * k]);
  }
}

template <typename T>
__global__ void __launch_bounds__(128) qkv_rope_kv_kernel(float* __restrict__ qkv, RowMeta m,
                                                          const float* __restrict__ rc,
                                                          const float* __restrict__ rs, int Hq, KVLayer kv,
                                                          T* __restrict__ q_out, int M, int zero, int nparts_,
                                                          L2Pf pf) {
  l2pf_issue(pf);
  pdl_wait();
  l2pf_issue(pf, 1);
  pdl_trigger();
  const int n_v = (M + VROWS - 1) / VROWS * kv.kv_heads * ((kv.head_dim + 31) / 32);
  if ((int)blockIdx.x < n_v) {          // V-transpose CTAs first (fewer, longer), then rope
    v_transpose_block<T>(qkv, m, M, Hq, kv, blockIdx.x, zero);
    return;
  }
  const int rb = blockIdx.x - n_v;
  const int nparts = nparts_, r = rb / nparts, part = rb % nparts;
  const int hd = kv.head_dim, half = hd / 2, Hkv = kv.kv_heads;
  const int ld = (Hq + 2 * Hkv) * hd;
  float* row = qkv + (size_t)r * ld;
  const int tid = part * blockDim.x + threadIdx.x, nthr = nparts * blockDim.x;
  const int p = m.pos[r];
  T* qo = q_out + (size_t)r * Hq * hd;
  if (p < 0) {
    for (int i = tid; i < Hq * hd; i += nthr) qo[i] = from_f32<T>(0.f);
  } else {
    const float* c = rc + (size_t)p * half;
    const float* sn = rs + (size_t)p * half;
    const int kp = m.kvpos[r];
    const int page = kv.block_table[(size_t)m.req[r] * kv.pages_per_req + kp / kv.page_size];
    const int slot = kp % kv.page_size;
    T* base = (T*)kv.base;
    // rotated q (Hq heads) and k (Hkv heads): (Hq + Hkv) * half rotation pairs.
    // All of a thread's loads are issued before its first store (up to RP pairs per
    // pass): the stores go through pointers the compiler cannot prove disjoint from
    // the scratch row, so an interleaved loop serialised one memory round trip per
    // pair (c4: 5 pairs per thread, qkv_rope ~1 ms per layer in the launch list)
    constexpr int RP = 8;
    const int npairs = (Hq + Hkv) * half;
    if ((half & 3) == 0) {
      // 4 consecutive rotation pairs per item: float4 loads of both halves and of the
      // cos / sin rows, 4-element stores (8 bytes of bf16)
      const int nq4 = npairs / 4, half4 = half / 4;
      constexpr int RQ = 4;
      for (int i0 = tid; i0 < nq4; i0 += RQ * nthr) {
        float4 x1[RQ], x2[RQ], cc[RQ], ss[RQ];
#pragma unroll
        for (int u = 0; u < RQ; ++u) {
          const int i = i0 + u * nthr;
          if (i < nq4) {
            const int h = i / half4, j = (i % half4) * 4;
            x1[u] = *(const float4*)(row + h * hd + j);
            x2[u] = *(const float4*)(row + h * hd + j + half);
            cc[u] = *(const float4*)(c + j);
            ss[u] = *(const float4*)(sn + j);
          }
        }
#pragma unroll
        for (int u = 0; u < RQ; ++u) {
          const int i = i0 + u * nthr;
          if (i >= nq4) break;
          const int h = i / half4, j = (i % half4) * 4;
          const float4 a = x1[u], b2 = x2[u], co = cc[u], si = ss[u];
          const float4 y1 = make_float4(a.x * co.x - b2.x * si.x, a.y * co.y - b2.y * si.y, a.z * co.z - b2.z * si.z,
                                        a.w * co.w - b2.w * si.w);
          const float4 y2 = make_float4(b2.x * co.x + a.x * si.x, b2.y * co.y + a.y * si.y, b2.z * co.z + a.z * si.z,
                                        b2.w * co.w + a.w * si.w);
          T* d1;
          T* d2;
          if (h < Hq) {
            d1 = qo + h * hd + j;
            d2 = d1 + half;
          } else {
            d1 = base + kv_offset(page, 0, Hkv, h - Hq, kv.page_size, hd, slot, j);
            d2 = d1 + half;
          }
          store4<T>(d1, y1);
          store4<T>(d2, y2);
        }
      }
    } else
    for (int i0 = tid; i0 < npairs; i0 += RP * nthr) {
      float x1[RP], x2[RP], cc[RP], ss[RP];
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int i = i0 + u * nthr;
        if (i < npairs) {
          const int h = i / half, j = i % half;
          x1[u] = row[h * hd + j];
          x2[u] = row[h * hd + j + half];
          cc[u] = c[j];
          ss[u] = sn[j];
        }
      }
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int i = i0 + u * nthr;
        if (i >= npairs) break;
        const int h = i / half, j = i % half;
        const float y1 = x1[u] * cc[u] - x2[u] * ss[u], y2 = x2[u] * cc[u] + x1[u] * ss[u];
        if (h < Hq) {
          qo[h * hd + j] = from_f32<T>(y1);
          qo[h * hd + j + half] = from_f32<T>(y2);
        } else {
          base[kv_offset(page, 0, Hkv, h - Hq, kv.page_size, hd, slot, j)] = from_f32<T>(y1);
          base[kv_offset(page, 0, Hkv, h - Hq, kv.page_size, hd, slot, j + half)] = from_f32<T>(y2);
        }
      }
    }
  }
  // Each element was read by exactly this thread (same tid -> same indices), so
  // re-zeroing the scratch needs no cross-CTA barrier: zero what this thread read.
  if (!zero) return;   // a data-parallel GEMM stored (not accumulated) this scratch
  if (p >= 0 && (half & 3) == 0) {   // the quads this thread read (vectorised path above)
    const int half4 = half / 4;
    for (int i = tid; i < (Hq + Hkv) * half4; i += nthr) {
      const int h = i / half4, j = (i % half4) * 4;
      *(float4*)(row + h * hd + j) = make_float4(0.f, 0.f, 0.f, 0.f);
      *(float4*)(row + h * hd + j + half) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (p >= 0) {
    for (int i = tid; i < (Hq + Hkv) * half; i += nthr) {
      const int h = i / half, j = i % half;
      row[h * hd + j] = 0.f;
      row[h * hd + j + half] = 0.f;
    }
  } else {
    for (int i = tid; i < (Hq + Hkv) * hd; i += nthr) row[i] = 0.f;   // V columns: the V CTAs
  }
}

void launch_qkv_rope_kv(float* qkv, int M, const RowMeta& m, const float* rope_cos,
                        const float* rope_sin, int Hq, const KVLayer& kv, void* q_out, DType dt,
                        cudaStream_t st, bool zero) {
  const L2Pf pf = take_l2pf();
  if (M <= 0) return;
  // q/k CTAs per row: 8 at decode sizes (c2: M = 65, latency-bound, spread wide);
  // at large M a row per CTA -- c3's 2080 x 8 tiny CTAs spent more time in CTA
  // turnaround and the per-CTA metadata chain than in their 2.5 pairs per thread
  static const int parts_env = [] { const char* e = getenv("HSD_ROPE_PARTS"); return e ? atoi(e) : 0; }();
  const int nparts = parts_env > 0 ? std::min(parts_env, ROPE_PARTS)
                                   : std::max(1, std::min(ROPE_PARTS, (num_sms() * 8) / std::max(M, 1)));
  const int grid = M * nparts + (M + VROWS - 1) / VROWS * kv.kv_heads * ((kv.head_dim + 31) / 32);
  if (dt == DT_F32)
    launch_k(qkv_rope_kv_kernel<float>, dim3(grid), 128, 0, st, qkv, m, rope_cos, rope_sin, Hq, kv, (float*)q_out, M, zero ? 1 : 0, nparts, pf);
  else
    launch_k(qkv_rope_kv_kernel<bf16>, dim3(grid), 128, 0, st, qkv, m, rope_cos, rope_sin, Hq, kv, (bf16*)q_out, M, zero ? 1 : 0, nparts, pf);
}

// ------------------------------------------------------------------ SwiGLU
// gu row = 2f values with gate/up INTERLEAVED in GU_GROUP (16) feature groups
// (weight rows of W_gu are stored that way so the data-parallel tcgen05 GEMM can
// fuse SwiGLU into its epilogue: a 32-row TMEM lane quarter holds 16 gates and
// their 16 ups, exchanged by one warp shuffle): feature i's gate is column
// 2*GU_GROUP*(i/GU_GROUP) + i%GU_GROUP and its up value GU_GROUP columns later.
// out[i] = silu(gate) * up. grid (M, f/4/256), f % 64 == 0.
template <typename T>
__global__ void swiglu_kernel(float* __restrict__ gu, int f, T* __restrict__ out,
                              const int32_t* __restrict__ pos, L2Pf pf) {
  l2pf_issue(pf);
  pdl_wait();
  l2pf_issue(pf, 1);
  pdl_trigger();
  const int r = blockIdx.x;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;   // float4 index
  if (4 * i >= f) return;
  const int col = 2 * GU_GROUP * ((4 * i) / GU_GROUP) + (4 * i) % GU_GROUP;
  float4* ga = (float4*)(gu + (size_t)r * 2 * f + col);
  float4* gb = (float4*)(gu + (size_t)r * 2 * f + col + GU_GROUP);
  const float4 a = *ga, u = *gb;
  *ga = make_float4(0.f, 0.f, 0.f, 0.f);   // re-zero the GEMM scratch (see qkv_rope_kv)
  *gb = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool active = pos == nullptr || pos[r] >= 0;
  auto sl = [](float x) { return x / (1.0f + expf(-x)); };
  if (active) Vec4<T>::store(out + (size_t)r * f + 4 * i, sl(a.x) * u.x, sl(a.y) * u.y, sl(a.z) * u.z, sl(a.w) * u.w);
  else Vec4<T>::store(out + (size_t)r * f + 4 * i, 0.f, 0.f, 0.f, 0.f);
}

void launch_swiglu(float* gu, int M, int f, void* out, DType dt, const int32_t* pos, cudaStream_t st) {
  const L2Pf pf = take_l2pf();
  if (M <= 0) return;
  dim3 grid(M, (f / 4 + 255) / 256);
  if (dt == DT_F32) launch_k(swiglu_kernel<float>, grid, 256, 0, st, gu, f, (float*)out, pos, pf);
  else launch_k(swiglu_kernel<bf16>, grid, 256, 0, st, gu, f, (bf16*)out, pos, pf);
}

// gate rows [0,f) and up rows [f,2f) of src -> interleaved GU_GROUP-row groups in dst
template <typename T>
__global__ void interleave_gu_kernel(const T* __restrict__ src, int f, int n, T* __restrict__ dst) {
  const int r = blockIdx.x;                       // destination row
  const int g = r / (2 * GU_GROUP), o = r % (2 * GU_GROUP);
  const int srow = o < GU_GROUP ? g * GU_GROUP + o : f + g * GU_GROUP + (o - GU_GROUP);
  for (int c = threadIdx.x; c < n; c += blockDim.x) dst[(size_t)r * n + c] = src[(size_t)srow * n + c];
}

void launch_interleave_gu(const void* src, int f, int n, void* dst, DType dt, cudaStream_t st) {
  if (dt == DT_F32) interleave_gu_kernel<float><<<2 * f, 256, 0, st>>>((const float*)src, f, n, (float*)dst);
  else interleave_gu_kernel<bf16><<<2 * f, 256, 0, st>>>((const bf16*)src, f, n, (bf16*)dst);
}

// ------------------------------------------------------------------ argmax
// lowest index among maxima (reading R8)
__global__ void argmax_rows_kernel(const float* __restrict__ x, int V, const int32_t* __restrict__ pos,
                                   int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  int r = blockIdx.x;
  if (pos && pos[r] < 0) {
    if (threadIdx.x == 0) out[r] = -1;
    return;
  }
  const float* xr = x + (size_t)r * V;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    float v = xr[i];
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
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
    if (lane == 0) out[r] = bi;
  }
}

// token-level AR draft input (EAGLE-style, R27): t = argmax of the draft logits row
// (columns in rank order when perm != null; ties -> lowest TOKEN id), then the fc
// input row [h_i ; E(t)] (h from the fp32 chain state)
template <typename T>
__global__ void token_ar_input_kernel(const float* __restrict__ L, size_t ldl, int V, const int32_t* __restrict__ perm,
                                      const float* __restrict__ h, int n, const T* __restrict__ E, T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  const int r = blockIdx.x;
  const float* xr = L + (size_t)r * ldl;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const int t = perm ? perm[i] : i;
    if (better(xr[i], t, bv, bi)) { bv = xr[i]; bi = t; }
  }
  warp_argmax(bv, bi);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
    warp_argmax(bv, bi);
    if (lane == 0) si[0] = bi;
  }
  __syncthreads();
  const int tok = si[0];
  T* o = out + (size_t)r * 2 * n;
  const T* e = E + (size_t)tok * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    o[i] = from_f32<T>(h[(size_t)r * n + i]);
    o[n + i] = e[i];
  }
}

void launch_token_ar_input(const float* L, size_t ldl, int V, const int32_t* perm, const float* h, int M, int n,
                           const void* E, DType dt, void* out, cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32)
    launch_k(token_ar_input_kernel<float>, M, 1024, 0, st, L, ldl, V, perm, h, n, (const float*)E, (float*)out);
  else
    launch_k(token_ar_input_kernel<bf16>, M, 1024, 0, st, L, ldl, V, perm, h, n, (const bf16*)E, (bf16*)out);
}

void launch_argmax_rows(const float* x, int M, int V, const int32_t* pos, int32_t* out, cudaStream_t st) {
  if (M <= 0) return;
  launch_k(argmax_rows_kernel, M, 1024, 0, st, x, V, pos, out);
}

// ------------------------------------------------------------------ draft input
// out[r] = [H_{j-1} (fp32 -> T) ; E(t_j)]   (W_fc input, reading R1)
template <typename T>
__global__ void draft_concat_kernel(const float* __restrict__ Hprev, const int32_t* __restrict__ tok,
                                    const int32_t* __restrict__ pos, const int32_t* __restrict__ slot,
                                    const T* __restrict__ E, int n, T* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x;
  T* o = out + (size_t)r * 2 * n;
  bool active = pos[r] >= 0;
  const bool with_e = !(slot && slot[r] == -2);   // -2: the root pair without its token (R26)
  const float* h = Hprev + (size_t)r * n;
  const T* e = E + (size_t)(active ? tok[r] : 0) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    o[i] = active ? from_f32<T>(h[i]) : from_f32<T>(0.f);
    o[n + i] = active && with_e ? e[i] : from_f32<T>(0.f);
  }
}

void launch_draft_concat(const float* Hprev, const int32_t* tok, const int32_t* pos, const int32_t* slot,
                         const void* E, DType dt, int M, int n, void* out, cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32)
    launch_k(draft_concat_kernel<float>, M, 256, 0, st, Hprev, tok, pos, slot, (const float*)E, n, (float*)out);
  else
    launch_k(draft_concat_kernel<bf16>, M, 256, 0, st, Hprev, tok, pos, slot, (const bf16*)E, n, (bf16*)out);
}
