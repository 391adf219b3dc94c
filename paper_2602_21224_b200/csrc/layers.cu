// layers.cu -- row-wise kernels of the Llama decoder used by draft, verify and
// prefill passes: RMSNorm, embedding gather, RoPE + paged KV write, SwiGLU,
// argmax, draft-input concat (reading R1).
#include "kernels.cuh"

// ------------------------------------------------------------------ RMSNorm
// out[r] = x[r] / sqrt(mean(x[r]^2) + eps) (gain 1). Inactive rows -> 0.
template <typename T>
__global__ void rmsnorm_kernel(const float* __restrict__ x, int n, float eps, T* __restrict__ out,
                               const int32_t* __restrict__ pos) {
  __shared__ float red[32];
  int r = blockIdx.x;
  const float* xr = x + (size_t)r * n;
  T* o = out + (size_t)r * n;
  bool active = pos == nullptr || pos[r] >= 0;
  if (!active) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = from_f32<T>(0.f);
    return;
  }
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += xr[i] * xr[i];
  s = block_sum(s, red);
  float inv = 1.0f / sqrtf(s / (float)n + eps);
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = from_f32<T>(xr[i] * inv);
}

void launch_rmsnorm(const float* x, int M, int n, float eps, void* out, DType dt, const int32_t* pos,
                    cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32) rmsnorm_kernel<float><<<M, 256, 0, st>>>(x, n, eps, (float*)out, pos);
  else rmsnorm_kernel<bf16><<<M, 256, 0, st>>>(x, n, eps, (bf16*)out, pos);
}

// ------------------------------------------------------------------ embedding
template <typename T>
__global__ void embed_kernel(const T* __restrict__ E, const int32_t* __restrict__ tok,
                             const int32_t* __restrict__ pos, int n, float* __restrict__ x) {
  int r = blockIdx.x;
  float* xr = x + (size_t)r * n;
  if (pos && pos[r] < 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) xr[i] = 0.f;
    return;
  }
  const T* e = E + (size_t)tok[r] * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) xr[i] = to_f32(e[i]);
}

void launch_embed(const void* E, DType dt, const int32_t* tok, const int32_t* pos, int M, int n, float* x,
                  cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32) embed_kernel<float><<<M, 256, 0, st>>>((const float*)E, tok, pos, n, x);
  else embed_kernel<bf16><<<M, 256, 0, st>>>((const bf16*)E, tok, pos, n, x);
}

// ------------------------------------------------------------------ RoPE + KV write
// qkv row layout: [q (Hq*hd) | k (Hkv*hd) | v (Hkv*hd)], fp32 from the GEMM.
// Llama rotate_half convention: x' = x*cos + rotate_half(x)*sin with angle
// pos * theta^(-2i/hd); cos/sin tables precomputed on the host in double.
template <typename T>
__global__ void qkv_rope_kv_kernel(const float* __restrict__ qkv, RowMeta m, const float* __restrict__ rc,
                                   const float* __restrict__ rs, int Hq, KVLayer kv, T* __restrict__ q_out) {
  int r = blockIdx.x;
  int hd = kv.head_dim, half = hd / 2, Hkv = kv.kv_heads;
  int ld = (Hq + 2 * Hkv) * hd;
  const float* row = qkv + (size_t)r * ld;
  int p = m.pos[r];
  T* qo = q_out + (size_t)r * Hq * hd;
  if (p < 0) {
    for (int i = threadIdx.x; i < Hq * hd; i += blockDim.x) qo[i] = from_f32<T>(0.f);
    return;
  }
  const float* c = rc + (size_t)p * half;
  const float* s = rs + (size_t)p * half;
  // q heads
  for (int i = threadIdx.x; i < Hq * half; i += blockDim.x) {
    int h = i / half, j = i % half;
    float x1 = row[h * hd + j], x2 = row[h * hd + j + half];
    qo[h * hd + j] = from_f32<T>(x1 * c[j] - x2 * s[j]);
    qo[h * hd + j + half] = from_f32<T>(x2 * c[j] + x1 * s[j]);
  }
  // k (rotated) and v into the paged cache at kvpos
  int kp = m.kvpos[r];
  int page = kv.block_table[(size_t)m.req[r] * kv.pages_per_req + kp / kv.page_size];
  int slot = kp % kv.page_size;
  T* base = (T*)kv.base;
  for (int i = threadIdx.x; i < Hkv * half; i += blockDim.x) {
    int h = i / half, j = i % half;
    const float* kr = row + Hq * hd + h * hd;
    float x1 = kr[j], x2 = kr[j + half];
    size_t off = ((((size_t)page * 2 + 0) * Hkv + h) * kv.page_size + slot) * hd;
    base[off + j] = from_f32<T>(x1 * c[j] - x2 * s[j]);
    base[off + j + half] = from_f32<T>(x2 * c[j] + x1 * s[j]);
  }
  for (int i = threadIdx.x; i < Hkv * hd; i += blockDim.x) {
    int h = i / hd, j = i % hd;
    size_t off = ((((size_t)page * 2 + 1) * Hkv + h) * kv.page_size + slot) * hd;
    base[off + j] = from_f32<T>(row[(Hq + Hkv) * hd + i]);
  }
}

void launch_qkv_rope_kv(const float* qkv, int M, const RowMeta& m, const float* rope_cos,
                        const float* rope_sin, int Hq, const KVLayer& kv, void* q_out, DType dt,
                        cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32)
    qkv_rope_kv_kernel<float><<<M, 128, 0, st>>>(qkv, m, rope_cos, rope_sin, Hq, kv, (float*)q_out);
  else
    qkv_rope_kv_kernel<bf16><<<M, 128, 0, st>>>(qkv, m, rope_cos, rope_sin, Hq, kv, (bf16*)q_out);
}

// ------------------------------------------------------------------ SwiGLU
// gu row = [gate (f) | up (f)] -> silu(gate) * up
template <typename T>
__global__ void swiglu_kernel(const float* __restrict__ gu, int f, T* __restrict__ out,
                              const int32_t* __restrict__ pos) {
  int r = blockIdx.x;
  const float* g = gu + (size_t)r * 2 * f;
  T* o = out + (size_t)r * f;
  bool active = pos == nullptr || pos[r] >= 0;
  for (int i = threadIdx.x; i < f; i += blockDim.x) {
    float a = g[i], u = g[f + i];
    o[i] = from_f32<T>(active ? (a / (1.0f + expf(-a))) * u : 0.f);
  }
}

void launch_swiglu(const float* gu, int M, int f, void* out, DType dt, const int32_t* pos, cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32) swiglu_kernel<float><<<M, 256, 0, st>>>(gu, f, (float*)out, pos);
  else swiglu_kernel<bf16><<<M, 256, 0, st>>>(gu, f, (bf16*)out, pos);
}

// ------------------------------------------------------------------ argmax
// lowest index among maxima (reading R8)
__global__ void argmax_rows_kernel(const float* __restrict__ x, int V, const int32_t* __restrict__ pos,
                                   int32_t* __restrict__ out) {
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

void launch_argmax_rows(const float* x, int M, int V, const int32_t* pos, int32_t* out, cudaStream_t st) {
  if (M <= 0) return;
  argmax_rows_kernel<<<M, 512, 0, st>>>(x, V, pos, out);
}

// ------------------------------------------------------------------ draft input
// out[r] = [H_{j-1} (fp32 -> T) ; E(t_j)]   (W_fc input, reading R1)
template <typename T>
__global__ void draft_concat_kernel(const float* __restrict__ Hprev, const int32_t* __restrict__ tok,
                                    const int32_t* __restrict__ pos, const T* __restrict__ E, int n,
                                    T* __restrict__ out) {
  int r = blockIdx.x;
  T* o = out + (size_t)r * 2 * n;
  bool active = pos[r] >= 0;
  const float* h = Hprev + (size_t)r * n;
  const T* e = E + (size_t)(active ? tok[r] : 0) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    o[i] = active ? from_f32<T>(h[i]) : from_f32<T>(0.f);
    o[n + i] = active ? e[i] : from_f32<T>(0.f);
  }
}

void launch_draft_concat(const float* Hprev, const int32_t* tok, const int32_t* pos, const void* E,
                         DType dt, int M, int n, void* out, cudaStream_t st) {
  if (M <= 0) return;
  if (dt == DT_F32)
    draft_concat_kernel<float><<<M, 256, 0, st>>>(Hprev, tok, pos, (const float*)E, n, (float*)out);
  else
    draft_concat_kernel<bf16><<<M, 256, 0, st>>>(Hprev, tok, pos, (const bf16*)E, n, (bf16*)out);
}
