// init.cu -- on-device weight generation (Philox4x32-10, reading R23) and the
// token-info table build (PAPER.md:290-296 collapse, :223 RMSNorm, :404-406
// hot-token sparsity, reading R5).
#include "kernels.cuh"

// w[e] = fp32(scale) * (2u - 1), u = (x>>8) * 2^-24, x = word e%4 of
// Philox(counter = (e/4 lo, e/4 hi, 0, 0), key = (seed, tid)).
template <typename T>
__global__ void philox_fill_kernel(T* __restrict__ out, size_t count, uint32_t seed, uint32_t tid,
                                   float scale) {
  size_t nblk = (count + 3) / 4;
  for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < nblk; b += (size_t)gridDim.x * blockDim.x) {
    u32x4 c = {(uint32_t)(b & 0xffffffffu), (uint32_t)(b >> 32), 0u, 0u};
    u32x4 r = philox4x32_10(c, seed, tid);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      size_t e = b * 4 + i;
      if (e < count) {
        float u = (float)(lane_of(r, i) >> 8) * 5.9604644775390625e-08f;
        float t = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);   // exact
        out[e] = from_f32<T>(__fmul_rn(scale, t));
      }
    }
  }
}

void launch_philox_fill(void* out, DType dt, size_t count, uint32_t seed, uint32_t tid, float scale,
                        cudaStream_t st) {
  size_t nblk = (count + 3) / 4;
  int grid = (int)((nblk + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  if (dt == DT_F32) philox_fill_kernel<float><<<grid, 256, 0, st>>>((float*)out, count, seed, tid, scale);
  else philox_fill_kernel<bf16><<<grid, 256, 0, st>>>((bf16*)out, count, seed, tid, scale);
}

// Table rows: E' chunk [rows, V] fp32 with columns in rank order -> RMSNorm over
// the FULL row (eps 1e-6, no gain, R4) -> keep the first Vh (hot) columns.
template <typename T>
__global__ void table_rows_kernel(const float* __restrict__ E, int V, int Vh, T* __restrict__ table) {
  __shared__ float red[32];
  int r = blockIdx.x;
  const float* e = E + (size_t)r * V;
  float s = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += e[i] * e[i];
  s = block_sum(s, red);
  float inv = 1.0f / sqrtf(s / (float)V + 1e-6f);
  T* o = table + (size_t)r * Vh;
  for (int i = threadIdx.x; i < Vh; i += blockDim.x) o[i] = from_f32<T>(e[i] * inv);
}

// FP8 variant (reading R25): the same RMSNorm row, then one scale per row
// s = max_j |row[j]| / 448 over the stored (hot) columns and e4m3 codes
// RNE(row / s) with saturation (cvt.rn.satfinite.e4m3x2.f32).
__global__ void table_rows_fp8_kernel(const float* __restrict__ E, int V, int Vh, __nv_fp8_storage_t* __restrict__ table,
                                      float* __restrict__ scale) {
  __shared__ float red[32];
  __shared__ float s_sc;
  int r = blockIdx.x;
  const float* e = E + (size_t)r * V;
  float s = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += e[i] * e[i];
  s = block_sum(s, red);
  const float inv = 1.0f / sqrtf(s / (float)V + 1e-6f);
  float amax = 0.f;
  for (int i = threadIdx.x; i < Vh; i += blockDim.x) amax = fmaxf(amax, fabsf(e[i] * inv));
  amax = block_max(amax, red);
  if (threadIdx.x == 0) {
    s_sc = amax > 0.f ? amax / 448.0f : 1.0f;
    scale[r] = s_sc;
  }
  __syncthreads();
  const float sc = s_sc;
  __nv_fp8_storage_t* o = table + (size_t)r * Vh;
  for (int i = threadIdx.x; i < Vh; i += blockDim.x)
    o[i] = __nv_cvt_float_to_fp8(__fdiv_rn(e[i] * inv, sc), __NV_SATFINITE, __NV_E4M3);
}

void launch_table_rows_fp8(const float* E, int rows, int V, int Vh, void* table, float* scale, cudaStream_t st) {
  if (rows <= 0) return;
  table_rows_fp8_kernel<<<rows, 512, 0, st>>>(E, V, Vh, (__nv_fp8_storage_t*)table, scale);
}

void launch_table_rows(const float* E, int rows, int V, int Vh, const int32_t* /*unused*/, void* table,
                       DType dt, cudaStream_t st) {
  if (rows <= 0) return;
  if (dt == DT_F32) table_rows_kernel<float><<<rows, 512, 0, st>>>(E, V, Vh, (float*)table);
  else table_rows_kernel<bf16><<<rows, 512, 0, st>>>(E, V, Vh, (bf16*)table);
}

// dst[r] = src[idx[r]] as fp32 (idx = null -> identity)
template <typename T>
__global__ void gather_rows_f32_kernel(const T* __restrict__ src, const int32_t* __restrict__ idx, int n,
                                       float* __restrict__ dst) {
  int r = blockIdx.x;
  const T* s = src + (size_t)(idx ? idx[r] : r) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[(size_t)r * n + i] = to_f32(s[i]);
}

void launch_gather_rows_f32(const void* src, DType dt, const int32_t* idx, int rows, int n, float* dst,
                            cudaStream_t st) {
  if (rows <= 0) return;
  if (dt == DT_F32) gather_rows_f32_kernel<float><<<rows, 256, 0, st>>>((const float*)src, idx, n, dst);
  else gather_rows_f32_kernel<bf16><<<rows, 256, 0, st>>>((const bf16*)src, idx, n, dst);
}
