// gemm_simt.cu -- SIMT FFMA GEMM, C[M,N] (+)= A[M,K] W[N,K]^T.
// The fp32-verify path: every output accumulates k = 0..K-1 in
// order with one FFMA per step (no split-K), so results are deterministic and
// independent of the launch shape. Also the fallback for bf16 when tcgen05 is
// disabled. Operands are K-major (nn.Linear layout).
#include "kernels.cuh"

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ A, int lda,
                                                        const T* __restrict__ W, int ldw,
                                                        float* __restrict__ C, int ldc, int M, int N, int K,
                                                        int accumulate) {
  pdl_wait();
  pdl_trigger();
  __shared__ float As[BK][BM + 4];
  __shared__ float Ws[BK][BN + 4];
  int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  int lr = tid >> 2, lk = (tid & 3) * 4;
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int k = k0 + lk + i;
      int am = m0 + lr, wn = n0 + lr;
      As[lk + i][lr] = (am < M && k < K) ? to_f32(A[(size_t)am * lda + k]) : 0.f;
      Ws[lk + i][lr] = (wn < N && k < K) ? to_f32(W[(size_t)wn * ldw + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float* c = C + (size_t)m * ldc + n;
      *c = accumulate ? *c + acc[i][j] : acc[i][j];
    }
  }
}
}  // namespace

void gemm_simt(const void* A, int lda, const void* W, int ldw, DType dt, float* C, int ldc, int M, int N,
               int K, bool accumulate, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  if (dt == DT_F32)
    launch_k(gemm_simt_kernel<float>, grid, 256, 0, st, (const float*)A, lda, (const float*)W, ldw, C, ldc, M, N, K,
                                                  accumulate);
  else
    launch_k(gemm_simt_kernel<bf16>, grid, 256, 0, st, (const bf16*)A, lda, (const bf16*)W, ldw, C, ldc, M, N, K,
                                                 accumulate);
}
