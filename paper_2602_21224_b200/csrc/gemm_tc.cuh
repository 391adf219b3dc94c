// gemm_tc.cuh -- tcgen05 (5th-gen tensor core) bf16 GEMM, C[M,N] (+)= A[M,K] W[N,K]^T.
#pragma once
#include "common.cuh"

bool gemm_tc_supported(int M, int N, int K, int lda, int ldw);
// returns the number of kernels launched
// accumulate=false && c_zeroed=false: C is cleared first (memset); c_zeroed=true
// promises C is already zero (the engine's scratch buffers are re-zeroed by
// their consumer kernels), which saves the memset node.
int gemm_tc_bf16(const bf16* A, int lda, const bf16* W, int ldw, float* C, int ldc, int M, int N, int K,
                 bool accumulate, cudaStream_t st, bool c_zeroed = false);
// true when the GEMM runs data-parallel (at least one output tile per SM)
// K / accumulate: 0 / false when unknown (store epilogue)
bool gemm_tc_dp(int M, int N, int K = 0, bool accumulate = false);
// the gate/up GEMM can fuse SwiGLU into its epilogue (data-parallel shapes)
bool gemm_tc_swiglu_ok(int M, int N, int K);
// data-parallel gate/up GEMM with the SwiGLU fused into the epilogue: W rows are
// interleaved in 64-row groups (gate rows g*64.., then the matching up rows),
// H[M, N/2] = silu(gate) * up in bf16. Returns 0 (nothing launched) when the
// shape would not run data-parallel; the caller then uses the plain path.
int gemm_tc_swiglu_bf16(const bf16* A, int lda, const bf16* W, int ldw, bf16* H, int ldh, int M, int N, int K,
                        cudaStream_t st);
