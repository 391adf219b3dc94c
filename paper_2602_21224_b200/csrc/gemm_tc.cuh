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
