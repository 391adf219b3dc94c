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
// interleaved in 16-row groups (gate rows g*16.., then the matching up rows),
// H[M, N/2] = silu(gate) * up in bf16. Returns 0 (nothing launched) when the
// shape would not run data-parallel; the caller then uses the plain path.
int gemm_tc_swiglu_bf16(const bf16* A, int lda, const bf16* W, int ldw, bf16* H, int ldh, int M, int N, int K,
                        cudaStream_t st);

// Fused QKV epilogue (verify pass, data-parallel CTA-pair shapes): the QKV GEMM's
// accumulators go straight to RoPE-rotated bf16 q rows and rotated K / plain V
// rows in the paged cache -- the work of qkv_rope_kv, without the fp32 QKV row.
struct QkvEpi {
  const int32_t* pos;          // [M] RoPE position, -1 = inactive row (q row zeroed, no KV write)
  const int32_t* kvpos;        // [M] cache position of the row's K / V
  const int32_t* req;          // [M] block-table row
  const float* rc;             // [max_pos, hd/2] cos
  const float* rs;             // [max_pos, hd/2] sin
  bf16* q_out;                 // [M, Hq, hd]
  void* kv_base;               // KV pool of the layer (see KVLayer)
  const int32_t* block_table;
  int pages_per_req, page_size, Hq, Hkv, hd;
};
bool gemm_tc_qkv_ok(int M, int N, int K, int hd, int Hq, int Hkv);
// returns the number of kernels launched (0: not applicable, nothing launched)
int gemm_tc_qkv_bf16(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K, const QkvEpi& e,
                     cudaStream_t st);
