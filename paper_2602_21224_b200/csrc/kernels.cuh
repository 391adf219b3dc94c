// kernels.cuh -- launcher declarations shared by the engine (product side).
#pragma once
#include <string>
#include "common.cuh"

// Per-row metadata of one forward pass (rows are padded; pos < 0 = inactive).
struct RowMeta {
  const int32_t* tok;    // [M] token (embedding input), may be null
  const int32_t* pos;    // [M] RoPE position, -1 = inactive row
  const int32_t* kvpos;  // [M] cache position the row's K/V is written to
  const int32_t* req;    // [M] request index (block-table row)
  const int32_t* klo;    // [M] unconditional visible keys [klo, khi)
  const int32_t* khi;
  const int32_t* slot;   // [M] tree slot (-1 = none); tree keys at tbase[req] + s
  const int32_t* tbase;  // [b] first cache position of the tree region
  const uint64_t* anc;   // [b, t_max, anc_words] ancestor masks
  int t_max, anc_words;
};

// Paged KV pool of one layer. Block (page p, kind 0=K / 1=V, kv head h) holds
// page_size*hd elements at ((p*2 + kind)*Hkv + h)*page_size*hd:
//   K: element (slot, d) at slot*hd + d      ([page_size][hd], hd contiguous)
//   V: element (slot, d) at d*page_size + slot ([hd][page_size], TRANSPOSED so that
//      V^T tiles are K-major UMMA operands for O += P V in the tcgen05 kernel).
struct KVLayer {
  void* base;
  const int32_t* block_table;  // [b, pages_per_req]
  int pages_per_req, page_size, kv_heads, head_dim;
};

HSD_DEV size_t kv_offset(int page, int kind, int Hkv, int h, int ps, int hd, int slot, int d) {
  size_t blk = (((size_t)page * 2 + kind) * Hkv + h) * (size_t)ps * hd;
  return blk + (kind == 0 ? (size_t)slot * hd + d : (size_t)d * ps + slot);
}

// init.cu
void launch_philox_fill(void* out, DType dt, size_t count, uint32_t seed, uint32_t tid, float scale,
                        cudaStream_t st);
void launch_table_rows_fp8(const float* E, int rows, int V, int Vh, void* table, float* scale, cudaStream_t st);
void launch_table_rows(const float* E, int rows, int V, int Vh, const int32_t* col_of_rank,
                       void* table, DType dt, cudaStream_t st);
void launch_gather_rows_f32(const void* src, DType dt, const int32_t* idx, int rows, int n, float* dst,
                            cudaStream_t st);

// gemm_simt.cu: C[M,N] (+)= A[M,K] W[N,K]^T, fp32 accumulation, fixed k order.
void gemm_simt(const void* A, int lda, const void* W, int ldw, DType dt, float* C, int ldc, int M, int N,
               int K, bool accumulate, cudaStream_t st);

// layers.cu
void launch_rmsnorm(const float* x, int M, int n, float eps, void* out, DType dt, const int32_t* pos,
                    cudaStream_t st);
void launch_embed(const void* E, DType dt, const int32_t* tok, const int32_t* pos, int M, int n, float* x,
                  cudaStream_t st);
// zero: re-zero the fp32 scratch rows after reading them (the stream-K GEMMs
// accumulate into a zero scratch); false when a data-parallel GEMM stored them
void launch_qkv_rope_kv(float* qkv, int M, const RowMeta& m, const float* rope_cos,
                        const float* rope_sin, int Hq, const KVLayer& kv, void* q_out, DType dt,
                        cudaStream_t st, bool zero = true);
void launch_swiglu(float* gu, int M, int f, void* out, DType dt, const int32_t* pos, cudaStream_t st);
void launch_interleave_gu(const void* src, int f, int n, void* dst, DType dt, cudaStream_t st);
void launch_argmax_rows(const float* x, int M, int V, const int32_t* pos, int32_t* out, cudaStream_t st);
void launch_token_ar_input(const float* L, size_t ldl, int V, const int32_t* perm, const float* h, int M, int n,
                           const void* E, DType dt, void* out, cudaStream_t st);
void launch_draft_concat(const float* Hprev, const int32_t* tok, const int32_t* pos, const int32_t* slot,
                         const void* E, DType dt, int M, int n, void* out, cudaStream_t st);

// attention.cu (SIMT, any precision) and attention_tc.cu (tcgen05, bf16, hd 64/128)
bool attention_tc_supported(int hd, int page_size, DType dt);
int launch_attention_tc(const void* q, int M, int rows_per_req, int n_req, const RowMeta& m, const KVLayer& kv,
                        int Hq, int max_keys, void* out, float* ws, size_t ws_floats, size_t kv_layer_elems,
                        cudaStream_t st);
void launch_attention(const void* q, int M, int rows_per_req, int n_req, const RowMeta& m, const KVLayer& kv,
                      int Hq, DType dt, int max_keys, void* out, float* ws, size_t ws_floats,
                      cudaStream_t st);
size_t attention_ws_floats(int M, int Hq, int hd, int max_splits);

// shard.cu: vocab-sharded lm_head -- partial argmax / merge /
// column scatter kernels and the run-time-loaded NCCL entry points
#define HSD_MAX_SHARDS 16
#define HSD_SHARD_KG 16   // Gumbel candidates kept per row and shard (stochastic + vocab shards)
// stochastic acceptance over a vocab-sharded head (shard.cu): per-row records of a
// shard's columns, then their merge into lse / tree-token logits / Gumbel top-KG
void launch_stoch_part(const float* x, int rows, int ld, int w, int col0, int T, const int32_t* tree_tok,
                       const int32_t* req_id, const int32_t* step, uint32_t seed, float temperature, float* out,
                       cudaStream_t st);
void launch_stoch_merge(const float* part, int G, size_t sstride, int row0, int M, int T, float* lse, float* tl,
                        float* gv, int32_t* gi, cudaStream_t st);
size_t stoch_record_floats(int T);
void launch_argmax_part(const float* x, int rows, int ld, int w, int col0, float* outv, int32_t* outi,
                        cudaStream_t st);
void launch_argmax_merge(const float* pv, const int32_t* pi, int S, int stride, int row0, int M,
                         const int32_t* pos, int32_t* out, cudaStream_t st);
void launch_scatter_cols(const float* src, size_t src_stride, int rows, int S, const int* lo, float* dst, int ld,
                         cudaStream_t st);
bool shard_nccl_unique_id(uint8_t* out, std::string& err);
bool shard_nccl_init(void** comm, int nranks, const uint8_t* id_bytes, int rank, std::string& err);
void shard_nccl_destroy(void* comm);
bool shard_allgather(const void* send, void* recv, size_t bytes, void* comm, cudaStream_t st, std::string& err);
bool shard_alltoallv(const char* send, const size_t* send_off, const size_t* send_bytes, char* recv,
                     const size_t* recv_off, const size_t* recv_bytes, int nranks, void* comm, cudaStream_t st,
                     std::string& err);
