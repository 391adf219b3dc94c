// accept.cuh -- parameters of the S3/S4 kernels (accept.cu).
#pragma once
#include "common.cuh"

struct AcceptParams {
  int mode;                 // 0 greedy, 1 stochastic
  int append;               // 1: the dedicated verify of the re-sampled tree (fusion off): tokens go
                            // after the step's first n_emitted; a request with t_n == 0 is skipped
                            // (acc_n = -1)
  int N, t_max, V;
  float temperature;
  uint32_t seed;
  const int32_t* req_id;    // [b] global request id per slot (random streams)
  const int32_t *t_tok, *t_par, *t_n;
  const int32_t* argmax;    // [b, t_max] (greedy)
  const float* logits;      // [b, t_max, V] (stochastic)
  // stochastic with a vocab-sharded head (no full logits rows): per verify row the
  // merged lse of l / T, the tree-token logits [t_max], the Gumbel top-KG (value desc)
  const float *sh_lse, *sh_tl, *sh_gv;
  const int32_t* sh_gi;
  const int32_t* step;
  int32_t *acc_n, *acc_slots, *bonus, *emitted, *n_emitted;
};

struct CompactParams {
  void* kv_base;            // layer 0 base; layer l at + l * layer_stride elements
  size_t layer_stride;
  const int32_t* block_table;
  int pages_per_req, page_size, kv_heads, head_dim, N;
  const int32_t *acc_n, *acc_slots, *p;
};

struct CommitParams {
  int N, t_max, hidden;
  int append;               // 1: draft pairs appended after the step's first n_pend (acc_n < 0: skip)
  const float* Hverify;     // [b, t_max, n]
  const int32_t *acc_n, *acc_slots, *emitted, *bonus, *n_emitted;
  float* pend_H;            // [b, N+1, n]
  int32_t *pend_tok, *n_pend, *root_tok, *p, *step;
};

void launch_walk(const AcceptParams& P, int n_req, cudaStream_t st);
// the Alg. 2 pending tree [b, Br+1] (creation order) as a verify tree [b, t_max]:
// BFS, siblings by (log-joint desc, token asc) (R8), ancestor bitmasks; t_n = 0
// for a request without a re-sampled tree
void launch_pending_as_tree(const int32_t* pt_n, const int32_t* pt_tok, const int32_t* pt_par,
                            const int32_t* pt_depth, const float* pt_lj, int br1, int32_t* t_n, int32_t* t_tok,
                            int32_t* t_par, int32_t* t_depth, float* t_lj, uint64_t* t_anc, int t_max, int anc_words,
                            int n_req, cudaStream_t st);
void launch_compact(const CompactParams& P, int n_req, int layers, DType dt, cudaStream_t st);
void launch_commit(const CommitParams& P, int n_req, cudaStream_t st);
void launch_gumbel_debug(const float* logits, int ld, int V, float temperature, uint32_t seed, int req, int step,
                         int n, const int32_t* row, const int32_t* slot, int32_t* out, cudaStream_t st);
