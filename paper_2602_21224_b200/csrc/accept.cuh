// accept.cuh -- parameters of the S3/S4 kernels (accept.cu).
#pragma once
#include "common.cuh"

struct AcceptParams {
  int mode;                 // 0 greedy, 1 stochastic
  int N, t_max, V;
  float temperature;
  uint32_t seed;
  const int32_t* req_id;    // [b] global request id per slot (random streams)
  const int32_t *t_tok, *t_par, *t_n;
  const int32_t* argmax;    // [b, t_max] (greedy)
  const float* logits;      // [b, t_max, V] (stochastic)
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
  const float* Hverify;     // [b, t_max, n]
  const int32_t *acc_n, *acc_slots, *emitted, *bonus;
  float* pend_H;            // [b, N+1, n]
  int32_t *pend_tok, *n_pend, *root_tok, *p, *step;
};

void launch_walk(const AcceptParams& P, int n_req, cudaStream_t st);
void launch_compact(const CompactParams& P, int n_req, int layers, DType dt, cudaStream_t st);
void launch_commit(const CommitParams& P, int n_req, cudaStream_t st);
void launch_gumbel_debug(const float* logits, int ld, int V, float temperature, uint32_t seed, int req, int step,
                         int n, const int32_t* row, const int32_t* slot, int32_t* out, cudaStream_t st);
