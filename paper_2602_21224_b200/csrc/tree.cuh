// tree.cuh -- parameters of the K-TREE kernel (tree.cu).
#pragma once
#include "common.cuh"

#define HSD_MAX_PLANT_DEPTH_DEV 16
#define HSD_MAX_BR1 64     // B_r + 1 capacity of the pending tree (host-checked)
enum { TREE_MODE_FRESH = 0, TREE_MODE_RESAMPLE = 1 };

struct TreeParams {
  int N, k, B, Br, r, V, Vh, t_max, anc_words;
  int fusion, resample, zero_table;
  const float* L;            // [b, N, V] draft logits, columns in rank order
  const void* table;         // [Vh, Vh] token-info bias, rank-indexed
  DType tdt;
  const float* tscale;       // non-null: table holds e4m3 codes, row r scaled by tscale[r] (R25)
  const int32_t* perm;       // [V] rank -> token (null = identity)
  const int32_t* rank_of;    // [V] token -> rank (null = identity)
  const int32_t* root_tok;   // [b] last committed token
  int32_t *pt_n, *pt_tok, *pt_par, *pt_depth;   // pending re-sampled tree [b, Br+1]
  float* pt_lj;
  int32_t *t_n, *t_tok, *t_par, *t_depth;       // linearised tree [b, t_max]
  float* t_lj;
  uint64_t* t_anc;           // [b, t_max, anc_words]
  const int32_t* acc_n;      // [b] accepted count m (resample mode)
  const int32_t* bonus;      // [b] bonus token (resample mode)
  const int32_t* p;          // [b] root position
  const int32_t* step;       // step counter (device)
  const int32_t* plant;      // [b, plant_stride] or null
  int plant_stride;
  float plant_rates[HSD_MAX_PLANT_DEPTH_DEV];
  uint32_t seed;
  const int32_t* req_id;     // [b] global request id per slot (plant stream)
  int* err;
  L2Pf pf;                   // weights of a later GEMM to prefetch into L2 (common.cuh)
  unsigned long long* trace; // debug phase trace (HSD_TREE_TRACE) or null
};

void launch_tree(const TreeParams& P, int mode, int n_req, cudaStream_t st);
void tree_trace_init();   // debug: HSD_TREE_TRACE phase trace buffer
