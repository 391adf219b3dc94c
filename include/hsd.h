/*
 * hsd.h -- C ABI of the B200-native hidden-state tree speculative decoder
 * (arXiv 2602.21224, "Make Every Draft Count", system name Lyanna).
 *
 * One library call = one stage of the per-step draft-tree verify-and-reuse loop
 * (section 3 Overview). Citations: P:<line> = PAPER.md line.
 *
 * Conventions (all entry points):
 *  - Every call is asynchronous on the stream given to hsd_init_model, except
 *    where stated ("synchronous"). Outputs go into CALLER-OWNED buffers whose
 *    location (host or device) is stated per argument.
 *  - Host-checkable preconditions (contract violations: bad sizes, k > V,
 *    B < 1, N < 1, token outside [0, V), more requests than max_batch, wrong call
 *    order) return HSD_EINVAL / HSD_ESTATE BEFORE any launch, with text in
 *    hsd_last_error(). Device-side violations set a device error word that is
 *    surfaced as HSD_EDEVICE by hsd_sync().
 *  - A context owns all its device memory (weights, paged KV pools, the
 *    token-info table, workspace); it is used by one host thread at a time.
 *  - Layout words: "row-major [a, b]" means element (i, j) at i*b + j.
 *  - Requests are independent. Random streams use the GLOBAL request id
 *    (req_offset + local index) so batch sharding across GPUs never changes a
 *    result.
 */
#ifndef HSD_H
#define HSD_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hsd_ctx hsd_ctx;

typedef enum {
  HSD_OK = 0,
  HSD_EINVAL = -1,   /* contract violation (host-checked, nothing launched)   */
  HSD_ENOMEM = -2,   /* device allocation failed                               */
  HSD_ECUDA = -3,    /* CUDA runtime / launch error                            */
  HSD_ENCCL = -4,    /* reserved: collective error                             */
  HSD_ESTATE = -5,   /* call order violated (e.g. verify before build)         */
  HSD_EUNSUP = -6,   /* configuration not supported by this build              */
  HSD_EDEVICE = -7   /* a kernel detected a violation on the device            */
} hsd_status;

enum { HSD_FP32_VERIFY = 0, HSD_BF16 = 1 };          /* hsd_config.precision   */
enum { HSD_GREEDY = 0, HSD_STOCHASTIC = 1 };         /* hsd_config.accept_mode */
enum {                                               /* hsd_config.flags       */
  HSD_FLAG_RESAMPLE = 1u << 0,  /* Alg. 2 re-sampling              */
  HSD_FLAG_FUSION = 1u << 1,    /* verification fusion. RESAMPLE
                                   without FUSION = the paper's ablation:
                                   the re-sampled tree is verified by a dedicated
                                   extra target pass inside the same step        */
  HSD_FLAG_PLANTED = 1u << 2,   /* planted-continuation perf mode (DESIGN R24) */
  HSD_FLAG_ZERO_TABLE = 1u << 3,/* token info off: Alg. 1 == beam tree */
  HSD_FLAG_TCGEN05 = 1u << 4,   /* bf16 GEMMs on tcgen05 (else SIMT FFMA)       */
  HSD_FLAG_TABLE_FP8 = 1u << 5, /* token-info table as e4m3 codes + a per-row
                                   fp32 scale (DESIGN R25)        */
  HSD_FLAG_NO_FIRST_TOKEN = 1u << 6, /* "w/o first token" (Table 4, P:511-533;
                                   R26): the root pair -- the ground-truth token
                                   just committed -- enters the draft as
                                   W_fc [H; 0], without its embedding            */
  HSD_FLAG_TOKEN_AR = 1u << 7   /* token-level AR draft (EAGLE-style, NEXT-2;
                                   R27): each chain step feeds back
                                   its own top-1 token, x = W_fc [h_i; E(t_i)],
                                   with one lm_head GEMV per step instead of the
                                   one-pass head (not with the sharded head)     */
};

#define HSD_MAX_PLANT_DEPTH 16

typedef struct {
  /* target model shape (Llama decoder)                   */
  int32_t vocab, hidden, layers, q_heads, kv_heads, head_dim, ffn;
  float rope_theta, rms_eps;
  /* tree / method parameters: N steps (tree depth), branch k, budget B
     (non-root nodes), re-sample budget B_r and threshold r,
     hot tokens V_h (0 = dense table), low-rank d (R7; 0 -> hidden/16)  */
  int32_t steps_N, branch_k, budget_B, resample_budget_Br, resample_threshold_r;
  int32_t hot_tokens, table_rank;
  /* capacity                                                                 */
  int32_t max_batch, max_ctx, page_size;
  int32_t precision;    /* HSD_FP32_VERIFY | HSD_BF16                          */
  int32_t accept_mode;  /* HSD_GREEDY | HSD_STOCHASTIC                         */
  float temperature;    /* stochastic mode only                                */
  uint64_t seed;        /* Philox seed for weights and sampling (R23)           */
  uint32_t flags;       /* HSD_FLAG_*                                          */
  int32_t req_offset;   /* global id of local request 0 (batch sharding)       */
  /* HOST pointer, vocab entries, rank -> token id (rank 0 = most frequent);
     required when hot_tokens > 0 (defines the hot set, R5), else may be NULL.
     Copied during hsd_init_model.                                            */
  const int32_t* vocab_perm;
  /* planted mode: acceptance rates a_1..a_N (R24)                            */
  float plant_rates[HSD_MAX_PLANT_DEPTH];
  /* Vocab-sharded lm_head (BASELINE configs[4]). Greedy, and
   * stochastic through per-row (max, sum exp, Gumbel top-16, tree-token logit)
   * records merged across shards (R29; needs branch_k + B_r < 16,
   * else HSD_EUNSUP; the token-AR draft is not combined with sharding ->
   * HSD_EUNSUP). shard_mode != HSD_SHARD_NONE splits
   * the two per-step heads -- the draft one-pass logits (S1a) and the
   * verify head (S2) -- by vocabulary column: shard s owns columns
   * [lo_s, lo_{s+1}), lo_s = floor(s*V/G / 128) * 128, lo_G = V, G =
   * vocab_shards. Verify: every shard computes its columns for ALL rows, a
   * per-row partial argmax (max value, lowest token id) over its columns, and
   * the partials are merged exactly (the global argmax is the best partial).
   * Draft: every shard computes its columns for all rows and an all-to-all
   * returns each row owner its full fp32 logits rows (bit-identical columns).
   *  HSD_SHARD_NCCL: G = number of processes (one per GPU), shard_rank = this
   *    process; normalised rows are all-gathered and partials / logits slices
   *    exchanged with NCCL (nccl_id = hsd_nccl_unique_id() bytes of shard 0,
   *    broadcast by the caller). Every shard must prefill the same number of
   *    requests. Each process keeps the full W_head (prefill's first-token
   *    head stays local).
   *  HSD_SHARD_SIM: one process computes all G column slices itself and runs
   *    the same partial / merge / scatter kernels, the collectives replaced by
   *    the buffers they would fill -- the single-GPU test of the sharded
   *    arithmetic. shard_rank must be 0.
   * In sharded mode hsd_verify_view.logits is NULL (no full logits rows).     */
  int32_t vocab_shards, shard_rank, shard_mode;
  uint8_t nccl_id[128];
} hsd_config;

enum { HSD_SHARD_NONE = 0, HSD_SHARD_NCCL = 1, HSD_SHARD_SIM = 2 };   /* hsd_config.shard_mode */

/* Write a fresh NCCL unique id (128 bytes, HOST buffer `out`) for the shard
 * group; call on shard 0 only and broadcast the bytes to the other shards.
 * NCCL is loaded at run time (dlopen "libnccl.so.2"): HSD_ENCCL if it cannot
 * be loaded or the call fails. Synchronous, no device work.                 */
hsd_status hsd_nccl_unique_id(uint8_t* out);

/* Fill *cfg with neutral defaults (flags RESAMPLE|FUSION, B_r 4, r 1, page 64). */
void hsd_config_defaults(hsd_config* cfg);

/* Create a context on `device`, allocate every pool and generate the weights on
 * the device from Philox (R23), precompute RoPE tables, and build the
 * token-info table W_collapsed = W_E W1 W2 with row RMSNorm and 2-D hot pruning
 * (P:290-296). `cuda_stream` is a cudaStream_t (NULL = legacy
 * default stream). Synchronous. On failure *out is NULL.                      */
hsd_status hsd_init_model(const hsd_config* cfg, int device, void* cuda_stream, hsd_ctx** out);

/* Prefill `n_req` (<= max_batch) requests. h_tokens: HOST row-major
 * [n_req, stride] int32 prompt tokens, request r uses h_tokens[r*stride ...
 * + h_lens[r]). h_lens: HOST [n_req], 2 <= len <= max_ctx. Capacity: the KV
 * pool holds max_pos >= max_ctx + T + N positions per slot; a step writes KV up
 * to p + T - 1 and commits at most N + 1 tokens, so hsd_step / hsd_build_tree
 * return HSD_ESTATE (nothing launched) once a slot's committed length p could
 * reach max_pos - T (the host tracks p + (N + 1) per step and re-reads the
 * device's p when that bound gets tight). Slot r's global request id (random
 * streams, R13 / R22 / R24) is req_offset + r. Runs the target causally over each prompt (writes KV), picks the
 * first token (argmax, or Gumbel sample in stochastic mode, R22), and runs the
 * draft layer over pairs (H_{j-1}, t_j), j = 1..len-1 (R1). d_first: DEVICE
 * [n_req] int32 output (may be NULL). Resets the step counter.              */
hsd_status hsd_prefill(hsd_ctx* ctx, int32_t n_req, const int32_t* h_tokens, int32_t stride,
                       const int32_t* h_lens, int32_t* d_first);

/* Continuous batching (the serving layer around the path,
 * P:428): replace the request in batch slot `slot` (0 <= slot < the prefilled
 * n_req) by a new prompt h_tokens (HOST [len] int32, 2 <= len <= max_ctx,
 * ragged: any length per slot) while the other slots keep their state. Runs the
 * same per-request prefill as hsd_prefill (target KV + H, first token, draft
 * prefill) for that slot only and clears its pending re-sampled tree; the step
 * graph stays valid (no shape change). d_first: DEVICE [n_req] int32 or NULL
 * (entry `slot` written). Synchronous. HSD_ESTATE before hsd_prefill or inside a
 * staged step; HSD_EUNSUP with the NCCL vocab-sharded head (every shard would have
 * to admit in lockstep). req_id (>= 0, else HSD_EINVAL): the admitted request's
 * GLOBAL id for every random stream (first-token Gumbel, acceptance uniforms,
 * planting) -- the caller gives each admitted request a fresh id, so it never
 * reuses the noise of the slot's earlier requests.                             */
hsd_status hsd_admit(hsd_ctx* ctx, int32_t slot, const int32_t* h_tokens, int32_t len, int32_t req_id,
                     int32_t* d_first);

/* Paged KV (P:95's cache): the block table maps (slot r, logical
 * page i) to a physical page of the KV pools -- every kernel that reads or writes
 * K / V (prefill, qkv_rope_kv, tree attention, compaction, the draft layer) goes
 * through it. h_table: HOST [max_batch, pages_per_req] int32, a permutation of
 * [0, max_batch * pages_per_req) (pages_per_req = hsd_get_tensor("block_table")
 * dims[1]); copied. The KV contents are not moved, so set it before hsd_prefill
 * (the default is the identity). HSD_EINVAL if not a permutation; HSD_ESTATE
 * inside a staged step. Drops the captured step graphs.                       */
hsd_status hsd_set_block_table(hsd_ctx* ctx, const int32_t* h_table);

/* Planted mode only: HOST row-major [n_req, stride] greedy continuation tokens
 * indexed by absolute position (R24). Copied. */
hsd_status hsd_set_plant(hsd_ctx* ctx, const int32_t* h_plant, int32_t stride);

/* Read-only device view of the current draft tree (valid until the next
 * mutating call). Arrays are row-major per request, T_max = B + B_r + 1 slots:
 * tok [b, T_max] int32, par [b, T_max] int32 (-1 root), depth [b, T_max] int32,
 * logjoint [b, T_max] float, n [b] int32 node count, anc [b, T_max, anc_words]
 * uint64 ancestor bitmask (bit s of row u set iff slot s is u or an ancestor
 * of u; P:95 tree attention).                                                 */
typedef struct {
  const int32_t* tok; const int32_t* par; const int32_t* depth; const float* logjoint;
  const int32_t* n; const uint64_t* anc;
  int32_t batch, t_max, anc_words;
} hsd_tree_view;

/* Read-only device view of the last verification: logits [b, T_max, vocab]
 * float32 (target logits per slot), argmax [b, T_max] int32, hidden
 * [b, T_max, hidden] float32 (pre-final-norm H).                             */
typedef struct {
  const float* logits; const int32_t* argmax; const float* hidden;
  int32_t batch, t_max, vocab, hidden_dim;
} hsd_verify_view;

/* S0 + S1: draft chain, one-pass logits, Alg. 1 tree
 * (P:310-353), prune to B, fuse the pending re-sampled tree and prune
 * to B + B_r, linearise + ancestor masks. `out` may be NULL. */
hsd_status hsd_build_tree(hsd_ctx* ctx, hsd_tree_view* out);

/* Replace the tree built by hsd_build_tree with a caller tree (teacher
 * forcing in parity tests). HOST arrays [n_req, t_max] tok/par/depth and
 * [n_req] n; slots depth-major, parents before children. */
hsd_status hsd_force_tree(hsd_ctx* ctx, const int32_t* h_tok, const int32_t* h_par,
                          const int32_t* h_depth, const int32_t* h_n);

/* S2: target forward over the tree slots with tree-masked attention over the
 * paged KV cache + the tree; writes the slots' K/V at cache
 * positions p..p+T-1. `out` may be NULL. Requires hsd_build_tree. */
hsd_status hsd_verify_tree(hsd_ctx* ctx, hsd_verify_view* out);

/* S3 + S4: acceptance walk (greedy P:378 / stochastic R13), KV compaction of
 * the accepted path, hidden-state gather for the next draft prefill, and Alg. 2
 * re-sampling into the pending tree. d_emitted: DEVICE [b, N+1]
 * int32 (accepted draft tokens then the bonus token; unused entries -1);
 * d_n_emitted: DEVICE [b] int32 (m+1). Either may be NULL. Requires
 * hsd_verify_tree. */
hsd_status hsd_accept_and_compact(hsd_ctx* ctx, int32_t* d_emitted, int32_t* d_n_emitted);

/* One whole step = build_tree + verify_tree + accept_and_compact, captured in
 * a CUDA graph on first use and replayed afterwards (no host sync inside). */
hsd_status hsd_step(hsd_ctx* ctx, int32_t* d_emitted, int32_t* d_n_emitted);

/* hsd_step with HOST outputs: emitted [b, N+1] and n [b] are copied
 * device->host inside the call (synchronous). The end-to-end API. */
hsd_status hsd_step_host(hsd_ctx* ctx, int32_t* h_emitted, int32_t* h_n_emitted);

/* Wait for the context stream; returns HSD_EDEVICE if a kernel flagged a
 * violation (and resets the flag), HSD_ECUDA on a CUDA error. Synchronous. */
hsd_status hsd_sync(hsd_ctx* ctx);

/* Debug/test access to named device tensors (e.g. "kv", "draft_logits",
 * "table", "pos", "pend_tok", "acc_slots", "bonus"). Fills a device pointer,
 * dtype code (0 f32, 1 bf16, 2 i32, 3 u64, 4 u8) and up to 4 dims. With
 * HSD_FLAG_TABLE_FP8, "table" is u8 e4m3 codes [Vh, Vh] and "table_scale" f32 [Vh]. */
typedef struct { void* ptr; int32_t dtype; int32_t ndim; int64_t dims[4]; } hsd_tensor;
hsd_status hsd_get_tensor(hsd_ctx* ctx, const char* name, hsd_tensor* out);

/* Kernel-category profiling (measurement support, not part of the method).
 * enable != 0: subsequent hsd_step / staged calls run EAGERLY and every launch
 * is bracketed by CUDA events on the ctx stream; counters reset. Categories:
 * "gemm_verify", "gemm_draft", "head_verify", "head_draft", "attn_verify",
 * "attn_draft", "tree", "resample", "walk", "compact", "rowwise".
 * hsd_profile_read returns the summed event time (ms), the launch count and
 * the ALGORITHMIC bytes / flops of those launches (GEMM: weights + activations
 * + outputs once; compaction: rows moved). Any out-pointer may be NULL.
 * Synchronous.                                                               */
hsd_status hsd_profile(hsd_ctx* ctx, int enable);
hsd_status hsd_profile_read(hsd_ctx* ctx, const char* category, double* total_ms, int64_t* launches,
                            double* bytes, double* flops);

/* Test hook: one GEMM of the library, C[M,N] (+)= A[M,K] W[N,K]^T, DEVICE
 * pointers, row-major with leading dimensions lda/ldw/ldc (elements).
 * dtype 0 = fp32 operands (SIMT FFMA kernel), 1 = bf16 operands; use_tc = 1
 * selects the tcgen05 kernel (bf16 only); use_tc = 2 the data-parallel tcgen05
 * kernel with SwiGLU fused in the epilogue (W rows gate/up interleaved in 16-row
 * groups; C is then a bf16 [M, N/2] output with leading dimension ldc; only for
 * shapes with >= 4 output tiles per SM, else HSD_EUNSUP). Otherwise C is fp32.
 * Asynchronous on `stream`.
 * Returns HSD_EUNSUP if use_tc is requested for an unsupported shape.        */
hsd_status hsd_debug_gemm(const void* A, int32_t lda, const void* W, int32_t ldw, float* C, int32_t ldc,
                          int32_t M, int32_t N, int32_t K, int32_t accumulate, int32_t dtype, int32_t use_tc,
                          void* stream);

/* Test hook: n independent Gumbel-max draws with the stochastic walk's own device
 * code (reading R13; PAPER.md:449 leaves T > 0 unspecified): draw i returns
 * argmax_v (l_v / T - log(-log U_v)) over row d_row[i] of the DEVICE fp32 logits
 * [*, ld] (v < V), with U_v the sampling uniform of the Gumbel Philox stream
 * (seed, 0x5EED0002), counter (v/4, d_slot[i], step, req), word v%4 (DESIGN.md
 * section 4). d_row, d_slot, d_out: DEVICE int32 [n]. Asynchronous on `stream`.
 * HSD_EINVAL on null pointers, ld < V or temperature <= 0.                   */
hsd_status hsd_debug_gumbel(const float* d_logits, int32_t ld, int32_t V, float temperature, uint64_t seed,
                            int32_t req, int32_t step, int32_t n, const int32_t* d_row, const int32_t* d_slot,
                            int32_t* d_out, void* stream);

/* Number of this library's kernels launched on the ctx since creation. */
int64_t hsd_kernel_launches(const hsd_ctx* ctx);

/* Measurement: per-launch device time of the verify GEMMs INSIDE graph-replayed
 * steps (no events between launches). enable != 0: the next hsd_step recaptures
 * its graph with every verify GEMM launch stamping %globaltimer at CTA entry
 * (minimum over CTAs) and exit (maximum) into a device buffer indexed by (step
 * counter mod 64, launch); enable == 0 drops the stamped graph. Synchronous.
 * HSD_ESTATE inside a staged step.                                           */
hsd_status hsd_kstamp(hsd_ctx* ctx, int enable);
/* Read the stamps (synchronous): *avg_us = mean (exit - entry) over every stamped
 * launch of every stamped replay still in the buffer, *samples their count,
 * *bytes_per_launch / *flops_per_launch the mean algorithmic bytes / flops of one
 * stamped launch (the same accounting as hsd_profile). HOST outputs, may be NULL.
 * HSD_ESTATE if no stamped graph ran.                                         */
hsd_status hsd_kstamp_read(hsd_ctx* ctx, double* avg_us, int64_t* samples, double* bytes_per_launch,
                           double* flops_per_launch);
/* The same for the verify tree-attention launches (the tcgen05 kernel plus its
 * split merge when there is one): *avg_us from the first return from
 * griddepcontrol.wait to the last CTA exit of the merge, *samples as above.   */
hsd_status hsd_kstamp_read_attention(hsd_ctx* ctx, double* avg_us, int64_t* samples);

hsd_status hsd_destroy(hsd_ctx* ctx);
const char* hsd_last_error(const hsd_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HSD_H */
