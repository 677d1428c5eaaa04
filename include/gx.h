/* gx.h — C ABI of the B200 Galvatron-plan executor (libgx.so).
 *
 * Everything crossing this boundary is a plain C type: pointers, sizes, flags, JSON text.
 * Device buffers are caller-owned; every compute call is stream-ordered on the caller's
 * cudaStream_t (passed as void*).  No exceptions cross the ABI: every entry point returns
 * an int status mirroring the reference CLI's exit codes (proj/tools/parplan_main.cc:40-42:
 * 0 ok, 1 config/validation error, 2 infeasible) extended with 3 = CUDA error and
 * 4 = NCCL error.  gx_last_error() returns the message of the calling thread's last failure.
 *
 * Three groups of entry points:
 *   gx_plan_*   the plan/search side (reference interface: proj/include/parplan/planner.h,
 *               oracle.h, cost_model.h, strategy.h), JSON in / JSON out;
 *   gx_exec_*   the plan executor: one context per process (one or more local ranks),
 *               runs the Transformer-layer fwd/bwd + optimizer step under a plan;
 *   gx_k_*      individual sm_100a kernels (exposed for parity tests and the profiler).
 */
#ifndef GX_H_
#define GX_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GX_API __attribute__((visibility("default")))
#else
#define GX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GX_OK 0
#define GX_ERR_CONFIG 1
#define GX_ERR_INFEASIBLE 2
#define GX_ERR_CUDA 3
#define GX_ERR_NCCL 4
#define GX_ERR_GUARD 5 /* brute-force oracle guard tripped (parplan::GuardError) */

#define GX_OUT_BF16 0
#define GX_OUT_F32 1
#define GX_OUT_F32_ACC 2
#define GX_OUT_F32_SPLIT 3  /* split-K: out is [splits][M][ldo] fp32, split s stores slice s */

/* ------------------------------------------------------------------ library */
GX_API const char* gx_last_error(void);
GX_API int gx_version(void);

/* ------------------------------------------------------------------ plan / search
 * Reference interface replaced: parplan::Optimize (proj/include/parplan/planner.h:164-167)
 * with PlanToJson (planner.h:169-170).  Inputs are the reference's JSON schemas
 * (model_ir.cc:69-95, cluster.cc:47-61, cost_model.cc:47-66); `batches` is the candidate
 * list (NULL/0 = DefaultBatchCandidates, planner.cc:404-408).  On success writes the plan
 * JSON (PlanToJson schema) into out[0..cap); returns 2 with the diagnostic in
 * gx_last_error() when no plan exists.  *needed receives the full length + 1. */
GX_API int gx_plan_optimize(const char* model_json, const char* cluster_json, const char* profile_json,
                     const int* batches, int num_batches, int prune, const char* guideline,
                     int num_threads, char* out, size_t cap, size_t* needed);

/* parplan::ExhaustivePlan (proj/include/parplan/oracle.h:46-50) — guarded brute force. */
GX_API int gx_plan_exhaustive(const char* model_json, const char* cluster_json,
                       const char* profile_json, const int* batches, int num_batches, int prune,
                       const char* guideline, char* out, size_t cap, size_t* needed);

/* parplan::DpSearch (planner.h:109-112) over layers [begin,end) of the model.  Writes
 * {"feasible", "cost_ms", "assignment": [strategy strings], "peak_memory_bytes"}. */
GX_API int gx_plan_dp_search(const char* model_json, int begin, int end, int64_t budget_bytes,
                      int group_size, int prune, int batch_per_group, double bandwidth_gbps,
                      const char* profile_json, char* out, size_t cap, size_t* needed);

/* parplan::EstimateLayerCost + EstimateMemory (cost_model.h:107-127) for one layer spec
 * and one strategy string.  Writes {"feasible", forward_ms, backward_ms,
 * comm_ms_unoverlapped, total_ms, params_bytes, grads_bytes, optimizer_bytes,
 * activation_bytes}. */
GX_API int gx_plan_estimate(int64_t param_bytes, int64_t act_bytes_per_sample, double fwd_ms,
                     const char* strategy, int batch_per_group, double bandwidth_gbps,
                     const char* profile_json, char* out, size_t cap, size_t* needed);

/* parplan::TransformationCostMs (cost_model.h:139-141). */
GX_API int gx_plan_transformation_ms(int64_t param_bytes, int64_t act_bytes_per_sample,
                              const char* prev_strategy, const char* cur_strategy,
                              int batch_per_group, double bandwidth_gbps, double* out_ms);

/* parplan::EnumerateStrategies (strategy.h:90) -> StrategySetToJson. */
GX_API int gx_plan_enumerate(int group_size, int prune, char* out, size_t cap, size_t* needed);

/* parplan::ExhaustiveDp (oracle.h:39-44) with the gx_plan_dp_search signature/output. */
GX_API int gx_plan_exhaustive_dp(const char* model_json, int begin, int end, int64_t budget_bytes,
                                 int group_size, int prune, int batch_per_group,
                                 double bandwidth_gbps, const char* profile_json, char* out,
                                 size_t cap, size_t* needed);

/* parplan::PartitionPipeline (planner.h:44-48): writes [[begin,end],...] or null. */
GX_API int gx_plan_partition(const char* model_json, int pp_degree, const char* guideline,
                             char* out, size_t cap, size_t* needed);

/* parplan::StagePipelineCostMs (planner.h:50-54). */
GX_API int gx_plan_pipeline_cost(const double* stage_costs_ms, int n, int pp_degree,
                                 int micro_batches, double* out_ms);

/* parplan::CollectiveVolumeBytes (cost_model.h:70-73); kind 0 AR, 1 AG, 2 RS. */
GX_API int gx_plan_collective_bytes(int kind, int degree, double payload_bytes, double* out);

/* ModelFromJson / ClusterFromJson / ProfileFromJson validation; kind = "model" |
 * "cluster" | "profile".  Returns 1 with the field-naming message on failure. */
GX_API int gx_plan_validate(const char* kind, const char* json_text);

/* parplan::GroupBandwidthGbps (cluster.h:51). */
GX_API int gx_plan_bandwidth(const char* cluster_json, int group_size, double* out_gbps);

/* Message of the calling thread's last gx_plan_* failure (also mirrored in gx_last_error). */
GX_API const char* gx_plan_last_error(void);

/* ------------------------------------------------------------------ executor
 * One gx_exec per process.  config_json:
 *   {"plan": <PlanToJson object>, "model": <model json, layers carry "shape">,
 *    "world_size": N, "local_ranks": [...],            (default: all ranks -> sim mode)
 *    "comm": "sim" | "nccl", "nccl_id_hex": "<256 hex chars>" (nccl mode),
 *    "dropout_attn": p, "dropout_hidden": p, "seed": s, "optimizer": true,
 *    "lr", "beta1", "beta2", "eps", "weight_decay", "device": cuda ordinal (optional)}
 * Layer "shape": {"hidden", "heads", "head_dim", "seq", "ffn", "kind"} with kind
 *   "encoder" (pre-LN BERT/ViT layer), "causal" (decoder-only self-attention),
 *   "decoder" (T5: causal self-attention + cross-attention over the first decoder layer's
 *   input + MLP; decoder layers are the model's suffix) or "window" (Swin: "window"
 *   tokens per attention window, window-major; "shift": true = SW-MSA; "rel_pos": true =
 *   learned relative-position bias; "merge": true = patch merging of a [4*seq, hidden/2]
 *   input first).
 * Parameters cross the boundary in the canonical unsharded fp32 order
 * ln1_g ln1_b ln2_g ln2_b b_qkv b_o b_1 b_2 w_qkv w_o w_1 w_2 (row-major, [out][in]), then
 * mln_g mln_b w_m (merging layers) or ln3_g ln3_b b_q2 b_kv2 b_o2 w_q2 w_kv2 w_o2 (decoder
 * layers), then rpb [heads][(2 side - 1)^2] (rel_pos window layers); the executor slices each
 * rank's TP slice and SDP shard.  Batches are global bf16
 * [batch*seq][hidden] arrays; each rank copies only its own rows. */
typedef struct gx_exec gx_exec;
GX_API int gx_exec_create(const char* config_json, gx_exec** out);
GX_API int gx_exec_destroy(gx_exec* ex);
GX_API int gx_exec_set_layer_params(gx_exec* ex, int layer, const float* canonical, int64_t n);
/* what: 0 = fp32 master params, 1 = synchronised fp32 gradients of the last step. */
GX_API int gx_exec_export_layer(gx_exec* ex, int layer, int what, float* canonical, int64_t n);
GX_API int gx_exec_load_batch(gx_exec* ex, const void* x_host, const void* target_host);
/* Device-resident batch: the copies are ordered after the legacy default stream; buffers
 * written on any other stream must be complete (synchronised) before the call. */
GX_API int gx_exec_load_batch_device(gx_exec* ex, const void* x_dev, const void* target_dev);
/* One training step (fwd + loss + bwd + grad sync + AdamW) on the loaded batch.
 * flags bit 0: replay as a CUDA graph (captured on first use); bit 1: instrumented run that
 * brackets every launch with CUDA events (read back with gx_exec_profile_report). */
GX_API int gx_exec_run(gx_exec* ex, int flags);
/* `warmup` untimed runs, then `steps` runs timed with CUDA events on the executor's stream;
 * *ms_per_run = device time / steps (the parplan CLI's `run` and `profile`). */
GX_API int gx_exec_time(gx_exec* ex, int flags, int warmup, int steps, double* ms_per_run);
/* Per-category device time / launches / algorithmic flops+bytes of the last instrumented
 * run, plus per-GEMM-launch (ms, flops) pairs: the per-strategy profiler's raw data. */
GX_API int gx_exec_profile_report(gx_exec* ex, char* out, size_t cap, size_t* needed);
/* Deterministic synthetic parameters on the device (value depends only on seed, layer and
 * canonical index, never on the sharding): LN gains 1, biases 0, weights N(0, std^2). */
GX_API int gx_exec_init_params(gx_exec* ex, uint64_t seed, float std_dev);
GX_API int gx_exec_loss(gx_exec* ex, float* out);
/* Wait for the step(s) in flight, polling the NCCL communicators' asynchronous errors; after
 * timeout_ms (<= 0: none) or on a communicator error the communicators are aborted and
 * GX_ERR_NCCL returned instead of hanging (ncclCommGetAsyncError / ncclCommAbort).
 * gx_exec_loss and gx_exec_step use it with config "sync_timeout_ms" (default 600000). */
GX_API int gx_exec_sync(gx_exec* ex, int64_t timeout_ms);
/* load_batch + run + loss: the end-to-end call (host buffers in, loss out). */
GX_API int gx_exec_step(gx_exec* ex, const void* x_host, const void* target_host, int use_graph,
                        float* loss_out);
/* what: 0 = model output y, 1 = gradient w.r.t. the model input; global bf16 layout. */
GX_API int gx_exec_export_output(gx_exec* ex, int what, void* host_bf16);
GX_API int gx_exec_stream(gx_exec* ex, void** stream_out);
GX_API int gx_exec_info(gx_exec* ex, char* out, size_t cap, size_t* needed);
GX_API int gx_exec_canonical_size(int hidden, int ffn, int64_t* out);
/* Host-only view of the executor for config_json with "comm": "dryrun": communication groups
 * (member lists), per-layer data chunks and pipeline send/recv lists of the local ranks.
 * Touches no device; used to check multi-process rank logic on CPU. */
GX_API int gx_exec_topology(const char* config_json, char* out, size_t cap, size_t* needed);
/* ncclGetUniqueId -> 256 hex chars + NUL (rank 0 creates, torch.distributed broadcasts). */
GX_API int gx_nccl_unique_id(char* out_hex, size_t cap);
GX_API int64_t gx_launch_count(void);

/* ------------------------------------------------------------------ kernels */
typedef struct gx_gemm_epilogue {
  int out_kind;               /* GX_OUT_BF16 | GX_OUT_F32 | GX_OUT_F32_ACC | GX_OUT_F32_SPLIT */
  void* out;                  /* [M][ldo] */
  int64_t ldo;
  float alpha;                /* acc scale */
  const void* bias;           /* bf16 [N] or NULL */
  int gelu;                   /* out = gelu(acc + bias); aux = acc + bias (bf16); 2: aux = gelu'(acc + bias) */
  void* aux;
  int64_t ld_aux;
  const void* residual;       /* bf16 [M][ld_res]: out = residual + dropout(acc + bias) */
  int64_t ld_res;
  int64_t row_offset;         /* global row of local row 0 (dropout counter) */
  int64_t col_offset;         /* global column of local column 0 (dropout counter) */
  int64_t drop_ld;            /* global row length used by the dropout counter */
  uint32_t drop_threshold;    /* thr8 = round(p * 256): byte threshold; 0 disables dropout */
  float drop_scale;           /* 256 / (256 - thr8) */
  uint64_t seed;
  uint64_t site;
  int gelu_bwd;               /* out = acc * gelu'(aux) (aux = bf16 pre-activation, read); 2: out = acc * aux */
  const uint64_t* seed_offset;/* optional device counter added to seed (per-step masks) */
  /* debug: when set, CTA b writes %globaltimer stamps [b][0..7] (entry, after PDL wait,
   * first TMA issued, first stage landed, last MMA issued, first accumulator ready, epilogue
   * done, exit) and SM clock stamps [b][8..15] of epilogue warp 4 (before / after the TMEM
   * loads of its first two chunks; first block: math start / end, staged, store issued) --
   * see scripts/gemm_trace.py */
  unsigned long long* trace;
} gx_gemm_epilogue;

/* C[M,N] = A[M,K] * B[N,K]^T with the epilogue above.  a_mn_major: A stored [K][lda]
 * (else [M][lda]); b_mn_major: B stored [K][ldb] (else [N][ldb]).  tile_n: 0 = auto. */
GX_API int gx_k_gemm_bf16(const void* a, int64_t lda, int a_mn_major, const void* b, int64_t ldb,
                   int b_mn_major, int M, int N, int K, const gx_gemm_epilogue* ep,
                   int tile_n, void* stream);

/* Fused multi-head attention over a token-major qkv buffer ([M=batch*seq][3][heads][d],
 * row stride ld_qkv).  fwd writes ctx ([M][heads*d], ld_ctx) and lse (fp32 [batch*heads][seq],
 * log2 domain); bwd reads qkv, ctx, lse, dctx and writes dqkv (qkv layout) using the fp32
 * workspaces dq_accum ([ceil(seq/128)][batch*heads*round_up(seq,4)*d] fp32: per-key-tile dQ
 * partials) and
 * dsum ([batch*heads*seq], zero-initialised once by the caller; left reset).  head_dim 32-80
 * (multiples of 16) and seq <= 512 run on tcgen05/TMEM (attention_tc.cu: every BASELINE shape,
 * with the masks and biases below); head_dim 128 or longer sequences on mma.sync.  Windowed
 * (Swin) attention is this call with batch = samples * windows and seq = window.  Dropout
 * element (q,k) of global (sample_offset+b, head_offset+h) follows csrc/kernels/attention.cu. */
typedef struct gx_attention_args {
  int batch, seq, heads, head_dim;
  int heads_total, head_offset;
  int64_t sample_offset;
  float scale;
  const void* qkv;
  int64_t ld_qkv;
  void* ctx;
  int64_t ld_ctx;
  void* lse;
  const void* dctx;
  void* dqkv;
  void* dq_accum;
  void* dsum;
  uint32_t drop_threshold;
  float drop_scale;
  uint64_t seed;
  uint64_t site;
  const uint64_t* seed_offset; /* optional device counter added to seed */
  void* mask;                  /* uint16 keep bits [batch*heads][seq][ceil(seq/64)][4]:
                                  written by fwd, read by bwd (when dropout is on) */
  unsigned long long* trace;   /* debug: per-CTA %globaltimer stamps (tcgen05 kernels), or NULL */
  int causal;                  /* 1: query q attends keys k <= q only (decoder self-attention) */
  /* Swin shifted windows (SW-MSA): with win_shift > 0 the batch is samples x (grid/side)^2
   * windows of side win_side over a win_grid-wide grid rolled by win_shift; q and k attend
   * only when they come from the same region of the unrolled grid. */
  int win_grid, win_side, win_shift;
  /* Swin relative-position bias (seq = rpb_side^2 window tokens): scores get
   * rpb[head][(dy + side - 1) * (2 side - 1) + dx + side - 1] (bf16 [heads][(2 side - 1)^2],
   * this call's heads); bwd writes each (window, head)'s table gradient to rpb_dpart (fp32
   * [batch*heads][(2 side - 1)^2], seq <= 64) for gx_k_rpb_grad to sum over the batch in
   * order.  rpb NULL = no bias. */
  const void* rpb;
  void* rpb_dpart;
  int rpb_side;
  /* T5 relative attention bias (tcgen05 path): scores get relb[head][relb_map[k - q + seq - 1]]
   * (bf16 [heads][relb_buckets] learned table, int8 relb_map[2 seq - 1] = the T5 bucket of
   * each relative position, bidirectional or causal); bwd writes per-(sequence x head, key
   * block) fp32 partial sums of dS over each relative position to relb_dpart
   * ([batch*heads][ceil(seq/128)][2 seq - 1]) for gx_k_relb_grad.  relb NULL = no bias. */
  const void* relb;
  const void* relb_map;
  int relb_buckets;
  void* relb_dpart;
} gx_attention_args;

GX_API int gx_k_attention_fwd(const gx_attention_args* args, void* stream);
/* Tests: fill every SM's shared memory with 0xFF (NaN) bytes, so a kernel launched next that
 * reads shared memory it never wrote produces NaN. */
GX_API int gx_k_poison_smem(void* stream);
GX_API int gx_k_attention_bwd(const gx_attention_args* args, void* stream);

/* LayerNorm over rows of h (bf16 in/out, fp32 statistics, eps 1e-5).
 * fwd: y = (x-mean)*rstd*gamma + beta; writes mean/rstd (fp32 [rows]).
 * bwd: dx = LN'(dy) (+ dres if non-NULL); dgamma/dbeta (fp32 [h]) are ACCUMULATED. */
GX_API int gx_k_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y,
                              void* mean, void* rstd, int rows, int h, void* stream);
GX_API int gx_k_layernorm_bwd(const void* dy, const void* x, const void* mean, const void* rstd,
                              const void* gamma, const void* dres, void* dx, void* dgamma,
                              void* dbeta, int rows, int h, void* stream);

/* Dropout sites share one parameter block: element (r, c) of a [rows][cols] local tensor is
 * global element (row_offset + r) * drop_ld + (col_offset + c) of the site's Philox stream. */
typedef struct gx_dropout {
  uint32_t threshold;         /* thr8 = round(p * 256), 0 = off */
  float scale;                /* 256 / (256 - thr8) */
  uint64_t seed, site;
  int64_t row_offset, col_offset, drop_ld;
  const uint64_t* seed_offset; /* optional device counter added to seed */
} gx_dropout;

/* out = residual + dropout(x + bias)      (bf16; bias may be NULL) */
GX_API int gx_k_bias_dropout_add(const void* x, const void* bias, const void* residual, void* out,
                                 int rows, int cols, const gx_dropout* d, void* stream);
/* dz = dropout_mask(dy) (may alias dy when dropout is off); dbias[c] += sum_r dz[r][c] (fp32). */
GX_API int gx_k_dropout_bwd_colsum(const void* dy, void* dz, void* dbias, int rows, int cols,
                                   const gx_dropout* d, void* stream);
/* acc[c] += sum_r x[r][c] (x bf16 [rows][ld], acc fp32) */
GX_API int gx_k_colsum(const void* x, int64_t ld, void* acc, int rows, int cols, void* stream);
/* MSE: loss += sum (y-t)^2 * inv_count (fp32 scalar); dy = 2 (y-t) * inv_count (bf16). */
GX_API int gx_k_mse_loss(const void* y, const void* target, void* dy, void* loss, int64_t n,
                         float inv_count, void* stream);
/* AdamW over n fp32 elements; writes the bf16 compute copy. bias corrections precomputed. */
GX_API int gx_k_adamw(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n,
                      float lr, float beta1, float beta2, float eps, float weight_decay,
                      float bc1, float bc2, void* stream);
/* fp32 -> bf16 */
/* Swin patch merging between window-major token layouts (window side window_side, input
 * grid 2*grid_out, channels c in): backward = 0 gathers [samples*4*grid_out^2][c] into
 * [samples*grid_out^2][4c] (2x2 neighbours in (dy,dx) order (0,0) (1,0) (0,1) (1,1));
 * backward = 1 scatters the merged gradient back.  c % 8 == 0. */
GX_API int gx_k_patch_merge(const void* src, void* dst, int samples, int grid_out,
                            int window_side, int channels, int backward, void* stream);
/* Swin cyclic shift between window-major layouts of a grid x grid token grid: inverse = 0
 * rolls by -shift in both axes (torch.roll(x, (-shift, -shift))), inverse = 1 rolls back. */
/* Swin relative-position-bias gradient: grad[h][e] (+)= sum over b of dpart[b*heads + h][e]
 * (fixed order: deterministic). */
GX_API int gx_k_rpb_grad(const void* dpart, int batch, int heads, int side, void* grad,
                         int accumulate, void* stream);
/* T5 relative attention bias gradient: grad[h][b] (+)= fixed-order sum over the sequence tiles
 * `tiles`, key blocks and relative positions d (map[d] == b) of the backward's relb_dpart. */
GX_API int gx_k_relb_grad(const void* dpart, int tiles, int heads, int seq, const void* map,
                          int buckets, void* grad, int accumulate, void* stream);
GX_API int gx_k_window_roll(const void* src, void* dst, int samples, int grid, int window_side,
                            int shift, int channels, int inverse, void* stream);
GX_API int gx_k_cast_bf16(const void* src, void* dst, int64_t n, void* stream);

/* Split-K GEMM: out_f32[M,N] += A * B^T, each of `splits` K-slices reduce-adding its fp32
 * partial via TMA (caller zeroes out_f32 for a plain product).  splits <= 0 picks the plan
 * the executor uses (CTA-pair 256-wide tiles, one wave).  tile_n as in gx_k_gemm_bf16. */
GX_API int gx_k_gemm_bf16_splitk(const void* a, int64_t lda, int a_mn_major, const void* b,
                                 int64_t ldb, int b_mn_major, int M, int N, int K, void* out_f32,
                                 int64_t ldo, int splits, int tile_n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GX_H_ */
