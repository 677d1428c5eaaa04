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

/* ------------------------------------------------------------------ kernels */
typedef struct gx_gemm_epilogue {
  int out_kind;               /* GX_OUT_BF16 | GX_OUT_F32 | GX_OUT_F32_ACC */
  void* out;                  /* [M][ldo] */
  int64_t ldo;
  float alpha;                /* acc scale */
  const void* bias;           /* bf16 [N] or NULL */
  int gelu;                   /* out = gelu(acc + bias); aux = acc + bias (bf16) */
  void* aux;
  int64_t ld_aux;
  const void* residual;       /* bf16 [M][ld_res]: out = residual + dropout(acc + bias) */
  int64_t ld_res;
  int64_t row_offset;         /* global row of local row 0 (dropout counter) */
  int64_t col_offset;         /* global column of local column 0 (dropout counter) */
  int64_t drop_ld;            /* global row length used by the dropout counter */
  uint32_t drop_threshold;    /* p * 2^32; 0 disables dropout */
  float drop_scale;           /* 1 / (1 - p) */
  uint64_t seed;
  uint64_t site;
} gx_gemm_epilogue;

/* C[M,N] = A[M,K] * B[N,K]^T with the epilogue above.  a_mn_major: A stored [K][lda]
 * (else [M][lda]); b_mn_major: B stored [K][ldb] (else [N][ldb]).  tile_n: 0 = auto. */
GX_API int gx_k_gemm_bf16(const void* a, int64_t lda, int a_mn_major, const void* b, int64_t ldb,
                   int b_mn_major, int M, int N, int K, const gx_gemm_epilogue* ep,
                   int tile_n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GX_H_ */
