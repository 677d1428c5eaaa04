// executor.h — runs Transformer-layer forward/backward + AdamW under a Galvatron plan.
//
// Input: a plan in the reference's PlanToJson schema (proj/src/planner.cc:483-521) and a
// model in the reference's model schema with per-layer "shape" objects.  Semantics of each
// strategy follow the reference cost model, which is the executor's contract:
//   * memory / shard sizes      EstimateMemory      (proj/src/cost_model.cc:119-143)
//   * communication schedule    EstimateLayerCost   (proj/src/cost_model.cc:145-213)
//       TP: activation all-reduce in forward and backward (serial);
//       SDP: parameter all-gather before forward and again before backward,
//            gradient reduce-scatter; DP: gradient all-reduce of the owned shard
//   * inter-layer relayout      TransformationCostMs (proj/src/cost_model.cc:215-241):
//       equal degrees -> no-op; D grows -> local slice (bwd: all-gather);
//       D shrinks -> all-gather of D_prev/D_cur shards (bwd: local slice)
//   * pipeline                  GPipe with the plan's micro-batch count
//                               (StagePipelineCostMs, planner.cc:138-159)
// Rank mapping: stage p owns ranks [p*g, (p+1)*g); inside a stage TP
// groups are contiguous runs of t ranks, data (DP/SDP) groups are stride-t.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "comm.h"

namespace gx {

struct Deg {
  int dp = 1, sdp = 1, tp = 1;
  int data() const { return dp * sdp; }
};

struct Shape {
  int h = 0, heads = 0, hd = 0, seq = 0, ffn = 0;
  int win = 0;  // tokens per attention window (kind "window"); == seq for full attention
  int windows() const { return seq / win; }
  // Swin patch merging at the layer input: the input is [4*seq, h/2] per sample (a grid of
  // side 2G, window-major), 2x2 neighbours are concatenated, LayerNorm'd and projected to h.
  bool merge = false;
  // decoder layers: causal self-attention (kind "causal", "decoder"); "decoder" adds a
  // cross-attention sublayer over the memory (the input of the model's first decoder layer)
  bool causal = false, cross = false;
  int shift = 0;  // Swin SW-MSA: tokens rolled by -shift in both grid axes around attention
  bool rpb = false;  // Swin relative-position bias table [heads][(2 side - 1)^2]
  // T5: RMSNorm for every LayerNorm of the layer (gain only, eps 1e-6), and the bucketed
  // relative attention bias of the self-attention (relb buckets, 0 = none; max distance 128)
  bool rms = false;
  int relb = 0;
  int rpb_n() const {  // table entries per head
    int w = 1;
    while (w * w < win) ++w;
    return (2 * w - 1) * (2 * w - 1);
  }
  int in_h() const { return merge ? h / 2 : h; }
  int in_seq() const { return merge ? 4 * seq : seq; }
};

// Offsets (elements) of one layer's tensors inside its flat per-rank parameter buffer.
struct Slot {
  int64_t off = 0, n = 0;
};
struct Layout {
  Slot ln1g, ln1b, ln2g, ln2b, bqkv, bo, b1, b2, wqkv, wo, w1, w2;
  Slot mlng, mlnb, wm;  // patch merging (empty unless Shape::merge): LN(2h) and [h][2h]
  // cross-attention (empty unless Shape::cross): LN3, q / kv / out projections
  Slot ln3g, ln3b, bq2, bkv2, bo2, wq2, wkv2, wo2;
  Slot rpb;  // Swin relative-position bias, this rank's heads (gradient accumulated)
  Slot relb;  // T5 relative attention bias [heads / tp][buckets] (gradient accumulated)
  int64_t acc_end = 0;  // [0, acc_end): params whose grads accumulate with atomics
  int64_t total = 0;    // padded to a multiple of 64 * sdp
  int64_t shard() const { return total; }
};
Layout make_layout(const Shape& s, int tp, int sdp);
// Canonical (unsharded, unpadded) flat order used at the host boundary:
// ln1_g ln1_b ln2_g ln2_b b_qkv b_o b_1 b_2 w_qkv w_o w_1 w_2
int64_t canonical_size(const Shape& s);

class Executor;
// On failure *err holds the message and *code (when non-null) the gx error code.
std::unique_ptr<Executor> create_executor(const std::string& config_json, std::string* err,
                                          int* code = nullptr);

class Executor {
 public:
  virtual ~Executor() = default;
  virtual int set_layer_params(int layer, const float* canonical, int64_t n) = 0;
  virtual int export_layer(int layer, int what, float* canonical, int64_t n) = 0;  // 0 params 1 grads
  virtual int load_batch(const void* x_host, const void* target_host) = 0;
  virtual int load_batch_device(const void* x_dev, const void* target_dev) = 0;
  virtual int run(bool use_graph) = 0;
  virtual int loss(float* out) = 0;
  // stream synchronisation with communicator failure detection (timeout_ms <= 0: no limit)
  virtual int sync(int64_t timeout_ms) = 0;
  virtual int export_output(void* host_bf16, int what) = 0;  // 0 final y, 1 input grad dx
  virtual cudaStream_t stream() const = 0;
  virtual std::string info() const = 0;
  // bit 0: CUDA graph, bit 1: instrumented (per-launch events) variant
  virtual int run2(bool use_graph, bool profile) = 0;
  virtual std::string profile_report() const = 0;
  virtual int init_params(uint64_t seed, float std_dev) = 0;
  // Groups, data chunks and pipeline transfers of the local ranks (no device state needed).
  virtual std::string topology() const = 0;
};

}  // namespace gx
