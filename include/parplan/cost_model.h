// parplan/cost_model.h — memory O(l,s), time c(l,s) and relayout R(l,s',s) of Eq. 1.
// Interface: reference proj/include/parplan/cost_model.h:28-143.  These formulas are also
// the executor's contract: EstimateMemory fixes each device's shard sizes, EstimateLayerCost
// the communication schedule (serial SDP gather + TP syncs, gradient sync overlapped with
// backward), TransformationCostMs the Slice-Gather between layers.
#ifndef GX_PARPLAN_COST_MODEL_H_
#define GX_PARPLAN_COST_MODEL_H_

#include <cstdint>
#include <optional>
#include <string>

#include <nlohmann/json_fwd.hpp>

#include "parplan/common.h"
#include "parplan/model_ir.h"
#include "parplan/strategy.h"

namespace parplan {

struct CostProfile {
  double backward_multiplier = 2.0;         // backward compute / forward compute
  double overlap_slowdown = 1.3;            // contention factor on overlapped bwd + grad sync
  double optimizer_state_multiplier = 2.0;  // optimizer bytes per parameter byte
  double tp_activation_replication = 0.25;  // rho: replicated activation fraction under TP
  int64_t memory_granularity_bytes = 64 * kMiB;

  friend bool operator==(const CostProfile&, const CostProfile&) = default;
};

void ValidateProfile(const CostProfile& profile);
CostProfile ProfileFromJson(const nlohmann::json& j);
nlohmann::json ProfileToJson(const CostProfile& profile);
CostProfile LoadProfile(const std::string& path);

// ceil(bytes / granularity).
int MemoryUnits(double bytes, int64_t granularity_bytes);

enum class CollectiveKind { kAllReduce, kAllGather, kReduceScatter };

// Ring bytes per device: all-reduce 2(d-1)/d, all-gather / reduce-scatter (d-1)/d.
double CollectiveVolumeBytes(CollectiveKind kind, int degree, double payload_bytes);

struct MemoryBreakdown {
  double params_bytes = 0.0;
  double grads_bytes = 0.0;
  double optimizer_bytes = 0.0;
  double activation_bytes = 0.0;

  double total_bytes() const {
    return params_bytes + grads_bytes + optimizer_bytes + activation_bytes;
  }
};

struct LayerCost {
  double forward_ms = 0.0;
  double backward_ms = 0.0;
  double comm_ms_unoverlapped = 0.0;
  double total_ms = 0.0;
};

std::optional<MemoryBreakdown> EstimateMemory(const LayerSpec& layer,
                                              const HybridStrategy& strategy,
                                              int batch_per_group,
                                              const CostProfile& profile);

std::optional<LayerCost> EstimateLayerCost(const LayerSpec& layer,
                                           const HybridStrategy& strategy,
                                           int batch_per_group, double bandwidth_gbps,
                                           const CostProfile& profile);

double TransformationCostMs(const LayerSpec& layer, const HybridStrategy& prev,
                            const HybridStrategy& cur, int batch_per_group,
                            double bandwidth_gbps);

}  // namespace parplan

#endif  // GX_PARPLAN_COST_MODEL_H_
