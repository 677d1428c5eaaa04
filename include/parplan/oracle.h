// parplan/oracle.h — guarded brute-force counterparts of DpSearch / Optimize.
// Interface: reference proj/include/parplan/oracle.h:28-52.
#ifndef GX_PARPLAN_ORACLE_H_
#define GX_PARPLAN_ORACLE_H_

#include <cstdint>
#include <span>
#include <vector>

#include "parplan/cluster.h"
#include "parplan/cost_model.h"
#include "parplan/model_ir.h"
#include "parplan/planner.h"
#include "parplan/strategy.h"

namespace parplan {

inline constexpr int64_t kOracleEnumerationLimit = 1'000'000;

DpResult ExhaustiveDp(std::span<const LayerSpec> layers, int64_t memory_budget_bytes,
                      const StrategySet& strategies, int batch_per_group, double bandwidth_gbps,
                      const CostProfile& profile);

PlanOutcome ExhaustivePlan(const ModelSpec& model, const ClusterSpec& cluster,
                           const CostProfile& profile, const std::vector<int>& batch_candidates,
                           const PlannerOptions& options = {});

}  // namespace parplan

#endif  // GX_PARPLAN_ORACLE_H_
