// plan_capi.cc — extern "C" surface of the plan/search layer (gx_plan_* in include/gx.h).
//
// JSON text in, JSON text out; C++ exceptions are caught here and mapped to the status
// codes of include/gx.h (ValidationError -> 1, infeasible -> 2, GuardError -> 5).
//
// The same translation unit is also compiled by oracle/Makefile against the reference
// planner sources renamed to namespace parplan_ref (-Dparplan=parplan_ref) with
// -DGX_PLAN_PREFIX=ref_plan_, giving the test-only checker an identical C surface.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "parplan/cluster.h"
#include "parplan/cost_model.h"
#include "parplan/model_ir.h"
#include "parplan/oracle.h"
#include "parplan/planner.h"
#include "parplan/strategy.h"

#ifndef GX_PLAN_PREFIX
#define GX_PLAN_PREFIX gx_plan_
#define GX_PLAN_SET_ERROR 1
#include "gx_internal.h"
#endif

#define GX_CAT2(a, b) a##b
#define GX_CAT(a, b) GX_CAT2(a, b)
#define GX_FN(name) GX_CAT(GX_PLAN_PREFIX, name)

#if defined(__GNUC__)
#define GX_EXPORT extern "C" __attribute__((visibility("default")))
#else
#define GX_EXPORT extern "C"
#endif

namespace {

using nlohmann::json;

thread_local std::string g_plan_error;

int Fail(int code, const std::string& msg) {
  g_plan_error = msg;
#ifdef GX_PLAN_SET_ERROR
  gx::set_error(code, msg.c_str());
#endif
  return code;
}

int Emit(const std::string& text, char* out, size_t cap, size_t* needed) {
  if (needed != nullptr) *needed = text.size() + 1;
  if (out == nullptr || cap == 0) return 0;
  if (cap < text.size() + 1) return Fail(1, "output buffer too small");
  std::memcpy(out, text.c_str(), text.size() + 1);
  return 0;
}

parplan::CostProfile ProfileOrDefault(const char* profile_json) {
  if (profile_json == nullptr || profile_json[0] == '\0') return parplan::CostProfile{};
  return parplan::ProfileFromJson(json::parse(profile_json));
}

parplan::PlannerOptions Options(int prune, const char* guideline, int threads) {
  parplan::PlannerOptions o;
  o.prune = prune != 0;
  if (guideline != nullptr && guideline[0] != '\0')
    o.guideline = parplan::PpGuidelineFromName(guideline);
  o.num_threads = threads;
  return o;
}

std::vector<int> Batches(const int* batches, int n) {
  if (batches == nullptr || n <= 0) return parplan::DefaultBatchCandidates();
  return std::vector<int>(batches, batches + n);
}

template <typename F>
int Guarded(F&& body) {
  try {
    return body();
  } catch (const parplan::GuardError& e) {
    return Fail(5, e.what());
  } catch (const parplan::ValidationError& e) {
    return Fail(1, e.what());
  } catch (const json::exception& e) {
    return Fail(1, std::string("json: ") + e.what());
  } catch (const std::exception& e) {
    return Fail(1, e.what());
  }
}

int EmitOutcome(const parplan::PlanOutcome& outcome, const parplan::ModelSpec& model,
                const parplan::CostProfile& profile, char* out, size_t cap, size_t* needed) {
  if (!outcome.plan) {
    Emit(outcome.diagnostic, out, cap, needed);
    return Fail(2, outcome.diagnostic);
  }
  return Emit(parplan::PlanToJson(*outcome.plan, model, profile).dump(), out, cap, needed);
}

}  // namespace

GX_EXPORT const char* GX_FN(last_error)(void) { return g_plan_error.c_str(); }

GX_EXPORT int GX_FN(optimize)(const char* model_json, const char* cluster_json,
                              const char* profile_json, const int* batches, int num_batches,
                              int prune, const char* guideline, int num_threads, char* out,
                              size_t cap, size_t* needed) {
  return Guarded([&] {
    const parplan::ModelSpec model = parplan::ModelFromJson(json::parse(model_json));
    const parplan::ClusterSpec cluster = parplan::ClusterFromJson(json::parse(cluster_json));
    const parplan::CostProfile profile = ProfileOrDefault(profile_json);
    const auto outcome = parplan::Optimize(model, cluster, profile, Batches(batches, num_batches),
                                           Options(prune, guideline, num_threads));
    return EmitOutcome(outcome, model, profile, out, cap, needed);
  });
}

GX_EXPORT int GX_FN(exhaustive)(const char* model_json, const char* cluster_json,
                                const char* profile_json, const int* batches, int num_batches,
                                int prune, const char* guideline, char* out, size_t cap,
                                size_t* needed) {
  return Guarded([&] {
    const parplan::ModelSpec model = parplan::ModelFromJson(json::parse(model_json));
    const parplan::ClusterSpec cluster = parplan::ClusterFromJson(json::parse(cluster_json));
    const parplan::CostProfile profile = ProfileOrDefault(profile_json);
    const auto outcome = parplan::ExhaustivePlan(model, cluster, profile,
                                                 Batches(batches, num_batches),
                                                 Options(prune, guideline, 1));
    return EmitOutcome(outcome, model, profile, out, cap, needed);
  });
}

namespace {
int DpCommon(bool exhaustive, const char* model_json, int begin, int end, int64_t budget,
             int group_size, int prune, int batch, double bw, const char* profile_json,
             char* out, size_t cap, size_t* needed) {
  return Guarded([&] {
    const parplan::ModelSpec model = parplan::ModelFromJson(json::parse(model_json));
    if (begin < 0 || end > model.num_layers() || begin > end)
      return Fail(1, "dp_search: bad layer range");
    const parplan::CostProfile profile = ProfileOrDefault(profile_json);
    const parplan::StrategySet set = parplan::EnumerateStrategies(group_size, prune != 0);
    const auto span = std::span<const parplan::LayerSpec>(model.layers).subspan(begin, end - begin);
    const parplan::DpResult r =
        exhaustive ? parplan::ExhaustiveDp(span, budget, set, batch, bw, profile)
                   : parplan::DpSearch(span, budget, set, batch, bw, profile);
    json j;
    j["feasible"] = r.feasible;
    j["cost_ms"] = r.cost_ms;
    j["peak_memory_bytes"] = r.peak_memory_bytes;
    json a = json::array();
    for (const auto& s : r.assignment) a.push_back(s.ToString());
    j["assignment"] = std::move(a);
    return Emit(j.dump(), out, cap, needed);
  });
}
}  // namespace

GX_EXPORT int GX_FN(dp_search)(const char* model_json, int begin, int end, int64_t budget,
                               int group_size, int prune, int batch, double bw,
                               const char* profile_json, char* out, size_t cap, size_t* needed) {
  return DpCommon(false, model_json, begin, end, budget, group_size, prune, batch, bw,
                  profile_json, out, cap, needed);
}

GX_EXPORT int GX_FN(exhaustive_dp)(const char* model_json, int begin, int end, int64_t budget,
                                   int group_size, int prune, int batch, double bw,
                                   const char* profile_json, char* out, size_t cap,
                                   size_t* needed) {
  return DpCommon(true, model_json, begin, end, budget, group_size, prune, batch, bw,
                  profile_json, out, cap, needed);
}

GX_EXPORT int GX_FN(estimate)(int64_t param_bytes, int64_t act_bytes, double fwd_ms,
                              const char* strategy, int batch, double bw,
                              const char* profile_json, char* out, size_t cap, size_t* needed) {
  return Guarded([&] {
    parplan::LayerSpec layer;
    layer.param_bytes = param_bytes;
    layer.activation_bytes_per_sample = act_bytes;
    layer.fwd_time_per_sample_ms = fwd_ms;
    const parplan::CostProfile profile = ProfileOrDefault(profile_json);
    const parplan::HybridStrategy s = parplan::StrategyFromString(strategy ? strategy : "");
    const auto cost = parplan::EstimateLayerCost(layer, s, batch, bw, profile);
    const auto mem = parplan::EstimateMemory(layer, s, batch, profile);
    json j;
    j["feasible"] = cost.has_value() && mem.has_value();
    if (cost) {
      j["forward_ms"] = cost->forward_ms;
      j["backward_ms"] = cost->backward_ms;
      j["comm_ms_unoverlapped"] = cost->comm_ms_unoverlapped;
      j["total_ms"] = cost->total_ms;
    }
    if (mem) {
      j["params_bytes"] = mem->params_bytes;
      j["grads_bytes"] = mem->grads_bytes;
      j["optimizer_bytes"] = mem->optimizer_bytes;
      j["activation_bytes"] = mem->activation_bytes;
      j["total_bytes"] = mem->total_bytes();
      j["memory_units"] = parplan::MemoryUnits(mem->total_bytes(), profile.memory_granularity_bytes);
    }
    return Emit(j.dump(), out, cap, needed);
  });
}

GX_EXPORT int GX_FN(transformation_ms)(int64_t param_bytes, int64_t act_bytes, const char* prev,
                                       const char* cur, int batch, double bw, double* out_ms) {
  return Guarded([&] {
    parplan::LayerSpec layer;
    layer.param_bytes = param_bytes;
    layer.activation_bytes_per_sample = act_bytes;
    parplan::HybridStrategy a = parplan::StrategyFromString(prev ? prev : "");
    parplan::HybridStrategy b = parplan::StrategyFromString(cur ? cur : "");
    *out_ms = parplan::TransformationCostMs(layer, a, b, batch, bw);
    return 0;
  });
}

GX_EXPORT int GX_FN(enumerate)(int group_size, int prune, char* out, size_t cap,
                               size_t* needed) {
  return Guarded([&] {
    return Emit(parplan::StrategySetToJson(parplan::EnumerateStrategies(group_size, prune != 0)).dump(),
                out, cap, needed);
  });
}

GX_EXPORT int GX_FN(partition)(const char* model_json, int pp_degree, const char* guideline,
                               char* out, size_t cap, size_t* needed) {
  return Guarded([&] {
    const parplan::ModelSpec model = parplan::ModelFromJson(json::parse(model_json));
    const auto ranges = parplan::PartitionPipeline(
        model, pp_degree, parplan::PpGuidelineFromName(guideline ? guideline : "layers"));
    json j = nullptr;
    if (ranges) {
      j = json::array();
      for (const auto& [b, e] : *ranges) j.push_back(json::array({b, e}));
    }
    return Emit(j.dump(), out, cap, needed);
  });
}

GX_EXPORT int GX_FN(pipeline_cost)(const double* stage_costs, int n, int pp_degree,
                                   int micro_batches, double* out_ms) {
  return Guarded([&] {
    *out_ms = parplan::StagePipelineCostMs(std::vector<double>(stage_costs, stage_costs + n),
                                           pp_degree, micro_batches);
    return 0;
  });
}

GX_EXPORT int GX_FN(collective_bytes)(int kind, int degree, double payload, double* out_bytes) {
  return Guarded([&] {
    const parplan::CollectiveKind k = kind == 0   ? parplan::CollectiveKind::kAllReduce
                                      : kind == 1 ? parplan::CollectiveKind::kAllGather
                                                  : parplan::CollectiveKind::kReduceScatter;
    *out_bytes = parplan::CollectiveVolumeBytes(k, degree, payload);
    return 0;
  });
}

GX_EXPORT int GX_FN(validate)(const char* kind, const char* text) {
  return Guarded([&] {
    const std::string k = kind ? kind : "";
    const json j = json::parse(text);
    if (k == "model") {
      parplan::ModelFromJson(j);
    } else if (k == "cluster") {
      parplan::ClusterFromJson(j);
    } else if (k == "profile") {
      parplan::ProfileFromJson(j);
    } else {
      return Fail(1, "validate: unknown kind '" + k + "'");
    }
    return 0;
  });
}

GX_EXPORT int GX_FN(bandwidth)(const char* cluster_json, int group_size, double* out_gbps) {
  return Guarded([&] {
    *out_gbps = parplan::GroupBandwidthGbps(parplan::ClusterFromJson(json::parse(cluster_json)),
                                            group_size);
    return 0;
  });
}
