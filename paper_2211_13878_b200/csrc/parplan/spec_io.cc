// spec_io.cc — model / cluster / cost-profile value types: validation and JSON I/O.
//
// Semantics follow the reference planner's L0 inputs:
//   model   : reference proj/src/model_ir.cc:41-142 (ids by position, unknown keys ignored)
//   cluster : reference proj/src/cluster.cc:25-97
//   profile : reference proj/src/cost_model.cc:27-90 (every key optional)
#include <fstream>
#include <sstream>

#include <nlohmann/json.hpp>

#include "parplan/cluster.h"
#include "parplan/cost_model.h"
#include "parplan/model_ir.h"

namespace parplan {

using nlohmann::json;

namespace {

json ReadJsonFile(const std::string& path, const char* what) {
  std::ifstream file(path);
  if (!file.good()) throw ValidationError(std::string(what) + ": cannot open " + path);
  json j;
  try {
    file >> j;  // non-strict: trailing content after the first value is ignored
    return j;
  } catch (const json::exception& e) {
    throw ValidationError(std::string(what) + ": parse error in " + path + ": " + e.what());
  }
}

}  // namespace

// ------------------------------------------------------------------------------ model

int64_t ModelSpec::TotalParamBytes() const {
  int64_t sum = 0;
  for (const LayerSpec& l : layers) sum += l.param_bytes;
  return sum;
}

int64_t ModelSpec::TotalActivationBytesPerSample() const {
  int64_t sum = 0;
  for (const LayerSpec& l : layers) sum += l.activation_bytes_per_sample;
  return sum;
}

void ValidateModel(const ModelSpec& model) {
  if (model.layers.empty()) throw ValidationError("model: layers must contain at least one layer");
  if (model.dtype_bytes <= 0) throw ValidationError("model: dtype_bytes must be positive");
  for (std::size_t i = 0; i < model.layers.size(); ++i) {
    const LayerSpec& l = model.layers[i];
    const std::string field = "model: layers[" + std::to_string(i) + "].";
    if (l.id != static_cast<int>(i))
      throw ValidationError(field + "id must equal its position " + std::to_string(i));
    if (l.param_bytes < 0) throw ValidationError(field + "param_bytes must be >= 0");
    if (l.activation_bytes_per_sample < 0)
      throw ValidationError(field + "activation_bytes_per_sample must be >= 0");
    // written as !(x >= 0) so NaN is rejected too
    if (!(l.fwd_time_per_sample_ms >= 0.0))
      throw ValidationError(field + "fwd_time_per_sample_ms must be >= 0");
  }
}

ModelSpec ModelFromJson(const json& j) {
  ModelSpec model;
  try {
    model.dtype_bytes = j.value("dtype_bytes", 4);
    const json& arr = j.at("layers");
    if (!arr.is_array()) throw ValidationError("model: layers must be an array");
    model.layers.reserve(arr.size());
    for (const json& item : arr) {
      LayerSpec l;
      l.id = static_cast<int>(model.layers.size());
      l.param_bytes = item.at("param_bytes").get<int64_t>();
      l.activation_bytes_per_sample = item.at("activation_bytes_per_sample").get<int64_t>();
      l.fwd_time_per_sample_ms = item.at("fwd_time_per_sample_ms").get<double>();
      l.name = item.value("name", std::string());
      model.layers.push_back(std::move(l));
    }
  } catch (const json::exception& e) {
    throw ValidationError(std::string("model: malformed description: ") + e.what());
  }
  ValidateModel(model);
  return model;
}

json ModelToJson(const ModelSpec& model) {
  json arr = json::array();
  for (const LayerSpec& l : model.layers) {
    json item;
    item["param_bytes"] = l.param_bytes;
    item["activation_bytes_per_sample"] = l.activation_bytes_per_sample;
    item["fwd_time_per_sample_ms"] = l.fwd_time_per_sample_ms;
    if (!l.name.empty()) item["name"] = l.name;
    arr.push_back(std::move(item));
  }
  json out;
  out["dtype_bytes"] = model.dtype_bytes;
  out["layers"] = std::move(arr);
  return out;
}

ModelSpec LoadModel(const std::string& path) { return ModelFromJson(ReadJsonFile(path, "model")); }

ModelSpec UniformModel(int num_layers, int64_t param_bytes, int64_t activation_bytes_per_sample,
                       double fwd_time_per_sample_ms) {
  if (num_layers < 1) throw ValidationError("uniform model: num_layers must be >= 1");
  ModelSpec model;
  for (int i = 0; i < num_layers; ++i) {
    LayerSpec l;
    l.id = i;
    l.param_bytes = param_bytes;
    l.activation_bytes_per_sample = activation_bytes_per_sample;
    l.fwd_time_per_sample_ms = fwd_time_per_sample_ms;
    model.layers.push_back(l);
  }
  ValidateModel(model);
  return model;
}

// ---------------------------------------------------------------------------- cluster

void ValidateCluster(const ClusterSpec& c) {
  if (!IsPowerOfTwo(c.num_devices))
    throw ValidationError("cluster: num_devices must be a power of two");
  if (!IsPowerOfTwo(c.island_size))
    throw ValidationError("cluster: island_size must be a power of two");
  if (c.num_devices % c.island_size != 0)
    throw ValidationError("cluster: island_size must divide num_devices");
  if (!(c.inter_island_bw_gbps > 0.0))
    throw ValidationError("cluster: inter_island_bw_gbps must be > 0");
  if (c.intra_island_bw_gbps < c.inter_island_bw_gbps)
    throw ValidationError("cluster: intra_island_bw_gbps must be >= inter_island_bw_gbps");
  if (c.memory_budget_bytes <= 0) throw ValidationError("cluster: memory_budget_bytes must be > 0");
}

ClusterSpec ClusterFromJson(const json& j) {
  ClusterSpec c;
  try {
    c.num_devices = j.at("num_devices").get<int>();
    c.memory_budget_bytes = j.at("memory_budget_bytes").get<int64_t>();
    c.island_size = j.at("island_size").get<int>();
    c.intra_island_bw_gbps = j.at("intra_island_bw_gbps").get<double>();
    c.inter_island_bw_gbps = j.at("inter_island_bw_gbps").get<double>();
  } catch (const json::exception& e) {
    throw ValidationError(std::string("cluster: malformed description: ") + e.what());
  }
  ValidateCluster(c);
  return c;
}

json ClusterToJson(const ClusterSpec& c) {
  json out;
  out["num_devices"] = c.num_devices;
  out["memory_budget_bytes"] = c.memory_budget_bytes;
  out["island_size"] = c.island_size;
  out["intra_island_bw_gbps"] = c.intra_island_bw_gbps;
  out["inter_island_bw_gbps"] = c.inter_island_bw_gbps;
  return out;
}

ClusterSpec LoadCluster(const std::string& path) {
  return ClusterFromJson(ReadJsonFile(path, "cluster"));
}

double GroupBandwidthGbps(const ClusterSpec& c, int group_size) {
  if (!IsPowerOfTwo(group_size))
    throw ValidationError("group_bandwidth: group_size must be a power of two");
  if (group_size > c.num_devices)
    throw ValidationError("group_bandwidth: group_size exceeds the device count");
  if (group_size <= c.island_size) return c.intra_island_bw_gbps;
  return c.inter_island_bw_gbps;
}

// ---------------------------------------------------------------------------- profile

void ValidateProfile(const CostProfile& p) {
  if (!(p.backward_multiplier > 0.0))
    throw ValidationError("profile: backward_multiplier must be > 0");
  if (!(p.overlap_slowdown >= 1.0)) throw ValidationError("profile: overlap_slowdown must be >= 1");
  if (!(p.optimizer_state_multiplier >= 0.0))
    throw ValidationError("profile: optimizer_state_multiplier must be >= 0");
  if (!(p.tp_activation_replication >= 0.0 && p.tp_activation_replication <= 1.0))
    throw ValidationError("profile: tp_activation_replication must be in [0, 1]");
  if (p.memory_granularity_bytes <= 0)
    throw ValidationError("profile: memory_granularity_bytes must be > 0");
}

CostProfile ProfileFromJson(const json& j) {
  CostProfile p;
  try {
    p.backward_multiplier = j.value("backward_multiplier", p.backward_multiplier);
    p.overlap_slowdown = j.value("overlap_slowdown", p.overlap_slowdown);
    p.optimizer_state_multiplier =
        j.value("optimizer_state_multiplier", p.optimizer_state_multiplier);
    p.tp_activation_replication = j.value("tp_activation_replication", p.tp_activation_replication);
    p.memory_granularity_bytes = j.value("memory_granularity_bytes", p.memory_granularity_bytes);
  } catch (const json::exception& e) {
    throw ValidationError(std::string("profile: malformed description: ") + e.what());
  }
  ValidateProfile(p);
  return p;
}

json ProfileToJson(const CostProfile& p) {
  json out;
  out["backward_multiplier"] = p.backward_multiplier;
  out["overlap_slowdown"] = p.overlap_slowdown;
  out["optimizer_state_multiplier"] = p.optimizer_state_multiplier;
  out["tp_activation_replication"] = p.tp_activation_replication;
  out["memory_granularity_bytes"] = p.memory_granularity_bytes;
  return out;
}

CostProfile LoadProfile(const std::string& path) {
  return ProfileFromJson(ReadJsonFile(path, "profile"));
}

}  // namespace parplan
