// parplan_cli.cc — the `parplan` command line, a drop-in for the reference front-end
// (proj/tools/parplan_main.cc) on top of this repo's planner, plus the executor-facing
// subcommands SURVEY.md §8(f)1 asks for.
//
//   parplan plan        --model M --cluster C [--profile P] [--batches 8,16] [--pp-guideline
//                       layers|params|memory|time] [--no-prune] [--out plan.json]
//   parplan enumerate   --group-size G [--no-prune] [--out set.json]
//   parplan estimate    --model M --cluster C [--profile P] [--strategy S] [--batch B] [--csv F]
//   parplan sweep       --model M --cluster C --budgets 8,12 [planner flags] [--csv F]
//   parplan oracle-plan (flags of plan; exhaustive search, small instances only)
//   parplan run         planner flags | --plan plan.json, [--shape h,heads,seq,ffn] [--steps K]
//                       [--warmup W] ...  -> executes the plan on B200 (libgx.so)
//   parplan profile     --model M [--shape ...] [--batch B] --out-model F --out-profile F
//                       -> measures fwd time / backward multiplier on B200 for the search
//
// Exit codes follow the reference (parplan_main.cc:40-42): 0 ok, 1 configuration / usage
// error ("error: ..." on stderr), 2 infeasible ("infeasible: ..." on stderr).  Output text,
// JSON and CSV formats are the reference's (PrintPlanSummary parplan_main.cc:111-125,
// RunEstimate 167-213, RunSweep 215-252); PLANNER_THREADS sets the search's thread count
// (parplan_main.cc:73-75).  The reference parses flags with CLI11 (absent from this image);
// the parser here is a small table-driven one accepting the same spellings: `--flag value`,
// `--flag=value`, comma (or space) separated lists.
//
// `run` / `profile` load libgx.so lazily (dlopen, next to this binary or $GX_LIB), so the
// planning subcommands work on machines without a GPU stack.
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <nlohmann/json.hpp>

#include "gx.h"
#include "parplan/cluster.h"
#include "parplan/common.h"
#include "parplan/cost_model.h"
#include "parplan/model_ir.h"
#include "parplan/oracle.h"
#include "parplan/planner.h"
#include "parplan/strategy.h"

namespace {

using nlohmann::json;

enum Exit : int { kOk = 0, kConfig = 1, kInfeasible = 2 };

// ------------------------------------------------------------------------------ arguments

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// One declared option of a subcommand.  Values are stored as text and converted by the
// typed accessors, so a bad number is reported against the flag that carried it.
struct OptSpec {
  std::string name;  // without the leading "--"
  enum Kind { kValue, kList, kFlag } kind = kValue;
  bool required = false;
  std::string help;
  std::vector<std::string> choices;  // empty: any value
  enum Type { kText, kInt, kReal } type = kText;  // checked while parsing, like CLI11
};

class Args {
 public:
  Args(std::string cmd, std::vector<OptSpec> specs) : cmd_(std::move(cmd)), specs_(std::move(specs)) {}

  void parse(const std::vector<std::string>& tok) {
    for (size_t i = 0; i < tok.size(); ++i) {
      const std::string& t = tok[i];
      if (t.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + t + "'");
      std::string name = t.substr(2), inline_value;
      bool has_inline = false;
      if (const size_t eq = name.find('='); eq != std::string::npos) {
        inline_value = name.substr(eq + 1);
        name = name.substr(0, eq);
        has_inline = true;
      }
      const OptSpec* s = find(name);
      if (s == nullptr) throw UsageError("unknown option --" + name + " for '" + cmd_ + "'");
      std::vector<std::string>& vals = values_[name];
      if (s->kind == OptSpec::kFlag) {
        if (has_inline) throw UsageError("--" + name + " takes no value");
        vals.push_back("1");
        continue;
      }
      std::vector<std::string> raw;
      if (has_inline) {
        raw.push_back(inline_value);
      } else {
        if (i + 1 >= tok.size()) throw UsageError("--" + name + " needs a value");
        raw.push_back(tok[++i]);
        // lists also take further space-separated items up to the next option
        while (s->kind == OptSpec::kList && i + 1 < tok.size() && tok[i + 1].rfind("--", 0) != 0)
          raw.push_back(tok[++i]);
      }
      if (s->kind == OptSpec::kValue) {
        vals.assign(1, raw[0]);
      } else {
        for (const std::string& r : raw) {
          std::stringstream ss(r);
          std::string item;
          while (std::getline(ss, item, ',')) {
            if (!item.empty()) vals.push_back(item);
          }
        }
      }
      for (const std::string& v : vals) {
        if (s->type == OptSpec::kInt) (void)to_int(name, v);
        if (s->type == OptSpec::kReal) (void)to_double(name, v);
      }
      if (!s->choices.empty()) {
        for (const std::string& v : vals) {
          if (std::find(s->choices.begin(), s->choices.end(), v) == s->choices.end())
            throw UsageError("--" + name + ": '" + v + "' not in {" + join(s->choices) + "}");
        }
      }
    }
    for (const OptSpec& s : specs_) {
      if (s.required && !has(s.name)) throw UsageError("--" + s.name + " is required");
    }
  }

  bool has(const std::string& n) const { return values_.count(n) != 0; }
  std::string str(const std::string& n, const std::string& dflt = "") const {
    const auto it = values_.find(n);
    return it == values_.end() || it->second.empty() ? dflt : it->second.back();
  }
  int integer(const std::string& n, int dflt) const {
    return has(n) ? to_int(n, str(n)) : dflt;
  }
  double real(const std::string& n, double dflt) const {
    return has(n) ? to_double(n, str(n)) : dflt;
  }
  std::vector<int> ints(const std::string& n) const {
    std::vector<int> out;
    if (const auto it = values_.find(n); it != values_.end())
      for (const std::string& v : it->second) out.push_back(to_int(n, v));
    return out;
  }
  std::vector<double> reals(const std::string& n) const {
    std::vector<double> out;
    if (const auto it = values_.find(n); it != values_.end())
      for (const std::string& v : it->second) out.push_back(to_double(n, v));
    return out;
  }

  std::string usage() const {
    std::string u = "usage: parplan " + cmd_;
    for (const OptSpec& s : specs_) {
      std::string item = "--" + s.name + (s.kind == OptSpec::kFlag ? "" : " <v>");
      u += s.required ? " " + item : " [" + item + "]";
    }
    u += "\n";
    for (const OptSpec& s : specs_) u += "  --" + s.name + std::string(std::max<size_t>(1, 16 - s.name.size()), ' ') + s.help + "\n";
    return u;
  }

 private:
  static std::string join(const std::vector<std::string>& v) {
    std::string o;
    for (const std::string& s : v) o += (o.empty() ? "" : ",") + s;
    return o;
  }
  const OptSpec* find(const std::string& n) const {
    for (const OptSpec& s : specs_)
      if (s.name == n) return &s;
    return nullptr;
  }
  static int to_int(const std::string& n, const std::string& v) {
    size_t used = 0;
    int x = 0;
    try {
      x = std::stoi(v, &used);
    } catch (const std::exception&) {
      used = std::string::npos;
    }
    if (used != v.size()) throw UsageError("--" + n + ": '" + v + "' is not an integer");
    return x;
  }
  static double to_double(const std::string& n, const std::string& v) {
    size_t used = 0;
    double x = 0;
    try {
      x = std::stod(v, &used);
    } catch (const std::exception&) {
      used = std::string::npos;
    }
    if (used != v.size()) throw UsageError("--" + n + ": '" + v + "' is not a number");
    return x;
  }

  std::string cmd_;
  std::vector<OptSpec> specs_;
  std::map<std::string, std::vector<std::string>> values_;
};

std::vector<OptSpec> planner_opts() {
  return {
      {"model", OptSpec::kValue, true, "model description JSON", {}},
      {"cluster", OptSpec::kValue, true, "cluster description JSON", {}},
      {"profile", OptSpec::kValue, false, "cost profile JSON", {}},
      {"batches", OptSpec::kList, false, "global batch size candidates (ascending)", {}, OptSpec::kInt},
      {"pp-guideline", OptSpec::kValue, false, "pipeline partition guideline",
       {"layers", "params", "memory", "time"}},
      {"no-prune", OptSpec::kFlag, false, "keep strategies mixing dp and sdp", {}},
  };
}

std::vector<OptSpec> with(std::vector<OptSpec> base, std::vector<OptSpec> extra) {
  base.insert(base.end(), extra.begin(), extra.end());
  return base;
}

// ------------------------------------------------------------------------------ planning

struct PlannerInputs {
  parplan::ModelSpec model;
  parplan::ClusterSpec cluster;
  parplan::CostProfile profile;
  parplan::PlannerOptions options;
  std::vector<int> batches;
};

PlannerInputs load_inputs(const Args& a) {
  PlannerInputs in;
  in.model = parplan::LoadModel(a.str("model"));
  in.cluster = parplan::LoadCluster(a.str("cluster"));
  in.profile = a.str("profile").empty() ? parplan::CostProfile{} : parplan::LoadProfile(a.str("profile"));
  in.options.guideline = parplan::PpGuidelineFromName(a.str("pp-guideline", "layers"));
  in.options.prune = !a.has("no-prune");
  if (const char* env = std::getenv("PLANNER_THREADS")) in.options.num_threads = std::max(1, std::atoi(env));
  in.batches = a.ints("batches");
  if (in.batches.empty()) in.batches = parplan::DefaultBatchCandidates();
  return in;
}

std::string gib(double bytes) {
  char b[32];
  std::snprintf(b, sizeof(b), "%.2f GiB", bytes / static_cast<double>(parplan::kGiB));
  return b;
}

// "[name] xN | [name] xM": runs of consecutive layers with one strategy (Fig. 8 style).
std::string ribbon(const parplan::StageAssignment& st) {
  std::string out;
  for (size_t i = 0, j; i < st.strategies.size(); i = j) {
    for (j = i + 1; j < st.strategies.size() && st.strategies[j] == st.strategies[i]; ++j) {
    }
    std::string name = st.strategies[i].ToString();
    if (name.empty()) name = "serial";
    if (!out.empty()) out += " | ";
    out += "[" + name + "] x" + std::to_string(j - i);
  }
  return out;
}

void print_summary(const parplan::ParallelPlan& p) {
  std::printf("batch size       %d\n", p.batch_size);
  std::printf("pp degree        %d  (micro-batches: %d)\n", p.pp_degree, p.micro_batches);
  std::printf("iteration time   %.3f ms\n", p.iteration_time_ms);
  std::printf("throughput       %.3f samples/s\n", p.throughput_samples_per_sec);
  for (size_t s = 0; s < p.stages.size(); ++s) {
    const parplan::StageAssignment& st = p.stages[s];
    std::printf("stage %zu  layers [%d,%d)  cost %.3f ms  peak %s\n", s, st.begin_layer,
                st.end_layer, st.stage_cost_ms, gib(st.peak_memory_bytes).c_str());
    std::printf("  %s\n", ribbon(st).c_str());
  }
}

void write_text(const std::string& path, const std::string& text) {
  std::ofstream f(path);
  if (!f) throw parplan::ValidationError("cannot write " + path);
  f << text;
}

void emit_json(const json& j, const std::string& path) {
  if (path.empty()) {
    std::cout << j.dump(2) << "\n";
  } else {
    write_text(path, j.dump(2) + "\n");
  }
}

// plan / oracle-plan.  Returns the plan JSON through *plan_json when non-null (run).
int cmd_plan(const Args& a, bool exhaustive, json* plan_json = nullptr, bool quiet = false) {
  const PlannerInputs in = load_inputs(a);
  const parplan::PlanOutcome r =
      exhaustive ? parplan::ExhaustivePlan(in.model, in.cluster, in.profile, in.batches, in.options)
                 : parplan::Optimize(in.model, in.cluster, in.profile, in.batches, in.options);
  if (!r.feasible()) {
    std::cerr << "infeasible: " << r.diagnostic << "\n";
    return kInfeasible;
  }
  if (!quiet) print_summary(*r.plan);
  const json j = parplan::PlanToJson(*r.plan, in.model, in.profile);
  if (plan_json != nullptr) {
    *plan_json = j;
    if (!a.str("out").empty() && !quiet) emit_json(j, a.str("out"));
  } else {
    emit_json(j, a.str("out"));
  }
  return kOk;
}

int cmd_enumerate(const Args& a) {
  const parplan::StrategySet set = parplan::EnumerateStrategies(a.integer("group-size", 0), !a.has("no-prune"));
  emit_json(parplan::StrategySetToJson(set), a.str("out"));
  return kOk;
}

int cmd_estimate(const Args& a) {
  const parplan::ModelSpec model = parplan::LoadModel(a.str("model"));
  const parplan::ClusterSpec cluster = parplan::LoadCluster(a.str("cluster"));
  const parplan::CostProfile profile =
      a.str("profile").empty() ? parplan::CostProfile{} : parplan::LoadProfile(a.str("profile"));
  const std::string text = a.str("strategy");
  const int batch = a.integer("batch", 8);
  const parplan::HybridStrategy s = parplan::StrategyFromString(text);
  const double bw = parplan::GroupBandwidthGbps(cluster, s.group_size);

  std::string csv =
      "layer,forward_ms,backward_ms,comm_ms_unoverlapped,total_ms,params_bytes,grads_bytes,"
      "optimizer_bytes,activation_bytes,total_bytes\n";
  std::printf("strategy %s  batch %d  bandwidth %.1f GB/s\n", text.empty() ? "serial" : text.c_str(),
              batch, bw);
  std::printf("%5s %12s %12s %12s %12s %14s %14s\n", "layer", "fwd(ms)", "bwd(ms)", "comm(ms)",
              "total(ms)", "memory", "activations");
  for (const parplan::LayerSpec& l : model.layers) {
    const auto c = parplan::EstimateLayerCost(l, s, batch, bw, profile);
    const auto m = parplan::EstimateMemory(l, s, batch, profile);
    if (!c || !m) {
      std::cerr << "infeasible: batch " << batch
                << " cannot be split across the data-parallel replicas\n";
      return kInfeasible;
    }
    std::printf("%5d %12.4f %12.4f %12.4f %12.4f %14s %14s\n", l.id, c->forward_ms, c->backward_ms,
                c->comm_ms_unoverlapped, c->total_ms, gib(m->total_bytes()).c_str(),
                gib(m->activation_bytes).c_str());
    char row[512];
    std::snprintf(row, sizeof(row), "%d,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g\n", l.id,
                  c->forward_ms, c->backward_ms, c->comm_ms_unoverlapped, c->total_ms,
                  m->params_bytes, m->grads_bytes, m->optimizer_bytes, m->activation_bytes,
                  m->total_bytes());
    csv += row;
  }
  if (!a.str("csv").empty()) write_text(a.str("csv"), csv);
  return kOk;
}

int cmd_sweep(const Args& a) {
  PlannerInputs in = load_inputs(a);
  std::string csv = "budget_gb,batch_size,pp_degree,throughput_samples_per_s\n";
  for (const double gb : a.reals("budgets")) {
    if (!(gb > 0.0)) throw parplan::ValidationError("sweep: budgets must be positive");
    in.cluster.memory_budget_bytes = static_cast<int64_t>(gb * static_cast<double>(parplan::kGiB));
    const parplan::PlanOutcome r = parplan::Optimize(in.model, in.cluster, in.profile, in.batches, in.options);
    char row[160];
    if (r.feasible()) {
      std::snprintf(row, sizeof(row), "%g,%d,%d,%.6f\n", gb, r.plan->batch_size, r.plan->pp_degree,
                    r.plan->throughput_samples_per_sec);
    } else {
      std::snprintf(row, sizeof(row), "%g,OOM,OOM,OOM\n", gb);
    }
    csv += row;
  }
  std::cout << csv;
  if (!a.str("csv").empty()) write_text(a.str("csv"), csv);
  return kOk;
}

// ------------------------------------------------------------------------------ executor

// The gx_exec_* entry points, resolved from libgx.so at first use.
struct GxLib {
  decltype(&gx_last_error) last_error = nullptr;
  decltype(&gx_exec_create) create = nullptr;
  decltype(&gx_exec_destroy) destroy = nullptr;
  decltype(&gx_exec_init_params) init_params = nullptr;
  decltype(&gx_exec_load_batch) load_batch = nullptr;
  decltype(&gx_exec_time) time = nullptr;
  decltype(&gx_exec_loss) loss = nullptr;
  decltype(&gx_exec_info) info = nullptr;
  decltype(&gx_exec_step) step = nullptr;
  decltype(&gx_nccl_unique_id) nccl_id = nullptr;

  static const GxLib& get() {
    static GxLib lib = load();
    return lib;
  }

 private:
  static GxLib load() {
    std::string path;
    if (const char* e = std::getenv("GX_LIB")) {
      path = e;
    } else {
      std::error_code ec;
      const auto self = std::filesystem::read_symlink("/proc/self/exe", ec);
      path = (ec ? std::filesystem::path(".") : self.parent_path()) / "libgx.so";
    }
    void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) throw parplan::ValidationError(std::string("cannot load executor library: ") + dlerror());
    GxLib L;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (fn == nullptr) throw parplan::ValidationError(std::string("executor library lacks ") + name);
    };
    sym(L.last_error, "gx_last_error");
    sym(L.create, "gx_exec_create");
    sym(L.destroy, "gx_exec_destroy");
    sym(L.init_params, "gx_exec_init_params");
    sym(L.load_batch, "gx_exec_load_batch");
    sym(L.time, "gx_exec_time");
    sym(L.loss, "gx_exec_loss");
    sym(L.info, "gx_exec_info");
    sym(L.step, "gx_exec_step");
    sym(L.nccl_id, "gx_nccl_unique_id");
    return L;
  }
};

// Executor failures map to the CLI's codes: infeasible stays 2, everything else is 1.
struct ExecError : std::runtime_error {
  int code;
  ExecError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void gx_check(int rc, const char* what) {
  if (rc == GX_OK) return;
  throw ExecError(rc == GX_ERR_INFEASIBLE ? kInfeasible : kConfig,
                  std::string(what) + ": " + GxLib::get().last_error());
}

class Executor {
 public:
  explicit Executor(const json& cfg) { gx_check(GxLib::get().create(cfg.dump().c_str(), &h_), "gx_exec_create"); }
  ~Executor() {
    if (h_ != nullptr) GxLib::get().destroy(h_);
  }
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;
  gx_exec* get() const { return h_; }
  json info() const {
    size_t need = 0;
    gx_check(GxLib::get().info(h_, nullptr, 0, &need), "gx_exec_info");
    std::string buf(need, '\0');
    gx_check(GxLib::get().info(h_, buf.data(), need, &need), "gx_exec_info");
    return json::parse(buf.c_str());
  }

 private:
  gx_exec* h_ = nullptr;
};

// "hidden,heads,seq,ffn" -> the executor's per-layer shape object (encoder layer).
json parse_shape(const std::string& text) {
  std::vector<int> v;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) {
    size_t used = 0;
    int x = 0;
    try {
      x = std::stoi(item, &used);
    } catch (const std::exception&) {
      used = std::string::npos;
    }
    if (used != item.size() || x <= 0) throw UsageError("--shape: '" + text + "' is not hidden,heads,seq,ffn");
    v.push_back(x);
  }
  if (v.size() != 4 || v[0] % v[1] != 0) throw UsageError("--shape: '" + text + "' is not hidden,heads,seq,ffn");
  return {{"hidden", v[0]}, {"heads", v[1]}, {"head_dim", v[0] / v[1]}, {"seq", v[2]}, {"ffn", v[3]},
          {"kind", "encoder"}};
}

json read_json(const std::string& path, const char* what) {
  std::ifstream f(path);
  if (!f) throw parplan::ValidationError(std::string("cannot open ") + what + " file " + path);
  try {
    return json::parse(f);
  } catch (const json::exception& e) {
    throw parplan::ValidationError(std::string("malformed ") + what + " JSON " + path + ": " + e.what());
  }
}

// The model file as JSON with an executor shape on every layer (the reference ignores unknown
// keys, model_ir.cc:69-95, so shaped files stay valid planner inputs).
json shaped_model(const Args& a) {
  json m = read_json(a.str("model"), "model");
  (void)parplan::ModelFromJson(m);  // the planner's validation
  const bool override_all = a.has("shape");
  const json shape = override_all ? parse_shape(a.str("shape")) : json();
  json& layers = m.at("layers");
  for (size_t i = 0; i < layers.size(); ++i) {
    if (override_all) {
      layers[i]["shape"] = shape;
    } else if (!layers[i].contains("shape")) {
      throw parplan::ValidationError("model layer " + std::to_string(i) +
                                     " has no executor shape (add \"shape\" or pass --shape)");
    }
  }
  return m;
}

// Deterministic synthetic bf16 batch (Box-Muller over a 64-bit LCG), like bench.py's data.
std::vector<uint16_t> synthetic_bf16(size_t n, uint64_t seed) {
  std::vector<uint16_t> out(n);
  uint64_t s = seed * 6364136223846793005ull + 1442695040888963407ull;
  auto uni = [&]() {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return (static_cast<double>(s >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  };
  for (size_t i = 0; i < n; ++i) {
    const float x = static_cast<float>(std::sqrt(-2.0 * std::log(uni())) * std::cos(6.283185307179586 * uni()));
    uint32_t b;
    std::memcpy(&b, &x, 4);
    out[i] = static_cast<uint16_t>((b + 0x7fffu + ((b >> 16) & 1u)) >> 16);  // round to nearest even
  }
  return out;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e == nullptr || *e == '\0' ? dflt : std::atoi(e);
}

// Rank 0 creates the NCCL id and publishes it through a file as "<launch id> <hex>"; the other
// ranks poll for a file carrying THEIR launch id, so a leftover of an earlier (e.g. crashed)
// launch on the same path is never read.  The launch id is shared by every rank of one launch:
// $PARPLAN_LAUNCH_ID, else torchrun's $TORCHELASTIC_RUN_ID.  Without either, only a file
// written after this process started (minus a few seconds of launch skew) is accepted.
// Rank 0 removes the file once its communicator exists (NCCL init is collective, so every rank
// has read it by then).
std::string launch_id() {
  for (const char* name : {"PARPLAN_LAUNCH_ID", "TORCHELASTIC_RUN_ID"}) {
    const char* e = std::getenv(name);
    if (e != nullptr && *e != '\0') return e;
  }
  return "-";
}

const auto kProcessStart = std::filesystem::file_time_type::clock::now();

std::string exchange_nccl_id(const std::string& path, int rank) {
  const std::string nonce = launch_id();
  if (rank == 0) {
    char hex[257];
    gx_check(GxLib::get().nccl_id(hex, sizeof(hex)), "gx_nccl_unique_id");
    std::error_code ec;
    std::filesystem::remove(path, ec);  // a stale id must not outlive this launch's start
    const std::string tmp = path + ".tmp";
    write_text(tmp, nonce + " " + hex);
    std::filesystem::rename(tmp, path);
    return hex;
  }
  const auto not_before = kProcessStart - std::chrono::seconds(5);
  for (int i = 0; i < 1200; ++i) {
    std::error_code ec;
    const auto mtime = std::filesystem::last_write_time(path, ec);
    std::ifstream f(path);
    std::string tag, hex;
    if (!ec && f && (f >> tag >> hex) && hex.size() == 256 && tag == nonce &&
        (nonce != "-" || mtime >= not_before))
      return hex;
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
  }
  throw parplan::ValidationError("timed out waiting for the NCCL id in " + path);
}

int cmd_run(const Args& a) {
  json model = shaped_model(a);
  json plan;
  int world = 0;
  const int rank = env_int("RANK", 0);
  if (a.has("plan")) {
    plan = read_json(a.str("plan"), "plan");
    const parplan::ClusterSpec cluster = parplan::LoadCluster(a.str("cluster"));
    world = cluster.num_devices;
  } else {
    const int rc = cmd_plan(a, false, &plan, /*quiet=*/rank != 0);
    if (rc != kOk) return rc;
    world = parplan::LoadCluster(a.str("cluster")).num_devices;
  }
  const int env_world = env_int("WORLD_SIZE", 1);
  const bool nccl = env_world > 1;
  if (nccl && env_world != world)
    throw parplan::ValidationError("WORLD_SIZE " + std::to_string(env_world) +
                                   " does not match the cluster's num_devices " + std::to_string(world));
  const float p = static_cast<float>(a.real("dropout", 0.0));
  json cfg = {{"plan", plan},
              {"model", model},
              {"world_size", world},
              {"comm", nccl ? "nccl" : "sim"},
              {"dropout_attn", p},
              {"dropout_hidden", p},
              {"seed", a.integer("seed", 1234)},
              {"lr", a.real("lr", 1e-4)},
              {"optimizer", !a.has("no-optimizer")},
              {"device", env_int("LOCAL_RANK", a.integer("device", 0))}};
  if (a.has("enforce-budget"))
    cfg["memory_cap_bytes"] = parplan::LoadCluster(a.str("cluster")).memory_budget_bytes;
  const char* port = std::getenv("MASTER_PORT");
  const std::string id_file = a.str("nccl-id-file", "/tmp/parplan_nccl_" + std::string(port ? port : "0") + ".id");
  if (nccl) {
    cfg["local_ranks"] = json::array({rank});
    cfg["nccl_id_hex"] = exchange_nccl_id(id_file, rank);
  }
  Executor ex(cfg);
  if (nccl && rank == 0) {  // every rank has joined the communicator, so has read the id
    std::error_code ec;
    std::filesystem::remove(id_file, ec);
  }
  const GxLib& L = GxLib::get();
  gx_check(L.init_params(ex.get(), static_cast<uint64_t>(a.integer("seed", 1234)), 0.02f), "init_params");
  const json& l0 = model.at("layers").front().at("shape");
  const json& ll = model.at("layers").back().at("shape");
  const int B = plan.at("batch_size").get<int>();
  const auto x = synthetic_bf16(static_cast<size_t>(B) * l0.at("seq").get<int>() * l0.at("hidden").get<int>(), 1);
  const auto y = synthetic_bf16(static_cast<size_t>(B) * ll.at("seq").get<int>() * ll.at("hidden").get<int>(), 2);
  gx_check(L.load_batch(ex.get(), x.data(), y.data()), "load_batch");
  const int steps = std::max(1, a.integer("steps", 10));
  const int warmup = std::max(0, a.integer("warmup", 3));
  const int flags = a.has("no-graph") ? 0 : 1;
  double ms = 0;
  gx_check(L.time(ex.get(), flags, warmup, steps, &ms), "gx_exec_time");
  float loss = 0.f;
  gx_check(L.loss(ex.get(), &loss), "loss");
  // end to end: host batch in, loss out, every step (gx_exec_step)
  float e2e_loss = 0.f;
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) gx_check(L.step(ex.get(), x.data(), y.data(), flags, &e2e_loss), "gx_exec_step");
  const double e2e_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / steps;
  const json info = ex.info();
  if (rank == 0) {
    const char* mode = nccl ? "nccl" : (world > 1 ? "sim (all ranks on one device)" : "1 device");
    std::printf("executor         world %d  comm %s\n", world, mode);
    std::printf("step time        %.3f ms  (device, %d steps after %d warm-up)\n", ms, steps, warmup);
    std::printf("end-to-end       %.3f ms/step  (host batch in, loss out)\n", e2e_ms);
    std::printf("throughput       %.3f samples/s\n", B / (ms / 1e3));
    std::printf("loss             %.6f  (step %d)\n", loss, warmup + steps);
    if (!a.str("report").empty()) {
      const json rep = {{"plan", plan},           {"world_size", world},   {"comm", nccl ? "nccl" : "sim"},
                        {"steps", steps},         {"warmup", warmup},      {"ms_per_step", ms},
                        {"e2e_ms_per_step", e2e_ms}, {"samples_per_s", B / (ms / 1e3)},
                        {"loss", loss},           {"e2e_loss", e2e_loss},  {"info", info}};
      write_text(a.str("report"), rep.dump(2) + "\n");
    }
  }
  if (!std::isfinite(loss) || !std::isfinite(e2e_loss)) {
    std::cerr << "error: non-finite loss\n";
    return kConfig;
  }
  return kOk;
}

// Time `shapes` run in sequence (serial strategy, `batch` samples, graph replay).
double time_layers(const std::vector<json>& shapes, int batch, bool forward_only, int warmup,
                   int steps, int device) {
  json layers = json::array(), plan_layers = json::array();
  for (size_t i = 0; i < shapes.size(); ++i) {
    layers.push_back({{"param_bytes", 1}, {"activation_bytes_per_sample", 1},
                      {"fwd_time_per_sample_ms", 1.0}, {"shape", shapes[i]}});
    plan_layers.push_back({{"id", static_cast<int>(i)}, {"strategy", ""}});
  }
  const int n = static_cast<int>(shapes.size());
  const json model = {{"dtype_bytes", 4}, {"layers", layers}};
  const json plan = {{"pp_degree", 1},
                     {"micro_batches", 1},
                     {"batch_size", batch},
                     {"stages", json::array({{{"layer_range", {0, n}}, {"layers", plan_layers}}})}};
  const json cfg = {{"plan", plan},         {"model", model},        {"world_size", 1},
                    {"comm", "sim"},        {"forward_only", forward_only}, {"optimizer", false},
                    {"dropout_attn", 0.1},  {"dropout_hidden", 0.1}, {"device", device}};
  Executor ex(cfg);
  const GxLib& L = GxLib::get();
  gx_check(L.init_params(ex.get(), 1, 0.02f), "init_params");
  const json& f = shapes.front();
  const json& z = shapes.back();
  const auto x = synthetic_bf16(static_cast<size_t>(batch) * f.at("seq").get<int>() * f.at("hidden").get<int>(), 3);
  const auto y = synthetic_bf16(static_cast<size_t>(batch) * z.at("seq").get<int>() * z.at("hidden").get<int>(), 4);
  gx_check(L.load_batch(ex.get(), x.data(), y.data()), "load_batch");
  double ms = 0;
  gx_check(L.time(ex.get(), 1, warmup, steps, &ms), "gx_exec_time");
  return ms;
}

double round_to(double x, int digits) {
  const double f = std::pow(10.0, digits);
  return std::nearbyint(x * f) / f;
}

// Measures the planner's time inputs on this GPU: fwd_time_per_sample_ms per
// layer (LayerSpec, model_ir.h:34) and backward_multiplier (CostProfile, cost_model.h:46),
// as paper_2211_13878_b200/profiler.py does, and writes them in the reference schemas.
int cmd_profile(const Args& a) {
  json model = shaped_model(a);
  parplan::CostProfile prof =
      a.str("profile").empty() ? parplan::CostProfile{} : parplan::LoadProfile(a.str("profile"));
  const int batch = a.integer("batch", 4);
  if (batch <= 0) throw UsageError("--batch must be positive");
  const int steps = std::max(1, a.integer("steps", 20)), warmup = std::max(0, a.integer("warmup", 3));
  const int device = a.integer("device", 0);
  std::map<std::string, std::pair<double, double>> measured;  // shape -> (fwd, fwd+bwd) ms
  std::vector<std::string> order;
  json raw = json::array();
  json prev;  // the previous layer's shape: a patch-merging layer is timed behind it
  auto time_layer = [&](const json& shape, bool fwd_only) {
    if (!shape.value("merge", false)) return time_layers({shape}, batch, fwd_only, warmup, steps, device);
    return time_layers({prev, shape}, batch, fwd_only, warmup, steps, device) -
           time_layers({prev}, batch, fwd_only, warmup, steps, device);
  };
  for (json& layer : model.at("layers")) {
    const std::string key = layer.at("shape").dump();
    if (measured.count(key) == 0) {
      const double fwd = time_layer(layer.at("shape"), true);
      const double full = time_layer(layer.at("shape"), false);
      measured[key] = {fwd, full};
      order.push_back(key);
      raw.push_back({{"shape", layer.at("shape")}, {"batch", batch}, {"fwd_ms", fwd}, {"fwd_bwd_ms", full}});
      std::printf("shape %s  batch %d  fwd %.4f ms  fwd+bwd %.4f ms\n", key.c_str(), batch, fwd, full);
    }
    layer["fwd_time_per_sample_ms"] = round_to(measured[key].first / batch, 6);
    prev = layer.at("shape");
  }
  double sum = 0;
  int cnt = 0;
  for (const std::string& k : order) {
    const auto [fwd, full] = measured[k];
    if (fwd > 0) {
      sum += (full - fwd) / fwd;
      ++cnt;
    }
  }
  if (cnt > 0) prof.backward_multiplier = round_to(sum / cnt, 4);
  std::printf("backward_multiplier %.4f\n", prof.backward_multiplier);
  (void)parplan::ModelFromJson(model);  // the written files must load back into the planner
  parplan::ValidateProfile(prof);
  const json pj = parplan::ProfileToJson(prof);
  if (!a.str("out-model").empty()) write_text(a.str("out-model"), model.dump(2) + "\n");
  if (!a.str("out-profile").empty()) write_text(a.str("out-profile"), pj.dump(2) + "\n");
  if (a.str("out-model").empty() && a.str("out-profile").empty())
    std::cout << json({{"model", model}, {"profile", pj}, {"raw", raw}}).dump(2) << "\n";
  return kOk;
}

// ------------------------------------------------------------------------------ dispatch

struct Command {
  std::string name, help;
  std::vector<OptSpec> opts;
  std::function<int(const Args&)> run;
};

std::vector<Command> commands() {
  const std::vector<OptSpec> exec_opts = {
      {"shape", OptSpec::kValue, false, "executor layer shape hidden,heads,seq,ffn (all layers)", {}},
      {"steps", OptSpec::kValue, false, "timed steps", {}, OptSpec::kInt},
      {"warmup", OptSpec::kValue, false, "untimed warm-up steps", {}, OptSpec::kInt},
      {"device", OptSpec::kValue, false, "CUDA device (LOCAL_RANK wins when set)", {}, OptSpec::kInt},
  };
  return {
      {"plan", "search for the best plan",
       with(planner_opts(), {{"out", OptSpec::kValue, false, "write the plan JSON here", {}}}),
       [](const Args& a) { return cmd_plan(a, false); }},
      {"enumerate", "dump the strategy set for a group",
       {{"group-size", OptSpec::kValue, true, "device group size", {}, OptSpec::kInt},
        {"no-prune", OptSpec::kFlag, false, "keep strategies mixing dp and sdp", {}},
        {"out", OptSpec::kValue, false, "write the JSON here", {}}},
       cmd_enumerate},
      {"estimate", "per-layer costs and memory for one strategy",
       {{"model", OptSpec::kValue, true, "model JSON", {}},
        {"cluster", OptSpec::kValue, true, "cluster JSON", {}},
        {"profile", OptSpec::kValue, false, "cost profile JSON", {}},
        {"strategy", OptSpec::kValue, false, "strategy string, e.g. tp:2,dp:4 (empty = serial)", {}},
        {"batch", OptSpec::kValue, false, "samples per group", {}, OptSpec::kInt},
        {"csv", OptSpec::kValue, false, "write the table as CSV here", {}}},
       cmd_estimate},
      {"sweep", "plan across memory budgets, emit CSV",
       with(planner_opts(), {{"budgets", OptSpec::kList, true, "memory budgets in GiB", {}, OptSpec::kReal},
                             {"csv", OptSpec::kValue, false, "also write the CSV here", {}}}),
       cmd_sweep},
      {"oracle-plan", "exhaustive reference search (small instances only)",
       with(planner_opts(), {{"out", OptSpec::kValue, false, "write the plan JSON here", {}}}),
       [](const Args& a) { return cmd_plan(a, true); }},
      {"run", "execute a plan (searched, or --plan) on B200 and time it",
       with(with(planner_opts(), exec_opts),
            {{"plan", OptSpec::kValue, false, "plan JSON to execute (skips the search)", {}},
             {"out", OptSpec::kValue, false, "write the searched plan JSON here", {}},
             {"report", OptSpec::kValue, false, "write a JSON run report here", {}},
             {"dropout", OptSpec::kValue, false, "attention/hidden dropout probability", {}, OptSpec::kReal},
             {"seed", OptSpec::kValue, false, "parameter / dropout seed", {}, OptSpec::kInt},
             {"lr", OptSpec::kValue, false, "AdamW learning rate", {}, OptSpec::kReal},
             {"no-optimizer", OptSpec::kFlag, false, "skip the AdamW update", {}},
             {"no-graph", OptSpec::kFlag, false, "launch kernels eagerly instead of a CUDA graph", {}},
             {"enforce-budget", OptSpec::kFlag, false, "cap device memory at the cluster budget", {}},
             {"nccl-id-file", OptSpec::kValue, false, "NCCL id rendezvous file (WORLD_SIZE > 1)", {}}}),
       cmd_run},
      {"profile", "measure layer times on B200 and write planner inputs",
       with({{"model", OptSpec::kValue, true, "model JSON", {}},
             {"profile", OptSpec::kValue, false, "base cost profile JSON", {}},
             {"batch", OptSpec::kValue, false, "samples per timed layer run", {}, OptSpec::kInt},
             {"out-model", OptSpec::kValue, false, "write the measured model JSON here", {}},
             {"out-profile", OptSpec::kValue, false, "write the measured profile JSON here", {}}},
            exec_opts),
       cmd_profile},
  };
}

void top_usage(std::ostream& os, const std::vector<Command>& cmds) {
  os << "hybrid-parallelism planner for layered models (B200 executor)\n"
        "usage: parplan <subcommand> [options]   (parplan <subcommand> --help)\n";
  for (const Command& c : cmds) os << "  " << c.name << std::string(14 - c.name.size(), ' ') << c.help << "\n";
}

}  // namespace

int main(int argc, char** argv) {
  const std::vector<Command> cmds = commands();
  if (argc < 2) {
    top_usage(std::cerr, cmds);
    return kConfig;
  }
  const std::string sub = argv[1];
  if (sub == "--help" || sub == "-h") {
    top_usage(std::cout, cmds);
    return kOk;
  }
  const auto it = std::find_if(cmds.begin(), cmds.end(), [&](const Command& c) { return c.name == sub; });
  if (it == cmds.end()) {
    std::cerr << "error: unknown subcommand '" << sub << "'\n";
    top_usage(std::cerr, cmds);
    return kConfig;
  }
  std::vector<std::string> tok(argv + 2, argv + argc);
  Args args(it->name, it->opts);
  if (std::find(tok.begin(), tok.end(), "--help") != tok.end() ||
      std::find(tok.begin(), tok.end(), "-h") != tok.end()) {
    std::cout << it->help << "\n" << args.usage();
    return kOk;
  }
  try {
    args.parse(tok);
    return it->run(args);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n" << args.usage();
    return kConfig;
  } catch (const ExecError& e) {
    std::cerr << (e.code == kInfeasible ? "infeasible: " : "error: ") << e.what() << "\n";
    return e.code;
  } catch (const std::exception& e) {  // ValidationError, GuardError, I/O
    std::cerr << "error: " << e.what() << "\n";
    return kConfig;
  }
}
