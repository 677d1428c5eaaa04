// executor.cc — the plan executor (see executor.h for the contract and the reference
// semantics each piece follows).
//
// Execution model: a set of *local ranks* is driven in lockstep.  NCCL mode has exactly one
// local rank per process (one GPU each); sim mode places every rank of the world on this
// device and routes collectives through SimComm.  Each layer's forward/backward is split
// into phases that end at a collective, and the driver runs phase k for every local rank of
// the stage before phase k+1, so the same code path serves both modes.
#include "executor_impl.h"

namespace gx {

using xi::json;
using xi::pad64;

Layout make_layout(const Shape& s, int tp, int sdp) {
  Layout L;
  int64_t off = 0;
  auto put = [&](Slot& slot, int64_t n) {
    slot.off = off;
    slot.n = n;
    off += pad64(n);
  };
  const int64_t h = s.h, f = s.ffn;
  put(L.ln1g, h);
  put(L.ln1b, h);
  put(L.ln2g, h);
  put(L.ln2b, h);
  put(L.bqkv, 3 * h / tp);
  put(L.bo, h);
  put(L.b1, f / tp);
  put(L.b2, h);
  const int64_t mc = s.merge ? 2 * h : 0;  // merged channels (4 x h/2)
  put(L.mlng, mc);
  put(L.mlnb, mc);
  const int64_t xh = s.cross ? h : 0, xht = s.cross ? h / tp : 0;
  put(L.ln3g, xh);
  put(L.ln3b, xh);
  put(L.bq2, xht);
  put(L.bkv2, 2 * xht);
  put(L.bo2, xh);
  put(L.rpb, s.rpb ? static_cast<int64_t>(s.heads / tp) * s.rpb_n() : 0);
  put(L.relb, static_cast<int64_t>(s.heads / tp) * s.relb);
  L.acc_end = off;
  put(L.wqkv, 3 * h / tp * h);
  put(L.wo, h * (h / tp));
  put(L.w1, f / tp * h);
  put(L.w2, h * (f / tp));
  put(L.wm, s.merge ? h * mc : 0);  // replicated across TP ranks (identical gradients)
  put(L.wq2, xht * h);
  put(L.wkv2, 2 * xht * h);
  put(L.wo2, h * xht);
  const int64_t q = 64 * static_cast<int64_t>(sdp);
  L.total = (off + q - 1) / q * q;
  return L;
}

int64_t canonical_size(const Shape& s) {
  const int64_t h = s.h, f = s.ffn;
  const int64_t merge = s.merge ? 4 * h + 2 * h * h : 0;  // mln_g, mln_b (2h each), w_m [h][2h]
  // ln3_g ln3_b b_q2 b_kv2(2h) b_o2, w_q2 [h][h], w_kv2 [2h][h], w_o2 [h][h]
  const int64_t cross = s.cross ? 6 * h + 4 * h * h : 0;
  const int64_t rpb = s.rpb ? static_cast<int64_t>(s.heads) * s.rpb_n() : 0;
  const int64_t relb = static_cast<int64_t>(s.heads) * s.relb;  // T5 table [heads][buckets]
  return 4 * h + 3 * h + h + f + h + 3 * h * h + h * h + f * h + h * f + merge + cross + rpb +
         relb;
}

namespace xi {

// Canonical index of local flat element `j` of rank (tp degree t, tp index tr); -1 = padding.
int64_t canon_index(const Shape& s, const Layout& L, int t, int tr, int64_t j) {
  const int64_t h = s.h, f = s.ffn, ht = h / t, ft = f / t;
  // canonical offsets (tp = 1, unpadded)
  const int64_t c_ln1g = 0, c_ln1b = h, c_ln2g = 2 * h, c_ln2b = 3 * h, c_bqkv = 4 * h,
                c_bo = 7 * h, c_b1 = 8 * h, c_b2 = 8 * h + f, c_wqkv = 9 * h + f,
                c_wo = c_wqkv + 3 * h * h, c_w1 = c_wo + h * h, c_w2 = c_w1 + f * h;
  auto in = [&](const Slot& sl, int64_t& k) {
    if (j < sl.off || j >= sl.off + sl.n) return false;
    k = j - sl.off;
    return true;
  };
  int64_t k = 0;
  if (in(L.ln1g, k)) return c_ln1g + k;
  if (in(L.ln1b, k)) return c_ln1b + k;
  if (in(L.ln2g, k)) return c_ln2g + k;
  if (in(L.ln2b, k)) return c_ln2b + k;
  if (in(L.bo, k)) return c_bo + k;
  if (in(L.b2, k)) return c_b2 + k;
  if (in(L.bqkv, k)) return c_bqkv + (k / ht) * h + tr * ht + k % ht;
  if (in(L.b1, k)) return c_b1 + tr * ft + k;
  if (in(L.wqkv, k)) {
    const int64_t row = k / h, col = k % h;
    return c_wqkv + ((row / ht) * h + tr * ht + row % ht) * h + col;
  }
  if (in(L.w1, k)) return c_w1 + (tr * ft + k / h) * h + k % h;
  if (in(L.wo, k)) return c_wo + (k / ht) * h + tr * ht + k % ht;
  if (in(L.w2, k)) return c_w2 + (k / ft) * f + tr * ft + k % ft;
  const int64_t c_m = c_w2 + h * f;  // patch merging, after w_2, unsharded by TP
  if (in(L.mlng, k)) return c_m + k;
  if (in(L.mlnb, k)) return c_m + 2 * h + k;
  if (in(L.wm, k)) return c_m + 4 * h + k;
  if (in(L.ln3g, k)) return c_m + k;  // cross-attention shares the base (never both)
  if (in(L.ln3b, k)) return c_m + h + k;
  if (in(L.bq2, k)) return c_m + 2 * h + tr * ht + k;
  if (in(L.bkv2, k)) return c_m + 3 * h + (k / ht) * h + tr * ht + k % ht;
  if (in(L.bo2, k)) return c_m + 5 * h + k;
  if (in(L.wq2, k)) return c_m + 6 * h + (tr * ht + k / h) * h + k % h;
  if (in(L.wkv2, k)) {
    const int64_t row = k / h, col = k % h;
    return c_m + 6 * h + h * h + ((row / ht) * h + tr * ht + row % ht) * h + col;
  }
  if (in(L.wo2, k)) return c_m + 6 * h + 3 * h * h + (k / ht) * h + tr * ht + k % ht;
  if (in(L.rpb, k)) return c_m + (s.merge ? 4 * h + 2 * h * h : 0) + tr * L.rpb.n + k;
  if (in(L.relb, k)) return c_m + (s.cross ? 6 * h + 4 * h * h : 0) + tr * L.relb.n + k;
  return -1;
}

// T5's relative-position bucket of d = k - q (the published bucketing; pinned against
// transformers' T5Attention in tests/test_layer_oracle.py), bidirectional unless causal,
// max distance 128, computed in double as oracle/layer_oracle.py::t5_buckets does.
std::vector<int8_t> t5_bucket_map(int seq, bool bidirectional, int buckets) {
  std::vector<int8_t> out(2 * seq - 1);
  for (int i = 0; i < 2 * seq - 1; ++i) {
    int n = -(i - (seq - 1));  // query - key
    int nb = buckets, ret = 0;
    if (bidirectional) {
      nb /= 2;
      ret = n < 0 ? nb : 0;
      n = n < 0 ? -n : n;
    } else {
      n = n > 0 ? n : 0;
    }
    const int max_exact = nb / 2;
    int v = n;
    if (n >= max_exact) {
      v = max_exact + static_cast<int>(std::log(static_cast<double>(n) / max_exact) /
                                       std::log(128.0 / max_exact) * (nb - max_exact));
      v = std::min(v, nb - 1);
    }
    out[i] = static_cast<int8_t>(ret + v);
  }
  return out;
}

// Byte-threshold dropout (philox.cuh): thr8 = round(p * 256); kept values scale by
// 256 / (256 - thr8) so the expectation is exact at the effective rate thr8 / 256.
uint32_t threshold_of(float p) {
  if (p <= 0.f) return 0u;
  const int t = static_cast<int>(p * 256.f + 0.5f);
  return static_cast<uint32_t>(t > 255 ? 255 : (t < 1 ? 1 : t));
}
float scale_of(float p) {
  const uint32_t t = threshold_of(p);
  return t == 0u ? 1.f : 256.f / static_cast<float>(256u - t);
}

int ExecutorImpl::init(const json& cfg, std::string* err) {
  try {
    plan_ = cfg.at("plan");
    model_ = cfg.at("model");
    world_ = cfg.at("world_size").get<int>();
    const std::string comm_kind = cfg.value("comm", std::string("sim"));
    // one process per GPU without torch (the parplan CLI): the caller names its device
    if (cfg.contains("device") && comm_kind != "dryrun") {
      const int dev = cfg.at("device").get<int>();
      if (cudaSetDevice(dev) != cudaSuccess) {
        cudaGetLastError();
        *err = "executor: cannot select CUDA device " + std::to_string(dev);
        return kErrCuda;
      }
    }
    sim_ = comm_kind == "sim" || comm_kind == "dryrun";
    comm_kind_ = comm_kind;
    if (comm_kind != "sim" && comm_kind != "dryrun" && comm_kind != "nccl" && comm_kind != "null") {
      *err = "executor: comm must be sim, nccl, null or dryrun";
      return kErrConfig;
    }
    dry_run_ = comm_kind == "dryrun";
    p_attn_ = cfg.value("dropout_attn", 0.0f);
    p_hidden_ = cfg.value("dropout_hidden", 0.0f);
    seed_ = cfg.value("seed", static_cast<uint64_t>(1234));
    lr_ = cfg.value("lr", 1e-4f);
    b1_ = cfg.value("beta1", 0.9f);
    b2_ = cfg.value("beta2", 0.999f);
    eps_ = cfg.value("eps", 1e-8f);
    wd_ = cfg.value("weight_decay", 0.0f);
    optimizer_ = cfg.value("optimizer", true);
    forward_only_ = cfg.value("forward_only", false);
    splitk_ = cfg.value("splitk", true);
    mem_cap_ = cfg.value("memory_cap_bytes", static_cast<int64_t>(0));
    sync_timeout_ms_ = cfg.value("sync_timeout_ms", sync_timeout_ms_);
    wgrad_stream_ = cfg.value("wgrad_stream", true);
    comm_stream_ = cfg.value("comm_stream", true);
    trace_ = cfg.value("trace", false);
    thr_attn_ = threshold_of(p_attn_);
    thr_hidden_ = threshold_of(p_hidden_);

    P_ = plan_.at("pp_degree").get<int>();
    m_ = plan_.at("micro_batches").get<int>();
    B_ = plan_.at("batch_size").get<int>();
    if (world_ % P_ != 0) {
      *err = "executor: world_size must be a multiple of pp_degree";
      return kErrConfig;
    }
    g_ = world_ / P_;
    if (B_ % m_ != 0) {
      *err = "executor: micro_batches must divide batch_size";
      return kErrConfig;
    }
    Bm_ = B_ / m_;
    const json& layers = model_.at("layers");
    L_ = static_cast<int>(layers.size());
    deg_.assign(L_, Deg{});
    shape_.assign(L_, Shape{});
    for (int l = 0; l < L_; ++l) {
      const json& sh = layers[l].at("shape");
      Shape s;
      s.h = sh.at("hidden").get<int>();
      s.heads = sh.at("heads").get<int>();
      s.hd = sh.value("head_dim", s.h / s.heads);
      s.seq = sh.at("seq").get<int>();
      s.ffn = sh.at("ffn").get<int>();
      const std::string kind = sh.value("kind", std::string("encoder"));
      // "window": Swin-style windowed self-attention -- the sample's seq tokens are stored
      // window-major (window w holds tokens [w*win, (w+1)*win)) and attention runs inside
      // each window; everything else is the encoder layer.
      if (kind == "encoder" || kind == "causal" || kind == "decoder") {
        s.win = s.seq;
        s.causal = kind != "encoder";
        s.cross = kind == "decoder";
      } else if (kind == "window") {
        s.win = sh.value("window", 49);
        if (s.win <= 0 || s.seq % s.win != 0) {
          *err = "executor: window layer needs seq to be a multiple of window";
          return kErrConfig;
        }
      } else {
        *err = "executor: layer kind '" + kind + "' not supported (encoder, causal, decoder, window)";
        return kErrConfig;
      }
      if (kind == "window" && sh.value("shift", false)) {  // SW-MSA (Swin's odd blocks)
        const int g = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.seq))));
        const int ws = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.win))));
        if (g * g != s.seq || ws * ws != s.win || g % ws != 0) {
          *err = "executor: shifted windows need a square token grid tiled by square windows";
          return kErrConfig;
        }
        s.shift = g > ws ? ws / 2 : 0;  // one window covers the grid: Swin skips the shift
      }
      s.rpb = kind == "window" && sh.value("rel_pos", false);
      {
        const std::string norm = sh.value("norm", std::string("layer"));
        if (norm != "layer" && norm != "rms") {
          *err = "executor: shape norm must be \"layer\" or \"rms\"";
          return kErrConfig;
        }
        s.rms = norm == "rms";
      }
      s.relb = sh.value("rel_bias", 0);
      if (s.relb < 0 || s.relb > 127 || (s.relb > 0 && (kind == "window" || s.hd > 64))) {
        *err = "executor: rel_bias (T5 buckets, 1..127) needs a full-attention layer with "
               "head_dim <= 64";
        return kErrConfig;
      }
      s.merge = sh.value("merge", false);
      if (s.merge) {
        const int g = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.seq))));
        const int ws = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.win))));
        if (kind != "window" || g * g != s.seq || ws * ws != s.win || g % ws != 0 ||
            (s.h / 2) % 8 != 0 || s.h % 2 != 0) {
          *err = "executor: patch merging needs a window layer with a square token grid tiled by "
                 "square windows and hidden/2 a multiple of 8";
          return kErrConfig;
        }
        if (l == 0) {
          *err = "executor: the first layer cannot merge patches (its input is the model input)";
          return kErrConfig;
        }
      }
      if (s.hd * s.heads != s.h) {
        *err = "executor: heads * head_dim must equal hidden";
        return kErrConfig;
      }
      shape_[l] = s;
    }
    for (const json& st : plan_.at("stages")) {
      const int b = st.at("layer_range")[0].get<int>(), e = st.at("layer_range")[1].get<int>();
      stage_range_.push_back({b, e});
      for (const json& jl : st.at("layers")) {
        const int id = jl.at("id").get<int>();
        const auto hs = parplan::StrategyFromString(jl.at("strategy").get<std::string>());
        const auto dd = hs.DimDegrees();
        if (hs.group_size != g_) {
          *err = "executor: strategy group size does not match world_size / pp_degree";
          return kErrConfig;
        }
        deg_[id] = Deg{dd.dp, dd.sdp, dd.tp};
      }
    }
    if (static_cast<int>(stage_range_.size()) != P_) {
      *err = "executor: plan stage count != pp_degree";
      return kErrConfig;
    }
    for (int l = 0; l < L_; ++l) {
      const Shape& s = shape_[l];
      const Deg& d = deg_[l];
      if (s.heads % d.tp || s.ffn % d.tp || s.h % d.tp) {
        *err = "executor: tp degree must divide heads, hidden and ffn";
        return kErrConfig;
      }
      if ((s.h / d.tp) % 8 || (s.ffn / d.tp) % 8) {
        *err = "executor: hidden/tp and ffn/tp must be multiples of 8";
        return kErrConfig;
      }
      // d.data() > Bm_ is allowed: GPipe splits each micro-batch over the data replicas, so
      // with the planner's 1-sample micro-batches (A14, planner.cc:343-349) some replicas
      // idle for a micro-batch; their gradients enter the reductions as zeros.
      if (s.cross) {  // T5 decoder layers (SPEC.md:67 flattens encoder + decoder)
        if (dec0_ < 0) dec0_ = l;
        const Shape& s0 = shape_[dec0_];
        // the memory (the first decoder layer's input) travels with the activations across
        // the decoder's stage boundaries, chunked like them: one data degree and shape
        if (d.data() != deg_[dec0_].data() || s.h != s0.h || s.seq != s0.seq) {
          *err = "executor: decoder layers must share one data degree and shape (the memory "
                 "is the first decoder layer's input)";
          return kErrConfig;
        }
      } else if (dec0_ >= 0) {
        *err = "executor: decoder layers must be the model's last layers";
        return kErrConfig;
      }
      if (l > 0 && (s.in_h() != shape_[l - 1].h || s.in_seq() != shape_[l - 1].seq)) {
        *err = "executor: layer " + std::to_string(l) +
               " input shape differs from the previous layer's output (only patch merging, "
               "\"merge\": true, changes hidden and tokens between layers)";
        return kErrConfig;
      }
    }
    inv_count_ = 1.0f / (static_cast<float>(B_) * shape_.back().seq * shape_.back().h);

    std::vector<int> local;
    if (cfg.contains("local_ranks")) {
      local = cfg.at("local_ranks").get<std::vector<int>>();
    } else {
      for (int r = 0; r < world_; ++r) local.push_back(r);
    }
    if (sim_) {
      comm_ = make_sim_comm(world_);
    } else if (comm_kind == "null") {
      // per-GPU proxy: one rank's share of a world_-rank plan on this device, every
      // collective / transfer a no-op (timing of the rank's compute only; values are junk)
      if (local.size() != 1) {
        *err = "executor: null comm drives exactly one local rank";
        return kErrConfig;
      }
      comm_ = make_null_comm(world_);
    } else {
      if (local.size() != 1) {
        *err = "executor: nccl mode drives exactly one local rank";
        return kErrConfig;
      }
      std::string hex = cfg.at("nccl_id_hex").get<std::string>();
      std::string id(hex.size() / 2, '\0');
      for (size_t i = 0; i < id.size(); ++i)
        id[i] = static_cast<char>(std::stoi(hex.substr(2 * i, 2), nullptr, 16));
      NcclOptions no;
      no.min_ctas = cfg.value("nccl_min_ctas", no.min_ctas);
      no.max_ctas = cfg.value("nccl_max_ctas", no.max_ctas);
      no.timeout_ms = cfg.value("nccl_timeout_ms", no.timeout_ms);
      comm_ = make_nccl_comm(world_, local[0], id, no, err);
      if (!comm_) return kErrNccl;
    }
    if (dry_run_) {
      for (int r : local) {
        auto rc = std::make_unique<RankCtx>();
        rc->rank = r;
        rc->stage = r / g_;
        rc->idx = r % g_;
        ranks_.push_back(std::move(rc));
      }
      const int rc = build_groups();
      if (rc != kOk) *err = gx_last_error();
      return rc;
    }
    if (cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&join_event_, cudaEventDisableTiming) != cudaSuccess) {
      *err = "executor: side stream creation failed";
      return kErrCuda;
    }
    // the data-gradient chain gets the highest priority, the wgrad stream the next
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, hi_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&wg_, cudaStreamNonBlocking,
                                     hi_prio < lo_prio ? hi_prio + 1 : lo_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&cs_, cudaStreamNonBlocking,
                                     hi_prio < lo_prio ? hi_prio + 1 : lo_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&pp_, cudaStreamNonBlocking, hi_prio) != cudaSuccess) {
      *err = "executor: cudaStreamCreate failed";
      return kErrCuda;
    }
    ls_ = stream_;
    for (int r : local) {
      auto rc = std::make_unique<RankCtx>();
      rc->rank = r;
      rc->stage = r / g_;
      rc->idx = r % g_;
      ranks_.push_back(std::move(rc));
    }
  } catch (const std::exception& e) {
    *err = std::string("executor config: ") + e.what();
    return kErrConfig;
  }
  int rc = build_groups();
  if (rc != kOk) {
    *err = gx_last_error();
    return rc;
  }
  for (auto& r : ranks_) {
    rc = allocate(*r);
    if (rc != kOk) {
      *err = gx_last_error();
      return rc;
    }
  }
  return kOk;
}

int ExecutorImpl::build_groups() {
  // Identical registration order on every process (NCCL splits are world collectives).
  for (int s = 0; s < P_; ++s) {
    const int base = s * g_;
    for (int l = stage_range_[s].first; l < stage_range_[s].second; ++l) {
      const Deg& d = deg_[l];
      for (int i = 0; i < g_; ++i) {
        const int tr = i % d.tp, dr = i / d.tp, sr = dr % d.sdp, pr = dr / d.sdp;
        std::vector<int> tp, sdp, dp;
        for (int j = 0; j < d.tp; ++j) tp.push_back(base + dr * d.tp + j);
        for (int j = 0; j < d.sdp; ++j) sdp.push_back(base + (pr * d.sdp + j) * d.tp + tr);
        for (int j = 0; j < d.dp; ++j) dp.push_back(base + (j * d.sdp + sr) * d.tp + tr);
        const int gtp = d.tp > 1 ? comm_->add_group(tp) : -1;
        const int gsdp = d.sdp > 1 ? comm_->add_group(sdp) : -1;
        const int gdp = d.dp > 1 ? comm_->add_group(dp) : -1;
        int gx = -1;
        Xin xin = Xin::kStageInput;
        if (l > stage_range_[s].first) {
          const Deg& p = deg_[l - 1];
          if (p.data() == d.data()) {
            xin = Xin::kSame;
          } else if (d.data() > p.data()) {
            // slice forward; backward all-gathers dY over the k sub-chunks of the prev chunk
            xin = Xin::kSlice;
            const int c = i / p.tp, k = p.tp / d.tp;
            std::vector<int> mem;
            for (int r = 0; r < k; ++r) mem.push_back(base + c * p.tp + r * d.tp + i % d.tp);
            gx = comm_->add_group(mem);
          } else {
            xin = Xin::kGather;
            const int j = i / d.tp, k = d.tp / p.tp;
            std::vector<int> mem;
            for (int r = 0; r < k; ++r) mem.push_back(base + j * d.tp + r * p.tp + i % p.tp);
            gx = comm_->add_group(mem);
          }
        }
        for (auto& rc : ranks_) {
          if (rc->rank != base + i) continue;
          RankLayer L;
          L.layer = l;
          L.sh = shape_[l];
          L.d = d;
          L.tr = tr;
          L.dr = dr;
          L.sr = sr;
          L.pr = pr;
          L.g_tp = gtp;
          L.g_sdp = gsdp;
          L.g_dp = gdp;
          L.g_xin = gx;
          L.xin = xin;
          rc->layers.push_back(std::move(L));
        }
      }
    }
  }
  return comm_->finalize();
}

std::string ExecutorImpl::topology() const {
  json j;
  j["world_size"] = world_;
  j["pp_degree"] = P_;
  j["group_size"] = g_;
  j["micro_batches"] = m_;
  j["batch_size"] = B_;
  json ranks = json::array();
  auto members = [&](int gid) {
    return gid < 0 ? json(nullptr) : json(comm_->group(gid).ranks);
  };
  for (const auto& r : ranks_) {
    json jr;
    jr["rank"] = r->rank;
    jr["stage"] = r->stage;
    jr["idx"] = r->idx;
    json layers = json::array();
    for (const RankLayer& L : r->layers) {
      json jl;
      jl["layer"] = L.layer;
      jl["dp"] = L.d.dp;
      jl["sdp"] = L.d.sdp;
      jl["tp"] = L.d.tp;
      jl["tp_rank"] = L.tr;
      jl["data_rank"] = L.dr;
      jl["tp_group"] = members(L.g_tp);
      jl["sdp_group"] = members(L.g_sdp);
      jl["dp_group"] = members(L.g_dp);
      jl["relayout"] = L.xin == Xin::kSame ? "same" : L.xin == Xin::kSlice ? "slice"
                       : L.xin == Xin::kGather ? "gather" : "stage_input";
      jl["relayout_group"] = members(L.g_xin);
      json ch = json::array();
      for (int mb = 0; mb < m_; ++mb) {
        int64_t lo, hi;
        chunk(L.d, r->idx, mb, lo, hi);
        ch.push_back({lo, hi});
      }
      jl["chunks"] = ch;
      layers.push_back(jl);
    }
    jr["layers"] = layers;
    json pp = json::array();
    for (int mb = 0; mb < m_; ++mb) {
      for (int kind = 0; kind < 4; ++kind) {
        const bool exists = (kind == 0 && r->stage + 1 < P_) || (kind == 1 && r->stage > 0) ||
                            (kind == 2 && r->stage > 0) || (kind == 3 && r->stage + 1 < P_);
        if (!exists) continue;
        for (const Xfer& x : pp_plan(r->stage, r->idx, mb, kind))
          pp.push_back({{"mb", mb}, {"kind", kind}, {"peer", x.peer}, {"lo", x.lo}, {"hi", x.hi}});
      }
    }
    jr["pp"] = pp;
    ranks.push_back(jr);
  }
  j["ranks"] = ranks;
  j["groups"] = json::array();
  for (int g = 0; g < comm_->num_groups(); ++g) j["groups"].push_back(comm_->group(g).ranks);
  return j.dump();
}

std::string ExecutorImpl::info() const {
  json j;
  j["world_size"] = world_;
  j["pp_degree"] = P_;
  j["micro_batches"] = m_;
  j["batch_size"] = B_;
  j["comm"] = comm_kind_;
  j["launches_per_step"] = launches_per_step_;
  j["steps_run"] = steps_run_;
  json ranks = json::array();
  for (const auto& r : ranks_) {
    json jr;
    jr["rank"] = r->rank;
    jr["stage"] = r->stage;
    jr["device_bytes"] = r->arena.bytes();
    jr["memory_cap_bytes"] = r->arena.cap();
    int64_t in_rows = 0, tgt_rows = 0;  // rows of this rank's host batch slice (load_batch)
    for (int mb = 0; mb < m_; ++mb) {
      if (r->stage == 0) in_rows += r->layers.front().acts[mb].samples * r->layers.front().sh.in_seq();
      if (r->stage == P_ - 1) tgt_rows += r->layers.back().acts[mb].rows;
    }
    jr["input_rows"] = in_rows;
    jr["target_rows"] = tgt_rows;
    // the planner's per-device estimate for this rank's stage (EstimateMemory, A7)
    if (plan_.contains("stages") && r->stage < static_cast<int>(plan_["stages"].size()))
      jr["plan_estimate_bytes"] = plan_["stages"][r->stage].value("peak_memory_bytes", int64_t{0});
    int64_t params = 0, opt = 0, grads = 0;
    for (const RankLayer& L : r->layers) {
      params += L.shard_n * 4 + L.lay.total * 2;
      opt += 2 * L.shard_n * 4;
      grads += L.lay.total * 4 + (L.d.sdp > 1 ? L.shard_n * 4 : 0);
    }
    jr["param_bytes"] = params;
    jr["optimizer_bytes"] = opt;
    jr["grad_bytes"] = grads;
    ranks.push_back(jr);
  }
  j["ranks"] = ranks;
  return j.dump();
}

}  // namespace xi

std::unique_ptr<Executor> create_executor(const std::string& config_json, std::string* err,
                                          int* code) {
  json cfg;
  try {
    cfg = json::parse(config_json);
  } catch (const std::exception& e) {
    *err = std::string("executor: bad config json: ") + e.what();
    if (code != nullptr) *code = kErrConfig;
    return nullptr;
  }
  auto ex = std::make_unique<xi::ExecutorImpl>();
  const int rc = ex->init(cfg, err);
  if (rc != kOk) {
    if (code != nullptr) *code = rc;
    return nullptr;
  }
  return ex;
}

}  // namespace gx
