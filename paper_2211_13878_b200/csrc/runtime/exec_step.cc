// exec_step.cc -- the training step: GPipe schedule over the local ranks, stream forks / joins,
// CUDA-graph capture and replay, device timing, the profile report, sync and loss
#include "executor_impl.h"

namespace gx {
namespace xi {

// ------------------------------------------------------------------------- the step
int ExecutorImpl::step_once() {
  fork_used_ = 0;
  tr_used_ = 0;
  tmark("step_begin", stream_);
  side_used_ = false;
  wg_used_ = false;
  cs_used_ = false;
  pp_used_ = false;
  wg_active_ = wgrad_stream_ && !profiling_;
  ls_ = stream_;
  for (auto& r : ranks_) r->wg_pending[0] = r->wg_pending[1] = false;
  auto in_stage = [&](int st) {
    std::vector<RankCtx*> v;
    for (auto& r : ranks_)
      if (r->stage == st) v.push_back(r.get());
    return v;
  };
  for (auto& r : ranks_) {
    for (RankLayer& L : r->layers)
      for (Acts& a : L.acts) a.ln1_ready = false;
    GX_TRY(bump_step(r->step, nullptr, stream_));
    GX_TRY(cuda_check(cudaMemsetAsync(r->loss, 0, 4, stream_), "memset loss"));
    for (RankLayer& L : r->layers)
      GX_TRY(cuda_check(cudaMemsetAsync(L.gfull, 0, grad_zero_bytes(*r, L), stream_), "memset grads"));
  }
  // ---------------------------------------------------------------- forward (GPipe)
  for (int mb = 0; mb < m_; ++mb) {
    for (int st = 0; st < P_; ++st) {
      auto R = in_stage(st);
      if (R.empty()) continue;
      if (st > 0) GX_TRY(pp_exchange(R, mb, true, false));
      const int nl = static_cast<int>(R[0]->layers.size());
      for (int li = 0; li < nl; ++li) {
        for (RankCtx* r : R) GX_TRY(xin_fwd(*r, li, mb));
        if (mb == 0) {
          // SDP parameters: gathered on stream_ for the stage's first layer, prefetched on
          // cs_ one layer ahead for the rest (the all-gather overlaps the previous layer)
          const bool pre = li > 0 && prefetched_;
          for (RankCtx* r : R) {
            if (r->layers[li].d.sdp <= 1) continue;
            if (pre)
              GX_TRY(cuda_check(cudaStreamWaitEvent(stream_, r->gath_ev[li], 0), "gather wait"));
            else
              GX_TRY(gather_params(*r, li, stream_));
          }
          prefetched_ = false;
          if (comm_on_cs() && li + 1 < nl && R[0]->layers[li + 1].d.sdp > 1) {
            GX_TRY(fork(stream_, cs_));
            cs_used_ = true;
            for (RankCtx* r : R) GX_TRY(gather_params(*r, li + 1, cs_));
            // recorded after every rank posted: a simulated collective runs at the last post
            for (RankCtx* r : R)
              GX_TRY(cuda_check(cudaEventRecord(r->gath_ev[li + 1], cs_), "gather done"));
            prefetched_ = true;
          }
        }
        const int phases = tp_phases(R[0]->layers[li]);
        for (int ph = 0; ph < phases; ++ph)
          for (RankCtx* r : R) GX_TRY(fwd_phase(*r, li, mb, ph));
      }
      if (st + 1 < P_) GX_TRY(pp_exchange(R, mb, true, true));
    }
  }
  tmark("fwd_end", stream_);
  // --------------------------------------------------------------- backward (GPipe)
  for (int mb = m_ - 1; mb >= 0 && !forward_only_; --mb) {
    for (int st = P_ - 1; st >= 0; --st) {
      auto R = in_stage(st);
      if (R.empty()) continue;
      for (RankCtx* r : R) {
        r->cur = 0;
        if (st == P_ - 1) {
          const RankLayer& Lz = r->layers.back();
          const Acts& a = Lz.acts[mb];
          const int64_t n = static_cast<int64_t>(a.rows) * Lz.sh.h;
          int64_t off = 0;
          for (int k = 0; k < mb; ++k) off += Lz.acts[k].rows;
          if (n > 0)
            GX_TRY(mse_loss(a.y, r->target + off * Lz.sh.h, r->gbuf[0], Lz.tr == 0 ? r->loss
                                                                                      : r->loss_dummy,
                            n, inv_count_, stream_, r->loss_ws));
        }
      }
      if (st + 1 < P_) GX_TRY(pp_exchange(R, mb, false, false));
      const int nl = static_cast<int>(R[0]->layers.size());
      for (int li = nl - 1; li >= 0; --li) {
        // SDP: the forward all-gather's copy stays resident through backward (B200 HBM
        // allows it), so the cost model's second gather (cost_model.cc:186-195) is elided.
        const int tp = R[0]->layers[li].d.tp;
        tmark("bwd_begin L" + std::to_string(R[0]->layers[li].layer), stream_);
        if (tp > 1) {
          for (int ph = 0; ph < tp_bwd_phases(R[0]->layers[li]); ++ph)
            for (RankCtx* r : R) GX_TRY(bwd_phase(*r, li, mb, ph));
        } else {
          for (RankCtx* r : R) GX_TRY(bwd_phase(*r, li, mb, 0));
        }
        if (mb == 0)
          for (int ph = 0; ph < 3; ++ph)
            for (RankCtx* r : R) GX_TRY(sync_phase(*r, li, ph));
        if (li > 0) {
          for (RankCtx* r : R) GX_TRY(xin_bwd(*r, li, mb));
          // the relayout leaves dY of layer li-1 in gbuf[cur] (kSame flips cur instead)
        } else {
          for (RankCtx* r : R) r->cur ^= 1;  // dX of the stage's first layer now in gbuf[cur]
        }
      }
      for (RankCtx* r : R) r->cur ^= 1;  // pp_bwd(send) / export read gbuf[cur ^ 1]
      if (st > 0) {
        GX_TRY(pp_exchange(R, mb, false, true));
      } else {
        for (RankCtx* r : R) {
          const RankLayer& F = r->layers.front();
          const Acts& a = F.acts[mb];
          if (a.rows > 0)
            GX_TRY(cuda_check(cudaMemcpyAsync(r->dx_out + r->in_row_off[mb] * F.sh.h,
                                              r->gbuf[r->cur ^ 1],
                                              static_cast<size_t>(a.rows) * F.sh.h * 2,
                                              cudaMemcpyDeviceToDevice, stream_),
                              "export dx"));
        }
      }
    }
  }
  tmark("bwd_chain_end", stream_);
  if (wg_used_) {  // join the wgrad stream
    GX_TRY(fork(wg_, stream_));
  }
  tmark("wgrad_joined", stream_);
  if (cs_used_) GX_TRY(fork(cs_, stream_));  // ... and the gradient-collective stream
  if (pp_used_) GX_TRY(fork(pp_, stream_));  // ... and the pipeline stream
  if (side_used_) {  // join the optimizer stream before the step completes
    GX_TRY(cuda_check(cudaEventRecord(join_event_, side_), "join record"));
    GX_TRY(cuda_check(cudaStreamWaitEvent(stream_, join_event_, 0), "join wait"));
  }
  tmark("step_end", stream_);
  for (auto& r : ranks_) GX_TRY(comm_->world_sum(r->rank, r->loss, stream_));
  // next step draws fresh dropout masks
  for (auto& r : ranks_) GX_TRY(bump_step(nullptr, r->seed_off, stream_));
  return kOk;
}

int ExecutorImpl::run2(bool use_graph, bool profile) {
  profiling_ = profile;
  ev_used_ = 0;
  recs_.clear();
  if (!use_graph) {
    const int64_t before = launch_count();
    const int rc = step_once();
    profiling_ = false;
    GX_TRY(rc);
    launches_per_step_ = launch_count() - before;
    ++steps_run_;
    return kOk;
  }
  cudaGraphExec_t& exec = profile ? pgraph_exec_ : graph_exec_;
  cudaGraph_t& graph = profile ? pgraph_ : graph_;
  if (exec == nullptr) {
    GX_TRY(cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal),
                      "begin capture"));
    capturing_ = true;
    const int64_t before = launch_count();
    const int rc = step_once();
    if (!profile) launches_per_step_ = launch_count() - before;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(stream_, &g);
    capturing_ = false;
    if (rc != kOk) {
      profiling_ = false;
      return rc;
    }
    GX_TRY(cuda_check(e, "end capture"));
    graph = g;
    // Node priorities (cudaGraphInstantiateFlagUseNodePriority) were measured slower: the
    // weight-gradient stream starves and the data-gradient chain then waits on its buffers.
    GX_TRY(cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate"));
    if (profile) prof_recs_ = recs_;
  }
  profiling_ = false;
  GX_TRY(cuda_check(cudaGraphLaunch(exec, stream_), "graph launch"));
  if (profile) recs_ = prof_recs_;
  ++steps_run_;
  return kOk;
}

std::string ExecutorImpl::profile_report() const {
  static const char* kNames[kNumCats] = {"gemm", "attention_fwd", "attention_bwd", "layernorm",
                                         "elementwise", "optimizer", "comm"};
  cudaStreamSynchronize(stream_);
  double ms[kNumCats] = {}, fl[kNumCats] = {}, by[kNumCats] = {};
  int64_t n[kNumCats] = {};
  json launches = json::array();
  static const char* kKinds[kNumCommKinds] = {"tp_all_reduce", "sdp_all_gather",
                                              "sdp_reduce_scatter", "dp_all_reduce",
                                              "relayout_all_gather", "pp_send_recv"};
  double kms[kNumCommKinds] = {}, kby[kNumCommKinds] = {}, kbus[kNumCommKinds] = {};
  int64_t kn[kNumCommKinds] = {};
  for (const Rec& r : recs_) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) continue;
    ms[r.cat] += t;
    fl[r.cat] += r.flops;
    by[r.cat] += r.bytes;
    n[r.cat] += 1;
    if (r.cat == kGemm) launches.push_back({t, r.flops});
    if (r.cat == kComm && r.kind >= 0) {
      kms[r.kind] += t;
      kby[r.kind] += r.bytes;
      kbus[r.kind] += r.bus;
      kn[r.kind] += 1;
    }
  }
  json j;
  double total = 0;
  for (int c = 0; c < kNumCats; ++c) {
    j["categories"][kNames[c]] = {{"ms", ms[c]}, {"launches", n[c]}, {"flops", fl[c]},
                                  {"bytes", by[c]}};
    total += ms[c];
  }
  float span = 0.f;
  if (!recs_.empty()) cudaEventElapsedTime(&span, recs_.front().a, recs_.back().b);
  j["sum_ms"] = total;
  j["span_ms"] = span;
  j["gemm_launches"] = launches;
  j["comm_kinds"] = json::object();
  for (int k = 0; k < kNumCommKinds; ++k)
    if (kn[k] > 0)
      j["comm_kinds"][kKinds[k]] = {{"ms", kms[k]}, {"bytes", kby[k]}, {"bus_bytes", kbus[k]},
                                    {"launches", kn[k]}};
  if (trace_ && tr_used_ > 0) {
    cudaDeviceSynchronize();
    json tl = json::array();
    for (size_t i = 0; i < tr_used_; ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, tr_[0].second, tr_[i].second);
      tl.push_back({tr_[i].first, t});
    }
    j["trace"] = tl;
  }
  return j.dump();
}

// Waits for the executor stream like cudaStreamSynchronize, but polls the communicators'
// asynchronous errors meanwhile and gives up after timeout_ms: a dead or hung peer aborts the
// communicators (NCCL kernels blocked on it return) and surfaces as GX_ERR_NCCL instead of a
// hang (SURVEY.md §5 failure detection).
int ExecutorImpl::sync(int64_t timeout_ms) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(stream_);
    if (e == cudaSuccess) return kOk;
    if (e != cudaErrorNotReady) return cuda_check(e, "executor sync");
    if (comm_ != nullptr) {
      const int rc = comm_->poll_async();
      if (rc != kOk) {
        comm_->abort();
        return rc;
      }
    }
    if (timeout_ms > 0 &&
        std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms)) {
      if (comm_ != nullptr) comm_->abort();
      return set_error(kErrNccl, ("executor: step did not complete within " +
                                  std::to_string(timeout_ms) + " ms (communicators aborted)").c_str());
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

int ExecutorImpl::loss(float* out) {
  float v = 0.f;
  GX_TRY(cuda_check(cudaMemcpyAsync(&v, ranks_.front()->loss, 4, cudaMemcpyDeviceToHost, stream_),
                    "loss d2h"));
  GX_TRY(sync(sync_timeout_ms_));
  *out = v;
  return kOk;
}

}  // namespace xi
}  // namespace gx
