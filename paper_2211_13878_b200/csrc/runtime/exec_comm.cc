// exec_comm.cc -- gradient collectives (DP all-reduce, SDP reduce-scatter) and the optimizer,
// SDP parameter gathers, strategy-transition relayouts (Slice / Gather), pipeline transfers
#include "executor_impl.h"

namespace gx {
namespace xi {

// Gradient synchronisation + optimizer after the layer's last backward micro-batch.
int ExecutorImpl::sync_phase(RankCtx& r, int li, int phase) {
  RankLayer& L = r.layers[li];
  const int par = li & 1;
  const bool syncs = L.d.sdp > 1 || L.d.dp > 1;
  if (synced_on_cs_.size() < r.layers.size()) synced_on_cs_.assign(r.layers.size(), 0);
  cudaStream_t cst = syncs && comm_on_cs() ? cs_ : stream_;
  if (phase == 0) {
    if (syncs && cst == cs_) {  // after everything the gradients came from on stream_ ...
      GX_TRY(fork(stream_, cs_));
      cs_used_ = true;
    }
    synced_on_cs_[li] = cst == cs_;
    // ... and on the wgrad stream
    if (wg_active_ && syncs)
      GX_TRY(cuda_check(cudaStreamWaitEvent(cst, r.wg_done[par], 0), "wgrad join"));
    if (L.d.sdp > 1)
      return c_reduce_scatter(kSdpReduceScatter, L.g_sdp, r.rank, L.gfull, L.gshard,
                                   static_cast<size_t>(L.shard_n), DType::kF32, cst);
    if (L.d.dp > 1)
      return c_all_reduce(kDpAllReduce, L.g_dp, r.rank, L.gfull, static_cast<size_t>(L.lay.total),
                               DType::kF32, cst);
    return kOk;
  }
  if (phase == 1) {
    if (L.d.sdp > 1 && L.d.dp > 1)
      return c_all_reduce(kDpAllReduce, L.g_dp, r.rank, L.gshard, static_cast<size_t>(L.shard_n),
                               DType::kF32, cst);
    return kOk;
  }
  const bool on_cs = synced_on_cs_[li] != 0;
  if (phase == 2 && optimizer_) {
    if (profiling_) {  // instrumented runs keep everything on one stream
      if (on_cs) GX_TRY(fork(cs_, stream_));
      return timed(kOptim, 0, 30.0 * L.shard_n, [&] {
        return adamw_dev(L.master, L.gshard, L.m, L.v, L.pshard, L.shard_n, lr_, b1_, b2_, eps_,
                         wd_, r.step, stream_);
      });
    }
    // side stream, after this layer's data-gradient chain, its weight gradients and their
    // collectives
    GX_TRY(fork(stream_, side_));
    if (wg_active_)
      GX_TRY(cuda_check(cudaStreamWaitEvent(side_, r.wg_done[par], 0), "fork wait wgrad"));
    if (on_cs) GX_TRY(fork(cs_, side_));
    side_used_ = true;
    tmark("opt_begin L" + std::to_string(L.layer), side_);
    GX_TRY(adamw_dev(L.master, L.gshard, L.m, L.v, L.pshard, L.shard_n, lr_, b1_, b2_, eps_, wd_,
                     r.step, side_, 2 * num_sms()));
    tmark("opt_end L" + std::to_string(L.layer), side_);
  }
  return kOk;
}

int ExecutorImpl::gather_params(RankCtx& r, int li, cudaStream_t st) {
  RankLayer& L = r.layers[li];
  if (L.d.sdp <= 1) return kOk;
  std::vector<size_t> counts(L.d.sdp, static_cast<size_t>(L.shard_n));
  return c_all_gather(kSdpAllGather, L.g_sdp, r.rank, L.pshard, L.pfull, counts, DType::kBF16, st);
}

// Forward relayout into layer li (same stage): only the all-gather case moves data.
int ExecutorImpl::xin_fwd(RankCtx& r, int li, int mb) {
  RankLayer& L = r.layers[li];
  if (L.xin != Xin::kGather) return kOk;
  const RankLayer& Pv = r.layers[li - 1];
  const Acts& p = Pv.acts[mb];
  const CommGroup& grp = comm_->group(L.g_xin);
  std::vector<size_t> counts;
  for (int member : grp.ranks) {
    int64_t lo, hi;
    chunk(Pv.d, member % g_, mb, lo, hi);
    counts.push_back(static_cast<size_t>((hi - lo) * L.sh.in_seq() * L.sh.in_h()));
  }
  return c_all_gather(kRelayout, L.g_xin, r.rank, p.y, L.acts[mb].in(), counts, DType::kBF16, stream_);
}

// Backward relayout out of layer li: dX (gbuf[cur^1], layout li) -> dY of layer li-1 in
// gbuf[cur] after the call.
int ExecutorImpl::xin_bwd(RankCtx& r, int li, int mb) {
  RankLayer& L = r.layers[li];
  const RankLayer& Pv = r.layers[li - 1];
  bf16* dX = r.gbuf[r.cur ^ 1];
  bf16* dYp = r.gbuf[r.cur];
  const int64_t h = L.sh.in_h(), seq = L.sh.in_seq();  // the relayout moves layer li's input
  if (L.xin == Xin::kSame) {
    r.cur ^= 1;
    return kOk;
  }
  if (L.xin == Xin::kGather) {
    // forward gathered k chunks; backward keeps this rank's own sub-chunk
    const Acts& a = L.acts[mb];
    const Acts& p = Pv.acts[mb];
    const int64_t off = (p.sample0 - a.sample0) * seq * h;
    if (p.rows == 0) return kOk;
    return cuda_check(cudaMemcpyAsync(dYp, dX + off, static_cast<size_t>(p.rows) * h * 2,
                                      cudaMemcpyDeviceToDevice, stream_),
                      "xin_bwd slice");
  }
  // forward sliced; backward all-gathers the sub-chunk gradients of the previous chunk
  const CommGroup& grp = comm_->group(L.g_xin);
  std::vector<size_t> counts;
  for (int member : grp.ranks) {
    int64_t lo, hi;
    chunk(L.d, member % g_, mb, lo, hi);
    counts.push_back(static_cast<size_t>((hi - lo) * seq * h));
  }
  return c_all_gather(kRelayout, L.g_xin, r.rank, dX, dYp, counts, DType::kBF16, stream_);
}

// Pipeline-boundary transfer lists (pure functions of the plan, shared by the executor and
// the dry-run topology export).  kind 0: forward send (this stage's last layer output to the
// next stage), 1: forward receive, 2: backward send (first layer's input gradient to the
// previous stage), 3: backward receive.  Each entry is (peer global rank, sample range); a
// sender is paired with the receiver of equal tp-residue so every receiver gets each
// overlapping sample range exactly once.
std::vector<ExecutorImpl::Xfer> ExecutorImpl::pp_plan(int stage, int idx, int mb, int kind) const {
  std::vector<Xfer> out;
  const bool fwd = kind < 2;
  const bool send = kind == 0 || kind == 2;
  // (my layer, other stage, other layer) for this boundary
  const int other = fwd ? (send ? stage + 1 : stage - 1) : (send ? stage - 1 : stage + 1);
  const int my_layer = (fwd == send) ? stage_range_[stage].second - 1 : stage_range_[stage].first;
  const int ot_layer = (fwd == send) ? stage_range_[other].first : stage_range_[other].second - 1;
  const Deg& me = deg_[my_layer];
  const Deg& ot = deg_[ot_layer];
  int64_t mlo, mhi;
  chunk(me, idx, mb, mlo, mhi);
  if (send) {
    for (int j = 0; j < g_; ++j) {
      if (j % me.tp != idx % me.tp) continue;
      int64_t lo2, hi2;
      chunk(ot, j, mb, lo2, hi2);
      const int64_t lo = std::max(mlo, lo2), hi = std::min(mhi, hi2);
      if (hi > lo) out.push_back(Xfer{other * g_ + j, lo, hi});
    }
  } else {
    for (int c = 0; c < ot.data(); ++c) {
      int64_t lo1, hi1;
      chunk(ot, c * ot.tp, mb, lo1, hi1);
      const int64_t lo = std::max(mlo, lo1), hi = std::min(mhi, hi1);
      if (hi > lo) out.push_back(Xfer{other * g_ + c * ot.tp + idx % ot.tp, lo, hi});
    }
  }
  return out;
}

// Forward boundary: send this stage's last layer output / receive the first layer input.
int ExecutorImpl::pp_fwd(RankCtx& r, int mb, bool send, cudaStream_t st) {
  const RankLayer& L = send ? r.layers.back() : r.layers.front();
  const Acts& my = L.acts[mb];
  const int64_t hs = send ? static_cast<int64_t>(L.sh.seq) * L.sh.h
                          : static_cast<int64_t>(L.sh.in_seq()) * L.sh.in_h();
  for (const Xfer& x : pp_plan(r.stage, r.idx, mb, send ? 0 : 1)) {
    const size_t bytes = static_cast<size_t>((x.hi - x.lo) * hs) * 2;
    const int64_t off = (x.lo - my.sample0) * hs;
    if (send) {
      GX_TRY(comm_->send(r.rank, x.peer, my.y + off, bytes, st));
    } else {
      GX_TRY(comm_->recv(r.rank, x.peer, my.in() + off, bytes, st));
    }
    // decoder stages: the memory follows, same rows (decoders share data degree and shape)
    if (send && dec0_ >= 0 && r.stage >= stage_of_layer(dec0_))
      GX_TRY(comm_->send(r.rank, x.peer, r.mem(mb) + off, bytes, st));
    if (!send && !r.mem_in.empty())
      GX_TRY(comm_->recv(r.rank, x.peer, r.mem_in[mb] + off, bytes, st));
  }
  return kOk;
}

// Backward boundary: send the first layer's input gradient (gbuf[cur ^ 1]) / receive the
// last layer's output gradient into gbuf[cur].
int ExecutorImpl::pp_bwd(RankCtx& r, int mb, bool send, cudaStream_t st) {
  const RankLayer& L = send ? r.layers.front() : r.layers.back();
  const Acts& my = L.acts[mb];
  const int64_t hs = send ? static_cast<int64_t>(L.sh.in_seq()) * L.sh.in_h()
                          : static_cast<int64_t>(L.sh.seq) * L.sh.h;
  bf16* dx_src = nullptr;
  float* dmem_src = nullptr;
  if (send) {  // private per-micro-batch copies (stream_), read by the send on `st`
    int64_t off_in = 0, off_rows = 0;
    for (int k = 0; k < mb; ++k) {
      off_in += static_cast<int64_t>(L.acts[k].samples) * hs;
      off_rows += L.acts[k].rows;
    }
    dx_src = r.pp_dx_send + off_in;
    if (my.samples > 0)
      GX_TRY(cuda_check(cudaMemcpyAsync(dx_src, r.gbuf[r.cur ^ 1], static_cast<size_t>(my.samples) * hs * 2,
                                        cudaMemcpyDeviceToDevice, stream_), "pp dx copy"));
    if (!r.mem_in.empty()) {
      dmem_src = r.pp_dmem_send + off_rows * L.sh.h;
      if (my.rows > 0)
        GX_TRY(cuda_check(cudaMemcpyAsync(dmem_src, r.dmem, static_cast<size_t>(my.rows) * L.sh.h * 4,
                                          cudaMemcpyDeviceToDevice, stream_), "pp dmem copy"));
    }
  }
  for (const Xfer& x : pp_plan(r.stage, r.idx, mb, send ? 2 : 3)) {
    const size_t bytes = static_cast<size_t>((x.hi - x.lo) * hs) * 2;
    const int64_t off = (x.lo - my.sample0) * hs;
    if (send) {
      GX_TRY(comm_->send(r.rank, x.peer, dx_src + off, bytes, st));
    } else {
      GX_TRY(comm_->recv(r.rank, x.peer, r.gbuf[r.cur] + off, bytes, st));
    }
    // decoder stages: dL/dmemory summed over this stage's decoder layers goes back (fp32)
    if (send && dmem_src != nullptr)
      GX_TRY(comm_->send(r.rank, x.peer, dmem_src + off, bytes * 2, st));
    if (!send && r.dmem_from_next)
      GX_TRY(comm_->recv(r.rank, x.peer, r.dmem + off, bytes * 2, st));
  }
  return kOk;
}

}  // namespace xi
}  // namespace gx
