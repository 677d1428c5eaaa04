// exec_memory.cc -- device buffers of every local rank (arena with the plan's memory cap), parameters
// in and out in the canonical order, batches, and the exported outputs
#include "executor_impl.h"

namespace gx {
namespace xi {

int ExecutorImpl::allocate(RankCtx& r) {
  Arena& A = r.arena;
  A.set_cap(static_cast<size_t>(mem_cap_));
  int64_t max_rows = 0, max_h = 0, max_f = 0, max_q = 0, max_c = 0, max_lse = 0, max_m = 0,
          max_x = 0;
  bool any_shift = false;
  int64_t max_rpb = 0, max_relb = 0;
  for (size_t li = 0; li < r.layers.size(); ++li) {
    RankLayer& L = r.layers[li];
    const Shape& s = L.sh;
    const int t = L.d.tp;
    L.lay = make_layout(s, t, L.d.sdp);
    L.shard_n = L.lay.total / L.d.sdp;
    L.master = A.a<float>(L.shard_n);
    L.m = A.a<float>(L.shard_n);
    L.v = A.a<float>(L.shard_n);
    L.gfull = A.a<float>(L.lay.total);
    L.gshard = L.d.sdp > 1 ? A.a<float>(L.shard_n) : L.gfull;
    L.pshard = A.a<bf16>(L.shard_n);
    L.pfull = L.d.sdp > 1 ? A.a<bf16>(L.lay.total) : L.pshard;
    if (L.m != nullptr) cudaMemset(L.m, 0, L.shard_n * 4);
    if (L.v != nullptr) cudaMemset(L.v, 0, L.shard_n * 4);
    L.acts.resize(m_);
    for (int mb = 0; mb < m_; ++mb) {
      Acts& a = L.acts[mb];
      int64_t lo, hi;
      chunk(L.d, r.idx, mb, lo, hi);
      a.sample0 = lo;
      a.samples = static_cast<int>(hi - lo);
      a.rows = a.samples * s.seq;
      if (a.rows == 0) r.idle_chunks = true;
      const int64_t rows = a.rows;
      const int64_t h = s.h, ht = s.h / t, ft = s.ffn / t;
      const int64_t in_rows = static_cast<int64_t>(a.samples) * s.in_seq();
      // layer input: alias into the previous layer's output where the relayout allows
      bf16* xin = nullptr;
      if (L.xin == Xin::kSame) {
        xin = r.layers[li - 1].acts[mb].y;
      } else if (L.xin == Xin::kSlice) {
        const Acts& p = r.layers[li - 1].acts[mb];
        xin = p.y + (a.sample0 - p.sample0) * s.in_seq() * s.in_h();
      } else {
        xin = A.a<bf16>(in_rows * s.in_h());
      }
      if (s.merge) {
        a.xm = xin;
        a.mg = A.a<bf16>(rows * 2 * h);
        a.mln = A.a<bf16>(rows * 2 * h);
        a.meanm = A.a<float>(rows);
        a.rstdm = A.a<float>(rows);
        a.x = A.a<bf16>(rows * h);
        max_m = std::max(max_m, rows * 2 * h);
      } else {
        a.x = xin;
      }
      max_h = std::max(max_h, in_rows * s.in_h());  // gbuf also carries the input gradient
      a.ln1 = A.a<bf16>(rows * h);
      a.qkv = A.a<bf16>(rows * 3 * ht);
      a.ctx = A.a<bf16>(rows * ht);
      a.x1 = A.a<bf16>(rows * h);
      a.ln2 = A.a<bf16>(rows * h);
      a.pre = A.a<bf16>(rows * ft);
      a.gel = A.a<bf16>(rows * ft);
      a.y = A.a<bf16>(rows * h);
      if (s.cross) {
        a.x2 = A.a<bf16>(rows * h);
        a.ln3 = A.a<bf16>(rows * h);
        a.qkv2 = A.a<bf16>(rows * 3 * ht);
        a.ctx2 = A.a<bf16>(rows * ht);
        a.lse2 = A.a<float>(static_cast<int64_t>(a.samples) * (s.heads / t) * s.seq);
        if (thr_attn_ != 0u)
          a.amask2 = A.a<uint16_t>(static_cast<int64_t>(a.samples) * (s.heads / t) * s.seq *
                                   ((s.seq + 63) / 64) * 4);
        a.mean3 = s.rms ? nullptr : A.a<float>(rows);  // (null mean: RMSNorm)
        a.rstd3 = A.a<float>(rows);
        max_x = std::max(max_x, rows * h);
      }
      if (s.rpb)
        max_rpb = std::max<int64_t>(max_rpb, static_cast<int64_t>(a.samples) * s.windows() *
                                                 (s.heads / t) * s.rpb_n());
      if (s.relb)
        max_relb = std::max<int64_t>(max_relb, static_cast<int64_t>(a.samples) * (s.heads / t) *
                                                   ((s.seq + 127) / 128) * (2 * s.seq - 1));
      if (s.shift > 0) {
        a.ln1r = A.a<bf16>(rows * h);
        a.ctxr = A.a<bf16>(rows * ht);
        any_shift = true;
      }
      a.lse = A.a<float>(static_cast<int64_t>(a.samples) * (s.heads / t) * s.seq);
      if (thr_attn_ != 0u)
        a.amask = A.a<uint16_t>(static_cast<int64_t>(a.samples) * (s.heads / t) * s.seq *
                                ((s.win + 63) / 64) * 4);
      a.mean1 = s.rms ? nullptr : A.a<float>(rows);  // (null mean: RMSNorm)
      a.rstd1 = A.a<float>(rows);
      a.mean2 = s.rms ? nullptr : A.a<float>(rows);
      a.rstd2 = A.a<float>(rows);
      max_rows = std::max(max_rows, rows);
      max_h = std::max(max_h, rows * h);
      max_f = std::max(max_f, rows * ft);
      max_q = std::max(max_q, rows * 3 * ht);
      max_c = std::max(max_c, rows * ht);
      max_lse = std::max(max_lse, static_cast<int64_t>(a.samples) * (s.heads / t) * s.seq);
    }
  }
  r.partial = A.a<bf16>(max_h);
  for (int p = 0; p < 2; ++p) {
    r.dzb[p] = A.a<bf16>(max_h);
    r.dpreb[p] = A.a<bf16>(max_f);
    r.doutb[p] = A.a<bf16>(max_h);
    r.dqkvb[p] = A.a<bf16>(max_q);
    r.lnfold[p][0] = A.a<float>(max_h);
    r.lnfold[p][1] = A.a<float>(max_h);
    if (cudaEventCreateWithFlags(&r.wg_done[p], cudaEventDisableTiming) != cudaSuccess)
      return set_error(kErrCuda, "executor: event creation failed");
  }
  r.dx1 = A.a<bf16>(max_h);
  r.dctx = A.a<bf16>(max_c);
  r.da = A.a<bf16>(max_h);
  r.gbuf[0] = A.a<bf16>(max_h);
  r.gbuf[1] = A.a<bf16>(max_h);
  // tcgen05 attention: one dQ partial per 128-key tile, columns padded to 4 rows (the slack
  // covers ceil(seq / 128) x round_up(seq, 4) <= 5 seq)
  r.dq_acc = A.a<float>(5 * max_c);
  if (any_shift) {
    r.dctxr = A.a<bf16>(max_c);
    r.rollbuf = A.a<bf16>(max_h);
  }
  if (max_rpb > 0) r.rpb_part = A.a<float>(max_rpb);
  if (max_relb > 0) r.relb_part = A.a<float>(max_relb);
  for (RankLayer& L : r.layers)
    if (L.sh.relb > 0) {
      const std::vector<int8_t> map = t5_bucket_map(L.sh.seq, !L.sh.causal, L.sh.relb);
      L.relb_map = A.a<int8_t>(static_cast<int64_t>(map.size()));
      if (L.relb_map != nullptr &&
          cudaMemcpy(L.relb_map, map.data(), map.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return set_error(kErrCuda, "executor: relb map upload failed");
    }
  if (max_x > 0) {
    int64_t hx = 0;
    for (const RankLayer& L : r.layers) hx = std::max<int64_t>(hx, L.sh.h);
    r.ln_ws_x = A.a<float>(layernorm_bwd_ws_floats(static_cast<int>(hx)));
    if (r.ln_ws_x != nullptr)
      cudaMemset(r.ln_ws_x, 0, layernorm_bwd_ws_floats(static_cast<int>(hx)) * sizeof(float));
    r.dout2 = A.a<bf16>(max_x);
    r.dqkv2 = A.a<bf16>(3 * max_x);
    r.dmem = A.a<float>(max_x);
    for (size_t i = 0; i < r.layers.size(); ++i)
      if (r.layers[i].layer == dec0_) r.dec_li = static_cast<int>(i);
    const int s0 = stage_of_layer(dec0_);
    r.dmem_from_next = r.stage >= s0 && r.stage + 1 < P_;
    if (r.stage > s0) {
      r.mem_in.resize(m_);
      for (int mb = 0; mb < m_; ++mb)
        r.mem_in[mb] = A.a<bf16>(static_cast<int64_t>(r.layers.front().acts[mb].rows) *
                                 r.layers.front().sh.h);
    }
  }
  r.acc32 = A.a<float>(static_cast<int64_t>(kMaxSplits) * max_h);
  {
    int64_t max_hdim = 0;
    for (const RankLayer& L : r.layers) max_hdim = std::max<int64_t>(max_hdim, L.sh.h);
    r.ln_ws = A.a<float>(layernorm_bwd_ws_floats(static_cast<int>(max_hdim)));
    if (max_m > 0) {
      r.ln_ws_m = A.a<float>(layernorm_bwd_ws_floats(static_cast<int>(2 * max_hdim)));
      if (r.ln_ws_m != nullptr)
        cudaMemset(r.ln_ws_m, 0, layernorm_bwd_ws_floats(static_cast<int>(2 * max_hdim)) * 4);
      r.dmg1 = A.a<bf16>(max_m);
      r.dmg2 = A.a<bf16>(max_m);
    }
    int64_t max_cols = 0;
    for (const RankLayer& L : r.layers)
      max_cols = std::max<int64_t>({max_cols, L.sh.h, L.sh.ffn / L.d.tp, 3 * L.sh.h / L.d.tp});
    for (float*& w : r.cs_ws) {
      w = A.a<float>(colsum_ws_floats(static_cast<int>(max_cols)));
      if (w != nullptr)
        cudaMemset(w, 0, colsum_ws_floats(static_cast<int>(max_cols)) * sizeof(float));
    }
    if (r.ln_ws != nullptr)
      cudaMemset(r.ln_ws, 0, layernorm_bwd_ws_floats(static_cast<int>(max_hdim)) * sizeof(float));
  }
  r.dsum = A.a<float>(max_lse);
  if (r.dsum != nullptr) cudaMemset(r.dsum, 0, max_lse * sizeof(float));  // attention tickets
  r.loss = A.a<float>(1);
  r.loss_dummy = A.a<float>(1);
  r.loss_ws = A.a<float>(kLossBlocks + 1);
  if (r.loss_ws != nullptr) cudaMemset(r.loss_ws, 0, (kLossBlocks + 1) * sizeof(float));
  r.step = A.a<int64_t>(1);
  r.gath_ev.resize(r.layers.size(), nullptr);
  for (auto& e : r.gath_ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return set_error(kErrCuda, "executor: event creation failed");
  r.seed_off = A.a<uint64_t>(1);
  if (r.step != nullptr) cudaMemset(r.step, 0, 8);
  if (r.seed_off != nullptr) cudaMemset(r.seed_off, 0, 8);
  // stage input (first stage) / targets (last stage) for all micro-batches of this rank
  const RankLayer& first = r.layers.front();
  const RankLayer& last = r.layers.back();
  r.in_row_off.assign(m_, 0);
  int64_t tot = 0;
  for (int mb = 0; mb < m_; ++mb) {
    r.in_row_off[mb] = tot;
    tot += (r.stage == 0 ? first.acts[mb].rows : last.acts[mb].rows);
  }
  r.in_rows_total = tot;
  if (r.stage == 0) {
    int64_t rows_all = 0;
    for (int mb = 0; mb < m_; ++mb) rows_all += first.acts[mb].rows;
    r.x_in = A.a<bf16>(rows_all * first.sh.h);
    r.dx_out = A.a<bf16>(rows_all * first.sh.h);
    int64_t off = 0;
    for (int mb = 0; mb < m_; ++mb) {
      // first layer reads its input straight from the staged batch
      r.layers.front().acts[mb].x = r.x_in + off * first.sh.h;
      off += first.acts[mb].rows;
    }
  }
  if (r.stage == P_ - 1) {
    int64_t rows_all = 0;
    for (int mb = 0; mb < m_; ++mb) rows_all += last.acts[mb].rows;
    r.target = A.a<bf16>(rows_all * last.sh.h);
  }
  if (r.stage > 0) {
    int64_t in_all = 0, rows_all = 0;
    for (int mb = 0; mb < m_; ++mb) {
      in_all += static_cast<int64_t>(first.acts[mb].samples) * first.sh.in_seq() * first.sh.in_h();
      rows_all += first.acts[mb].rows;
    }
    r.pp_dx_send = A.a<bf16>(in_all);
    if (!r.mem_in.empty()) r.pp_dmem_send = A.a<float>(rows_all * first.sh.h);
  }
  if (A.failed()) (void)cudaGetLastError();  // no stale error for the next caller's checks
  if (A.over_cap())
    return set_error(kErrInfeasible, ("executor: rank " + std::to_string(r.rank) +
                                      " needs more than its memory cap of " +
                                      std::to_string(mem_cap_) + " bytes").c_str());
  if (A.failed()) return set_error(kErrCuda, "executor: out of device memory");
  return cuda_check(cudaDeviceSynchronize(), "executor allocate");
}

// ------------------------------------------------------------------------- parameters
int ExecutorImpl::set_layer_params(int layer, const float* canonical, int64_t n) {
  if (layer < 0 || layer >= L_) return set_error(kErrConfig, "set_layer_params: bad layer");
  if (n != canonical_size(shape_[layer])) return set_error(kErrConfig, "set_layer_params: size");
  for (auto& r : ranks_) {
    for (RankLayer& L : r->layers) {
      if (L.layer != layer) continue;
      std::vector<float> shard(L.shard_n, 0.f);
      const int64_t lo = static_cast<int64_t>(L.sr) * L.shard_n;
      for (int64_t j = 0; j < L.shard_n; ++j) {
        const int64_t c = canon_index(L.sh, L.lay, L.d.tp, L.tr, lo + j);
        if (c >= 0) shard[j] = canonical[c];
      }
      // Same stream as the cast below: a pageable cudaMemcpy may return before its DMA
      // lands, and stream_ does not synchronise with the legacy default stream.
      GX_TRY(cuda_check(cudaMemcpyAsync(L.master, shard.data(), L.shard_n * 4,
                                        cudaMemcpyHostToDevice, stream_),
                        "set_layer_params"));
      GX_TRY(cuda_check(cudaStreamSynchronize(stream_), "set_layer_params h2d"));
      GX_TRY(cast_bf16(L.master, L.pshard, L.shard_n, stream_));
      GX_TRY(cuda_check(cudaMemsetAsync(L.m, 0, L.shard_n * 4, stream_), "memset m"));
      GX_TRY(cuda_check(cudaMemsetAsync(L.v, 0, L.shard_n * 4, stream_), "memset v"));
      if (L.d.sdp > 1) {  // keep a gathered copy valid for inspection; fwd re-gathers
        GX_TRY(cuda_check(cudaMemsetAsync(L.pfull, 0, L.lay.total * 2, stream_), "memset"));
      }
    }
  }
  return cuda_check(cudaStreamSynchronize(stream_), "set_layer_params sync");
}

int ExecutorImpl::export_layer(int layer, int what, float* canonical, int64_t n) {
  if (layer < 0 || layer >= L_) return set_error(kErrConfig, "export_layer: bad layer");
  if (n != canonical_size(shape_[layer])) return set_error(kErrConfig, "export_layer: size");
  GX_TRY(cuda_check(cudaStreamSynchronize(stream_), "export sync"));
  for (int64_t i = 0; i < n; ++i) canonical[i] = std::nanf("");
  for (auto& r : ranks_) {
    for (RankLayer& L : r->layers) {
      if (L.layer != layer || L.pr != 0) continue;  // one DP replica holds every shard
      std::vector<float> shard(L.shard_n);
      if (what == 2) {  // bf16 compute copy of this rank's shard
        std::vector<uint16_t> b(L.shard_n);
        GX_TRY(cuda_check(cudaMemcpy(b.data(), L.pshard, L.shard_n * 2, cudaMemcpyDeviceToHost),
                          "export_layer"));
        for (int64_t j = 0; j < L.shard_n; ++j) {
          const uint32_t u = static_cast<uint32_t>(b[j]) << 16;
          std::memcpy(&shard[j], &u, 4);
        }
      } else {
        const float* src = what == 0 ? L.master : L.gshard;
        GX_TRY(cuda_check(cudaMemcpy(shard.data(), src, L.shard_n * 4, cudaMemcpyDeviceToHost),
                          "export_layer"));
      }
      const int64_t lo = static_cast<int64_t>(L.sr) * L.shard_n;
      for (int64_t j = 0; j < L.shard_n; ++j) {
        const int64_t c = canon_index(L.sh, L.lay, L.d.tp, L.tr, lo + j);
        if (c >= 0) canonical[c] = shard[j];
      }
    }
  }
  return kOk;
}

int ExecutorImpl::init_params(uint64_t seed, float std_dev) {
  for (auto& r : ranks_) {
    for (RankLayer& L : r->layers) {
      InitLayout il{};
      const Slot* slots[kInitSlots] = {
          &L.lay.ln1g, &L.lay.ln1b, &L.lay.ln2g, &L.lay.ln2b, &L.lay.bqkv, &L.lay.bo,
          &L.lay.b1,   &L.lay.b2,   &L.lay.wqkv, &L.lay.wo,   &L.lay.w1,   &L.lay.w2,
          &L.lay.mlng, &L.lay.mlnb, &L.lay.wm,   &L.lay.ln3g, &L.lay.ln3b, &L.lay.bq2,
          &L.lay.bkv2, &L.lay.bo2,  &L.lay.wq2,  &L.lay.wkv2, &L.lay.wo2,  &L.lay.rpb,
          &L.lay.relb};
      il.extra = L.sh.merge ? 1 : (L.sh.cross ? 2 : 0);
      for (int i = 0; i < kInitSlots; ++i) {
        il.off[i] = slots[i]->off;
        il.n[i] = slots[i]->n;
      }
      il.h = L.sh.h;
      il.f = L.sh.ffn;
      il.t = L.d.tp;
      il.tr = L.tr;
      il.lo = static_cast<int64_t>(L.sr) * L.shard_n;
      GX_TRY(gx::init_params(L.master, L.shard_n, il, seed, static_cast<uint64_t>(L.layer), std_dev,
                             stream_));
      GX_TRY(cast_bf16(L.master, L.pshard, L.shard_n, stream_));
      GX_TRY(cuda_check(cudaMemsetAsync(L.m, 0, L.shard_n * 4, stream_), "memset m"));
      GX_TRY(cuda_check(cudaMemsetAsync(L.v, 0, L.shard_n * 4, stream_), "memset v"));
    }
  }
  return cuda_check(cudaStreamSynchronize(stream_), "init_params");
}

// ------------------------------------------------------------------------------ inputs
int ExecutorImpl::load_batch(const void* x_host, const void* target_host) {
  for (auto& rp : ranks_) {
    RankCtx& r = *rp;
    for (int mb = 0; mb < m_; ++mb) {
      if (r.stage == 0 && x_host != nullptr) {
        const RankLayer& F = r.layers.front();
        const Acts& a = F.acts[mb];
        const size_t row_bytes = static_cast<size_t>(F.sh.h) * 2;
        GX_TRY(cuda_check(
            cudaMemcpyAsync(r.x_in + r.in_row_off[mb] * F.sh.h,
                            static_cast<const char*>(x_host) + a.sample0 * F.sh.seq * row_bytes,
                            a.rows * row_bytes, cudaMemcpyHostToDevice, stream_),
            "load_batch x"));
      }
      if (r.stage == P_ - 1 && target_host != nullptr) {
        const RankLayer& Lz = r.layers.back();
        const Acts& a = Lz.acts[mb];
        const size_t row_bytes = static_cast<size_t>(Lz.sh.h) * 2;
        int64_t off = 0;
        for (int k = 0; k < mb; ++k) off += Lz.acts[k].rows;
        GX_TRY(cuda_check(
            cudaMemcpyAsync(r.target + off * Lz.sh.h,
                            static_cast<const char*>(target_host) + a.sample0 * Lz.sh.seq * row_bytes,
                            a.rows * row_bytes, cudaMemcpyHostToDevice, stream_),
            "load_batch target"));
      }
    }
  }
  return kOk;
}

int ExecutorImpl::load_batch_device(const void* x_dev, const void* target_dev) {
  // The caller produced the buffers on its own stream; our streams are non-blocking, so order
  // the copies after the legacy default stream explicitly (callers on other streams must
  // synchronise them first -- the Python wrapper does).
  {
    cudaEvent_t ev = nullptr;
    GX_TRY(cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "load event"));
    cudaError_t e = cudaEventRecord(ev, cudaStreamLegacy);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream_, ev, 0);
    cudaEventDestroy(ev);
    GX_TRY(cuda_check(e, "load_batch_device order"));
  }
  for (auto& rp : ranks_) {
    RankCtx& r = *rp;
    for (int mb = 0; mb < m_; ++mb) {
      if (r.stage == 0 && x_dev != nullptr) {
        const RankLayer& F = r.layers.front();
        const Acts& a = F.acts[mb];
        const size_t row_bytes = static_cast<size_t>(F.sh.h) * 2;
        GX_TRY(cuda_check(
            cudaMemcpyAsync(r.x_in + r.in_row_off[mb] * F.sh.h,
                            static_cast<const char*>(x_dev) + a.sample0 * F.sh.seq * row_bytes,
                            a.rows * row_bytes, cudaMemcpyDeviceToDevice, stream_),
            "load_batch_device x"));
      }
      if (r.stage == P_ - 1 && target_dev != nullptr) {
        const RankLayer& Lz = r.layers.back();
        const Acts& a = Lz.acts[mb];
        const size_t row_bytes = static_cast<size_t>(Lz.sh.h) * 2;
        int64_t off = 0;
        for (int k = 0; k < mb; ++k) off += Lz.acts[k].rows;
        GX_TRY(cuda_check(
            cudaMemcpyAsync(r.target + off * Lz.sh.h,
                            static_cast<const char*>(target_dev) + a.sample0 * Lz.sh.seq * row_bytes,
                            a.rows * row_bytes, cudaMemcpyDeviceToDevice, stream_),
            "load_batch_device target"));
      }
    }
  }
  return kOk;
}

int ExecutorImpl::export_output(void* host, int what) {
  // what: 0 = model output, 1 = model input gradient, 2 + l = output of layer l,
  // 1000 + 16*l + k = activation k of layer l (debug: 0 x 1 ln1 2 x1 3 ln2 4 gel 5 y), [rows][h|ffn]
  GX_TRY(cuda_check(cudaStreamSynchronize(stream_), "export sync"));
  if (what >= 1000) {
    const int l = (what - 1000) / 16, k = (what - 1000) % 16;
    for (auto& rp : ranks_) {
      for (const RankLayer& L : rp->layers) {
        if (L.layer != l || L.tr != 0) continue;
        const int64_t w = k == 4 ? L.sh.ffn / L.d.tp : L.sh.h;
        for (int mb = 0; mb < m_; ++mb) {
          const Acts& a = L.acts[mb];
          const bf16* src = k == 0 ? a.x : k == 1 ? a.ln1 : k == 2 ? a.x1 : k == 3 ? a.ln2 : k == 4 ? a.gel : a.y;
          if (a.rows > 0)
            GX_TRY(cuda_check(cudaMemcpy(static_cast<char*>(host) + a.sample0 * L.sh.seq * w * 2, src,
                                         a.rows * w * 2, cudaMemcpyDeviceToHost), "export act"));
        }
      }
    }
    return kOk;
  }
  for (auto& rp : ranks_) {
    RankCtx& r = *rp;
    const RankLayer* Lp = nullptr;
    if (what == 0 && r.stage == P_ - 1) Lp = &r.layers.back();
    if (what == 1 && r.stage == 0) Lp = &r.layers.front();
    if (what >= 2)
      for (const RankLayer& L : r.layers)
        if (L.layer == what - 2) Lp = &L;
    if (Lp == nullptr || Lp->tr != 0) continue;
    const RankLayer& L = *Lp;
    const size_t rb = static_cast<size_t>(L.sh.h) * 2;
    int64_t off = 0;
    for (int mb = 0; mb < m_; ++mb) {
      const Acts& a = L.acts[mb];
      const void* src = what != 1 ? static_cast<const void*>(a.y)
                                  : static_cast<const void*>(r.dx_out + off * L.sh.h);
      if (a.rows > 0)
        GX_TRY(cuda_check(cudaMemcpy(static_cast<char*>(host) + a.sample0 * L.sh.seq * rb, src,
                                     a.rows * rb, cudaMemcpyDeviceToHost),
                          "export_output"));
      off += a.rows;
    }
  }
  return kOk;
}

}  // namespace xi
}  // namespace gx
