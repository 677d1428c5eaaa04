// exec_backward.cc -- backward phases of a layer: data-gradient chain on the compute stream, weight
// gradients (+ bias / LayerNorm column sums) on the wgrad stream
#include "executor_impl.h"

namespace gx {
namespace xi {

// -------------------------------------------------------------------- backward phases
// dY in gbuf[cur]; dX goes to gbuf[cur ^ 1].
int ExecutorImpl::bwd_phase(RankCtx& r, int li, int mb, int phase) {
  RankLayer& L = r.layers[li];
  Acts& A = L.acts[mb];
  const Shape& s = L.sh;
  const int t = L.d.tp;
  const int rows = A.rows;
  const int h = s.h, ht = s.h / t, ft = s.ffn / t;
  const bf16* P = L.pfull;
  float* G = L.gfull;
  const int l = L.layer;
  const int64_t row_off = A.sample0 * s.seq;
  const bool first_mb = mb == m_ - 1;  // backward visits micro-batches in reverse
  const int wk = first_mb && !r.idle_chunks ? kOutF32 : kOutF32Accumulate;
  bf16* dY = r.gbuf[r.cur];
  bf16* dX = r.gbuf[r.cur ^ 1];
  if (rows == 0) return kOk;
  const int par = li & 1;
  bf16 *dz = r.dzb[par], *dpre = r.dpreb[par], *dout = r.doutb[par], *dqkv = r.dqkvb[par];
  // Weight-gradient epilogue for a weight slot: fp32 gradient into G (written on the first
  // backward micro-batch, accumulated on the others).
  auto wgrad_ep = [&](const Slot& slot, int64_t ldo) {
    gx_gemm_epilogue w = epi();
    w.ldo = ldo;
    w.out_kind = wk;
    w.out = G + slot.off;
    return w;
  };
  gx_dropout d{};
  d.threshold = thr_hidden_;
  d.scale = scale_of(p_hidden_);
  d.seed = seed_;
  d.row_offset = row_off;
  d.drop_ld = h;
  d.seed_offset = r.seed_off;
  if (phase == 0) {
    // this parity's buffers are free once the wgrads that last read them are done
    if (r.wg_pending[par]) {
      GX_TRY(cuda_check(cudaStreamWaitEvent(stream_, r.wg_done[par], 0), "wgrad wait"));
      r.wg_pending[par] = false;
    }
    d.site = 3ull * l + 2;
    GX_TRY(timed(kElementwise, 0, 4.0 * rows * h, [&] { return dropout_bwd_colsum(dY, dz, G + L.lay.b2.off, rows, h, d, stream_, r.cs_ws[0]); }));
    const gx_gemm_epilogue w2 = wgrad_ep(L.lay.w2, ft);
    // dW2 = dz^T gel, as early as its inputs exist
    GX_TRY(on_wgrad([&] { return gemm(dz, h, true, A.gel, ft, true, h, ft, rows, w2); }));
    gx_gemm_epilogue e = epi();
    e.out_kind = kOutBF16;
    e.out = dpre;
    e.ldo = ft;
    e.gelu_bwd = 2;
    e.aux = A.pre;
    e.ld_aux = ft;
    GX_TRY(gemm(dz, h, false, P + L.lay.w2.off, ft, true, rows, ft, h, e));  // dz W2 * gelu'
    GX_TRY(on_wgrad([&]() -> int {
      GX_TRY(timed(kElementwise, 0, 2.0 * rows * h, [&] { return colsum(dpre, ft, G + L.lay.b1.off, rows, ft, ls_, r.cs_ws[ls_ == stream_ ? 0 : 1]); }));
      const gx_gemm_epilogue w1 = wgrad_ep(L.lay.w1, h);
      return gemm(dpre, ft, true, A.ln2, h, true, ft, h, rows, w1);  // dW1 = dpre^T ln2
    }));
    int sp_c = 1;
    if (t == 1)
      GX_TRY(gemm_splitk(r, dpre, ft, P + L.lay.w1.off, h, true, rows, h, ft, &sp_c));
    r.dc_slices = sp_c;
    if (sp_c == 1) {
      // fp32 (one slice in acc32): LN2's backward reads the unrounded gradient, and TP partial
      // sums are all-reduced in fp32 -- bf16 rounding of the partials before the LayerNorm's
      // column sums cost up to 1.03e-2 relative error on dgamma (SURVEY 8(d) bar: 1e-2)
      gx_gemm_epilogue c = epi();
      c.out_kind = kOutF32;
      c.out = r.acc32;
      c.ldo = h;
      GX_TRY(gemm(dpre, ft, false, P + L.lay.w1.off, h, true, rows, h, ft, c));  // dpre W1
    }
    if (t > 1)
      return c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.acc32, static_cast<size_t>(rows) * h,
                          DType::kF32, stream_);
    phase = 1;
  }
  // TP decoder layers: [MLP] [LN2 + cross attention] [LN3 + self-attention] [LN1] (+ [dmem
  // all-reduce] [dmem add] on the first decoder layer); every other layer: [MLP] [LN2 +
  // self-attention] [LN1]
  const bool xtp = s.cross && t > 1;
  const int ln1_ph = xtp ? 3 : 2;
  if (phase == 1 || (xtp && phase == 2)) {
   if (phase == 1) {
    const void* dc_in = r.acc32;
    // LN2 backward with the out-projection's dropout backward + bias gradient fused in:
    // dx1 = residual-stream gradient, dout = dropout_mask(dx1), dbo += colsum(dout)
    // (row pass on the critical path; the dgamma / dbeta / dbias column pass rides the wgrad
    // stream from the row pass's fp32 copy of dy)
    // (decoder layers: LN2 sits on x2 and the dropout below it is the cross sublayer's)
    const bool xd = s.cross;
    d.site = xd ? 3ull * L_ + 2ull * l + 1 : 3ull * l + 1;
    bf16* const xr = xd ? A.x2 : A.x1;
    bf16* const dz2 = xd ? r.dout2 : dout;
    float* fold2 = r.lnfold[par][0];
    GX_TRY(timed(kNorm, 0, 10.0 * rows * h, [&] { return layernorm_bwd_rows(dc_in, xr, A.mean2, A.rstd2, P + L.lay.ln2g.off, dY, r.dx1,
                         rows, h, stream_, true, &d, dz2, r.dc_slices,
                         static_cast<int64_t>(rows) * h, fold2); }));
    GX_TRY(on_wgrad([&] {
      return timed(kNorm, 0, 8.0 * rows * h, [&] { return layernorm_bwd_cols(fold2, true, xr, A.mean2, A.rstd2, dz2,
                         G + L.lay.ln2g.off, G + L.lay.ln2b.off, G + (xd ? L.lay.bo2 : L.lay.bo).off, rows, h, r.ln_ws, ls_); });
    }));
    if (xd) {
      // the wgrad-stream LN2 column pass above reads dout2 / fold2: let it finish first
      if (wg_active_) GX_TRY(fork(wg_, stream_));
      GX_TRY(cross_bwd_attn(r, li, mb, wgrad_ep));  // -> dc3 (TP: partial) in r.acc32 (fp32)
      if (t > 1)
        return c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.acc32, static_cast<size_t>(rows) * h,
                            DType::kF32, stream_);
    }
   }
    if (s.cross) GX_TRY(cross_bwd_ln3(r, li, mb, dout));  // dx1, dout (self-attention)
    const gx_gemm_epilogue wo = wgrad_ep(L.lay.wo, ht);
    // dWo = dout^T ctx
    GX_TRY(on_wgrad([&] { return gemm(dout, h, true, A.ctx, ht, true, h, ht, rows, wo); }));
    gx_gemm_epilogue c = epi();
    c.out_kind = kOutBF16;
    c.out = r.dctx;
    c.ldo = ht;
    GX_TRY(gemm(dout, h, false, P + L.lay.wo.off, ht, true, rows, ht, h, c));  // dout Wo
    gx_attention_args at{};
    at.batch = A.samples * s.windows();  // one attention sequence per window
    at.seq = s.win;
    at.heads = s.heads / t;
    at.head_dim = s.hd;
    at.heads_total = s.heads;
    at.head_offset = L.tr * (s.heads / t);
    at.sample_offset = A.sample0 * s.windows();
    at.scale = 1.f / std::sqrt(static_cast<float>(s.hd));
    if (s.shift > 0)  // the attention saw rolled tokens: roll its output gradient likewise
      GX_TRY(timed(kElementwise, 0, 4.0 * rows * ht, [&] {
        return window_roll(r.dctx, r.dctxr, A.samples, grid_of(s), side_of(s), s.shift, ht,
                           false, stream_);
      }));
    at.qkv = A.qkv;
    at.ld_qkv = 3 * ht;
    at.ctx = s.shift > 0 ? A.ctxr : A.ctx;
    at.ld_ctx = ht;
    at.lse = A.lse;
    set_window_mask(at, s);
    if (s.rpb) {
      at.rpb = P + L.lay.rpb.off;
      at.rpb_side = side_of(s);
      at.rpb_dpart = r.rpb_part;
    }
    if (s.relb) {
      at.relb = P + L.lay.relb.off;
      at.relb_map = L.relb_map;
      at.relb_buckets = s.relb;
      at.relb_dpart = r.relb_part;
    }
    at.dctx = s.shift > 0 ? r.dctxr : r.dctx;
    at.dqkv = dqkv;
    at.dq_accum = r.dq_acc;
    at.dsum = r.dsum;
    at.drop_threshold = thr_attn_;
    at.drop_scale = scale_of(p_attn_);
    at.seed = seed_;
    at.site = 3ull * l;
    at.seed_offset = r.seed_off;
    at.mask = A.amask;
    at.causal = s.causal ? 1 : 0;
    {
      const double af = 10.0 * A.samples * (s.heads / t) * double(s.seq) * s.win * s.hd;
      GX_TRY(timed(kAttnBwd, af, 2.0 * rows * 8 * ht, [&] { return attention_bwd(at, stream_); }));
    }
    if (s.relb)  // T5 table gradient: fixed-order sum over sequences, key blocks, positions
      GX_TRY(timed(kElementwise, 0, 4.0 * A.samples * (s.heads / t) * ((s.seq + 127) / 128) *
                                        (2.0 * s.seq - 1), [&] {
        const int wpt = s.seq <= 64 ? 128 / s.seq : 1;  // sequences per attention tile
        return relb_grad(r.relb_part, (A.samples + wpt - 1) / wpt, s.heads / t, s.seq,
                         L.relb_map, s.relb, G + L.lay.relb.off, true, stream_);
      }));
    if (s.rpb)  // table gradient: fixed-order sum of the per-window score gradients
      GX_TRY(timed(kElementwise, 0, 4.0 * A.samples * s.windows() * (s.heads / t) * s.rpb_n(), [&] {
        return rpb_grad(r.rpb_part, A.samples * s.windows(), s.heads / t, side_of(s),
                        G + L.lay.rpb.off, true, stream_);
      }));
    GX_TRY(on_wgrad([&]() -> int {
      GX_TRY(timed(kElementwise, 0, 2.0 * rows * h, [&] { return colsum(dqkv, 3 * ht, G + L.lay.bqkv.off, rows, 3 * ht, ls_, r.cs_ws[ls_ == stream_ ? 0 : 1]); }));
      const gx_gemm_epilogue wq = wgrad_ep(L.lay.wqkv, h);
      return gemm(dqkv, 3 * ht, true, s.shift > 0 ? A.ln1r : A.ln1, h, true, 3 * ht, h, rows,
                  wq);  // dWqkv
    }));
    int sp_a = 1;
    if (t == 1 && s.shift == 0)  // (SW-MSA rolls dA back before LN1: keep it bf16)
      GX_TRY(gemm_splitk(r, dqkv, 3 * ht, P + L.lay.wqkv.off, h, true, rows, h, 3 * ht, &sp_a));
    r.da_slices = sp_a;
    if (sp_a == 1) {
      gx_gemm_epilogue a = epi();
      a.out_kind = s.shift > 0 ? kOutBF16 : kOutF32;  // fp32 into LN1's backward, as for LN2
      a.out = s.shift > 0 ? static_cast<void*>(r.da) : static_cast<void*>(r.acc32);
      a.ldo = h;
      GX_TRY(gemm(dqkv, 3 * ht, false, P + L.lay.wqkv.off, h, true, rows, h, 3 * ht, a));
      if (s.shift > 0) {  // LN1 (and the residual) live in the unrolled order
        GX_TRY(timed(kElementwise, 0, 8.0 * rows * h, [&] {
          return window_roll(r.da, r.rollbuf, A.samples, grid_of(s), side_of(s), s.shift, h, true,
                             stream_);
        }));
        GX_TRY(cuda_check(cudaMemcpyAsync(r.da, r.rollbuf, static_cast<size_t>(rows) * h * 2,
                                          cudaMemcpyDeviceToDevice, stream_),
                          "sw-msa da"));
      }
    }
    if (s.shift > 0) r.da_slices = 0;  // bf16 in r.da
    if (t > 1)
      return r.da_slices == 0
                 ? c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.da, static_cast<size_t>(rows) * h,
                                DType::kBF16, stream_)
                 : c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.acc32,
                                static_cast<size_t>(rows) * h, DType::kF32, stream_);
    phase = 2;
  }
  if (phase == ln1_ph) {
    const void* da_in = r.da_slices ? static_cast<const void*>(r.acc32) : static_cast<const void*>(r.da);
    float* fold1 = r.lnfold[par][1];
    GX_TRY(timed(kNorm, 0, 8.0 * rows * h, [&] { return layernorm_bwd_rows(da_in, A.x, A.mean1, A.rstd1, P + L.lay.ln1g.off, r.dx1, dX,
                         rows, h, stream_, r.da_slices > 0, nullptr, nullptr,
                         std::max(1, r.da_slices), static_cast<int64_t>(rows) * h, fold1); }));
    GX_TRY(on_wgrad([&]() -> int {
      GX_TRY(timed(kNorm, 0, 8.0 * rows * h, [&] { return layernorm_bwd_cols(fold1, true, A.x, A.mean1, A.rstd1, nullptr,
                           G + L.lay.ln1g.off, G + L.lay.ln1b.off, nullptr,
                           rows, h, r.ln_ws, ls_); }));
      if (wg_active_) {  // the last reader of this parity's buffers
        GX_TRY(cuda_check(cudaEventRecord(r.wg_done[par], wg_), "wgrad done"));
        r.wg_pending[par] = true;
      }
      return kOk;
    }));
    if (s.merge) GX_TRY(merge_bwd(r, L, A, dX, wgrad_ep(L.lay.wm, 2 * h)));
    if (li == r.dec_li && t > 1)  // TP ranks hold per-head partial sums of dL/dmem
      return c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.dmem, static_cast<size_t>(rows) * h, DType::kF32,
                          stream_);
    phase = ln1_ph + 1;
  }
  if (phase == ln1_ph + 1 && li == r.dec_li) {
    // this input is also every decoder layer's memory: dX += dL/dmem
    gx_dropout off{};
    GX_TRY(timed(kElementwise, 0, 8.0 * rows * h, [&] {
      return bias_dropout_add(r.dmem, nullptr, dX, dX, rows, h, off, stream_, true);
    }));
  }
  return kOk;
}

// Decoder cross-attention sublayer, backward (main stream).  In: r.dx1 = dL/dx2 (the residual
// gradient below the MLP), r.dout2 = its dropout-masked copy (bo2's gradient already taken).
// Out: r.dx1 = dL/dx1, dout = dL/d(self-attention out-projection) with bo's gradient, and
// dL/dmem accumulated into r.dmem.
int ExecutorImpl::cross_bwd_attn(RankCtx& r, int li, int mb,
                                 const std::function<gx_gemm_epilogue(const Slot&, int64_t)>& wgrad_ep) {
  RankLayer& L = r.layers[li];
  Acts& A = L.acts[mb];
  const Shape& s = L.sh;
  const int rows = A.rows, h = s.h, t = L.d.tp, ht = h / t;
  const bf16* P = L.pfull;
  float* G = L.gfull;
  const bf16* mem = r.mem(mb);
  gx_gemm_epilogue c = epi();
  c.out_kind = kOutBF16;
  c.out = r.dctx;
  c.ldo = ht;
  GX_TRY(gemm(r.dout2, h, false, P + L.lay.wo2.off, ht, true, rows, ht, h, c));  // dout2 Wo2
  GX_TRY(gemm(r.dout2, h, true, A.ctx2, ht, true, h, ht, rows, wgrad_ep(L.lay.wo2, ht)));
  gx_attention_args at = cross_args(r, L, A);
  at.dctx = r.dctx;
  at.dqkv = r.dqkv2;
  GX_TRY(timed(kAttnBwd, 10.0 * A.samples * (s.heads / t) * double(s.seq) * s.seq * s.hd,
               2.0 * rows * 8 * ht, [&] { return attention_bwd(at, stream_); }));
  // weight / bias gradients of the q and kv projections (this rank's heads)
  GX_TRY(colsum(r.dqkv2, 3 * ht, G + L.lay.bq2.off, rows, ht, stream_, r.cs_ws[0]));
  GX_TRY(gemm(r.dqkv2, 3 * ht, true, A.ln3, h, true, ht, h, rows, wgrad_ep(L.lay.wq2, h)));
  GX_TRY(colsum(r.dqkv2 + ht, 3 * ht, G + L.lay.bkv2.off, rows, 2 * ht, stream_, r.cs_ws[0]));
  GX_TRY(gemm(r.dqkv2 + ht, 3 * ht, true, mem, h, true, 2 * ht, h, rows, wgrad_ep(L.lay.wkv2, h)));
  // memory gradient (TP: partial over heads): the last decoder layer starts the sum
  gx_gemm_epilogue m = epi();
  m.out_kind = li + 1 == static_cast<int>(r.layers.size()) && !r.dmem_from_next
                   ? kOutF32 : kOutF32Accumulate;
  m.out = r.dmem;
  m.ldo = h;
  GX_TRY(gemm(r.dqkv2 + ht, 3 * ht, false, P + L.lay.wkv2.off, h, true, rows, h, 2 * ht, m));
  c.out_kind = kOutF32;  // fp32 into LN3's backward (and the TP all-reduce), as for LN2
  c.out = r.acc32;
  c.ldo = h;
  return gemm(r.dqkv2, 3 * ht, false, P + L.lay.wq2.off, h, true, rows, h, ht, c);  // dq Wq2
}

// LN3 backward: dx1 = dx2 + LN3'(dc3), with the self-attention out-projection's dropout
// backward and bias gradient fused in (as LN2's backward does for non-decoder layers).
int ExecutorImpl::cross_bwd_ln3(RankCtx& r, int li, int mb, bf16* dout) {
  RankLayer& L = r.layers[li];
  Acts& A = L.acts[mb];
  const Shape& s = L.sh;
  const int rows = A.rows, h = s.h;
  const bf16* P = L.pfull;
  float* G = L.gfull;
  const int l = L.layer;
  gx_dropout d{};
  d.threshold = thr_hidden_;
  d.scale = scale_of(p_hidden_);
  d.seed = seed_;
  d.site = 3ull * l + 1;
  d.row_offset = A.sample0 * s.seq;
  d.drop_ld = h;
  d.seed_offset = r.seed_off;
  return timed(kNorm, 0, 18.0 * rows * h, [&] {
    return layernorm_bwd(r.acc32, A.x1, A.mean3, A.rstd3, P + L.lay.ln3g.off, r.dx1, r.dx1,
                         G + L.lay.ln3g.off, G + L.lay.ln3b.off, rows, h, r.ln_ws_x, stream_,
                         true, &d, dout, G + L.lay.bo.off, 1, static_cast<int64_t>(rows) * h);
  });
}

// Patch-merging backward (main stream, after LN1's backward left dL/dx in dX):
// dmln = dX Wm, dWm = dX^T mln, LayerNorm(2h) backward, then the 2x2 scatter writes the input
// gradient [4*rows][h/2] over dX (both readers of dX ran before it on this stream).
int ExecutorImpl::merge_bwd(RankCtx& r, RankLayer& L, Acts& A, bf16* dX,
                            const gx_gemm_epilogue& wm_ep) {
  const Shape& s = L.sh;
  const int rows = A.rows, h = s.h;
  const bf16* P = L.pfull;
  float* G = L.gfull;
  gx_gemm_epilogue c = epi();
  c.out_kind = kOutBF16;
  c.out = r.dmg1;
  c.ldo = 2 * h;
  GX_TRY(gemm(dX, h, false, P + L.lay.wm.off, 2 * h, true, rows, 2 * h, h, c));  // dX Wm
  GX_TRY(gemm(dX, h, true, A.mln, 2 * h, true, h, 2 * h, rows, wm_ep));          // dWm
  GX_TRY(timed(kNorm, 0, 12.0 * rows * h, [&] {
    return layernorm_bwd(r.dmg1, A.mg, A.meanm, A.rstdm, P + L.lay.mlng.off, nullptr, r.dmg2,
                         G + L.lay.mlng.off, G + L.lay.mlnb.off, rows, 2 * h, r.ln_ws_m, stream_);
  }));
  const int g = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.seq))));
  const int ws = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.win))));
  return timed(kElementwise, 0, 2.0 * rows * 2 * h * 2, [&] {
    return patch_merge(r.dmg2, dX, A.samples, g, ws, h / 2, true, stream_);
  });
}

}  // namespace xi
}  // namespace gx
