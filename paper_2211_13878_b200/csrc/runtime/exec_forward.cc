// exec_forward.cc -- forward phases of a layer: LN -> QKV -> attention -> out-projection (+ residual,
// next LN) -> MLP, the decoder's cross-attention sublayer; each phase ends at a collective
#include "executor_impl.h"

namespace gx {
namespace xi {

// --------------------------------------------------------------------- forward phases
// Phase 0 runs after the layer input is in place.  tp == 1: one phase (all epilogues fused
// into the GEMMs).  tp > 1: phases end at the two activation all-reduces.
int ExecutorImpl::fwd_phase(RankCtx& r, int li, int mb, int phase) {
  RankLayer& L = r.layers[li];
  Acts& A = L.acts[mb];
  const Shape& s = L.sh;
  const int t = L.d.tp;
  const int rows = A.rows;
  const int h = s.h, ht = s.h / t, ft = s.ffn / t;
  const bf16* P = L.pfull;
  const int l = L.layer;
  const int64_t row_off = A.sample0 * s.seq;
  if (rows == 0) return kOk;
  bool ln2_ready = false, ln3_ready = false;
  if (phase == 0) {
    if (s.merge) {  // Swin patch merging: gather 2x2 -> LayerNorm(2h) -> x = mln Wm^T
      const int g = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.seq))));
      const int ws = static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.win))));
      GX_TRY(timed(kElementwise, 0, 2.0 * rows * 2 * h * 2, [&] {
        return patch_merge(A.xm, A.mg, A.samples, g, ws, h / 2, false, stream_);
      }));
      GX_TRY(timed(kNorm, 0, 8.0 * rows * h, [&] {
        return layernorm_fwd(A.mg, P + L.lay.mlng.off, P + L.lay.mlnb.off, A.mln, A.meanm,
                             A.rstdm, rows, 2 * h, stream_);
      }));
      gx_gemm_epilogue e = epi();
      e.out_kind = kOutBF16;
      e.out = A.x;
      e.ldo = h;
      GX_TRY(gemm(A.mln, 2 * h, false, P + L.lay.wm.off, 2 * h, false, rows, h, 2 * h, e));
    }
    if (!A.ln1_ready)
      GX_TRY(timed(kNorm, 0, 4.0 * rows * h, [&] { return layernorm_fwd(A.x, P + L.lay.ln1g.off, P + L.lay.ln1b.off, A.ln1, A.mean1, A.rstd1,
                           rows, h, stream_); }));
    const bf16* qkv_in = A.ln1;
    if (s.shift > 0) {  // SW-MSA: roll the (per-token) LN1 output, attend, roll the context back
      GX_TRY(timed(kElementwise, 0, 4.0 * rows * h, [&] {
        return window_roll(A.ln1, A.ln1r, A.samples, grid_of(s), side_of(s), s.shift, h, false,
                           stream_);
      }));
      qkv_in = A.ln1r;
    }
    gx_gemm_epilogue e = epi();
    e.out_kind = kOutBF16;
    e.out = A.qkv;
    e.ldo = 3 * ht;
    e.bias = P + L.lay.bqkv.off;
    GX_TRY(gemm(qkv_in, h, false, P + L.lay.wqkv.off, h, false, rows, 3 * ht, h, e));
    gx_attention_args at{};
    at.batch = A.samples * s.windows();  // one attention sequence per window
    at.seq = s.win;
    at.heads = s.heads / t;
    at.head_dim = s.hd;
    at.heads_total = s.heads;
    at.head_offset = L.tr * (s.heads / t);
    at.sample_offset = A.sample0 * s.windows();
    at.scale = 1.f / std::sqrt(static_cast<float>(s.hd));
    at.qkv = A.qkv;
    at.ld_qkv = 3 * ht;
    at.ctx = s.shift > 0 ? A.ctxr : A.ctx;
    at.ld_ctx = ht;
    at.lse = A.lse;
    set_window_mask(at, s);
    if (s.rpb) {
      at.rpb = P + L.lay.rpb.off;
      at.rpb_side = side_of(s);
    }
    if (s.relb) {  // T5 relative bias of this rank's heads
      at.relb = P + L.lay.relb.off;
      at.relb_map = L.relb_map;
      at.relb_buckets = s.relb;
    }
    at.drop_threshold = thr_attn_;
    at.drop_scale = scale_of(p_attn_);
    at.seed = seed_;
    at.site = 3ull * l;
    at.seed_offset = r.seed_off;
    at.mask = A.amask;
    at.causal = s.causal ? 1 : 0;
    {
      const double af = 4.0 * A.samples * (s.heads / t) * double(s.seq) * s.win * s.hd;
      GX_TRY(timed(kAttnFwd, af, 2.0 * rows * 4 * ht, [&] { return attention_fwd(at, stream_); }));
    }
    if (s.shift > 0)
      GX_TRY(timed(kElementwise, 0, 4.0 * rows * ht, [&] {
        return window_roll(A.ctxr, A.ctx, A.samples, grid_of(s), side_of(s), s.shift, ht, true,
                           stream_);
      }));
    gx_gemm_epilogue o = epi();
    o.out_kind = kOutBF16;
    o.ldo = h;
    if (t == 1) {
      // split-K out-projection -> one row pass: slice sum + bias + dropout + residual + LN2
      int sp = 1;
      GX_TRY(gemm_splitk(r, A.ctx, ht, P + L.lay.wo.off, ht, false, rows, h, ht, &sp));
      if (sp > 1) {
        gx_dropout d{};
        d.threshold = thr_hidden_;
        d.scale = scale_of(p_hidden_);
        d.seed = seed_;
        d.site = 3ull * l + 1;
        d.row_offset = row_off;
        d.drop_ld = h;
        d.seed_offset = r.seed_off;
        // (decoder layers: the LayerNorm that follows is the cross sublayer's LN3)
        GX_TRY(timed(kNorm, 0, (4.0 * sp + 8.0) * rows * h, [&] {
          return residual_layernorm(r.acc32, sp, static_cast<int64_t>(rows) * h, P + L.lay.bo.off,
                                    A.x, A.x1, d, P + (s.cross ? L.lay.ln3g : L.lay.ln2g).off,
                                    P + (s.cross ? L.lay.ln3b : L.lay.ln2b).off,
                                    s.cross ? A.ln3 : A.ln2, s.cross ? A.mean3 : A.mean2,
                                    s.cross ? A.rstd3 : A.rstd2, rows, h, stream_);
        }));
        (s.cross ? ln3_ready : ln2_ready) = true;
      } else {
        o.out = A.x1;
        o.bias = P + L.lay.bo.off;
        o.residual = A.x;
        o.ld_res = h;
        o.row_offset = row_off;
        o.drop_ld = h;
        o.drop_threshold = thr_hidden_;
        o.drop_scale = scale_of(p_hidden_);
        o.seed = seed_;
        o.site = 3ull * l + 1;
        o.seed_offset = r.seed_off;
        GX_TRY(gemm(A.ctx, ht, false, P + L.lay.wo.off, ht, false, rows, h, ht, o));
      }
    } else {
      o.out = r.partial;
      GX_TRY(gemm(A.ctx, ht, false, P + L.lay.wo.off, ht, false, rows, h, ht, o));
      return c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.partial, static_cast<size_t>(rows) * h,
                               DType::kBF16, stream_);
    }
  }
  // the MLP's residual-stream input: x1, or -- after a decoder's cross sublayer -- x2
  bf16* const xr = s.cross ? A.x2 : A.x1;
  // TP phases: [attention] [cross (decoders)] [MLP] [final residual]
  const int mlp_ph = t > 1 ? (s.cross ? 2 : 1) : 0;
  if (t > 1 && s.cross && phase == 1) {
    GX_TRY(timed(kElementwise, 0, 6.0 * rows * h, [&] {
      return bias_dropout_add(r.partial, P + L.lay.bo.off, A.x, A.x1, rows, h,
                              hidden_drop(r, 3ull * l + 1, row_off, h), stream_);
    }));
    GX_TRY(cross_fwd(r, li, mb, false));  // leaves the out-projection partial in r.partial
    return c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.partial, static_cast<size_t>(rows) * h, DType::kBF16,
                        stream_);
  }
  if (phase == mlp_ph) {
    if (t > 1) {  // the all-reduced sublayer output below the MLP: + bias, dropout, residual
      const bool xd = s.cross;
      GX_TRY(timed(kElementwise, 0, 6.0 * rows * h, [&] {
        return bias_dropout_add(r.partial, P + (xd ? L.lay.bo2 : L.lay.bo).off, xd ? A.x1 : A.x,
                                xr, rows, h,
                                hidden_drop(r, xd ? 3ull * L_ + 2ull * l + 1 : 3ull * l + 1,
                                            row_off, h),
                                stream_);
      }));
    }
    if (s.cross && t == 1) GX_TRY(cross_fwd(r, li, mb, ln3_ready));
    if (!ln2_ready)
      GX_TRY(timed(kNorm, 0, 4.0 * rows * h, [&] { return layernorm_fwd(xr, P + L.lay.ln2g.off, P + L.lay.ln2b.off, A.ln2, A.mean2, A.rstd2,
                           rows, h, stream_); }));
    gx_gemm_epilogue e = epi();
    e.out_kind = kOutBF16;
    e.out = A.gel;
    e.ldo = ft;
    e.bias = P + L.lay.b1.off;
    e.gelu = 2;  // A.pre receives gelu'(pre-activation) for the backward's plain multiply
    e.aux = A.pre;
    e.ld_aux = ft;
    GX_TRY(gemm(A.ln2, h, false, P + L.lay.w1.off, h, false, rows, ft, h, e));
    gx_gemm_epilogue o = epi();
    o.out_kind = kOutBF16;
    o.ldo = h;
    if (t == 1) {
      int sp = 1;
      GX_TRY(gemm_splitk(r, A.gel, ft, P + L.lay.w2.off, ft, false, rows, h, ft, &sp));
      if (sp > 1) {  // split-K partials summed in fp32, then bias + dropout + residual
        gx_dropout d{};
        d.threshold = thr_hidden_;
        d.scale = scale_of(p_hidden_);
        d.seed = seed_;
        d.site = 3ull * l + 2;
        d.row_offset = row_off;
        d.drop_ld = h;
        d.seed_offset = r.seed_off;
        // ... and the next layer's LN1 in the same row pass when its input aliases this
        // output and its LayerNorm parameters are resident (no SDP gather pending)
        Acts* nxt = nullptr;
        const bf16* PN = nullptr;
        if (li + 1 < static_cast<int>(r.layers.size())) {
          RankLayer& N1 = r.layers[li + 1];
          if (N1.xin == Xin::kSame && N1.d.sdp == 1 && N1.sh.h == h) {
            nxt = &N1.acts[mb];
            PN = N1.pfull;
          }
        }
        GX_TRY(timed(kNorm, 0, (4.0 * sp + 8.0) * rows * h, [&] {
          return residual_layernorm(r.acc32, sp, static_cast<int64_t>(rows) * h, P + L.lay.b2.off,
                                    xr, A.y, d,
                                    nxt ? PN + r.layers[li + 1].lay.ln1g.off : nullptr,
                                    nxt ? PN + r.layers[li + 1].lay.ln1b.off : nullptr,
                                    nxt ? nxt->ln1 : nullptr, nxt ? nxt->mean1 : nullptr,
                                    nxt ? nxt->rstd1 : nullptr, rows, h, stream_);
        }));
        if (nxt != nullptr) nxt->ln1_ready = true;
        return kOk;
      }
      o.out = A.y;
      o.bias = P + L.lay.b2.off;
      o.residual = xr;
      o.ld_res = h;
      o.row_offset = row_off;
      o.drop_ld = h;
      o.drop_threshold = thr_hidden_;
      o.drop_scale = scale_of(p_hidden_);
      o.seed = seed_;
      o.site = 3ull * l + 2;
      o.seed_offset = r.seed_off;
      return gemm(A.gel, ft, false, P + L.lay.w2.off, ft, false, rows, h, ft, o);
    }
    o.out = r.partial;
    GX_TRY(gemm(A.gel, ft, false, P + L.lay.w2.off, ft, false, rows, h, ft, o));
    return c_all_reduce(kTpAllReduce, L.g_tp, r.rank, r.partial, static_cast<size_t>(rows) * h,
                             DType::kBF16, stream_);
  }
  if (t > 1 && phase == mlp_ph + 1) {
    gx_dropout d = hidden_drop(r, 3ull * l + 2, row_off, h);
    return timed(kElementwise, 0, 6.0 * rows * h, [&] {
      return bias_dropout_add(r.partial, P + L.lay.b2.off, xr, A.y, rows, h, d, stream_);
    });
  }
  return kOk;
}

// Decoder cross-attention sublayer, forward (tp == 1): x2 = x1 + drop(attn(q, k, v) Wo2 + bo2)
// with q = LN3(x1) Wq2 + bq2 and k, v = mem Wkv2 + bkv2, mem = the input of the model's first
// decoder layer (the encoder output).  q and kv are written side by side into one
// [rows][3h] buffer so the self-attention kernels serve unchanged (non-causal).
int ExecutorImpl::cross_fwd(RankCtx& r, int li, int mb, bool ln3_ready) {
  RankLayer& L = r.layers[li];
  Acts& A = L.acts[mb];
  const Shape& s = L.sh;
  const int rows = A.rows, h = s.h, t = L.d.tp, ht = h / t;
  const bf16* P = L.pfull;
  const int l = L.layer;
  const bf16* mem = r.mem(mb);
  if (!ln3_ready)
    GX_TRY(timed(kNorm, 0, 4.0 * rows * h, [&] {
      return layernorm_fwd(A.x1, P + L.lay.ln3g.off, P + L.lay.ln3b.off, A.ln3, A.mean3, A.rstd3,
                           rows, h, stream_);
    }));
  // (TP: this rank's heads -- q2 / kv2 column-parallel, the out-projection row-parallel)
  gx_gemm_epilogue e = epi();
  e.out_kind = kOutBF16;
  e.out = A.qkv2;
  e.ldo = 3 * ht;
  e.bias = P + L.lay.bq2.off;
  GX_TRY(gemm(A.ln3, h, false, P + L.lay.wq2.off, h, false, rows, ht, h, e));  // q2
  e.out = A.qkv2 + ht;
  e.bias = P + L.lay.bkv2.off;
  GX_TRY(gemm(mem, h, false, P + L.lay.wkv2.off, h, false, rows, 2 * ht, h, e));  // k2 v2
  gx_attention_args at = cross_args(r, L, A);
  GX_TRY(timed(kAttnFwd, 4.0 * A.samples * (s.heads / t) * double(s.seq) * s.seq * s.hd,
               2.0 * rows * 4 * ht, [&] { return attention_fwd(at, stream_); }));
  gx_gemm_epilogue o = epi();
  o.out_kind = kOutBF16;
  o.ldo = h;
  if (t > 1) {  // partial sums; the caller all-reduces and adds bias + dropout + residual
    o.out = r.partial;
    return gemm(A.ctx2, ht, false, P + L.lay.wo2.off, ht, false, rows, h, ht, o);
  }
  o.out = A.x2;
  o.bias = P + L.lay.bo2.off;
  o.residual = A.x1;
  o.ld_res = h;
  o.row_offset = A.sample0 * s.seq;
  o.drop_ld = h;
  o.drop_threshold = thr_hidden_;
  o.drop_scale = scale_of(p_hidden_);
  o.seed = seed_;
  o.site = 3ull * L_ + 2ull * l + 1;
  o.seed_offset = r.seed_off;
  return gemm(A.ctx2, h, false, P + L.lay.wo2.off, h, false, rows, h, h, o);
}

gx_attention_args ExecutorImpl::cross_args(RankCtx& r, const RankLayer& L, const Acts& A) const {
  const Shape& s = L.sh;
  const int t = L.d.tp;
  gx_attention_args at{};
  at.batch = A.samples;
  at.seq = s.seq;
  at.heads = s.heads / t;
  at.head_dim = s.hd;
  at.heads_total = s.heads;
  at.head_offset = L.tr * (s.heads / t);
  at.sample_offset = A.sample0;
  at.scale = 1.f / std::sqrt(static_cast<float>(s.hd));
  at.qkv = A.qkv2;
  at.ld_qkv = 3 * s.h / t;
  at.ctx = A.ctx2;
  at.ld_ctx = s.h / t;
  at.lse = A.lse2;
  at.drop_threshold = thr_attn_;
  at.drop_scale = scale_of(p_attn_);
  at.seed = seed_;
  at.site = 3ull * L_ + 2ull * L.layer;
  at.seed_offset = r.seed_off;
  at.mask = A.amask2;
  at.dq_accum = r.dq_acc;
  at.dsum = r.dsum;
  return at;
}

}  // namespace xi
}  // namespace gx
