// executor.cc — the plan executor (see executor.h for the contract and the reference
// semantics each piece follows).
//
// Execution model: a set of *local ranks* is driven in lockstep.  NCCL mode has exactly one
// local rank per process (one GPU each); sim mode places every rank of the world on this
// device and routes collectives through SimComm.  Each layer's forward/backward is split
// into phases that end at a collective, and the driver runs phase k for every local rank of
// the stage before phase k+1, so the same code path serves both modes.
#include "executor.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <functional>
#include <sstream>

#include <nlohmann/json.hpp>

#include "../kernels/gx_internal.h"
#include "parplan/strategy.h"

namespace gx {

using nlohmann::json;

namespace {

int64_t pad64(int64_t n) { return (n + 63) / 64 * 64; }

#define GX_TRY(expr)                 \
  do {                               \
    const int gx_rc_ = (expr);       \
    if (gx_rc_ != kOk) return gx_rc_; \
  } while (0)

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return kOk;
  return set_error(kErrCuda, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

}  // namespace

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

namespace {

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

// ------------------------------------------------------------------ device allocations
// Per-rank device arena with an optional byte cap (E15: the per-GPU memory budget E of the
// plan).  Exceeding the cap fails the allocation like an OOM.
class Arena {
 public:
  ~Arena() {
    for (void* p : ptrs_) cudaFree(p);
  }
  void set_cap(size_t cap) { cap_ = cap; }
  size_t cap() const { return cap_; }
  bool over_cap() const { return over_cap_; }
  void* alloc(size_t bytes) {
    if (bytes == 0) return nullptr;
    if (cap_ != 0 && bytes_ + bytes > cap_) {
      failed_ = over_cap_ = true;
      return nullptr;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, (bytes + 255) / 256 * 256) != cudaSuccess) {
      failed_ = true;
      return nullptr;
    }
    ptrs_.push_back(p);
    bytes_ += bytes;
    // GX_POISON=1 (debug): fill fresh allocations with NaN bit patterns, so a read of memory
    // the step never wrote shows up as a NaN instead of depending on what was there before
    static const bool poison = [] {
      const char* e = std::getenv("GX_POISON");
      return e != nullptr && e[0] == '1';
    }();
    if (poison) cudaMemset(p, 0xFF, (bytes + 255) / 256 * 256);
    return p;
  }
  template <typename T>
  T* a(int64_t n) {
    return static_cast<T*>(alloc(static_cast<size_t>(n) * sizeof(T)));
  }
  bool failed() const { return failed_; }
  size_t bytes() const { return bytes_; }

 private:
  std::vector<void*> ptrs_;
  size_t bytes_ = 0;
  size_t cap_ = 0;
  bool failed_ = false, over_cap_ = false;
};

using bf16 = __nv_bfloat16;

struct Acts {
  int64_t sample0 = 0;  // first global sample of this chunk (within the iteration)
  int samples = 0;
  int rows = 0;  // samples * seq
  bf16 *x = nullptr, *ln1 = nullptr, *qkv = nullptr, *ctx = nullptr, *x1 = nullptr,
       *ln2 = nullptr, *pre = nullptr, *gel = nullptr, *y = nullptr;
  float *lse = nullptr, *mean1 = nullptr, *rstd1 = nullptr, *mean2 = nullptr, *rstd2 = nullptr;
  uint16_t* amask = nullptr;  // attention dropout keep bits (fwd -> bwd)
  // patch merging (Shape::merge): xm = layer input [4*rows][h/2], mg = gathered [rows][2h],
  // mln = LayerNorm(mg); x = mln Wm^T is then the residual-stream input of the block
  bf16 *xm = nullptr, *mg = nullptr, *mln = nullptr;
  float *meanm = nullptr, *rstdm = nullptr;
  bf16* in() const { return xm != nullptr ? xm : x; }  // what the previous layer feeds
  bf16 *ln1r = nullptr, *ctxr = nullptr;  // SW-MSA: LN1 output / context in rolled order
  // decoder cross-attention sublayer: x2 = x1 + drop(attn(LN3(x1) Wq2, mem Wkv2) Wo2 + bo2)
  bf16 *x2 = nullptr, *ln3 = nullptr, *qkv2 = nullptr, *ctx2 = nullptr;
  float *lse2 = nullptr, *mean3 = nullptr, *rstd3 = nullptr;
  uint16_t* amask2 = nullptr;
  bool ln1_ready = false;     // LN1 already produced by the previous layer's fused epilogue
  bool dz_ready = false;      // backward: dz / db2 already produced by the next layer's LN1 bwd
};

enum class Xin { kSame, kSlice, kGather, kStageInput };

struct RankLayer {
  int layer = 0;  // global layer id
  Shape sh;
  Deg d;
  int tr = 0, dr = 0, sr = 0, pr = 0;
  int g_tp = -1, g_sdp = -1, g_dp = -1, g_xin = -1;  // group ids (-1: none)
  Xin xin = Xin::kStageInput;
  Layout lay;
  int64_t shard_n = 0;
  float *master = nullptr, *m = nullptr, *v = nullptr, *gfull = nullptr, *gshard = nullptr;
  bf16 *pshard = nullptr, *pfull = nullptr;
  int8_t* relb_map = nullptr;  // T5: bucket of each relative position k - q + seq - 1
  std::vector<Acts> acts;  // per micro-batch
};

// T5's relative-position bucket of d = k - q (the published bucketing; pinned against
// transformers' T5Attention in tests/test_layer_oracle.py), bidirectional unless causal,
// max distance 128, computed in double as oracle/layer_oracle.py::t5_buckets does.
static std::vector<int8_t> t5_bucket_map(int seq, bool bidirectional, int buckets) {
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

struct RankCtx {
  int rank = 0, stage = 0, idx = 0;
  std::vector<RankLayer> layers;  // this stage's layers in order
  Arena arena;
  // scratch
  bf16 *partial = nullptr, *dx1 = nullptr, *dctx = nullptr, *da = nullptr;
  // Gradients the weight-gradient GEMMs read, double-buffered by layer parity: layer l's
  // wgrads run on the wgrad stream while layer l-1's data-gradient chain writes the other
  // buffer.  wg_done[p] marks the last wgrad that read buffer set p.
  bf16 *dzb[2] = {nullptr, nullptr}, *dpreb[2] = {nullptr, nullptr},
       *doutb[2] = {nullptr, nullptr}, *dqkvb[2] = {nullptr, nullptr};
  float* lnfold[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [parity][LN2, LN1] fp32 dy
  cudaEvent_t wg_done[2] = {nullptr, nullptr};
  bool wg_pending[2] = {false, false};
  bf16* gbuf[2] = {nullptr, nullptr};
  float *dq_acc = nullptr, *dsum = nullptr;
  float* ln_ws = nullptr;  // LayerNorm-backward block partials
  float* ln_ws_m = nullptr;  // ... for the patch-merging LayerNorm (main stream only)
  float* ln_ws_x = nullptr;  // ... for the decoder's LN3 (main stream only)
  bf16 *dmg1 = nullptr, *dmg2 = nullptr;  // patch-merging backward scratch [rows][2h]
  // decoder backward: the cross sublayer's dropout-masked output gradient, its dqkv, and the
  // memory gradient accumulated over the decoder layers (fp32, added to the first decoder
  // layer's input gradient)
  bf16 *dout2 = nullptr, *dqkv2 = nullptr;
  bf16 *dctxr = nullptr, *rollbuf = nullptr;  // SW-MSA backward scratch (rolled dctx, da)
  float* rpb_part = nullptr;  // relative-position bias: per-(window, head) score gradients
  float* relb_part = nullptr;  // T5 bias: per-(sequence x head, key block) relative-position sums
  float* dmem = nullptr;
  int dec_li = -1;  // local index of the model's first decoder layer on this rank, or -1
  // stages after the first decoder layer's: the memory received with each micro-batch's
  // activations, and whether dL/dmem arrives from the next (decoder) stage in backward
  std::vector<bf16*> mem_in;
  bool dmem_from_next = false;
  const bf16* mem(int mb) const {
    return dec_li >= 0 ? layers[dec_li].acts[mb].x : mem_in[mb];
  }
  float* cs_ws[2] = {nullptr, nullptr};  // column-sum workspaces: [0] main stream, [1] wgrad stream
  float* acc32 = nullptr;  // split-K fp32 slices [kMaxSplits][rows][h]
  bf16 *x_in = nullptr, *target = nullptr;  // [m micro-batches of this rank's rows][h]
  bf16* dx_out = nullptr;                   // first stage: input gradient per micro-batch
  // stages > 0: the input gradient (and dL/dmemory) each backward micro-batch sends to the
  // previous stage, copied out of the ping-pong gradient buffers so the send (on the pipeline
  // stream) overlaps the next micro-batch's backward instead of fencing it
  bf16* pp_dx_send = nullptr;
  float* pp_dmem_send = nullptr;
  float *loss = nullptr, *loss_dummy = nullptr;
  float* loss_ws = nullptr;  // deterministic loss reduction: block partials + ticket
  std::vector<cudaEvent_t> gath_ev;   // SDP parameter all-gather of layer li done (prefetch)
  int64_t* step = nullptr;
  uint64_t* seed_off = nullptr;
  int64_t in_rows_total = 0;
  std::vector<int64_t> in_row_off;  // per micro-batch offset (rows) into x_in / target
  int cur = 0;                      // index of gbuf holding the current dY
  bool idle_chunks = false;  // some (layer, micro-batch) chunk of this rank has no samples:
                             // gradients are zeroed whole each step and always accumulated
  int dc_slices = 0, da_slices = 0;  // fp32 slices pending in acc32 (da: 0 = bf16 in r.da)
};

// --------------------------------------------------------------------------------------
float scale_of(float p);  // dropout keep-scale for probability p (defined below)

class ExecutorImpl final : public Executor {
 public:
  int init(const json& cfg, std::string* err);
  int set_layer_params(int layer, const float* canonical, int64_t n) override;
  int export_layer(int layer, int what, float* canonical, int64_t n) override;
  int load_batch(const void* x_host, const void* target_host) override;
  int load_batch_device(const void* x_dev, const void* target_dev) override;
  int run(bool use_graph) override { return run2(use_graph, false); }
  int run2(bool use_graph, bool profile) override;
  int loss(float* out) override;
  int sync(int64_t timeout_ms) override;
  int export_output(void* host_bf16, int what) override;
  cudaStream_t stream() const override { return stream_; }
  std::string info() const override;
  ~ExecutorImpl() override {
    if (graph_exec_ != nullptr) cudaGraphExecDestroy(graph_exec_);
    if (graph_ != nullptr) cudaGraphDestroy(graph_);
    if (pgraph_exec_ != nullptr) cudaGraphExecDestroy(pgraph_exec_);
    if (pgraph_ != nullptr) cudaGraphDestroy(pgraph_);
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
    for (auto& t : tr_) cudaEventDestroy(t.second);
    for (cudaEvent_t e : fork_events_) cudaEventDestroy(e);
    if (join_event_ != nullptr) cudaEventDestroy(join_event_);
    for (auto& r : ranks_) {
      for (cudaEvent_t e : r->wg_done)
        if (e != nullptr) cudaEventDestroy(e);
      for (cudaEvent_t e : r->gath_ev)
        if (e != nullptr) cudaEventDestroy(e);
    }
    ranks_.clear();
    comm_.reset();
    if (stream_ != nullptr) cudaStreamDestroy(stream_);
    if (side_ != nullptr) cudaStreamDestroy(side_);
    if (cs_ != nullptr) cudaStreamDestroy(cs_);
    if (pp_ != nullptr) cudaStreamDestroy(pp_);
    if (wg_ != nullptr) cudaStreamDestroy(wg_);
  }

 private:
  // topology helpers
  int stage_of_layer(int l) const {
    for (int s = 0; s < P_; ++s)
      if (l >= stage_range_[s].first && l < stage_range_[s].second) return s;
    return -1;
  }
  void chunk(const Deg& d, int idx, int mb, int64_t& lo, int64_t& hi) const {
    const int t = d.tp, D = d.data();
    const int c = idx / t;
    const int64_t base = static_cast<int64_t>(mb) * Bm_;
    lo = base + static_cast<int64_t>(c) * Bm_ / D;
    hi = base + static_cast<int64_t>(c + 1) * Bm_ / D;
  }
  int build_groups();
  int allocate(RankCtx& r);
  int step_once();

  // per-phase work
  int fwd_phase(RankCtx& r, int li, int mb, int phase);
  int bwd_phase(RankCtx& r, int li, int mb, int phase);
  int merge_bwd(RankCtx& r, RankLayer& L, Acts& A, bf16* dX, const gx_gemm_epilogue& wm_ep);
  // phases of a layer's forward / backward: TP splits them at its all-reduces (a decoder's
  // cross sublayer adds one)
  int tp_phases(const RankLayer& L) const {
    return L.d.tp > 1 ? (L.sh.cross ? 4 : 3) : 1;
  }
  int tp_bwd_phases(const RankLayer& L) const {
    return L.d.tp > 1 ? (L.sh.cross ? (L.layer == dec0_ ? 5 : 4) : 3) : 1;
  }
  gx_dropout hidden_drop(const RankCtx& r, uint64_t site, int64_t row_off, int ld) const {
    gx_dropout d{};
    d.threshold = thr_hidden_;
    d.scale = scale_of(p_hidden_);
    d.seed = seed_;
    d.site = site;
    d.row_offset = row_off;
    d.drop_ld = ld;
    d.seed_offset = r.seed_off;
    return d;
  }
  static int grid_of(const Shape& s) {
    return static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.seq))));
  }
  static int side_of(const Shape& s) {
    return static_cast<int>(std::lround(std::sqrt(static_cast<double>(s.win))));
  }
  static void set_window_mask(gx_attention_args& at, const Shape& s) {
    if (s.shift > 0) {
      at.win_grid = grid_of(s);
      at.win_side = side_of(s);
      at.win_shift = s.shift;
    }
  }
  int cross_fwd(RankCtx& r, int li, int mb, bool ln3_ready);
  int cross_bwd_attn(RankCtx& r, int li, int mb,
                     const std::function<gx_gemm_epilogue(const Slot&, int64_t)>& wgrad_ep);
  int cross_bwd_ln3(RankCtx& r, int li, int mb, bf16* dout);
  gx_attention_args cross_args(RankCtx& r, const RankLayer& L, const Acts& A) const;
  int sync_phase(RankCtx& r, int li, int phase);
  int xin_fwd(RankCtx& r, int li, int mb);
  int xin_bwd(RankCtx& r, int li, int mb);
  int gather_params(RankCtx& r, int li, cudaStream_t st);
  bool prefetched_ = false;  // the current layer's SDP gather was prefetched on cs_
  int pp_fwd(RankCtx& r, int mb, bool send, cudaStream_t st);
  int pp_bwd(RankCtx& r, int mb, bool send, cudaStream_t st);
  // One pipeline-boundary exchange of every rank in R on the pipeline stream pp_ (E12/E13):
  // forked after the producer's work on stream_; receives are joined back before the
  // consumer runs, sends (of activations / private gradient copies that nothing overwrites
  // within the step) only at the step end.
  int pp_exchange(const std::vector<RankCtx*>& R, int mb, bool fwd, bool send) {
    const bool side = pp_ != nullptr && !profiling_;
    cudaStream_t st = side ? pp_ : stream_;
    if (side) GX_TRY(fork(stream_, pp_));
    double bytes = 0;  // rows this exchange moves (send or receive side), bf16
    for (RankCtx* r : R) {
      const bool out = fwd == send;  // the stage's output rows (else its input rows)
      const RankLayer& L = out ? r->layers.back() : r->layers.front();
      const double hs = out ? 1.0 * L.sh.seq * L.sh.h : 1.0 * L.sh.in_seq() * L.sh.in_h();
      for (const Xfer& x : pp_plan(r->stage, r->idx, mb, fwd ? (send ? 0 : 1) : (send ? 2 : 3)))
        bytes += 2.0 * hs * static_cast<double>(x.hi - x.lo);
    }
    return timed(kComm, 0, bytes, [&]() -> int {
      GX_TRY(comm_->group_start());
      for (RankCtx* r : R) GX_TRY(fwd ? pp_fwd(*r, mb, send, st) : pp_bwd(*r, mb, send, st));
      GX_TRY(comm_->group_end());
      if (side) {
        pp_used_ = true;
        if (!send) GX_TRY(fork(pp_, stream_));
      }
      return kOk;
    }, kPpSendRecv, bytes);
  }
  cudaStream_t pp_ = nullptr;
  bool pp_used_ = false;
  struct Xfer {
    int peer;
    int64_t lo, hi;  // global sample range within the iteration
  };
  std::vector<Xfer> pp_plan(int stage, int idx, int mb, int kind) const;

 public:
  std::string topology() const override;

 private:

  // ------------------------------------------------------------ kernel profiler
  // Categories of launched work; every launch site goes through timed(), which (when
  // profiling) brackets it with CUDA events on the executor stream.  Inside graph capture
  // the events become external event-record nodes, so a replay of the instrumented graph
  // yields per-launch device durations of exactly the kernels the plain graph runs.
  enum Cat { kGemm, kAttnFwd, kAttnBwd, kNorm, kElementwise, kOptim, kComm, kNumCats };
  // collective classes of the plan, reported with their NCCL bus bytes
  enum CommKind { kTpAllReduce, kSdpAllGather, kSdpReduceScatter, kDpAllReduce, kRelayout,
                  kPpSendRecv, kNumCommKinds };
  struct Rec {
    int cat;
    double flops, bytes;
    cudaEvent_t a, b;
    int kind = -1;      // CommKind of a kComm record
    double bus = 0.0;   // NCCL bus bytes (ring convention, cost_model.cc:97-117)
  };
  template <class F>
  int timed(int cat, double flops, double bytes, F&& f, int kind = -1, double bus = 0.0) {
    if (!profiling_) return f();
    cudaEvent_t a = next_event(), b = next_event();
    record_event(a);
    const int rc = f();
    record_event(b);
    recs_.push_back(Rec{cat, flops, bytes, a, b, kind, bus});
    return rc;
  }
  cudaEvent_t next_event() {
    if (ev_used_ == events_.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      events_.push_back(e);
    }
    return events_[ev_used_++];
  }
  void record_event(cudaEvent_t e) {
    if (capturing_)
      cudaEventRecordWithFlags(e, stream_, cudaEventRecordExternal);
    else
      cudaEventRecord(e, stream_);
  }
  int c_all_reduce(int kind, int g, int rank, void* buf, size_t n, DType t, cudaStream_t st) {
    const double d = static_cast<double>(comm_->group(g).ranks.size());
    const double bytes = 1.0 * n * dtype_bytes(t);
    return timed(kComm, 0, 2.0 * bytes, [&] { return comm_->all_reduce(g, rank, buf, n, t, st); },
                 kind, 2.0 * (d - 1.0) / d * bytes);
  }
  int c_reduce_scatter(int kind, int g, int rank, const void* a, void* b, size_t n, DType t,
                       cudaStream_t st) {
    const double d = static_cast<double>(comm_->group(g).ranks.size());
    const double bytes = 1.0 * n * dtype_bytes(t) * d;
    return timed(kComm, 0, bytes,
                 [&] { return comm_->reduce_scatter(g, rank, a, b, n, t, st); }, kind,
                 (d - 1.0) / d * bytes);
  }
  int c_all_gather(int kind, int g, int rank, const void* a, void* b, const std::vector<size_t>& c,
                   DType t, cudaStream_t st) {
    size_t n = 0;
    for (size_t x : c) n += x;
    const double d = static_cast<double>(comm_->group(g).ranks.size());
    const double bytes = 1.0 * n * dtype_bytes(t);
    return timed(kComm, 0, bytes, [&] { return comm_->all_gather(g, rank, a, b, c, t, st); },
                 kind, (d - 1.0) / d * bytes);
  }
  // Split-K into r.acc32 (fp32 slices [splits][M][N], summed in order by the consumer) when
  // it pays (small M*N, long K); *used = split count, 1 meaning "not split" (nothing launched).
  int gemm_splitk(RankCtx& r, const void* a, int64_t lda, const void* b, int64_t ldb, bool bmn,
                  int M, int N, int K, int* used) {
    *used = 1;
    // below ~2K of K the un-split GEMM with its fused epilogue wins (measured at M = 512:
    // out-projection K = 1280 split + row pass 19.8 us vs fused 10.4 + LayerNorm 5.5 us)
    if (!splitk_ || K < 2048) return kOk;
    int tile = 0;
    const int sp = splitk_plan(M, N, K, &tile);
    if (sp < 2) return kOk;
    gx_gemm_epilogue e{};
    e.alpha = 1.f;
    e.drop_scale = 1.f;
    e.out_kind = kOutF32Split;
    e.out = r.acc32;
    e.ldo = N;
    const double flops = 2.0 * M * N * K;
    const double bytes = 2.0 * (static_cast<double>(M) * K + static_cast<double>(N) * K) + 4.0 * M * N;
    GX_TRY(timed(kGemm, flops, bytes, [&] {
      return gemm_bf16(GemmOperand{a, lda, false}, GemmOperand{b, ldb, bmn}, M, N, K, e, stream_,
                       tile, sp);
    }));
    *used = sp;
    return kOk;
  }
  int gemm(const void* a, int64_t lda, bool amn, const void* b, int64_t ldb, bool bmn, int M, int N,
           int K, const gx_gemm_epilogue& ep) {
    const double flops = 2.0 * M * N * K;
    const double bytes = 2.0 * (static_cast<double>(M) * K + static_cast<double>(N) * K) +
                         (ep.out_kind == kOutBF16 ? 2.0 : 4.0) * M * N;
    return timed(kGemm, flops, bytes, [&] {
      return gemm_bf16(GemmOperand{a, lda, amn}, GemmOperand{b, ldb, bmn}, M, N, K, ep, ls_);
    });
  }
 public:
  std::string profile_report() const override;
  int init_params(uint64_t seed, float std_dev) override;
 private:
  gx_gemm_epilogue epi() const {
    gx_gemm_epilogue e{};
    e.alpha = 1.f;
    e.drop_scale = 1.f;
    return e;
  }
  // config
  json plan_, model_;
  int world_ = 1, P_ = 1, g_ = 1, m_ = 1, B_ = 1, Bm_ = 1, L_ = 0;
  std::vector<std::pair<int, int>> stage_range_;
  std::vector<Deg> deg_;
  std::vector<Shape> shape_;
  bool sim_ = true;
  std::string comm_kind_ = "sim";
  float p_attn_ = 0.f, p_hidden_ = 0.f;
  uint32_t thr_attn_ = 0, thr_hidden_ = 0;
  uint64_t seed_ = 1234;
  float lr_ = 1e-4f, b1_ = 0.9f, b2_ = 0.999f, eps_ = 1e-8f, wd_ = 0.f;
  bool optimizer_ = true;
  bool forward_only_ = false;  // profiler / debugging: skip loss, backward and optimizer
  bool splitk_ = true;         // split-K for long-K / small-MN GEMMs (cfg "splitk")
  int64_t mem_cap_ = 0;  // per-rank device-byte cap (cfg "memory_cap_bytes"; 0 = none)
  int64_t sync_timeout_ms_ = 600000;  // loss() / step(): watchdog limit (cfg "sync_timeout_ms")
  int dec0_ = -1;         // first decoder (cross-attention) layer, or -1
  bool dry_run_ = false;       // topology only: no device state (host-logic tests)
  float inv_count_ = 1.f;

  std::unique_ptr<Comm> comm_;
  std::vector<std::unique_ptr<RankCtx>> ranks_;
  cudaStream_t stream_ = nullptr;
  // AdamW of layer l runs on side_ while layer l-1's backward runs on stream_ (HBM-bound
  // optimizer under tensor-bound GEMMs); joined back before the step ends.
  cudaStream_t side_ = nullptr;
  // Gradient collectives (DP all-reduce, SDP reduce-scatter) of layer l run on cs_ beside
  // layer l-1's backward (the overlap EstimateLayerCost models, cost_model.cc:200-206); the
  // optimizer of layer l waits for them.  comm_stream_ = false keeps them on stream_.
  cudaStream_t cs_ = nullptr;
  bool comm_stream_ = true, cs_used_ = false;
  std::vector<char> synced_on_cs_;  // per local layer index: this step's sync ran on cs_
  bool comm_on_cs() const { return comm_stream_ && !profiling_ && cs_ != nullptr; }
  // Weight-gradient GEMMs (and the bias column sums) of the backward run on wg_, forked
  // from stream_ as soon as their inputs exist, so they fill the SMs the data-gradient
  // chain (the critical path) leaves idle.  ls_ is the stream gemm() launches on.
  cudaStream_t wg_ = nullptr;
  cudaStream_t ls_ = nullptr;
  bool wgrad_stream_ = true;  // cfg "wgrad_stream": false keeps the wgrads on stream_
  bool fuse_dz_ = false;      // previous layer's dropout bwd inside LN1 bwd (cfg "fuse_dz")
  // AdamW of each layer runs on the side stream as a resident grid of 2 blocks per SM
  // (64-register blocks): enough HBM parallelism without crowding the backward's GEMMs off
  // their SMs (DESIGN.md §7.2 lists the placements measured and rejected).
  // gradient bytes cleared before a step: the atomically accumulated head of the buffer, or
  // all of it when some chunk of the rank is empty (its weight-gradient GEMMs may not run)
  static size_t grad_zero_bytes(const RankCtx& r, const RankLayer& L) {
    return static_cast<size_t>(r.idle_chunks ? L.lay.total : L.lay.acc_end) * 4;
  }
  bool wg_active_ = false;    // this capture forks (off while profiling)
  bool wg_used_ = false;
  int fork(cudaStream_t from, cudaStream_t to) {
    if (fork_events_.size() <= static_cast<size_t>(fork_used_)) {
      cudaEvent_t e;
      GX_TRY(cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event"));
      fork_events_.push_back(e);
    }
    cudaEvent_t e = fork_events_[fork_used_++];
    GX_TRY(cuda_check(cudaEventRecord(e, from), "fork record"));
    return cuda_check(cudaStreamWaitEvent(to, e, 0), "fork wait");
  }
  // Runs f with launches on the wgrad stream (after everything already on stream_).
  template <class F>
  int on_wgrad(F&& f) {
    if (!wg_active_) return f();
    GX_TRY(fork(stream_, wg_));
    wg_used_ = true;
    ls_ = wg_;
    const int rc = f();
    ls_ = stream_;
    return rc;
  }
  std::vector<cudaEvent_t> fork_events_;
  cudaEvent_t join_event_ = nullptr;
  // Eager-mode timeline (cfg "trace"): timing events recorded on the stream each mark names,
  // reported by profile_report() as ms since the step's first mark.
  bool trace_ = false;
  std::vector<std::pair<std::string, cudaEvent_t>> tr_;
  size_t tr_used_ = 0;
  void tmark(const std::string& name, cudaStream_t st) {
    if (!trace_ || capturing_) return;
    if (tr_used_ == tr_.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      tr_.push_back({name, e});
    }
    tr_[tr_used_].first = name;
    cudaEventRecord(tr_[tr_used_].second, st);
    ++tr_used_;
  }
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  cudaGraph_t pgraph_ = nullptr;  // instrumented (profiling) variant
  cudaGraphExec_t pgraph_exec_ = nullptr;
  bool profiling_ = false, capturing_ = false;
  int fork_used_ = 0;
  bool side_used_ = false;
  std::vector<cudaEvent_t> events_;
  size_t ev_used_ = 0;
  std::vector<Rec> recs_, prof_recs_;
  double last_profile_ms_ = 0;
  int64_t steps_run_ = 0;
  int64_t launches_per_step_ = 0;
};

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
    fuse_dz_ = cfg.value("fuse_dz", false);
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
  r.dq_acc = A.a<float>(4 * max_c);  // tcgen05 attention: one dQ partial per 128-key tile
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
    if (!A.dz_ready)
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
    // When this layer's input is the previous layer's output (same rows), the previous
    // layer's MLP dropout backward rides along: dz_{l-1} = dropout_mask(dX), db2_{l-1} +=
    // colsum(dz_{l-1}) -- its phase 0 then starts straight at the GEMMs.
    Acts* prev = nullptr;
    RankLayer* Lp = nullptr;
    if (fuse_dz_ && li > 0 && L.xin == Xin::kSame && r.layers[li - 1].sh.h == h) {
      Lp = &r.layers[li - 1];
      prev = &Lp->acts[mb];
    }
    gx_dropout dp{};
    bf16* dz_prev = nullptr;
    if (prev != nullptr) {
      const int pp = (li - 1) & 1;
      if (r.wg_pending[pp]) {  // that parity's buffers are free once their wgrads are done
        GX_TRY(cuda_check(cudaStreamWaitEvent(stream_, r.wg_done[pp], 0), "wgrad wait"));
        r.wg_pending[pp] = false;
      }
      dp.threshold = thr_hidden_;
      dp.scale = scale_of(p_hidden_);
      dp.seed = seed_;
      dp.site = 3ull * Lp->layer + 2;
      dp.row_offset = prev->sample0 * Lp->sh.seq;
      dp.drop_ld = h;
      dp.seed_offset = r.seed_off;
      dz_prev = r.dzb[pp];
    }
    float* fold1 = r.lnfold[par][1];
    GX_TRY(timed(kNorm, 0, 8.0 * rows * h, [&] { return layernorm_bwd_rows(da_in, A.x, A.mean1, A.rstd1, P + L.lay.ln1g.off, r.dx1, dX,
                         rows, h, stream_, r.da_slices > 0, prev ? &dp : nullptr, dz_prev,
                         std::max(1, r.da_slices), static_cast<int64_t>(rows) * h, fold1); }));
    GX_TRY(on_wgrad([&]() -> int {
      GX_TRY(timed(kNorm, 0, 8.0 * rows * h, [&] { return layernorm_bwd_cols(fold1, true, A.x, A.mean1, A.rstd1, dz_prev,
                           G + L.lay.ln1g.off, G + L.lay.ln1b.off, prev ? Lp->gfull + Lp->lay.b2.off : nullptr,
                           rows, h, r.ln_ws, ls_); }));
      if (wg_active_) {  // the last reader of this parity's buffers
        GX_TRY(cuda_check(cudaEventRecord(r.wg_done[par], wg_), "wgrad done"));
        r.wg_pending[par] = true;
      }
      return kOk;
    }));
    if (prev != nullptr) prev->dz_ready = true;
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
      for (Acts& a : L.acts) a.ln1_ready = a.dz_ready = false;
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

}  // namespace

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
  auto ex = std::make_unique<ExecutorImpl>();
  const int rc = ex->init(cfg, err);
  if (rc != kOk) {
    if (code != nullptr) *code = rc;
    return nullptr;
  }
  return ex;
}

}  // namespace gx
