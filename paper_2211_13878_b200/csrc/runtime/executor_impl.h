// executor_impl.h -- internals of the plan executor, shared by its translation units:
//   executor.cc       configuration, parameter layouts, communicator groups, topology / info
//   exec_memory.cc    device arena and buffers, parameters in / out, batches, outputs
//   exec_forward.cc   forward phases (self-attention, cross-attention, MLP)
//   exec_backward.cc  backward phases (data gradients; weight gradients on the wgrad stream)
//   exec_comm.cc      gradient collectives + optimizer, SDP gathers, relayouts, pipeline
//   exec_step.cc      the step driver (GPipe schedule, streams, CUDA graph), timing, reports
#pragma once
#include "executor.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <thread>

#include <nlohmann/json.hpp>

#include "../kernels/gx_internal.h"
#include "parplan/strategy.h"

#define GX_TRY(expr)                  \
  do {                                \
    const int gx_rc_ = (expr);        \
    if (gx_rc_ != kOk) return gx_rc_; \
  } while (0)

namespace gx {
namespace xi {

using nlohmann::json;

inline int64_t pad64(int64_t n) { return (n + 63) / 64 * 64; }

inline int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return kOk;
  return set_error(kErrCuda, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

// Canonical index of local flat element `j` of rank (tp degree t, tp index tr); -1 = padding.
int64_t canon_index(const Shape& s, const Layout& L, int t, int tr, int64_t j);
// T5 relative-attention bucket of every relative position (executor.cc)
std::vector<int8_t> t5_bucket_map(int seq, bool bidirectional, int buckets);
uint32_t threshold_of(float p);  // dropout byte threshold of probability p (executor.cc)

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
    const int sp = splitk_plan(M, N, K, &tile, bmn);
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

}  // namespace xi
}  // namespace gx
