// comm.cc — SimComm (single-device simulated world) and NcclComm (one rank per GPU).
#include "comm.h"

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstring>
#include <deque>

#include "../kernels/gx_internal.h"

namespace gx {

int Comm::add_group(std::vector<int> ranks) {
  std::sort(ranks.begin(), ranks.end());
  for (size_t i = 0; i < groups_.size(); ++i)
    if (groups_[i].ranks == ranks) return static_cast<int>(i);
  groups_.push_back(CommGroup{std::move(ranks)});
  return static_cast<int>(groups_.size()) - 1;
}

namespace {

int cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return kOk;
  return set_error(kErrCuda, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

// =================================================================== simulated world
class SimComm final : public Comm {
 public:
  explicit SimComm(int world) : world_(world) {}

  int finalize() override { return kOk; }

  int all_reduce(int gid, int rank, void* buf, size_t count, DType t, cudaStream_t s) override {
    Pending& p = post(gid, rank, Kind::kAllReduce);
    p.recv[p.me] = buf;
    p.count = count;
    if (!complete(p, gid)) return kOk;
    PtrPack pk{};
    pk.n = static_cast<int>(p.recv.size());
    for (int j = 0; j < pk.n; ++j) pk.p[j] = p.recv[j];
    int rc = sum_ptrs(pk, p.recv[0], static_cast<int64_t>(count), t == DType::kBF16, s);
    for (size_t j = 1; j < p.recv.size() && rc == kOk; ++j)
      rc = cuda_ok(cudaMemcpyAsync(p.recv[j], p.recv[0], count * dtype_bytes(t),
                                   cudaMemcpyDeviceToDevice, s),
                   "sim all_reduce copy");
    pending_.erase(gid);
    return rc;
  }

  int reduce_scatter(int gid, int rank, const void* send, void* recv, size_t count, DType t,
                     cudaStream_t s) override {
    Pending& p = post(gid, rank, Kind::kReduceScatter);
    p.send[p.me] = send;
    p.recv[p.me] = recv;
    p.count = count;
    if (!complete(p, gid)) return kOk;
    const int n = static_cast<int>(p.send.size());
    int rc = kOk;
    for (int j = 0; j < n && rc == kOk; ++j) {
      PtrPack pk{};
      pk.n = n;
      for (int i = 0; i < n; ++i)
        pk.p[i] = static_cast<const char*>(p.send[i]) + j * count * dtype_bytes(t);
      rc = sum_ptrs(pk, p.recv[j], static_cast<int64_t>(count), t == DType::kBF16, s);
    }
    pending_.erase(gid);
    return rc;
  }

  int all_gather(int gid, int rank, const void* send, void* recv,
                 const std::vector<size_t>& counts, DType t, cudaStream_t s) override {
    Pending& p = post(gid, rank, Kind::kAllGather);
    p.send[p.me] = send;
    p.recv[p.me] = recv;
    p.counts = counts;
    if (!complete(p, gid)) return kOk;
    const int n = static_cast<int>(p.send.size());
    const size_t eb = dtype_bytes(t);
    int rc = kOk;
    size_t displ = 0;
    for (int j = 0; j < n && rc == kOk; ++j) {
      for (int i = 0; i < n && rc == kOk; ++i) {
        if (p.counts[j] == 0) continue;
        if (static_cast<const char*>(p.recv[i]) + displ * eb == p.send[j]) continue;
        rc = cuda_ok(cudaMemcpyAsync(static_cast<char*>(p.recv[i]) + displ * eb, p.send[j],
                                     p.counts[j] * eb, cudaMemcpyDeviceToDevice, s),
                     "sim all_gather copy");
      }
      displ += p.counts[j];
    }
    pending_.erase(gid);
    return rc;
  }

  int send(int rank, int peer, const void* buf, size_t bytes, cudaStream_t s) override {
    auto& q = p2p_[{rank, peer}];
    if (!q.recvs.empty()) {
      void* dst = q.recvs.front();
      q.recvs.pop_front();
      return cuda_ok(cudaMemcpyAsync(dst, buf, bytes, cudaMemcpyDeviceToDevice, s), "sim p2p");
    }
    q.sends.push_back({buf, bytes});
    return kOk;
  }

  int recv(int rank, int peer, void* buf, size_t bytes, cudaStream_t s) override {
    auto& q = p2p_[{peer, rank}];
    if (!q.sends.empty()) {
      const auto [src, n] = q.sends.front();
      q.sends.pop_front();
      if (n != bytes) return set_error(kErrConfig, "sim p2p: size mismatch");
      return cuda_ok(cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToDevice, s), "sim p2p");
    }
    q.recvs.push_back(buf);
    return kOk;
  }

  int world_sum(int rank, float* v, cudaStream_t s) override {
    (void)rank;
    scalars_.push_back(v);
    if (static_cast<int>(scalars_.size()) < world_) return kOk;
    PtrPack pk{};
    int rc = kOk;
    // world may exceed 16: fold in chunks into scalars_[0]
    size_t i = 1;
    while (i < scalars_.size() && rc == kOk) {
      pk.n = 1;
      pk.p[0] = scalars_[0];
      while (i < scalars_.size() && pk.n < 16) pk.p[pk.n++] = scalars_[i++];
      rc = sum_ptrs(pk, scalars_[0], 1, false, s);
    }
    for (size_t j = 1; j < scalars_.size() && rc == kOk; ++j)
      rc = cuda_ok(cudaMemcpyAsync(scalars_[j], scalars_[0], 4, cudaMemcpyDeviceToDevice, s),
                   "sim world_sum");
    scalars_.clear();
    return rc;
  }

 private:
  enum class Kind { kAllReduce, kReduceScatter, kAllGather };
  struct Pending {
    Kind kind;
    int posted = 0;
    int me = 0;
    size_t count = 0;
    std::vector<size_t> counts;
    std::vector<const void*> send;
    std::vector<void*> recv;
  };

  Pending& post(int gid, int rank, Kind k) {
    auto it = pending_.find(gid);
    if (it == pending_.end()) {
      Pending p;
      p.kind = k;
      const size_t n = groups_[gid].ranks.size();
      p.send.assign(n, nullptr);
      p.recv.assign(n, nullptr);
      it = pending_.emplace(gid, std::move(p)).first;
    }
    Pending& p = it->second;
    p.me = groups_[gid].index_of(rank);
    p.posted += 1;
    return p;
  }
  bool complete(const Pending& p, int gid) const {
    return p.posted == static_cast<int>(groups_[gid].ranks.size());
  }

  struct Queue {
    std::deque<std::pair<const void*, size_t>> sends;
    std::deque<void*> recvs;
  };
  int world_;
  std::map<int, Pending> pending_;
  std::map<std::pair<int, int>, Queue> p2p_;
  std::vector<float*> scalars_;
};

// ======================================================================== NCCL world
ncclDataType_t nccl_type(DType t) { return t == DType::kBF16 ? ncclBfloat16 : ncclFloat32; }

class NcclComm final : public Comm {
 public:
  NcclComm(int world, int rank, const NcclOptions& opt)
      : world_size_(world), rank_(rank), opt_(opt) {}
  ~NcclComm() override {
    for (ncclComm_t c : comms_)
      if (c != nullptr) ncclCommDestroy(c);
    if (world_ != nullptr) ncclCommDestroy(world_);
  }

  // Nonblocking communicators: creation returns at once and is polled with a deadline, so a
  // rank whose peers never arrive fails with an error instead of hanging the job.
  int init(const std::string& id_bytes, std::string* err) {
    ncclUniqueId id;
    if (id_bytes.size() != sizeof(id.internal)) {
      *err = "nccl: unique id must be 128 bytes";
      return kErrConfig;
    }
    std::memcpy(id.internal, id_bytes.data(), sizeof(id.internal));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    if (opt_.min_ctas > 0) cfg.minCTAs = opt_.min_ctas;
    if (opt_.max_ctas > 0) cfg.maxCTAs = opt_.max_ctas;
    ncclResult_t r = ncclCommInitRankConfig(&world_, world_size_, id, rank_, &cfg);
    if (r == ncclSuccess || r == ncclInProgress) r = wait_ready(world_);
    if (r != ncclSuccess) {
      *err = std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r) +
             (r == ncclInProgress ? " (timed out waiting for the other ranks)" : "");
      if (world_ != nullptr) ncclCommAbort(world_);
      world_ = nullptr;
      return kErrNccl;
    }
    return kOk;
  }

  int finalize() override {
    comms_.assign(groups_.size(), nullptr);
    for (size_t g = 0; g < groups_.size(); ++g) {
      if (groups_[g].ranks.size() <= 1) continue;
      const int idx = groups_[g].index_of(rank_);
      ncclComm_t c = nullptr;
      // the child inherits the parent's config (nonblocking, CTA budget)
      ncclResult_t r = ncclCommSplit(world_, idx >= 0 ? 0 : NCCL_SPLIT_NOCOLOR,
                                     idx >= 0 ? idx : 0, &c, nullptr);
      if (r == ncclInProgress) r = wait_ready(world_);
      if (r == ncclSuccess && c != nullptr) r = wait_ready(c);
      if (r != ncclSuccess) return nccl_fail(r, "ncclCommSplit");
      comms_[g] = c;
    }
    return kOk;
  }

  int all_reduce(int gid, int, void* buf, size_t count, DType t, cudaStream_t s) override {
    if (groups_[gid].ranks.size() <= 1) return kOk;
    return done(comms_[gid], ncclAllReduce(buf, buf, count, nccl_type(t), ncclSum, comms_[gid], s),
                "ncclAllReduce");
  }

  int reduce_scatter(int gid, int, const void* send, void* recv, size_t count, DType t,
                     cudaStream_t s) override {
    if (groups_[gid].ranks.size() <= 1) {
      if (send == recv) return kOk;
      return cuda_ok(cudaMemcpyAsync(recv, send, count * dtype_bytes(t), cudaMemcpyDeviceToDevice,
                                     s),
                     "reduce_scatter copy");
    }
    return done(comms_[gid],
                ncclReduceScatter(send, recv, count, nccl_type(t), ncclSum, comms_[gid], s),
                "ncclReduceScatter");
  }

  int all_gather(int gid, int rank, const void* send, void* recv,
                 const std::vector<size_t>& counts, DType t, cudaStream_t s) override {
    const CommGroup& g = groups_[gid];
    const size_t eb = dtype_bytes(t);
    if (g.ranks.size() <= 1) {
      if (send == recv) return kOk;
      return cuda_ok(cudaMemcpyAsync(recv, send, counts[0] * eb, cudaMemcpyDeviceToDevice, s),
                     "all_gather copy");
    }
    const bool equal = std::all_of(counts.begin(), counts.end(),
                                   [&](size_t c) { return c == counts[0]; });
    if (equal)
      return done(comms_[gid], ncclAllGather(send, recv, counts[0], nccl_type(t), comms_[gid], s),
                  "ncclAllGather");
    const int me = g.index_of(rank);
    ncclGroupStart();
    size_t displ = 0;
    for (size_t j = 0; j < counts.size(); ++j) {
      char* dst = static_cast<char*>(recv) + displ * eb;
      const void* src = static_cast<int>(j) == me ? send : dst;
      const ncclResult_t r =
          ncclBroadcast(src, dst, counts[j], nccl_type(t), static_cast<int>(j), comms_[gid], s);
      if (r != ncclSuccess && r != ncclInProgress) {
        ncclGroupEnd();
        return nccl_fail(r, "ncclBroadcast");
      }
      displ += counts[j];
    }
    return done(comms_[gid], ncclGroupEnd(), "ncclGroupEnd");
  }

  int send(int, int peer, const void* buf, size_t bytes, cudaStream_t s) override {
    return done(world_, ncclSend(buf, bytes, ncclUint8, peer, world_, s), "ncclSend");
  }
  int recv(int, int peer, void* buf, size_t bytes, cudaStream_t s) override {
    return done(world_, ncclRecv(buf, bytes, ncclUint8, peer, world_, s), "ncclRecv");
  }
  int group_start() override { return nccl_ok(ncclGroupStart(), "ncclGroupStart"); }
  int group_end() override { return done(world_, ncclGroupEnd(), "ncclGroupEnd"); }

  int world_sum(int, float* v, cudaStream_t s) override {
    return done(world_, ncclAllReduce(v, v, 1, ncclFloat32, ncclSum, world_, s),
                "ncclAllReduce(loss)");
  }

  int poll_async() override {
    auto check = [](ncclComm_t c) {
      ncclResult_t a = ncclSuccess;
      if (c != nullptr && ncclCommGetAsyncError(c, &a) == ncclSuccess && a != ncclSuccess &&
          a != ncclInProgress)
        return nccl_fail(a, "NCCL asynchronous error");
      return static_cast<int>(kOk);
    };
    int rc = check(world_);
    for (ncclComm_t c : comms_)
      if (rc == kOk) rc = check(c);
    return rc;
  }

  void abort() override {
    for (ncclComm_t& c : comms_)
      if (c != nullptr) {
        ncclCommAbort(c);
        c = nullptr;
      }
    if (world_ != nullptr) ncclCommAbort(world_);
    world_ = nullptr;
  }

 private:
  static int nccl_fail(ncclResult_t r, const char* what) {
    return set_error(kErrNccl, (std::string(what) + ": " + ncclGetErrorString(r)).c_str());
  }
  static int nccl_ok(ncclResult_t r, const char* what) {
    return r == ncclSuccess ? kOk : nccl_fail(r, what);
  }
  // Nonblocking communicator: poll until the communicator leaves ncclInProgress (or the
  // deadline passes, reported as ncclInProgress).
  ncclResult_t wait_ready(ncclComm_t c) const {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      ncclResult_t a = ncclSuccess;
      const ncclResult_t q = ncclCommGetAsyncError(c, &a);
      if (q != ncclSuccess) return q;
      if (a != ncclInProgress) return a;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(opt_.timeout_ms))
        return ncclInProgress;
      std::this_thread::yield();
    }
  }
  // An enqueue on a nonblocking communicator may return ncclInProgress: wait for it.
  int done(ncclComm_t c, ncclResult_t r, const char* what) const {
    if (r == ncclInProgress) r = wait_ready(c);
    return nccl_ok(r, what);
  }
  int world_size_, rank_;
  NcclOptions opt_;
  ncclComm_t world_ = nullptr;
  std::vector<ncclComm_t> comms_;
};

// =========================================================== no-op world (per-GPU proxy)
class NullComm final : public Comm {
 public:
  int finalize() override { return kOk; }
  int all_reduce(int, int, void*, size_t, DType, cudaStream_t) override { return kOk; }
  int reduce_scatter(int, int, const void*, void*, size_t, DType, cudaStream_t) override {
    return kOk;
  }
  int all_gather(int, int, const void*, void*, const std::vector<size_t>&, DType,
                 cudaStream_t) override {
    return kOk;
  }
  int send(int, int, const void*, size_t, cudaStream_t) override { return kOk; }
  int recv(int, int, void*, size_t, cudaStream_t) override { return kOk; }
  int world_sum(int, float*, cudaStream_t) override { return kOk; }
};

}  // namespace

std::unique_ptr<Comm> make_null_comm(int) { return std::make_unique<NullComm>(); }

std::unique_ptr<Comm> make_sim_comm(int world_size) {
  return std::make_unique<SimComm>(world_size);
}

std::unique_ptr<Comm> make_nccl_comm(int world_size, int rank, const std::string& unique_id,
                                     const NcclOptions& opt, std::string* err) {
  auto c = std::make_unique<NcclComm>(world_size, rank, opt);
  if (c->init(unique_id, err) != kOk) return nullptr;
  return c;
}

}  // namespace gx
