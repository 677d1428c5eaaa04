// comm.h — the executor's collective layer: a pool of communication groups (created once,
// PAPER.md:338) with two backends behind one interface:
//   NcclComm  one process per GPU, one ncclComm_t per group split from the world comm
//             (ncclCommSplit), NVLink/NVSwitch transport chosen by NCCL;
//   SimComm   every rank of a (small) world lives in this process on one device; a
//             collective completes when the last member of its group has posted its
//             buffers (ranks are stepped in lockstep by the executor), using device copies
//             and a fixed-order fp32 reduction.  This is how multi-rank plans are executed
//             and checked on a single B200.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace gx {

enum class DType { kBF16, kF32 };

inline size_t dtype_bytes(DType t) { return t == DType::kBF16 ? 2 : 4; }

struct CommGroup {
  std::vector<int> ranks;  // global ranks, ascending; member index = position
  int index_of(int rank) const {
    for (size_t i = 0; i < ranks.size(); ++i)
      if (ranks[i] == rank) return static_cast<int>(i);
    return -1;
  }
};

class Comm {
 public:
  virtual ~Comm() = default;

  // Registers a group (idempotent on identical member lists); returns its id.
  int add_group(std::vector<int> ranks);
  const CommGroup& group(int id) const { return groups_[id]; }
  int num_groups() const { return static_cast<int>(groups_.size()); }

  // Called once after every group is registered (NCCL: collective over the world).
  virtual int finalize() = 0;

  // In-place sum over the group.
  virtual int all_reduce(int gid, int rank, void* buf, size_t count, DType t, cudaStream_t s) = 0;
  // send: count*members elements; recv: this member's count-element slice of the sum.
  virtual int reduce_scatter(int gid, int rank, const void* send, void* recv, size_t count,
                             DType t, cudaStream_t s) = 0;
  // Variable-count all-gather: member j contributes counts[j] elements; recv holds the
  // concatenation in member order.  (Equal counts use ncclAllGather.)
  virtual int all_gather(int gid, int rank, const void* send, void* recv,
                         const std::vector<size_t>& counts, DType t, cudaStream_t s) = 0;
  // Point-to-point: rows handed between pipeline stages.  A batch of sends/recvs posted
  // between group_start()/group_end() completes together.
  virtual int send(int rank, int peer, const void* buf, size_t bytes, cudaStream_t s) = 0;
  virtual int recv(int rank, int peer, void* buf, size_t bytes, cudaStream_t s) = 0;
  virtual int group_start() { return 0; }
  virtual int group_end() { return 0; }
  // Scalar fp32 sum over the world (loss reporting).
  virtual int world_sum(int rank, float* dev_scalar, cudaStream_t s) = 0;
  // Failure detection: an asynchronous communicator error (a peer died, a
  // network fault) as kErrNccl, else kOk.  abort() tears every communicator down so kernels
  // blocked on a dead peer return and the process can exit instead of hanging.
  virtual int poll_async() { return 0; }
  virtual void abort() {}

 protected:
  std::vector<CommGroup> groups_;
};

std::unique_ptr<Comm> make_sim_comm(int world_size);
// Every collective and transfer is a no-op: one rank of a larger world run alone on one GPU
// (bench.py's per-GPU proxy of an N-GPU plan).
std::unique_ptr<Comm> make_null_comm(int world_size);
// NCCL communicator options (E13): a CTA budget so collectives overlapped with GEMMs leave
// SMs to them, and a timeout for communicator creation (nonblocking init, polled).
struct NcclOptions {
  int min_ctas = 0;        // 0 = NCCL default
  int max_ctas = 16;       // per collective; NVSwitch (NVLS) needs few CTAs for full bandwidth
  int timeout_ms = 120000;  // init / split / in-progress polling limit
};
// unique_id: the 128-byte ncclUniqueId shared by all ranks (rank 0 creates it).
std::unique_ptr<Comm> make_nccl_comm(int world_size, int rank, const std::string& unique_id,
                                     const NcclOptions& opt, std::string* err);

}  // namespace gx
