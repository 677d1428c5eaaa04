// exec_capi.cc — extern "C" surface of the plan executor (gx_exec_* in include/gx.h).
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "../kernels/gx_internal.h"
#include "executor.h"

struct gx_exec {
  std::unique_ptr<gx::Executor> impl;
};

namespace {
int bad(const char* m) { return gx::set_error(gx::kErrConfig, m); }
}  // namespace

extern "C" {

int gx_exec_create(const char* config_json, gx_exec** out) {
  if (config_json == nullptr || out == nullptr) return bad("exec_create: NULL argument");
  std::string err;
  int code = gx::kOk;
  auto impl = gx::create_executor(config_json, &err, &code);
  if (!impl) {
    if (code == gx::kErrInfeasible) return gx::set_error(code, err.c_str());  // memory cap
    const bool nccl = err.find("nccl") != std::string::npos;
    const bool cuda = err.find("CUDA") != std::string::npos || err.find("cuda") != std::string::npos ||
                      err.find("memory") != std::string::npos;
    return gx::set_error(nccl ? gx::kErrNccl : (cuda ? gx::kErrCuda : gx::kErrConfig), err.c_str());
  }
  *out = new gx_exec{std::move(impl)};
  return gx::kOk;
}

int gx_exec_destroy(gx_exec* ex) {
  delete ex;
  return gx::kOk;
}

int gx_exec_set_layer_params(gx_exec* ex, int layer, const float* c, int64_t n) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->set_layer_params(layer, c, n);
}

int gx_exec_export_layer(gx_exec* ex, int layer, int what, float* c, int64_t n) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->export_layer(layer, what, c, n);
}

int gx_exec_load_batch(gx_exec* ex, const void* x, const void* t) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->load_batch(x, t);
}

int gx_exec_load_batch_device(gx_exec* ex, const void* x, const void* t) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->load_batch_device(x, t);
}

int gx_exec_run(gx_exec* ex, int flags) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->run2((flags & 1) != 0, (flags & 2) != 0);
}

int gx_exec_time(gx_exec* ex, int flags, int warmup, int steps, double* ms_per_run) {
  if (ex == nullptr || ms_per_run == nullptr) return bad("exec_time: NULL argument");
  if (steps <= 0 || warmup < 0) return bad("exec_time: steps must be > 0 and warmup >= 0");
  for (int i = 0; i < warmup; ++i) {
    const int rc = gx_exec_run(ex, flags);
    if (rc != gx::kOk) return rc;
  }
  auto st = static_cast<cudaStream_t>(ex->impl->stream());
  cudaEvent_t a = nullptr, b = nullptr;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) {
    cudaGetLastError();
    return gx::set_error(gx::kErrCuda, "exec_time: cudaEventCreate failed");
  }
  int rc = gx::kOk;
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = gx::check_launch("exec_time warm-up");
  if (rc == gx::kOk) {
    cudaEventRecord(a, st);
    for (int i = 0; i < steps && rc == gx::kOk; ++i) rc = gx_exec_run(ex, flags);
    cudaEventRecord(b, st);
  }
  float ms = 0.f;
  if (rc == gx::kOk) {
    if (cudaEventSynchronize(b) != cudaSuccess || cudaEventElapsedTime(&ms, a, b) != cudaSuccess)
      rc = gx::set_error(gx::kErrCuda, "exec_time: event timing failed");
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (rc == gx::kOk) *ms_per_run = static_cast<double>(ms) / steps;
  return rc;
}

int gx_exec_profile_report(gx_exec* ex, char* out, size_t cap, size_t* needed) {
  if (ex == nullptr) return bad("exec: NULL handle");
  const std::string s = ex->impl->profile_report();
  if (needed != nullptr) *needed = s.size() + 1;
  if (out == nullptr || cap == 0) return gx::kOk;
  if (cap < s.size() + 1) return bad("profile_report: buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return gx::kOk;
}

int gx_exec_init_params(gx_exec* ex, uint64_t seed, float std_dev) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->init_params(seed, std_dev);
}

int gx_exec_loss(gx_exec* ex, float* out) {
  if (ex == nullptr || out == nullptr) return bad("exec: NULL argument");
  return ex->impl->loss(out);
}

int gx_exec_sync(gx_exec* ex, int64_t timeout_ms) {
  if (ex == nullptr) return bad("exec: NULL handle");
  return ex->impl->sync(timeout_ms);
}

int gx_exec_step(gx_exec* ex, const void* x, const void* t, int use_graph, float* loss_out) {
  if (ex == nullptr) return bad("exec: NULL handle");
  int rc = ex->impl->load_batch(x, t);
  if (rc == gx::kOk) rc = ex->impl->run(use_graph != 0);
  if (rc == gx::kOk && loss_out != nullptr) rc = ex->impl->loss(loss_out);
  return rc;
}

int gx_exec_export_output(gx_exec* ex, int what, void* host) {
  if (ex == nullptr || host == nullptr) return bad("exec: NULL argument");
  return ex->impl->export_output(host, what);
}

int gx_exec_stream(gx_exec* ex, void** s) {
  if (ex == nullptr || s == nullptr) return bad("exec: NULL argument");
  *s = ex->impl->stream();
  return gx::kOk;
}

int gx_exec_info(gx_exec* ex, char* out, size_t cap, size_t* needed) {
  if (ex == nullptr) return bad("exec: NULL handle");
  const std::string s = ex->impl->info();
  if (needed != nullptr) *needed = s.size() + 1;
  if (out == nullptr || cap == 0) return gx::kOk;
  if (cap < s.size() + 1) return bad("exec_info: buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return gx::kOk;
}

int gx_exec_topology(const char* config_json, char* out, size_t cap, size_t* needed) {
  if (config_json == nullptr) return bad("exec_topology: NULL config");
  std::string cfg = config_json;
  // force the device-free dry-run mode
  std::string err;
  auto impl = gx::create_executor(cfg, &err);
  if (!impl) return gx::set_error(gx::kErrConfig, err.c_str());
  const std::string s = impl->topology();
  if (needed != nullptr) *needed = s.size() + 1;
  if (out == nullptr || cap == 0) return gx::kOk;
  if (cap < s.size() + 1) return bad("exec_topology: buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return gx::kOk;
}

int gx_exec_canonical_size(int hidden, int ffn, int64_t* out) {
  gx::Shape s;
  s.h = hidden;
  s.ffn = ffn;
  *out = gx::canonical_size(s);
  return gx::kOk;
}

int gx_nccl_unique_id(char* out_hex, size_t cap) {
  if (out_hex == nullptr || cap < 257) return bad("nccl_unique_id: need 257 bytes");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess)
    return gx::set_error(gx::kErrNccl, (std::string("ncclGetUniqueId: ") + ncclGetErrorString(r)).c_str());
  for (int i = 0; i < 128; ++i)
    std::snprintf(out_hex + 2 * i, 3, "%02x", static_cast<unsigned char>(id.internal[i]));
  return gx::kOk;
}

}  // extern "C"
