// errors.cc — thread-local last-error storage behind gx_last_error().
#include <cuda_runtime.h>

#include <atomic>
#include <string>

#include "../kernels/gx_internal.h"

namespace gx {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

int64_t launch_count() { return g_launches.load(); }

int set_error(int code, const char* msg) {
  g_last_error = msg == nullptr ? "" : msg;
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    g_launches.fetch_add(1);
    return kOk;
  }
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(kErrCuda, m.c_str());
}

}  // namespace gx

extern "C" const char* gx_last_error(void) { return gx::g_last_error.c_str(); }
extern "C" int gx_version(void) { return 1; }
extern "C" int64_t gx_launch_count(void) { return gx::launch_count(); }
