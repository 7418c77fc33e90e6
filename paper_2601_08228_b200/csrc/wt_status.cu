// Thread-local error string + version for the C ABI (include/wten_b200.h).
#include <stdarg.h>
#include <stdio.h>

#include <map>
#include <mutex>
#include <utility>

#include "wt_common.cuh"

namespace wt {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: kernel launch failed: %s", what, cudaGetErrorString(e));
    return WT_ERR_CUDA;
  }
  return WT_OK;
}

int smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{dev, kernel}];
  if (have >= bytes) return WT_OK;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    set_error("cudaFuncSetAttribute(MaxDynamicSharedMemorySize = %d) failed: %s", bytes,
              cudaGetErrorString(e));
    return WT_ERR_CUDA;
  }
  have = bytes;
  return WT_OK;
}

}  // namespace wt

extern "C" int wt_version(void) { return 100; }

extern "C" const char* wt_last_error(void) { return wt::g_last_error; }
