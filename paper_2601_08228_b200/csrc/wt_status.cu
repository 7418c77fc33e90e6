// Thread-local error string + version for the C ABI (include/wten_b200.h).
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
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

// Test / diagnostic switches (wt_set_option): the production defaults unless a
// test or a diagnostics tool changes them.
static std::atomic<int> g_options[WT_OPT_COUNT] = {
    {0},  // WT_OPT_SVD_SPLIT: 0 = host rule, else forced cluster split S
    {0},  // WT_OPT_SVD_CTAS_PER_SM: 0 = host rule, else cap on resident sweep CTAs per SM
    {1},  // WT_OPT_SVD_PAIR_SKIP: clean-pair skip on
    {1},  // WT_OPT_SVD_PERSIST: persistent dependency-scheduled sweeps on
    {1},  // WT_OPT_SVD_PRECOND: Gram-eigenbasis preconditioner on
    {0},  // WT_OPT_SVD_PROFILE: per-phase cycle counters on stderr
    {0},  // WT_OPT_SVD_TRACE: per-sweep convergence trace on stderr
    {0},  // WT_OPT_EIG_PROFILE: preconditioner phase times on stderr
    {1},  // WT_OPT_EIG_TWOSTAGE: two-stage tridiagonalization (eig_sbr.cuh) where eligible
    {1},  // WT_OPT_GEMM_TMA: K3 large tiles through the tensor-map variant
    {0},  // WT_OPT_EIG_SPLIT: 0 = host rule, 1 = never, 2 / 3 / 4 = always split the two-stage reduction into that many groups on their own streams
};

int option(int which) { return (which >= 0 && which < WT_OPT_COUNT) ? g_options[which].load() : 0; }

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

extern "C" int wt_version(void) { return 200; }

extern "C" int wt_set_option(int which, int value) {
  if (which < 0 || which >= WT_OPT_COUNT) {
    wt::set_error("wt_set_option: unknown option %d", which);
    return WT_ERR_INVALID;
  }
  return wt::g_options[which].exchange(value);
}

extern "C" const char* wt_last_error(void) { return wt::g_last_error; }
