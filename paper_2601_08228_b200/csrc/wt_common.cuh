// Shared helpers for the wten_b200 sm_100a kernels: status plumbing for the
// C ABI, PTX wrappers for the bulk-async (TMA 1-D) copy engine and mbarriers,
// and the FP64 DMMA fragment op.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/wten_b200.h"

namespace wt {

// ---------------------------------------------------------------- status ----
void set_error(const char* fmt, ...);
int check_launch(const char* what);
int option(int which);  // wt_set_option's table (production defaults unless a test changed them)

// K3 with per-matrix limits (device arrays, nullable): the inner dimension of
// matrix b is min(K, klim[b]) (operands beyond it read as zeros) and output
// column tiles starting at or beyond nlim[b] are skipped (not written).
// lower = 1 computes only the tiles that touch the lower triangle (j <= i) --
// symmetric rank-2k updates whose upper part is never read.
int gemm_f64_lim(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                 const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                 int64_t strideB, double beta, double* C, int64_t ldc, int64_t strideC,
                 int64_t batch, const int* klim, const int* nlim, void* stream, int lower = 0);

// K4 preconditioner (eig.cu): for the batch of m x n matrices X given as Xt
// (row r of Xt = column r of X, pitch ldx, stride sx; n <= m) writes the kk
// columns of X V0 as the rows of Yt (pitch ldy, stride sy), V0 = the kk leading
// eigenvectors of X^T X (Householder tridiagonalization, bisection, inverse
// iteration, Newton-Schulz), descending.  Matrices whose basis fails the
// orthogonality check get V0 = I[:, :kk].
size_t eig_workspace_bytes(int64_t n, int64_t batch);
// kmask (nullable, device): per-matrix K limit of the Gram and X V0 GEMMs, 0 for
// an all-zero slice (its Gram and X V0 are written as zeros without the k loop).
int eig_precondition(const double* Xt, double* Yt, int64_t m, int64_t n, int64_t ldx, int64_t sx,
                     int64_t batch, int64_t kk, int64_t ldy, int64_t sy, void* ws, size_t ws_bytes, int* n_fallback,
                     cudaStream_t st, const int* kmask = nullptr, int* h_flags = nullptr);
// (h_flags, host, nullable, needs n_fallback: per matrix 1 = preconditioned, 0 = fell back to V0 = I)
// wt_scale_cols_f64 with an optional per-matrix column limit (columns >= clim[b] untouched).
int scale_cols_lim(double* M, int64_t rows, int64_t ncols, int64_t ld, int64_t strideM,
                   const double* s, int64_t q, int64_t batch, int mode, double tol,
                   const int* clim, void* stream);

// wt_orthonormal_fixup_f64 with general strides: element (row i, vector j) at M[i * si + j * sj].
int ortho_fixup_strided(double* M, int64_t rows, int64_t r, int64_t si, int64_t sj, int64_t strideM,
                        const double* s, int64_t q, int64_t batch, double tau, void* stream, int skip_zero);
// (skip_zero: matrices whose largest singular value is 0 are left untouched)

#define WT_REQUIRE(cond, ...)        \
  do {                               \
    if (!(cond)) {                   \
      ::wt::set_error(__VA_ARGS__);  \
      return WT_ERR_INVALID;         \
    }                                \
  } while (0)

#define WT_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ::wt::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),      \
                      __FILE__, __LINE__);                                         \
      return WT_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

// Raise a kernel's dynamic shared-memory limit to `bytes` on the CURRENT
// device (the attribute is per device; cached per (device, kernel), thread-safe).
int smem_attr(const void* kernel, int bytes);
template <typename K>
inline int ensure_smem(K kernel, size_t bytes) {
  return smem_attr(reinterpret_cast<const void*>(kernel), (int)bytes);
}

constexpr int kNumSMs = 148;  // B200; queried at runtime where it matters

inline int num_sms() {
  static const int n = [] {  // thread-safe one-time init (one GPU model per process)
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0 ? v
                                                                                                : kNumSMs;
  }();
  return n;
}

// ------------------------------------------------------- async copy (PTX) ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine (SASS UBLKCP),
// completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Ampere-style cp.async (LDGSTS) with zero-fill: copies `src_bytes` (0 or N)
// and zero-fills the rest of the N-byte destination.
template <int N>
__device__ __forceinline__ void cp_async_zfill(void* dst_smem, const void* src, bool valid) {
  int sz = valid ? N : 0;
  if constexpr (N == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst_smem)),
                 "l"(src), "r"(sz)
                 : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(dst_smem)),
                 "l"(src), "n"(N), "r"(sz)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------ readback -----
// A few ints from device memory into PAGE-LOCKED host memory by a one-warp
// kernel that stores straight into the mapped host block, not by cudaMemcpyAsync:
// a 4-byte copy queues on the D2H copy engine behind whatever bulk transfer other
// streams have in flight (a 256 MiB chunk holds it for ~5 ms; K4's ~8 readbacks
// per call took it from 17.8 to 47 ms under sp_w_svd_many's PCIe traffic).
// Ordered on `st` like the copy it replaces: valid after the stream is synchronised.
static __global__ void readback_ints_kernel(const int* __restrict__ src, int* __restrict__ dst_host, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst_host[i] = src[i];
  __threadfence_system();
}
inline cudaError_t readback_ints(int* h_pinned, const int* d_src, int n, cudaStream_t st) {
  int* h_dev = nullptr;  // (unified addressing: the same pointer; asked for rather than assumed)
  if (n <= 0) return cudaSuccess;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_dev), h_pinned, 0) != cudaSuccess || h_dev == nullptr) {
    (void)cudaGetLastError();
    return cudaMemcpyAsync(h_pinned, d_src, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost, st);
  }
  readback_ints_kernel<<<1, n < 256 ? 32 : 256, 0, st>>>(d_src, h_dev, n);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- DMMA -----
// D(8x8) += A(8x4, row) * B(4x8, col) in FP64 on the tensor pipe (SASS DMMA.884).
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
//            c = {C[lane/4][2*(lane%4)], C[lane/4][2*(lane%4)+1]}.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

}  // namespace wt
