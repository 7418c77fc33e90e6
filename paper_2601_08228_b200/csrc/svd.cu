// K4: batched one-sided block-Jacobi SVD in FP64 (Gram and rotation tiles on
// the DMMA tensor pipe).  Replaces _stack_svd (decomposition.py:64-67), i.e.
// LAPACK dgesdd over every wavelet-domain slice.
//
// Algorithm:
//   X (m x n, n <= m, columns contiguous) is the slice oriented so that the
//   short side is orthogonalised: X = A^T when n1 <= n2 (columns = rows of A),
//   X = A otherwise.  Columns are grouped in blocks of 16; each sweep visits
//   every block pair once in round-robin order (nblk-1 rounds of nblk/2
//   disjoint pairs, one CTA per pair and matrix).  Per pair:
//     1. G = Z^T Z for the 32-column panel Z = [X_I X_J] (DMMA on the 10 upper
//        8x8 tiles, rows streamed through shared memory with cp.async double
//        buffering, rows split over the warps, fixed-order tree reduction);
//     2. if every |G_ij| <= tol sqrt(G_ii G_jj) (+ a null-column floor) the
//        pair is skipped; otherwise one sweep of cyclic parallel two-sided
//        Jacobi on G in shared memory (16 disjoint rotations per step) gives Q;
//     3. Z <- Z Q (DMMA, streamed again -- mostly from L2 -- written back).
//   Before every sweep the columns are reordered by descending norm.  A sweep
//   in which no pair exceeded tol retires the matrix: later launches only run
//   over the compacted list of matrices still iterating.
//   Finally sigma_c = ||X_c|| and the columns are sorted descending; the
//   normalised columns are the long-side singular vectors.
// Everything is deterministic: fixed reduction orders, no floating atomics.
#include <stdlib.h>

#include <string.h>

#include <algorithm>
#include <vector>

#include "wt_common.cuh"

#ifndef WT_SVD_THREADS
#define WT_SVD_THREADS 256
#endif
#ifndef WT_SVD_MINB
#define WT_SVD_MINB 3
#endif
#ifndef WT_EIG_WARPS
#define WT_EIG_WARPS WT_SVD_THREADS / 32
#endif
#ifndef WT_SVD_FLATRED
#define WT_SVD_FLATRED 1
#endif
#ifndef WT_SVD_SPIN_NS
#define WT_SVD_SPIN_NS 100
#endif
#ifndef WT_SVD_LIGHT_RELEASE
#define WT_SVD_LIGHT_RELEASE 1
#endif
#ifndef WT_SVD_NZ
#define WT_SVD_NZ 3
#endif

namespace wt {
// diagnostics of the last wt_svd_jacobi_f64 call on this thread
static thread_local int g_last_sweeps = 0;
static thread_local long long g_last_rotations = 0;
static thread_local long long g_last_panel_rows = 0;
static thread_local int g_last_hb = 16;
static thread_local int g_last_fallbacks = -1;  // -1: no preconditioning; else matrices that fell back to V0 = I
}  // namespace wt

#define SVD_NS hb16
#define SVD_HB 16
#include "svd_impl.cuh"
#undef SVD_NS
#undef SVD_HB

using namespace wt;

// Sweeps used by the last wt_svd_jacobi_f64 call on this thread (diagnostics).
extern "C" int wt_svd_last_sweeps(void) { return g_last_sweeps; }

// Matrices of the last call that were not preconditioned (V0 = I fallback), or
// -1 if the call ran without the preconditioner (diagnostics).
extern "C" int wt_svd_last_fallbacks(void) { return g_last_fallbacks; }

// FP64 flops executed by the Jacobi iteration of the last call on this thread:
// every rotated pair visit = Gram (upper 8x8 tiles) + Z Q on an mpad x BW
// panel: 2 * mpad * BW^2 * (Gram tile fraction + 1).
extern "C" double wt_svd_last_jacobi_flops(void) {
  const double bw = 2.0 * g_last_hb;
  const double t = bw / 8.0, gram = t * (t + 1.0) / 2.0 / (t * t);
  return (double)g_last_rotations * 2.0 * (double)g_last_panel_rows * bw * bw * (gram + 1.0);
}

extern "C" size_t wt_svd_workspace_bytes(int64_t n1, int64_t n2, int64_t batch) {
  if (n1 < 0 || n2 < 0 || batch < 0) return 0;
  return hb16::workspace_bytes(n1, n2, batch);
}

extern "C" int wt_svd_jacobi_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1,
                                 int64_t n2, int64_t batch, double* sigma, double* vec,
                                 int64_t nvec, int* info, double tol, int max_sweeps,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && batch >= 0, "svd: bad shape %lld x %lld", (long long)n1,
             (long long)n2);
  if (batch == 0) return WT_OK;
  if (batch > 65535) {  // grid.y limit: chunks of matrices through a prefix of the workspace
    const int64_t q = n1 < n2 ? n1 : n2, ln = n1 < n2 ? n2 : n1;
    WT_REQUIRE(workspace_bytes >= wt_svd_workspace_bytes(n1, n2, 65535),
               "svd: workspace too small for 65535-matrix chunks");
    long long sweeps = 0, rotations = 0;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
      const int64_t nb = std::min<int64_t>(65535, batch - b0);
      int e = wt_svd_jacobi_f64(A + b0 * strideA, lda, strideA, n1, n2, nb, sigma + b0 * q,
                                vec ? vec + b0 * nvec * ln : vec, nvec, info + b0, tol, max_sweeps,
                                workspace, workspace_bytes, stream);
      if (e) return e;
      sweeps = std::max<long long>(sweeps, g_last_sweeps);
      rotations += g_last_rotations;
    }
    g_last_sweeps = (int)sweeps;
    g_last_rotations = rotations;
    return WT_OK;
  }
  g_last_hb = 16;
  return hb16::jacobi(A, lda, strideA, n1, n2, batch, sigma, vec, nvec, info, tol, max_sweeps,
                      workspace, workspace_bytes, stream);
}

extern "C" size_t wt_svd_topk_workspace_bytes(int64_t n1, int64_t n2, int64_t batch, int64_t k) {
  if (n1 < 1 || n2 < 1 || batch < 0 || k < 1) return 0;
  return hb16::topk_layout(n1, n2, batch, k).total;
}

extern "C" int wt_svd_topk_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1, int64_t n2, int64_t batch,
                               int64_t k, double* sigma, double* vec, int64_t nvec, int* info, double tol,
                               int max_sweeps, void* workspace, size_t workspace_bytes, void* stream) {
  WT_REQUIRE(batch <= 65535, "svd_topk: batch above 65535");
  g_last_hb = 16;
  return hb16::jacobi_topk(A, lda, strideA, n1, n2, batch, k, sigma, vec, nvec, info, tol, max_sweeps, workspace,
                           workspace_bytes, stream);
}
