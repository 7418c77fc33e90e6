// K5 / K6 / K7: the SVD epilogues of the decomposition path as single C-ABI
// calls, composed stream-ordered from K3 (wt_gemm_f64) and the column-scale /
// copy kernels of util.cu.  All use the long-side singular vectors K4 returns
// (right vectors when n1 <= n2, left vectors otherwise), so the short-side
// factor is never formed explicitly:
//   right side:  T = A V_r  (n1 x r)      recon = T V_r^T      pinv = V diag(s+^2) (A V)^T
//   left side:   T = A^T U_r (n2 x r)     recon = U_r T^T      pinv = (A^T U) diag(s+^2) U^T
// which equal U_r diag(s_r) V_r^T (decomposition.py:70-72) and V diag(s+) U^T
// (decomposition.py:157-163) because A V = U diag(s) and A^T U = V diag(s).
#include "wt_common.cuh"

extern "C" int wt_svd_truncate_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1,
                                   int64_t n2, int64_t batch, const double* vec, int64_t nvec,
                                   int64_t r, double* recon, int64_t ldr, int64_t strideR,
                                   double* T, void* stream) {
  const int64_t q = n1 < n2 ? n1 : n2, ln = n1 < n2 ? n2 : n1;
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && batch >= 0, "svd_truncate: bad shape");
  WT_REQUIRE(r >= 1 && r <= q && r <= nvec, "svd_truncate: rank %lld outside [1, %lld]",
             (long long)r, (long long)(q < nvec ? q : nvec));
  WT_REQUIRE(T != nullptr && recon != nullptr && A != nullptr && vec != nullptr,
             "svd_truncate: null pointer");
  if (batch == 0) return WT_OK;
  const int64_t sV = nvec * ln, sT = q * r;
  int st;
  if (n1 <= n2) {
    // T = A V_r^T-stored-rows: (n1 x n2) x (r x n2)^T
    st = wt_gemm_f64(0, 1, n1, r, n2, 1.0, A, lda, strideA, vec, ln, sV, 0.0, T, r, sT, batch, stream);
    if (st) return st;
    return wt_gemm_f64(0, 0, n1, n2, r, 1.0, T, r, sT, vec, ln, sV, 0.0, recon, ldr, strideR, batch,
                       stream);
  }
  // T = A^T U_r: A stored (n1 x n2) read transposed, U_r rows (r x n1) read transposed
  st = wt_gemm_f64(1, 1, n2, r, n1, 1.0, A, lda, strideA, vec, ln, sV, 0.0, T, r, sT, batch, stream);
  if (st) return st;
  return wt_gemm_f64(1, 1, n1, n2, r, 1.0, vec, ln, sV, T, r, sT, 0.0, recon, ldr, strideR, batch,
                     stream);
}

extern "C" int wt_svd_factors_f64(const double* T, const double* vec, int64_t nvec,
                                  const double* sigma, int64_t n1, int64_t n2, int64_t batch,
                                  int64_t r, double* U, double* V, void* stream) {
  const int64_t q = n1 < n2 ? n1 : n2, ln = n1 < n2 ? n2 : n1;
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && batch >= 0, "svd_factors: bad shape");
  WT_REQUIRE(r >= 1 && r <= q && r <= nvec, "svd_factors: bad rank %lld", (long long)r);
  WT_REQUIRE(T && vec && sigma && U && V, "svd_factors: null pointer");
  if (batch == 0) return WT_OK;
  const int64_t sV = nvec * ln, sT = q * r;
  // short-side factor = T / sigma (column j scaled by 1/s_j, 0 for s_j == 0)
  double* shortf = n1 <= n2 ? U : V;
  double* longf = n1 <= n2 ? V : U;
  const int64_t srows = n1 <= n2 ? n1 : n2;
  int st = wt_copy2d_f64(T, r, sT, shortf, r, srows * r, srows, r, batch, 0, stream);
  if (st) return st;
  st = wt_scale_cols_f64(shortf, srows, r, r, srows * r, sigma, q, batch, WT_SCALE_DIV, 0.0, stream);
  if (st) return st;
  // (A v_j) / s_j is orthogonal only to ~eps s_max / s_j and zero for s_j = 0:
  // re-orthonormalise in sigma order (LAPACK's U and V are orthonormal blocks)
  st = wt_orthonormal_fixup_f64(shortf, srows, r, r, srows * r, sigma, q, batch, 1.0, stream);
  if (st) return st;
  // long-side factor = first r long-side vectors, transposed to (ln x r); the
  // numerically null ones (s_j <= ~1e-12 s_max: the Jacobi test leaves their
  // directions unconstrained; zero vectors for s_j = 0) are completed likewise
  st = wt_copy2d_f64(vec, ln, sV, longf, r, ln * r, ln, r, batch, 1, stream);
  if (st) return st;
  return wt_orthonormal_fixup_f64(longf, ln, r, r, ln * r, sigma, q, batch, 1e-12, stream);
}

namespace {
// k_b = #{i : s_i > tol * s_0 and s_i > 0} (sigma descending): the columns
// WT_SCALE_PINV2 keeps (decomposition.py:160-161).
__global__ void pinv_rank_kernel(const double* __restrict__ s, int64_t q, double tol, int* rank) {
  const int64_t b = blockIdx.x;
  const double smax = s[b * q];
  int cnt = 0;
  for (int64_t i = threadIdx.x; i < q; i += blockDim.x) {
    const double v = s[b * q + i];
    cnt += (v > tol * smax && v > 0.0) ? 1 : 0;
  }
  __shared__ int tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  atomicAdd(&tot, cnt);  // integer: order-independent
  __syncthreads();
  if (threadIdx.x == 0) rank[b] = tot;
}
}  // namespace

extern "C" int wt_pinv_from_svd_ranked_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1,
                                           int64_t n2, int64_t batch, const double* sigma,
                                           const double* vec, double tol, double* out, int64_t ldo,
                                           int64_t strideO, double* T, int* rank_ws, void* stream) {
  const int64_t q = n1 < n2 ? n1 : n2, ln = n1 < n2 ? n2 : n1;
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && batch >= 0, "pinv_from_svd: bad shape");
  WT_REQUIRE(A && sigma && vec && out && T, "pinv_from_svd: null pointer");
  if (batch == 0) return WT_OK;
  if (rank_ws) {
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
      const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
      pinv_rank_kernel<<<(unsigned)nb, 128, 0, (cudaStream_t)stream>>>(sigma + b0 * q, q, tol,
                                                                       rank_ws + b0);
    }
    if (int e = wt::check_launch("pinv_rank_kernel")) return e;
  }
  const int64_t sV = q * ln, sT = q * q;
  int st;
  if (n1 <= n2) {
    // T = A V (n1 x q) = U diag(s), first k_b columns; scale by s+^2 -> U diag(s+);
    // out = V T^T (n2 x n1) over the k_b kept terms
    st = wt::gemm_f64_lim(0, 1, n1, q, n2, 1.0, A, lda, strideA, vec, ln, sV, 0.0, T, q, sT, batch,
                          nullptr, rank_ws, stream);
    if (st) return st;
    st = wt::scale_cols_lim(T, n1, q, q, sT, sigma, q, batch, WT_SCALE_PINV2, tol, rank_ws, stream);
    if (st) return st;
    return wt::gemm_f64_lim(1, 1, n2, n1, q, 1.0, vec, ln, sV, T, q, sT, 0.0, out, ldo, strideO,
                            batch, rank_ws, nullptr, stream);
  }
  // T = A^T U (n2 x q) = V diag(s), first k_b columns; out = T diag(s+^2) U^T (n2 x n1)
  st = wt::gemm_f64_lim(1, 1, n2, q, n1, 1.0, A, lda, strideA, vec, ln, sV, 0.0, T, q, sT, batch,
                        nullptr, rank_ws, stream);
  if (st) return st;
  st = wt::scale_cols_lim(T, n2, q, q, sT, sigma, q, batch, WT_SCALE_PINV2, tol, rank_ws, stream);
  if (st) return st;
  return wt::gemm_f64_lim(0, 0, n2, n1, q, 1.0, T, q, sT, vec, ln, sV, 0.0, out, ldo, strideO, batch,
                          rank_ws, nullptr, stream);
}

extern "C" int wt_pinv_from_svd_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1,
                                    int64_t n2, int64_t batch, const double* sigma,
                                    const double* vec, double tol, double* out, int64_t ldo,
                                    int64_t strideO, double* T, void* stream) {
  return wt_pinv_from_svd_ranked_f64(A, lda, strideA, n1, n2, batch, sigma, vec, tol, out, ldo,
                                     strideO, T, nullptr, stream);
}
