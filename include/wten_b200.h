/*
 * wten_b200 -- C ABI of the B200 (sm_100a) hot path of the w-product framework.
 *
 * This is the drop-in boundary for the reference package `wten`
 * (/root/reference/pkg/src/wten).  The reference is pure Python/numpy, so
 * there is no reference C header; each entry point below names the reference
 * function (file:line) whose arithmetic it replaces.  The Python mirror of the
 * reference API (paper_2601_08228_b200/{lifting,algebra,decomposition}.py)
 * binds these symbols with ctypes; INTEGRATION.md shows the equivalent stub a
 * `wten` maintainer would add.
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *     caller-owned, float64.  `stream` is a cudaStream_t (NULL = legacy default).
 *   - Every call is stream-ordered and returns an int status (WT_OK = 0).  On a
 *     non-zero status `wt_last_error()` returns a thread-local message.
 *   - Validation that the reference performs in Python (LevelError, ShapeError,
 *     RankError) stays in the Python layer, which calls these only with valid
 *     arguments; the ABI re-checks and returns WT_ERR_INVALID instead of raising.
 *
 * Tensor layouts
 *   - Spatial tensor: (n1, n2, p) C-contiguous, tube (mode-3) axis fastest,
 *     exactly the reference layout (tensor.py:1-5).  "tube" q = i*n2 + j.
 *   - Pyramid, slice-major (WT_LAYOUT_SLICE_MAJOR): p matrices of n1 x n2 rows-
 *     major, blocks in order [d1 | d2 | ... | dL | sL]; detail level j occupies
 *     slices [p - p/2^(j-1), p - p/2^j), the smooth stack the last p/2^L slices.
 *   - Pyramid, tube-major (WT_LAYOUT_TUBE_MAJOR): same block order, each block an
 *     (n1, n2, k) C-contiguous array -- the reference's own per-level arrays
 *     (lifting.py:24-34), used by the numpy drop-in path.
 *   - `slice_base`: the output/input buffer starts at packed slice index
 *     slice_base (compact buffers for the sparse variants, e.g. only [dL|sL]).
 */
#ifndef WTEN_B200_H
#define WTEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WT_OK 0
#define WT_ERR_INVALID 1     /* bad argument (shape / level / layout)            */
#define WT_ERR_CUDA 2        /* CUDA runtime error (launch / memory)             */
#define WT_ERR_UNSUPPORTED 3 /* valid but not implemented configuration          */

#define WT_LAYOUT_SLICE_MAJOR 0
#define WT_LAYOUT_TUBE_MAJOR 1

/* level_mask bit 0 = smooth sL, bit j (1..L) = detail level j. */
#define WT_MASK_ALL (~(uint64_t)0)

/* ABI version (major*100 + minor). */
int wt_version(void);
/* Thread-local description of the last failing call on this thread. */
const char* wt_last_error(void);

/*
 * K1 -- forward multilevel lazy lifting along mode 3, all L levels in one pass.
 * Replaces forward_w (lifting.py:77-94) with _lift_once (lifting.py:63-66) and
 * the tube->slice staging copies of slicewise_matmul (algebra.py:26-27) and
 * _stack_svd (decomposition.py:66).  Bit-exact with the reference.
 *   x      : (n1, n2, p) spatial tensor, tube-fastest, contiguous
 *   levels : 0 <= levels, 2^levels | p   (levels = 0 is a pure tube->slice transpose)
 *   out    : pyramid in `layout`, starting at packed slice `slice_base`
 *   level_mask : which blocks to write (others are computed but not stored)
 */
int wt_lift_fwd_f64(const double* x, int64_t n1, int64_t n2, int64_t p, int levels,
                    double* out, int layout, int64_t slice_base, uint64_t level_mask,
                    void* stream);

/*
 * K2 -- inverse multilevel lifting (lifting.py:114-120, _unlift_once :69-74).
 * Blocks not in level_mask are treated as exactly zero and never read
 * (sp_w_svd / sp_pinv_w zero the finer details, decomposition.py:152,201).
 */
int wt_lift_inv_f64(const double* pyr, int64_t n1, int64_t n2, int64_t p, int levels,
                    int layout, int64_t slice_base, uint64_t level_mask, double* y,
                    void* stream);

/*
 * K1 / K2 with the rows -> slices exchange fused in (multi-GPU, sharded.py).
 * Same transform; packed slice s (slice_base <= s < p) of the caller's tubes is
 * stored to / loaded from (double*)slice_ptrs[s - slice_base] + tube, where
 * slice_ptrs (a DEVICE array) may point into other GPUs' symmetric-memory
 * buffers: the stores / loads of the lifting kernel are the all-to-all.
 */
int wt_lift_fwd_f64_peer(const double* x, int64_t n1, int64_t n2, int64_t p, int levels,
                         const unsigned long long* slice_ptrs, int64_t slice_base,
                         uint64_t level_mask, void* stream);
int wt_lift_inv_f64_peer(const unsigned long long* slice_ptrs, int64_t n1, int64_t n2, int64_t p,
                         int levels, int64_t slice_base, uint64_t level_mask, double* y,
                         void* stream);

/*
 * K3 -- strided-batched FP64 GEMM on the DMMA tensor pipe (mma.sync f64).
 * Replaces the per-slice cblas_dgemm of slicewise_matmul (algebra.py:18-28),
 * _truncated_blocks (decomposition.py:70-72) and _pinv_stack (:162).
 * Row-major: C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b], b < batch,
 * op(A) is M x K (transA: A stored K x M), op(B) is K x N (transB: B stored N x K).
 */
int wt_gemm_f64(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                int64_t strideB, double beta, double* C, int64_t ldc, int64_t strideC,
                int64_t batch, void* stream);

/*
 * The whole w-product C = inverse_w(face_product(forward_w(A), forward_w(B)))
 * (reference algebra.py:43-51) in one call: K1 on A (n1 x n2 x p) and B
 * (n2 x n3 x p), one K3 over all p wavelet slices, K2 into C (n1 x n3 x p), all
 * C-contiguous device arrays.  `workspace` holds the three packed pyramids
 * (wt_w_product_workspace_bytes).  A call repeating the previous call's exact
 * arguments on the same host thread replays a CUDA graph of the four launches.
 */
size_t wt_w_product_workspace_bytes(int64_t n1, int64_t n2, int64_t n3, int64_t p);
int wt_w_product_f64(const double* a, const double* b, int64_t n1, int64_t n2, int64_t n3, int64_t p,
                     int levels, double* c, void* workspace, size_t workspace_bytes, void* stream);

/*
 * K4 -- batched one-sided block-Jacobi SVD (Gram/rotation tiles on DMMA).
 * Replaces _stack_svd (decomposition.py:64-67, LAPACK dgesdd).
 * For each b < batch, A[b] is an n1 x n2 row-major matrix (lda, strideA).
 * Outputs, q = min(n1, n2):
 *   sigma[b*q + i]      singular values, descending
 *   vec[b*nvec*len + i*len + t], i < nvec <= q:
 *       the i-th singular vector on the LONG side (len = max(n1, n2)):
 *       right vector v_i if n1 <= n2, else left vector u_i; unit norm
 *       (zero vector when sigma_i == 0).
 *   info[b] : 0 ok, 1 non-finite input/result, 2 no convergence in max_sweeps.
 * The short-side vectors follow from one GEMM with A (wt_svd_truncate_f64 /
 * wt_svd_factors_f64 / wt_pinv_from_svd_f64).
 * `workspace` must hold wt_svd_workspace_bytes(n1, n2, min(batch, 65535)) bytes
 * (larger batches run in chunks of 65535 matrices through that workspace).
 * tol <= 0 selects the default; max_sweeps <= 0 selects 80.
 * The call synchronizes `stream` once per sweep to test convergence.
 */
size_t wt_svd_workspace_bytes(int64_t n1, int64_t n2, int64_t batch);
int wt_svd_jacobi_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1, int64_t n2,
                      int64_t batch, double* sigma, double* vec, int64_t nvec, int* info,
                      double tol, int max_sweeps, void* workspace, size_t workspace_bytes,
                      void* stream);

/*
 * K4, leading triplets only: the k largest singular values (descending) of every
 * slice and their long-side singular vectors (nvec <= k), same conventions as
 * wt_svd_jacobi_f64.  The Jacobi sweeps run on X V0[:, :k], V0 the k leading
 * eigenvectors of X^T X -- the rank-r truncation of sp_w_svd (reference
 * decomposition.py:140-154, which needs no other singular value) with k well
 * above r (3 <= min(n1, n2) <= 2048; batch <= 65535).
 */
size_t wt_svd_topk_workspace_bytes(int64_t n1, int64_t n2, int64_t batch, int64_t k);
int wt_svd_topk_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1, int64_t n2, int64_t batch, int64_t k,
                    double* sigma, double* vec, int64_t nvec, int* info, double tol, int max_sweeps,
                    void* workspace, size_t workspace_bytes, void* stream);

/*
 * K5/K6/K7 helpers: scale the columns of a batch of row-major matrices,
 * M[b][i][j] *= f(s[b*q + j]) for j < ncols, where f is
 *   WT_SCALE_MUL (s), WT_SCALE_DIV (1/s, 0 if s == 0),
 *   WT_SCALE_PINV2 (1/s^2 if s > tol*s[b*q+0] and s > 0, else 0) -- the
 *   _pinv_stack cutoff rule (decomposition.py:160-161) applied twice.
 */
#define WT_SCALE_MUL 0
#define WT_SCALE_DIV 1
#define WT_SCALE_PINV2 2
int wt_scale_cols_f64(double* M, int64_t rows, int64_t ncols, int64_t ld, int64_t strideM,
                      const double* s, int64_t q, int64_t batch, int mode, double tol,
                      void* stream);

/* Strided batched 2-D copy / transpose: dst[b][i][j] = src[b][j][i] (trans) or
 * src[b][i][j]; rows x cols of dst.  Used for the slicewise transpose
 * (tensor.py:50-52) and the sharded row<->slice exchange permutations. */
int wt_copy2d_f64(const double* src, int64_t lds, int64_t strideS, double* dst, int64_t ldd,
                  int64_t strideD, int64_t rows, int64_t cols, int64_t batch, int trans,
                  void* stream);

/*
 * K5 / K6 / K7 -- the SVD epilogues, from K4's outputs (sigma, the long-side
 * vectors `vec`: nvec rows of length max(n1, n2)) and the matrices A that K4
 * decomposed (unchanged by K4).  Composed stream-ordered from K3 + the column
 * scaling / copy kernels; no hidden allocation.
 *
 * wt_svd_truncate_f64 -- _truncated_blocks (decomposition.py:70-72): rank-r
 *   reconstruction recon[b] (n1 x n2, pitch ldr) = U_r diag(s_r) V_r^T, via
 *   T = A V_r (n1 <= n2) or T = A^T U_r (n1 > n2); T (batch x min(n1,n2) x r,
 *   caller-allocated) keeps that projection for wt_svd_factors_f64.
 * wt_svd_factors_f64 -- _factor_blocks (decomposition.py:75-82): U (batch, n1, r)
 *   and V (batch, n2, r) row-major from T, vec and sigma (1/s of a zero
 *   singular value gives a zero column).
 * wt_pinv_from_svd_f64 -- _pinv_stack (decomposition.py:157-163): out[b]
 *   (n2 x n1, pitch ldo) = V diag(s+) U^T with s+ = 1/s for s > tol * s_max,
 *   else 0; needs the full K4 output (nvec = min(n1, n2)) and T of
 *   batch x min(n1,n2)^2 doubles.
 */
int wt_svd_truncate_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1, int64_t n2,
                        int64_t batch, const double* vec, int64_t nvec, int64_t r, double* recon,
                        int64_t ldr, int64_t strideR, double* T, void* stream);
int wt_svd_factors_f64(const double* T, const double* vec, int64_t nvec, const double* sigma,
                       int64_t n1, int64_t n2, int64_t batch, int64_t r, double* U, double* V,
                       void* stream);
int wt_pinv_from_svd_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1, int64_t n2,
                         int64_t batch, const double* sigma, const double* vec, double tol,
                         double* out, int64_t ldo, int64_t strideO, double* T, void* stream);
/* Same result as wt_pinv_from_svd_f64, with the GEMMs limited per slice to the
 * k_b kept singular values (s > tol * s_max): the projection computes only
 * k_b columns of T and the assembly sums only k_b terms, so an all-zero slice
 * (k_b = 0) costs no GEMM work and yields exact zeros.  rank_ws: batch ints
 * (device, caller-owned); on return rank_ws[b] = k_b. */
int wt_pinv_from_svd_ranked_f64(const double* A, int64_t lda, int64_t strideA, int64_t n1,
                                int64_t n2, int64_t batch, const double* sigma, const double* vec,
                                double tol, double* out, int64_t ldo, int64_t strideO, double* T,
                                int* rank_ws, void* stream);

/* Comparator-DFT helper: out[t][k] = x[t][k] - x[t][0] over ntubes tubes of p
 * samples (tube-fastest).  The t-product baselines FFT these deltas and add
 * p * x[t][0] to DC, so constant tubes transform to exact zeros off DC, as
 * np.fft.fft does (reference baselines.py:68,118,129). */
int wt_tube_delta_f64(const double* x, int64_t ntubes, int64_t p, double* out, void* stream);

/* Slicewise transpose of a spatial tensor (reference tensor.py:50-52):
 * y (n2, n1, p) with y[j][i][:] = x[i][j][:], both C-contiguous, tube-fastest:
 * one pass of whole-tube copies (no trip through the slice-major layout). */
int wt_tube_transpose_f64(const double* x, int64_t n1, int64_t n2, int64_t p, double* y,
                          void* stream);

/* n int32 values from device memory into PAGE-LOCKED host memory, then a
 * synchronisation of `stream`: a one-warp kernel stores straight into the mapped
 * host block instead of a copy-engine copy, so a status readback (K4's info
 * vector: the reference's LinAlgError check, decomposition.py:66) does not queue
 * behind bulk transfers other streams have in flight.  host_pinned must come
 * from cudaMallocHost / cudaHostAlloc / a pinned torch tensor. */
int wt_readback_i32(const int* src, int* host_pinned, int64_t n, void* stream);

/* Orthonormal completion of singular-vector columns: M[b] is rows x r (pitch ld,
 * stride strideM), its columns in the order of s[b*q + 0 ..] (descending).  Every
 * column j with s_j <= tau * s_0 (or s_j == 0 / non-finite) is re-orthonormalised
 * against columns 0..j-1 (classical Gram-Schmidt twice); a column with no
 * independent part (zero singular value) becomes the first unit vector that has
 * one.  The short-side factor (A v_j) / s_j of wt_svd_factors_f64 and
 * tensor.matrix_svd goes through it with tau = 1, the long-side vectors with
 * tau = 0 -- LAPACK returns orthonormal U and V for rank-deficient slices too
 * (reference tensor.py:70-77, decomposition.py:75-82). */
int wt_orthonormal_fixup_f64(double* M, int64_t rows, int64_t r, int64_t ld, int64_t strideM,
                             const double* s, int64_t q, int64_t batch, double tau, void* stream);

/* S[b] (r x r, row-major) = diag(s[b*q + 0 .. r-1]) for b < batch: the S factor
 * blocks of w_svd (reference decomposition.py:75-82). */
int wt_diag_blocks_f64(const double* s, int64_t q, int64_t r, int64_t batch, double* S, void* stream);

/* inverse_tensor's singularity rule (reference algebra.py:77-83, np.linalg.inv ->
 * LAPACK dgetrf): Gaussian elimination with partial pivoting, IN PLACE on the batch
 * of n x n row-major matrices W (pass a copy); info[b] = 1 + the first column with
 * an exactly zero pivot, else 0. */
int wt_lu_pivot_check_f64(double* W, int64_t n, int64_t batch, int* info, void* stream);

/* Deterministic per-band reductions used by the quality metrics (PSNR/SSIM,
 * PAPER.md:876-887) and parity norms: x, y are spatial tensors viewed as
 * (n tubes, nslices bands) tube-major; out[k] = sum over tubes of f(x, y) with
 * f = x*x (mode 0), (x-y)^2 (mode 1), x (mode 2), x*y (mode 3).  Fixed
 * reduction tree, bit-reproducible.  `out` must hold
 * wt_slice_reduce_scratch(n, nslices) bytes (the tail is scratch). */
size_t wt_slice_reduce_scratch(int64_t n, int64_t nslices);
int wt_slice_reduce_f64(const double* x, const double* y, int64_t n, int64_t nslices,
                        int mode, double* out, void* stream);

/* Imaging helpers either side of the path.
 * The reference ships no code for them (SPEC-only), so these build the operands
 * of BASELINE configs[2..4] directly in HBM.
 *
 * wt_toeplitz_tensor_f64: the slice-constant symmetric Toeplitz operator
 * out[i][j][k] = c[|i - j|] (0 beyond nc), (n, n, p) tube-fastest.
 *
 * wt_gauss_smooth2d_f64: separable reflect-mode ("half-sample symmetric")
 * Gaussian filter over axes 0 and 1 of x (n1, n2, e), e fastest, with the
 * half-kernel w[0..radius] (w[0] = centre tap); tmp and out hold n1*n2*e doubles.
 *
 * wt_hsi_mix_f64: out[pix][k] = clip(sum_j ab[pix][j] spectra[j][k] + sigma z, lo, hi)
 * with z = noise[pix][k] when `noise` is given, else standard normals from the
 * Philox-4x32-10 stream keyed by `seed` (counter pix * ceil(p / 2) + k / 2, Box-Muller
 * pair for bands k, k + 1); at most 32 endmembers. */
int wt_toeplitz_tensor_f64(const double* c, int64_t nc, int64_t n, int64_t p, double* out, void* stream);
int wt_gauss_smooth2d_f64(const double* x, int64_t n1, int64_t n2, int64_t e, const double* w,
                          int64_t radius, double* tmp, double* out, void* stream);
int wt_hsi_mix_f64(const double* ab, const double* spectra, int64_t npix, int64_t e, int64_t p,
                   double noise_sigma, const double* noise, uint64_t seed, double lo, double hi,
                   double* out, void* stream);

/* Test / diagnostic switches (process-wide; the defaults are the production
 * choices).  Returns the previous value, or WT_ERR_INVALID for an unknown option.
 * Used by the test suite to force scheduling variants whose results must not
 * change (or change only at rounding level), and by the tools/ diagnostics. */
#define WT_OPT_SVD_SPLIT 0        /* 0: host rule; S = 1, 2, 4, 8: forced cluster-split sweeps */
#define WT_OPT_SVD_CTAS_PER_SM 1  /* 0: host rule; k: at most k resident sweep CTAs per SM */
#define WT_OPT_SVD_PAIR_SKIP 2    /* 1: skip pair visits certified clean (default) */
#define WT_OPT_SVD_PERSIST 3      /* 1: one persistent launch per sweep (default); 0: one per round */
#define WT_OPT_SVD_PRECOND 4      /* 1: Gram-eigenbasis preconditioner for n >= 128 (default) */
#define WT_OPT_SVD_PROFILE 5      /* 1: K4 per-visit phase cycle counters on stderr */
#define WT_OPT_SVD_TRACE 6        /* 1: K4 per-sweep convergence trace on stderr */
#define WT_OPT_EIG_PROFILE 7      /* 1: preconditioner phase times on stderr */
#define WT_OPT_EIG_TWOSTAGE 8     /* 1: two-stage tridiagonalization for wide Grams in leading-triplet mode (default) */
#define WT_OPT_GEMM_TMA 9         /* 1: K3 large tiles fed by tensor-map TMA boxes (default); 0: cp.async ring */
#define WT_OPT_EIG_SPLIT 10       /* 0: host rule; 1: never; 2, 3, 4: always run the two-stage reduction as that many groups of matrices on their own streams */
#define WT_OPT_COUNT 11
int wt_set_option(int option, int value);

/* Sweeps used by the last wt_svd_jacobi_f64 call on the calling thread, and
 * the FP64 flops its Jacobi iteration executed (Gram + rotation tiles of every
 * rotated pair visit) -- the denominator-free work measure for the roofline. */
int wt_svd_last_sweeps(void);
/* Matrices of the last wt_svd_jacobi_f64 call (this thread) whose Gram-eigenbasis
 * preconditioner fell back to the identity, or -1 when the call ran without it. */
int wt_svd_last_fallbacks(void);
double wt_svd_last_jacobi_flops(void);

#ifdef __cplusplus
}
#endif

#endif /* WTEN_B200_H */
