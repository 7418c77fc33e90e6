// Small memory-bound helpers around the hot path:
//   * column scaling (epilogues K5/K6/K7: Sigma, Sigma^-1, pinv cutoff weights),
//   * strided batched 2-D copy / transpose (slicewise transpose tensor.py:50-52,
//     sharded row<->slice permutations),
//   * deterministic per-band reductions (PSNR/SSIM moments, Frobenius norms).
#include <algorithm>

#include "wt_common.cuh"

namespace wt {
namespace {

// CTA (x, b): rows x, x + gridDim.x, ... of matrix b; threads own columns, so
// each thread forms its column factors once (no per-element index division)
// and every row access is coalesced.  clim (nullable): columns >= clim[b] are
// left untouched (the ranked pseudo-inverse never reads them).
__global__ void scale_cols_kernel(double* __restrict__ M, int64_t rows, int64_t ncols, int64_t ld,
                                  int64_t sM, const double* __restrict__ s, int64_t q, int mode,
                                  double tol, const int* __restrict__ clim) {
  const int64_t b = blockIdx.y;
  const int64_t nc = clim ? std::min<int64_t>(ncols, std::max(clim[b], 0)) : ncols;
  const double* sb = s + b * q;
  const double smax = sb[0];
  double* Mb = M + b * sM;
  for (int64_t j = threadIdx.x; j < nc; j += blockDim.x) {
    const double sv = sb[j];
    double f;
    if (mode == WT_SCALE_MUL) {
      f = sv;
    } else if (mode == WT_SCALE_DIV) {
      f = sv != 0.0 ? 1.0 / sv : 0.0;
    } else {  // WT_SCALE_PINV2: 1/s applied twice on kept values (decomposition.py:160-161);
              // (x / s) / s, never x * (1/s)^2: 1/s^2 overflows for s < ~1.5e-154
      const double inv = (sv > tol * smax && sv > 0.0) ? 1.0 / sv : 0.0;
      for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) Mb[i * ld + j] = (Mb[i * ld + j] * inv) * inv;
      continue;
    }
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) Mb[i * ld + j] *= f;
  }
}

template <bool TRANS>
__global__ void copy2d_kernel(const double* __restrict__ src, int64_t lds, int64_t sS,
                              double* __restrict__ dst, int64_t ldd, int64_t sD, int64_t rows,
                              int64_t cols) {
  // 32x32 tiles through shared memory so both sides are coalesced when TRANS.
  __shared__ double tile[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const double* S = src + b * sS;
  double* D = dst + b * sD;
  if (TRANS) {
    // dst[r][c] = src[c][r]: read src rows c0.., cols r0..
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int64_t sr = c0 + k, sc = r0 + threadIdx.x;
      if (sr < cols && sc < rows) tile[k][threadIdx.x] = S[sr * lds + sc];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int64_t dr = r0 + k, dc = c0 + threadIdx.x;
      if (dr < rows && dc < cols) D[dr * ldd + dc] = tile[threadIdx.x][k];
    }
  } else {
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int64_t r = r0 + k, c = c0 + threadIdx.x;
      if (r < rows && c < cols) D[r * ldd + c] = S[r * lds + c];
    }
  }
}

// Per-band partial sums over a chunk of tubes: x is (ntubes, p) tube-major.
__global__ void band_reduce_partial(const double* __restrict__ x, const double* __restrict__ y,
                                    int64_t ntubes, int64_t p, int mode, int64_t tubes_per_cta,
                                    double* __restrict__ part) {
  __shared__ double red[8][33];
  const int64_t k = (int64_t)blockIdx.y * 32 + threadIdx.x;
  const int64_t q0 = (int64_t)blockIdx.x * tubes_per_cta;
  const int64_t q1 = std::min<int64_t>(q0 + tubes_per_cta, ntubes);
  double acc = 0.0;
  if (k < p) {
    for (int64_t q = q0 + threadIdx.y; q < q1; q += 8) {
      const double a = x[q * p + k];
      double v;
      switch (mode) {
        case 0: v = a * a; break;
        case 1: { const double d = a - y[q * p + k]; v = d * d; } break;
        case 2: v = a; break;
        default: v = a * y[q * p + k]; break;
      }
      acc += v;
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && k < p) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += red[t][threadIdx.x];
    part[(int64_t)blockIdx.x * p + k] = s;
  }
}

__global__ void band_reduce_final(const double* __restrict__ part, int64_t nparts, int64_t p,
                                  double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p;
       k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i < nparts; ++i) s += part[i * p + k];
    out[k] = s;
  }
}

}  // namespace
}  // namespace wt

using namespace wt;

int wt::scale_cols_lim(double* M, int64_t rows, int64_t ncols, int64_t ld, int64_t strideM,
                       const double* s, int64_t q, int64_t batch, int mode, double tol,
                       const int* clim, void* stream) {
  WT_REQUIRE(rows >= 0 && ncols >= 0 && batch >= 0 && ncols <= q && ld >= ncols,
             "scale_cols: bad arguments");
  WT_REQUIRE(mode >= WT_SCALE_MUL && mode <= WT_SCALE_PINV2, "scale_cols: bad mode %d", mode);
  if (rows == 0 || ncols == 0 || batch == 0) return WT_OK;
  const int threads = ncols >= 256 ? 256 : (int)((ncols + 31) / 32 * 32);
  // enough CTAs to cover the GPU several times over, each streaming a few rows
  const int64_t want = std::max<int64_t>(1, 8 * num_sms() / std::max<int64_t>(batch, 1));
  const unsigned gx = (unsigned)std::min<int64_t>(rows, want);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {  // grid.y limit
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    scale_cols_kernel<<<dim3(gx, (unsigned)nb), threads, 0, (cudaStream_t)stream>>>(
        M + b0 * strideM, rows, ncols, ld, strideM, s + b0 * q, q, mode, tol,
        clim ? clim + b0 : nullptr);
  }
  return check_launch("wt_scale_cols_f64");
}

extern "C" int wt_scale_cols_f64(double* M, int64_t rows, int64_t ncols, int64_t ld,
                                 int64_t strideM, const double* s, int64_t q, int64_t batch,
                                 int mode, double tol, void* stream) {
  return scale_cols_lim(M, rows, ncols, ld, strideM, s, q, batch, mode, tol, nullptr, stream);
}

extern "C" int wt_copy2d_f64(const double* src, int64_t lds, int64_t strideS, double* dst,
                             int64_t ldd, int64_t strideD, int64_t rows, int64_t cols,
                             int64_t batch, int trans, void* stream) {
  WT_REQUIRE(rows >= 0 && cols >= 0 && batch >= 0, "copy2d: negative size");
  if (rows == 0 || cols == 0 || batch == 0) return WT_OK;
  WT_REQUIRE((cols + 31) / 32 < (1LL << 31), "copy2d: too many columns");
  constexpr int64_t kRowChunk = 65535LL * 32;  // grid.y limit
  dim3 block(32, 8);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {  // grid.z limit
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    for (int64_t r0 = 0; r0 < rows; r0 += kRowChunk) {
      const int64_t nr = std::min<int64_t>(kRowChunk, rows - r0);
      // dst rows r0.. read src rows r0.. (copy) or src columns r0.. (transpose)
      const double* S = src + b0 * strideS + (trans ? r0 : r0 * lds);
      double* D = dst + b0 * strideD + r0 * ldd;
      dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((nr + 31) / 32), (unsigned)nb);
      if (trans)
        copy2d_kernel<true><<<grid, block, 0, (cudaStream_t)stream>>>(S, lds, strideS, D, ldd,
                                                                      strideD, nr, cols);
      else
        copy2d_kernel<false><<<grid, block, 0, (cudaStream_t)stream>>>(S, lds, strideS, D, ldd,
                                                                       strideD, nr, cols);
    }
  }
  return check_launch("wt_copy2d_f64");
}

// Tube deltas for the comparator DFT: out[t][k] = x[t][k] - x[t][0] (so out[t][0] = 0).
// DFT(x) = DFT(out) + p x_0 e_0: constant tubes then give exactly zero off-DC
// coefficients, as an FFT's butterflies do (baselines.py:68 np.fft.fft).
__global__ void tube_delta_kernel(const double* __restrict__ x, int64_t total, int64_t p,
                                  double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    out[e] = __dsub_rn(x[e], x[e - e % p]);
  }
}

extern "C" int wt_tube_delta_f64(const double* x, int64_t ntubes, int64_t p, double* out,
                                 void* stream) {
  WT_REQUIRE(ntubes >= 0 && p >= 1, "tube_delta: bad shape");
  const int64_t total = ntubes * p;
  if (total == 0) return WT_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  tube_delta_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, total, p, out);
  return check_launch("wt_tube_delta_f64");
}

size_t wt_band_reduce_parts(int64_t ntubes) {
  return (size_t)std::max<int64_t>(1, std::min<int64_t>(1184, (ntubes + 63) / 64));
}

extern "C" int wt_slice_reduce_f64(const double* x, const double* y, int64_t n, int64_t nslices,
                                   int mode, double* out, void* stream) {
  // x, y: spatial (n tubes, nslices bands) tube-major; out[k] = sum over tubes.
  // `out` must hold nslices * (1 + parts) doubles: the tail is scratch.
  WT_REQUIRE(n >= 0 && nslices >= 1, "slice_reduce: bad shape");
  WT_REQUIRE(mode >= 0 && mode <= 3, "slice_reduce: bad mode %d", mode);
  WT_REQUIRE((mode != 1 && mode != 3) || y != nullptr, "slice_reduce: y required");
  const int64_t parts = (int64_t)wt_band_reduce_parts(n);
  const int64_t per = (n + parts - 1) / parts;
  double* part = out + nslices;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)parts, (unsigned)((nslices + 31) / 32));
  WT_REQUIRE(grid.y <= 65535, "slice_reduce: too many bands");
  band_reduce_partial<<<grid, dim3(32, 8), 0, st>>>(x, y, n, nslices, mode, std::max<int64_t>(per, 1), part);
  if (int e = check_launch("band_reduce_partial")) return e;
  band_reduce_final<<<(unsigned)std::min<int64_t>((nslices + 255) / 256, 1024), 256, 0, st>>>(
      part, parts, nslices, out);
  return check_launch("band_reduce_final");
}

extern "C" size_t wt_slice_reduce_scratch(int64_t n, int64_t nslices) {
  return (size_t)nslices * (1 + wt_band_reduce_parts(n)) * sizeof(double);
}

namespace wt {
namespace {
// one warp per tube: source tubes in order (coalesced reads across warps), each
// tube copied with 16-byte vectors when p is even and the tubes 16-byte aligned
template <bool V2>
__global__ void tube_transpose_kernel(const double* __restrict__ x, int64_t n1, int64_t n2, int64_t p,
                                      double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  const int64_t nt = n1 * n2;
  for (int64_t t = blockIdx.x * wpb + (threadIdx.x >> 5); t < nt; t += (int64_t)gridDim.x * wpb) {
    const int64_t i = t / n2, j = t - i * n2;
    const double* src = x + t * p;
    double* dst = y + (j * n1 + i) * p;
    if (V2) {
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(dst);
      for (int64_t k = lane; k < p / 2; k += 32) d2[k] = s2[k];
    } else {
      for (int64_t k = lane; k < p; k += 32) dst[k] = src[k];
    }
  }
}
}  // namespace
}  // namespace wt

extern "C" int wt_tube_transpose_f64(const double* x, int64_t n1, int64_t n2, int64_t p, double* y,
                                     void* stream) {
  WT_REQUIRE(n1 >= 0 && n2 >= 0 && p >= 0, "tube_transpose: negative dimension");
  if (n1 * n2 * p == 0) return WT_OK;
  WT_REQUIRE(x && y, "tube_transpose: null pointer");
  const int64_t nt = n1 * n2;
  const unsigned grid = (unsigned)std::min<int64_t>((nt + 7) / 8, (int64_t)num_sms() * 16);
  const bool v2 = p % 2 == 0 && (uintptr_t)x % 16 == 0 && (uintptr_t)y % 16 == 0;
  if (v2)
    tube_transpose_kernel<true><<<grid, 256, 0, (cudaStream_t)stream>>>(x, n1, n2, p, y);
  else
    tube_transpose_kernel<false><<<grid, 256, 0, (cudaStream_t)stream>>>(x, n1, n2, p, y);
  return check_launch("wt_tube_transpose_f64");
}

// ----------------------------------------------------- orthonormal columns --
// Short-side singular vectors formed as (A v_j) / s_j lose orthogonality like
// eps s_max / s_j and are zero for s_j = 0 (K6, tensor.matrix_svd).  For every
// column j with s_j <= tau * s_max (in descending-sigma order) this kernel
// re-orthonormalises it against columns 0..j-1 by classical Gram-Schmidt done
// twice, and replaces a column with no independent part left (zero singular
// value) by the first unit vector e_k that has one -- so the columns are
// orthonormal to rounding, as LAPACK's are, and U diag(s) V^T is unchanged up
// to s_j times the correction.  One CTA per matrix; deterministic.
namespace wt {
namespace ortho {
constexpr int OT = 256;

__device__ double ortho_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < OT / 32; ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(OT) ortho_fixup_kernel(double* __restrict__ M, int64_t rows, int64_t r,
                                                         int64_t ld, int64_t cs, int64_t sM,
                                                         const double* __restrict__ s, int64_t q, double tau,
                                                         int skip_zero) {
  // element (row i, column j) at Mb[i * ld + j * cs]: (ld, 1) for rows x r blocks, (1, vector pitch)
  // for K4's vectors-as-rows output
  extern __shared__ double osm[];  // dots [r], red [8]
  double* dots = osm;
  double* red = osm + r;
  const int64_t b = blockIdx.x;
  double* Mb = M + b * sM;
  const double* sb = s + b * q;
  const double smax = sb[0];
  if (skip_zero && !(smax > 0.0)) return;  // an all-zero matrix: nothing refers to its vectors (K4's own pass)
  int64_t next_e = 0;  // next unit-vector candidate
  for (int64_t j = 0; j < r; ++j) {
    const double sj = sb[j];
    if (sj > tau * smax && sj > 0.0 && isfinite(sj)) continue;  // orthogonal to rounding already
    bool fresh = false;
    for (int attempt = 0; attempt <= rows; ++attempt) {
      if (fresh) {  // candidate e_k
        for (int64_t i = threadIdx.x; i < rows; i += OT) Mb[i * ld + j * cs] = (i == next_e) ? 1.0 : 0.0;
        ++next_e;
        __syncthreads();
      }
      double nrm0 = 0.0;
      for (int64_t i = threadIdx.x; i < rows; i += OT) nrm0 = fma(Mb[i * ld + j * cs], Mb[i * ld + j * cs], nrm0);
      nrm0 = sqrt(ortho_block_sum(nrm0, red));
      if (!(nrm0 > 0.0) || !isfinite(nrm0)) {  // nothing to orthogonalise: take a unit vector
        fresh = true;
        continue;
      }
      for (int pass = 0; pass < 2; ++pass) {
        // dots with the previous columns (warp per column, lanes over rows)
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int64_t c = warp; c < j; c += OT / 32) {
          double d = 0.0;
          for (int64_t i = lane; i < rows; i += 32) d = fma(Mb[i * ld + c * cs], Mb[i * ld + j * cs], d);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (lane == 0) dots[c] = d;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < rows; i += OT) {
          double v = Mb[i * ld + j * cs];
          for (int64_t c = 0; c < j; ++c) v = fma(-dots[c], Mb[i * ld + c * cs], v);
          Mb[i * ld + j * cs] = v;
        }
        __syncthreads();
      }
      double nrm = 0.0;
      for (int64_t i = threadIdx.x; i < rows; i += OT) nrm = fma(Mb[i * ld + j * cs], Mb[i * ld + j * cs], nrm);
      nrm = sqrt(ortho_block_sum(nrm, red));
      if (nrm > 0.5 * nrm0) {  // an independent direction survived: normalise it
        const double inv = 1.0 / nrm;
        for (int64_t i = threadIdx.x; i < rows; i += OT) Mb[i * ld + j * cs] *= inv;
        __syncthreads();
        break;
      }
      if (!fresh && nrm > 1e-8 * nrm0) {  // mostly dependent but not empty: keep its independent part
        const double inv = 1.0 / nrm;
        for (int64_t i = threadIdx.x; i < rows; i += OT) Mb[i * ld + j * cs] *= inv;
        __syncthreads();
        // one more round of orthogonalisation in the next attempt
        continue;
      }
      fresh = true;
    }
  }
}
}  // namespace ortho
}  // namespace wt

namespace wt {
int ortho_fixup_strided(double* M, int64_t rows, int64_t r, int64_t si, int64_t sj, int64_t strideM,
                        const double* s, int64_t q, int64_t batch, double tau, void* stream, int skip_zero) {
  if (batch == 0 || r == 0) return WT_OK;
  WT_REQUIRE(batch <= 2147483647, "orthonormal_fixup: batch too large");
  const size_t smem = sizeof(double) * (size_t)(r + ortho::OT / 32);
  if (int e = ensure_smem(ortho::ortho_fixup_kernel, smem)) return e;
  ortho::ortho_fixup_kernel<<<(unsigned)batch, ortho::OT, smem, (cudaStream_t)stream>>>(M, rows, r, si, sj, strideM,
                                                                                         s, q, tau, skip_zero);
  return check_launch("wt_orthonormal_fixup_f64");
}
}  // namespace wt

extern "C" int wt_orthonormal_fixup_f64(double* M, int64_t rows, int64_t r, int64_t ld, int64_t strideM,
                                        const double* s, int64_t q, int64_t batch, double tau, void* stream) {
  WT_REQUIRE(rows >= 0 && r >= 0 && r <= q && r <= rows && batch >= 0 && ld >= r, "orthonormal_fixup: bad shape");
  return wt::ortho_fixup_strided(M, rows, r, ld, 1, strideM, s, q, batch, tau, stream, 0);
}

// ------------------------------------------------------------ LU pivots --
// inverse_tensor's singularity rule (algebra.py:77-83: np.linalg.inv raises
// LinAlgError when LAPACK dgetrf meets an exactly zero pivot): Gaussian
// elimination with partial pivoting on a copy of every n x n slice; info[b] =
// 1 + the first column whose pivot is exactly zero, else 0.  One CTA per slice
// (off the hot path: only the ring constructor inverse_tensor calls it).
namespace wt {
namespace ortho {
__global__ void __launch_bounds__(OT) lu_pivot_kernel(double* __restrict__ W, int64_t n, int64_t sW,
                                                      int* __restrict__ info) {
  __shared__ double sval[OT / 32];
  __shared__ int64_t sidx[OT / 32];
  __shared__ int64_t piv;
  const int64_t b = blockIdx.x;
  double* A = W + b * sW;
  int res = 0;
  for (int64_t k = 0; k < n; ++k) {
    // pivot: largest |A[i][k]|, i >= k (lowest index on ties, as idamax)
    double best = -1.0;
    int64_t bi = n;
    for (int64_t i = k + threadIdx.x; i < n; i += OT) {
      const double v = fabs(A[i * n + k]);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { sval[threadIdx.x >> 5] = best; sidx[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bv = sval[0];
      int64_t bx = sidx[0];
      for (int w = 1; w < OT / 32; ++w)
        if (sval[w] > bv || (sval[w] == bv && sidx[w] < bx)) { bv = sval[w]; bx = sidx[w]; }
      piv = bv == 0.0 ? -1 : (bx < n ? bx : k);  // (a NaN column: no pivot order; the inverse check reports it)
    }
    __syncthreads();
    const int64_t p = piv;
    if (p < 0) { res = (int)k + 1; break; }  // exactly singular (uniform)
    if (p != k)
      for (int64_t c = threadIdx.x; c < n; c += OT) {
        const double t = A[k * n + c];
        A[k * n + c] = A[p * n + c];
        A[p * n + c] = t;
      }
    __syncthreads();
    const double inv = 1.0 / A[k * n + k];
    for (int64_t e = threadIdx.x; e < (n - k - 1) * (n - k); e += OT) {
      const int64_t i = k + 1 + e / (n - k), c = k + e % (n - k);
      const double l = A[i * n + k] * inv;
      if (c > k) A[i * n + c] = fma(-l, A[k * n + c], A[i * n + c]);
    }
    __syncthreads();
    for (int64_t i = k + 1 + threadIdx.x; i < n; i += OT) A[i * n + k] *= inv;
    __syncthreads();
  }
  if (threadIdx.x == 0) info[b] = res;
}
}  // namespace ortho
}  // namespace wt

extern "C" int wt_lu_pivot_check_f64(double* W, int64_t n, int64_t batch, int* info, void* stream) {
  WT_REQUIRE(n >= 0 && batch >= 0, "lu_pivot_check: bad shape");
  if (batch == 0) return WT_OK;
  if (n == 0) return cudaMemsetAsync(info, 0, sizeof(int) * (size_t)batch, (cudaStream_t)stream) == cudaSuccess
                         ? WT_OK : WT_ERR_CUDA;
  wt::ortho::lu_pivot_kernel<<<(unsigned)batch, wt::ortho::OT, 0, (cudaStream_t)stream>>>(W, n, n * n, info);
  return check_launch("wt_lu_pivot_check_f64");
}

// ------------------------------------------------------- diagonal blocks --
// S[b] (r x r row-major) = diag(s[b*q + 0 .. r-1]): the S factor blocks of
// w_svd (decomposition.py:75-82, _factor_blocks' np.diag per slice).
namespace wt {
namespace ortho {
__global__ void diag_blocks_kernel(const double* __restrict__ s, int64_t q, int64_t r, int64_t batch,
                                   double* __restrict__ S) {
  const int64_t total = batch * r * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / (r * r), rc = e - b * r * r, i = rc / r, j = rc - i * r;
    S[e] = i == j ? s[b * q + i] : 0.0;
  }
}
}  // namespace ortho
}  // namespace wt

extern "C" int wt_diag_blocks_f64(const double* s, int64_t q, int64_t r, int64_t batch, double* S, void* stream) {
  WT_REQUIRE(r >= 0 && r <= q && batch >= 0, "diag_blocks: bad shape");
  const int64_t total = batch * r * r;
  if (total == 0) return WT_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 4096);
  wt::ortho::diag_blocks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(s, q, r, batch, S);
  return check_launch("wt_diag_blocks_f64");
}

extern "C" int wt_readback_i32(const int* src, int* host_pinned, int64_t n, void* stream) {
  WT_REQUIRE(n >= 0 && n <= (int64_t)1 << 30, "readback: bad count %lld", (long long)n);
  if (n == 0) return WT_OK;
  WT_REQUIRE(src && host_pinned, "readback: null pointer");
  WT_CUDA(wt::readback_ints(host_pinned, src, (int)n, (cudaStream_t)stream));
  WT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return WT_OK;
}
