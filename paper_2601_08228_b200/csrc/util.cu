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
    } else {  // WT_SCALE_PINV2: (1/s)^2 on kept values (decomposition.py:160-161)
      const double inv = (sv > tol * smax && sv > 0.0) ? 1.0 / sv : 0.0;
      f = inv * inv;
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
