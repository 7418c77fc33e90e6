// Imaging helpers either side of the hot path (SPEC.md:447-548,
// BASELINE.json configs[2..4]): built in HBM so the 268 MB - 2 GiB operands of the
// deblur / w-svd configurations never cross PCIe.
//   * slice-constant Toeplitz blur operators,
//   * the synthetic-cube generator's heavy stages: reflect-mode Gaussian smoothing of the
//     abundance maps, abundances x spectra mixing, additive noise, clipping.
// All three are HBM-write-bound streaming kernels (8 B written per element).
#include <algorithm>

#include "wt_common.cuh"

namespace wt {
namespace img {

// out[i][j][k] = c[|i - j|] for |i - j| < nc, else 0; (n, n, p) tube-fastest.
// CTA (jc, i): row i, columns [jc * JT, ...); threads stream the row's (j, k) pairs.
constexpr int JT = 64;
__global__ void toeplitz_kernel(const double* __restrict__ c, int nc, int n, int p, double* __restrict__ out) {
  const int i = blockIdx.y, j0 = blockIdx.x * JT, j1 = min(n, j0 + JT);
  double* row = out + ((int64_t)i * n + j0) * p;
  const int total = (j1 - j0) * p;
  if ((p & 1) == 0) {
    const int p2 = p >> 1;
    for (int t = threadIdx.x; t < (total >> 1); t += blockDim.x) {
      const int j = j0 + t / p2, d = abs(i - j);
      const double v = d < nc ? c[d] : 0.0;
      reinterpret_cast<double2*>(row)[t] = make_double2(v, v);
    }
  } else {
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int j = j0 + t / p, d = abs(i - j);
      row[t] = d < nc ? c[d] : 0.0;
    }
  }
}

// scipy.ndimage 'reflect' (half-sample symmetric): ... c b a | a b c d | d c b ...
__device__ __forceinline__ int reflect(int i, int n) {
  const int per = 2 * n;
  i %= per;
  if (i < 0) i += per;
  return i < n ? i : per - 1 - i;
}

// One axis pass of the separable filter on x (n1, n2, e), e fastest:
// y[c] = x[c] w[0] + sum_{l = R .. 1} (x[c - l] + x[c + l]) w[l], farthest taps first,
// products and sums rounded separately (no contraction) so the result does not
// depend on the compiler's fusion choices.
__global__ void smooth_axis_kernel(const double* __restrict__ x, int n1, int n2, int e, int axis,
                                   const double* __restrict__ w, int radius, double* __restrict__ y) {
  const int64_t total = (int64_t)n1 * n2 * e;
  const int64_t stride = axis == 0 ? (int64_t)n2 * e : e;
  const int len = axis == 0 ? n1 : n2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = t / e;
    const int c = axis == 0 ? (int)(pix / n2) : (int)(pix % n2);
    const double* line = x + (t - (int64_t)c * stride);
    double acc = __dmul_rn(line[(int64_t)c * stride], w[0]);
    for (int l = radius; l >= 1; --l) {
      const double a = line[(int64_t)reflect(c - l, len) * stride];
      const double b = line[(int64_t)reflect(c + l, len) * stride];
      acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(a, b), w[l]));
    }
    y[t] = acc;
  }
}

// Philox-4x32-10 (Salmon et al. 2011), counter = (lo, hi, 0, 0), key = seed.
__device__ __forceinline__ uint4 philox(uint64_t ctr, uint64_t seed) {
  uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0u, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t h0 = __umulhi(0xD2511F53u, c0), l0 = 0xD2511F53u * c0;
    const uint32_t h1 = __umulhi(0xCD9E8D57u, c2), l1 = 0xCD9E8D57u * c2;
    c0 = h1 ^ c1 ^ k0;
    c1 = l1;
    c2 = h0 ^ c3 ^ k1;
    c3 = l0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {  // [0, 1)
  return (double)(((uint64_t)(hi >> 5) << 26) | (uint64_t)(lo >> 6)) * (1.0 / 9007199254740992.0);
}
// Two independent standard normals of element pair `pair` (Box-Muller).
__device__ __forceinline__ double2 normal_pair(uint64_t pair, uint64_t seed) {
  const uint4 r = philox(pair, seed);
  const double u1 = 1.0 - u53(r.x, r.y), u2 = u53(r.z, r.w);  // u1 in (0, 1]
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(rad * c, rad * s);
}

// out[pix][k] = clip(sum_j ab[pix][j] S[j][k] + sigma z, lo, hi).  A thread owns one band
// pair (k, k + 1) with its 2 x e spectra values in registers and walks the CTA's pixels;
// the pixels' abundances are staged in shared memory (broadcast reads).  z: noise[pix][k]
// if given, else the Philox stream at counter pix * ceil(p / 2) + k / 2.
constexpr int MIX_PIX = 32;   // pixels per staged tile
constexpr int MIX_T = 128;    // threads per CTA
template <int EMAX>
__global__ void __launch_bounds__(MIX_T) mix_kernel(const double* __restrict__ ab, const double* __restrict__ spectra,
                                                    int64_t npix, int e, int p, double sigma,
                                                    const double* __restrict__ noise, uint64_t seed, double lo,
                                                    double hi, double* __restrict__ out) {
  __shared__ double sab[MIX_PIX * EMAX];
  const int pp = (p + 1) >> 1;
  const bool vec = (p & 1) == 0;
  const int64_t ntiles = (npix + MIX_PIX - 1) / MIX_PIX;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t pix0 = tile * MIX_PIX;
    const int np = (int)min((int64_t)MIX_PIX, npix - pix0);
    __syncthreads();
    for (int t = threadIdx.x; t < np * e; t += MIX_T) sab[(t / e) * EMAX + (t % e)] = ab[pix0 * e + t];
    __syncthreads();
    for (int kp = threadIdx.x; kp < pp; kp += MIX_T) {
      const int k = 2 * kp;
      const bool two = k + 1 < p;
      double s0[EMAX], s1[EMAX];
#pragma unroll
      for (int j = 0; j < EMAX; ++j) {
        s0[j] = j < e ? spectra[j * p + k] : 0.0;
        s1[j] = (j < e && two) ? spectra[j * p + k + 1] : 0.0;
      }
      for (int i = 0; i < np; ++i) {
        const int64_t pix = pix0 + i;
        double v0 = 0.0, v1 = 0.0;
#pragma unroll
        for (int j = 0; j < EMAX; ++j) {
          const double a = sab[i * EMAX + j];   // zero-padded beyond e by s0/s1 = 0
          v0 = fma(j < e ? a : 0.0, s0[j], v0);
          v1 = fma(j < e ? a : 0.0, s1[j], v1);
        }
        if (sigma != 0.0) {
          double z0, z1 = 0.0;
          if (noise) {
            z0 = noise[pix * p + k];
            if (two) z1 = noise[pix * p + k + 1];
          } else {
            const double2 g = normal_pair((uint64_t)(pix * pp + kp), seed);
            z0 = g.x;
            z1 = g.y;
          }
          v0 = fma(sigma, z0, v0);
          v1 = fma(sigma, z1, v1);
        }
        v0 = fmin(fmax(v0, lo), hi);
        v1 = fmin(fmax(v1, lo), hi);
        double* o = out + pix * p + k;
        if (vec) {
          *reinterpret_cast<double2*>(o) = make_double2(v0, v1);
        } else {
          o[0] = v0;
          if (two) o[1] = v1;
        }
      }
    }
  }
}

}  // namespace img
}  // namespace wt

extern "C" int wt_toeplitz_tensor_f64(const double* c, int64_t nc, int64_t n, int64_t p, double* out, void* stream) {
  WT_REQUIRE(nc >= 0 && n >= 0 && p >= 0, "toeplitz_tensor: bad shape");
  WT_REQUIRE(n < 65536 && (int64_t)wt::img::JT * p < (1ll << 30), "toeplitz_tensor: n < 65536 and p < 2^24 supported");
  if (n == 0 || p == 0) return WT_OK;
  dim3 grid((unsigned)((n + wt::img::JT - 1) / wt::img::JT), (unsigned)n);
  wt::img::toeplitz_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(c, (int)std::min<int64_t>(nc, n), (int)n, (int)p, out);
  return wt::check_launch("wt_toeplitz_tensor_f64");
}

extern "C" int wt_gauss_smooth2d_f64(const double* x, int64_t n1, int64_t n2, int64_t e, const double* w,
                                     int64_t radius, double* tmp, double* out, void* stream) {
  WT_REQUIRE(n1 >= 0 && n2 >= 0 && e >= 0 && radius >= 0, "gauss_smooth2d: bad shape");
  WT_REQUIRE(n1 < (1ll << 30) && n2 < (1ll << 30) && radius < (1ll << 20), "gauss_smooth2d: extents too large");
  const int64_t total = n1 * n2 * e;
  if (total == 0) return WT_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)wt::num_sms() * 16);
  wt::img::smooth_axis_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, (int)n1, (int)n2, (int)e, 0, w, (int)radius, tmp);
  wt::img::smooth_axis_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(tmp, (int)n1, (int)n2, (int)e, 1, w, (int)radius, out);
  return wt::check_launch("wt_gauss_smooth2d_f64");
}

template <int EMAX>
static int launch_mix(const double* ab, const double* spectra, int64_t npix, int e, int p, double sigma,
                      const double* noise, uint64_t seed, double lo, double hi, double* out, cudaStream_t st) {
  const int64_t ntiles = (npix + wt::img::MIX_PIX - 1) / wt::img::MIX_PIX;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)wt::num_sms() * 16);
  wt::img::mix_kernel<EMAX><<<grid, wt::img::MIX_T, 0, st>>>(ab, spectra, npix, e, p, sigma, noise, seed, lo, hi, out);
  return wt::check_launch("wt_hsi_mix_f64");
}

extern "C" int wt_hsi_mix_f64(const double* ab, const double* spectra, int64_t npix, int64_t e, int64_t p,
                              double noise_sigma, const double* noise, uint64_t seed, double lo, double hi,
                              double* out, void* stream) {
  WT_REQUIRE(npix >= 0 && e >= 0 && p >= 0 && p < (1ll << 30), "hsi_mix: bad shape");
  WT_REQUIRE(e <= 32, "hsi_mix: at most 32 endmembers");
  if (npix * p == 0) return WT_OK;
  if (e <= 12)
    return launch_mix<12>(ab, spectra, npix, (int)e, (int)p, noise_sigma, noise, seed, lo, hi, out, (cudaStream_t)stream);
  return launch_mix<32>(ab, spectra, npix, (int)e, (int)p, noise_sigma, noise, seed, lo, hi, out, (cudaStream_t)stream);
}
