// K1 / K2: fused multilevel lazy-lifting transform along mode 3 (the tube axis).
//
// Reference semantics (bit-exact):
//   forward level (lifting.py:63-66):  d = x[2k] - x[2k+1];  s = x[2k+1] + d/2
//   inverse level (lifting.py:69-74):  x[2k+1] = s - d/2;    x[2k] = d + x[2k+1]
// Halving is exact in IEEE-754, so __dmul_rn(d, 0.5) == d/2 and every result is
// the same correctly-rounded double the numpy reference produces.
//
// B200 design:
//   * A CTA owns a tile of TQ consecutive tubes x CT consecutive bands (CT a
//     multiple of 2^L: lifting has no halo across 2^L-band chunks), so all L
//     levels run in one pass over HBM: 8 B read + 8 B written per element.
//   * The tile is staged in shared memory by the TMA bulk-copy engine
//     (cp.async.bulk, one copy per tube row, mbarrier completion) -- the
//     tube-major input rows are contiguous.  Row pitch CT+2 doubles makes the
//     (2k, 2k+1) pair reads conflict-free double2 LDS.
//   * Slice-major outputs are written with consecutive threads on consecutive
//     tubes: every packed slice row segment is a contiguous TQ*8-byte burst.
//   * Inverse: the finished tube rows go back to HBM with bulk shared->global
//     copies.
#include <algorithm>

#include "wt_common.cuh"

namespace wt {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxTileElems = 8192;                 // TQ * CT
constexpr int kMaxItems = kMaxTileElems / 2 / kThreads;  // register staging depth (16)

struct LiftGeom {
  int64_t ntubes, p;
  int L;
  int TQ, CT, LDT;  // tile tubes, tile bands, smem row pitch (doubles)
  int64_t slice_base;
  int layout;
  uint64_t mask;
};

__host__ __device__ __forceinline__ int64_t detail_off(int64_t p, int j) {
  // first packed slice of detail level j (1-based): p - p/2^(j-1)
  return p - (p >> (j - 1));
}
__host__ __device__ __forceinline__ int64_t smooth_off(int64_t p, int L) { return p - (p >> L); }

// Output/input address of element k (0-based within the block) of packed block
// `blk_off` (first slice), holding `cnt` slices, for tube q.
__device__ __forceinline__ int64_t pyr_index(const LiftGeom& g, int64_t blk_off, int64_t cnt,
                                             int64_t q, int64_t k) {
  if (g.layout == WT_LAYOUT_SLICE_MAJOR) return (blk_off + k - g.slice_base) * g.ntubes + q;
  return (blk_off - g.slice_base) * g.ntubes + q * cnt + k;
}

// Stage rows [q0, q0+tq) x [t0, t0+CT) of the tube-major tensor into smem.
__device__ __forceinline__ void load_tile(double* tile, const double* __restrict__ x,
                                          const LiftGeom& g, int64_t q0, int tq, int64_t t0,
                                          bool bulk, uint64_t* bar) {
  if (bulk) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) mbar_expect_tx(bar, (uint32_t)(tq * g.CT * 8));
      __syncwarp();
      for (int r = threadIdx.x; r < tq; r += 32)
        bulk_g2s(tile + r * g.LDT, x + (q0 + r) * g.p + t0, (uint32_t)(g.CT * 8), bar);
    }
    mbar_wait(bar, 0);
  } else {
    const int n = tq * g.CT;
    for (int e = threadIdx.x; e < n; e += kThreads) {
      int r = e / g.CT, t = e - r * g.CT;
      tile[r * g.LDT + t] = __ldg(x + (q0 + r) * g.p + t0 + t);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) lift_fwd_kernel(const double* __restrict__ x,
                                                            double* __restrict__ out,
                                                            LiftGeom g, bool bulk) {
  extern __shared__ __align__(128) double tile[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t q0 = (int64_t)blockIdx.x * g.TQ;
  const int tq = (int)(g.ntubes - q0 < g.TQ ? g.ntubes - q0 : g.TQ);
  const int64_t t0 = (int64_t)blockIdx.y * g.CT;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  load_tile(tile, x, g, q0, tq, t0, bulk, &bar);

  const bool tube_out = g.layout == WT_LAYOUT_TUBE_MAJOR;
  int ell = g.CT;
  if (g.L == 0) {  // pure tube-major -> slice-major transpose
    if (g.mask & 1) {
      const int n = tq * ell;
      for (int e = threadIdx.x; e < n; e += kThreads) {
        int r, k;
        if (tube_out) { r = e / ell; k = e - r * ell; } else { k = e / tq; r = e - k * tq; }
        out[pyr_index(g, 0, g.p, q0 + r, t0 + k)] = tile[r * g.LDT + k];
      }
    }
    return;
  }
  for (int j = 1; j <= g.L; ++j) {
    const int half = ell >> 1;
    const int n = tq * half;
    const bool last = (j == g.L);
    const bool want_d = (g.mask >> j) & 1;
    const bool want_s = last && (g.mask & 1);
    const int64_t dcnt = g.p >> j;
    const int64_t doff = detail_off(g.p, j);
    const int64_t kbase = t0 >> j;
    double sreg[kMaxItems];
#pragma unroll
    for (int it = 0; it < kMaxItems; ++it) {
      const int e = threadIdx.x + it * kThreads;
      if (e < n) {
        int r, k;
        if (tube_out) { r = e / half; k = e - r * half; } else { k = e / tq; r = e - k * tq; }
        const double2 v = *reinterpret_cast<const double2*>(tile + r * g.LDT + 2 * k);
        const double d = __dsub_rn(v.x, v.y);
        const double s = __dadd_rn(v.y, __dmul_rn(d, 0.5));
        if (want_d) out[pyr_index(g, doff, dcnt, q0 + r, kbase + k)] = d;
        if (last) {
          if (want_s) out[pyr_index(g, smooth_off(g.p, g.L), dcnt, q0 + r, kbase + k)] = s;
        } else {
          sreg[it] = s;
        }
      }
    }
    if (last) break;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kMaxItems; ++it) {
      const int e = threadIdx.x + it * kThreads;
      if (e < n) {
        int r, k;
        if (tube_out) { r = e / half; k = e - r * half; } else { k = e / tq; r = e - k * tq; }
        tile[r * g.LDT + k] = sreg[it];
      }
    }
    __syncthreads();
    ell = half;
  }
}

__global__ void __launch_bounds__(kThreads) lift_inv_kernel(const double* __restrict__ pyr,
                                                            double* __restrict__ y, LiftGeom g,
                                                            bool bulk) {
  extern __shared__ __align__(128) double tile[];
  const int64_t q0 = (int64_t)blockIdx.x * g.TQ;
  const int tq = (int)(g.ntubes - q0 < g.TQ ? g.ntubes - q0 : g.TQ);
  const int64_t t0 = (int64_t)blockIdx.y * g.CT;
  const bool tube_in = g.layout == WT_LAYOUT_TUBE_MAJOR;

  // coarsest smooth block -> smem
  {
    const int ms = g.CT >> g.L;
    const int n = tq * ms;
    const int64_t scnt = g.p >> g.L;
    const int64_t soff = smooth_off(g.p, g.L);
    const bool have = g.mask & 1;
    for (int e = threadIdx.x; e < n; e += kThreads) {
      int r, k;
      if (tube_in) { r = e / ms; k = e - r * ms; } else { k = e / tq; r = e - k * tq; }
      tile[r * g.LDT + k] = have ? __ldg(pyr + pyr_index(g, soff, scnt, q0 + r, (t0 >> g.L) + k)) : 0.0;
    }
  }
  __syncthreads();
  for (int j = g.L; j >= 1; --j) {
    const int half = g.CT >> j;
    const int n = tq * half;
    const bool have_d = (g.mask >> j) & 1;
    const int64_t dcnt = g.p >> j;
    const int64_t doff = detail_off(g.p, j);
    const int64_t kbase = t0 >> j;
    double2 oreg[kMaxItems];
#pragma unroll
    for (int it = 0; it < kMaxItems; ++it) {
      const int e = threadIdx.x + it * kThreads;
      if (e < n) {
        int r, k;
        if (tube_in) { r = e / half; k = e - r * half; } else { k = e / tq; r = e - k * tq; }
        const double s = tile[r * g.LDT + k];
        const double d = have_d ? __ldg(pyr + pyr_index(g, doff, dcnt, q0 + r, kbase + k)) : 0.0;
        const double x1 = __dsub_rn(s, __dmul_rn(d, 0.5));
        oreg[it] = make_double2(__dadd_rn(d, x1), x1);
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kMaxItems; ++it) {
      const int e = threadIdx.x + it * kThreads;
      if (e < n) {
        int r, k;
        if (tube_in) { r = e / half; k = e - r * half; } else { k = e / tq; r = e - k * tq; }
        *reinterpret_cast<double2*>(tile + r * g.LDT + 2 * k) = oreg[it];
      }
    }
    __syncthreads();
  }
  // tile rows -> tube-major output
  if (bulk) {
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x < 32) {
      for (int r = threadIdx.x; r < tq; r += 32)
        bulk_s2g(y + (q0 + r) * g.p + t0, tile + r * g.LDT, (uint32_t)(g.CT * 8));
      bulk_commit();
      bulk_wait_all();
    }
  } else {
    const int n = tq * g.CT;
    for (int e = threadIdx.x; e < n; e += kThreads) {
      int r = e / g.CT, t = e - r * g.CT;
      y[(q0 + r) * g.p + t0 + t] = tile[r * g.LDT + t];
    }
  }
}

// ----------------------------------------------------------------------------
// Per-level fallback for 2^L-band chunks larger than one tile (L > 13): one
// launch per level through stream-ordered scratch.  Same arithmetic, any L.
__global__ void lift_fwd_level(const double* __restrict__ src, int64_t len, double* __restrict__ dst,
                               double* __restrict__ out, LiftGeom g, int j) {
  const int64_t half = len / 2, total = g.ntubes * half;
  const bool want_d = (g.mask >> j) & 1, last = (j == g.L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / half, k = e - q * half;
    const double a = src[q * len + 2 * k], b = src[q * len + 2 * k + 1];
    const double d = __dsub_rn(a, b);
    const double s = __dadd_rn(b, __dmul_rn(d, 0.5));
    if (want_d) out[pyr_index(g, detail_off(g.p, j), half, q, k)] = d;
    if (!last) dst[q * half + k] = s;
    else if (g.mask & 1) out[pyr_index(g, smooth_off(g.p, g.L), half, q, k)] = s;
  }
}

__global__ void lift_inv_level(const double* __restrict__ src, const double* __restrict__ pyr,
                               double* __restrict__ dst, LiftGeom g, int j) {
  const int64_t half = g.p >> j, total = g.ntubes * half;
  const bool have_d = (g.mask >> j) & 1, top = (j == g.L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / half, k = e - q * half;
    const double s = top ? ((g.mask & 1) ? pyr[pyr_index(g, smooth_off(g.p, g.L), half, q, k)] : 0.0)
                         : src[q * half + k];
    const double d = have_d ? pyr[pyr_index(g, detail_off(g.p, j), half, q, k)] : 0.0;
    const double x1 = __dsub_rn(s, __dmul_rn(d, 0.5));
    dst[q * 2 * half + 2 * k] = __dadd_rn(d, x1);
    dst[q * 2 * half + 2 * k + 1] = x1;
  }
}

int levelwise_forward(const double* x, double* out, const LiftGeom& g, cudaStream_t st) {
  double *t0 = nullptr, *t1 = nullptr;
  const size_t bytes = sizeof(double) * (size_t)g.ntubes * (size_t)(g.p / 2);
  WT_CUDA(cudaMallocAsync(&t0, bytes, st));
  WT_CUDA(cudaMallocAsync(&t1, bytes, st));
  const double* src = x;
  int64_t len = g.p;
  for (int j = 1; j <= g.L; ++j) {
    double* dst = (j & 1) ? t0 : t1;
    const int64_t total = g.ntubes * (len / 2);
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
    lift_fwd_level<<<grid, 256, 0, st>>>(src, len, dst, out, g, j);
    src = dst;
    len /= 2;
  }
  WT_CUDA(cudaFreeAsync(t0, st));
  WT_CUDA(cudaFreeAsync(t1, st));
  return check_launch("wt_lift_fwd_f64 (levelwise)");
}

int levelwise_inverse(const double* pyr, double* y, const LiftGeom& g, cudaStream_t st) {
  double *t0 = nullptr, *t1 = nullptr;
  const size_t bytes = sizeof(double) * (size_t)g.ntubes * (size_t)(g.p / 2);
  WT_CUDA(cudaMallocAsync(&t0, bytes, st));
  WT_CUDA(cudaMallocAsync(&t1, bytes, st));
  const double* src = nullptr;
  for (int j = g.L; j >= 1; --j) {
    double* dst = j == 1 ? y : ((j & 1) ? t0 : t1);
    const int64_t total = g.ntubes * (g.p >> j);
    const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
    lift_inv_level<<<grid, 256, 0, st>>>(src, pyr, dst, g, j);
    src = dst;
  }
  WT_CUDA(cudaFreeAsync(t0, st));
  WT_CUDA(cudaFreeAsync(t1, st));
  return check_launch("wt_lift_inv_f64 (levelwise)");
}

// Choose the tile: TQ tubes x CT bands, CT = 2^L * d with d | p/2^L.
int plan_tiles(LiftGeom& g) {
  const int64_t unit = (int64_t)1 << g.L;
  const int64_t munits = g.p / unit;
  for (int tq = 32; tq >= 1; tq >>= 1) {
    const int64_t cap = kMaxTileElems / tq;
    if (unit > cap) continue;
    int64_t best = 0;
    for (int64_t d = 1; d <= munits && unit * d <= cap; ++d)
      if (munits % d == 0) best = d;
    g.TQ = tq;
    g.CT = (int)(unit * best);
    g.LDT = g.CT + (g.CT % 2 == 0 ? 2 : 1);
    return WT_OK;
  }
  return WT_ERR_UNSUPPORTED;  // caller switches to the per-level path
}

int validate(int64_t n1, int64_t n2, int64_t p, int levels, int layout, int64_t slice_base) {
  WT_REQUIRE(n1 >= 0 && n2 >= 0 && p >= 1, "lifting: bad shape (%lld, %lld, %lld)",
             (long long)n1, (long long)n2, (long long)p);
  WT_REQUIRE(levels >= 0 && levels < 63 && (p % ((int64_t)1 << levels)) == 0,
             "lifting: 2**%d does not divide slice count %lld", levels, (long long)p);
  WT_REQUIRE(layout == WT_LAYOUT_SLICE_MAJOR || layout == WT_LAYOUT_TUBE_MAJOR,
             "lifting: unknown layout %d", layout);
  WT_REQUIRE(slice_base >= 0 && slice_base < p, "lifting: slice_base %lld out of range",
             (long long)slice_base);
  return WT_OK;
}

// dst (b x a) = transpose of src (a x b), both densely row-major, through
// wt_copy2d_f64 in batches that respect its grid limits.
int transpose_dense(const double* src, int64_t a, int64_t b, double* dst, cudaStream_t st) {
  constexpr int64_t kRows = 1 << 20;  // dst rows per batch item (grid.y = kRows / 32)
  int64_t done = 0;
  while (done < b) {
    const int64_t rows = std::min<int64_t>(kRows, b - done);
    const int64_t batch = std::min<int64_t>((b - done) / rows, 65535);
    int e = wt_copy2d_f64(src + done, b, rows, dst + done * a, a, rows * a, rows, a, batch, 1, st);
    if (e) return e;
    done += rows * batch;
  }
  return WT_OK;
}

// Tube-major (reference-layout) pyramids through the slice-major fast kernels:
// each packed block is one dense transpose away from the other layout, so the
// TUBE layout costs one extra HBM pass per block instead of the one-tile-per-CTA
// per-level kernel above (~1.3-3.3 TB/s, tools/lift_tq_probe.py round 1).
template <typename F>
int for_each_block(int64_t p, int L, int64_t slice_base, uint64_t mask, F f) {
  for (int j = 1; j <= L + 1; ++j) {
    const bool smooth = j > L;
    const int64_t off = smooth ? smooth_off(p, L) : detail_off(p, j);
    const int64_t cnt = p >> (smooth ? L : j);
    if (!((mask >> (smooth ? 0 : j)) & 1) || off < slice_base) continue;
    if (int e = f(off - slice_base, cnt)) return e;
  }
  return WT_OK;
}

}  // namespace

int lift_fwd_fast(const double* x, int64_t ntubes, int64_t p, int L, double* out,
                  int64_t slice_base, uint64_t mask, cudaStream_t st,
                  const unsigned long long* tab = nullptr);
int lift_inv_fast(const double* pyr, int64_t ntubes, int64_t p, int L, double* y,
                  int64_t slice_base, uint64_t mask, cudaStream_t st,
                  const unsigned long long* tab = nullptr);
}  // namespace wt

using namespace wt;

extern "C" int wt_lift_fwd_f64(const double* x, int64_t n1, int64_t n2, int64_t p, int levels,
                               double* out, int layout, int64_t slice_base, uint64_t level_mask,
                               void* stream) {
  int st = validate(n1, n2, p, levels, layout, slice_base);
  if (st) return st;
  LiftGeom g{n1 * n2, p, levels, 0, 0, 0, slice_base, layout, level_mask};
  if (g.ntubes == 0) return WT_OK;
  if (levels == 0 && layout == WT_LAYOUT_SLICE_MAJOR && slice_base == 0 && (level_mask & 1)) {
    // level 0 is the plain tube -> slice relayout (slicewise_matmul staging,
    // algebra.py:26-27): one dense transpose at copy bandwidth
    st = transpose_dense(x, g.ntubes, p, out, (cudaStream_t)stream);
    return st ? st : check_launch("wt_lift_fwd_f64 (level 0)");
  }
  if (layout == WT_LAYOUT_SLICE_MAJOR) {
    st = lift_fwd_fast(x, g.ntubes, p, levels, out, slice_base, level_mask, (cudaStream_t)stream);
    if (st != WT_ERR_UNSUPPORTED) return st;
  } else if (levels >= 1 && p % 2 == 0 && (uintptr_t)x % 16 == 0) {
    cudaStream_t cs = (cudaStream_t)stream;
    double* tmp = nullptr;
    WT_CUDA(cudaMallocAsync(&tmp, (size_t)(p - slice_base) * g.ntubes * sizeof(double), cs));
    st = lift_fwd_fast(x, g.ntubes, p, levels, tmp, slice_base, level_mask, cs);
    if (st == WT_OK)
      st = for_each_block(p, levels, slice_base, level_mask, [&](int64_t o, int64_t cnt) {
        return transpose_dense(tmp + o * g.ntubes, cnt, g.ntubes, out + o * g.ntubes, cs);
      });
    WT_CUDA(cudaFreeAsync(tmp, cs));
    if (st != WT_ERR_UNSUPPORTED) return st ? st : check_launch("wt_lift_fwd_f64 (tube layout)");
  }
  if (plan_tiles(g) != WT_OK) return levelwise_forward(x, out, g, (cudaStream_t)stream);
  const bool bulk = (g.CT % 2 == 0) && (p % 2 == 0) && ((uintptr_t)x % 16 == 0);
  const size_t smem = (size_t)g.TQ * g.LDT * sizeof(double);
  if (int e = ensure_smem(lift_fwd_kernel, kMaxTileElems * 8 + 4096)) return e;
  dim3 grid((unsigned)((g.ntubes + g.TQ - 1) / g.TQ), (unsigned)(p / g.CT));
  WT_REQUIRE(grid.y <= 65535, "lifting: too many band chunks");
  lift_fwd_kernel<<<grid, kThreads, smem, (cudaStream_t)stream>>>(x, out, g, bulk);
  return check_launch("wt_lift_fwd_f64");
}

extern "C" int wt_lift_inv_f64(const double* pyr, int64_t n1, int64_t n2, int64_t p, int levels,
                               int layout, int64_t slice_base, uint64_t level_mask, double* y,
                               void* stream) {
  int st = validate(n1, n2, p, levels, layout, slice_base);
  if (st) return st;
  LiftGeom g{n1 * n2, p, levels, 0, 0, 0, slice_base, layout, level_mask};
  if (g.ntubes == 0) return WT_OK;
  if (levels == 0 && layout == WT_LAYOUT_SLICE_MAJOR && slice_base == 0 && (level_mask & 1)) {
    st = transpose_dense(pyr, p, g.ntubes, y, (cudaStream_t)stream);  // slices -> tubes
    return st ? st : check_launch("wt_lift_inv_f64 (level 0)");
  }
  if (layout == WT_LAYOUT_SLICE_MAJOR) {
    st = lift_inv_fast(pyr, g.ntubes, p, levels, y, slice_base, level_mask, (cudaStream_t)stream);
    if (st != WT_ERR_UNSUPPORTED) return st;
  } else if (levels >= 1 && p % 2 == 0 && g.ntubes % 2 == 0 && (uintptr_t)y % 16 == 0) {
    cudaStream_t cs = (cudaStream_t)stream;
    double* tmp = nullptr;
    WT_CUDA(cudaMallocAsync(&tmp, (size_t)(p - slice_base) * g.ntubes * sizeof(double), cs));
    st = for_each_block(p, levels, slice_base, level_mask, [&](int64_t o, int64_t cnt) {
      return transpose_dense(pyr + o * g.ntubes, g.ntubes, cnt, tmp + o * g.ntubes, cs);
    });
    if (st == WT_OK) st = lift_inv_fast(tmp, g.ntubes, p, levels, y, slice_base, level_mask, cs);
    WT_CUDA(cudaFreeAsync(tmp, cs));
    if (st != WT_ERR_UNSUPPORTED) return st ? st : check_launch("wt_lift_inv_f64 (tube layout)");
  }
  if (plan_tiles(g) != WT_OK) return levelwise_inverse(pyr, y, g, (cudaStream_t)stream);
  const bool bulk = (g.CT % 2 == 0) && (p % 2 == 0) && ((uintptr_t)y % 16 == 0);
  const size_t smem = (size_t)g.TQ * g.LDT * sizeof(double);
  if (int e = ensure_smem(lift_inv_kernel, kMaxTileElems * 8 + 4096)) return e;
  dim3 grid((unsigned)((g.ntubes + g.TQ - 1) / g.TQ), (unsigned)(p / g.CT));
  WT_REQUIRE(grid.y <= 65535, "lifting: too many band chunks");
  lift_inv_kernel<<<grid, kThreads, smem, (cudaStream_t)stream>>>(pyr, y, g, bulk);
  return check_launch("wt_lift_inv_f64");
}

extern "C" int wt_lift_fwd_f64_peer(const double* x, int64_t n1, int64_t n2, int64_t p, int levels,
                                    const unsigned long long* slice_ptrs, int64_t slice_base,
                                    uint64_t level_mask, void* stream) {
  int st = validate(n1, n2, p, levels, WT_LAYOUT_SLICE_MAJOR, slice_base);
  if (st) return st;
  WT_REQUIRE(slice_ptrs != nullptr, "lifting: null slice pointer table");
  if (n1 * n2 == 0) return WT_OK;
  // dummy non-null base: every address comes from the table
  st = lift_fwd_fast(x, n1 * n2, p, levels, reinterpret_cast<double*>(16), slice_base, level_mask,
                     (cudaStream_t)stream, slice_ptrs);
  if (st == WT_ERR_UNSUPPORTED)
    set_error("wt_lift_fwd_f64_peer: needs levels >= 1, even p, 16-byte aligned x");
  return st;
}

extern "C" int wt_lift_inv_f64_peer(const unsigned long long* slice_ptrs, int64_t n1, int64_t n2,
                                    int64_t p, int levels, int64_t slice_base, uint64_t level_mask,
                                    double* y, void* stream) {
  int st = validate(n1, n2, p, levels, WT_LAYOUT_SLICE_MAJOR, slice_base);
  if (st) return st;
  WT_REQUIRE(slice_ptrs != nullptr, "lifting: null slice pointer table");
  if (n1 * n2 == 0) return WT_OK;
  st = lift_inv_fast(reinterpret_cast<const double*>(16), n1 * n2, p, levels, y, slice_base,
                     level_mask, (cudaStream_t)stream, slice_ptrs);
  if (st == WT_ERR_UNSUPPORTED)
    set_error("wt_lift_inv_f64_peer: needs levels >= 1, even p, even n1*n2, aligned y");
  return st;
}
