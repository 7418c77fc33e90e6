// K1 / K2 hot path: persistent, double-buffered lifting kernels for the
// slice-major pyramid (the layout the face GEMM and the SVD consume).
//
// Same arithmetic as lift.cu (bit-exact with lifting.py:63-74); the difference
// is the schedule:
//   * persistent CTAs (grid = SMs x resident CTAs) walk the tiles; the next
//     tile's input is in flight while the current one is lifted;
//   * forward input tiles arrive by TMA bulk copies (one per tube row, mbarrier
//     completion), inverse input rows by 16-byte cp.async;
//   * levels are processed in register-blocked stages of up to 3 levels: a
//     thread takes 2^W consecutive values of one tube, runs W levels in
//     registers and emits every detail directly -- one barrier per stage
//     instead of two per level (ncu: the per-level version was index-math and
//     barrier bound at L = 8);
//   * the tile height TQ (tubes) is a compile-time constant, so every index
//     split is a shift/mask; consecutive threads own consecutive tubes, so each
//     packed slice row is written / read as TQ*8-byte bursts.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>

#include "wt_common.cuh"

namespace wt {
namespace fast {

constexpr int kT = 256;
constexpr int kMaxElems = 4096;  // TQ * CT per tile (32 KB)
constexpr int kMaxTmaLevels = 12;

struct FGeom {
  int64_t ntubes, p;
  int L, CT;
  int LDT;         // forward: tube-major tile pitch (CT + 2)
  int LDA0, LDA1;  // stage buffers: CT/8 + 2, CT/64 + 2
  int64_t slice_base;
  uint64_t mask;
  uint32_t nqt, ntiles;
  // Optional per-slice row pointers (peer / symmetric-memory addressing): when
  // set, packed slice s of this rank's tubes lives at (double*)tab[s - slice_base]
  // (+ tube index) instead of out + (s - slice_base) * ntubes.  This is how the
  // sharded pipeline fuses its rows -> slices exchange into K1 / K2: the stores
  // (loads) go straight to (from) the owning GPU's buffer over NVLink.
  const unsigned long long* tab;
  int inv_path;  // K2: from this L up (0 = never), levels above 3 by per-thread ancestor chains
};

__device__ __forceinline__ double* slice_row(const FGeom& g, double* base, int64_t s) {
  return g.tab ? reinterpret_cast<double*>(g.tab[s - g.slice_base])
               : base + (s - g.slice_base) * g.ntubes;
}

__device__ __forceinline__ int64_t doff(int64_t p, int j) { return p - (p >> (j - 1)); }
__device__ __forceinline__ int64_t soff(int64_t p, int L) { return p - (p >> L); }

template <int TQ>
__device__ __forceinline__ void tile_at(const FGeom g, uint32_t t, int64_t& q0, int& tq, int64_t& t0) {
  const uint32_t qt = t % g.nqt, ct = t / g.nqt;
  q0 = (int64_t)qt * TQ;
  tq = (int)(g.ntubes - q0 < TQ ? g.ntubes - q0 : TQ);
  t0 = (int64_t)ct * g.CT;
}

// ------------------------------------------------------------- forward ----
// W levels after level l0 on `len` smooth values per tube held in src (pitch ps).
template <int TQ, int W>
__device__ __forceinline__ void fwd_stage(const double* src, int ps, double* dst, int pd, int l0,
                                          int len, const FGeom g, double* __restrict__ out,
                                          int64_t q0, int tq, int64_t t0) {
  // A thread lifts the same 2^W-band chunk of TWO adjacent tubes (r, r+1), so
  // every detail / smooth output is one 16-byte store (adjacent tubes are
  // adjacent in a packed slice row): half the store instructions, full sectors.
  constexpr int V = 1 << W;
  constexpr int HQ = TQ / 2;
  const int items = HQ * (len >> W);
  const bool last = (l0 + W == g.L);
  for (int e = threadIdx.x; e < items; e += kT) {
    const int r = 2 * (e & (HQ - 1)), c = e / HQ;
    if (r >= tq) continue;
    const bool two = r + 1 < tq;
    double v[2][V];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < V; i += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(src + (r + h) * ps + c * V + i);
        v[h][i] = t2.x;
        v[h][i + 1] = t2.y;
      }
    auto put = [&](int64_t s, double a, double b) {
      double* o = slice_row(g, out, s) + q0 + r;
      if (two && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
        *reinterpret_cast<double2*>(o) = make_double2(a, b);
      } else {
        o[0] = a;
        if (two) o[1] = b;
      }
    };
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int lev = l0 + w + 1;
      const int n = V >> (w + 1);
      const bool want = (g.mask >> lev) & 1;
      const int64_t s0 = doff(g.p, lev) + (t0 >> lev) + (int64_t)c * n;
#pragma unroll
      for (int i = 0; i < (V >> 1); ++i) {
        if (i < n) {
          double d[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            d[h] = __dsub_rn(v[h][2 * i], v[h][2 * i + 1]);
            v[h][i] = __dadd_rn(v[h][2 * i + 1], __dmul_rn(d[h], 0.5));
          }
          if (want) put(s0 + i, d[0], d[1]);
        }
      }
    }
    if (last) {
      if (g.mask & 1) put(soff(g.p, g.L) + (t0 >> g.L) + c, v[0][0], v[1][0]);
    } else {
      dst[r * pd + c] = v[0][0];
      if (two) dst[(r + 1) * pd + c] = v[1][0];
    }
  }
}

template <int TQ>
__global__ void __launch_bounds__(kT) fwd_persistent(const double* __restrict__ x,
                                                     double* __restrict__ out, FGeom g) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  // pointer arithmetic on `sm` (not arrays of pointers) keeps every access LDS/STS
  const int tile_sz = TQ * g.LDT;
  double* const aux0 = sm + 2 * tile_sz;
  double* const aux1 = aux0 + TQ * g.LDA0;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t t, int buf) {
    if (threadIdx.x < 32) {
      int64_t q0, t0;
      int tq;
      tile_at<TQ>(g, t, q0, tq, t0);
      if (threadIdx.x == 0) mbar_expect_tx(&bar[buf], (uint32_t)(tq * g.CT * 8));
      __syncwarp();
      for (int r = threadIdx.x; r < tq; r += 32)
        bulk_g2s(sm + buf * tile_sz + r * g.LDT, x + (q0 + r) * g.p + t0, (uint32_t)(g.CT * 8), &bar[buf]);
    }
  };
  uint32_t t = blockIdx.x;
  if (t < g.ntiles) issue(t, 0);
  for (int i = 0; t < g.ntiles; ++i, t += gridDim.x) {
    const int buf = i & 1;
    if (t + gridDim.x < g.ntiles) issue(t + gridDim.x, buf ^ 1);
    mbar_wait(&bar[buf], (i >> 1) & 1);
    int64_t q0, t0;
    int tq;
    tile_at<TQ>(g, t, q0, tq, t0);
    const double* src = sm + buf * tile_sz;
    int ps = g.LDT, len = g.CT, l0 = 0, stage = 0;
    while (l0 < g.L) {
      const int W = min(3, g.L - l0);
      double* dst = (stage & 1) ? aux1 : aux0;
      const int pd = (stage & 1) ? g.LDA1 : g.LDA0;
      if (W == 3) fwd_stage<TQ, 3>(src, ps, dst, pd, l0, len, g, out, q0, tq, t0);
      else if (W == 2) fwd_stage<TQ, 2>(src, ps, dst, pd, l0, len, g, out, q0, tq, t0);
      else fwd_stage<TQ, 1>(src, ps, dst, pd, l0, len, g, out, q0, tq, t0);
      l0 += W;
      len >>= W;
      if (l0 < g.L) {
        __syncthreads();
        src = dst;
        ps = pd;
        ++stage;
      }
    }
    fence_proxy_async_smem();  // generic reads of `buf` before its TMA refill
    __syncthreads();  // tile buffer `buf` is refilled by the next iteration's issue
  }
  if (g.tab) __threadfence_system();  // peer stores: system-scope release before the exchange barrier
}

// Deep-L variant (L > 3): ONE tile buffer of TQ = 32 tubes x CT bands.  Stage 0
// reads the whole input tile into registers, so the next tile's TMA load is
// issued right after stage 0's barrier and overlaps the later stages.
template <int TQ>
__global__ void __launch_bounds__(kT) fwd_persistent1(const double* __restrict__ x,
                                                      double* __restrict__ out, FGeom g) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  double* const aux0 = sm + TQ * g.LDT;
  double* const aux1 = aux0 + TQ * g.LDA0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t t) {
    if (threadIdx.x < 32) {
      int64_t q0, t0;
      int tq;
      tile_at<TQ>(g, t, q0, tq, t0);
      if (threadIdx.x == 0) mbar_expect_tx(&bar, (uint32_t)(tq * g.CT * 8));
      __syncwarp();
      for (int r = threadIdx.x; r < tq; r += 32)
        bulk_g2s(sm + r * g.LDT, x + (q0 + r) * g.p + t0, (uint32_t)(g.CT * 8), &bar);
    }
  };
  uint32_t t = blockIdx.x;
  if (t < g.ntiles) issue(t);
  for (int i = 0; t < g.ntiles; ++i, t += gridDim.x) {
    mbar_wait(&bar, i & 1);
    int64_t q0, t0;
    int tq;
    tile_at<TQ>(g, t, q0, tq, t0);
    const double* src = sm;
    int ps = g.LDT, len = g.CT, l0 = 0, stage = 0;
    while (l0 < g.L) {
      const int W = min(3, g.L - l0);
      double* dst = (stage & 1) ? aux1 : aux0;
      const int pd = (stage & 1) ? g.LDA1 : g.LDA0;
      if (W == 3) fwd_stage<TQ, 3>(src, ps, dst, pd, l0, len, g, out, q0, tq, t0);
      else if (W == 2) fwd_stage<TQ, 2>(src, ps, dst, pd, l0, len, g, out, q0, tq, t0);
      else fwd_stage<TQ, 1>(src, ps, dst, pd, l0, len, g, out, q0, tq, t0);
      l0 += W;
      len >>= W;
      if (l0 < g.L) {
        if (stage == 0) fence_proxy_async_smem();  // tile reads before the TMA refill
        __syncthreads();
        if (stage == 0 && t + gridDim.x < g.ntiles) issue(t + gridDim.x);  // tile buffer is free
        src = dst;
        ps = pd;
        ++stage;
      }
    }
    __syncthreads();
  }
  if (g.tab) __threadfence_system();  // peer stores: system-scope release before the exchange barrier
}

// Shallow variant (L = W <= 3, one stage): ONE 32 x 256 tile buffer; every
// thread first pulls its 2^W-band chunks of two tubes into registers, one CTA
// barrier frees the buffer, the next tile's TMA load is issued, and the lift +
// stores run while it is in flight.
template <int W>
__global__ void __launch_bounds__(kT) fwd_shallow(const double* __restrict__ x,
                                                  double* __restrict__ out, FGeom g) {
  constexpr int TQ = 32, CT = 256, V = 1 << W, HQ = TQ / 2;
  constexpr int ITEMS = HQ * (CT >> W), MAXI = ITEMS / kT;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int LDT = CT + 2;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t t) {
    if (threadIdx.x < 32) {
      int64_t q0, t0;
      int tq;
      tile_at<TQ>(g, t, q0, tq, t0);
      if (threadIdx.x == 0) mbar_expect_tx(&bar, (uint32_t)(tq * CT * 8));
      __syncwarp();
      for (int r = threadIdx.x; r < tq; r += 32)
        bulk_g2s(sm + r * LDT, x + (q0 + r) * g.p + t0, (uint32_t)(CT * 8), &bar);
    }
  };
  uint32_t t = blockIdx.x;
  if (t < g.ntiles) issue(t);
  for (int it = 0; t < g.ntiles; ++it, t += gridDim.x) {
    mbar_wait(&bar, it & 1);
    int64_t q0, t0;
    int tq;
    tile_at<TQ>(g, t, q0, tq, t0);
    double v[MAXI][2][V];
#pragma unroll
    for (int k = 0; k < MAXI; ++k) {
      const int e = threadIdx.x + k * kT;
      const int r = 2 * (e & (HQ - 1)), c = e / HQ;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < V; i += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(sm + (r + h) * LDT + c * V + i);
          v[k][h][i] = t2.x;
          v[k][h][i + 1] = t2.y;
        }
    }
    fence_proxy_async_smem();                          // reads before the TMA refill
    __syncthreads();                                   // the tile buffer is free
    if (t + gridDim.x < g.ntiles) issue(t + gridDim.x);
#pragma unroll
    for (int k = 0; k < MAXI; ++k) {
      const int e = threadIdx.x + k * kT;
      const int r = 2 * (e & (HQ - 1)), c = e / HQ;
      if (r >= tq) continue;
      const bool two = r + 1 < tq;
      auto put = [&](int64_t s, double a, double b) {
        double* o = slice_row(g, out, s) + q0 + r;
        if (two && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
          *reinterpret_cast<double2*>(o) = make_double2(a, b);
        } else {
          o[0] = a;
          if (two) o[1] = b;
        }
      };
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int lev = w + 1;
        const int n = V >> (w + 1);
        const bool want = (g.mask >> lev) & 1;
        const int64_t s0 = doff(g.p, lev) + (t0 >> lev) + (int64_t)c * n;
#pragma unroll
        for (int i = 0; i < (V >> 1); ++i) {
          if (i < n) {
            double d[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              d[h] = __dsub_rn(v[k][h][2 * i], v[k][h][2 * i + 1]);
              v[k][h][i] = __dadd_rn(v[k][h][2 * i + 1], __dmul_rn(d[h], 0.5));
            }
            if (want) put(s0 + i, d[0], d[1]);
          }
        }
      }
      if (g.mask & 1) put(soff(g.p, W) + (t0 >> W) + c, v[k][0][0], v[k][1][0]);
    }
  }
  if (g.tab) __threadfence_system();  // peer stores: system-scope release before the exchange barrier
}

// ------------------------------------------------------------- inverse ----
// Tile-local rows of the prefetched slice-major input follow the packed order
// [d1 | ... | dL | sL] with the tile's CT bands in place of p.
__device__ __forceinline__ int drow(int CT, int j) { return CT - (CT >> (j - 1)); }

// s_hi[c] of tube r from s_L and the D = L - hi details on c's ancestor chain
// (loads first, then the dependent unlift chain; same roundings as level by level).
template <int TQ, int D>
__device__ __forceinline__ double path_chain(const double* __restrict__ I, int CT, int L, int hi,
                                             int c, int r, uint64_t mask, bool have_s, int srow) {
  double d[D];
#pragma unroll
  for (int u = 0; u < D; ++u) {
    const int j = L - u;
    d[u] = ((mask >> j) & 1) ? I[(drow(CT, j) + (c >> (j - hi))) * TQ + r] : 0.0;
  }
  double sv = have_s ? I[(srow + (c >> (L - hi))) * TQ + r] : 0.0;
#pragma unroll
  for (int u = 0; u < D; ++u) {
    const int j = L - u;
    const double x1 = __dsub_rn(sv, __dmul_rn(d[u], 0.5));
    sv = ((c >> (j - hi - 1)) & 1) ? x1 : __dadd_rn(d[u], x1);
  }
  return sv;
}

// Levels hi .. hi-W+1: each thread expands one s_hi value into 2^W values of
// s_{hi-W} using the prefetched details; the final stage (down to level 1)
// stores the 2^W consecutive bands straight to y.
template <int TQ, int W>
__device__ __forceinline__ void inv_stage(const double* __restrict__ I,
                                          const double* __restrict__ ssrc, int pss, bool s_in,
                                          double* __restrict__ dst, int pd, int hi, const FGeom g,
                                          double* __restrict__ y, int64_t q0, int tq, int64_t t0,
                                          bool path = false) {
  constexpr int V = 1 << W;
  const int CT = g.CT;
  const int nval = CT >> hi;
  const int items = TQ * nval;
  const bool final_stage = (hi - W == 0);
  const bool have_s = g.mask & 1;
  const int srow = CT - (CT >> g.L);
  for (int e = threadIdx.x; e < items; e += kT) {
    const int r = e & (TQ - 1), c = e / TQ;
    if (r >= tq) continue;
    double v[V];
    if (path) {
      // s_hi[c] straight from s_L along c's ancestor chain (levels L .. hi+1):
      // the same two roundings per level as the level-by-level inverse, no
      // stage barriers (lifting.py:69-74).  Depths are compile-time so every
      // detail load of the chain is issued before the dependent arithmetic
      // (ncu: the rolled loop waited on each shared load in turn).
      switch (g.L - hi) {
        case 4: v[0] = path_chain<TQ, 4>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        case 5: v[0] = path_chain<TQ, 5>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        case 6: v[0] = path_chain<TQ, 6>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        case 7: v[0] = path_chain<TQ, 7>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        case 8: v[0] = path_chain<TQ, 8>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        case 9: v[0] = path_chain<TQ, 9>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        case 10: v[0] = path_chain<TQ, 10>(I, CT, g.L, hi, c, r, g.mask, have_s, srow); break;
        default: {
          double sv = have_s ? I[(srow + (c >> (g.L - hi))) * TQ + r] : 0.0;
          for (int j = g.L; j > hi; --j) {
            const int k = c >> (j - hi);
            const double d = ((g.mask >> j) & 1) ? I[(drow(CT, j) + k) * TQ + r] : 0.0;
            const double x1 = __dsub_rn(sv, __dmul_rn(d, 0.5));
            sv = ((c >> (j - hi - 1)) & 1) ? x1 : __dadd_rn(d, x1);
          }
          v[0] = sv;
        }
      }
    } else {
      v[0] = s_in ? (have_s ? I[(srow + c) * TQ + r] : 0.0) : ssrc[r * pss + c];
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int lev = hi - w;
      const int n = 1 << w;
      const bool have_d = (g.mask >> lev) & 1;
      const double* dr = I + (drow(CT, lev) + c * n) * TQ + r;
#pragma unroll
      for (int i = (V >> 1) - 1; i >= 0; --i) {
        if (i < n) {
          const double d = have_d ? dr[i * TQ] : 0.0;
          const double x1 = __dsub_rn(v[i], __dmul_rn(d, 0.5));
          v[2 * i] = __dadd_rn(d, x1);
          v[2 * i + 1] = x1;
        }
      }
    }
    if (final_stage) {
      double* o = y + (q0 + r) * g.p + t0 + (int64_t)c * V;
#pragma unroll
      for (int i = 0; i < V; i += 2) *reinterpret_cast<double2*>(o + i) = make_double2(v[i], v[i + 1]);
    } else {
      double* o = dst + r * pd + c * V;
#pragma unroll
      for (int i = 0; i < V; i += 2) *reinterpret_cast<double2*>(o + i) = make_double2(v[i], v[i + 1]);
    }
  }
}

// One 2-D TMA descriptor per detail level j (box: TQ tubes x CT>>j slices of the
// packed buffer viewed as [slices][tubes]); the smooth block reuses level L's.
struct TmaMaps {
  CUtensorMap m[kMaxTmaLevels + 1];
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

template <int TQ, bool TMA>
__global__ void __launch_bounds__(kT) inv_persistent(const double* __restrict__ pyr,
                                                     double* __restrict__ y, FGeom g,
                                                     const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int CT = g.CT;
  // pointer arithmetic on `sm` (not arrays of pointers) keeps every access LDS/STS
  double* const aux0 = sm + 2 * CT * TQ;
  double* const aux1 = aux0 + TQ * g.LDA0;
  constexpr int CPR = TQ / 2;  // 16-byte chunks per row
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  auto issue = [&](uint32_t t, int buf) {
    int64_t q0, t0;
    int tq;
    tile_at<TQ>(g, t, q0, tq, t0);
    double* dstb = sm + buf * (CT * TQ);
    if (TMA) {
      // thread 0 issues one 2-D TMA box per level block (SASS UTMALDG);
      // out-of-range tubes of the last tile arrive zero-filled
      if (threadIdx.x == 0) {
        uint32_t bytes = 0;
        for (int j = 1; j <= g.L + 1; ++j)
          if ((g.mask >> (j > g.L ? 0 : j)) & 1) bytes += (CT >> min(j, g.L)) * TQ * 8;
        mbar_expect_tx(&bar[buf], bytes);
        for (int j = 1; j <= g.L + 1; ++j) {
          const bool smooth = j > g.L;
          if (!((g.mask >> (smooth ? 0 : j)) & 1)) continue;
          const int row0 = smooth ? CT - (CT >> g.L) : drow(CT, j);
          const int64_t s0 = smooth ? soff(g.p, g.L) + (t0 >> g.L) : doff(g.p, j) + (t0 >> j);
          tma_load_2d(dstb + row0 * TQ, &maps.m[smooth ? g.L : j], (int)q0,
                      (int)(s0 - g.slice_base), &bar[buf]);
        }
      }
      return;
    }
    for (int j = 1; j <= g.L + 1; ++j) {
      const bool smooth = j > g.L;
      if (!((g.mask >> (smooth ? 0 : j)) & 1)) continue;
      const int rows = smooth ? (CT >> g.L) : (CT >> j);
      const int row0 = smooth ? CT - (CT >> g.L) : drow(CT, j);
      const int64_t s0 = smooth ? soff(g.p, g.L) + (t0 >> g.L) : doff(g.p, j) + (t0 >> j);
      for (int e = threadIdx.x; e < rows * CPR; e += kT) {
        const int rr = e / CPR, v = (e % CPR) * 2;
        const bool ok = v < tq;
        const double* src = slice_row(g, const_cast<double*>(pyr), s0 + rr) + q0 + (ok ? v : 0);
        cp_async_zfill<16>(dstb + (row0 + rr) * TQ + v, src, ok);
      }
    }
    cp_async_commit();
  };
  uint32_t t = blockIdx.x;
  if (t < g.ntiles) issue(t, 0);
  else if (!TMA) cp_async_commit();
  for (int i = 0; t < g.ntiles; ++i, t += gridDim.x) {
    const int buf = i & 1;
    if (t + gridDim.x < g.ntiles) issue(t + gridDim.x, buf ^ 1);
    else if (!TMA) cp_async_commit();
    if (TMA) {
      mbar_wait(&bar[buf], (i >> 1) & 1);
    } else {
      cp_async_wait<1>();
      __syncthreads();
    }
    int64_t q0, t0;
    int tq;
    tile_at<TQ>(g, t, q0, tq, t0);
    const double* I = sm + buf * (CT * TQ);
    int hi = g.L, stage = 0;
    const double* ssrc = nullptr;
    int pss = 0;
    if (g.inv_path && g.L >= g.inv_path) {  // one barrier-free pass: levels L..4 by ancestor chains
      inv_stage<TQ, 3>(I, ssrc, pss, false, aux0, g.LDA0, 3, g, y, q0, tq, t0, true);
      hi = 0;
    }
    while (hi > 0) {
      const int W = (hi - 1) % 3 + 1;  // top stage absorbs the remainder: final stage is 3 wide
      double* dst = (stage & 1) ? aux1 : aux0;
      const int pd = g.LDA0;
      const bool s_in = (hi == g.L);
      if (W == 3) inv_stage<TQ, 3>(I, ssrc, pss, s_in, dst, pd, hi, g, y, q0, tq, t0);
      else if (W == 2) inv_stage<TQ, 2>(I, ssrc, pss, s_in, dst, pd, hi, g, y, q0, tq, t0);
      else inv_stage<TQ, 1>(I, ssrc, pss, s_in, dst, pd, hi, g, y, q0, tq, t0);
      hi -= W;
      if (hi > 0) {
        __syncthreads();
        ssrc = dst;
        pss = pd;
        ++stage;
      }
    }
    // No proxy fence before the TMA refill of this buffer (issued right after
    // the barrier): every shared-memory load of the tile has been consumed by
    // the lift and the global stores before the thread reaches the barrier, so
    // no read is still in flight.  (A fence here costs 4%.  The single-buffered
    // kernels that hold raw tile values across the barrier do fence: without
    // it inv_shallow read refilled data.)
    __syncthreads();  // input buffer / stage buffers are reused by later tiles
  }
  if (!TMA) cp_async_wait<0>();
}

// Tile height cap.  Forward: taller tiles write longer runs per packed slice
// row (TQ * 8 bytes); measured at config 2 (tools/lift_tq_probe.py, round 1,
// GB/s): L=1-3 best at 32 (+2%), L=4-6 at 64 (+7..14%), L=7 at 32 (+14%), L=8
// needs CT = 256 so stays at 16 (L >= 6 take fwd_persistent1).  Inverse: 16 (taller tiles cost 30%: the
// tube-major final stores scatter over more tubes per warp).
int tq_max(bool fwd, int L) {
  if (!fwd) return 16;
  return (L >= 4 && L <= 6) ? 64 : 32;
}

bool plan(FGeom& g, int& TQ, bool fwd) {
  const int64_t unit = (int64_t)1 << g.L;
  const int64_t munits = g.p / unit;
  for (int tq = tq_max(fwd, g.L); tq >= 2; tq >>= 1) {
    const int64_t cap = kMaxElems / tq;
    if (unit > cap) continue;
    int64_t best = 0;
    for (int64_t d = 1; d <= munits && unit * d <= cap; ++d)
      if (munits % d == 0) best = d;
    TQ = tq;
    g.CT = (int)(unit * best);
    g.LDT = g.CT + 2;
    g.LDA0 = std::max(2, g.CT / 8) + 2;
    g.LDA1 = std::max(2, g.CT / 64) + 2;
    const int64_t nqt = (g.ntubes + tq - 1) / tq;
    const int64_t ntiles = nqt * (g.p / g.CT);
    if (ntiles >= (1LL << 31)) return false;
    g.nqt = (uint32_t)nqt;
    g.ntiles = (uint32_t)ntiles;
    return true;
  }
  return false;
}

template <typename K, typename... Extra>
int launch(K kern, size_t smem, uint32_t ntiles, cudaStream_t st, const double* a, double* b,
           const FGeom& g, const char* what, const Extra&... extra) {
  if (int e = ensure_smem(kern, smem)) return e;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)num_sms() * per_sm);
  kern<<<grid, kT, smem, st>>>(a, b, g, extra...);
  return check_launch(what);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // function-local static: initialised once, thread-safe (concurrent first calls)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// Descriptors for the packed buffer [nslices][ntubes] with boxes TQ x (CT >> j).
bool make_maps(TmaMaps& M, const double* pyr, const FGeom& g, int TQ) {
  auto enc = encode_fn();
  if (!enc || g.L > kMaxTmaLevels) return false;
  const int64_t nslices = g.p - g.slice_base;
  const cuuint64_t dims[2] = {(cuuint64_t)g.ntubes, (cuuint64_t)nslices};
  const cuuint64_t strides[1] = {(cuuint64_t)g.ntubes * sizeof(double)};
  const cuuint32_t estr[2] = {1, 1};
  for (int j = 1; j <= g.L; ++j) {
    const cuuint32_t box[2] = {(cuuint32_t)TQ, (cuuint32_t)(g.CT >> j)};
    if (enc(&M.m[j], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(pyr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

}  // namespace fast

// Returns WT_ERR_UNSUPPORTED when the fast path does not apply (caller falls back).
int lift_fwd_fast(const double* x, int64_t ntubes, int64_t p, int L, double* out,
                  int64_t slice_base, uint64_t mask, cudaStream_t st,
                  const unsigned long long* tab) {
  using namespace fast;
  if (L < 1 || p % 2 || (uintptr_t)x % 16) return WT_ERR_UNSUPPORTED;
  FGeom g{ntubes, p, L, 0, 0, 0, 0, slice_base, mask, 0, 0, tab};
  int TQ = 0;
  if (!plan(g, TQ, true)) return WT_ERR_UNSUPPORTED;
  const size_t smem = ((size_t)2 * TQ * g.LDT + (size_t)TQ * (g.LDA0 + g.LDA1)) * sizeof(double);
  // L = 6..8: single-buffered 32-tube tiles of 256 bands (fwd_persistent1);
  // measured at config 2 (tools/lift_tq_probe.py, TB/s): L=6 5.58 -> 5.96,
  // L=7 5.83 -> 5.89, L=8 5.09 -> 5.89; L=4, 5 tie with the TQ=64 tiles.
  const int64_t unit = (int64_t)1 << g.L;
  if (g.L <= 3 && g.p % 256 == 0) {
    FGeom g1 = g;
    g1.CT = 256;
    g1.LDT = 258;
    g1.nqt = (uint32_t)((g.ntubes + 31) / 32);
    g1.ntiles = (uint32_t)(g1.nqt * (g.p / 256));
    const size_t smem1 = (size_t)32 * 258 * sizeof(double);
    if (g.L == 1) return launch(fwd_shallow<1>, smem1, g1.ntiles, st, x, out, g1, "wt_lift_fwd_f64");
    if (g.L == 2) return launch(fwd_shallow<2>, smem1, g1.ntiles, st, x, out, g1, "wt_lift_fwd_f64");
    return launch(fwd_shallow<3>, smem1, g1.ntiles, st, x, out, g1, "wt_lift_fwd_f64");
  }
  if (unit >= 64 && unit <= 256 && g.p % 256 == 0) {
    FGeom g1 = g;
    constexpr int TQ1 = 32;
    {
      g1.CT = 256;
      g1.LDT = g1.CT + 2;
      g1.LDA0 = std::max(2, g1.CT / 8) + 2;
      g1.LDA1 = std::max(2, g1.CT / 64) + 2;
      g1.nqt = (uint32_t)((g.ntubes + TQ1 - 1) / TQ1);
      g1.ntiles = (uint32_t)(g1.nqt * (g.p / g1.CT));
      const size_t smem1 = ((size_t)TQ1 * g1.LDT + (size_t)TQ1 * (g1.LDA0 + g1.LDA1)) * sizeof(double);
      return launch(fwd_persistent1<32>, smem1, g1.ntiles, st, x, out, g1, "wt_lift_fwd_f64");
    }
  }
  switch (TQ) {
    case 64: return launch(fwd_persistent<64>, smem, g.ntiles, st, x, out, g, "wt_lift_fwd_f64");
    case 32: return launch(fwd_persistent<32>, smem, g.ntiles, st, x, out, g, "wt_lift_fwd_f64");
    case 16: return launch(fwd_persistent<16>, smem, g.ntiles, st, x, out, g, "wt_lift_fwd_f64");
    case 8: return launch(fwd_persistent<8>, smem, g.ntiles, st, x, out, g, "wt_lift_fwd_f64");
    case 4: return launch(fwd_persistent<4>, smem, g.ntiles, st, x, out, g, "wt_lift_fwd_f64");
    default: return launch(fwd_persistent<2>, smem, g.ntiles, st, x, out, g, "wt_lift_fwd_f64");
  }
}

int lift_inv_fast(const double* pyr, int64_t ntubes, int64_t p, int L, double* y,
                  int64_t slice_base, uint64_t mask, cudaStream_t st,
                  const unsigned long long* tab) {
  using namespace fast;
  if (L < 1 || p % 2 || ntubes % 2 || (uintptr_t)y % 16 || (uintptr_t)pyr % 16)
    return WT_ERR_UNSUPPORTED;
  FGeom g{ntubes, p, L, 0, 0, 0, 0, slice_base, mask, 0, 0, tab};
  // measured at config 2 (tools/lift_tq_probe.py, 3 alternating runs): L = 7
  // +2% over the staged inverse, L = 8 even, L = 4..6 -2..7% (the chains'
  // redundant loads outweigh the saved barriers while the top levels are short)
  g.inv_path = 7;
  int TQ = 0;
  if (!plan(g, TQ, false)) return WT_ERR_UNSUPPORTED;
  const size_t smem = ((size_t)2 * g.CT * TQ + (size_t)2 * TQ * g.LDA0) * sizeof(double);
  if (smem > 200 * 1024) return WT_ERR_UNSUPPORTED;
  TmaMaps maps{};  // host copy, passed by value as a __grid_constant__ parameter
  // TMA boxes: 16 tubes (128-byte rows) x <= 256 slices, 16-byte-multiple stride
  if (!tab && TQ >= 16 && (g.CT >> 1) <= 256 &&
      make_maps(maps, pyr, g, TQ)) {
    if (TQ == 64)
      return launch(inv_persistent<64, true>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
    if (TQ == 32)
      return launch(inv_persistent<32, true>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
    return launch(inv_persistent<16, true>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
  }
  switch (TQ) {
    case 16: return launch(inv_persistent<16, false>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
    case 8: return launch(inv_persistent<8, false>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
    case 4: return launch(inv_persistent<4, false>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
    default: return launch(inv_persistent<2, false>, smem, g.ntiles, st, pyr, y, g, "wt_lift_inv_f64", maps);
  }
}

}  // namespace wt
