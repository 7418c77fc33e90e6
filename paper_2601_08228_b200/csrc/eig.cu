// K4 preconditioner: the eigenbasis V0 of the Gram X^T X of every slice, so
// that the one-sided Jacobi sweeps start from X V0 (nearly orthogonal columns,
// quadratic convergence from the first sweep) instead of from X.
//
// Why: plain cyclic one-sided Jacobi spends 9-15 of its 12-17 sweeps on the
// wavelet slices of configs 3-5 with pair cosines still at 0.3-0.9
// (profiles/r01_summary.md, convergence traces); started from X V0 it needs 3
// (tools/jacobi_precond_probe.py).  The Gram squares the
// condition number, so V0 is only a preconditioner: the FP64 Jacobi on X V0
// keeps its own convergence test and delivers the singular values, so the
// accuracy is that of the Jacobi method (replacing _stack_svd,
// decomposition.py:64-67, as before).
//
// Pipeline (all batched over the slices, stream-ordered, FP64):
//   1. G = X^T X                                   K3 GEMM
//   2. G = Q T Q^T, T tridiagonal                  panels of NB columns:
//        tridiag_panel<C> (lazy latrd-style column updates, lower-triangle
//        symv, one CTA or a C-CTA cluster per matrix; rows of the trailing
//        block dealt cyclically over the cluster, partial sums exchanged in
//        distributed shared memory) + the symmetric rank-2NB trailing update
//        on K3 (lower tiles only).  The panel's Householder vectors overwrite
//        its (dead) columns of G.
//   3. eigenvalues of T: bisection, one thread per eigenvalue (Sturm counts
//      by the scaled determinant recurrence: one FMA per step on the chain)
//   4. eigenvectors of T: inverse iteration (2 solves with the LDL^T factors of
//      T - lambda I), one thread per eigenvalue              -> Z
//   5. Newton-Schulz Z <- Z (3 I - Z^T Z) / 2 until orthogonal to rounding
//      (K3; matrices where it cannot converge fall back to V0 = I)
//   6. V0 = Q Z: compact-WY blocks of 64 / 128 reflectors (larft + 3 K3 GEMMs each)
//   7. Y = X V0                                      K3 GEMM
// Deterministic: fixed thread -> data maps and reduction orders.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "wt_common.cuh"

namespace wt {
namespace eig {

constexpr int NB_MAX = 32;  // tridiagonalization panel width: 16 or 32 (panel_shape)
constexpr int NBT = 128;   // back-transformation block (reflectors per compact-WY block)
constexpr int PT = 256;    // panel kernel threads
constexpr int NW = PT / 32;
#ifndef WT_EIG_CH
#define WT_EIG_CH 256
#endif
#ifndef WT_EIG_RB
#define WT_EIG_RB 4
#endif
constexpr int CH = WT_EIG_CH;  // symv column chunk (CH / 64 double2 register accumulators per lane)
constexpr int NCH2 = CH / 64;
constexpr int RB = WT_EIG_RB;  // rows per warp in flight in the symv
static_assert(RB == 4, "the symv's row-sum reduction handles exactly 4 rows per warp");
static_assert(CH >= 2 * NB_MAX + 1, "the y partials alias the symv's per-warp accumulators");
constexpr int MAXR = 256;  // own rows per CTA (the panel's V, W rows of a CTA live in shared memory)
constexpr int PREF_R = 128;  // preferred own rows per CTA (two CTAs per SM)

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return (int)r;
}
template <typename T>
__device__ __forceinline__ T* cl_map(T* p, int rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<T*>(out);
}
template <int C>
__device__ __forceinline__ void csync() {
  if constexpr (C > 1) cl_sync(); else __syncthreads();
}
template <int C, typename T>
__device__ __forceinline__ const T* remote(const T* p, int rank) {
  if constexpr (C > 1) return cl_map(const_cast<T*>(p), rank);
  else return p;
}

// deterministic CTA sum (warp shuffles, then warps in order); result valid in every thread
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) s += red[w];
  return s;
}

struct PanelSmem {
  static size_t bytes(int n, int C, int NB) {
    const int R = (n + C - 1) / C;
    const int VP = 2 * NB + 2;
    return sizeof(double) * ((size_t)R * VP + 10 + 3 * (size_t)n + 2 + 2 * (size_t)R + (size_t)NW * CH + 4 + 2 +
                             2 * NB + 2 * NW + 7 * NB);
  }
};

// One panel (columns k0 .. k0+jb-1) of the lower Householder tridiagonalization
// (LAPACK dsytrd / dlatrd semantics, lower storage).  Per column k:
//   a   = A[k:, k] - V W[k, :]^T - W V[k, :]^T          (lazy panel updates)
//   v   = Householder vector of a[k+1:], tau, e[k] = beta, d[k] = a[k]
//   p   = A22 v - V (W^T v) - W (V^T v)                 (A22 = A[k+1:, k+1:], pre-panel)
//   w   = tau p - (tau^2 / 2)(p^T v - 2 (W^T v).(V^T v)) v
// Rows are dealt cyclically over the C CTAs of a cluster (row i -> CTA i % C,
// local row i / C); a CTA keeps its rows of the panel's V and W in shared
// memory, so the lazy updates never wait on global memory.  VW = [V | W] and
// WV = [W | V] (n x 2NB, row-major, global) feed the trailing update A22 -=
// VW WV^T on K3; the panel's V block overwrites its dead columns of A.
// Two cluster barriers per column: S1 (my rows' updated column entries and
// norm partials; every CTA then forms the whole v from the owners' entries)
// and S3 (symv partials); w of row k+1, needed by every CTA's next lazy
// update, is evaluated redundantly by every CTA with its owner's expression.
template <int C, int NB>
__global__ void __launch_bounds__(PT, 2) tridiag_panel(double* __restrict__ Gall, double* __restrict__ VWall,
                                                    double* __restrict__ WVall, double* __restrict__ dall,
                                                    double* __restrict__ eall, double* __restrict__ tauall,
                                                    const int* __restrict__ flag, int n, int k0, float l2keep) {
  static_assert(NB == 16 || NB == 32, "panel width");
  constexpr int VP = 2 * NB + 2;  // shared pitch of a [V | W] row (even: 16-byte aligned rows)
  extern __shared__ __align__(16) double sm[];
  const int R = (n + C - 1) / C;  // local rows (upper bound)
  double* vws = sm;                    // [R][VP]  my rows of [V | W]
  double* vsm = vws + ((R * VP + 1) & ~1);  // [n + 2]  v (full; 16-byte aligned, zero beyond n)
  // (every array starts 16-byte aligned: double2 accesses)
  double* aw = vsm + ((n + 3) & ~1);   // [n]  my rows' updated column entries a_i (DSMEM-visible)
  double* csum = aw + ((n + 1) & ~1);  // [n]  CTA partial column part of A22 v (DSMEM-visible)
  double* prow = csum + ((n + 1) & ~1);  // [R]  my rows: row part of A22 v
  double* diag = prow + ((R + 1) & ~1);  // [R]  my rows: A[i][i] (pre-panel)
  double* wacc = diag + ((R + 1) & ~1);  // [NW][CH] per-warp column accumulators
  double* part1 = wacc + NW * CH;      // [4]  ss, alpha (S1)
  double* part3 = part1 + 4;           // [2 + 2NB] pv, -, yW[NB], yV[NB] (S3)
  double* red = part3 + 2 + 2 * NB;    // [2NW]
  double* ys = red + 2 * NW;           // [2NB] cluster sums of yW, yV
  double* rk = ys + 2 * NB;            // [2NB] row k of [V | W]
  double* dpan = rk + 2 * NB;          // [3NB] d, e, tau of the panel's columns (written at the end)
  double* ywacc = wacc;                // [NW][2NB + 1] per-warp partials of yW, yV, v^T A22 v (aliases
                                       // wacc: written after the symv's last flush has been consumed)
  const int rank = C == 1 ? 0 : cl_rank();
  const int b = blockIdx.x / C;
  if (!flag[b]) return;  // cluster-uniform
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = Gall + (int64_t)b * n * n;
  // L2 policy of the symv loads: the fraction l2keep of the trailing blocks' lines
  // (by address hash) is kept (evict_last), the rest streams (evict_first), so a
  // batch whose trailing blocks exceed L2 keeps most of them resident across the
  // panel's columns instead of thrashing all of them
  uint64_t l2pol = 0;
  if constexpr (C > 1)
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(l2pol) : "f"(l2keep));
  double* VW = VWall + (int64_t)b * n * 2 * NB;
  double* WV = WVall + (int64_t)b * n * 2 * NB;
  double* d = dall + (int64_t)b * n;
  double* e = eall + (int64_t)b * n;
  double* tau = tauall + (int64_t)b * n;
  const int jb = min(NB, n - k0);
  const int nloc = (n - rank + C - 1) / C;  // my rows: i = rank + C q, q < nloc
  auto row_of = [&](int q) { return rank + C * q; };
  auto q_first = [&](int lo) { return lo <= rank ? 0 : (lo - rank + C - 1) / C; };  // first q with row >= lo

  for (int q = tid; q < nloc; q += PT) {
    diag[q] = A[(int64_t)row_of(q) * n + row_of(q)];
    for (int t = 0; t < 2 * NB; ++t) vws[q * VP + t] = 0.0;
  }
  for (int i = tid; i < n + 2; i += PT) vsm[i] = 0.0;
  // prefetch of my rows' entries of column k (pre-panel values)
  double anext[(MAXR + PT - 1) / PT];
#pragma unroll
  for (int u = 0; u < (MAXR + PT - 1) / PT; ++u) {
    const int q = tid + u * PT;
    anext[u] = (q < nloc && row_of(q) >= k0) ? A[(int64_t)row_of(q) * n + k0] : 0.0;
  }
  __syncthreads();

  for (int j = 0; j < jb; ++j) {
    const int k = k0 + j;
    // ---------------- A: column update of my rows i >= k -------------------
    double ss = 0.0, alpha_own = 0.0;
#pragma unroll
    for (int u = 0; u < (MAXR + PT - 1) / PT; ++u) {
      const int q = tid + u * PT;
      const int i = row_of(q);
      if (q < nloc && i >= k) {
        // a = A[i][k] - V[i, :j] W[k, :j]^T - W[i, :j] V[k, :j]^T in four independent chains
        const double* ri = vws + q * VP;
        double a0 = anext[u], a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int t = 0;
        for (; t + 2 <= j; t += 2) {
          const double2 v2 = *reinterpret_cast<const double2*>(ri + t);
          const double2 w2 = *reinterpret_cast<const double2*>(ri + NB + t);
          const double2 kv = *reinterpret_cast<const double2*>(rk + t);
          const double2 kw = *reinterpret_cast<const double2*>(rk + NB + t);
          a0 = fma(-v2.x, kw.x, a0);
          a1 = fma(-w2.x, kv.x, a1);
          a2 = fma(-v2.y, kw.y, a2);
          a3 = fma(-w2.y, kv.y, a3);
        }
        if (t < j) {
          a0 = fma(-ri[t], rk[NB + t], a0);
          a1 = fma(-ri[NB + t], rk[t], a1);
        }
        const double a = (a0 + a1) + (a2 + a3);
        aw[i] = a;
        if (i >= k + 2) ss = fma(a, a, ss);
        if (i == k) dpan[j] = a;
        if (i == k + 1) alpha_own = a;
      }
    }
    // (only the owner of row k+1 contributes alpha)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
      alpha_own += __shfl_xor_sync(0xffffffffu, alpha_own, o);
    }
    if (lane == 0) {
      red[warp] = ss;
      red[NW + warp] = alpha_own;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        s0 += red[w];
        s1 += red[NW + w];
      }
      part1[0] = s0;
      part1[1] = s1;
    }
    csync<C>();  // S1
    // ---------------- B: Householder vector ---------------------------------
    double sst = 0.0;
#pragma unroll
    for (int r = 0; r < C; ++r) sst += remote<C>(part1, r)[0];
    const double alpha = remote<C>(part1, (k + 1) % C)[1];
    double tk = 0.0, scale = 0.0, beta = alpha;
    const bool last = k >= n - 2;
    if (!last && sst > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, sst)), alpha);
      tk = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (tid == 0) {
      dpan[NB + j] = beta;  // e[k] (k < n - 1)
      dpan[2 * NB + j] = k < n - 1 ? tk : 0.0;
    }
    if (k == n - 1) break;  // the last column only has its diagonal
    // v for every row of the trailing block, from the owners' a values (no
    // barrier between: the a values stay untouched until after the next S3)
    {
      // (all remote loads first, then the stores: the DSMEM latencies overlap)
      constexpr int VI = (C * MAXR + PT - 1) / PT;  // n <= C MAXR
      double av_r[VI];
#pragma unroll
      for (int u = 0; u < VI; ++u) {
        const int i = tid + u * PT;
        av_r[u] = (i < n && i >= k + 2) ? remote<C>(aw, i % C)[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < VI; ++u) {
        const int i = tid + u * PT;
        if (i < n) vsm[i] = i >= k + 2 ? av_r[u] * scale : (i == k + 1 && tk != 0.0 ? 1.0 : 0.0);
      }
    }
    __syncthreads();
    for (int q = tid; q < nloc; q += PT) vws[q * VP + j] = vsm[row_of(q)];
    // L2 prefetch of my rows' part of the next column's symv (A22 is constant
    // within the panel): one bulk prefetch per row, issued a column ahead
    if (C > 1 && j + 1 < jb) {  // (single-CTA shapes: batches that fit L2, measured faster without)
      const int c0 = (k + 2) & ~1;
      for (int q = q_first(k + 2) + tid; q < nloc; q += PT) {
        const int i = row_of(q);
        const int len = ((i + 1 - c0) * 8 + 15) & ~15;
        if (len > 0 && (n & 1) == 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A + (int64_t)i * n + c0), "r"(len)
                       : "memory");
      }
    }
    // prefetch of my rows' entries of the next column (not changed by this panel);
    // issued here so that no load is outstanding at the cluster barrier S1
    // (their release semantics wait for it), consumed by the next column's step A
#pragma unroll
    for (int u = 0; u < (MAXR + PT - 1) / PT; ++u) {
      const int q = tid + u * PT;
      const int i = row_of(q);
      anext[u] = (q < nloc && k + 1 < n && i >= k + 1) ? A[(int64_t)i * n + k + 1] : 0.0;
    }
    // ---------------- C: p = A22 v (lower triangle, my rows) ----------------
    // row part  prow[q] = sum_{c = k+1}^{i} A[i][c] v[c]
    // col part  csum[c] = sum_{my rows i > c} A[i][c] v[i]
    const int cstart = (k + 1) & ~1;  // 16-byte aligned double2 loads (n even)
    const int qk = q_first(k + 1);
    for (int q = qk + tid; q < nloc; q += PT) prow[q] = 0.0;
    __syncthreads();
    double yv_l = 0.0, yw_l = 0.0;  // lane t: sum over my rows of V[i][t] v_i, W[i][t] v_i
    for (int cb = cstart; cb < n; cb += CH) {
      double acc[NCH2][2];
#pragma unroll
      for (int t = 0; t < NCH2; ++t) acc[t][0] = acc[t][1] = 0.0;
      // my rows with entries in this chunk: i >= max(k+1, cb); RB rows per warp at a time
      const int q0 = q_first(max(k + 1, cb));
      for (int qb = q0 + warp * RB; qb < nloc; qb += NW * RB) {
        double av[RB][NCH2][2];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int q = qb + r;
          const int i = row_of(q);
          const double* Ar = A + (int64_t)i * n;
          const int cend = min(i, cb + CH - 1);  // inclusive (diagonal)
#pragma unroll
          for (int t = 0; t < NCH2; ++t) {
            const int c = cb + 64 * t + 2 * lane;
            av[r][t][0] = av[r][t][1] = 0.0;
            if (q < nloc && c <= cend) {
              if ((n & 1) == 0) {
                double x0, x1;
                if constexpr (C > 1) {  // (the single-CTA shapes serve batches that fit L2)
                  asm("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                      : "=d"(x0), "=d"(x1) : "l"(Ar + c), "l"(l2pol));
                } else {
                  const double2 x = *reinterpret_cast<const double2*>(Ar + c);
                  x0 = x.x;
                  x1 = x.y;
                }
                av[r][t][0] = x0;
                av[r][t][1] = c + 1 <= cend ? x1 : 0.0;  // (upper triangle beyond the diagonal)
              } else {
                av[r][t][0] = Ar[c];
                if (c + 1 <= cend) av[r][t][1] = Ar[c + 1];
              }
            }
          }
        }
        // row parts: v[c] = 0 for c <= k, so columns left of the block need no mask;
        // column parts include the diagonal (subtracted again in step D)
        double rp[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int i = row_of(qb + r);
          const double vi = qb + r < nloc ? vsm[i] : 0.0;
          if (cb == cstart && qb + r < nloc) {  // every row >= k+1 is visited in the first chunk
            // NB = 32: lane t sums V[i][t] v_i and W[i][t] v_i; NB = 16: lane t < 32
            // sums column t of the contiguous [V | W] row
            yv_l = fma(vws[(qb + r) * VP + lane], vi, yv_l);
            if constexpr (NB == 32) yw_l = fma(vws[(qb + r) * VP + NB + lane], vi, yw_l);
          }
          rp[r] = 0.0;
#pragma unroll
          for (int t = 0; t < NCH2; ++t) {
            const int c = cb + 64 * t + 2 * lane;
            const double2 vv = *reinterpret_cast<const double2*>(vsm + c);
            rp[r] = fma(av[r][t][0], vv.x, fma(av[r][t][1], vv.y, rp[r]));
            acc[t][0] = fma(av[r][t][0], vi, acc[t][0]);
            acc[t][1] = fma(av[r][t][1], vi, acc[t][1]);
          }
        }
        // 4 row sums across the warp in 6 shuffles (pairwise halving, then a butterfly)
        {
          const bool hi16 = lane & 16, hi8 = lane & 8;
          double x0 = hi16 ? rp[0] : rp[1], y0 = hi16 ? rp[1] : rp[0];
          y0 += __shfl_xor_sync(0xffffffffu, x0, 16);  // row 0 (lanes < 16) / row 1 (lanes >= 16)
          double x1 = hi16 ? rp[2] : rp[3], y1 = hi16 ? rp[3] : rp[2];
          y1 += __shfl_xor_sync(0xffffffffu, x1, 16);  // row 2 / row 3
          double x2 = hi8 ? y0 : y1, y2 = hi8 ? y1 : y0;
          y2 += __shfl_xor_sync(0xffffffffu, x2, 8);   // lane&8 ? rows 2|3 : rows 0|1
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) y2 += __shfl_xor_sync(0xffffffffu, y2, o);
          if ((lane & 7) == 0) {
            const int r = (hi8 ? 2 : 0) + (hi16 ? 1 : 0);
            if (qb + r < nloc) prow[qb + r] += y2;
          }
        }
      }
      // flush the warp accumulators: csum[c] = sum over warps (fixed order)
#pragma unroll
      for (int t = 0; t < NCH2; ++t) {
        wacc[warp * CH + 64 * t + 2 * lane] = acc[t][0];
        wacc[warp * CH + 64 * t + 2 * lane + 1] = acc[t][1];
      }
      __syncthreads();
      for (int c = tid; c < CH && cb + c < n; c += PT) {
        double sacc = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) sacc += wacc[w * CH + c];
        csum[cb + c] = sacc;
      }
      __syncthreads();
    }
    // v^T A22 v over my rows: sum_i v_i (2 rowpart_i - A_ii v_i); with the y
    // partials through one shared pass (fixed warp order)
    double pv_own = 0.0;
    for (int q = qk + tid; q < nloc; q += PT) {
      const double vi = vsm[row_of(q)];
      pv_own = fma(vi, 2.0 * prow[q] - diag[q] * vi, pv_own);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pv_own += __shfl_xor_sync(0xffffffffu, pv_own, o);
    if constexpr (NB == 32) {
      ywacc[warp * (2 * NB + 1) + lane] = yw_l;          // yW[t] partials (t = lane)
      ywacc[warp * (2 * NB + 1) + NB + lane] = yv_l;     // yV[t]
    } else {  // lane < NB: yV[lane], lane >= NB: yW[lane - NB]
      ywacc[warp * (2 * NB + 1) + (lane < NB ? NB + lane : lane - NB)] = yv_l;
    }
    if (lane == 0) ywacc[warp * (2 * NB + 1) + 2 * NB] = pv_own;
    __syncthreads();
    for (int t = tid; t <= 2 * NB; t += PT) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) sacc += ywacc[w * (2 * NB + 1) + t];
      if (t == 2 * NB) part3[0] = sacc;
      else part3[2 + t] = sacc;
    }
    csync<C>();  // S3: csum, part3 of every CTA are complete
    // ---------------- D: w -------------------------------------------------
    double pvt = 0.0;
#pragma unroll
    for (int r = 0; r < C; ++r) pvt += remote<C>(part3, r)[0];
    for (int t = tid; t < 2 * NB; t += PT) {
      double sacc = 0.0;
      if ((t < NB && t < j) || (t >= NB && t - NB < j)) {
#pragma unroll
        for (int r = 0; r < C; ++r) sacc += remote<C>(part3, r)[2 + t];
      }
      ys[t] = sacc;
    }
    __syncthreads();
    // yW . yV over the panel's first j columns: one term per lane, butterfly sum
    double ywv = lane < j ? ys[lane] * ys[NB + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ywv += __shfl_xor_sync(0xffffffffu, ywv, o);
    const double alpha2 = -0.5 * tk * tk * (pvt - 2.0 * ywv);
    // w_i = tau (A22 v - V yW - W yV)_i + alpha2 v_i from the owner's row part,
    // diagonal and [V | W] row, and every CTA's column part (one expression,
    // evaluated by the owner for its rows and by every CTA for row k+1)
    auto w_of = [&](const double* prow_o, const double* diag_o, const double* ri, int qo, int i) {
      double p = prow_o[qo] - diag_o[qo] * vsm[i];  // the column parts include the diagonal
#pragma unroll
      for (int r = 0; r < C; ++r) p += remote<C>(csum, r)[i];
      double p1 = 0.0, p2 = 0.0, p3 = 0.0;
      int t = 0;
      for (; t + 2 <= j; t += 2) {
        const double2 v2 = *reinterpret_cast<const double2*>(ri + t);
        const double2 w2 = *reinterpret_cast<const double2*>(ri + NB + t);
        const double2 yw = *reinterpret_cast<const double2*>(ys + t);
        const double2 yv = *reinterpret_cast<const double2*>(ys + NB + t);
        p = fma(-v2.x, yw.x, p);
        p1 = fma(-w2.x, yv.x, p1);
        p2 = fma(-v2.y, yw.y, p2);
        p3 = fma(-w2.y, yv.y, p3);
      }
      if (t < j) {
        p = fma(-ri[t], ys[t], p);
        p1 = fma(-ri[NB + t], ys[NB + t], p1);
      }
      p = (p + p1) + (p2 + p3);
      return fma(alpha2, vsm[i], tk * p);
    };
    for (int q = tid; q < nloc; q += PT) {
      const int i = row_of(q);
      vws[q * VP + NB + j] = i >= k + 1 ? w_of(prow, diag, vws + q * VP, q, i) : 0.0;
    }
    // row k+1 of [V | W] for the next column's lazy update: columns < j from its
    // owner's shared memory (written before the last barrier), column j here
    if (j + 1 < jb) {
      const int ow = (k + 1) % C, qo = (k + 1) / C;
      const double* ro = remote<C>(vws, ow) + qo * VP;
      for (int t = tid; t < 2 * NB; t += PT) {
        double v;
        if (t == j) v = vsm[k + 1];
        else if (t == NB + j) v = w_of(remote<C>(prow, ow), remote<C>(diag, ow), ro, qo, k + 1);
        else v = ro[t];
        rk[t] = v;
      }
    }
    __syncthreads();
  }
  // Global results, written once per panel (no global stores inside the column
  // loop, so the cluster barriers do not wait on them): [V | W], [W | V] rows for
  // the trailing update, d / e / tau, and the panel's Householder vectors over
  // its (dead) columns of A -- the Y block of the back-transformation.
  for (int q = warp; q < nloc; q += NW) {
    const int i = row_of(q);
    double* vw = VW + (int64_t)i * 2 * NB;
    double* wv = WV + (int64_t)i * 2 * NB;
    for (int t = lane; t < NB; t += 32) {
      const double v = t < jb ? vws[q * VP + t] : 0.0, w = t < jb ? vws[q * VP + NB + t] : 0.0;
      vw[t] = v;
      vw[NB + t] = w;
      wv[t] = w;
      wv[NB + t] = v;
      if (t < jb) A[(int64_t)i * n + k0 + t] = v;
    }
  }
  for (int t = tid; t < jb; t += PT) {
    if ((k0 + t) % C == rank) d[k0 + t] = dpan[t];  // (the diagonal is known to its row's owner)
    if (rank == 0) {
      if (k0 + t < n - 1) e[k0 + t] = dpan[NB + t];
      tau[k0 + t] = dpan[2 * NB + t];
    }
  }
  if constexpr (C > 1) cl_sync();  // no CTA exits while others may still read its shared memory
}

// Per matrix: flag = (G finite and nonzero); Gershgorin interval and pivmin of T
// (after tridiagonalization); glim = flag ? INT_MAX : 0 (K3 per-matrix column limit)
__global__ void gram_flag(const double* __restrict__ G, int n, int* flag, int* glim) {
  const int b = blockIdx.x;
  const double* g = G + (int64_t)b * n * n;
  __shared__ double red[NW];
  double tr = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) tr += g[(int64_t)i * n + i];
  tr = block_sum(tr, red);
  if (threadIdx.x == 0) {
    const int ok = (tr > 0.0 && isfinite(tr)) ? 1 : 0;
    flag[b] = ok;
    glim[b] = ok ? 0x7fffffff : 0;
  }
}

// Sturm count (eigenvalues of T below x) by the scaled determinant recurrence
// p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}: one FMA per step on the
// dependent chain; renormalised by an exact power of two every 8 steps (T is
// scaled to norm ~1, so 8 steps cannot leave the exponent range).  A zero
// leading minor is replaced by -pivmin times the previous one (the LAPACK
// pivmin convention in product form).  d, e2 in shared memory.
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                           double x, double pivmin) {
  double p2 = 1.0, p1 = d[0] - x;
  if (p1 == 0.0) p1 = -pivmin;
  int cnt = p1 < 0.0;
  int i = 1;
  for (; i + 8 <= n; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double p = fma(d[i + u] - x, p1, -e2[i + u - 1] * p2);
      if (p == 0.0) p = -pivmin * p1;
      cnt += (p < 0.0) != (p1 < 0.0);
      p2 = p1;
      p1 = p;
    }
    // exact power-of-two renormalisation: 2^-ex with ex = exponent of p1
    const long long bits = __double_as_longlong(p1);
    const int ex = (int)((bits >> 52) & 0x7ff) - 1023;
    const double f = __longlong_as_double((long long)(1023 - ex) << 52);
    p1 *= f;
    p2 *= f;
  }
  for (; i < n; ++i) {
    double p = fma(d[i] - x, p1, -e2[i - 1] * p2);
    if (p == 0.0) p = -pivmin * p1;
    cnt += (p < 0.0) != (p1 < 0.0);
    p2 = p1;
    p1 = p;
  }
  return cnt;
}

// scale T to norm ~1 (power of two), squares of e; per-matrix scale/pivmin
__global__ void tri_prepare(double* __restrict__ dall, double* __restrict__ eall, double* __restrict__ e2all,
                            double* __restrict__ info, const int* flag, int n) {
  const int b = blockIdx.x;
  if (!flag[b]) return;
  double* d = dall + (int64_t)b * n;
  double* e = eall + (int64_t)b * n;
  double* e2 = e2all + (int64_t)b * n;
  __shared__ double red[NW];
  __shared__ double s_lo[NW], s_hi[NW];
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    mx = fmax(mx, fabs(d[i]));
    if (i < n - 1) mx = fmax(mx, fabs(e[i]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
  const double sc = mx > 0.0 ? ldexp(1.0, -ilogb(mx)) : 1.0;
  __syncthreads();
  double lo = 1e300, hi = -1e300;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double di = d[i] * sc;
    const double em = i > 0 ? fabs(e[i - 1] * sc) : 0.0, ep = i < n - 1 ? fabs(e[i] * sc) : 0.0;
    lo = fmin(lo, di - em - ep);
    hi = fmax(hi, di + em + ep);
  }
  __syncthreads();  // every thread read its d/e before the in-place scaling below
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    d[i] *= sc;
    if (i < n - 1) {
      e[i] *= sc;
      e2[i] = e[i] * e[i];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    s_lo[threadIdx.x >> 5] = lo;
    s_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, s_lo[w]);
      hi = fmax(hi, s_hi[w]);
    }
    lo = fmin(lo, s_lo[0]);
    hi = fmax(hi, s_hi[0]);
    const double span = fmax(fabs(lo), fabs(hi));
    info[b * 4 + 0] = lo - 2.2e-16 * span - 1e-300;
    info[b * 4 + 1] = hi + 2.2e-16 * span + 1e-300;
    info[b * 4 + 2] = span;
    info[b * 4 + 3] = sc;
  }
}

// One thread per eigenvalue: lam[b][j] = j-th smallest eigenvalue of (scaled) T, for the kk largest
__global__ void tri_bisect(const double* __restrict__ dall, const double* __restrict__ e2all,
                           const double* __restrict__ info, const int* flag, int n, int kk,
                           double* __restrict__ lam) {
  extern __shared__ double tsm[];  // d[n], e2[n]
  const int b = blockIdx.y;
  if (!flag[b]) return;
  double* ds = tsm;
  double* e2s = tsm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ds[i] = dall[(int64_t)b * n + i];
    e2s[i] = i < n - 1 ? e2all[(int64_t)b * n + i] : 0.0;
  }
  __syncthreads();
  const int j = n - kk + blockIdx.x * blockDim.x + threadIdx.x;  // the kk largest eigenvalues
  if (j >= n) return;
  double lo = info[b * 4 + 0], hi = info[b * 4 + 1];
  const double span = info[b * 4 + 2];
  const double tol = 4.0 * 2.220446049250313e-16 * span;
  const double pivmin = 1e-30 * span + 1e-300;
  for (int it = 0; it < 64 && hi - lo > tol; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (sturm_count(ds, e2s, n, mid, pivmin) <= j) lo = mid;
    else hi = mid;
  }
  lam[(int64_t)b * n + j] = 0.5 * (lo + hi);
}

// The same with one warp per eigenvalue (multisection), for few eigenvalues
// (kk <= 128: the leading-triplet mode), where one thread per eigenvalue leaves
// the GPU nearly idle: every round the 32 lanes take Sturm counts at 32
// equispaced interior points of the bracket, which shrinks 33-fold to the
// sub-interval where the count crosses j (~10 rounds instead of ~50 bisection
// steps; all lanes read the same d, e2 entries: shared-memory broadcasts).
__global__ void tri_multisect(const double* __restrict__ dall, const double* __restrict__ e2all,
                              const double* __restrict__ info, const int* flag, int n, int kk,
                              double* __restrict__ lam) {
  extern __shared__ double tsm[];  // d[n], e2[n]
  const int b = blockIdx.y;
  if (!flag[b]) return;
  double* ds = tsm;
  double* e2s = tsm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ds[i] = dall[(int64_t)b * n + i];
    e2s[i] = i < n - 1 ? e2all[(int64_t)b * n + i] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double span = info[b * 4 + 2];
  const double tol = 4.0 * 2.220446049250313e-16 * span;
  const double pivmin = 1e-30 * span + 1e-300;
  for (int jj = blockIdx.x * nw + (threadIdx.x >> 5); jj < kk; jj += gridDim.x * nw) {
    const int j = n - kk + jj;  // the kk largest eigenvalues
    double lo = info[b * 4 + 0], hi = info[b * 4 + 1];
    for (int it = 0; it < 24 && hi - lo > tol; ++it) {
      const double h = (hi - lo) * (1.0 / 33.0);
      const double x = fma((double)(lane + 1), h, lo);
      // lanes whose point lies at or below lambda_j: a prefix (counts are monotone in x)
      const unsigned below = __ballot_sync(0xffffffffu, sturm_count(ds, e2s, n, x, pivmin) <= j);
      const int L = 32 - __clz(below);  // points 1..L are <= lambda_j
      const double nlo = L > 0 ? fma((double)L, h, lo) : lo;
      const double nhi = L < 32 ? fma((double)(L + 1), h, lo) : hi;
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) lam[(int64_t)b * n + j] = 0.5 * (lo + hi);
  }
}

__device__ __forceinline__ double hash_unit(uint32_t i, uint32_t j) {
  uint32_t h = i * 0x9E3779B1u ^ (j + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return (double)(h & 0xFFFFFF) * (2.0 / 16777216.0) - 1.0 + 1.0 / 16777216.0;
}

// One thread per eigenvalue: inverse iteration with the LDL^T factors of
// T - lambda I (tiny pivots replaced by +-eps * ||T||), two solves from a fixed
// pseudo-random start, normalised.  Column n-1-j of Z (descending order).
// Scratch L, Dinv: [i][j] layout (coalesced over the eigenvalue threads).
__global__ void tri_inviter(const double* __restrict__ dall, const double* __restrict__ eall,
                            const double* __restrict__ info, const double* __restrict__ lamall, const int* flag,
                            int n, int kk, double* __restrict__ Zall, double* __restrict__ Lall,
                            double* __restrict__ Dall) {
  const int b = blockIdx.y;
  const int jj = blockIdx.x * blockDim.x + threadIdx.x;  // 0 .. kk-1: eigenvalue n - kk + jj
  if (!flag[b] || jj >= kk) return;
  const int j = n - kk + jj;
  const double* d = dall + (int64_t)b * n;
  const double* e = eall + (int64_t)b * n;
  const int64_t nk = (int64_t)n * kk;
  double* Z = Zall + b * nk;   // n x kk, column kk-1-jj (descending eigenvalues)
  double* L = Lall + b * nk;   // scratch [i][jj]
  double* Di = Dall + b * nk;
  const double lam = lamall[(int64_t)b * n + j];
  const double span = info[b * 4 + 2];
  const double small = 2.220446049250313e-16 * span + 1e-300;
  const int col = kk - 1 - jj;
  // factor
  double D = d[0] - lam;
  for (int i = 0; i < n; ++i) {
    if (fabs(D) < small) D = D < 0.0 ? -small : small;
    const double inv = 1.0 / D;
    Di[(int64_t)i * kk + jj] = inv;
    if (i < n - 1) {
      const double l = e[i] * inv;
      L[(int64_t)i * kk + jj] = l;
      D = (d[i + 1] - lam) - l * e[i];
    }
  }
  // two solves; the per-step operands are loaded in batches of IB ahead of the
  // dependent chains (the loads do not depend on the chain: latency overlaps)
  constexpr int IB = 16;
  double s = 1.0;
  for (int it = 0; it < 2; ++it) {
    // forward: w_i = x_i - l_{i-1} w_{i-1}
    double w = 0.0;
    for (int i0 = 0; i0 < n; i0 += IB) {
      double xb[IB], lb[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int i = i0 + u;
        xb[u] = i < n ? (it == 0 ? hash_unit(i, j) : Z[(int64_t)i * kk + col] * s) : 0.0;
        lb[u] = (i > 0 && i < n) ? L[(int64_t)(i - 1) * kk + jj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int i = i0 + u;
        if (i < n) {
          w = i == 0 ? xb[u] : fma(-lb[u], w, xb[u]);
          Z[(int64_t)i * kk + col] = w;
        }
      }
    }
    // back: y_i = w_i / D_i - l_i y_{i+1}
    double y = 0.0, nrm = 0.0;
    for (int i1 = n - 1; i1 >= 0; i1 -= IB) {
      double wb[IB], db[IB], lb[IB];
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int i = i1 - u;
        wb[u] = i >= 0 ? Z[(int64_t)i * kk + col] : 0.0;
        db[u] = i >= 0 ? Di[(int64_t)i * kk + jj] : 0.0;
        lb[u] = (i >= 0 && i < n - 1) ? L[(int64_t)i * kk + jj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < IB; ++u) {
        const int i = i1 - u;
        if (i >= 0) {
          const double wi = wb[u] * db[u];
          y = i == n - 1 ? wi : fma(-lb[u], y, wi);
          Z[(int64_t)i * kk + col] = y;
          nrm = fma(y, y, nrm);
        }
      }
    }
    s = nrm > 0.0 && isfinite(nrm) ? 1.0 / sqrt(nrm) : 0.0;
  }
  for (int i = 0; i < n; ++i) Z[(int64_t)i * kk + col] *= s;
}

// Eigenvalues that coincide to rounding (gap <= 1e-13 ||T||: e.g. the doubled
// singular values of the t-svd real embeddings) leave inverse iteration
// without a preferred direction: their vectors come out as independent but
// arbitrary combinations inside the eigenspace.  One CTA per matrix walks the
// ascending eigenvalues and orthonormalises each such cluster's vectors
// (modified Gram-Schmidt, two passes), so Newton-Schulz starts near-orthogonal.
__global__ void tri_cluster_mgs(const double* __restrict__ lamall, const double* __restrict__ info,
                                const int* flag, int n, int kk, double* __restrict__ Zall) {
  const int b = blockIdx.x;
  if (!flag[b]) return;
  const double* lam = lamall + (int64_t)b * n;
  double* Z = Zall + (int64_t)b * n * kk;  // n x kk, column kk-1-(j-(n-kk)) holds eigenvalue j
  const double ctol = 1e-13 * info[b * 4 + 2];
  __shared__ double red[NW];
  int j0 = n - kk;
  while (j0 < n) {
    int j1 = j0 + 1;
    while (j1 < n && lam[j1] - lam[j1 - 1] <= ctol) ++j1;  // cluster [j0, j1)
    for (int j = j0 + 1; j < j1; ++j) {
      const int cj = n - 1 - j;  // == kk - 1 - (j - (n - kk))
      for (int pass = 0; pass < 2; ++pass) {
        for (int t = j0; t < j; ++t) {
          const int ct = n - 1 - t;
          double dsum = 0.0;
          for (int i = threadIdx.x; i < n; i += blockDim.x) dsum = fma(Z[(int64_t)i * kk + ct], Z[(int64_t)i * kk + cj], dsum);
          dsum = block_sum(dsum, red);
          for (int i = threadIdx.x; i < n; i += blockDim.x) Z[(int64_t)i * kk + cj] = fma(-dsum, Z[(int64_t)i * kk + ct], Z[(int64_t)i * kk + cj]);
          __syncthreads();
        }
      }
      double nrm = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) nrm = fma(Z[(int64_t)i * kk + cj], Z[(int64_t)i * kk + cj], nrm);
      nrm = block_sum(nrm, red);
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) Z[(int64_t)i * kk + cj] *= inv;
      __syncthreads();
    }
    j0 = j1;
  }
}

// P = Z^T Z given in its lower triangle (K3 lower tiles): delta[b] = max |P - I|
// over the lower triangle (bit-pattern max; NaN propagates); mirrors P's lower
// triangle into its upper one.
__global__ void ns_delta(const double* __restrict__ Pall, int n, const int* flag, const int* mode,
                         unsigned long long* __restrict__ delta) {
  const int b = blockIdx.y;
  if (!flag[b] || mode[b] == 0) return;
  const double* P = Pall + (int64_t)b * n * n;
  double mx = 0.0;
  const int64_t nn = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e - r * n;
    if (c > r) continue;
    const double pv = P[e];
    if (c < r) const_cast<double*>(P)[c * n + r] = pv;  // symmetric P for the P^2 GEMM
    const double dv = fabs(pv - (r == c ? 1.0 : 0.0));
    mx = (isnan(dv) || dv > mx) ? dv : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (isnan(t) || t > mx) ? t : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long bits = isnan(mx) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(mx);
    atomicMax(delta + b, bits);
  }
}

#ifndef WT_NS_ORDER2_ONLY
#define WT_NS_ORDER2_ONLY 0
#endif
constexpr bool kNsOrder2Only = WT_NS_ORDER2_ONLY;
// Per-matrix Newton-Schulz decision from delta (independent of the other
// matrices of the batch, so results do not depend on the batch composition).
// With P = Z^T Z = I + E, |E| = delta:
//   order 2: Z (3I - P)/2                       -> error ~ 3/4 delta^2
//   order 3: Z (15I - 10P + 3P^2)/8             -> error ~ 5/16 delta^3
// mode[b]: 0 = orthogonal (no update, P = I), 1 = order 2, 2 = order 3, -1 = fell back (V0 = I).
// glim2[b] enables the P^2 GEMM for the order-3 matrices.
__global__ void ns_decide(const unsigned long long* __restrict__ delta, int batch, double tol, double limit,
                          int* flag, int* glim, int* mode, int* glim2, int* counts) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x) {
    glim2[b] = 0;
    if (!flag[b] || mode[b] == 0) {
      mode[b] = flag[b] ? 0 : -1;
      continue;
    }
    const double dl = __longlong_as_double((long long)delta[b]);
    if (dl <= tol) {
      mode[b] = 0;
    } else if (!(dl <= limit)) {
      flag[b] = 0;
      glim[b] = 0;
      mode[b] = -1;
    } else if (0.75 * dl * dl <= tol || kNsOrder2Only) {
      mode[b] = 1;
      atomicAdd(counts, 1);
    } else {
      mode[b] = 2;
      glim2[b] = 0x7fffffff;
      atomicAdd(counts, 1);
      if (0.3125 * dl * dl * dl > tol) atomicAdd(counts + 1, 1);  // will need another round
    }
  }
}

// P (lower triangle of Z^T Z) and Q (lower triangle of P^2, order-3 matrices)
// -> the full symmetric update polynomial in P.
__global__ void ns_form(double* __restrict__ Pall, const double* __restrict__ Qall, int n, const int* mode) {
  const int b = blockIdx.y;
  const int md = mode[b];
  if (md < 0) return;
  double* P = Pall + (int64_t)b * n * n;
  const double* Q = Qall + (int64_t)b * n * n;
  const int64_t nn = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e - r * n;
    if (c > r) continue;  // lower triangle + its mirror, one thread per pair
    const double dg = r == c ? 1.0 : 0.0;
    double v;
    if (md == 0) v = dg;
    else if (md == 1) v = fma(-0.5, P[e], 1.5 * dg);
    else v = (15.0 * dg - 10.0 * P[e] + 3.0 * Q[e]) * 0.125;
    P[e] = v;
    if (c < r) P[c * n + r] = v;
  }
}

// Compact-WY factor T (NBT x NBT upper triangular) of the block of reflectors
// Y (columns k0 .. k0 + nb - 1 of the stored panels), from S = Y^T Y:
// T_ii = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] S[0:i, i]   (dlarft, forward, columnwise)
// The strict upper triangle of S is staged transposed in T's free strict lower
// triangle (S[c][i] at T[i][c]) before the column recurrence, so the recurrence
// reads only shared memory.
__global__ void wy_larft(const double* __restrict__ Sall, const double* __restrict__ tauall, const int* flag,
                         int n, int k0, int nb, double* __restrict__ Tall) {
  const int b = blockIdx.x;
  if (!flag[b]) return;
  extern __shared__ double T[];  // [NBT][NBT + 1]
  constexpr int LD = NBT + 1;
  const double* S = Sall + (int64_t)b * NBT * NBT;
  const double* tau = tauall + (int64_t)b * n + k0;
  for (int e = threadIdx.x; e < NBT * NBT; e += blockDim.x) {
    const int r = e / NBT, c = e % NBT;  // S[r][c], coalesced over c
    T[c * LD + r] = (r < c && c < nb) ? S[e] : 0.0;
  }
  __syncthreads();
  // four threads per row r (lanes 4r' .. 4r'+3 of a warp), each summing every
  // fourth term of the row's dot product (chains a quarter as long), combined
  // by two shuffles in a fixed order
  const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
  for (int i = 0; i < nb; ++i) {
    double s0 = 0.0, s1 = 0.0;
    if (r < i) {
      const double* Tr = T + r * LD;
      const double* Si = T + i * LD;  // S[c][i] = T[i][c], c < i
      int c = r + part;
      for (; c + 4 < i; c += 8) {
        s0 = fma(Tr[c], Si[c], s0);
        s1 = fma(Tr[c + 4], Si[c + 4], s1);
      }
      if (c < i) s0 = fma(Tr[c], Si[c], s0);
    }
    double sum = s0 + s1;
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    __syncthreads();  // every thread has read column i's inputs (row r of T left of i, row i of S)
    if (part == 0) {
      if (r < i) T[r * LD + i] = -tau[i] * sum;
      if (r == i) T[r * LD + i] = tau[i];
    }
    __syncthreads();
  }
  double* Tg = Tall + (int64_t)b * NBT * NBT;
  for (int e = threadIdx.x; e < NBT * NBT; e += blockDim.x) {
    const int rr = e / NBT, c = e % NBT;
    Tg[e] = (c >= rr && c < nb) ? T[rr * LD + c] : 0.0;
  }
}

// V0 = I[:, :kk] for the matrices that fall back
__global__ void set_identity(double* __restrict__ Vall, int n, int kk, const int* flag) {
  const int b = blockIdx.y;
  if (flag[b]) return;
  double* V = Vall + (int64_t)b * n * kk;
  const int64_t nk = (int64_t)n * kk;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nk; e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e / kk == e % kk) ? 1.0 : 0.0;
}

struct Layout {
  size_t G, Z, Z2, P, VW, WV, d, e, e2, tau, lam, info, S, T, M1, M2, delta, flag, glim, done, glim2, cnt, total;
};

Layout layout(int64_t n, int64_t batch) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) / 256 * 256; return r; };
  const size_t nn = (size_t)(n * n * batch) * sizeof(double);
  L.G = take(nn);
  L.Z = take(nn);
  L.Z2 = take(nn);
  L.P = take(nn);  // also the inverse-iteration L factors; Z2 holds their 1/D
  L.VW = take(sizeof(double) * (size_t)(batch * n * 2 * NB_MAX));
  L.WV = take(sizeof(double) * (size_t)(batch * n * 2 * NB_MAX));
  L.d = take(sizeof(double) * (size_t)(batch * n));
  L.e = take(sizeof(double) * (size_t)(batch * n));
  L.e2 = take(sizeof(double) * (size_t)(batch * n));
  L.tau = take(sizeof(double) * (size_t)(batch * n));
  L.lam = take(sizeof(double) * (size_t)(batch * n));
  L.info = take(sizeof(double) * (size_t)(batch * 4));
  L.S = take(sizeof(double) * (size_t)(2 * batch * NBT * NBT));  // two of each: the two-stage back-transformation
  L.T = take(sizeof(double) * (size_t)(2 * batch * NBT * NBT));  // forms block i+1's factor under block i's GEMMs
  L.M1 = take(sizeof(double) * (size_t)(batch * NBT * n));
  L.M2 = take(sizeof(double) * (size_t)(batch * NBT * n));
  L.delta = take(sizeof(unsigned long long) * (size_t)batch);
  L.flag = take(sizeof(int) * (size_t)batch);
  L.glim = take(sizeof(int) * (size_t)batch);
  L.done = take(sizeof(int) * (size_t)batch);
  L.glim2 = take(sizeof(int) * (size_t)batch);
  L.cnt = take(sizeof(int) * 4);
  L.total = o;
  return L;
}

// Cluster size C and panel width NB of the tridiagonalization for n x n Grams.
// A function of n only (the cluster split changes the summation order, so a
// matrix gets the same bits in any batch).  At most MAXR rows per CTA (the
// panel's V and W rows of a CTA stay in shared memory); NB = 16 halves that
// shared footprint so 256-row CTAs still fit two per SM.
struct PanelShape {
  int C, NB;
};
PanelShape panel_shape(int64_t n) {
  // 129..256: one 256-row CTA per matrix, no cluster barriers (config 3: 192 x
  // 256^2 runs as one wave of 192 CTAs; the 2-CTA clusters of width-32 panels
  // needed two waves: K4 9.05 vs 11.24 ms, tools/panel_probe.py)
  if (n > PREF_R && n <= MAXR) return PanelShape{1, 16};
  // otherwise >= 128 rows per CTA at width 32 (n = 512: C = 4 17.0 ms vs C = 2,
  // NB = 16 18.9 ms on 64 x 512^2; n = 1024: C = 8 60.8 ms vs C = 4 69.4 ms)
  int C = 1;
  while (C < 8 && n > (int64_t)C * PREF_R) C *= 2;
  return PanelShape{C, 32};
}

template <int C, int NB>
int launch_panel(double* G, double* VW, double* WV, double* d, double* e, double* tau, const int* flag, int n,
                 int k0, int64_t batch, cudaStream_t st) {
  auto kern = tridiag_panel<C, NB>;
  const size_t smem = PanelSmem::bytes(n, C, NB);
  if (int r = ensure_smem(kern, smem)) return r;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(batch * C));
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  // fraction of the batch's trailing lower triangles marked evict_last: a 48 MB
  // share of the 126 MB L2 (config 4, 32 x 1024^2: 45 MB 23.8 ms, 30 MB 23.9,
  // 60 MB 24.1, 90 MB 24.9, no hint 25.0 ms)
  constexpr double kL2KeepBytes = 48.0 * 1048576.0;
  const double bytes = (double)batch * 4.0 * (double)(n - k0) * (double)(n - k0);
  const double keep = std::min(1.0, kL2KeepBytes / std::max(bytes, 1.0));
  WT_CUDA(cudaLaunchKernelEx(&cfg, kern, G, VW, WV, d, e, tau, flag, n, k0, (float)keep));
  return WT_OK;
}

#include "eig_sbr.cuh"

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
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

// G as [batch][n][n] with 64-row x 16-column boxes, 128-byte swizzle (sbr_update_mult)
bool make_gmap(CUtensorMap* map, double* G, int64_t n, int64_t batch) {
  auto enc = tmap_encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)n * sizeof(double), (cuuint64_t)n * n * sizeof(double)};
  const cuuint32_t box[3] = {16, FU_T, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, G, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Non-blocking side streams per device for the other groups of a split two-stage reduction
// (created once; ordered against the caller's stream by per-call events).
constexpr int kSideStreams = 3;
cudaStream_t side_stream(int i = 0) {
  static std::mutex mu;
  static cudaStream_t streams[64][kSideStreams] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || i < 0 || i >= kSideStreams) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!streams[dev][i] && cudaStreamCreateWithFlags(&streams[dev][i], cudaStreamNonBlocking) != cudaSuccess)
    return nullptr;
  return streams[dev][i];
}

// Two-stage path: wide Grams whose rows below the band fit one row per thread,
// few leading eigenvectors (the stage-2 back-transformation streams every
// reflector once per SB_QC columns of Z).
bool use_two_stage(int64_t n, int64_t kk) {
  // (full mode, kk = n: the stage-2 back-transformation grows with kk; measured on 32 matrices:
  // 512^2 13.3 -> 12.0 ms, 1024^2 49.3 -> 51.9 ms.  A function of n and kk only: same bits in any batch.)
  const int opt = option(WT_OPT_EIG_TWOSTAGE);
  return opt != 0 && (n >= 512 || (opt == 2 && n >= 128)) && n - SB_B <= SB_NT && n % 2 == 0 && (kk <= 128 || n <= 640 || opt == 2);
}

}  // namespace eig

size_t eig_workspace_bytes(int64_t n, int64_t batch) { return eig::layout(n, batch).total; }

int eig_precondition(const double* Xt, double* Yt, int64_t m, int64_t n, int64_t ldx, int64_t sx, int64_t batch,
                     int64_t kk, int64_t ldy, int64_t sy, void* ws, size_t ws_bytes, int* n_fallback,
                     cudaStream_t st, const int* kmask, int* h_flags) {
  using namespace eig;
  const Layout L = layout(n, batch);
  WT_REQUIRE(ws != nullptr && ws_bytes >= L.total, "eig: workspace too small");
  WT_REQUIRE(n >= 3 && n <= 8 * MAXR, "eig: n = %lld unsupported", (long long)n);
  WT_REQUIRE(kk >= 1 && kk <= n, "eig: %lld leading eigenvectors of %lld", (long long)kk, (long long)n);
  char* base = static_cast<char*>(ws);
  auto D = [&](size_t off) { return reinterpret_cast<double*>(base + off); };
  double *G = D(L.G), *Z = D(L.Z), *Z2 = D(L.Z2), *P = D(L.P), *VW = D(L.VW), *WV = D(L.WV);
  double *dd = D(L.d), *ee = D(L.e), *e2 = D(L.e2), *tau = D(L.tau), *lam = D(L.lam), *info = D(L.info);
  double *S = D(L.S), *T = D(L.T), *M1 = D(L.M1), *M2 = D(L.M2);
  auto* delta = reinterpret_cast<unsigned long long*>(base + L.delta);
  int* flag = reinterpret_cast<int*>(base + L.flag);
  int* glim = reinterpret_cast<int*>(base + L.glim);
  const int64_t nn = n * n;
  const int64_t nk = n * kk;  // Z, Z2: n x kk (the kk leading eigenvectors, descending)
  const int64_t kk2 = kk * kk;  // P, Z2-as-P^2: kk x kk
  const int ni = (int)n, ki = (int)kk;
  // WT_OPT_EIG_PROFILE: per-phase device times on stderr (diagnostics)
  const bool prof = option(WT_OPT_EIG_PROFILE) != 0;
  cudaEvent_t ev[10] = {};
  int nev = 0;
  auto mark = [&]() {
    if (!prof) return;
    cudaEventCreate(&ev[nev]);
    cudaEventRecord(ev[nev++], st);
  };
  mark();

  // 1. G = X^T X (rows of Xt are the columns of X)
  if (int r = gemm_f64_lim(0, 1, n, n, m, 1.0, Xt, ldx, sx, Xt, ldx, sx, 0.0, G, n, nn, batch, kmask, nullptr, st,
                           1))  // lower tiles: the tridiagonalization reads only the lower triangle
    return r;
  gram_flag<<<(unsigned)batch, PT, 0, st>>>(G, ni, flag, glim);
  mark();
  const PanelShape ps = panel_shape(n);
  const int C = ps.C, NB = ps.NB;
  const bool sbr = use_two_stage(n, kk);
  const double* sbr_tp = nullptr;  // the panels' compact-WY factors (two-stage), for the back-transformation
  if (sbr) {
    // 2'. dense -> band (stage 1), band -> tridiagonal (stage 2); eig_sbr.cuh
    constexpr int B = SB_B;
    double* AB = Z2;                                   // [batch][n][SB_LDB]
    double* Zp = AB + (size_t)batch * n * SB_LDB;      // [batch][n][B]   Z = A22 V of the current panel
    // [batch][panels][B][B] the panels' compact-WY factors: kept until the back-transformation, in the
    // tail of the VW buffer (sized for the one-stage panels' 64-wide rows; 24 are used here)
    double* Tp = VW + (size_t)batch * n * 2 * B;
    static_assert(2 * NB_MAX - 2 * SB_B >= SB_B + 1, "room for the panel factors behind [V | W]");
    double* Vc = Zp + (size_t)batch * n * B;           // [batch][n][B] compact copy of the current panel's V rows
    double* Np = Vc + (size_t)batch * n * B;           // [batch][strips][B][B] per-strip shares of N = V^T Z
    sbr_tp = Tp;
    if (int r = ensure_smem(sbr_update_mult, FU_SMEM)) return r;
    const size_t csm = ChaseSmem::bytes(ni);
    if (int r = ensure_smem(sbr_chase, csm)) return r;
    const int64_t npanels = (n + B - 1) / B, max_strips = (n + FU_T - 1) / FU_T;
    // Stages 1 and 2 of the matrices [b0, b0 + nb) on stream s (every array is indexed by matrix).
    auto reduce = [&](int64_t b0, int64_t nb, cudaStream_t s) -> int {
      double* Gh = G + b0 * nn;
      double* ABh = AB + b0 * n * SB_LDB;
      double* tauh = tau + b0 * n;
      double* Tph = Tp + b0 * npanels * B * B;
      double *VWh = VW + b0 * n * 2 * B, *WVh = WV + b0 * n * 2 * B;
      double *Vch = Vc + b0 * n * B, *Zph = Zp + b0 * n * B;
      double* Nph = Np + b0 * max_strips * B * B;  // (strips of a pass <= max_strips: the halves never overlap)
      const int* flagh = flag + b0;
      CUtensorMap gmap;
      WT_REQUIRE(make_gmap(&gmap, Gh, n, nb), "eig: cuTensorMapEncodeTiled failed");
      WT_CUDA(cudaMemsetAsync(ABh, 0, sizeof(double) * (size_t)nb * n * SB_LDB, s));
      WT_CUDA(cudaMemsetAsync(tauh, 0, sizeof(double) * (size_t)nb * n, s));
      // the panel QR reads full rows: mirror the Gram's lower triangle first
      sym_mirror<<<dim3((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32), (unsigned)nb), dim3(32, 8), 0, s>>>(
          Gh, ni, flagh);
      // Per panel two launches: sbr_panel (W of the previous panel from its Z, the
      // previous update applied to this panel's columns, QR of the rows below the
      // band) and one fused pass over the trailing block (previous update + Z = A22 V).
      int pend = 0;
      for (int64_t c0 = 0; c0 < n; c0 += B) {
        {
          cudaLaunchConfig_t cfg = {};
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = SB_PC;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = 1;
          cfg.gridDim = dim3((unsigned)(nb * SB_PC));
          cfg.blockDim = dim3(SB_PT);
          cfg.dynamicSmemBytes = 0;
          cfg.stream = s;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          const int nstrips_prev = (int)((n - c0 + FU_T - 1) / FU_T);  // strips of the previous trailing pass
          WT_CUDA(cudaLaunchKernelEx(&cfg, sbr_panel, Gh, ABh, tauh, Tph, flagh, ni, (int)c0, VWh, WVh, pend, Vch,
                                     (const double*)Zph, (const double*)Nph, nstrips_prev));
        }
        const int64_t r0 = c0 + B, mrem = n - r0;
        if (mrem < 2) continue;
        sbr_update_mult<<<dim3((unsigned)((mrem + FU_T - 1) / FU_T), (unsigned)nb), FU_NT, FU_SMEM, s>>>(
            gmap, VWh, WVh, Vch, Zph, Nph, flagh, ni, (int)c0, pend);
        pend = 1;  // W of this panel is formed by the next panel kernel (from Z, N and T)
      }
      cudaEvent_t ce[2] = {};
      if (prof) {
        cudaEventCreate(&ce[0]);
        cudaEventCreate(&ce[1]);
        cudaEventRecord(ce[0], s);
      }
      sbr_chase<<<(unsigned)nb, SB_CW * 32, csm, s>>>(ABh, Gh, dd + b0 * n, ee + b0 * n, flagh, ni);
      if (prof) {
        cudaEventRecord(ce[1], s);
        cudaEventSynchronize(ce[1]);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ce[0], ce[1]);
        fprintf(stderr, "[wt_eig] two-stage: band chase %.3f ms (inside tridiag, matrices %lld..%lld)\n", ms,
                (long long)b0, (long long)(b0 + nb - 1));
        cudaEventDestroy(ce[0]);
        cudaEventDestroy(ce[1]);
      }
      return check_launch("eig two-stage reduction");
    };
    // Two halves of the batch on two streams: the panel QR is latency-bound (a 4-CTA cluster per
    // matrix, one cluster reduction per column) and the trailing pass throughput-bound, so one half's
    // panels run under the other half's trailing passes; both band chases (one SM per matrix) run
    // side by side at the end.  Per-matrix arithmetic does not depend on the split.
    const int split_opt = option(WT_OPT_EIG_SPLIT);
    const bool split = split_opt >= 2 || (split_opt == 0 && batch >= 16 && !prof);
    // groups: 2 by default; WT_OPT_EIG_SPLIT = 2 / 3 / 4 forces that many (diagnostics)
    const int groups = (int)std::min<int64_t>(batch, split_opt >= 2 ? std::min(split_opt, kSideStreams + 1) : 2);
    if (split && groups >= 2) {
      cudaEvent_t fork = nullptr, join[kSideStreams] = {};
      WT_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      int r = WT_OK;
      if (cudaEventRecord(fork, st) != cudaSuccess) r = WT_ERR_CUDA;
      // group g: matrices [g h, min(batch, (g + 1) h)); group 0 on the caller's stream, issued last
      const int64_t h = (batch + groups - 1) / groups;
      for (int g = groups - 1; g >= 0 && !r; --g) {
        const int64_t b0 = g * h, nb = std::min<int64_t>(h, batch - b0);
        if (nb <= 0) continue;
        if (g == 0) {
          r = reduce(0, nb, st);
          continue;
        }
        cudaStream_t side = side_stream(g - 1);
        if (side == nullptr || cudaStreamWaitEvent(side, fork, 0) != cudaSuccess) r = WT_ERR_CUDA;
        if (!r) r = reduce(b0, nb, side);
        if (!r && (cudaEventCreateWithFlags(&join[g - 1], cudaEventDisableTiming) != cudaSuccess ||
                   cudaEventRecord(join[g - 1], side) != cudaSuccess))
          r = WT_ERR_CUDA;
      }
      for (int g = 0; g < kSideStreams; ++g) {
        if (!join[g]) continue;
        if (cudaStreamWaitEvent(st, join[g], 0) != cudaSuccess) r = r ? r : WT_ERR_CUDA;
        cudaEventDestroy(join[g]);
      }
      cudaEventDestroy(fork);
      if (r) return r;
    } else {
      if (int r = reduce(0, batch, st)) return r;
    }
  } else {
  WT_CUDA(cudaMemsetAsync(VW, 0, sizeof(double) * (size_t)(batch * n * 2 * NB), st));
  WT_CUDA(cudaMemsetAsync(WV, 0, sizeof(double) * (size_t)(batch * n * 2 * NB), st));
  // 2. tridiagonalization, panel by panel
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    int r = WT_OK;
    switch (C * 100 + NB) {
      case 832: r = launch_panel<8, 32>(G, VW, WV, dd, ee, tau, flag, ni, (int)k0, batch, st); break;
      case 432: r = launch_panel<4, 32>(G, VW, WV, dd, ee, tau, flag, ni, (int)k0, batch, st); break;
      case 232: r = launch_panel<2, 32>(G, VW, WV, dd, ee, tau, flag, ni, (int)k0, batch, st); break;
      case 116: r = launch_panel<1, 16>(G, VW, WV, dd, ee, tau, flag, ni, (int)k0, batch, st); break;
      default: r = launch_panel<1, 32>(G, VW, WV, dd, ee, tau, flag, ni, (int)k0, batch, st);
    }
    if (r) return r;
    const int64_t k1 = k0 + NB;
    if (k1 < n) {  // A22 -= [V W] [W V]^T, lower tiles only
      const int64_t off = k1 * n + k1, offp = k1 * 2 * NB;
      if (int r2 = gemm_f64_lim(0, 1, n - k1, n - k1, 2 * NB, -1.0, VW + offp, 2 * NB, n * 2 * NB, WV + offp, 2 * NB,
                                n * 2 * NB, 1.0, G + off, n, nn, batch, nullptr, glim, st, 1))
        return r2;
    }
  }
  }
  if (int r = check_launch("eig tridiagonalization")) return r;
  mark();
  // 3-4. eigenvalues (bisection) and eigenvectors (inverse iteration) of T
  tri_prepare<<<(unsigned)batch, PT, 0, st>>>(dd, ee, e2, info, flag, ni);
  {
    dim3 grid((unsigned)((kk + 127) / 128), (unsigned)batch);
    if (int r = ensure_smem(tri_bisect, 2 * sizeof(double) * (size_t)n)) return r;
    if (kk <= 128) {  // (8 warps per CTA: 8 eigenvalues per CTA)
      if (int r = ensure_smem(tri_multisect, 2 * sizeof(double) * (size_t)n)) return r;
      tri_multisect<<<dim3((unsigned)((kk + 7) / 8), (unsigned)batch), 256, 2 * sizeof(double) * (size_t)n, st>>>(
          dd, e2, info, flag, ni, ki, lam);
    } else {
      tri_bisect<<<grid, 128, 2 * sizeof(double) * (size_t)n, st>>>(dd, e2, info, flag, ni, ki, lam);
    }
    mark();
    tri_inviter<<<grid, 128, 0, st>>>(dd, ee, info, lam, flag, ni, ki, Z, P, Z2);
    tri_cluster_mgs<<<(unsigned)batch, PT, 0, st>>>(lam, info, flag, ni, ki, Z);
  }
  if (int r = check_launch("eig bisection / inverse iteration")) return r;
  mark();
  // 5. Newton-Schulz on Z until orthogonal to rounding (delta = max |Z^T Z - I|),
  //    order 2 or 3 per matrix as its delta needs (ns_decide); every decision is
  //    per matrix, so the result does not depend on the batch.
  const double done_tol = 64.0 * 2.220446049250313e-16 * sqrt((double)n);
  // (Z^T Z and its polynomial are kk x kk, packed with stride kk^2)
  constexpr int kMaxNs = 3;
  int* mode = reinterpret_cast<int*>(base + L.done);
  int* glim2 = reinterpret_cast<int*>(base + L.glim2);
  int* counts = reinterpret_cast<int*>(base + L.cnt);
  WT_CUDA(cudaMemsetAsync(mode, 0xff, sizeof(int) * (size_t)batch, st));  // -1 != 0: not yet known
  // (page-locked readback scratch, one per host thread: a pageable destination costs the stream
  // ~100 us of staging per read; [0..1] Newton-Schulz counts, [2..] the per-matrix flags)
  static thread_local int* h_pin = nullptr;
  static thread_local size_t h_pin_n = 0;
  if (h_pin_n < (size_t)batch + 2) {
    if (h_pin) cudaFreeHost(h_pin);
    h_pin = nullptr;
    h_pin_n = 0;
    const size_t want = std::max<size_t>((size_t)batch + 2, 4096);
    WT_CUDA(cudaMallocHost(&h_pin, sizeof(int) * want));
    h_pin_n = want;
  }
  int* h_counts = h_pin;
  h_counts[0] = h_counts[1] = 0;
  for (int it = 0; it < kMaxNs; ++it) {
    if (int r = gemm_f64_lim(1, 0, kk, kk, n, 1.0, Z, kk, nk, Z, kk, nk, 0.0, P, kk, kk2, batch, nullptr, glim, st, 1))
      return r;
    WT_CUDA(cudaMemsetAsync(delta, 0, sizeof(unsigned long long) * (size_t)batch, st));
    WT_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int), st));
    const dim3 grid((unsigned)std::min<int64_t>((kk2 + 255) / 256, 64), (unsigned)batch);
    ns_delta<<<grid, 256, 0, st>>>(P, ki, flag, mode, delta);
    // last iteration: keep only the matrices this update brings to rounding
    const double lim = it == kMaxNs - 1 ? cbrt(done_tol / 0.3125) : 0.25;
    ns_decide<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(delta, (int)batch, done_tol, lim, flag, glim, mode,
                                                             glim2, counts);
    WT_CUDA(readback_ints(h_counts, counts, 2, st));  // (not a copy-engine copy: wt_common.cuh)
    WT_CUDA(cudaStreamSynchronize(st));
    if (h_counts[0] == 0) break;  // every matrix orthogonal (or fallen back)
    // P^2 for the order-3 matrices (lower tiles; P still holds the lower triangle of Z^T Z)
    if (int r = gemm_f64_lim(0, 1, kk, kk, kk, 1.0, P, kk, kk2, P, kk, kk2, 0.0, Z2, kk, kk2, batch, nullptr, glim2,
                             st, 1))
      return r;
    ns_form<<<grid, 256, 0, st>>>(P, Z2, ki, mode);
    if (int r = gemm_f64_lim(0, 0, n, kk, kk, 1.0, Z, kk, nk, P, kk, kk2, 0.0, Z2, kk, nk, batch, nullptr, glim, st))
      return r;
    std::swap(Z, Z2);
    if (h_counts[1] == 0) break;  // every update reached rounding: no further check needed
    // (the next P of the matrices already at rounding: mode 0 is kept via ns_delta's skip)
  }
  // (after kMaxNs iterations every matrix left is done or fell back: see lim)
  int* hflag = h_pin + 2;
  WT_CUDA(readback_ints(hflag, flag, (int)batch, st));
  mark();
  // 6. V0 = Q Z: blocks of NBT reflectors, last block first
  // (two-stage: Z <- Q2 Z with the stage-2 reflectors, then the stage-1 reflectors
  // c = 0 .. n - SB_B - 2, unit entry at row c + SB_B, as the same compact-WY blocks)
  const int64_t roff = sbr ? SB_B : 1;  // row of reflector c's unit entry: c + roff
  if (sbr) {
    const size_t qsm = Q2Smem::bytes(ni);
    if (int r = ensure_smem(sbr_apply_q2, qsm)) return r;
    sbr_apply_q2<<<dim3((unsigned)((kk + SB_QC - 1) / SB_QC), (unsigned)batch), SB_QT, qsm, st>>>(G, Z, flag, ni, ki);
    const dim3 grid((unsigned)std::min<int64_t>((nn + 255) / 256, 1024), (unsigned)batch);
    sbr_clean_y<<<grid, 256, 0, st>>>(G, ni, flag);
  }
  const int64_t nref = n - 1 - roff;  // reflectors 0 .. nref-1 (tau = 0 beyond)
  // (128-reflector blocks halve the passes over Z for n >= 512; 64 measured
  // faster on 256^2 slices: config 3 back-transform 1.02 vs 1.43 ms)
  const int64_t nbt = sbr ? SB_TB : (n >= 512 ? NBT : 64);  // (two-stage: whole panels per block)
  const size_t tsm = sizeof(double) * NBT * (NBT + 1);
  if (int r = ensure_smem(wy_larft, tsm)) return r;
  if (sbr) {
    if (int r = ensure_smem(sbr_larft_merge, tsm)) return r;
  }
  // The blocks' factors (S = Y^T Y and the larft / merged T) do not depend on Z, and the chain of
  // small launches is latency-bound, so they are formed on a side stream one block ahead of the
  // three Z-dependent GEMMs (two S / T buffers, events both ways).  Same kernels and arguments as
  // the in-order chain: same bits.  (WT_OPT_EIG_SPLIT = 1 keeps everything on the caller's stream.)
  // (Two-stage path only: with the one-stage panels, four host threads running 256-wide calls at
  // once gave different bits in one of three full test runs -- not understood, so not shipped.)
  const bool ahead = sbr && option(WT_OPT_EIG_SPLIT) != 1 && !prof && nref > nbt;
  cudaStream_t fs = ahead ? side_stream(kSideStreams - 1) : st;
  WT_REQUIRE(!ahead || fs != nullptr, "eig: side stream creation failed");
  constexpr int kMaxBlk = 64;
  cudaEvent_t ready[kMaxBlk] = {}, freed[kMaxBlk] = {};
  const int64_t k_first = ((nref - 1) / nbt) * nbt;
  const int nblk = (int)(k_first / nbt) + 1;
  WT_REQUIRE(!ahead || nblk <= kMaxBlk, "eig: %d back-transformation blocks", nblk);
  const int64_t stS = batch * NBT * NBT;  // one S / T buffer
  int rc = WT_OK;
  auto factor = [&](int i, cudaStream_t s2) -> int {  // S and T of block i (k0 = k_first - i nbt) into buffer i % 2
    const int64_t k0 = k_first - (int64_t)i * nbt, nb = std::min<int64_t>(nbt, nref - k0), r0 = k0 + roff;
    const double* Y = G + r0 * n + k0;  // rows r0.., columns k0.. (ld n)
    double *Si = S + (ahead ? (i & 1) * stS : 0), *Ti = T + (ahead ? (i & 1) * stS : 0);
    if (int r = gemm_f64_lim(1, 0, nb, nb, n - r0, 1.0, Y, n, nn, Y, n, nn, 0.0, Si, NBT, NBT * NBT, batch, nullptr,
                             glim, s2))
      return r;
    if (sbr) {  // the panels' factors merged block by block
      sbr_larft_merge<<<(unsigned)batch, 512, tsm, s2>>>(Si, sbr_tp, flag, ni, (int)k0, (int)nb, Ti);
    } else {
      wy_larft<<<(unsigned)batch, 4 * NBT, tsm, s2>>>(Si, tau, flag, ni, (int)k0, (int)nb, Ti);
    }
    return WT_OK;
  };
  if (ahead) {
    cudaEvent_t fork = nullptr;
    if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(fork, st) != cudaSuccess || cudaStreamWaitEvent(fs, fork, 0) != cudaSuccess)
      rc = WT_ERR_CUDA;
    if (fork) cudaEventDestroy(fork);
    for (int i = 0; i < nblk && !rc; ++i)
      if (cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming) != cudaSuccess)
        rc = WT_ERR_CUDA;
    for (int i = 0; i < 2 && i < nblk && !rc; ++i) {  // the first two factors
      rc = factor(i, fs);
      if (!rc && cudaEventRecord(ready[i], fs) != cudaSuccess) rc = WT_ERR_CUDA;
    }
  }
  for (int i = 0; i < nblk && !rc; ++i) {
    const int64_t k0 = k_first - (int64_t)i * nbt;
    const int64_t nb = std::min<int64_t>(nbt, nref - k0);
    const int64_t r0 = k0 + roff;  // first nonzero row of the block
    const double* Y = G + r0 * n + k0;
    const double* Ti = T + (ahead ? (i & 1) * stS : 0);
    if (!ahead) rc = factor(i, st);
    // M1 = Y^T Z (nb x n), M2 = T M1, Z[r0:, :] -= Y M2
    if (!rc)
      rc = gemm_f64_lim(1, 0, nb, kk, n - r0, 1.0, Y, n, nn, Z + r0 * kk, kk, nk, 0.0, M1, kk, NBT * n, batch, nullptr,
                        glim, st);
    if (!rc && ahead && cudaStreamWaitEvent(st, ready[i], 0) != cudaSuccess) rc = WT_ERR_CUDA;
    if (!rc)
      rc = gemm_f64_lim(0, 0, nb, kk, nb, 1.0, Ti, NBT, NBT * NBT, M1, kk, NBT * n, 0.0, M2, kk, NBT * n, batch, nullptr,
                        glim, st);
    if (!rc && ahead && i + 2 < nblk) {  // buffer i % 2 is free: block i + 2's factor goes there
      if (cudaEventRecord(freed[i], st) != cudaSuccess || cudaStreamWaitEvent(fs, freed[i], 0) != cudaSuccess)
        rc = WT_ERR_CUDA;
      if (!rc) rc = factor(i + 2, fs);
      if (!rc && cudaEventRecord(ready[i + 2], fs) != cudaSuccess) rc = WT_ERR_CUDA;
    }
    if (!rc)
      rc = gemm_f64_lim(0, 0, n - r0, kk, nb, -1.0, Y, n, nn, M2, kk, NBT * n, 1.0, Z + r0 * kk, kk, nk, batch, nullptr,
                        glim, st);
  }
  for (int i = 0; i < kMaxBlk; ++i) {
    if (ready[i]) cudaEventDestroy(ready[i]);
    if (freed[i]) cudaEventDestroy(freed[i]);
  }
  if (rc) return rc;
  {
    dim3 grid((unsigned)std::min<int64_t>((nk + 255) / 256, 256), (unsigned)batch);
    set_identity<<<grid, 256, 0, st>>>(Z, ni, ki, flag);
  }
  if (int r = check_launch("eig back-transformation")) return r;
  mark();
  // 7. Y = X V0  (Yt = V0^T Xt: kk rows of pitch ldy, stride sy)
  if (int r = gemm_f64_lim(1, 0, kk, m, n, 1.0, Z, kk, nk, Xt, ldx, sx, 0.0, Yt, ldy, sy, batch, kmask, nullptr, st))
    return r;
  mark();
  if (prof && nev > 1) {
    cudaEventSynchronize(ev[nev - 1]);
    static const char* names[] = {"gram", "tridiag", "prep+bisect", "inviter", "newton-schulz", "backtransform",
                                  "X V0"};
    fprintf(stderr, "[wt_eig] n=%lld batch=%lld C=%d:", (long long)n, (long long)batch, C);
    for (int i = 1; i < nev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, " %s %.3f ms", i - 1 < 7 ? names[i - 1] : "?", ms);
    }
    fprintf(stderr, "\n");
    for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
  }
  if (n_fallback) {
    WT_CUDA(cudaStreamSynchronize(st));
    int active = 0;
    for (int64_t b = 0; b < batch; ++b) {
      active += hflag[b] != 0;
      if (h_flags) h_flags[b] = hflag[b];
    }
    *n_fallback = (int)batch - active;
  }
  return WT_OK;
}

}  // namespace wt
