// K3: strided-batched FP64 GEMM on the B200 DMMA pipe.
//
// Replaces the per-slice cblas_dgemm calls of the reference:
//   slicewise_matmul   algebra.py:18-28       (face product, all levels at once)
//   _truncated_blocks  decomposition.py:70-72 (rank-r reconstruction)
//   _pinv_stack        decomposition.py:162   (V diag(s+) U^T assembly)
//
// sm_100a has no FP64 tcgen05 kind (ptxas rejects .kind::f64), so the FP64
// tensor path is the warp-level mma.sync m8n8k4 f64 (SASS DMMA.8x8x4) fed from
// registers.  Design: CTA tile BM x BN x 16, 3-stage cp.async (LDGSTS) ring in
// shared memory, row pitches padded to 4 (mod 16) doubles so every fragment
// LDS.64 is bank-conflict-free for both operand orientations, warp tile
// (BM/WM) x (BN/WN) held as DMMA accumulators.
//
// Row-major semantics: C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b].
#include <algorithm>

#include "wt_common.cuh"

namespace wt {
namespace {

#ifndef WT_GEMM_BK
#define WT_GEMM_BK 16
#endif
#ifndef WT_GEMM_STAGES
#define WT_GEMM_STAGES 3
#endif
constexpr int BK = WT_GEMM_BK;
constexpr int STAGES = WT_GEMM_STAGES;

struct GemmArgs {
  int64_t M, N, K;
  double alpha, beta;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  int64_t batch;
  const int* klim;  // per-matrix inner-dimension limit (nullable)
  const int* nlim;  // per-matrix output-column limit (nullable)
  int lower;        // 1: only tiles touching the lower triangle (n0 < m0 + BM) are computed
};

template <int BM, int BN, bool TA, bool TB>
struct SmemLayout {
  // Fragments are read for k pairs (2k, 2k+1) per lane.  k-contiguous tiles
  // ([m][k], [n][k]) are read as LDS.128 with a pitch = 8 (mod 16) doubles;
  // m/n-contiguous tiles ([k][m], [k][n]) as two LDS.64 with a pitch
  // = 2 (mod 16): both patterns are bank-conflict-free.
  static constexpr int A_LD = TA ? (BM + 2) : (BK + 8);
  static constexpr int A_ELEMS = TA ? BK * A_LD : BM * A_LD;
  static constexpr int B_LD = TB ? (BK + 8) : (BN + 2);
  static constexpr int B_ELEMS = TB ? BN * B_LD : BK * B_LD;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = (size_t)STAGES * STAGE_ELEMS * sizeof(double);
};

template <int BM, int BN, int WM, int WN, bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(WM* WN * 32, (WM * WN == 8 && BN == 64) ? 2 : 1) gemm_f64_kernel(GemmArgs g) {
  using SL = SmemLayout<BM, BN, TA, TB>;
  constexpr int NT = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int FM = WTM / 8, FN = WTN / 8;
  extern __shared__ __align__(128) double smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / WN) * WTM, wn0 = (warp % WN) * WTN;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  if (g.lower && n0 >= m0 + BM) return;  // tile strictly above the diagonal (symmetric updates)
  // Loader geometry, fixed for the whole kernel: each thread owns A_IT (B_IT)
  // 16-byte chunks of every stage at the same tile position; only the k offset
  // moves, so a stage's addresses are one multiply-add per chunk (ncu: the
  // per-chunk index math of the first version was 40% of the stall samples).
  constexpr int A_ROWS = TA ? BK : BM, A_COLS = TA ? BM : BK;
  constexpr int B_ROWS = TB ? BN : BK, B_COLS = TB ? BK : BN;
  constexpr int A_CH = A_ROWS * A_COLS / VEC, B_CH = B_ROWS * B_COLS / VEC;
  constexpr int A_IT = (A_CH + NT - 1) / NT, B_IT = (B_CH + NT - 1) / NT;
  int64_t a_go[A_IT], b_go[B_IT];  // global element offset at k0 = 0
  int a_so[A_IT], b_so[B_IT];      // shared element offset within a stage
  int a_k[A_IT], b_k[B_IT];        // k index of the chunk at k0 = 0 (-1: outside M / N)
#pragma unroll
  for (int it = 0; it < A_IT; ++it) {
    const int c = tid + it * NT;
    const int r = c / (A_COLS / VEC), cc = (c % (A_COLS / VEC)) * VEC;
    const int64_t gm = m0 + (TA ? cc : r);
    const int kk = TA ? r : cc;
    a_so[it] = r * SL::A_LD + cc;
    a_go[it] = TA ? (int64_t)kk * g.lda + gm : gm * g.lda + kk;
    a_k[it] = (c < A_CH && gm < g.M) ? kk : -1;
  }
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    const int c = tid + it * NT;
    const int r = c / (B_COLS / VEC), cc = (c % (B_COLS / VEC)) * VEC;
    const int64_t gn = n0 + (TB ? r : cc);
    const int kk = TB ? cc : r;
    b_so[it] = r * SL::B_LD + cc;
    b_go[it] = TB ? gn * g.ldb + kk : (int64_t)kk * g.ldb + gn;
    b_k[it] = (c < B_CH && gn < g.N) ? kk : -1;
  }
  const int64_t a_kstep = TA ? (int64_t)BK * g.lda : BK;  // element step per k tile
  const int64_t b_kstep = TB ? BK : (int64_t)BK * g.ldb;

  for (int64_t b = blockIdx.z; b < g.batch; b += gridDim.z) {
    if (g.nlim && n0 >= g.nlim[b]) continue;  // no output column of this tile is wanted
    const int64_t Kb = g.klim ? std::min<int64_t>(g.K, std::max(g.klim[b], 0)) : g.K;
    const int nk = (int)((Kb + BK - 1) / BK);
    const double* __restrict__ A = g.A + b * g.sA;
    const double* __restrict__ B = g.B + b * g.sB;
    double* __restrict__ C = g.C + b * g.sC;

    auto load_stage = [&](int stage, int kt) {
      double* As = smem + stage * SL::STAGE_ELEMS;
      double* Bs = As + SL::A_ELEMS;
      const int k0 = kt * BK;
#pragma unroll
      for (int it = 0; it < A_IT; ++it) {
        if (A_CH % NT != 0 && tid + it * NT >= A_CH) break;
        const bool ok = a_k[it] >= 0 && a_k[it] + k0 < Kb;
        cp_async_zfill<VEC * 8>(As + a_so[it], ok ? A + a_go[it] + kt * a_kstep : A, ok);
      }
#pragma unroll
      for (int it = 0; it < B_IT; ++it) {
        if (B_CH % NT != 0 && tid + it * NT >= B_CH) break;
        const bool ok = b_k[it] >= 0 && b_k[it] + k0 < Kb;
        cp_async_zfill<VEC * 8>(Bs + b_so[it], ok ? B + b_go[it] + kt * b_kstep : B, ok);
      }
    };

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nk) load_stage(s, s);
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) load_stage(nxt % STAGES, nxt);
        cp_async_commit();
      }
      const double* As = smem + (kt % STAGES) * SL::STAGE_ELEMS;
      const double* Bs = As + SL::A_ELEMS;
      // Each lane feeds the k-slot pair (2k, 2k+1), k = lane%4, of an 8-wide
      // k-step into two DMMAs (any fixed k -> slot map is valid as long as
      // the A and B fragments use the same one).
#pragma unroll
      for (int ks = 0; ks < BK; ks += 8) {
        double2 af[FM], bf[FN];
        const int kk = ks + 2 * (lane & 3);
#pragma unroll
        for (int i = 0; i < FM; ++i) {
          const int mm = wm0 + i * 8 + (lane >> 2);
          if (TA) af[i] = make_double2(As[kk * SL::A_LD + mm], As[(kk + 1) * SL::A_LD + mm]);
          else af[i] = *reinterpret_cast<const double2*>(As + mm * SL::A_LD + kk);
        }
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          const int nn = wn0 + j * 8 + (lane >> 2);
          if (TB) bf[j] = *reinterpret_cast<const double2*>(Bs + nn * SL::B_LD + kk);
          else bf[j] = make_double2(Bs[kk * SL::B_LD + nn], Bs[(kk + 1) * SL::B_LD + nn]);
        }
        // all even-k products first, then all odd-k ones: the two DMMAs that
        // accumulate into one tile are FM*FN instructions apart instead of
        // back to back (ncu: the dependent second DMMA was the top stall)
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // stage buffers are reused by the next batch item

    // epilogue: C = alpha*acc + beta*C
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int64_t gm = m0 + wm0 + i * 8 + (lane >> 2);
      if (gm >= g.M) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int64_t gn = n0 + wn0 + j * 8 + 2 * (lane & 3);
        double* cp = C + gm * g.ldc + gn;
        double v0 = g.alpha * acc[i][j][0], v1 = g.alpha * acc[i][j][1];
        if (gn + 1 < g.N && ((reinterpret_cast<uintptr_t>(cp) & 15) == 0)) {
          if (g.beta != 0.0) {
            const double2 o = *reinterpret_cast<const double2*>(cp);
            v0 = fma(g.beta, o.x, v0);
            v1 = fma(g.beta, o.y, v1);
          }
          *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
        } else {
          if (gn < g.N) cp[0] = g.beta != 0.0 ? fma(g.beta, cp[0], v0) : v0;
          if (gn + 1 < g.N) cp[1] = g.beta != 0.0 ? fma(g.beta, cp[1], v1) : v1;
        }
      }
    }
  }
}

__global__ void gemm_scale_kernel(double* C, int64_t M, int64_t N, int64_t ldc, int64_t sC,
                                  double beta) {
  double* Cb = C + (int64_t)blockIdx.y * sC;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * N;
       e += (int64_t)gridDim.x * blockDim.x) {
    double* p = Cb + (e / N) * ldc + e % N;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

template <int BM, int BN, int WM, int WN, bool TA, bool TB, int VEC>
int launch_cfg(const GemmArgs& g, cudaStream_t st) {
  using SL = SmemLayout<BM, BN, TA, TB>;
  auto kern = gemm_f64_kernel<BM, BN, WM, WN, TA, TB, VEC>;
  if (int e = ensure_smem(kern, SL::BYTES)) return e;
  dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM),
            (unsigned)std::min<int64_t>(g.batch, 65535));
  WT_REQUIRE(grid.y <= 65535, "gemm: M too large");
  kern<<<grid, WM * WN * 32, SL::BYTES, st>>>(g);
  return check_launch("wt_gemm_f64");
}

template <bool TA, bool TB, int VEC>
int dispatch_tile(const GemmArgs& g, cudaStream_t st) {
  const int64_t big_tiles = ((g.M + 127) / 128) * ((g.N + 127) / 128) * g.batch;
#ifndef WT_GEMM_BIG
#define WT_GEMM_BIG 1
#endif
#if WT_GEMM_BIG == 1
  // 128 x 64 CTA tiles, two CTAs per SM: one CTA's k-tile barrier overlaps the
  // other's DMMA stream.  4 warps of 64 x 32 warp tiles; up to 256 x 256
  // matrices 8 warps of 32 x 32 (more warps per SM where each matrix is only
  // a few tiles: 256^3 x 192 26.6 -> 28.1 TF/s; -4% at 512^3 and up)
  if (g.M >= 128 && g.N >= 64 && big_tiles >= num_sms()) {
    if (g.M <= 256 && g.N <= 256) return launch_cfg<128, 64, 4, 2, TA, TB, VEC>(g, st);
    return launch_cfg<128, 64, 2, 2, TA, TB, VEC>(g, st);
  }
#elif WT_GEMM_BIG == 4
  // 128 x 64 CTA tiles of 8 warps (32 x 32 warp tiles), two CTAs per SM
  if (g.M >= 128 && g.N >= 64 && big_tiles >= num_sms())
    return launch_cfg<128, 64, 4, 2, TA, TB, VEC>(g, st);
#elif WT_GEMM_BIG == 2
  if (g.M >= 64 && g.N >= 128 && big_tiles >= num_sms())
    return launch_cfg<64, 128, 2, 2, TA, TB, VEC>(g, st);
#elif WT_GEMM_BIG == 0
  if (g.M >= 128 && g.N >= 128 && big_tiles >= num_sms())
    return launch_cfg<128, 128, 2, 4, TA, TB, VEC>(g, st);
#endif
  if (g.M >= 64 && g.N >= 64) return launch_cfg<64, 64, 2, 2, TA, TB, VEC>(g, st);
  return launch_cfg<32, 32, 2, 2, TA, TB, VEC>(g, st);
}

template <bool TA, bool TB>
int dispatch_vec(const GemmArgs& g, cudaStream_t st) {
  // 16-byte cp.async needs every contiguous run to start 16-byte aligned.
  const int64_t a_extent = TA ? g.M : g.K, b_extent = TB ? g.K : g.N;
  bool v2 = (a_extent % 2 == 0) && (b_extent % 2 == 0) && (g.lda % 2 == 0) &&
            (g.ldb % 2 == 0) && (g.sA % 2 == 0 || g.batch == 1) &&
            (g.sB % 2 == 0 || g.batch == 1) && ((uintptr_t)g.A % 16 == 0) &&
            ((uintptr_t)g.B % 16 == 0);
  return v2 ? dispatch_tile<TA, TB, 2>(g, st) : dispatch_tile<TA, TB, 1>(g, st);
}

}  // namespace
}  // namespace wt

using namespace wt;

int wt::gemm_f64_lim(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                     int64_t strideB, double beta, double* C, int64_t ldc, int64_t strideC,
                     int64_t batch, const int* klim, const int* nlim, void* stream, int lower) {
  WT_REQUIRE(M >= 0 && N >= 0 && K >= 0 && batch >= 0, "gemm: negative dimension");
  if (M == 0 || N == 0 || batch == 0) return WT_OK;
  WT_REQUIRE(ldc >= N, "gemm: ldc < N");
  WT_REQUIRE(lda >= (transA ? M : K) || K == 0, "gemm: lda too small");
  WT_REQUIRE(ldb >= (transB ? K : N) || K == 0, "gemm: ldb too small");
  if (K == 0) {  // empty inner dimension: C = beta * C (numpy matmul gives zeros)
    WT_REQUIRE(batch <= 65535, "gemm: batch too large");
    dim3 grid((unsigned)std::min<int64_t>((M * N + 255) / 256, 1024), (unsigned)batch);
    gemm_scale_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(C, M, N, ldc, strideC, beta);
    return check_launch("wt_gemm_f64(K=0)");
  }
  GemmArgs g{M, N, K, alpha, beta, A, lda, strideA, B, ldb, strideB, C, ldc, strideC, batch, klim, nlim,
             lower};
  cudaStream_t st = (cudaStream_t)stream;
  if (!transA && !transB) return dispatch_vec<false, false>(g, st);
  if (!transA && transB) return dispatch_vec<false, true>(g, st);
  if (transA && !transB) return dispatch_vec<true, false>(g, st);
  return dispatch_vec<true, true>(g, st);
}

extern "C" int wt_gemm_f64(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                           const double* A, int64_t lda, int64_t strideA, const double* B,
                           int64_t ldb, int64_t strideB, double beta, double* C, int64_t ldc,
                           int64_t strideC, int64_t batch, void* stream) {
  return gemm_f64_lim(transA, transB, M, N, K, alpha, A, lda, strideA, B, ldb, strideB, beta, C,
                      ldc, strideC, batch, nullptr, nullptr, stream);
}
