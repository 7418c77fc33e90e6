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
#include <cuda.h>
#include <cudaTypedefs.h>

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


// ------------------------------------------------------------- TMA variant ---
// The same CTA / warp tiling fed by tensor-map boxes (cp.async.bulk.tensor, SASS
// UTMALDG) through a full / empty mbarrier ring instead of the cp.async ring and
// its CTA barrier per k tile: one elected thread issues the boxes of a stage, the
// four warps release a stage with one mbarrier arrive each.  Operands are 3-D
// tensors (inner extent, outer extent, batch) with the 128-byte swizzle:
//   k-contiguous operand ([m][k] / [n][k]):  one box {16 k, BM} per stage; a
//     fragment pair (k, k+1) is one LDS.128 at 16-byte unit ((k/2) ^ (row & 7));
//   m/n-contiguous operand ([k][m] / [k][n]): BM/16 boxes {16 m, 16 k}; a fragment
//     pair is two LDS.64 (rows k, k+1 of the box).
// Rows / columns / k beyond the matrices are zero-filled by the TMA unit, so edge
// tiles and K tails need no predicates.  Used for the large-tile case without
// per-matrix limits; everything else stays on the cp.async kernel.
constexpr int TSTAGES = 4;
struct TmaArgs {
  CUtensorMap a, b;
};

__device__ __forceinline__ void tma_box_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int BM, int BN, int WM, int WN, bool TA, bool TB>
__global__ void __launch_bounds__(WM* WN * 32, 2) gemm_f64_tma_kernel(GemmArgs g, const __grid_constant__ TmaArgs tm) {
  constexpr int NT = WM * WN * 32, NWARP = WM * WN;
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int FM = WTM / 8, FN = WTN / 8;
  constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8, STAGE_BYTES = A_BYTES + B_BYTES;
  static_assert(BK == 16 && A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzled boxes: 16 doubles per row");
  extern __shared__ __align__(1024) unsigned char tsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + TSTAGES * STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / WN) * WTM, wn0 = (warp % WN) * WTN;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (g.lower && n0 >= m0 + BM) return;
  const int b = blockIdx.z;
  const int nk = (int)((g.K + BK - 1) / BK);
  if ((smem_u32(tsm) & 1023u) != 0) __trap();
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int kt) {  // thread 0
    const int s = kt % TSTAGES, k0 = kt * BK;
    unsigned char* As = tsm + s * STAGE_BYTES;
    unsigned char* Bs = As + A_BYTES;
    mbar_expect_tx(full + s, STAGE_BYTES);
    if (!TA) tma_box_3d(As, &tm.a, k0, m0, b, full + s);
    else
      for (int c = 0; c < BM / 16; ++c) tma_box_3d(As + c * 2048, &tm.a, m0 + 16 * c, k0, b, full + s);
    if (TB) tma_box_3d(Bs, &tm.b, k0, n0, b, full + s);
    else
      for (int c = 0; c < BN / 16; ++c) tma_box_3d(Bs + c * 2048, &tm.b, n0 + 16 * c, k0, b, full + s);
  };
  if (tid == 0)
    for (int kt = 0; kt < TSTAGES - 1 && kt < nk; ++kt) issue(kt);

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int g8 = lane >> 2, q = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TSTAGES;
    // refill the stage released one iteration ago (its consumers are mostly through)
    if (tid == 0) {
      const int nxt = kt + TSTAGES - 1;
      if (nxt < nk) {
        if (nxt >= TSTAGES) mbar_wait(empty + nxt % TSTAGES, (uint32_t)(((nxt / TSTAGES) - 1) & 1));
        issue(nxt);
      }
    }
    __syncwarp();
    mbar_wait(full + s, (uint32_t)((kt / TSTAGES) & 1));
    const unsigned char* As = tsm + s * STAGE_BYTES;
    const unsigned char* Bs = As + A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 8) {
      double2 af[FM], bf[FN];
      const int kk = ks + 2 * q;
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int mm = wm0 + i * 8 + g8;
        if (!TA) {
          af[i] = *reinterpret_cast<const double2*>(As + mm * 128 + (((kk >> 1) ^ (mm & 7)) << 4));
        } else {  // box (mm / 16): rows k, 16-byte unit ((mm % 16) / 2) ^ (k & 7)
          const unsigned char* bx = As + (mm >> 4) * 2048 + (mm & 1) * 8;
          const int u = (mm & 15) >> 1;
          af[i].x = *reinterpret_cast<const double*>(bx + kk * 128 + ((u ^ (kk & 7)) << 4));
          af[i].y = *reinterpret_cast<const double*>(bx + (kk + 1) * 128 + ((u ^ ((kk + 1) & 7)) << 4));
        }
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int nn = wn0 + j * 8 + g8;
        if (TB) {
          bf[j] = *reinterpret_cast<const double2*>(Bs + nn * 128 + (((kk >> 1) ^ (nn & 7)) << 4));
        } else {
          const unsigned char* bx = Bs + (nn >> 4) * 2048 + (nn & 1) * 8;
          const int u = (nn & 15) >> 1;
          bf[j].x = *reinterpret_cast<const double*>(bx + kk * 128 + ((u ^ (kk & 7)) << 4));
          bf[j].y = *reinterpret_cast<const double*>(bx + (kk + 1) * 128 + ((u ^ ((kk + 1) & 7)) << 4));
        }
      }
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }
  double* __restrict__ C = g.C + (int64_t)b * g.sC;
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int64_t gm = m0 + wm0 + i * 8 + g8;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int64_t gn = n0 + wn0 + j * 8 + 2 * q;
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

PFN_cuTensorMapEncodeTiled_v12000 gemm_encode_fn() {
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

// operand stored as [outer][inner] rows of pitch ld (elements), matrices sX apart
bool operand_map(CUtensorMap* map, const double* P, int64_t inner, int64_t outer, int64_t ld, int64_t sX, int64_t batch,
                 int box_inner, int box_outer) {
  auto enc = gemm_encode_fn();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(P) & 15) || (ld & 1) || (batch > 1 && (sX & 1))) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(double), (cuuint64_t)(batch > 1 ? sX : ld * outer) * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(P), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// returns WT_OK when launched, -1 when the TMA variant does not apply (caller falls back)
template <bool TA, bool TB, int WM, int WN>
int launch_tma(const GemmArgs& g, cudaStream_t st) {
  constexpr int BM = 128, BN = 64;
  if (g.klim || g.nlim || g.batch > 65535 || option(WT_OPT_GEMM_TMA) == 0) return -1;
  TmaArgs tm;
  const bool okA = TA ? operand_map(&tm.a, g.A, g.M, g.K, g.lda, g.sA, g.batch, 16, 16)
                      : operand_map(&tm.a, g.A, g.K, g.M, g.lda, g.sA, g.batch, 16, BM);
  const bool okB = TB ? operand_map(&tm.b, g.B, g.K, g.N, g.ldb, g.sB, g.batch, 16, BN)
                      : operand_map(&tm.b, g.B, g.N, g.K, g.ldb, g.sB, g.batch, 16, 16);
  if (!okA || !okB) return -1;
  auto kern = gemm_f64_tma_kernel<BM, BN, WM, WN, TA, TB>;
  constexpr size_t smem = (size_t)TSTAGES * (BM + BN) * BK * 8 + 2 * TSTAGES * 8;
  if (int e = ensure_smem(kern, smem)) return e;
  dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM), (unsigned)g.batch);
  if (grid.y > 65535) return -1;
  kern<<<grid, WM * WN * 32, smem, st>>>(g, tm);
  return check_launch("wt_gemm_f64 (tma)");
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
    const bool small = g.M <= 256 && g.N <= 256;  // (8 warps of 32 x 32 there, see above)
    if (VEC == 2 && g.K >= 64) {  // tensor-map fed variant where it applies
      const int r = small ? launch_tma<TA, TB, 4, 2>(g, st) : launch_tma<TA, TB, 2, 2>(g, st);
      if (r >= 0) return r;
    }
    if (small) return launch_cfg<128, 64, 4, 2, TA, TB, VEC>(g, st);
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
