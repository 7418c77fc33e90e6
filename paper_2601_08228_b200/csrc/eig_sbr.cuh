// K4 preconditioner, two-stage tridiagonalization (successive band reduction)
// for the wide Grams (n >= 512) of the leading-triplet mode.  Included by eig.cu
// inside namespace wt::eig.
//
// Why: the one-stage reduction (tridiag_panel) runs one symv over the trailing
// block per column -- 46 GB of loads and ~2 us of barriers per column on the 32
// coarse 1024^2 slices of config 4 (22.7 of the 31 ms K4 call, ncu
// round-2 launch lists).  Two stages read and write the trailing block once per
// SB_B columns instead:
//   stage 1  dense -> band of half-width SB_B: per panel a Householder QR of the
//            rows below the band (sbr_panel, a 4-CTA cluster per matrix, a row per
//            thread in registers, one cluster reduction per column; it first forms
//            the previous panel's W = Z T - V (T^T V^T Z T) / 2 and applies that
//            panel's update to its own columns), and one fused pass over the
//            trailing block (sbr_update_mult: the previous panel's two-sided update
//            A22 -= V W^T + W V^T and Z = A22 V for this panel).
//   stage 2  band -> tridiagonal by column-wise bulge chasing (Lang 1993) with
//            the band (2 SB_B - 1 diagonals) in shared memory, one CTA per matrix,
//            one warp per sweep, sweeps pipelined two hops apart through
//            shared-memory progress counters (sbr_chase).
// The back-transformation applies the stage-2 reflectors to the eigenvectors of
// T (sbr_apply_q2: column groups of Z in shared memory, one warp per hop) and
// then the stage-1 reflectors as compact-WY blocks on K3 (eig.cu, step 6).
// tools/sbr_proto.py is the numpy statement of the same index conventions.
// Deterministic: fixed lane/thread -> data maps and reduction trees; the sweep
// pipeline only reorders operations on disjoint data.
#pragma once

constexpr int SB_B = 12;             // band half-width (2 SB_B - 1 diagonals x 1024 columns fit one CTA's shared memory)
constexpr int SB_LDB = 2 * SB_B;      // band storage: AB[c * SB_LDB + d] = A[c + d][c], d = 0 .. 2 SB_B - 1 (the last one a
                                      // scratch slot of the chase: always zero between hops)
constexpr int SB_NT = 1024;          // threads of the stage-1 kernels: one row below the band per thread
#ifndef WT_SB_CW
#define WT_SB_CW 32
#endif
constexpr int SB_CW = WT_SB_CW;            // chase warps per CTA
constexpr int SB_QC = 16;            // columns of Z per CTA in sbr_apply_q2
constexpr int SB_QT = 512;           // its threads
constexpr int SB_QD = 6;             // reflector-row buffers: rows travel SB_QD - 1 sweeps ahead
static_assert(SB_B <= 16 && SB_B % 2 == 0, "lane maps below assume an even band width of at most 16");

// Sum of 16 per-lane values over the 32 lanes of a warp in 16 shuffles: after the
// call, the lanes with (lane & 1) == 0 hold the total of value index
// idx = 8 * bit4 + 4 * bit3 + 2 * bit2 + bit1 of their lane number.
// f(i) yields the lane's value i (evaluated once).
template <typename F>
__device__ __forceinline__ double warp_sum16(F f, int lane, int& idx) {
  double v8[8];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double lo_v = f(i), hi_v = f(i + 8);
      const double send = hi ? lo_v : hi_v, keep = hi ? hi_v : lo_v;
      v8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  double v4[4];
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double send = hi ? v8[i] : v8[i + 4], keep = hi ? v8[i + 4] : v8[i];
      v4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  double v2[2];
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double send = hi ? v4[i] : v4[i + 2], keep = hi ? v4[i + 2] : v4[i];
      v2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
  double v1;
  {
    const bool hi = lane & 2;
    const double send = hi ? v2[0] : v2[1], keep = hi ? v2[1] : v2[0];
    v1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
  idx = ((lane & 16) ? 8 : 0) + ((lane & 8) ? 4 : 0) + ((lane & 4) ? 2 : 0) + ((lane & 2) ? 1 : 0);
  return v1;
}

// dlarfg on (alpha, ss = sum of squares of the tail): H x = beta e1, H = I - tau v v^T,
// v = [1; tail * scale]
__device__ __forceinline__ void house_gen(double alpha, double ss, double& beta, double& tau, double& scale) {
  // one rsqrt and one reciprocal on the dependent chain (the chase pays this
  // latency once per hop).  Columns whose norm is below 1e-140 of the scaled
  // Gram's unit magnitude are left alone (tau = 0): the neglected entries are far
  // below rounding of the band.
  const double nrm2 = fma(alpha, alpha, ss);
  if (ss > 0.0 && nrm2 > 1e-280) {
    const double nrm = nrm2 * rsqrt(nrm2);
    beta = -copysign(nrm, alpha);
    const double amb = alpha - beta;           // |amb| >= |beta|: no cancellation
    const double r = 1.0 / (beta * amb);
    tau = -amb * (r * amb);                    // (beta - alpha) / beta
    scale = r * beta;                          // 1 / (alpha - beta)
  } else {
    beta = alpha;
    tau = 0.0;
    scale = 0.0;
  }
}

// upper triangle <- lower triangle (the Gram comes from K3's lower-tiles mode; the
// panel QR and Z = A22 V read full rows).  grid (n/32, n/32, batch), block (32, 8).
__global__ void sym_mirror(double* __restrict__ Gall, int n, const int* __restrict__ flag) {
  const int b = blockIdx.z;
  if (!flag[b] || blockIdx.x < blockIdx.y) return;  // tiles (ty, tx) with tx >= ty
  __shared__ double tile[32][33];
  double* A = Gall + (int64_t)b * n * n;
  const int tx = blockIdx.x * 32, ty = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {  // lower tile (tx.., ty..)
    const int r = tx + i, c = ty + threadIdx.x;
    tile[i][threadIdx.x] = (r < n && c < n) ? A[(int64_t)r * n + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = ty + i, c = tx + threadIdx.x;
    if (r < n && c < n && c > r) A[(int64_t)r * n + c] = tile[threadIdx.x][i];
  }
}

// Before the stage-1 back-transformation: zero everything above the reflectors'
// unit entries (row < col + SB_B: the dead band and the consumed stage-2
// reflectors), so the panel columns are the explicit Y blocks.
__global__ void sbr_clean_y(double* __restrict__ Gall, int n, const int* __restrict__ flag) {
  const int b = blockIdx.y;
  if (!flag[b]) return;
  double* A = Gall + (int64_t)b * n * n;
  const int64_t nn = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e - r * n;
    if (r < c + SB_B) A[e] = 0.0;
  }
}

// Fused trailing pass of panel j (r0 = c0 + SB_B, m = n - r0 rows): one read and one
// write of A22 = A[r0:, r0:] do both
//   A22 -= VW WV^T          (the previous panel's two-sided update; upd = 0 for panel 0)
//   Z    = A22 V            (V = this panel's reflectors, rows of the compact copy Vc)
// One CTA per 64-row strip of A22 walks the strip's 64 x 64 tiles through a FU_ST-stage
// ring: a tile arrives as four 16-column boxes of a 3-D tensor map over G
// (cp.async.bulk.tensor, 128-byte swizzle: the accumulator-layout accesses below are
// bank-conflict-free; rows / columns beyond the matrix are zero-filled on load and
// clipped on store), the WV and V rows of its columns as two bulk copies.  The
// rank-24 product runs on the DMMA pipe; the updated 8 x 8 blocks, still in the
// accumulator layout (row g, columns 2q, 2q+1), are exactly the A-fragment pairs of
// the k-steps of block x V, so Z's partial needs no shared round trip.  Each warp
// owns 32 rows x 16 tile columns; the four column-owner warps of a row group are
// summed in a fixed order at the end (deterministic).  Ten bulk operations per tile
// (one per row, 193 per tile, held the first version at 3.2 us per tile).
// grid (ceil(m / 64), batch), 256 threads.
#ifndef WT_FU_ST
#define WT_FU_ST 4
#endif
#ifndef WT_FU_PD
#define WT_FU_PD 3
#endif
#ifndef WT_FU_OCC
#define WT_FU_OCC 1
#endif
constexpr int FU_T = 64, FU_K = 2 * SB_B, FU_NT = 256, FU_ST = WT_FU_ST, FU_PD = WT_FU_PD;  // ring stages, prefetch distance
static_assert(FU_PD >= 1 && FU_PD < FU_ST, "prefetch distance");
constexpr int FU_CB = FU_T * FU_T * 8;                              // tile bytes (4 boxes of 64 x 16)
constexpr int FU_STAGE_B = FU_CB + FU_T * FU_K * 8 + FU_T * SB_B * 8;  // 51200: a multiple of 1024
constexpr size_t FU_SMEM = (size_t)FU_ST * FU_STAGE_B + FU_T * FU_K * 8 + 8 * FU_ST;  // (FU_ST = 2, two CTAs per SM: 13.9 vs 13.3 ms)
static_assert(FU_STAGE_B % 1024 == 0, "swizzled boxes need 1024-byte aligned stages");

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}

__global__ void __launch_bounds__(FU_NT, WT_FU_OCC) sbr_update_mult(const __grid_constant__ CUtensorMap gmap,
                                                           const double* __restrict__ VWall,
                                                           const double* __restrict__ WVall,
                                                           const double* __restrict__ Vcall, double* __restrict__ Zall,
                                                           double* __restrict__ Npall,
                                                           const int* __restrict__ flag, int n, int c0, int upd) {
  constexpr int B = SB_B;
  const int b = blockIdx.y;
  if (!flag[b]) return;
  extern __shared__ __align__(1024) unsigned char fsm[];
  if ((smem_u32(fsm) & 1023u) != 0) __trap();  // swizzled boxes need 1024-byte aligned stages (no static shared memory here)
  double* VWs = reinterpret_cast<double*>(fsm + FU_ST * FU_STAGE_B);  // [FU_T][FU_K] the strip's rows of VW
  uint64_t* bars = reinterpret_cast<uint64_t*>(VWs + FU_T * FU_K);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = c0 + B, m = n - r0;
  const int i0 = blockIdx.x * FU_T;
  const int hrows = min(FU_T, m - i0);
  const int ntiles = (m + FU_T - 1) / FU_T;
  const double* VWb = VWall + ((int64_t)b * n + r0) * FU_K;
  const double* WVb = WVall + ((int64_t)b * n + r0) * FU_K;
  const double* Vcb = Vcall + ((int64_t)b * n + r0) * B;
  // no stale NaN bit patterns in the ring: leftovers of partial tiles meet zero blocks
  for (int e = tid; e < (FU_ST * FU_STAGE_B + FU_T * FU_K * 8) / 8; e += FU_NT) reinterpret_cast<double*>(fsm)[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < FU_ST; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();  // the generic-proxy zero fill precedes the bulk copies into the same bytes
  __syncthreads();
  // tile t -> stage t % FU_ST (thread 0 only)
  auto issue = [&](int t) {
    const int s = t % FU_ST, j0 = t * FU_T, wc = min(FU_T, m - j0);
    const int nbox = (wc + 15) / 16;
    unsigned char* st = fsm + s * FU_STAGE_B;
    uint32_t bytes = (uint32_t)(nbox * FU_T * 16 * 8 + wc * B * 8 + (upd ? wc * FU_K * 8 : 0));
    if (t == 0 && upd) bytes += (uint32_t)(hrows * FU_K * 8);
    mbar_expect_tx(bars + s, bytes);
    for (int c = 0; c < nbox; ++c) tma_load_3d(st + c * (FU_T * 16 * 8), &gmap, r0 + j0 + 16 * c, r0 + i0, b, bars + s);
    bulk_g2s(st + FU_CB + FU_T * FU_K * 8, Vcb + (int64_t)j0 * B, (uint32_t)(wc * B * 8), bars + s);
    if (upd) {
      bulk_g2s(st + FU_CB, WVb + (int64_t)j0 * FU_K, (uint32_t)(wc * FU_K * 8), bars + s);
      if (t == 0) bulk_g2s(VWs, VWb + (int64_t)i0 * FU_K, (uint32_t)(hrows * FU_K * 8), bars + s);
    }
  };
  if (tid == 0) {
    for (int t = 0; t < FU_PD && t < ntiles; ++t) issue(t);
  }
  const int g = lane >> 2, q = lane & 3;
  const int um0 = (warp >> 2) * 32, own = warp & 3;  // warp tile: rows um0 .. um0+31, tile columns 16 own .. 16 own + 15
  double zacc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) zacc[i][j][0] = zacc[i][j][1] = 0.0;
  for (int t = 0; t < ntiles; ++t) {
    const int s = t % FU_ST, j0 = t * FU_T, wc = min(FU_T, m - j0);
    unsigned char* st = fsm + s * FU_STAGE_B;
    unsigned char* Cb = st + own * (FU_T * 16 * 8);  // my 16-column box: [64 rows][128 B], 16-byte units XOR (row & 7)
    const double* WVs = reinterpret_cast<const double*>(st + FU_CB);
    const double* Vs = reinterpret_cast<const double*>(st + FU_CB + FU_T * FU_K * 8);  // [64][B]
    mbar_wait(bars + s, (uint32_t)((t / FU_ST) & 1));
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (upd) {
#pragma unroll
      for (int ks = 0; ks < FU_K; ks += 8) {
        double2 af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = *reinterpret_cast<const double2*>(VWs + (um0 + 8 * i + g) * FU_K + ks + 2 * q);
#pragma unroll
        for (int j = 0; j < 2; ++j)
          bf[j] = *reinterpret_cast<const double2*>(WVs + (16 * own + 8 * j + g) * FU_K + ks + 2 * q);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
      }
    }
    // updated blocks -> acc (zero-filled beyond the matrix by the loads), and back to the tile
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = um0 + 8 * i + g;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double2* p = reinterpret_cast<double2*>(Cb + r * 128 + (((4 * j + q) ^ g) << 4));
        double2 o = *p;
        o.x -= acc[i][j][0];
        o.y -= acc[i][j][1];
        if (upd) *p = o;
        const bool in = r < hrows && 16 * own + 8 * j + 2 * q < wc;  // (stale rows of VW / WV beyond the matrix)
        acc[i][j][0] = in ? o.x : 0.0;
        acc[i][j][1] = in ? o.y : 0.0;
      }
    }
    // Z[my rows] += updated blocks x V[my tile columns]
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double bx[2], by[2];
#pragma unroll
      for (int nf = 0; nf < 2; ++nf) {
        const int col = 8 * nf + g;  // (V has B = 12 columns: the fragment's columns 12..15 are zeros)
        bx[nf] = col < B ? Vs[(16 * own + 8 * j + 2 * q) * B + col] : 0.0;
        by[nf] = col < B ? Vs[(16 * own + 8 * j + 2 * q + 1) * B + col] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nf = 0; nf < 2; ++nf) dmma884(zacc[i][nf][0], zacc[i][nf][1], acc[i][j][0], bx[nf]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int nf = 0; nf < 2; ++nf) dmma884(zacc[i][nf][0], zacc[i][nf][1], acc[i][j][1], by[nf]);
    }
    if (upd) fence_proxy_async_smem();
    __syncthreads();  // the updated tile is complete; every warp is past tile t - 1's stage
    if (tid == 0) {
      if (upd) {
        const int nbox = (wc + 15) / 16;
        for (int c = 0; c < nbox; ++c) tma_store_3d(&gmap, r0 + j0 + 16 * c, r0 + i0, b, st + c * (FU_T * 16 * 8));
        bulk_commit();
      }
      // refill: tile t + FU_PD goes to the stage of tile t + FU_PD - FU_ST, whose stores
      // (FU_ST - FU_PD groups back) must have read their shared bytes
      if (t + FU_PD < ntiles) {
        if (upd) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(FU_ST - FU_PD) : "memory");
        issue(t + FU_PD);
      }
    }
  }
  // Z strip = sum over the four column-owner warps of a row group (fixed order), through the ring
  if (tid == 0 && upd) bulk_wait_all();
  __syncthreads();
  {
    double* zp = reinterpret_cast<double*>(fsm);  // [4][FU_T][16]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int nf = 0; nf < 2; ++nf)
        *reinterpret_cast<double2*>(zp + (own * FU_T + um0 + 8 * i + g) * 16 + 8 * nf + 2 * q) =
            make_double2(zacc[i][nf][0], zacc[i][nf][1]);
    __syncthreads();
    double* zs = zp + 4 * FU_T * 16;   // [FU_T][B] the summed strip
    double* vs = zs + FU_T * B;        // [FU_T][B] the strip's rows of V
    for (int e = tid; e < FU_T * (B / 2); e += FU_NT) {
      const int r = e / (B / 2), c = (e % (B / 2)) * 2;
      double2 sum = make_double2(0.0, 0.0), vv = make_double2(0.0, 0.0);
      if (r < hrows) {
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const double2 v = *reinterpret_cast<const double2*>(zp + (o * FU_T + r) * 16 + c);
          sum.x += v.x;
          sum.y += v.y;
        }
        *reinterpret_cast<double2*>(Zall + ((int64_t)b * n + r0 + i0 + r) * B + c) = sum;
        vv = *reinterpret_cast<const double2*>(Vcb + (int64_t)(i0 + r) * B + c);
      }
      *reinterpret_cast<double2*>(zs + r * B + c) = sum;
      *reinterpret_cast<double2*>(vs + r * B + c) = vv;
    }
    __syncthreads();
    // the strip's share of N = V^T Z (SB_B x SB_B; the next panel kernel sums the strips in order)
    if (tid < B * B) {
      const int k = tid / B, l = tid % B;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 4
      for (int r = 0; r < FU_T; r += 4) {
        s0 = fma(vs[r * B + k], zs[r * B + l], s0);
        s1 = fma(vs[(r + 1) * B + k], zs[(r + 1) * B + l], s1);
        s2 = fma(vs[(r + 2) * B + k], zs[(r + 2) * B + l], s2);
        s3 = fma(vs[(r + 3) * B + k], zs[(r + 3) * B + l], s3);
      }
      Npall[((int64_t)b * gridDim.x + blockIdx.x) * B * B + tid] = (s0 + s1) + (s2 + s3);
    }
  }
}

// ---------------------------------------------------------------- stage 1 ---
// Panel c0 (columns c0 .. c0 + SB_B - 1) of matrix b = blockIdx.x, A = G[b] full
// symmetric n x n (the panel's rows c0.. are current).
//   * the panel's diagonal block (rows c0 .. c0 + SB_B - 1) goes to the band AB;
//   * the rows below it (r0 = c0 + SB_B .. n - 1, thread t = row r0 + t) are QR
//     factorised: reflector c (global column c0 + c) has its unit entry at row
//     r0 + c; R goes to the band, the reflectors overwrite the panel columns of A
//     explicitly (zeros above the unit entry, 1 on it: the Y block of the
//     back-transformation and the B operand of Z = A22 V), tau to tau[c0 + c],
//     the compact-WY factor T (upper triangular, SB_B x SB_B) to Tp[b].
//   * pend = 1: the previous panel's two-sided update (A -= VW WV^T, rows >= c0) has
//     not reached this panel's columns yet (sbr_update_mult applies it to the block
//     right of them only): every thread applies it to its row on load.
constexpr int SB_PC = 4;               // CTAs of the panel kernel's cluster (rows dealt in contiguous quarters)
constexpr int SB_PT = SB_NT / SB_PC;   // its threads per CTA: one row below the band per thread
constexpr int SB_PW = SB_PT / 32;
__global__ void __launch_bounds__(SB_PT, 1) sbr_panel(double* __restrict__ Gall, double* __restrict__ ABall,
                                                     double* __restrict__ tauall, double* __restrict__ Tpall,
                                                     const int* __restrict__ flag, int n, int c0,
                                                     double* __restrict__ VWall, double* __restrict__ WVall, int pend,
                                                     double* __restrict__ Vcall, const double* __restrict__ Zall,
                                                     const double* __restrict__ Npall, int nstrips) {
  constexpr int B = SB_B;
  const int b = blockIdx.x / SB_PC;
  if (!flag[b]) return;  // cluster-uniform
  const int rank = cl_rank();
  double* A = Gall + (int64_t)b * n * n;
  double* AB = ABall + (int64_t)b * n * SB_LDB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gt = rank * SB_PT + tid;  // my row below the band: r0 + gt
  const int bw = min(B, n - c0);  // panel width
  const int r0 = c0 + B;
  const int m = max(n - r0, 0);            // rows below the band
  const int jb = max(min(B, m - 1), 0);    // reflectors of this panel
  __shared__ double wp[2][SB_PW][16];      // per-warp partial sums (double-buffered by column parity)
  __shared__ double gpart[2][16];          // this CTA's share of the column sums (read by the whole cluster)
  __shared__ double pivrow[2][16];         // the pivot row's entries (rank 0; read by the whole cluster)
  __shared__ double vdot[B][B];            // V[:, k]^T v_c, k < c
  __shared__ double Ts[B][B + 1];
  __shared__ double taus[B];
  __shared__ double coef[2][16];  // tau * v^T P[:, k] of the current column (k > c)
  __shared__ double hs[2][2];     // scale, beta

  __shared__ __align__(16) double wvs[B][2 * B];  // [W | V] rows of the panel's columns (pending update)
  __shared__ __align__(16) double Ns[B][B], Tq[B][B], NT[B][B], Ss[B][B];
  // ---- previous panel (columns c0 - B ..): W = Z T - V (T^T N T) / 2 from the trailing pass's Z and the
  //      per-strip shares of N = V^T Z; its rows are the rows r0p = c0 .. of this panel.  Every CTA forms S.
  if (pend) {
    if (tid < B * B) {
      Tq[tid / B][tid % B] = Tpall[((int64_t)b * ((n + B - 1) / B) + c0 / B - 1) * B * B + tid];
      double sN = 0.0;
      for (int q = 0; q < nstrips; ++q) sN += Npall[((int64_t)b * nstrips + q) * B * B + tid];
      Ns[tid / B][tid % B] = sN;
    }
    __syncthreads();
    if (tid < B * B) {  // NT = N T
      const int k = tid / B, l = tid % B;
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < B; ++j) a = fma(Ns[k][j], Tq[j][l], a);
      NT[k][l] = a;
    }
    __syncthreads();
    if (tid < B * B) {  // S = T^T (N T), halved
      const int k = tid / B, l = tid % B;
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < B; ++j) a = fma(Tq[j][k], NT[j][l], a);
      Ss[k][l] = 0.5 * a;
    }
    __syncthreads();
  }
  // [V | W] of the previous panel for global row grow (>= c0): vw[0:B] = V row, vw[B:2B] = W row
  auto prev_vw = [&](int grow, double* vw) {
    const double* zr = Zall + ((int64_t)b * n + grow) * B;
    const double* vr = Vcall + ((int64_t)b * n + grow) * B;
    double z[B];
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      const double2 x = *reinterpret_cast<const double2*>(zr + k), y = *reinterpret_cast<const double2*>(vr + k);
      z[k] = x.x;
      z[k + 1] = x.y;
      vw[k] = y.x;
      vw[k + 1] = y.y;
    }
#pragma unroll
    for (int l0 = 0; l0 < B; l0 += 4) {
      double w[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const double2 t01 = *reinterpret_cast<const double2*>(&Tq[k][l0]);
        const double2 t23 = *reinterpret_cast<const double2*>(&Tq[k][l0 + 2]);
        const double2 s01 = *reinterpret_cast<const double2*>(&Ss[k][l0]);
        const double2 s23 = *reinterpret_cast<const double2*>(&Ss[k][l0 + 2]);
        w[0] = fma(z[k], t01.x, fma(-vw[k], s01.x, w[0]));
        w[1] = fma(z[k], t01.y, fma(-vw[k], s01.y, w[1]));
        w[2] = fma(z[k], t23.x, fma(-vw[k], s23.x, w[2]));
        w[3] = fma(z[k], t23.y, fma(-vw[k], s23.y, w[3]));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) vw[B + l0 + u] = w[u];
    }
  };
  auto store_vw = [&](int grow, const double* vw) {  // rows of [V | W] and [W | V] for the trailing pass
    double* pv = VWall + ((int64_t)b * n + grow) * 2 * B;
    double* pw = WVall + ((int64_t)b * n + grow) * 2 * B;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      const double2 vv = make_double2(vw[k], vw[k + 1]), ww = make_double2(vw[B + k], vw[B + k + 1]);
      *reinterpret_cast<double2*>(pv + k) = vv;
      *reinterpret_cast<double2*>(pv + B + k) = ww;
      *reinterpret_cast<double2*>(pw + k) = ww;
      *reinterpret_cast<double2*>(pw + B + k) = vv;
    }
  };
  if (pend) {
    // the [W | V] rows of this panel's columns (global rows c0 .. c0 + bw - 1): every CTA needs them
    if (tid < bw) {
      double vw[2 * B];
      prev_vw(c0 + tid, vw);
#pragma unroll
      for (int k = 0; k < B; ++k) {
        wvs[tid][k] = vw[B + k];
        wvs[tid][B + k] = vw[k];
      }
      if (rank == SB_PC - 1) store_vw(c0 + tid, vw);
    }
    __syncthreads();
  }
  // my row's panel entries minus the pending update  sum_t [V | W][row][t] [W | V][c0 + k][t]
  auto load_row = [&](int grow, double* row, bool store) {
    const double* ar = A + (int64_t)grow * n + c0;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      const double2 x = *reinterpret_cast<const double2*>(ar + k);  // (n, c0 even: 16-byte aligned)
      row[k] = x.x;
      row[k + 1] = x.y;
    }
    if (pend) {
      double vw[2 * B];
      prev_vw(grow, vw);
      if (store) store_vw(grow, vw);
#pragma unroll
      for (int t = 0; t < 2 * B; t += 2) {
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const double2 w2 = *reinterpret_cast<const double2*>(&wvs[k][t]);
          row[k] = fma(-vw[t], w2.x, fma(-vw[t + 1], w2.y, row[k]));
        }
      }
    }
  };
  // diagonal block -> band (lower part); the last CTA has the fewest QR rows to load
  if (rank == SB_PC - 1 && tid < bw) {
    double drow[B];
    load_row(c0 + tid, drow, false);
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k <= tid) AB[(int64_t)(c0 + k) * SB_LDB + (tid - k)] = drow[k];
  }
  if (m <= 0) return;  // cluster-uniform
  const bool have = gt < m;
  double row[B];
#pragma unroll
  for (int k = 0; k < B; ++k) row[k] = 0.0;
  if (have) load_row(r0 + gt, row, true);
#pragma unroll
  for (int c = 0; c < B; ++c) {  // (unrolled: static register indices)
    if (c < jb) {
      const int pb = c & 1;
      // x = my row's entry of column c (rows below the pivot row c only)
      const double x = row[c];
      const double xt = (have && gt > c) ? x : 0.0;
      int idx;
      const double sum = warp_sum16([&](int i) { return i < B ? xt * row[i < B ? i : 0] : 0.0; }, lane, idx);
      if ((lane & 1) == 0) wp[pb][warp][idx] = sum;
      if (gt == c) {  // (rank 0)
#pragma unroll
        for (int k = 0; k < B; ++k) pivrow[pb][k] = row[k];
      }
      __syncthreads();
      if (tid < 16) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int w = 0; w < SB_PW; w += 2) {
          s0 += wp[pb][w][tid];
          s1 += wp[pb][w + 1][tid];
        }
        gpart[pb][tid] = s0 + s1;
      }
      cl_sync();  // every CTA's share and the pivot row are visible
      if (warp == 0) {  // cluster sums, reflector and update coefficients (every CTA, identically)
        double gk = 0.0, pk = 0.0;
        if (lane < 16) {
#pragma unroll
          for (int r = 0; r < SB_PC; ++r) gk += cl_map(&gpart[pb][lane], r)[0];
          pk = cl_map(&pivrow[pb][lane], 0)[0];
        }
        const double ss = __shfl_sync(0xffffffffu, gk, c);
        const double alpha = __shfl_sync(0xffffffffu, pk, c);
        double beta, tau, scale;
        house_gen(alpha, ss, beta, tau, scale);
        if (lane < B) {
          const double sk = fma(scale, gk, pk);  // v^T P[:, k] (k > c), V[:, k]^T v (k < c)
          coef[pb][lane] = tau * sk;
          if (lane < c) vdot[lane][c] = sk;
        }
        if (lane == 0) {
          hs[pb][0] = scale;
          hs[pb][1] = beta;
          taus[c] = tau;
        }
      }
      __syncthreads();
      if (have && gt >= c) {
        const double vi = gt == c ? 1.0 : x * hs[pb][0];
#pragma unroll
        for (int k = c + 1; k < B; ++k) row[k] = fma(-coef[pb][k], vi, row[k]);
        row[c] = gt == c ? hs[pb][1] : vi;
      }
    }
  }
  __syncthreads();
  // compact-WY factor: T_cc = tau_c, T[0:c, c] = -tau_c T[0:c, 0:c] vdot[0:c, c]
  if (rank == 0 && warp == 0) {
    for (int k = lane; k < B * (B + 1); k += 32) (&Ts[0][0])[k] = 0.0;
    __syncwarp();
    for (int c = 0; c < jb; ++c) {
      double acc = 0.0;
      if (lane < c)
        for (int j = lane; j < c; ++j) acc = fma(Ts[lane][j], vdot[j][c], acc);
      __syncwarp();
      if (lane < c) Ts[lane][c] = -taus[c] * acc;
      if (lane == c) Ts[c][c] = taus[c];
      __syncwarp();
    }
    double* Tp = Tpall + ((int64_t)b * ((n + B - 1) / B) + c0 / B) * B * B;  // [matrix][panel][B][B]
    for (int k = lane; k < B * B; k += 32) Tp[k] = Ts[k / B][k % B];
    if (lane < B) tauall[(int64_t)b * n + c0 + lane] = lane < jb ? taus[lane] : 0.0;
  }
  // R -> band: row i = gt, column k >= i: distance B + i - k
  if (have && gt < B) {
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k >= gt) AB[(int64_t)(c0 + k) * SB_LDB + (B + gt - k)] = row[k];
  }
  // explicit reflectors over the panel columns (columns >= jb: zeros)
  if (have) {
    double* ar = A + (int64_t)(r0 + gt) * n + c0;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      double2 o;
      o.x = (k < jb && gt >= k) ? (gt == k ? 1.0 : row[k]) : 0.0;
      o.y = (k + 1 < jb && gt >= k + 1) ? (gt == k + 1 ? 1.0 : row[k + 1]) : 0.0;
      *reinterpret_cast<double2*>(ar + k) = o;
      *reinterpret_cast<double2*>(Vcall + ((int64_t)b * n + r0 + gt) * B + k) = o;  // compact copy: bulk-copied tile rows
    }
  }
  cl_sync();  // no CTA exits while the others may still read its shared memory
}

// Compact-WY factor of a back-transformation block of up to SB_TB = 10 SB_B stage-1
// reflectors (whole panels, k0 a multiple of SB_TB) from the panels' own factors T_j
// and S = Y^T Y of the block (K3):  T[0:c, c:c+B] = -T[0:c, 0:c] S[0:c, c:c+B] T_j,
// nine merges of dense blocks instead of dlarft's 120 dependent columns (wy_larft:
// ~1 us per column).  One CTA per matrix; T in shared memory, written as NBT x NBT.
constexpr int SB_TB = 10 * SB_B;
__global__ void __launch_bounds__(512, 1) sbr_larft_merge(const double* __restrict__ Sall, const double* __restrict__ Tpall,
                                                         const int* __restrict__ flag, int n, int k0, int nb,
                                                         double* __restrict__ Tall) {
  constexpr int B = SB_B, LD = NBT + 1;
  const int b = blockIdx.x;
  if (!flag[b]) return;
  extern __shared__ double T[];       // [NBT][LD]
  __shared__ double X[SB_TB][B + 1];  // S[0:c, c:c+B] T_j
  __shared__ double Tj[B][B + 1];
  const double* S = Sall + (int64_t)b * NBT * NBT;
  const double* Tp = Tpall + ((int64_t)b * ((n + B - 1) / B) + k0 / B) * B * B;
  const int tid = threadIdx.x;
  for (int e = tid; e < NBT * LD; e += 512) T[e] = 0.0;
  __syncthreads();
  const int np = (nb + B - 1) / B;
  for (int j = 0; j < np; ++j) {
    const int c = j * B;
    if (tid < B * B) Tj[tid / B][tid % B] = Tp[(int64_t)j * B * B + tid];
    __syncthreads();
    if (tid < B * B && c + tid / B < NBT && c + tid % B < NBT) T[(c + tid / B) * LD + c + tid % B] = Tj[tid / B][tid % B];
    for (int e = tid; e < c * B; e += 512) {  // X = S[0:c, c:c+B] T_j
      const int r = e / B, l = e % B;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < B; ++k) acc = fma(c + k < nb ? S[(int64_t)r * NBT + c + k] : 0.0, Tj[k][l], acc);
      X[r][l] = acc;
    }
    __syncthreads();
    for (int e = tid; e < c * B; e += 512) {  // T[0:c, c:c+B] = -T[0:c, 0:c] X (T upper triangular)
      const int r = e / B, l = e % B;
      double a0 = 0.0, a1 = 0.0;
      int k = r;
      for (; k + 1 < c; k += 2) {
        a0 = fma(T[r * LD + k], X[k][l], a0);
        a1 = fma(T[r * LD + k + 1], X[k + 1][l], a1);
      }
      if (k < c) a0 = fma(T[r * LD + k], X[k][l], a0);
      T[r * LD + c + l] = -(a0 + a1);
    }
    __syncthreads();
  }
  double* Tg = Tall + (int64_t)b * NBT * NBT;
  for (int e = tid; e < NBT * NBT; e += 512) {
    const int rr = e / NBT, cc = e % NBT;
    Tg[e] = (cc >= rr && cc < nb) ? T[rr * LD + cc] : 0.0;
  }
}

// ---------------------------------------------------------------- stage 2 ---
struct ChaseSmem {
  static size_t bytes(int n) {
    return sizeof(double) * ((size_t)(n + 2 * SB_B) * SB_LDB + 2 * SB_CW * 16) + sizeof(int) * (size_t)(2 * n + 8);
  }
};

// Band -> tridiagonal.  One CTA per matrix, band in shared memory (2 SB_B zero
// columns appended, so every hop works on full SB_B x SB_B blocks without bounds
// checks: reflector components of rows beyond the matrix come out as zeros).
// Warp w runs the sweeps s = w, w + SB_CW, ...: sweep s annihilates column s below
// its subdiagonal with a reflector on rows s+1 .. s+B and chases the first column
// of every bulge down the band (hop h works on rows r0 = s + 1 + h B ..).  Sweep s
// may run hop h once sweep s - 1 has completed hop h + 1 (tools/sbr_proto.py
// checks the rule under random interleavings), so the kernel's time is 2 (n - 2)
// hop latencies whatever the number of warps: the hop is written for latency
// (lane = (row or column, half of the block's other index): 6-term chains,
// straight-line addressing).  The reflectors (tau in the unit entry's place) go
// to the dead upper triangle of G: VQ[s][row] = G[s * n + row].
__global__ void __launch_bounds__(SB_CW * 32, 1) sbr_chase(const double* __restrict__ ABall, double* __restrict__ Gall,
                                                          double* __restrict__ dall, double* __restrict__ eall,
                                                          const int* __restrict__ flag, int n) {
  constexpr int B = SB_B, HB = SB_B / 2, LDB = SB_LDB, LD1 = SB_LDB - 1;
  constexpr int DONE = 0x7fffffff;
  const int b = blockIdx.x;
  if (!flag[b]) return;
  extern __shared__ __align__(16) double csm[];
  double* AB = csm;                               // [n + 2B][LDB]
  double* vsh = AB + (size_t)(n + 2 * B) * LDB;   // [SB_CW][16] current reflector
  double* wsh = vsh + SB_CW * 16;                 // [SB_CW][16] w / next reflector
  // per sweep: diagonal-block updates completed (progD) and block right-applies + new reflectors completed (progA)
  volatile int* progD = reinterpret_cast<volatile int*>(wsh + SB_CW * 16);
  volatile int* progA = progD + n + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const double* src = ABall + (int64_t)b * n * LDB;
    for (int i = tid; i < n * LDB; i += SB_CW * 32) AB[i] = src[i];
    for (int i = n * LDB + tid; i < (n + 2 * B) * LDB; i += SB_CW * 32) AB[i] = 0.0;
    for (int i = tid; i < n; i += SB_CW * 32) {
      progD[i] = 0;
      progA[i] = 0;
    }
  }
  __syncthreads();
  double* VQ = Gall + (int64_t)b * n * n;
  double* vs = vsh + warp * 16;
  double* ws = wsh + warp * 16;
  const int i = lane & 15, hf = lane >> 4;  // block row (or column) and half of the other index
  const bool act = i < B;
  const int ic = act ? i : 0;
  const int kh = hf * HB;
  auto half_sum = [&](double x) {  // sum over the 16 lanes of a half, valid in every lane of it
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  for (int s = warp; s < n - 2; s += SB_CW) {
    int h = 0;
    // Sweep s's hop h works, in this order, on D(h) (two-sided update of its diagonal block), A(h) (right-
    // apply on the block below + the next reflector) and the left-apply on that block.  Against sweep s - 1
    // (blocks one row / column up): D(h) overlaps its D(h), its block h after the left-apply, and the corner
    // of its D(h + 1); A(h) overlaps in addition the first entry of its block h + 1 (the new beta).  So D(h)
    // waits for D(h + 1) of the previous sweep and A(h) for its A(h + 1): ~1.35 hops of lag instead of 2
    // (tools/sbr_proto.py checks the coarser rule; this one is checked by the bit-identical repetitions and
    // the one-stage comparison of tests/test_gpu_twostage.py).
    auto wait_on = [&](volatile int* prog, int need) {
      if (s > 0) {
#ifndef SBR_SLEEP
#define SBR_SLEEP 20
#endif
        while (prog[s - 1] < need) __nanosleep(SBR_SLEEP);
        __threadfence_block();
      }
    };
    auto publish = [&](volatile int* prog, int value) {
      __syncwarp();
      __threadfence_block();
      if (lane == 0) prog[s] = value;
    };
    wait_on(progA, 1);  // column s is final once the previous sweep's first block has its new reflector
    // first reflector: column s, rows s+1 .. s+B (zeros beyond the matrix)
    double tau, vi;
    {
      const double x = (act && hf == 0) ? AB[(size_t)s * LDB + 1 + ic] : 0.0;
      const double alpha = __shfl_sync(0xffffffffu, x, 0);
      const double ss = __shfl_sync(0xffffffffu, half_sum(i >= 1 ? x * x : 0.0), 0);
      double beta, scale;
      house_gen(alpha, ss, beta, tau, scale);
      vi = i == 0 ? 1.0 : x * scale;
      vi = __shfl_sync(0xffffffffu, vi, i);
      if (lane == 0) AB[(size_t)s * LDB + 1] = beta;
    }
    int r0 = s + 1;
    while (true) {
      const int L = min(B, n - r0);
      if (hf == 0 && i < L) VQ[(int64_t)s * n + r0 + i] = i == 0 ? tau : vi;
      if (lane < 16) vs[lane] = vi;
      __syncwarp();
      wait_on(progD, h + 2);
      // ---- D <- H D H on the symmetric block at r0: lane = (row i, columns kh .. kh + HB - 1)
      {
        double* lo = AB + (size_t)r0 * LDB + ic + kh * LD1;        // (i, k), k <= i:  + kk * LD1
        double* up = AB + (size_t)(r0 + ic) * LDB - ic + kh;       // (k, i), k > i:   + kk
        double dv[HB];
        double p = 0.0;
#pragma unroll
        for (int kk = 0; kk < HB; ++kk) {
          const double* q = (kh + kk <= ic) ? lo + kk * LD1 : up + kk;
          dv[kk] = *q;
          p = fma(dv[kk], vs[kh + kk], p);
        }
        p += __shfl_xor_sync(0xffffffffu, p, 16);
        p = act ? p * tau : 0.0;
        const double pv = __shfl_sync(0xffffffffu, half_sum(hf == 0 ? p * vi : 0.0), 0);
        const double wi = fma(-0.5 * tau * pv, vi, p);
        if (lane < 16) ws[lane] = wi;
        __syncwarp();  // every lane has read its part of D; w is visible
#pragma unroll
        for (int kk = 0; kk < HB; ++kk)
          if (act && kh + kk <= i) lo[kk * LD1] = dv[kk] - vi * ws[kh + kk] - wi * vs[kh + kk];
      }
      publish(progD, h + 1);
      const int R0 = r0 + B;
      const int M = min(B, n - R0);
      if (L < B || M < 1) break;
      wait_on(progA, h + 2);
      // ---- B block: rows R0 + i, columns r0 + k at distance B + i - k: right-apply, new reflector
      double tau2, v2;
      {
        double* bp = AB + (size_t)r0 * LDB + B + ic + kh * LD1;    // + kk * LD1
        double bv[HB];
        double xb = 0.0;
#pragma unroll
        for (int kk = 0; kk < HB; ++kk) {
          bv[kk] = bp[kk * LD1];
          xb = fma(bv[kk], vs[kh + kk], xb);
        }
        xb += __shfl_xor_sync(0xffffffffu, xb, 16);
        xb *= tau;
#pragma unroll
        for (int kk = 0; kk < HB; ++kk) bv[kk] = fma(-xb, vs[kh + kk], bv[kk]);  // B (I - tau v v^T)
        const double c0 = (hf == 0 && act) ? bv[0] : 0.0;  // first column of the block
        const double a0 = __shfl_sync(0xffffffffu, c0, 0);
        const double ss2 = __shfl_sync(0xffffffffu, half_sum(i >= 1 ? c0 * c0 : 0.0), 0);
        double beta2, scale2;
        house_gen(a0, ss2, beta2, tau2, scale2);
        v2 = i == 0 ? 1.0 : c0 * scale2;
        v2 = __shfl_sync(0xffffffffu, v2, i);
        if (hf == 0) bv[0] = i == 0 ? beta2 : 0.0;
        __syncwarp();  // (ws reuse: every lane is past the D update)
        if (lane < 16) ws[lane] = v2;
        if (act) {
#pragma unroll
          for (int kk = 0; kk < HB; ++kk) bp[kk * LD1] = bv[kk];
        }
        publish(progA, h + 1);  // (its __syncwarp orders the block's stores before the column reads below)
      }
      // ---- (I - tau2 v2 v2^T) B[:, k]: lane = (column k = i >= 1, rows kh .. kh + HB - 1)
      if (tau2 != 0.0) {
        double* cp = AB + (size_t)(r0 + ic) * LDB + B - ic + kh;
        double cv[HB];
        double y = 0.0;
#pragma unroll
        for (int rr = 0; rr < HB; ++rr) {
          cv[rr] = cp[rr];
          y = fma(ws[kh + rr], cv[rr], y);
        }
        y += __shfl_xor_sync(0xffffffffu, y, 16);
        y *= tau2;
        if (act && i >= 1) {
#pragma unroll
          for (int rr = 0; rr < HB; ++rr) cp[rr] = fma(-y, ws[kh + rr], cv[rr]);
        }
      }
      ++h;
      if (M < 2) break;
      r0 = R0;
      tau = tau2;
      vi = v2;
    }
    publish(progD, DONE);
    if (lane == 0) progA[s] = DONE;
  }
  __syncthreads();
  double* d = dall + (int64_t)b * n;
  double* e = eall + (int64_t)b * n;
  for (int i2 = tid; i2 < n; i2 += SB_CW * 32) {
    d[i2] = AB[(size_t)i2 * LDB];
    if (i2 < n - 1) e[i2] = AB[(size_t)i2 * LDB + 1];
  }
}

// Z <- Q2 Z for SB_QC columns of Z per CTA (blockIdx.x = column group, blockIdx.y
// = matrix): the sweeps' reflectors in reverse generation order (sweep n-3 first);
// the hops of one sweep act on disjoint rows, one warp per hop, lane = (column,
// row half).  The next sweep's reflector row is staged in shared memory while the
// current one is applied.
struct Q2Smem {
  static size_t bytes(int n) { return sizeof(double) * ((size_t)n * (SB_QC + 1) + SB_QD * (size_t)(n + 2)); }
};
__global__ void __launch_bounds__(SB_QT, 2) sbr_apply_q2(const double* __restrict__ Gall, double* __restrict__ Zall,
                                                        const int* __restrict__ flag, int n, int kk) {
  constexpr int B = SB_B, HB = SB_B / 2, LDZ = SB_QC + 1;
  const int b = blockIdx.y;
  if (!flag[b]) return;
  extern __shared__ __align__(16) double qsm[];
  double* Zs = qsm;                       // [n][LDZ]
  double* vbuf = Zs + (size_t)n * LDZ;    // [SB_QD][n + 2]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWQ = SB_QT / 32;
  const int col0 = blockIdx.x * SB_QC;
  const int ncol = min(SB_QC, kk - col0);
  double* Z = Zall + (int64_t)b * n * kk;
  const double* VQ = Gall + (int64_t)b * n * n;
  for (int e = tid; e < n * SB_QC; e += SB_QT) {
    const int r = e / SB_QC, c = e % SB_QC;
    Zs[r * LDZ + c] = c < ncol ? Z[(int64_t)r * kk + col0 + c] : 0.0;
  }
  const int slast = n - 3;
  if (slast < 0) return;
  // the reflector rows of the next SB_QD - 1 sweeps travel by cp.async while the current one is applied
  auto fetch = [&](int sw) {
    if (sw >= 0) {
      double* nb = vbuf + (sw % SB_QD) * (n + 2);
      for (int i = sw + 1 + tid; i < n; i += SB_QT) cp_async_zfill<8>(nb + i, VQ + (int64_t)sw * n + i, true);
    }
    cp_async_commit();
  };
  for (int d = 0; d < SB_QD - 1; ++d) fetch(slast - d);
  cp_async_wait<SB_QD - 2>();
  __syncthreads();
  const int cc = lane & 15, rh = lane >> 4;
  for (int s = slast; s >= 0; --s) {
    const double* vb = vbuf + (s % SB_QD) * (n + 2);
    fetch(s - (SB_QD - 1));
    for (int r0 = s + 1 + warp * B; r0 < n; r0 += NWQ * B) {
      const int L = min(B, n - r0);
      if (L < 2) break;
      const double tau = vb[r0];
      double vv[HB], zz[HB];
      double y = 0.0;
#pragma unroll
      for (int i = 0; i < HB; ++i) {
        const int r = rh * HB + i;
        vv[i] = r == 0 ? 1.0 : (r < L ? vb[r0 + r] : 0.0);
        zz[i] = r < L ? Zs[(r0 + r) * LDZ + cc] : 0.0;
        y = fma(vv[i], zz[i], y);
      }
      y += __shfl_xor_sync(0xffffffffu, y, 16);
      y *= tau;
#pragma unroll
      for (int i = 0; i < HB; ++i) {
        const int r = rh * HB + i;
        if (r < L) Zs[(r0 + r) * LDZ + cc] = fma(-y, vv[i], zz[i]);
      }
    }
    cp_async_wait<SB_QD - 2>();  // sweep s - 1's row has landed (only the newest SB_QD - 2 groups may be pending)
    __syncthreads();
  }
  for (int e = tid; e < n * SB_QC; e += SB_QT) {
    const int r = e / SB_QC, c = e % SB_QC;
    if (c < ncol) Z[(int64_t)r * kk + col0 + c] = Zs[r * LDZ + c];
  }
}
