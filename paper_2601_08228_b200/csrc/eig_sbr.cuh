// K4 preconditioner, two-stage tridiagonalization (successive band reduction)
// for the wide Grams (n >= 512) of the leading-triplet mode.  Included by eig.cu
// inside namespace wt::eig.
//
// Why: the one-stage reduction (tridiag_panel) runs one symv over the trailing
// block per column -- 46 GB of loads and ~2 us of barriers per column on the 32
// coarse 1024^2 slices of config 4 (22.7 of the 31 ms K4 call, ncu
// profiles/r02_bench_launches.csv).  Two stages read the trailing block three
// times per SB_B columns instead:
//   stage 1  dense -> band of half-width SB_B: per panel a Householder QR of the
//            rows below the band (sbr_panel, one 1024-thread CTA per matrix, a
//            row per thread in registers, one block reduction per column), Z =
//            A22 V on K3, W = Z T - V (T^T V^T Z T) / 2 (sbr_w), and the
//            two-sided update A22 -= V W^T + W V^T on K3.
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
constexpr int SB_LDB = 2 * SB_B - 1;  // band storage: AB[c * SB_LDB + d] = A[c + d][c], d = 0 .. 2 SB_B - 2
constexpr int SB_NT = 1024;          // threads of the stage-1 kernels: one row below the band per thread
constexpr int SB_CW = 16;            // chase warps per CTA
constexpr int SB_QC = 16;            // columns of Z per CTA in sbr_apply_q2
constexpr int SB_QT = 512;           // its threads
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
  if (ss > 0.0) {
    beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
    tau = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
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
__global__ void __launch_bounds__(SB_NT, 1) sbr_panel(double* __restrict__ Gall, double* __restrict__ ABall,
                                                     double* __restrict__ tauall, double* __restrict__ Tpall,
                                                     const int* __restrict__ flag, int n, int c0) {
  constexpr int B = SB_B;
  const int b = blockIdx.x;
  if (!flag[b]) return;
  double* A = Gall + (int64_t)b * n * n;
  double* AB = ABall + (int64_t)b * n * SB_LDB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bw = min(B, n - c0);  // panel width
  const int r0 = c0 + B;
  const int m = max(n - r0, 0);            // rows below the band
  const int jb = max(min(B, m - 1), 0);    // reflectors of this panel
  __shared__ double wp[2][32][16];         // per-warp partial sums (double-buffered by column parity)
  __shared__ double gsm[2][16];            // block sums
  __shared__ double pivrow[2][16];         // the pivot row's entries
  __shared__ double vdot[B][B];            // V[:, k]^T v_c, k < c
  __shared__ double Ts[B][B + 1];
  __shared__ double taus[B];

  // diagonal block -> band (lower part)
  if (tid < bw) {
    const double* ar = A + (int64_t)(c0 + tid) * n + c0;
    for (int k = 0; k <= tid; ++k) AB[(int64_t)(c0 + k) * SB_LDB + (tid - k)] = ar[k];
  }
  if (m <= 0) return;
  const bool have = tid < m;
  double row[B];
  {
    const double* ar = A + (int64_t)(r0 + tid) * n + c0;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      double2 x = make_double2(0.0, 0.0);
      if (have) x = *reinterpret_cast<const double2*>(ar + k);  // (n, c0 even: 16-byte aligned)
      row[k] = x.x;
      row[k + 1] = x.y;
    }
  }
  for (int c = 0; c < jb; ++c) {
    const int pb = c & 1;
    // x = my row's entry of column c (rows below the pivot row c only)
    double x = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k == c) x = row[k];
    const double xt = (have && tid > c) ? x : 0.0;
    int idx;
    const double sum = warp_sum16([&](int i) { return i < B ? xt * row[i < B ? i : 0] : 0.0; }, lane, idx);
    if ((lane & 1) == 0) wp[pb][warp][idx] = sum;
    if (tid == c) {
#pragma unroll
      for (int k = 0; k < B; ++k) pivrow[pb][k] = row[k];
    }
    __syncthreads();
    if (tid < 16) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int w = 0; w < 32; w += 4) {
        s0 += wp[pb][w][tid];
        s1 += wp[pb][w + 1][tid];
        s2 += wp[pb][w + 2][tid];
        s3 += wp[pb][w + 3][tid];
      }
      gsm[pb][tid] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    double alpha = 0.0, ss = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k == c) {
        alpha = pivrow[pb][k];
        ss = gsm[pb][k];
      }
    double beta, tau, scale;
    house_gen(alpha, ss, beta, tau, scale);
    if (tid == 0) {
      taus[c] = tau;
      for (int k = 0; k < c; ++k) vdot[k][c] = fma(scale, gsm[pb][k], pivrow[pb][k]);
    }
    if (have && tid >= c) {
      const double vi = tid == c ? 1.0 : x * scale;
#pragma unroll
      for (int k = 0; k < B; ++k) {
        if (k > c) {
          const double s = fma(scale, gsm[pb][k], pivrow[pb][k]);  // v^T P[:, k]
          row[k] = fma(-tau * s, vi, row[k]);
        } else if (k == c) {
          row[k] = tid == c ? beta : vi;
        }
      }
    }
  }
  __syncthreads();
  // compact-WY factor: T_cc = tau_c, T[0:c, c] = -tau_c T[0:c, 0:c] vdot[0:c, c]
  if (warp == 0) {
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
    double* Tp = Tpall + (int64_t)b * B * B;
    for (int k = lane; k < B * B; k += 32) Tp[k] = Ts[k / B][k % B];
    if (lane < B) tauall[(int64_t)b * n + c0 + lane] = lane < jb ? taus[lane] : 0.0;
  }
  // R -> band: row i = tid, column k >= i: distance B + i - k
  if (have && tid < B) {
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k >= tid) AB[(int64_t)(c0 + k) * SB_LDB + (B + tid - k)] = row[k];
  }
  // explicit reflectors over the panel columns (columns >= jb: zeros)
  if (have) {
    double* ar = A + (int64_t)(r0 + tid) * n + c0;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      double2 o;
      o.x = (k < jb && tid >= k) ? (tid == k ? 1.0 : row[k]) : 0.0;
      o.y = (k + 1 < jb && tid >= k + 1) ? (tid == k + 1 ? 1.0 : row[k + 1]) : 0.0;
      *reinterpret_cast<double2*>(ar + k) = o;
    }
  }
}

// W = Z T - V (T^T (V^T Z) T) / 2 for the panel at c0 (rows r0 = c0 + SB_B ..), Z = A22 V
// (m x SB_B, pitch SB_B) from K3; writes the rows of VW = [V | W] and WV = [W | V]
// (pitch 2 SB_B, row index = global row) for the rank-2 SB_B update on K3.
__global__ void __launch_bounds__(SB_NT, 1) sbr_w(const double* __restrict__ Gall, const double* __restrict__ Zall,
                                                 const double* __restrict__ Tpall, double* __restrict__ VWall,
                                                 double* __restrict__ WVall, const int* __restrict__ flag, int n,
                                                 int c0) {
  constexpr int B = SB_B;
  const int b = blockIdx.x;
  if (!flag[b]) return;
  const double* A = Gall + (int64_t)b * n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = c0 + B;
  const int m = n - r0;
  const bool have = tid < m;
  constexpr int HB = B / 2;
  __shared__ double wp[32][HB][16];  // per-warp partials of N = V^T Z (half of V's columns at a time)
  __shared__ double Ns[B][B], Ts[B][B], NT[B][B], Ss[B][B];
  for (int k = tid; k < B * B; k += SB_NT) (&Ts[0][0])[k] = Tpall[(int64_t)b * B * B + k];
  // (V is re-read from the panel columns where needed: z, v and w rows together
  // do not fit 64 registers)
  const double* vr = A + (int64_t)(r0 + (have ? tid : 0)) * n + c0;
  double z[B];
  {
    const double* zr = Zall + ((int64_t)b * n + r0 + tid) * B;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      double2 x = make_double2(0.0, 0.0);
      if (have) x = *reinterpret_cast<const double2*>(zr + k);
      z[k] = x.x;
      z[k + 1] = x.y;
    }
  }
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
#pragma unroll
    for (int kh = 0; kh < HB; ++kh) {
      int idx;
      const double vk = have ? vr[half * HB + kh] : 0.0;
      const double sum = warp_sum16([&](int i) { return i < B ? vk * z[i < B ? i : 0] : 0.0; }, lane, idx);
      if ((lane & 1) == 0) wp[warp][kh][idx] = sum;
    }
    __syncthreads();
    if (tid < HB * B) {
      const int kh = tid / B, l = tid % B;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int w = 0; w < 32; w += 4) {
        s0 += wp[w][kh][l];
        s1 += wp[w + 1][kh][l];
        s2 += wp[w + 2][kh][l];
        s3 += wp[w + 3][kh][l];
      }
      Ns[half * HB + kh][l] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
  }
  if (tid < B * B) {  // NT = N T
    const int k = tid / B, l = tid % B;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j) s = fma(Ns[k][j], Ts[j][l], s);
    NT[k][l] = s;
  }
  __syncthreads();
  if (tid < B * B) {  // S = T^T (N T), halved
    const int k = tid / B, l = tid % B;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j) s = fma(Ts[j][k], NT[j][l], s);
    Ss[k][l] = 0.5 * s;
  }
  __syncthreads();
  if (have) {
    double* vw = VWall + ((int64_t)b * n + r0 + tid) * 2 * B;
    double* wv = WVall + ((int64_t)b * n + r0 + tid) * 2 * B;
#pragma unroll 1
    for (int l0 = 0; l0 < B; l0 += 2) {
      double w0 = 0.0, w1 = 0.0, u0 = 0.0, u1 = 0.0;
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const double vk = vr[k];
        w0 = fma(z[k], Ts[k][l0], w0);
        w1 = fma(z[k], Ts[k][l0 + 1], w1);
        u0 = fma(vk, Ss[k][l0], u0);
        u1 = fma(vk, Ss[k][l0 + 1], u1);
      }
      const double2 ww = make_double2(w0 - u0, w1 - u1);
      const double2 vv = *reinterpret_cast<const double2*>(vr + l0);
      *reinterpret_cast<double2*>(vw + l0) = vv;
      *reinterpret_cast<double2*>(vw + B + l0) = ww;
      *reinterpret_cast<double2*>(wv + l0) = ww;
      *reinterpret_cast<double2*>(wv + B + l0) = vv;
    }
  }
}

// ---------------------------------------------------------------- stage 2 ---
struct ChaseSmem {
  static size_t bytes(int n) {
    return sizeof(double) * ((size_t)n * SB_LDB + 2 * SB_CW * 16) + sizeof(int) * (size_t)(n + 4);
  }
};

// Band -> tridiagonal.  One CTA per matrix, band in shared memory.  Warp w runs
// the sweeps s = w, w + SB_CW, ...: sweep s annihilates column s below its
// subdiagonal with a reflector on rows s+1 .. s+B and chases the first column of
// every bulge down the band (hop h works on rows r0 = s + 1 + h B ..).  Sweep s
// may run hop h once sweep s - 1 has completed hop h + 1 (tools/sbr_proto.py
// checks the rule under random interleavings).  The reflectors (tau in the unit
// entry's place) go to the dead upper triangle of G: VQ[s][row] = G[s * n + row].
__global__ void __launch_bounds__(SB_CW * 32, 1) sbr_chase(const double* __restrict__ ABall, double* __restrict__ Gall,
                                                          double* __restrict__ dall, double* __restrict__ eall,
                                                          const int* __restrict__ flag, int n) {
  constexpr int B = SB_B, LDB = SB_LDB;
  constexpr int DONE = 0x7fffffff;
  const int b = blockIdx.x;
  if (!flag[b]) return;
  extern __shared__ __align__(16) double csm[];
  double* AB = csm;                          // [n][LDB]
  double* vsh = AB + (size_t)n * LDB;        // [SB_CW][16] current reflector
  double* wsh = vsh + SB_CW * 16;            // [SB_CW][16] w / next reflector
  volatile int* prog = reinterpret_cast<volatile int*>(wsh + SB_CW * 16);  // [n] hops completed by sweep s
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const double* src = ABall + (int64_t)b * n * LDB;
    for (int i = tid; i < n * LDB; i += SB_CW * 32) AB[i] = src[i];
    for (int i = tid; i < n; i += SB_CW * 32) prog[i] = 0;
  }
  __syncthreads();
  double* VQ = Gall + (int64_t)b * n * n;
  double* vs = vsh + warp * 16;
  double* ws = wsh + warp * 16;
  auto lane_sum = [&](double x) {  // over the 16-lane halves (lanes >= 16 carry zeros)
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  for (int s = warp; s < n - 2; s += SB_CW) {
    int L = min(B, n - 1 - s);
    int h = 0;
    auto wait_prev = [&](int need) {
      if (s > 0) {
        while (prog[s - 1] < need) {
        }
        __threadfence_block();
      }
    };
    wait_prev(2);
    // first reflector: column s, rows s+1 .. s+L
    double x = (lane < L) ? AB[(size_t)s * LDB + 1 + lane] : 0.0;
    double alpha = __shfl_sync(0xffffffffu, x, 0);
    double ss = lane_sum((lane >= 1 && lane < L) ? x * x : 0.0);
    ss = __shfl_sync(0xffffffffu, ss, 0);
    double beta, tau, scale;
    house_gen(alpha, ss, beta, tau, scale);
    double vi = lane == 0 ? 1.0 : (lane < L ? x * scale : 0.0);
    if (lane == 0) AB[(size_t)s * LDB + 1] = beta;
    int r0 = s + 1;
    while (true) {
      // store the reflector (tau in the unit entry's place)
      if (lane < L) VQ[(int64_t)s * n + r0 + lane] = lane == 0 ? tau : vi;
      if (lane < 16) vs[lane] = vi;
      __syncwarp();
      // ---- D <- H D H on the symmetric L x L block at r0 (lower band storage)
      {
        double drow[B];
        double p = 0.0;
#pragma unroll
        for (int k = 0; k < B; ++k) {
          double a = 0.0;
          if (lane < L && k < L)
            a = k <= lane ? AB[(size_t)(r0 + k) * LDB + (lane - k)] : AB[(size_t)(r0 + lane) * LDB + (k - lane)];
          drow[k] = a;
          p = fma(a, vs[k], p);
        }
        p *= tau;
        double pv = lane_sum(lane < L ? p * vi : 0.0);
        pv = __shfl_sync(0xffffffffu, pv, 0);
        const double wi = fma(-0.5 * tau * pv, vi, p);
        if (lane < 16) ws[lane] = lane < L ? wi : 0.0;
        __syncwarp();  // every lane has read its row of D; w is visible
        if (lane < L) {
#pragma unroll
          for (int k = 0; k < B; ++k)
            if (k <= lane) AB[(size_t)(r0 + k) * LDB + (lane - k)] = drow[k] - vi * ws[k] - wi * vs[k];
        }
      }
      const int R0 = r0 + L;
      const int M = min(B, n - R0);
      if (L < B || M < 1) break;
      // ---- B block: rows R0 .. R0 + M - 1, columns r0 .. r0 + B - 1 (distance B + i - k)
      double tau2 = 0.0, v2 = 0.0;
      {
        double brow[B];
        double xb = 0.0;
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int dist = B + lane - k;
          double a = 0.0;
          if (lane < M && dist <= 2 * B - 2) a = AB[(size_t)(r0 + k) * LDB + dist];
          brow[k] = a;
          xb = fma(a, vs[k], xb);
        }
        xb *= tau;
#pragma unroll
        for (int k = 0; k < B; ++k) brow[k] = fma(-xb, vs[k], brow[k]);  // B (I - tau v v^T)
        if (M >= 2) {
          const double a0 = __shfl_sync(0xffffffffu, brow[0], 0);
          double ss2 = lane_sum((lane >= 1 && lane < M) ? brow[0] * brow[0] : 0.0);
          ss2 = __shfl_sync(0xffffffffu, ss2, 0);
          double beta2, scale2;
          house_gen(a0, ss2, beta2, tau2, scale2);
          v2 = lane == 0 ? 1.0 : (lane < M ? brow[0] * scale2 : 0.0);
          brow[0] = lane == 0 ? beta2 : 0.0;
        }
        __syncwarp();  // (ws reuse: every lane is past the D update)
        if (lane < 16) ws[lane] = v2;
        if (lane < M) {
#pragma unroll
          for (int k = 0; k < B; ++k) {
            const int dist = B + lane - k;
            if (dist <= 2 * B - 2) AB[(size_t)(r0 + k) * LDB + dist] = brow[k];
          }
        }
        __syncwarp();
        if (M >= 2 && lane >= 1 && lane < B) {  // (I - tau2 v2 v2^T) B[:, k], k = lane
          double* col = AB + (size_t)(r0 + lane) * LDB + (B - lane);  // rows i = 0 .. M-1 contiguous
          double cv[B];
          double y = 0.0;
#pragma unroll
          for (int i = 0; i < B; ++i) {
            cv[i] = i < M ? col[i] : 0.0;
            y = fma(ws[i], cv[i], y);
          }
          y *= tau2;
#pragma unroll
          for (int i = 0; i < B; ++i)
            if (i < M) col[i] = fma(-y, ws[i], cv[i]);
        }
      }
      __syncwarp();
      __threadfence_block();
      ++h;
      if (lane == 0) prog[s] = h;
      if (M < 2) break;
      r0 = R0;
      L = M;
      tau = tau2;
      vi = v2;
      wait_prev(h + 2);
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) prog[s] = DONE;
  }
  __syncthreads();
  double* d = dall + (int64_t)b * n;
  double* e = eall + (int64_t)b * n;
  for (int i = tid; i < n; i += SB_CW * 32) {
    d[i] = AB[(size_t)i * LDB];
    if (i < n - 1) e[i] = AB[(size_t)i * LDB + 1];
  }
}

// Z <- Q2 Z for SB_QC columns of Z per CTA (blockIdx.x = column group, blockIdx.y
// = matrix): the sweeps' reflectors in reverse generation order (sweep n-3 first);
// the hops of one sweep act on disjoint rows, one warp per hop, lane = (column,
// row half).  The next sweep's reflector row is staged in shared memory while the
// current one is applied.
struct Q2Smem {
  static size_t bytes(int n) { return sizeof(double) * ((size_t)n * (SB_QC + 1) + 2 * (size_t)(n + 2)); }
};
__global__ void __launch_bounds__(SB_QT, 1) sbr_apply_q2(const double* __restrict__ Gall, double* __restrict__ Zall,
                                                        const int* __restrict__ flag, int n, int kk) {
  constexpr int B = SB_B, HB = SB_B / 2, LDZ = SB_QC + 1;
  const int b = blockIdx.y;
  if (!flag[b]) return;
  extern __shared__ __align__(16) double qsm[];
  double* Zs = qsm;                       // [n][LDZ]
  double* vbuf = Zs + (size_t)n * LDZ;    // [2][n + 2]
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
  for (int i = slast + 1 + tid; i < n; i += SB_QT) vbuf[(slast & 1) * (n + 2) + i] = VQ[(int64_t)slast * n + i];
  __syncthreads();
  const int cc = lane & 15, rh = lane >> 4;
  for (int s = slast; s >= 0; --s) {
    const double* vb = vbuf + (s & 1) * (n + 2);
    if (s > 0) {  // stage the next sweep's reflectors
      double* nb = vbuf + ((s - 1) & 1) * (n + 2);
      for (int i = s + tid; i < n; i += SB_QT) nb[i] = VQ[(int64_t)(s - 1) * n + i];
    }
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
    __syncthreads();
  }
  for (int e = tid; e < n * SB_QC; e += SB_QT) {
    const int r = e / SB_QC, c = e % SB_QC;
    if (c < ncol) Z[(int64_t)r * kk + col0 + c] = Zs[r * LDZ + c];
  }
}
