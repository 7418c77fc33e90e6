// K4 implementation, included by svd.cu once per column-block width
// (SVD_NS, SVD_HB): see svd.cu for the algorithm.
namespace wt {
namespace SVD_NS {

constexpr int HB = SVD_HB;   // column block width (16 or 32)
constexpr int BW = 2 * HB;   // pair panel width
constexpr int kThreads = WT_SVD_THREADS;
constexpr int kWarps = kThreads / 32;
// rows per streamed chunk: 8 per warp in the 32-column Gram; the 64-column
// Gram splits 32-row chunks over warp pairs
constexpr int RCH = HB == 16 ? 8 * kWarps : 32;
constexpr int LDZ = RCH + 8; // chunk column pitch (doubles), = 8 mod 16: conflict-free LDS.128 Gram frags
constexpr int LDG = BW + 1;  // Gram / Q pitch
static_assert(kWarps == 4 || kWarps == 8, "K4 CTA shape: 4 or 8 warps");
constexpr double kFloorEps = 1e3 * 2.220446049250313e-16;  // null-column floor (see the test)
constexpr int kMaxInnerSweeps = 16;
constexpr int kSkipMaxBlocks = 128;  // pair-skip records: nblk^2 per matrix (<= 2048 columns)
constexpr int kMinBlocks = HB == 16 ? WT_SVD_MINB : 2;  // resident CTAs per SM (smem-limited)
constexpr int kEigWarps = WT_EIG_WARPS;
constexpr int kNZ = HB == 16 ? WT_SVD_NZ : 2;  // chunk buffers in the streamed Gram / rotation pipelines  // warps running the 32x32 eigen steps

__device__ __forceinline__ void eig_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEigWarps * 32) : "memory");
}

struct SvdWs {
  double* X;        // batch * npad * mpad (buffer 0)
  double* X2;       // batch * npad * mpad (buffer 1, target of the between-sweep reordering)
  int* xsel;        // batch: which buffer holds matrix b (reordering skips converged matrices)
  int* active;      // compacted list of the matrices still iterating (grid.y indexes it)
  unsigned long long* prof;  // optional phase-cycle counters (WT_SVD_PROFILE diagnostics)
  unsigned long long* offmax;  // batch  (bit pattern of a non-negative double)
  int* conv;        // batch: 1 = converged, 2 = non-finite
  int* pending;     // 1 counter (matrices still iterating)
  double* sig;      // batch * npad  (scratch for the final sort)
  int* perm;        // batch * npad
  int* bdone;       // batch * nblk: rounds of the current sweep finished per column block
  int* ticket;      // 1 counter: next visit of the current sweep (persistent sweeps)
  int* bver;        // batch * nblk: version of every column block (bumped when its data changes)
  unsigned long long* pclean;  // batch * nblk * nblk: (ver_I, ver_J) when pair (I, J) last tested clean
  double* scale;    // batch: power-of-two input scale (absmax_scale)
  double* gref;     // batch: largest squared column norm at the last reordering (null-column reference)
};

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

__device__ __forceinline__ double* mat_ptr(const SvdWs& ws, int64_t b, int64_t npad, int64_t mpad) {
  return (ws.xsel[b] ? ws.X2 : ws.X) + b * npad * mpad;
}

// ------------------------------------------------------------- copy in -----
// Per-matrix power-of-two scale that brings max |A_b| into [1, 2): the Gram
// entries the iteration forms (squares of the data) then stay far from the
// subnormal / overflow ranges, as LAPACK's dgesdd scales out-of-range inputs.
// The singular values are scaled back at the end (exact: powers of two).
// (two kernels: a grid over row blocks of every matrix max-reduces |A| into the
// scale slot as IEEE bits -- non-negative doubles and NaN order as unsigned
// integers -- then one thread per matrix turns the maximum into the scale)
__global__ void svd_absmax_part(const double* __restrict__ A, int64_t lda, int64_t sA, int64_t n1, int64_t n2,
                                unsigned long long* __restrict__ bits) {
  const int64_t b = blockIdx.y;
  unsigned long long mx = 0ull;
  for (int64_t row = blockIdx.x; row < n1; row += gridDim.x) {
    const double* a = A + b * sA + row * lda;
    for (int64_t c = threadIdx.x; c < n2; c += blockDim.x) {
      const unsigned long long v = (unsigned long long)__double_as_longlong(fabs(a[c]));
      mx = v > mx ? v : mx;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(bits + b, mx);
}

__global__ void svd_absmax_final(double* __restrict__ scale, int* __restrict__ nz, int64_t batch) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double mx = __longlong_as_double((long long)reinterpret_cast<const unsigned long long*>(scale)[b]);
  scale[b] = (mx > 0.0 && isfinite(mx)) ? ldexp(1.0, -ilogb(mx)) : 1.0;
  // K limit of the preconditioner's GEMMs on this slice: 0 for an all-zero slice
  // (its Gram and X V0 are zero: K3 writes the zero tiles without the k loop)
  if (nz) nz[b] = mx != 0.0 ? 0x7fffffff : 0;
}

int absmax_scale(const double* A, int64_t lda, int64_t sA, int64_t n1, int64_t n2, int64_t batch, double* scale,
                 cudaStream_t st, int* nz = nullptr) {
  WT_CUDA(cudaMemsetAsync(scale, 0, sizeof(double) * (size_t)batch, st));
  dim3 grid((unsigned)std::min<int64_t>(n1, std::max<int64_t>(1, 2048 / std::max<int64_t>(batch, 1))), (unsigned)batch);
  svd_absmax_part<<<grid, 256, 0, st>>>(A, lda, sA, n1, n2, reinterpret_cast<unsigned long long*>(scale));
  svd_absmax_final<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(scale, nz, batch);
  return check_launch("svd absmax scale");
}

__global__ void svd_copy_in(const double* __restrict__ A, int64_t lda, int64_t sA, bool right,
                            int64_t m, int64_t n, int64_t mpad, int64_t npad, const double* __restrict__ scale,
                            double* __restrict__ X) {
  const int64_t b = blockIdx.y;
  const int64_t total = npad * mpad;
  const double f = scale[b];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / mpad, r = e - c * mpad;
    double v = 0.0;
    if (c < n && r < m) v = f * (right ? A[b * sA + c * lda + r] : A[b * sA + r * lda + c]);
    X[b * total + e] = v;
  }
}

// ------------------------------------------------------ cluster helpers ----
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return (int)r;
}
// generic address of `p` (this CTA's shared memory) in CTA `rank` of the cluster
template <typename T>
__device__ __forceinline__ T* cluster_map(T* p, int rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<T*>(out);
}

// ---------------------------------------------------------- pair kernel ----
__device__ __forceinline__ double nanmax(double a, double b) {
  return (isnan(a) || isnan(b)) ? (a + b) : fmax(a, b);
}

// Rounds whose visits rotate only the block I x block J pairs.  cross = 0:
// none; cross = 1: every round but round 0; cross = F >= 2: all but F evenly
// spaced "full" rounds (round 0 and the last round among them), which also
// rotate the within-block pairs.
__host__ __device__ __forceinline__ int cross_only_round(int cross, int round, int nb) {
  if (!cross || round == 0) return 0;
  if (cross == 1) return 1;
  const int last = nb - 2;
  for (int j = 1; j < cross; ++j)
    if (round == (j * last) / (cross - 1)) return 0;
  return 1;
}

__device__ __forceinline__ int rr_index(int pos, int round, int nb) {
  // circle method: position 0 fixed, the others rotate by `round`
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (nb - 1);
}

struct PairSmem {
  double Z[kNZ][BW * LDZ];
  double G[1][BW * LDG];
  double Q[BW * LDG];
  double warp_off[kThreads / 32];
  double gmax;
  int any_rot;
  int skip;
  unsigned long long gmax_bits;
  long long ts[2];  // WT_SVD_PROFILE: end of the Gram stream, end of the reduction
};

// Squared column norms of the panel (the Gram's diagonal; after the eigen
// steps, that of the rotated panel) into ws.sig: the between-sweep reordering
// sorts by them instead of re-reading every matrix.  The last visit of a block
// in a sweep writes last (visits of a block are ordered by the block counters).
__device__ __forceinline__ void store_norms(const double* G, double* cn, int colI, int colJ) {
  if (threadIdx.x < BW) {
    const int c = threadIdx.x;
    cn[c < HB ? colI + c : colJ + c - HB] = G[c * LDG + c];
  }
}

__device__ __forceinline__ void load_chunk(double* Zs, const double* Xb, int64_t mpad, int colI,
                                           int colJ, int64_t r0) {
  // 32 columns x RCH rows, 16-byte cp.async; column c of the panel maps to
  // global column colI + c (c < 16) or colJ + c - 16.
  constexpr int VPC = RCH / 2;  // 16-byte vectors per column chunk
  for (int v = threadIdx.x; v < BW * VPC; v += kThreads) {
    const int c = v / VPC, rv = (v % VPC) * 2;
    const int gc = c < HB ? colI + c : colJ + c - HB;
    cp_async_zfill<16>(Zs + c * LDZ + rv, Xb + (int64_t)gc * mpad + r0 + rv, true);
  }
}

// One pair visit (matrix b, column blocks I and J).  Every early return is
// CTA-uniform (it depends on global flags / shared values only).
// SPLIT > 1: the visit is shared by the SPLIT CTAs of a thread-block cluster,
// CTA `rank` owning a contiguous range of the panel's row chunks.  Each CTA
// streams its rows' partial Gram, the partials are summed in rank order through
// distributed shared memory (every CTA ends with the same G, bit for bit), every
// CTA runs the same eigen steps redundantly (same Q) and rotates its own rows.
// The sweep kernel's cluster leader has already done the skip / converged checks.
template <int SPLIT>
__device__ __forceinline__ void pair_visit(PairSmem& S, const SvdWs& ws, int b, int I, int J,
                                           int64_t mpad, int64_t npad, double tol, int inner_sweeps,
                                           int cross_only, int rank = 0) {
  if (SPLIT == 1 && ws.conv[b]) return;
  const int colI = I * HB, colJ = J * HB;
  double* Xb = mat_ptr(ws, b, npad, mpad);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // A pair found clean whose two blocks have not changed since (same data, or
  // the same column sets after a reordering) is still clean: skip the visit
  // without touching the panel (the late sweeps are mostly such visits).
  const int nbk = (int)(npad / HB);
  if (SPLIT == 1 && ws.pclean) {
    if (tid == 0) {
      const unsigned long long cur =
          ((unsigned long long)(unsigned)__ldcg(ws.bver + (int64_t)b * nbk + I) << 32) |
          (unsigned)__ldcg(ws.bver + (int64_t)b * nbk + J);
      S.skip = __ldcg(ws.pclean + ((int64_t)b * nbk + I) * nbk + J) == cur;
    }
    __syncthreads();
    if (S.skip) return;
  }
  const int nch = (int)(mpad / RCH);
  // this CTA's row chunks [c0, c1) of the panel (all of them without a split)
  const int c0 = SPLIT == 1 ? 0 : (int)((int64_t)rank * nch / SPLIT);
  const int ncl = SPLIT == 1 ? nch : (int)((int64_t)(rank + 1) * nch / SPLIT) - c0;
  const bool lead = SPLIT == 1 || rank == 0;  // writes the visit's bookkeeping

  const long long t_start = clock64();
  // ---------------- 1. Gram G = Z^T Z: upper 10 of the 16 8x8 tiles --------
  // Rows are split over the 8 warps (warp w owns rows w*8 .. w*8+7 of every
  // chunk).  One LDS.128 per column group feeds two DMMAs: lane (r, k) holds
  // rows 2k and 2k+1, so the two products' k-slots are the even and the odd
  // rows -- any fixed row->slot map is valid for Z^T Z.  4 LDS.128 feed 20
  // DMMAs per warp per chunk; the 8 partial Grams are summed by a fixed tree.
  double acc[10][2];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < kNZ - 1; ++s0) {
    if (s0 < ncl) load_chunk(S.Z[s0], Xb, mpad, colI, colJ, (int64_t)(c0 + s0) * RCH);
    cp_async_commit();
  }
  for (int ch = 0; ch < ncl; ++ch) {
    const int nx = ch + kNZ - 1;
    if (nx < ncl) load_chunk(S.Z[nx % kNZ], Xb, mpad, colI, colJ, (int64_t)(c0 + nx) * RCH);
    cp_async_commit();
    cp_async_wait<kNZ - 1>();
    __syncthreads();
    const double* Zs = S.Z[ch % kNZ];
    double2 f[4];
#pragma unroll
    for (int tj = 0; tj < 4; ++tj)
      f[tj] = *reinterpret_cast<const double2*>(Zs + (tj * 8 + (lane >> 2)) * LDZ + warp * 8 + 2 * (lane & 3));
    int t = 0;
#pragma unroll
    for (int ta = 0; ta < 4; ++ta)
#pragma unroll
      for (int tb = ta; tb < 4; ++tb, ++t) {
        dmma884(acc[t][0], acc[t][1], f[ta].x, f[tb].x);
        dmma884(acc[t][0], acc[t][1], f[ta].y, f[tb].y);
      }
    __syncthreads();
  }
  if (tid == 0) S.ts[0] = clock64();
  {
#if WT_SVD_FLATRED
    // every warp parks its partial tiles in the (now free) chunk buffers; each
    // thread then sums fixed entries over the warps in warp order (deterministic),
    // writes them and their mirror into G and folds the diagonal into gmax
    // (shared 64-bit max of the bit patterns: non-negative doubles order as
    // integers; NaN is skipped like fmax does).  2 barriers instead of a tree.
    static_assert(kWarps * 10 * 64 <= kNZ * BW * LDZ, "partial tiles exceed the chunk buffers");
    double* red = S.Z[0];  // kWarps x 10 x 64 doubles
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      red[(warp * 10 + t) * 64 + 2 * lane] = acc[t][0];
      red[(warp * 10 + t) * 64 + 2 * lane + 1] = acc[t][1];
    }
    if (tid == 0) S.gmax_bits = 0ull;
    __syncthreads();
    if constexpr (SPLIT > 1) {
      // this CTA's partial after the warp sum, then the cluster's partials in rank order
      static_assert((kWarps + 1) * 640 <= kNZ * BW * LDZ, "cluster partial exceeds the chunk buffers");
      double* part = red + kWarps * 640;
      for (int e = tid; e < 640; e += kThreads) {
        double v = red[e];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) v += red[w * 640 + e];
        part[e] = v;
      }
      cluster_sync();
      for (int e = tid; e < 640; e += kThreads) {
        double v = *cluster_map(part + e, 0);
#pragma unroll
        for (int r = 1; r < SPLIT; ++r) v += *cluster_map(part + e, r);
        red[e] = v;  // own warp-0 partial slot is free: the loop below reads red[e] (w = 0 only)
      }
      __syncthreads();
    }
    for (int e = tid; e < 640; e += kThreads) {
      double v = red[e];
      if (SPLIT == 1) {
#pragma unroll
        for (int w = 1; w < kWarps; ++w) v += red[w * 640 + e];
      }
      const int t = e >> 6, l = (e & 63) >> 1, h = e & 1;
      // tile t -> (ta, tb), ta <= tb, in the order of the accumulation loop
      const int ta = t < 4 ? 0 : t < 7 ? 1 : t < 9 ? 2 : 3;
      const int tb = ta + t - (ta == 0 ? 0 : ta == 1 ? 4 : ta == 2 ? 7 : 9);
      const int r = ta * 8 + (l >> 2), c = tb * 8 + 2 * (l & 3) + h;
      if (ta < tb || r <= c) {
        S.G[0][r * LDG + c] = v;
        S.G[0][c * LDG + r] = v;
        if (r == c && !isnan(v)) atomicMax(&S.gmax_bits, (unsigned long long)__double_as_longlong(v));
      }
    }
    __syncthreads();
  }
#else
    // deterministic tree over the 8 warps through the (now free) chunk buffers
    double* red = S.Z[0];  // 4 x 10 x 64 doubles
#pragma unroll
    static_assert((kWarps / 2) * 10 * 64 <= kNZ * BW * LDZ, "tree buffer exceeds the chunk buffers");
    for (int half = kWarps / 2; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half) {
#pragma unroll
        for (int t = 0; t < 10; ++t) {
          red[((warp - half) * 10 + t) * 64 + 2 * lane] = acc[t][0];
          red[((warp - half) * 10 + t) * 64 + 2 * lane + 1] = acc[t][1];
        }
      }
      __syncthreads();
      if (warp < half) {
#pragma unroll
        for (int t = 0; t < 10; ++t) {
          acc[t][0] += red[(warp * 10 + t) * 64 + 2 * lane];
          acc[t][1] += red[(warp * 10 + t) * 64 + 2 * lane + 1];
        }
      }
      __syncthreads();
    }
    if (warp == 0) {  // C frag: row ta*8 + lane/4, col tb*8 + 2*(lane%4) + h; mirror below
      int t = 0;
#pragma unroll
      for (int ta = 0; ta < 4; ++ta)
#pragma unroll
        for (int tb = ta; tb < 4; ++tb, ++t)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = ta * 8 + (lane >> 2), c = tb * 8 + 2 * (lane & 3) + h;
            if (ta < tb || r <= c) {
              S.G[0][r * LDG + c] = acc[t][h];
              S.G[0][c * LDG + r] = acc[t][h];
            }
          }
      __syncwarp();
      double gm = S.G[0][lane * LDG + lane];  // largest squared column norm of the panel
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
      if (lane == 0) S.gmax = gm;
    }
    __syncthreads();
  }
#endif

  // ---------------- 2. convergence test on this pair -----------------------
  // Pair (i, j) is orthogonal enough when
  //   |g_ij| <= tol * sqrt(g_ii g_jj) + (1e3 eps)^2 * gmax,
  // the second term only matters for numerically-null columns (norm below
  // ~1e-13 |z_max|), whose directions are rounding noise and must not keep
  // the iteration alive; real columns are held to the relative tolerance.
  // `off` is the largest |g_ij| / (that bound) * tol, so off < tol <=> converged.
  if (tid == 0) S.ts[1] = clock64();
#if WT_SVD_FLATRED
  const double gmax = __longlong_as_double((long long)S.gmax_bits);
#else
  const double gmax = S.gmax;
#endif
  const double floor_c = kFloorEps * kFloorEps / tol;
  // Two numerically-null columns (both norms below 1e3 eps times the matrix's largest column norm at
  // the reordering before this sweep -- sigma_1 from the second sweep on) are left to each other: when
  // every column of a visit is null the panel-relative floor above is itself noise and such pairs
  // rotated for ever (rank-82 123 x 245 slices: 40 sweeps without progress, found by
  // tools/fuzz_parity.py).  Their singular values are below 1e-12 sigma_1, where the vectors are
  // re-orthonormalised by wt_orthonormal_fixup_f64 anyway.  (A null column is still rotated against
  // the real ones: K5's projector V_r V_r^T needs the null vectors out of the real subspace --
  // exempting every pair with a null column gave O(1) reconstruction errors in the same sweep.)
  const double kNull2 = kFloorEps * kFloorEps * ws.gref[b];
  {
    // 1 / max(sqrt(g_ii g_jj), floor_c g_max) = min(rsqrt(g_ii g_jj), 1 / (floor_c g_max)):
    // no sqrt and no division per pair (the test was ~10% of the kernel's stall samples)
    const double rfl = 1.0 / (floor_c * gmax);
    double mx = 0.0;
    auto test_pair = [&](int i, int j) {
      const double gii = S.G[0][i * LDG + i], gjj = S.G[0][j * LDG + j];
      const double gij = S.G[0][i * LDG + j];
      double c = 0.0;
      if (gij != 0.0 && fmax(gii, gjj) > kNull2) c = fabs(gij) * fmin(rsqrt(gii * gjj), rfl);
      if (isnan(gii) || isnan(gjj)) c = gii + gjj;
      mx = nanmax(mx, c);
    };
    if (cross_only && HB * HB == kThreads) {
      // cross-only visits answer for the block I x block J pairs alone (the
      // within-block pairs are tested and rotated at the sweep's round 0):
      // exactly one pair per thread
      test_pair(tid / HB, HB + tid % HB);
    } else
    for (int e = tid; e < BW * BW; e += kThreads) {
      const int i = e / BW, j = e % BW;
      if (i < j && !(cross_only && (i < HB) == (j < HB))) {
        const double gii = S.G[0][i * LDG + i], gjj = S.G[0][j * LDG + j];
        const double gij = S.G[0][i * LDG + j];
        double c = 0.0;
        if (gij != 0.0 && fmax(gii, gjj) > kNull2) c = fabs(gij) * fmin(rsqrt(gii * gjj), rfl);
        if (isnan(gii) || isnan(gjj)) c = gii + gjj;
        mx = nanmax(mx, c);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = nanmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) S.warp_off[warp] = mx;
  }
  __syncthreads();
  double off = 0.0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) off = nanmax(off, S.warp_off[w]);
  // NaN-propagating max through the bit pattern (non-negative doubles order as uint64)
  if (tid == 0) atomicMax(&ws.offmax[b], (unsigned long long)__double_as_longlong(off));
  if (!(off >= tol) || isinf(off)) {  // converged pair (or NaN / inf: recorded above)
    if (lead) store_norms(S.G[0], ws.sig + (int64_t)b * npad, colI, colJ);
    if (lead && ws.pclean && tid == 0 && off < tol)  // certified clean at the blocks' current versions
      __stcg(ws.pclean + ((int64_t)b * nbk + I) * nbk + J,
             ((unsigned long long)(unsigned)__ldcg(ws.bver + (int64_t)b * nbk + I) << 32) |
                 (unsigned)__ldcg(ws.bver + (int64_t)b * nbk + J));
    return;
  }
  if (lead && tid == 0) atomicAdd(ws.pending + 1, 1);  // rotated-pair counter (diagnostics)

  const long long t_gram = clock64();
  // ---------------- 3. eigen-decomposition of G (cyclic parallel Jacobi) ----
  // Only the first kEigWarps warps run the steps (named barrier 1); the rest
  // wait at the CTA barrier after it.  16 groups of TPG threads: group g owns
  // rotation pair g of every step, computes its (c, s) redundantly (no shared
  // round trip), then applies G <- G J, Q <- Q J (columns p, q) and, after a
  // barrier, G <- J^T G (rows p, q).  Fewer warps = fewer redundant FP64
  // rotation chains per SM: the step was issue-bound with all 8 warps (clock64
  // phase counters, WT_SVD_PROFILE).
  for (int e = tid; e < BW * BW; e += kThreads) {
    const int i = e / BW, j = e % BW;
    S.Q[i * LDG + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (warp < kEigWarps) {
    constexpr int TPG = kEigWarps * 32 / (BW / 2);  // threads per rotation group
    constexpr int RPT = BW / TPG;                   // rows (columns) per thread
    double* G = S.G[0];
    double* Q = S.Q;
    const int grp = tid / TPG, sub = tid % TPG;
    const double fl = floor_c * gmax;
    const double rot_floor = tol * tol * (fl * fl);
    const double tol2 = tol * tol;
    const double psc = gmax > 0.0 ? ldexp(1.0, -ilogb(gmax)) : 1.0;  // keeps a^2 + b^2 in range
    for (int sweep = 0; sweep < inner_sweeps; ++sweep) {
      int my_rot = 0;
      const int nsteps = cross_only ? HB : BW - 1;
      for (int step = 0; step < nsteps; ++step) {
        int p, q;
        if (cross_only) {  // block I x block J pairs only: 16 steps of 16 disjoint pairs
          p = grp;
          q = HB + (grp + step) % HB;
        } else {           // all 496 pairs of the 32 columns: 31 round-robin steps
          p = rr_index(grp, step, BW);
          q = rr_index(BW - 1 - grp, step, BW);
          if (p > q) { const int t = p; p = q; q = t; }
        }
        const double gpp = G[p * LDG + p], gqq = G[q * LDG + q], gpq = G[p * LDG + q];
        // rotate iff |g_pq| > tol * max(sqrt(g_pp g_qq), floor_c g_max)  (squared: no sqrt)
        const bool rot = gpq * gpq > fmax(tol2 * (gpp * gqq), rot_floor) && fmax(gpp, gqq) > kNull2;
        __syncwarp();
        double c = 1.0, s = 0.0;
        if (rot) {
          // Jacobi rotation from two rsqrt and no division (the dependent FP64
          // MUFU chain bounds the step): with a = g_qq - g_pp, b = 2 g_pq
          // (scaled by a power of two ~ 1/g_max), cos 2phi = |a| / r,
          // c = sqrt((1 + cos 2phi) / 2), s = sign(a) b / (2 r c), |phi| <= pi/4
          // -- the same rotation as Rutishauser's t = sgn(tau)/(|tau|+sqrt(1+tau^2)).
          const double a = (gqq - gpp) * psc, bb = 2.0 * gpq * psc;
          const double rinv = rsqrt(fma(a, a, bb * bb));
          const double h = fma(0.5, fabs(a) * rinv, 0.5);
          const double rh = rsqrt(h);
          c = h * rh;
          s = (a >= 0.0 ? 0.5 : -0.5) * bb * rinv * rh;
          // one Newton step on c^2 + s^2 = 1 keeps the accumulated Q orthogonal
          const double f = fma(-0.5, fma(c, c, s * s), 1.5);
          c *= f;
          s *= f;
          my_rot = 1;
          double ga[RPT], gb[RPT], qa[RPT], qb[RPT];
#pragma unroll
          for (int h = 0; h < RPT; ++h) {  // columns: G <- G J, Q <- Q J (loads first)
            const int i = sub + TPG * h;
            ga[h] = G[i * LDG + p];
            gb[h] = G[i * LDG + q];
            qa[h] = Q[i * LDG + p];
            qb[h] = Q[i * LDG + q];
          }
#pragma unroll
          for (int h = 0; h < RPT; ++h) {
            const int i = sub + TPG * h;
            G[i * LDG + p] = c * ga[h] - s * gb[h];
            G[i * LDG + q] = s * ga[h] + c * gb[h];
            Q[i * LDG + p] = c * qa[h] - s * qb[h];
            Q[i * LDG + q] = s * qa[h] + c * qb[h];
          }
        }
        eig_barrier();
        if (rot) {
          double ra[RPT], rb[RPT];
#pragma unroll
          for (int h = 0; h < RPT; ++h) {
            const int j = sub + TPG * h;
            ra[h] = G[p * LDG + j];
            rb[h] = G[q * LDG + j];
          }
#pragma unroll
          for (int h = 0; h < RPT; ++h) {  // rows: G <- J^T G
            const int j = sub + TPG * h;
            double np = c * ra[h] - s * rb[h], nq = s * ra[h] + c * rb[h];
            if (j == q) np = 0.0;  // annihilated pair
            if (j == p) nq = 0.0;
            G[p * LDG + j] = np;
            G[q * LDG + j] = nq;
          }
        }
        eig_barrier();
      }
      S.any_rot = 0;
      eig_barrier();
      if (my_rot) S.any_rot = 1;
      eig_barrier();
      if (!S.any_rot) break;
      eig_barrier();
    }
  }
  // (split: every CTA of the cluster has read the others' Gram partials, which
  // live in the chunk buffers the rotation stream refills next)
  if constexpr (SPLIT > 1) cluster_sync(); else __syncthreads();
  if (lead) store_norms(S.G[0], ws.sig + (int64_t)b * npad, colI, colJ);  // rotated Gram's diagonal
  const long long t_eig = clock64();
  // ---------------- 4. Z <- Z Q, streamed, written back in place -----------
  // warp w: chunk rows rt*16 .. rt*16+15 (two 8-row tiles) x output n-tiles
  // {2nh, 2nh+1}; its Q b-fragments Q[kk*4 + lane%4][n*8 + lane/4] stay in
  // registers for the whole stream.
  constexpr int RT = RCH / 16;  // 16-row tiles per chunk; warps = RT x 2 column halves
  const int rt = warp % RT, nh = warp / RT;
  double qf[8][2];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int j = 0; j < 2; ++j) qf[kk][j] = S.Q[(kk * 4 + (lane & 3)) * LDG + (2 * nh + j) * 8 + (lane >> 2)];
#pragma unroll
  for (int s0 = 0; s0 < kNZ - 1; ++s0) {
    if (s0 < ncl) load_chunk(S.Z[s0], Xb, mpad, colI, colJ, (int64_t)(c0 + s0) * RCH);
    cp_async_commit();
  }
  for (int ch = 0; ch < ncl; ++ch) {
    const int nx = ch + kNZ - 1;
    if (nx < ncl) load_chunk(S.Z[nx % kNZ], Xb, mpad, colI, colJ, (int64_t)(c0 + nx) * RCH);
    cp_async_commit();
    cp_async_wait<kNZ - 1>();
    __syncthreads();
    double* Zs = S.Z[ch % kNZ];
    double o[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) o[i][j][0] = o[i][j][1] = 0.0;
    // one LDS.128 per k-step: rows r0 + 2(lane/4) and +1 feed the "even" and
    // "odd" 8-row tiles; results go back as STS.128 row pairs
    const int r0 = rt * 16 + 2 * (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double2 a = *reinterpret_cast<const double2*>(Zs + (kk * 4 + (lane & 3)) * LDZ + r0);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        dmma884(o[0][j][0], o[0][j][1], a.x, qf[kk][j]);
        dmma884(o[1][j][0], o[1][j][1], a.y, qf[kk][j]);
      }
    }
    // results straight from the DMMA fragments to global, in place: a lane
    // holds rows r0, r0+1 of 4 output columns, so the 8 lanes sharing lane%4
    // write 128 contiguous bytes of one column (no smem round trip)
    const int64_t rbase = (int64_t)(c0 + ch) * RCH;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = (2 * nh + j) * 8 + 2 * (lane & 3) + h;
        const int gc = c < HB ? colI + c : colJ + c - HB;
        *reinterpret_cast<double2*>(Xb + (int64_t)gc * mpad + rbase + r0) =
            make_double2(o[0][j][h], o[1][j][h]);
      }
    __syncthreads();  // every warp has read the chunk before its buffer is refilled
  }
  if (lead && ws.pclean && tid == 0) {  // both blocks changed (the visit owns them exclusively)
    __stcg(ws.bver + (int64_t)b * nbk + I, __ldcg(ws.bver + (int64_t)b * nbk + I) + 1);
    __stcg(ws.bver + (int64_t)b * nbk + J, __ldcg(ws.bver + (int64_t)b * nbk + J) + 1);
  }
  if (lead && ws.prof && tid == 0) {
    atomicAdd(ws.prof + 0, (unsigned long long)(t_gram - t_start));
    atomicAdd(ws.prof + 1, (unsigned long long)(t_eig - t_gram));
    atomicAdd(ws.prof + 2, (unsigned long long)(clock64() - t_eig));
    atomicAdd(ws.prof + 3, 1ull);
    atomicAdd(ws.prof + 4, (unsigned long long)(S.ts[0] - t_start));
    atomicAdd(ws.prof + 5, (unsigned long long)(S.ts[1] - S.ts[0]));
  }
}

// One launch per round: CTA (x, y) visits pair x of active matrix y.
__global__ void __launch_bounds__(kThreads, kMinBlocks) svd_pair_kernel(SvdWs ws, int64_t mpad, int64_t npad,
                                                               int round, double tol, int inner_sweeps,
                                                               int cross_only) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PairSmem& S = *reinterpret_cast<PairSmem*>(smem_raw);
  const int nb = (int)(npad / HB);
  const int I = rr_index(blockIdx.x, round, nb), J = rr_index(nb - 1 - blockIdx.x, round, nb);
  pair_visit<1>(S, ws, ws.active[blockIdx.y], I, J, mpad, npad, tol, inner_sweeps, cross_only);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One persistent launch per sweep: CTAs take visits from a global ticket in
// (round, matrix, pair) order and start a visit as soon as the two visits of
// the previous round that held its blocks have finished (per-block round
// counters ws.bdone), so a round's tail overlaps the next round's start
// instead of draining the GPU at every kernel boundary.  A visit only waits on
// smaller tickets, which running CTAs already hold: no deadlock.
// SPLIT > 1 (launched with SPLIT-CTA clusters): the cluster is the unit that
// takes tickets; its leader CTA schedules (ticket, dependency wait, converged /
// clean-pair skip) and the others read the item from the leader's shared memory.
template <int SPLIT>
__global__ void __launch_bounds__(kThreads, SPLIT > 1 ? 2 : kMinBlocks) svd_sweep_kernel(SvdWs ws, int64_t mpad, int64_t npad,
                                                                int n_active, double tol, int inner_sweeps,
                                                                int cross) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PairSmem& S = *reinterpret_cast<PairSmem*>(smem_raw);
  __shared__ int s_item[5];  // ticket, (matrix, block I, block J) of the visit, skip (SPLIT > 1)
  const int nb = (int)(npad / HB);
  const int per_round = n_active * (nb / 2);
  const int total = per_round * (nb - 1);
  const int rank = SPLIT == 1 ? 0 : cluster_rank();
  for (;;) {
    if (threadIdx.x == 0 && rank == 0) {
      const int t = atomicAdd(ws.ticket, 1);
      s_item[0] = t;
      if (t < total) {
        const int round = t / per_round, rem = t - round * per_round;
        const int ai = rem / (nb / 2), k = rem - ai * (nb / 2);
        const int b = ws.active[ai];
        const int I = rr_index(k, round, nb), J = rr_index(nb - 1 - k, round, nb);
        s_item[1] = b;
        s_item[2] = I;
        s_item[3] = J;
        while (ld_acquire(ws.bdone + (int64_t)b * nb + I) < round) __nanosleep(WT_SVD_SPIN_NS);
        while (ld_acquire(ws.bdone + (int64_t)b * nb + J) < round) __nanosleep(WT_SVD_SPIN_NS);
        if (SPLIT > 1) {
          int skip = ws.conv[b] != 0;
          if (!skip && ws.pclean) {
            const unsigned long long cur =
                ((unsigned long long)(unsigned)__ldcg(ws.bver + (int64_t)b * nb + I) << 32) |
                (unsigned)__ldcg(ws.bver + (int64_t)b * nb + J);
            skip = __ldcg(ws.pclean + ((int64_t)b * nb + I) * nb + J) == cur;
          }
          s_item[4] = skip;
        }
      }
    }
    int t, b, I, J, skip = 0;
    if constexpr (SPLIT == 1) {
      __syncthreads();
      t = s_item[0], b = s_item[1], I = s_item[2], J = s_item[3];
    } else {
      cluster_sync();
      const int* li = cluster_map(s_item, 0);
      t = li[0], b = li[1], I = li[2], J = li[3], skip = li[4];
    }
    if (t >= total) {
      if constexpr (SPLIT > 1) cluster_sync();  // the leader's item stays readable until all have read it
      return;
    }
    const int round = t / per_round;
    const int cross_only = cross_only_round(cross, round, nb);
    if (!skip) pair_visit<SPLIT>(S, ws, b, I, J, mpad, npad, tol, inner_sweeps, cross_only, rank);
    if constexpr (SPLIT > 1) {
      __threadfence();  // every CTA's stores of the visit, before the leader's release below
      cluster_sync();
    } else {
      __syncthreads();  // every store of the visit precedes the release below (and s_item reuse)
    }
    if (threadIdx.x == 0 && rank == 0) {
#if WT_SVD_LIGHT_RELEASE
      // one acq_rel fence then two relaxed stores: a release of both counters
      // (the CTA / cluster barrier above orders every thread's stores first)
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      st_relaxed(ws.bdone + (int64_t)b * nb + I, round + 1);
      st_relaxed(ws.bdone + (int64_t)b * nb + J, round + 1);
#else
      __threadfence();
      st_release(ws.bdone + (int64_t)b * nb + I, round + 1);
      st_release(ws.bdone + (int64_t)b * nb + J, round + 1);
#endif
    }
  }
}

// ------------------------------------------------------ sweep bookkeeping --
__global__ void svd_end_sweep(SvdWs ws, int batch, double tol) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x) {
    if (ws.conv[b]) continue;
    const double off = __longlong_as_double((long long)ws.offmax[b]);
    if (isnan(off) || isinf(off)) ws.conv[b] = 2;
    else if (off < tol) ws.conv[b] = 1;
    else ws.active[atomicAdd(ws.pending, 1)] = b;  // order is irrelevant: matrices are independent
    ws.offmax[b] = 0ull;
  }
}

// ------------------------------------------------------------- finalize ----
// One CTA per matrix: column norms, descending sort (ties by index), sigma out.
__global__ void svd_norms_sort(SvdWs ws, int64_t mpad, int64_t npad, int64_t n, int npow2,
                               double* __restrict__ sigma, int* __restrict__ info, int max_sweeps_hit,
                               int use_cn = 0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* key = reinterpret_cast<double*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + npow2);
  const int b = sigma == nullptr ? ws.active[blockIdx.x] : blockIdx.x;
  if (sigma == nullptr && ws.conv[b]) return;  // reordering: converged matrices stay put
  const double* Xb = mat_ptr(ws, b, npad, mpad);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (sigma == nullptr && use_cn) {  // reordering from the norms the last visits left in ws.sig
    for (int c = threadIdx.x; c < npow2; c += blockDim.x) {
      key[c] = c < n ? ws.sig[(int64_t)b * npad + c] : -1.0;  // squared norms: same order
      idx[c] = c;
    }
  } else
  for (int c = warp; c < npow2; c += nw) {
    double s = 0.0;
    if (c < n) {
      for (int64_t r = lane; r < mpad; r += 32) {
        const double v = Xb[(int64_t)c * mpad + r];
        s = fma(v, v, s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (lane == 0) {
      // the reordering pass sorts squared norms (the units the visits leave in ws.sig)
      key[c] = c < n ? (sigma == nullptr ? s : sqrt(s)) : -1.0;
      idx[c] = c;
    }
  }
  __syncthreads();
  // bitonic sort: descending key, ascending index on ties; NaN sorts first
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const double ki = key[i], kl = key[l];
          const int ii = idx[i], il = idx[l];
          // "i before l" in final order?
          const bool i_first = (ki > kl) || (ki == kl && ii < il) || (isnan(ki) && !isnan(kl));
          const bool up = ((i & k) == 0);
          if (up != i_first) {
            key[i] = kl; key[l] = ki;
            idx[i] = il; idx[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  if (sigma == nullptr) {  // reordering pass between sweeps: permutation only
    // an all-zero matrix (largest norm exactly 0, e.g. the detail slices of a
    // slice-constant operator) is already diagonal: retire it before any visit
    if (threadIdx.x == 0 && key[0] == 0.0) ws.conv[b] = 1;
    if (threadIdx.x == 0) ws.gref[b] = key[0];
    for (int i = threadIdx.x; i < npad; i += blockDim.x) ws.perm[(int64_t)b * npad + i] = idx[i];
    // the norms follow their columns (blocks skipped in the next sweep keep them valid)
    for (int i = threadIdx.x; i < n; i += blockDim.x) ws.sig[(int64_t)b * npad + i] = key[i];
    if (ws.bver) {  // a block whose column set changed has new data
      const int nbk = (int)(npad / HB);
      for (int B = threadIdx.x; B < nbk; B += blockDim.x) {
        bool moved = false;
        for (int i = B * HB; i < (B + 1) * HB; ++i) moved |= (idx[i] / HB) != B;
        if (moved) ws.bver[(int64_t)b * nbk + B] += 1;
      }
    }
    return;
  }
  bool bad = false;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sigma[(int64_t)b * n + i] = key[i] / ws.scale[b];  // (exact: a power of two)
    ws.perm[(int64_t)b * npad + i] = idx[i];
    ws.sig[(int64_t)b * npad + i] = key[i];
    if (!isfinite(key[i])) bad = true;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    int st = 0;
    if (bad || ws.conv[b] == 2) st = 1;
    else if (ws.conv[b] == 0 && max_sweeps_hit) st = 2;
    info[b] = st;
  }
}

__global__ void svd_gather(SvdWs ws, int64_t mpad, int64_t npad, int64_t m, int64_t nvec,
                           double* __restrict__ vec) {
  const int64_t i = blockIdx.x, b = blockIdx.y;
  const int c = ws.perm[b * npad + i];
  const double s = ws.sig[b * npad + i];
  const double inv = (s > 0.0 && isfinite(s)) ? 1.0 / s : 0.0;
  const double* col = mat_ptr(ws, b, npad, mpad) + (int64_t)c * mpad;
  double* dst = vec + (b * nvec + i) * m;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) dst[r] = col[r] * inv;
}

// other[b][i] = cur[b][perm[b][i]] (whole columns) for every matrix still
// iterating; svd_flip then makes `other` current for those matrices.
__global__ void svd_permute_cols(SvdWs ws, int64_t mpad, int64_t npad) {
  const int64_t i = blockIdx.x, b = ws.active[blockIdx.y];
  if (ws.conv[b]) return;
  const int c = ws.perm[b * npad + i];
  const bool sel = ws.xsel[b];
  const double* cur = (sel ? ws.X2 : ws.X) + b * npad * mpad;
  double* oth = (sel ? ws.X : ws.X2) + b * npad * mpad;
  const double2* src = reinterpret_cast<const double2*>(cur + (int64_t)c * mpad);
  double2* dst = reinterpret_cast<double2*>(oth + i * mpad);
  for (int64_t r = threadIdx.x; r < mpad / 2; r += blockDim.x) dst[r] = src[r];
}

__global__ void svd_fill_int(int* a, int n, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
}

__global__ void svd_iota(int* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void svd_flip(SvdWs ws, int batch) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x)
    if (!ws.conv[b]) ws.xsel[b] ^= 1;
}

struct WsLayout {
  int64_t m, n, mpad, npad;
  size_t off_X, off_X2, off_xsel, off_active, off_off, off_conv, off_pending, off_sig, off_perm, off_bdone,
      off_bver, off_pclean, off_scale, off_gref, off_nz, off_eig, eig_bytes, total;
  bool skip;     // pair-skip bookkeeping (nblk <= kSkipMaxBlocks)
  bool precond;  // Gram-eigenbasis preconditioner (eig.cu) before the sweeps
};

// Slices with at least this many short-side columns start the sweeps from
// X V0, V0 = eigenbasis of X^T X (eig.cu): 3 sweeps instead of 12-17 on the
// config 3-5 slices.  Below it plain Jacobi is cheap enough.
constexpr int64_t kPrecondMinN = 128;
inline bool precond_enabled(int64_t n) {
  return option(WT_OPT_SVD_PRECOND) != 0 && n >= kPrecondMinN && n <= 2048;
}

WsLayout ws_layout(int64_t n1, int64_t n2, int64_t batch, bool allow_precond = true) {
  WsLayout L{};
  L.m = std::max(n1, n2);
  L.n = std::min(n1, n2);
  L.mpad = round_up(std::max<int64_t>(L.m, 1), RCH);
  L.npad = round_up(std::max<int64_t>(L.n, 1), BW);
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) / 256 * 256; return r; };
  L.off_X = take(sizeof(double) * (size_t)(batch * L.npad * L.mpad));
  L.off_X2 = take(sizeof(double) * (size_t)(batch * L.npad * L.mpad));
  L.off_xsel = take(sizeof(int) * (size_t)batch);
  L.off_active = take(sizeof(int) * (size_t)batch);
  L.off_off = take(sizeof(unsigned long long) * (size_t)batch);
  L.off_conv = take(sizeof(int) * (size_t)batch);
  L.off_pending = take(sizeof(int) * 4);
  L.off_sig = take(sizeof(double) * (size_t)(batch * L.npad));
  L.off_perm = take(sizeof(int) * (size_t)(batch * L.npad));
  L.off_bdone = take(sizeof(int) * (size_t)(batch * (L.npad / HB)));
  const int64_t nbk = L.npad / HB;
  L.skip = nbk <= kSkipMaxBlocks;
  L.off_bver = take(L.skip ? sizeof(int) * (size_t)(batch * nbk) : 0);
  L.off_pclean = take(L.skip ? sizeof(unsigned long long) * (size_t)(batch * nbk * nbk) : 0);
  L.off_scale = take(sizeof(double) * (size_t)batch);
  L.off_gref = take(sizeof(double) * (size_t)batch);
  L.off_nz = take(sizeof(int) * (size_t)batch);
  L.precond = allow_precond && precond_enabled(L.n);
  L.eig_bytes = L.precond ? eig_workspace_bytes(L.n, batch) : 0;
  L.off_eig = take(L.eig_bytes);
  L.total = o;
  return L;
}

}  // namespace SVD_NS
}  // namespace wt

namespace wt {
namespace SVD_NS {

// One persistent sweep launch; SPLIT > 1 runs every visit on a SPLIT-CTA
// cluster (rows split), as many clusters as can be resident.
template <int SPLIT>
int launch_sweep(const SvdWs& ws, int64_t mpad, int64_t npad, int n_active, double tol, int inner,
                 int cross, int64_t visits, int max_ctas, cudaStream_t st) {
  auto kern = svd_sweep_kernel<SPLIT>;
  if (int e = ensure_smem(kern, sizeof(PairSmem))) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = SPLIT;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sizeof(PairSmem);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = SPLIT > 1 ? 1 : 0;
  int64_t units = std::max(max_ctas / SPLIT, 1);
  if (SPLIT > 1) {
    cfg.gridDim = dim3((unsigned)(SPLIT * units));
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc <= 0) {
      (void)cudaGetLastError();  // clusters of this shape cannot be resident: caller runs S = 1
      return WT_ERR_UNSUPPORTED;
    }
    units = std::min<int64_t>(units, nc);
  }
  units = std::min<int64_t>(units, visits);
  cfg.gridDim = dim3((unsigned)(SPLIT * units));
  WT_CUDA(cudaLaunchKernelEx(&cfg, kern, ws, mpad, npad, n_active, tol, inner, cross));
  return WT_OK;
}

size_t workspace_bytes(int64_t n1, int64_t n2, int64_t batch) {
  if (n1 < 0 || n2 < 0 || batch < 0) return 0;
  return ws_layout(n1, n2, batch).total;
}

int jacobi(const double* A, int64_t lda, int64_t strideA, int64_t n1,
                                 int64_t n2, int64_t batch, double* sigma, double* vec,
                                 int64_t nvec, int* info, double tol, int max_sweeps,
                                 void* workspace, size_t workspace_bytes, void* stream, bool allow_precond = true) {
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && batch >= 0, "svd: bad shape %lld x %lld", (long long)n1,
             (long long)n2);
  if (batch == 0) return WT_OK;
  WT_REQUIRE(lda >= n2, "svd: lda < n2");
  const WsLayout L = ws_layout(n1, n2, batch, allow_precond);
  WT_REQUIRE(nvec >= 0 && nvec <= L.n, "svd: nvec %lld outside [0, %lld]", (long long)nvec,
             (long long)L.n);
  WT_REQUIRE(workspace != nullptr && workspace_bytes >= L.total,
             "svd: workspace too small (%zu < %zu)", workspace_bytes, L.total);
  int npow2 = 1;
  while (npow2 < L.npad) npow2 <<= 1;
  WT_REQUIRE(npow2 <= 8192, "svd: min(n1, n2) = %lld above the 8192 sort limit", (long long)L.n);
  cudaStream_t st = (cudaStream_t)stream;
  char* base = static_cast<char*>(workspace);
  SvdWs ws{reinterpret_cast<double*>(base + L.off_X), reinterpret_cast<double*>(base + L.off_X2),
           reinterpret_cast<int*>(base + L.off_xsel), reinterpret_cast<int*>(base + L.off_active),
           nullptr,
           reinterpret_cast<unsigned long long*>(base + L.off_off),
           reinterpret_cast<int*>(base + L.off_conv), reinterpret_cast<int*>(base + L.off_pending),
           reinterpret_cast<double*>(base + L.off_sig), reinterpret_cast<int*>(base + L.off_perm),
           reinterpret_cast<int*>(base + L.off_bdone), reinterpret_cast<int*>(base + L.off_pending) + 2,
           nullptr, nullptr, reinterpret_cast<double*>(base + L.off_scale),
           reinterpret_cast<double*>(base + L.off_gref)};
  const int pair_skip = option(WT_OPT_SVD_PAIR_SKIP);
  if (L.skip && pair_skip) {
    ws.bver = reinterpret_cast<int*>(base + L.off_bver);
    ws.pclean = reinterpret_cast<unsigned long long*>(base + L.off_pclean);
    const int64_t nbk = L.npad / HB;
    WT_CUDA(cudaMemsetAsync(ws.bver, 0, sizeof(int) * (size_t)(batch * nbk), (cudaStream_t)stream));
    WT_CUDA(cudaMemsetAsync(ws.pclean, 0xff, sizeof(unsigned long long) * (size_t)(batch * nbk * nbk),
                            (cudaStream_t)stream));
  }
  if (tol <= 0.0) tol = 4.0 * 2.220446049250313e-16 * sqrt((double)L.m) + 1e-15;
  if (max_sweeps <= 0) max_sweeps = 80;  // (full-rank slices take 3-17; rank-deficient ones without the preconditioner up to ~25)
  const bool right = n1 <= n2;

  {
    dim3 grid((unsigned)std::min<int64_t>((L.npad * L.mpad + 255) / 256, 4096), (unsigned)batch);
    if (int e = absmax_scale(A, lda, strideA, n1, n2, batch, ws.scale, st, reinterpret_cast<int*>(base + L.off_nz)))
      return e;
    svd_copy_in<<<grid, 256, 0, st>>>(A, lda, strideA, right, L.m, L.n, L.mpad, L.npad, ws.scale, ws.X);
    if (int e = check_launch("svd_copy_in")) return e;
  }
  WT_CUDA(cudaMemsetAsync(ws.offmax, 0, sizeof(unsigned long long) * batch, st));
  WT_CUDA(cudaMemsetAsync(ws.conv, 0, sizeof(int) * batch, st));
  WT_CUDA(cudaMemsetAsync(ws.xsel, 0, sizeof(int) * batch, st));
  g_last_fallbacks = -1;
  if (L.precond) {
    // X2 <- X V0 (rows n .. npad-1 of the column-major panels stay zero), then
    // every matrix starts from buffer 1
    WT_CUDA(cudaMemsetAsync(ws.X2, 0, sizeof(double) * (size_t)(batch * L.npad * L.mpad), st));
    int fallback = 0;
    if (int e = eig_precondition(ws.X, ws.X2, L.mpad, L.n, L.mpad, L.npad * L.mpad, batch, L.n, L.mpad,
                                 L.npad * L.mpad, base + L.off_eig, L.eig_bytes, &fallback, st,
                                 reinterpret_cast<const int*>(base + L.off_nz)))
      return e;
    g_last_fallbacks = fallback;
    svd_fill_int<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(ws.xsel, (int)batch, 1);
  }
  svd_iota<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(ws.active, (int)batch);
  int64_t n_active = batch;
  WT_CUDA(cudaMemsetAsync(ws.pending, 0, sizeof(int) * 3, st));

  if (int e = ensure_smem(svd_pair_kernel, sizeof(PairSmem))) return e;
  // Persistent sweeps (one launch per sweep, visits scheduled by block
  // dependencies) unless WT_SVD_PERSIST=0 (one launch per round).
  const int persist = option(WT_OPT_SVD_PERSIST);
  int sweep_ctas = 0;
  const int split_env = option(WT_OPT_SVD_SPLIT);
  int n_sms = kNumSMs;
  if (persist) {
    int dev = 0, per_sm = 0;
    WT_CUDA(cudaGetDevice(&dev));
    int sms = 0;
    WT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    n_sms = sms;
    // (the dynamic shared-memory limit must be raised before the occupancy
    // query, or the first call in a process sees 0 resident CTAs)
    if (int e = ensure_smem(svd_sweep_kernel<1>, sizeof(PairSmem))) return e;
    WT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, svd_sweep_kernel<1>, kThreads, sizeof(PairSmem)));
    if (const int cap = option(WT_OPT_SVD_CTAS_PER_SM)) per_sm = std::min(per_sm, std::max(1, cap));
    sweep_ctas = sms * std::max(per_sm, 1);
  }
  g_last_sweeps = 0;
  g_last_rotations = 0;
  int dbg_prev = 0;
  static thread_local unsigned long long* d_prof = nullptr;  // WT_SVD_PROFILE diagnostics
  const bool profile = option(WT_OPT_SVD_PROFILE) != 0;
  if (profile) {
    if (!d_prof) WT_CUDA(cudaMalloc(&d_prof, 8 * sizeof(unsigned long long)));
    WT_CUDA(cudaMemsetAsync(d_prof, 0, 8 * sizeof(unsigned long long), st));
    ws.prof = d_prof;
  }
  static thread_local int* h_pending = nullptr;  // per host thread: concurrent calls on other streams
  if (!h_pending) WT_CUDA(cudaMallocHost(&h_pending, 2 * sizeof(int)));  // [pending, rotated visits]
  h_pending[0] = h_pending[1] = 0;
  const int nb = (int)(L.npad / HB);
  // One inner Jacobi sweep per pair visit: measured on the config-3/4 slices it
  // needs the same number of outer sweeps as full diagonalisation (13 / 18) at
  // 2.4x / 1.6x less time (tools/svd_probe.py, round 1).
  constexpr int inner = 1;
  bool hit_max = true;
  // Full rounds visit every block once with the full 32-column inner sweep
  // (all within-block pairs); the other rounds rotate (and test) only the
  // cross-block pairs, so every column pair is still covered at least once per
  // sweep with 16 instead of 31 eigen steps per visit.  Round 0 alone full
  // (round 1: 256 columns -9%, 1024 -3.5%, 384 (t-svd embeddings) -22%, 128
  // +5%, hence only from 16 blocks up) cost 1-4 extra sweeps: the cross
  // rotations disturb the within-block pairs for a whole sweep.  F = nb / 8
  // evenly spaced full rounds (2..4, round 0 and the last among them) win back
  // the sweeps (session 3, tools/svd_concurrency.py, ms / sweeps): config 3
  // 20.5 / 14 -> 18.6 / 12 (F = 2), config 4 158 / 16 -> 143 / 15 (F = 4),
  // the config-5 operators' pseudo-inverse pair 28.1 -> 24.2 (F = 4),
  // 4 x 1024^2 33.7 / 15 -> 31.2 / 13.
  const int cross = nb >= 16 ? std::max(2, std::min(4, nb / 8)) : 0;
  // Reorder the columns by descending norm before every sweep: measured on the
  // config-3/4 slices 13 -> 12 and 17 -> 16 sweeps, -10% time (round 1).
  constexpr int sort_mode = 2;
  // From sweep 1 on, sort by the column norms the visits leave behind (no
  // pass over the matrices).
  constexpr int visit_norms = 1;
  const size_t sort_smem = (size_t)npow2 * (sizeof(double) + sizeof(int));
  if (int e = ensure_smem(svd_norms_sort, 8192 * (sizeof(double) + sizeof(int)))) return e;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (sort_mode == 2 || (sort_mode == 1 && sweep == 0)) {
      // columns in descending norm order before the sweep (de Rijk-style)
      svd_norms_sort<<<(unsigned)n_active, 512, sort_smem, st>>>(ws, L.mpad, L.npad, L.n, npow2,
                                                              nullptr, nullptr, 0,
                                                              sweep > 0 && visit_norms ? 1 : 0);
      svd_permute_cols<<<dim3((unsigned)L.npad, (unsigned)n_active), 128, 0, st>>>(ws, L.mpad, L.npad);
      svd_flip<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(ws, (int)batch);
      if (int e = check_launch("svd reorder")) return e;
    }
    if (persist && n_active * (int64_t)(nb / 2) * (nb - 1) < (1ll << 30)) {  // int tickets
      WT_CUDA(cudaMemsetAsync(ws.bdone, 0, sizeof(int) * (size_t)batch * nb, st));
      WT_CUDA(cudaMemsetAsync(ws.ticket, 0, sizeof(int), st));
      const int64_t visits = n_active * (int64_t)(nb / 2) * (nb - 1);
      // Latency-bound sweeps (too few concurrent visits to fill the resident
      // CTA slots: few matrices, e.g. the 8-GPU share of config 4 or the
      // config-5 operator slices).  Two levers, measured on one B200 (round 1,
      // tools/svd_concurrency.py, ms):
      //  * resident CTAs per SM: just enough for one round's visits, so that a
      //    visit does not share its SM when it need not (the persistent grid
      //    otherwise parks idle CTAs next to running visits): 4 x 1024^2
      //    38.7 -> 33.5 at 1 CTA/SM, 16 x 512^2 19.7 -> 17.7 and 24 x 256^2
      //    5.52 -> 5.14 at 2;
      //  * cluster-split visits (rows over S CTAs, partial Grams summed in
      //    DSMEM) while every visit still has SMs to itself and each CTA keeps
      //    >= 128 rows: 1 x 512^2 12.96 (S = 1) -> 10.68 (S = 4), 1 CTA/SM.
      // Throughput-bound batches (configs 3 and 4 on one GPU) keep S = 1 and
      // all resident CTAs.  WT_SVD_SPLIT forces S, WT_SVD_CTAS_PER_SM caps k.
      const int64_t conc = n_active * (int64_t)(nb / 2);
      int split = 1;
      if (split_env > 0) split = split_env;
      else
        while (split < 8 && L.mpad / (2 * split) >= 128 && conc * split * 2 <= n_sms) split *= 2;
      while (split > 1 && split > L.mpad / RCH) split >>= 1;  // at least one row chunk per CTA
      split = split >= 8 ? 8 : split >= 4 ? 4 : split >= 2 ? 2 : 1;
      const int64_t per_sm_max = std::max<int64_t>(sweep_ctas / std::max(n_sms, 1), 1);
      const int64_t k_sm = std::min<int64_t>(std::max<int64_t>((conc * split + n_sms - 1) / n_sms, 1), per_sm_max);
      const int max_ctas = (int)std::max<int64_t>(n_sms * k_sm, split);
      int e = WT_OK;
      switch (split) {
        case 8: e = launch_sweep<8>(ws, L.mpad, L.npad, (int)n_active, tol, inner, cross, visits, max_ctas, st); break;
        case 4: e = launch_sweep<4>(ws, L.mpad, L.npad, (int)n_active, tol, inner, cross, visits, max_ctas, st); break;
        case 2: e = launch_sweep<2>(ws, L.mpad, L.npad, (int)n_active, tol, inner, cross, visits, max_ctas, st); break;
        default: e = launch_sweep<1>(ws, L.mpad, L.npad, (int)n_active, tol, inner, cross, visits, max_ctas, st);
      }
      if (e == WT_ERR_UNSUPPORTED)
        e = launch_sweep<1>(ws, L.mpad, L.npad, (int)n_active, tol, inner, cross, visits, max_ctas, st);
      if (e) return e;
    } else {
      for (int round = 0; round < nb - 1; ++round) {
        svd_pair_kernel<<<dim3(nb / 2, (unsigned)n_active), kThreads, sizeof(PairSmem), st>>>(
            ws, L.mpad, L.npad, round, tol, inner, cross_only_round(cross, round, nb));
      }
    }
    if (int e = check_launch("svd_pair_kernel")) return e;
    if (option(WT_OPT_SVD_TRACE)) {  // per-sweep convergence trace (diagnostics only)
      std::vector<unsigned long long> h(batch);
      WT_CUDA(cudaMemcpyAsync(h.data(), ws.offmax, sizeof(unsigned long long) * batch,
                              cudaMemcpyDeviceToHost, st));
      WT_CUDA(cudaStreamSynchronize(st));
      double mx = 0.0;
      int active = 0;
      for (auto v : h) {
        double d;
        memcpy(&d, &v, sizeof(d));
        mx = std::max(mx, d);
        active += d >= tol;
      }
      int rotated = 0;
      WT_CUDA(cudaMemcpy(&rotated, ws.pending + 1, sizeof(int), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[wt_svd] sweep %d: max off %.3e (tol %.1e), %d/%lld matrices above tol, "
              "%d/%lld pair visits rotated\n", sweep, mx, tol, active, (long long)batch,
              rotated - dbg_prev, (long long)(nb / 2) * (nb - 1) * batch);
      dbg_prev = rotated;
    }
    WT_CUDA(cudaMemsetAsync(ws.pending, 0, sizeof(int), st));
    svd_end_sweep<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(ws, (int)batch, tol);
    WT_CUDA(readback_ints(h_pending, ws.pending, 2, st));  // (not a copy-engine copy: wt_common.cuh)
    WT_CUDA(cudaStreamSynchronize(st));
    g_last_sweeps = sweep + 1;
    if (*h_pending == 0) { hit_max = false; break; }
    n_active = *h_pending;  // svd_end_sweep compacted the survivors into ws.active
  }
  {
    g_last_rotations = h_pending[1];  // read back with the last sweep's pending count
    g_last_panel_rows = L.mpad;
  }
  if (profile) {
    unsigned long long h[8];
    WT_CUDA(cudaMemcpyAsync(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost, st));
    WT_CUDA(cudaStreamSynchronize(st));
    const double n = h[3] ? (double)h[3] : 1.0;
    fprintf(stderr, "[wt_svd] %llu rotated pair visits; mean cycles per visit: gram+test %.0f, "
            "eigen %.0f, rotate %.0f (gram: stream %.0f, reduce %.0f, test %.0f)\n", h[3], h[0] / n,
            h[1] / n, h[2] / n, h[4] / n, h[5] / n, (h[0] - h[4] - h[5]) / n);
  }
  {
    const size_t sm = (size_t)npow2 * (sizeof(double) + sizeof(int));
    if (int e = ensure_smem(svd_norms_sort, 8192 * (sizeof(double) + sizeof(int)))) return e;
    svd_norms_sort<<<(unsigned)batch, 512, sm, st>>>(ws, L.mpad, L.npad, L.n, npow2, sigma, info,
                                                     hit_max ? 1 : 0);
    if (int e = check_launch("svd_norms_sort")) return e;
  }
  if (nvec > 0) {
    svd_gather<<<dim3((unsigned)nvec, (unsigned)batch), 256, 0, st>>>(ws, L.mpad, L.npad, L.m,
                                                                       nvec, vec);
    if (int e = check_launch("svd_gather")) return e;
    // The normalised columns of numerically-null singular values (s_j <= 1e-12 s_0) are rounding
    // noise -- the convergence floor leaves them wherever they are, even parallel to a real vector
    // (two parallel columns of a 12 x 3 slice: the truncated reconstruction counted that direction
    // twice; tools/fuzz_parity.py) -- so they are completed orthonormally here, for every consumer
    // (K5's projector, K6, K7, matrix_svd), as LAPACK's vectors are.  All-zero matrices are skipped
    // (config 5's 224 zero detail slices would each cost a 512-vector Gram-Schmidt: 188 ms; K6 and
    // matrix_svd, which hand vectors out, complete those themselves).
    const int64_t rfix = std::min<int64_t>(nvec, L.n);
    if (int e = ortho_fixup_strided(vec, L.m, rfix, 1, L.m, nvec * L.m, sigma, L.n, batch, 1e-12, st, 1)) return e;
  }
  return WT_OK;
}


// ------------------------------------------------------- leading triplets --
// The k leading singular triplets only (sp-w-svd needs no more: its result is
// the rank-r reconstruction of the coarse slices, decomposition.py:140-154):
// X V0 with V0 the k leading eigenvectors of X^T X (eig.cu), then the one-sided
// Jacobi on that m x k matrix.  Its columns span the leading singular subspace
// to eps ||X||^2 / (s_k^2 - s_{k+1}^2), so with k well above r the rank-r
// truncation is that of the full SVD (tested against LAPACK / the oracle);
// the sweeps run on k columns instead of n.
struct TopkLayout {
  WsLayout inner;
  int64_t m, n, mpad, npad, k;
  size_t off_X, off_scale, off_nz, off_eig, eig_bytes, off_X1, off_inner, total;
};

TopkLayout topk_layout(int64_t n1, int64_t n2, int64_t batch, int64_t k) {
  TopkLayout T{};
  T.m = std::max(n1, n2);
  T.n = std::min(n1, n2);
  T.k = k;
  T.mpad = round_up(std::max<int64_t>(T.m, 1), RCH);
  T.npad = round_up(std::max<int64_t>(T.n, 1), BW);
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) / 256 * 256; return r; };
  T.off_X = take(sizeof(double) * (size_t)(batch * T.npad * T.mpad));
  T.off_scale = take(sizeof(double) * (size_t)batch);
  T.off_nz = take(sizeof(int) * (size_t)batch);
  T.eig_bytes = eig_workspace_bytes(T.n, batch);
  T.off_eig = take(T.eig_bytes);
  T.off_X1 = take(sizeof(double) * (size_t)(batch * k * T.mpad));
  T.inner = ws_layout(k, T.m, batch, false);
  T.off_inner = take(T.inner.total);
  T.total = o;
  return T;
}

__global__ void svd_unscale(double* __restrict__ sigma, int64_t k, int64_t batch, const double* __restrict__ scale) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < batch * k; e += (int64_t)gridDim.x * blockDim.x)
    sigma[e] /= scale[e / k];
}

int jacobi_topk(const double* A, int64_t lda, int64_t strideA, int64_t n1, int64_t n2, int64_t batch, int64_t k,
                double* sigma, double* vec, int64_t nvec, int* info, double tol, int max_sweeps, void* workspace,
                size_t workspace_bytes, void* stream) {
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && batch >= 0, "svd_topk: bad shape");
  if (batch == 0) return WT_OK;
  const TopkLayout T = topk_layout(n1, n2, batch, k);
  WT_REQUIRE(k >= 1 && k <= T.n && nvec >= 0 && nvec <= k, "svd_topk: k = %lld, nvec = %lld for min(n1, n2) = %lld",
             (long long)k, (long long)nvec, (long long)T.n);
  WT_REQUIRE(T.n >= 3 && T.n <= 2048, "svd_topk: min(n1, n2) = %lld outside [3, 2048]", (long long)T.n);
  WT_REQUIRE(lda >= n2, "svd_topk: lda < n2");
  WT_REQUIRE(workspace != nullptr && workspace_bytes >= T.total, "svd_topk: workspace too small (%zu < %zu)",
             workspace_bytes, T.total);
  cudaStream_t st = (cudaStream_t)stream;
  char* base = static_cast<char*>(workspace);
  double* X = reinterpret_cast<double*>(base + T.off_X);
  double* scale = reinterpret_cast<double*>(base + T.off_scale);
  double* X1 = reinterpret_cast<double*>(base + T.off_X1);
  const bool right = n1 <= n2;
  int* nz = reinterpret_cast<int*>(base + T.off_nz);
  if (int e = absmax_scale(A, lda, strideA, n1, n2, batch, scale, st, nz)) return e;
  {
    dim3 grid((unsigned)std::min<int64_t>((T.npad * T.mpad + 255) / 256, 4096), (unsigned)batch);
    svd_copy_in<<<grid, 256, 0, st>>>(A, lda, strideA, right, T.m, T.n, T.mpad, T.npad, scale, X);
    if (int e = check_launch("svd_topk copy-in")) return e;
  }
  int fallback = 0;
  std::vector<int> hflags((size_t)batch, 1);
  if (int e = eig_precondition(X, X1, T.mpad, T.n, T.mpad, T.npad * T.mpad, batch, k, T.mpad, k * T.mpad,
                               base + T.off_eig, T.eig_bytes, &fallback, st, nz, hflags.data()))
    return e;
  // rows of X1 are the k columns of X V0: the Jacobi on that (k x m) row-major matrix,
  // right side: its long-side vectors are X's (A's long side), its sigma X V0's
  if (int e = jacobi(X1, T.mpad, k * T.mpad, k, T.m, batch, sigma, vec, nvec, info, tol, max_sweeps,
                     base + T.off_inner, T.inner.total, stream, false))
    return e;
  svd_unscale<<<(unsigned)std::min<int64_t>((batch * k + 255) / 256, 4096), 256, 0, st>>>(sigma, k, batch, scale);
  if (int e = check_launch("svd_topk unscale")) return e;
  if (fallback > 0) {
    // Matrices without a usable eigenbasis (numerically rank-deficient Grams whose
    // inverse-iteration vectors Newton-Schulz could not repair, all-zero slices):
    // I[:, :k] does not span their leading subspace, so they take the full SVD
    // (which starts its Jacobi from X itself) and keep its k leading values /
    // nvec leading vectors.  Rare: scratch comes from the stream-ordered allocator.
    const int64_t ln = T.m;
    const size_t wsb1 = ws_layout(n1, n2, 1).total;
    const size_t sig_b = (sizeof(double) * (size_t)T.n + 255) / 256 * 256;
    const size_t vec_b = (sizeof(double) * (size_t)(std::max<int64_t>(nvec, 1) * ln) + 255) / 256 * 256;
    char* tmp = nullptr;
    WT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sig_b + vec_b + 256 + wsb1, st));
    double* sig1 = reinterpret_cast<double*>(tmp);
    double* vec1 = reinterpret_cast<double*>(tmp + sig_b);
    int* info1 = reinterpret_cast<int*>(tmp + sig_b + vec_b);
    int rc = WT_OK;
    for (int64_t b = 0; b < batch && rc == WT_OK; ++b) {
      if (hflags[(size_t)b]) continue;
      rc = jacobi(A + b * strideA, lda, strideA, n1, n2, 1, sig1, vec1, nvec, info1, tol, max_sweeps,
                  tmp + sig_b + vec_b + 256, wsb1, stream, true);
      if (rc != WT_OK) break;
      cudaMemcpyAsync(sigma + b * k, sig1, sizeof(double) * (size_t)k, cudaMemcpyDeviceToDevice, st);
      if (nvec > 0)
        cudaMemcpyAsync(vec + b * nvec * ln, vec1, sizeof(double) * (size_t)(nvec * ln), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(info + b, info1, sizeof(int), cudaMemcpyDeviceToDevice, st);
    }
    cudaFreeAsync(tmp, st);
    if (rc != WT_OK) return rc;
  }
  g_last_fallbacks = fallback;
  return check_launch("svd_topk");
}
}  // namespace SVD_NS
}  // namespace wt
