// vba_small.cu — fp64 Cholesky solve of a small SPD system in one CTA (sm_100a).
//
// np.linalg.solve(Hred, -gred) (solver.py:287; loopclosure.py:534 via solver._solve_step)
// for reduced systems of up to kSmallMaxN unknowns: the tracker's windows, BASELINE configs
// 0-2 (n = 105, 225), small pose graphs.  The 128-tile DAG (vba_chol.cu) spends 0.1-0.25 ms
// there: each 128-column diagonal tile is a serial task and tasks hand over through global
// flags.  Here one CTA keeps the whole lower triangle in shared memory as 8 x 8 blocks
// (column-major inside a block, blocks in packed lower order: a 4-row quarter column is one
// aligned 32-byte run) and never leaves the SM:
//   per 8-column panel p:  thread 0 factors the 8 x 8 diagonal block and inverts it in
//   registers (diag8); a thread per row below multiplies its 8-entry panel row by the
//   inverse (L_rp = A_rp X_pp^T); the rank-8 trailing update runs in 4 x 4 register blocks on
//   all threads, the next diagonal block first so thread 0 can factor it (look-ahead) while
//   the others finish;
// then the blocked forward (L y = b) and backward (L^T x = y) substitutions with the
// diagonal inverses.  The system is padded to a multiple of 8 with identity rows.  fp64
// throughout, fixed operation order (deterministic); a non-positive pivot sets *status (the
// reference's "singular reduced pose system" retry path, as the DAG).
#include <cuda_runtime.h>

#include "vba_internal.cuh"

namespace vba {

constexpr int kSmallThreads = 512;
constexpr int kSmallMaxN = 232;   // 29 x 30 / 2 blocks of 512 B + 3 vectors: <= 227 KB of shared memory

__host__ __device__ __forceinline__ int sm_nblk(int np) { return (np / 8) * (np / 8 + 1) / 2; }
size_t chol_small_smem(int n) {
  const int np = (n + 7) / 8 * 8;
  return ((size_t)sm_nblk(np) * 64 + 2 * np + 64) * sizeof(double);
}

// block (R, C), R >= C, of the packed block-lower storage: 64 doubles, column-major in
// 16-byte units (2 rows of a column); the unit index is XOR-swizzled with the block index
// so that threads touching the same logical unit of different blocks hit different banks
__device__ __forceinline__ int sbid(int R, int C) { return (R * (R + 1)) / 2 + C; }
__device__ __forceinline__ double* sunit(double* S, int b, int u) { return S + b * 64 + ((u ^ (b & 7)) << 1); }
__device__ __forceinline__ double& sel(double* S, int b, int r8, int c8) {
  return sunit(S, b, c8 * 4 + (r8 >> 1))[r8 & 1];
}

// factor + invert the diagonal block (p, p) in registers: L overwrites it (zeros above),
// X = L^-1 (row-major) goes to Xs, 1 / L_jj to rinv
__device__ __forceinline__ void small_diag8(double* S, int p, double* Xs, double* rinv_g, int* bad) {
  const int b = sbid(p, p);
  double l[8][8], x[8][8], rinv[8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) l[r][c] = (r >= c) ? sel(S, b, r, c) : 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double d = l[j][j];
    if (!(d > 0.0)) { *bad = 1; d = 1.0; }
    const double rs = rsqrt(d);
    rinv[j] = rs;
    l[j][j] = d * rs;
#pragma unroll
    for (int r = j + 1; r < 8; ++r) l[r][j] *= rs;
#pragma unroll
    for (int c = j + 1; c < 8; ++c)
#pragma unroll
      for (int r = c; r < 8; ++r) l[r][c] = fma(-l[r][j], l[c][j], l[r][c]);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < c) { x[r][c] = 0.0; continue; }
      double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int m = c; m < r; ++m) s = fma(-l[r][m], x[m][c], s);
      x[r][c] = s * rinv[r];
    }
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      // lower: L;  upper (r < c): X[c][r] = (L^-1)[c][r], kept for the substitutions
      sel(S, b, r, c) = r >= c ? l[r][c] : x[c][r];
      Xs[r * 8 + c] = x[r][c];
    }
#pragma unroll
  for (int j = 0; j < 8; ++j) rinv_g[8 * p + j] = rinv[j];
}

// quarter (rows 4 u0.., cols 4 v0..) of block (R, C) -= L_Rp L_Cp^T   (rank 8)
__device__ __forceinline__ void small_upd(double* S, int p, int R, int C, int u0, int v0) {
  const int bR = sbid(R, p), bC = sbid(C, p), bT = sbid(R, C);
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const double2 r01 = *reinterpret_cast<const double2*>(sunit(S, bR, m * 4 + 2 * u0));
    const double2 r23 = *reinterpret_cast<const double2*>(sunit(S, bR, m * 4 + 2 * u0 + 1));
    const double2 c01 = *reinterpret_cast<const double2*>(sunit(S, bC, m * 4 + 2 * v0));
    const double2 c23 = *reinterpret_cast<const double2*>(sunit(S, bC, m * 4 + 2 * v0 + 1));
    const double rv[4] = {r01.x, r01.y, r23.x, r23.y}, cv[4] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fma(rv[u], cv[v], acc[u][v]);
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int col = 4 * v0 + v;
    double2* d0 = reinterpret_cast<double2*>(sunit(S, bT, col * 4 + 2 * u0));
    double2* d1 = reinterpret_cast<double2*>(sunit(S, bT, col * 4 + 2 * u0 + 1));
    double2 a = *d0, b = *d1;
    a.x -= acc[0][v]; a.y -= acc[1][v]; b.x -= acc[2][v]; b.y -= acc[3][v];
    *d0 = a;
    *d1 = b;
  }
}

// work item q of the trailing update over the lower blocks of [p0, nb): block q / 4 in
// packed row order (rb >= cb), quarter q % 4 = (u, v); the upper quarter of a diagonal
// block (u = 0, v = 1) is skipped by the caller
__device__ __forceinline__ void small_quarter(int q, int p0, int& R, int& C, int& u, int& v) {
  const int bb = q >> 2, qq = q & 3;
  int rb = (int)((sqrtf(8.f * (float)bb + 1.f) - 1.f) * 0.5f);
  while ((rb + 1) * (rb + 2) / 2 <= bb) ++rb;
  while (rb * (rb + 1) / 2 > bb) --rb;
  R = p0 + rb;
  C = p0 + bb - rb * (rb + 1) / 2;
  u = qq >> 1;
  v = qq & 1;
}

__global__ void __launch_bounds__(kSmallThreads, 1) k_chol_small(const double* __restrict__ H, int64_t ld, int n,
                                                                 const double* __restrict__ rhs,
                                                                 double* __restrict__ x, int* __restrict__ status) {
  extern __shared__ __align__(16) double S[];
  const int np = (n + 7) / 8 * 8, nb = np / 8;
  double* y = S + (size_t)sm_nblk(np) * 64;
  double* rinv = y + np;     // 1 / L_jj
  double* Xs = rinv + np;    // 8 x 8 inverse of the current diagonal block
  __shared__ int bad;
  const int tid = threadIdx.x, nth = blockDim.x;
  if (tid == 0) bad = 0;
  // lower triangle of the column-major H into the blocks (identity padding); consecutive
  // threads along a column: coalesced reads
  for (int c = tid >> 5; c < np; c += nth >> 5)
    for (int r = c + (tid & 31); r < np; r += 32) {
      const double v = (r < n && c < n) ? H[(int64_t)c * ld + r] : (r == c ? 1.0 : 0.0);
      sel(S, sbid(r >> 3, c >> 3), r & 7, c & 7) = v;
    }
  for (int r = tid; r < np; r += nth) y[r] = r < n ? rhs[r] : 0.0;
  __syncthreads();
  if (tid == 0) small_diag8(S, 0, Xs, rinv, &bad);
  __syncthreads();
  for (int p = 0; p < nb; ++p) {
    // rows below the diagonal block: L_rp = A_rp X_pp^T (a row per thread)
    const int nr = np - 8 * (p + 1);
    for (int t = tid; t < nr; t += nth) {
      const int r = 8 * (p + 1) + t, b = sbid(r / 8, p), r8 = r % 8;
      double a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = sel(S, b, r8, m);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m <= c; ++m) s = fma(a[m], Xs[c * 8 + m], s);
        sel(S, b, r8, c) = s;
      }
    }
    __syncthreads();
    if (nr == 0) break;
    // trailing update, the next diagonal block's 3 quarters first (warp 0), then thread 0
    // factors it while the other warps finish the rest
    const int m = nb - p - 1, nq = 4 * m * (m + 1) / 2;
    if (tid < 32) {
      if (tid < 3) small_upd(S, p, p + 1, p + 1, tid == 0 ? 0 : 1, tid == 2 ? 1 : 0);
      __syncwarp();
      if (tid == 0) small_diag8(S, p + 1, Xs, rinv, &bad);
    } else {
      for (int q = 4 + tid - 32; q < nq; q += nth - 32) {   // block 0 = the next diagonal block
        int R, C, u, v;
        small_quarter(q, p + 1, R, C, u, v);
        if (R == C && u < v) continue;
        small_upd(S, p, R, C, u, v);
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *status = 1;
    return;
  }
  // forward substitution L y = b by 8-row blocks: y_p = X_pp (b_p - ...) with the inverse
  // kept in the diagonal block (8 threads, a row each), then the rows below
  for (int p = 0; p < nb; ++p) {
    const int b = sbid(p, p);
    double yr = 0.0;
    if (tid < 8) {
      yr = rinv[8 * p + tid] * y[8 * p + tid];
      for (int m = 0; m < tid; ++m) yr = fma(sel(S, b, m, tid), y[8 * p + m], yr);   // X[tid][m] at (m, tid)
    }
    __syncthreads();
    if (tid < 8) y[8 * p + tid] = yr;
    __syncthreads();
    for (int r = 8 * (p + 1) + tid; r < np; r += nth) {
      const int bl = sbid(r / 8, p), r8 = r % 8;
      double s = y[r];
#pragma unroll
      for (int m = 0; m < 8; ++m) s = fma(-sel(S, bl, r8, m), y[8 * p + m], s);
      y[r] = s;
    }
    __syncthreads();
  }
  // backward substitution L^T x = y: x_p = X_pp^T (y_p - ...), then the rows above
  for (int p = nb - 1; p >= 0; --p) {
    const int b = sbid(p, p);
    double xr = 0.0;
    if (tid < 8) {
      xr = rinv[8 * p + tid] * y[8 * p + tid];
      for (int m = tid + 1; m < 8; ++m) xr = fma(sel(S, b, tid, m), y[8 * p + m], xr);   // X[m][tid] at (tid, m)
    }
    __syncthreads();
    if (tid < 8) y[8 * p + tid] = xr;
    __syncthreads();
    for (int c = tid; c < 8 * p; c += nth) {   // y_c -= sum_m L[8p + m][c] x_{8p + m}
      const int bl = sbid(p, c / 8), c8 = c % 8;
      double s = y[c];
#pragma unroll
      for (int m = 0; m < 8; ++m) s = fma(-sel(S, bl, m, c8), y[8 * p + m], s);
      y[c] = s;
    }
    __syncthreads();
  }
  for (int r = tid; r < n; r += nth) x[r] = y[r];
}

int chol_small_solve(const double* H, int64_t ld, int n, const double* rhs, double* x, int* status, cudaStream_t st) {
  if (n <= 0 || n > kSmallMaxN) return 1;
  const size_t smem = chol_small_smem(n);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_chol_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_small_smem(kSmallMaxN));
    init = true;
  }
  k_chol_small<<<1, kSmallThreads, smem, st>>>(H, ld, n, rhs, x, status);
  launch_count();
  return 0;
}

}  // namespace vba
