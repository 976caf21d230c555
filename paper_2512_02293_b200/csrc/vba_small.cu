// vba_small.cu — fp64 Cholesky solve of a small SPD system in one CTA (sm_100a).
//
// np.linalg.solve(Hred, -gred) (solver.py:287) for reduced systems of a few hundred unknowns
// -- the tracker's windows, BASELINE configs 0-2 (n = 105, 225), small pose graphs.  The
// tile-DAG Cholesky (vba_chol.cu) spends ~0.1-0.25 ms there on its chain of 128-tile tasks
// handed between CTAs through global flags; here one CTA holds the packed lower
// triangle in shared memory (n <= kSmallN: n(n+1)/2 + n doubles <= 227 KB) and runs a
// right-looking blocked factorisation without leaving the SM (512 threads):
//   per 32-column panel: warp 0 factors the diagonal block (lane = row, the pivot column
//   broadcast by shuffles); the rows below solve against it (a row per thread, the diagonal
//   block read as a shared-memory broadcast); the trailing triangle takes the rank-32 update
//   in 4x4 register blocks (all warps);
// then the forward and backward substitutions in the same blocking.  fp64 throughout, fixed
// operation order (deterministic); a non-positive pivot sets *status (the reference's
// "singular reduced pose system" retry path).
#include <cuda_runtime.h>

#include "vba_internal.cuh"

namespace vba {

constexpr int kSmallThreads = 512;   // 128 registers per thread for the 32-wide row blocks

__device__ __forceinline__ int pidx(int r, int c) { return r * (r + 1) / 2 + c; }   // packed lower, row-major

__global__ void __launch_bounds__(kSmallThreads) k_chol_small(const double* __restrict__ H, int64_t ld, int n,
                                                              const double* __restrict__ rhs, double* __restrict__ x,
                                                              int* __restrict__ status) {
  extern __shared__ double S[];
  double* y = S + n * (n + 1) / 2;
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kSmallThreads / 32;
  if (tid == 0) bad = 0;
  // lower triangle of the column-major H: a warp per column, coalesced along its rows
  for (int c = warp; c < n; c += nw)
    for (int r = c + lane; r < n; r += 32) S[pidx(r, c)] = H[(int64_t)c * ld + r];
  for (int r = tid; r < n; r += kSmallThreads) y[r] = rhs[r];
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int b = min(32, n - c0);
    // 1. diagonal block: lane = row c0 + lane, a[c] = A[c0 + lane][c0 + c]
    if (warp == 0) {
      double a[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = (lane < b && c <= lane) ? S[pidx(c0 + lane, c0 + c)] : 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < b) {
          double d = __shfl_sync(0xffffffffu, a[j], j);
          if (!(d > 0.0)) {
            if (lane == 0) bad = 1;
            d = 1.0;
          }
          const double ljj = sqrt(d);
          const double lj = lane == j ? ljj : (lane > j ? a[j] / ljj : 0.0);
          a[j] = lj;
#pragma unroll
          for (int c = j + 1; c < 32; ++c) {
            const double lc = __shfl_sync(0xffffffffu, lj, c);
            if (lane >= c) a[c] = fma(-lj, lc, a[c]);
          }
        }
      }
      if (lane < b)
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c <= lane) S[pidx(c0 + lane, c0 + c)] = a[c];
    }
    __syncthreads();
    const int r0 = c0 + b, m = n - r0;
    if (m <= 0) break;
    // 2. panel rows below: L[r][c0 + c] = (A[r][c0 + c] - sum_{k<c} L[r][c0 + k] L[c0 + c][c0 + k]) / L_cc
    for (int t = tid; t < m; t += kSmallThreads) {
      const int r = r0 + t;
      double v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = c < b ? S[pidx(r, c0 + c)] : 0.0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c < b) {
          double s = v[c];
#pragma unroll
          for (int k = 0; k < c; ++k) s = fma(-v[k], S[pidx(c0 + c, c0 + k)], s);
          v[c] = s / S[pidx(c0 + c, c0 + c)];
        }
      }
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < b) S[pidx(r, c0 + c)] = v[c];
    }
    __syncthreads();
    // 3. trailing update A[r][c] -= sum_k L[r][c0 + k] L[c][c0 + k], r >= c >= r0, in 4x4 blocks
    const int nb = (m + 3) / 4, nblk = nb * (nb + 1) / 2;
    for (int q = tid; q < nblk; q += kSmallThreads) {
      int rb = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
      while ((rb + 1) * (rb + 2) / 2 <= q) ++rb;
      while (rb * (rb + 1) / 2 > q) --rb;
      const int cb = q - rb * (rb + 1) / 2;
      const int rr = r0 + 4 * rb, cc = r0 + 4 * cb;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] = 0.0;
      for (int k = 0; k < b; ++k) {
        double lr[4], lc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          lr[u] = rr + u < n ? S[pidx(rr + u, c0 + k)] : 0.0;
          lc[u] = cc + u < n ? S[pidx(cc + u, c0 + k)] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) acc[u][w] = fma(lr[u], lc[w], acc[u][w]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int r = rr + u, c = cc + w;
          if (r < n && c <= r) S[pidx(r, c)] -= acc[u][w];
        }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *status = 1;
    return;
  }
  // forward substitution L y = b, 32-row blocks
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int b = min(32, n - c0);
    if (warp == 0) {
      double yi = lane < b ? y[c0 + lane] : 0.0;
      for (int j = 0; j < b; ++j) {
        const double yj = __shfl_sync(0xffffffffu, yi, j) / S[pidx(c0 + j, c0 + j)];
        if (lane == j) yi = yj;
        else if (lane > j && lane < b) yi = fma(-S[pidx(c0 + lane, c0 + j)], yj, yi);
      }
      if (lane < b) y[c0 + lane] = yi;
    }
    __syncthreads();
    for (int r = c0 + b + tid; r < n; r += kSmallThreads) {
      double s = y[r];
      for (int k = 0; k < b; ++k) s = fma(-S[pidx(r, c0 + k)], y[c0 + k], s);
      y[r] = s;
    }
    __syncthreads();
  }
  // backward substitution L^T x = y, 32-row blocks from the end
  const int nblocks = (n + 31) / 32;
  for (int blk = nblocks - 1; blk >= 0; --blk) {
    const int c0 = 32 * blk, b = min(32, n - c0);
    if (warp == 0) {
      double xi = lane < b ? y[c0 + lane] : 0.0;
      for (int j = b - 1; j >= 0; --j) {
        const double xj = __shfl_sync(0xffffffffu, xi, j) / S[pidx(c0 + j, c0 + j)];
        if (lane == j) xi = xj;
        else if (lane < j) xi = fma(-S[pidx(c0 + j, c0 + lane)], xj, xi);
      }
      if (lane < b) y[c0 + lane] = xi;
    }
    __syncthreads();
    for (int r = tid; r < c0; r += kSmallThreads) {
      double s = y[r];
      for (int k = 0; k < b; ++k) s = fma(-S[pidx(c0 + k, r)], y[c0 + k], s);
      y[r] = s;
    }
    __syncthreads();
  }
  for (int r = tid; r < n; r += kSmallThreads) x[r] = y[r];
}

size_t chol_small_smem(int n) { return sizeof(double) * ((size_t)n * (n + 1) / 2 + (size_t)n); }

// Solves H x = b for n <= kSmallN (column-major H, leading dimension ld, lower triangle read);
// *status = 1 on a non-positive pivot.  Returns 1 (nothing launched) when n is too large.
int chol_small_solve(const double* H, int64_t ld, int n, const double* b, double* x, int* status, cudaStream_t st) {
  if (n <= 0) return 0;
  if (n > kSmallN) return 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_chol_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_small_smem(kSmallN));
    attr = true;
  }
  k_chol_small<<<1, kSmallThreads, chol_small_smem(n), st>>>(H, ld, n, b, x, status);
  launch_count();
  return 0;
}

}  // namespace vba
