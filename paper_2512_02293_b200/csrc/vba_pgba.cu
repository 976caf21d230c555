// vba_pgba.cu — Sim(3) pose-graph bundle adjustment (PGBA) on the GPU.
//
// Replaces vislam.loopclosure.solve_pgba (/root/reference/pkg/src/vislam/loopclosure.py:502-574)
// and its callees: total_pg_energy (:378-390), _PgLayout (:392-422), _linearize_pg (:425-475),
// _pg_apply (:489-499), the factors sim3_vision_residual (:225-307) and relative_pose_residual
// (residuals.py:364-380), the Sim(3) maps (geometry.py:230-370), and the shared damped Schur
// step solver._solve_step (loopclosure.py:27,534; solver.py:265-308).
//
// A pose graph is small next to a VI-BA window (hundreds of Sim(3) nodes, a handful of dense
// loop edges), so every factor is evaluated in fp64 -- no fp32 per-pixel stage -- and the
// path is latency-bound, not HBM-bound:
//   P1 k_pg_pixel    one thread per loop-edge pixel: the sqrt(w)-scaled rows
//                    [J_i (7) | J_j (7) | r | J_d] of both image components (fp64)
//   P2 k_pg_gram     one CTA per loop edge: the 15x15 Gram of [J_i | J_j | r] over its pixels
//                    in a fixed order -> H_ii, H_jj, H_ij, g_i, g_j, energy (fp64)
//   P3 k_pg_rel      one thread per relative edge: whitened Sim(3) log residual, J_i = W Jr^-1(r)
//                    Ad(S_j), J_j = -J_i (exact Jr^-1 via the block exponential, as the reference)
//   P4 k_pg_fill     one CTA per loop source: per-pixel Schur elimination of its disparities,
//                    F = sum_n u_n u_n^T / h_n, b = sum_n u_n g_n / h_n over its pose blocks
//   assembly         the shared block planner (vba_plan.h, k_assemble): damping, fill-in
//   solve            the shared reduced solve (fp64 tile-DAG Cholesky, or the tcgen05 split-fp16
//                    factor + fp64 refinement from 4 tiles up, vba_chol.cu)
//   P5 k_pg_backsub  per pixel dx_d = (-g_n - u_n . dx) / h_n, disparity floor (fp64)
//   P6 k_pg_retract  S <- S Exp(dx) for every free node (node 0 is the gauge)
// All sums have a fixed order: the solve is bitwise deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "vba_internal.cuh"
#include "vba_plan.h"

namespace vba {

constexpr int kPgRow = 32;      // doubles per pixel row record: 2 x (J_i 7, J_j 7, r, J_d)
constexpr int kPgRec = 168;     // doubles per factor record: Hii 49, Hjj 49, Hij 49, gi 7, gj 7, e 1 (+pad)
constexpr int kPgMaxPoses = 8;  // pose blocks per loop source (the source + distinct targets)
constexpr int kPgChunk = 32;    // pixels staged per step in k_pg_gram / k_pg_fill

struct PgGeo {     // per-thread constants of one loop edge
  double Rbc[9], pbc[3];
};

// ---------------------------------------------------------------------------
// fp64 Sim(3) helpers (geometry.py:230-370).  A state is q wxyz, t, s.
// ---------------------------------------------------------------------------
__device__ void sim3_wmat(const double* w, double sigma, double* W) {   // geometry.py:230-263
  const double theta = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9], K2[9];
  hat3(w, K);
  mat3_mul(K, K, K2);
  const double s = exp(sigma), eps = 1e-6;
  double A, B, C;
  if (fabs(sigma) < eps) {
    C = 1.0;
    if (theta < eps) {
      A = 0.5;
      B = 1.0 / 6.0;
    } else {
      const double t2 = theta * theta;
      A = (1.0 - cos(theta)) / t2;
      B = (theta - sin(theta)) / (t2 * theta);
    }
  } else {
    C = (s - 1.0) / sigma;
    if (theta < eps) {
      const double s2 = sigma * sigma;
      A = ((sigma - 1.0) * s + 1.0) / s2;
      B = (s * (0.5 * s2 - sigma + 1.0) - 1.0) / (s2 * sigma);
    } else {
      const double t2 = theta * theta, d = sigma * sigma + t2;
      A = (s * sigma * sin(theta) + theta * (1.0 - s * cos(theta))) / (theta * d);
      B = (C - ((s * cos(theta) - 1.0) * sigma + s * sin(theta) * theta) / d) / t2;
    }
  }
  for (int k = 0; k < 9; ++k) W[k] = A * K[k] + B * K2[k];
  W[0] += C;
  W[4] += C;
  W[8] += C;
}

// Gaussian elimination with partial pivoting, n <= 7 (row-major A[n*n], b[n] -> x[n]);
// the LAPACK gesv algorithm np.linalg.solve uses, without blocking.
__device__ void small_solve(double* A, double* b, int n) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int r = k + 1; r < n; ++r)
      if (fabs(A[r * n + k]) > fabs(A[p * n + k])) p = r;
    if (p != k) {
      for (int c = 0; c < n; ++c) {
        const double t = A[k * n + c];
        A[k * n + c] = A[p * n + c];
        A[p * n + c] = t;
      }
      const double t = b[k];
      b[k] = b[p];
      b[p] = t;
    }
    for (int r = k + 1; r < n; ++r) {
      const double f = A[r * n + k] / A[k * n + k];
      for (int c = k; c < n; ++c) A[r * n + c] -= f * A[k * n + c];
      b[r] -= f * b[k];
    }
  }
  for (int k = n - 1; k >= 0; --k) {
    double v = b[k];
    for (int c = k + 1; c < n; ++c) v -= A[k * n + c] * b[c];
    b[k] = v / A[k * n + k];
  }
}

// inverse of a 7x7 (Gauss-Jordan, partial pivoting); M is destroyed
__device__ void inv7(double* M, double* X) {
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) X[r * 7 + c] = r == c ? 1.0 : 0.0;
  for (int k = 0; k < 7; ++k) {
    int p = k;
    for (int r = k + 1; r < 7; ++r)
      if (fabs(M[r * 7 + k]) > fabs(M[p * 7 + k])) p = r;
    if (p != k)
      for (int c = 0; c < 7; ++c) {
        double t = M[k * 7 + c]; M[k * 7 + c] = M[p * 7 + c]; M[p * 7 + c] = t;
        t = X[k * 7 + c]; X[k * 7 + c] = X[p * 7 + c]; X[p * 7 + c] = t;
      }
    const double iv = 1.0 / M[k * 7 + k];
    for (int c = 0; c < 7; ++c) {
      M[k * 7 + c] *= iv;
      X[k * 7 + c] *= iv;
    }
    for (int r = 0; r < 7; ++r) {
      if (r == k) continue;
      const double f = M[r * 7 + k];
      if (f == 0.0) continue;
      for (int c = 0; c < 7; ++c) {
        M[r * 7 + c] -= f * M[k * 7 + c];
        X[r * 7 + c] -= f * X[k * 7 + c];
      }
    }
  }
}

__device__ void mat7_mul(const double* A, const double* B, double* C) {
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) {
      double v = 0.0;
      for (int k = 0; k < 7; ++k) v += A[r * 7 + k] * B[k * 7 + c];
      C[r * 7 + c] = v;
    }
}

// Jr^-1(xi) = phi(-ad_xi)^-1 with phi(A) = int_0^1 exp(A s) ds (geometry.py:357-370): scaling and
// squaring on the pair (E = exp(A), P = phi(A)) -- phi(2A) = P (E + I) / 2, exp(2A) = E^2 --
// from degree-16 Taylor series at A / 2^k (||A / 2^k|| <= 1/4).
__device__ void sim3_jr_inv(const double* xi, double* out) {
  double A[49];
  for (int k = 0; k < 49; ++k) A[k] = 0.0;
  const double *om = xi, *up = xi + 3, sg = xi[6];
  // -ad_xi (geometry.py:344-354)
  double H[9], U[9];
  hat3(om, H);
  hat3(up, U);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      A[r * 7 + c] = -H[r * 3 + c];
      A[(3 + r) * 7 + c] = -U[r * 3 + c];
      A[(3 + r) * 7 + 3 + c] = -(H[r * 3 + c] + (r == c ? sg : 0.0));
    }
  for (int r = 0; r < 3; ++r) A[(3 + r) * 7 + 6] = up[r];
  double nrm = 0.0;
  for (int r = 0; r < 7; ++r) {
    double s = 0.0;
    for (int c = 0; c < 7; ++c) s += fabs(A[r * 7 + c]);
    nrm = fmax(nrm, s);
  }
  int sq = 0;
  while (nrm > 0.25 && sq < 60) {
    nrm *= 0.5;
    ++sq;
  }
  const double sc = ldexp(1.0, -sq);
  for (int k = 0; k < 49; ++k) A[k] *= sc;
  // E = sum A^k / k!, P = sum A^k / (k+1)!  (Horner)
  double E[49], P[49], T[49];
  for (int k = 0; k < 49; ++k) E[k] = P[k] = 0.0;
  const int deg = 16;
  // P = I/1! + A/2! + A^2/3! + ...  via Horner: P = (I + A/(2) (I + A/3 (I + ...)))
  for (int k = 0; k < 7; ++k) P[k * 8] = 1.0;
  for (int m = deg; m >= 1; --m) {   // P <- I + A P / (m + 1)
    mat7_mul(A, P, T);
    for (int k = 0; k < 49; ++k) P[k] = T[k] / (double)(m + 1) + ((k % 8 == 0) ? 1.0 : 0.0);
  }
  // E = I + A P
  mat7_mul(A, P, E);
  for (int k = 0; k < 7; ++k) E[k * 8] += 1.0;
  for (int s = 0; s < sq; ++s) {
    for (int k = 0; k < 49; ++k) T[k] = E[k] + ((k % 8 == 0) ? 1.0 : 0.0);
    double P2[49];
    mat7_mul(P, T, P2);
    for (int k = 0; k < 49; ++k) P[k] = 0.5 * P2[k];
    mat7_mul(E, E, T);
    for (int k = 0; k < 49; ++k) E[k] = T[k];
  }
  inv7(P, out);
}

__device__ void s_compose(const double* a, const double* b, double* o) {   // geometry.py:296-301
  double R[9], t[3], q[4];
  qmat(a, R);
  mat3_vec(R, b + 4, t);
  qmul(a, b, q);
  qcanon(q);
  for (int k = 0; k < 4; ++k) o[k] = q[k];
  for (int k = 0; k < 3; ++k) o[4 + k] = a[7] * t[k] + a[4 + k];
  o[7] = a[7] * b[7];
}

__device__ void s_inverse(const double* a, double* o) {   // geometry.py:306-309
  double q[4] = {a[0], -a[1], -a[2], -a[3]};
  qcanon(q);
  double R[9], t[3];
  qmat(q, R);
  mat3_vec(R, a + 4, t);
  const double is = 1.0 / a[7];
  for (int k = 0; k < 4; ++k) o[k] = q[k];
  for (int k = 0; k < 3; ++k) o[4 + k] = -is * t[k];
  o[7] = is;
}

__device__ void s_log(const double* a, double* xi) {   // geometry.py:319-324
  qlog(a, xi);
  xi[6] = log(a[7]);
  double W[9], b[3] = {a[4], a[5], a[6]};
  sim3_wmat(xi, xi[6], W);
  small_solve(W, b, 3);
  xi[3] = b[0];
  xi[4] = b[1];
  xi[5] = b[2];
}

__device__ void s_exp(const double* xi, double* o) {   // geometry.py:311-317
  qexp(xi, o);
  double W[9];
  sim3_wmat(xi, xi[6], W);
  mat3_vec(W, xi + 3, o + 4);
  o[7] = exp(xi[6]);
}

__device__ void s_adjoint(const double* a, double* A) {   // geometry.py:329-339
  double R[9], H[9], HR[9];
  qmat(a, R);
  hat3(a + 4, H);
  mat3_mul(H, R, HR);
  for (int k = 0; k < 49; ++k) A[k] = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      A[r * 7 + c] = R[r * 3 + c];
      A[(3 + r) * 7 + c] = HR[r * 3 + c];
      A[(3 + r) * 7 + 3 + c] = a[7] * R[r * 3 + c];
    }
  for (int r = 0; r < 3; ++r) A[(3 + r) * 7 + 6] = -a[4 + r];
  A[48] = 1.0;
}

// ---------------------------------------------------------------------------
// P1: per-pixel rows of the loop vision factor (loopclosure.py:225-307), fp64
// ---------------------------------------------------------------------------
__global__ void k_pg_pixel(const int32_t* __restrict__ pix_edge, const int32_t* __restrict__ vi,
                           const int32_t* __restrict__ vj, const int64_t* __restrict__ voff,
                           const int64_t* __restrict__ doff, const double* __restrict__ state,
                           const double* __restrict__ disp, const double* __restrict__ pix,
                           const double* __restrict__ tgt, const double* __restrict__ wts, int64_t nrows,
                           double fx, double fy, double cx, double cy, PgGeo x, double* __restrict__ rows) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nrows) return;
  const int e = pix_edge[g];
  const int i = vi[e], j = vj[e];
  const int64_t n = g - voff[e];
  const double* Si = state + 8 * i;
  const double* Sj = state + 8 * j;
  const double d = disp[doff[i] + n];
  const double u = pix[2 * (doff[i] + n)], v = pix[2 * (doff[i] + n) + 1];
  double Ri[9], Rj[9];
  qmat(Si, Ri);
  qmat(Sj, Rj);
  const double s_i = Si[7], s_j = Sj[7];
  // backproject (residuals.py:81-87), chain of loopclosure.py:245-249
  const double z = 1.0 / d;
  const double Xi[3] = {(u - cx) / fx * z, (v - cy) / fy * z, z};
  double Yi[3], t3[3], Xw[3], Vj[3], Xc[3];
  mat3_vec(x.Rbc, Xi, Yi);
  for (int k = 0; k < 3; ++k) Yi[k] += x.pbc[k];
  mat3_vec(Ri, Yi, t3);
  for (int k = 0; k < 3; ++k) Xw[k] = s_i * t3[k] + Si[4 + k];
  for (int k = 0; k < 3; ++k) t3[k] = Xw[k] - Sj[4 + k];
  mat3T_vec(Rj, t3, Vj);
  for (int k = 0; k < 3; ++k) Vj[k] /= s_j;
  for (int k = 0; k < 3; ++k) t3[k] = Vj[k] - x.pbc[k];
  mat3T_vec(x.Rbc, t3, Xc);
  const bool valid = Xc[2] > 1e-6;
  const double zs = valid ? Xc[2] : 1.0;
  const double pu = fx * Xc[0] / zs + cx, pv = fy * Xc[1] / zs + cy;
  const double r0 = tgt[2 * (voff[e] + n)] - pu, r1 = tgt[2 * (voff[e] + n) + 1] - pv;
  const double P00 = fx / zs, P02 = -fx * Xc[0] / (zs * zs), P11 = fy / zs, P12 = -fy * Xc[1] / (zs * zs);
  // B = R_bc^T R_j^T / s_j, BRi = B R_i  (loopclosure.py:271-272)
  double RbcTRjT[9], B[9], BRi[9];
  double RbcT[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) RbcT[a * 3 + b] = x.Rbc[b * 3 + a];
  mat3_mulT(RbcT, Rj, RbcTRjT);
  for (int k = 0; k < 9; ++k) B[k] = RbcTRjT[k] / s_j;
  mat3_mul(B, Ri, BRi);
  // dX_c / d(theta_i, p_i, s_i), d(theta_j, p_j, s_j), d(d)
  double D[3][15];
  {
    double Hy[9], M1[9];
    hat3(Yi, Hy);
    mat3_mul(BRi, Hy, M1);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        D[a][b] = -s_i * M1[a * 3 + b];
        D[a][3 + b] = s_i * BRi[a * 3 + b];
      }
    double BY[3];
    mat3_vec(BRi, Yi, BY);
    for (int a = 0; a < 3; ++a) D[a][6] = s_i * BY[a];
    double Hv[9], M2[9];
    hat3(Vj, Hv);
    mat3_mul(RbcT, Hv, M2);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        D[a][7 + b] = M2[a * 3 + b];
        D[a][10 + b] = -RbcT[a * 3 + b];
      }
    double RV[3];
    mat3_vec(RbcT, Vj, RV);
    for (int a = 0; a < 3; ++a) D[a][13] = -RV[a];
    double C[9], CX[3];
    mat3_mul(BRi, x.Rbc, C);
    mat3_vec(C, Xi, CX);
    for (int a = 0; a < 3; ++a) D[a][14] = -s_i * CX[a] / d;
  }
  const double w0 = valid ? wts[2 * (voff[e] + n)] : 0.0, w1 = valid ? wts[2 * (voff[e] + n) + 1] : 0.0;
  const double sw0 = sqrt(w0), sw1 = sqrt(w1);
  double* o = rows + (int64_t)kPgRow * g;
  // row c: [J_i (7) | J_j (7) | r | J_d], J = -P dX_c, scaled by sqrt(w_c)
  for (int k = 0; k < 14; ++k) {
    o[k] = -sw0 * (P00 * D[0][k] + P02 * D[2][k]);
    o[16 + k] = -sw1 * (P11 * D[1][k] + P12 * D[2][k]);
  }
  o[14] = sw0 * r0;
  o[30] = sw1 * r1;
  o[15] = -sw0 * (P00 * D[0][14] + P02 * D[2][14]);
  o[31] = -sw1 * (P11 * D[1][14] + P12 * D[2][14]);
}

// ---------------------------------------------------------------------------
// P2: per loop edge, the 15x15 Gram of [J_i | J_j | r] (fixed pixel order) -> factor record
// ---------------------------------------------------------------------------
constexpr int kPgRange = 256;   // pixels (rows) per CTA of k_pg_gram / k_pg_fill: partials summed in order

// partial Grams: CTA (range x, edge y) over rows [r0 + x kPgRange, ...): 120 upper entries
// (energy only: 1) to part[(y * nrng + x) * 120]
__global__ void __launch_bounds__(128) k_pg_gram(const int64_t* __restrict__ voff, const double* __restrict__ rows,
                                                 int energy_only, int nrng, double* __restrict__ part) {
  __shared__ double S[kPgChunk][kPgRow + 1];
  const int e = blockIdx.y, tid = threadIdx.x;
  const int64_t r0 = voff[e] + (int64_t)blockIdx.x * kPgRange;
  const int64_t r1 = min(voff[e + 1], r0 + kPgRange);
  // thread t < 120 owns upper entry (a, b) of the 15x15 Gram (energy only: entry (14, 14))
  int a = -1, b = -1;
  if (energy_only) {
    if (tid == 0) a = b = 14;
  } else if (tid < 120) {
    int t = tid;
    for (a = 0; a < 15; ++a) {
      if (t < 15 - a) { b = a + t; break; }
      t -= 15 - a;
    }
  }
  double acc = 0.0;
  for (int64_t c0 = r0; c0 < r1; c0 += kPgChunk) {
    const int cnt = (int)(r1 - c0 < kPgChunk ? r1 - c0 : kPgChunk);
    __syncthreads();
    for (int k = tid; k < cnt * kPgRow; k += blockDim.x) S[k / kPgRow][k % kPgRow] = rows[kPgRow * c0 + k];
    __syncthreads();
    if (a >= 0)
      for (int p = 0; p < cnt; ++p) {
        acc += S[p][a] * S[p][b];
        acc += S[p][16 + a] * S[p][16 + b];
      }
  }
  if (energy_only) {
    if (tid == 0) part[((int64_t)e * nrng + blockIdx.x) * 120] = acc;
  } else if (tid < 120) {
    part[((int64_t)e * nrng + blockIdx.x) * 120 + tid] = acc;
  }
}

// per loop edge: the range partials summed in range order -> factor record
__global__ void __launch_bounds__(128) k_pg_gram_fin(const double* __restrict__ part, int nrng, int energy_only,
                                                     double* __restrict__ rec) {
  __shared__ double G[15][15];
  const int e = blockIdx.x, tid = threadIdx.x;
  double* o = rec + (int64_t)kPgRec * e;
  if (energy_only) {
    if (tid == 0) {
      double acc = 0.0;
      for (int x = 0; x < nrng; ++x) acc += part[((int64_t)e * nrng + x) * 120];
      o[161] = acc;
    }
    return;
  }
  if (tid < 120) {
    double acc = 0.0;
    for (int x = 0; x < nrng; ++x) acc += part[((int64_t)e * nrng + x) * 120 + tid];
    int t = tid, a = 0, b = 0;
    for (a = 0; a < 15; ++a) {
      if (t < 15 - a) { b = a + t; break; }
      t -= 15 - a;
    }
    G[a][b] = acc;
    G[b][a] = acc;
  }
  __syncthreads();
  for (int k = tid; k < 49; k += blockDim.x) {
    const int r = k / 7, c = k % 7;
    o[k] = G[r][c];               // H_ii
    o[49 + k] = G[7 + r][7 + c];  // H_jj
    o[98 + k] = G[r][7 + c];      // H_ij
  }
  if (tid < 7) {
    o[147 + tid] = G[tid][14];       // g_i = J_i^T r
    o[154 + tid] = G[7 + tid][14];   // g_j
  }
  if (tid == 0) o[161] = G[14][14];
}

// ---------------------------------------------------------------------------
// P3: relative pose factors (residuals.py:364-380), one thread per edge, fp64
// ---------------------------------------------------------------------------
__global__ void k_pg_rel(const double* __restrict__ relrec, const int32_t* __restrict__ ri,
                         const int32_t* __restrict__ rj, int R, const double* __restrict__ state,
                         const double* __restrict__ Wt, int energy_only, double* __restrict__ rec) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R) return;
  const double* m = relrec + (int64_t)VBA_PG_REL_REC * e;
  const double* Si = state + 8 * ri[e];
  const double* Sj = state + 8 * rj[e];
  double t1[8], t2[8], Sji[8], M[8], res[7];
  s_compose(m, Si, t1);          // T_meas S_i S_j^-1 (residuals.py:370)
  s_inverse(Sj, Sji);
  s_compose(t1, Sji, M);
  (void)t2;
  s_log(M, res);
  const double* W = Wt + 49 * (int64_t)e;   // whitening W = L^T (upper), constant per edge
  double wr[7];
  for (int r = 0; r < 7; ++r) {
    double v = 0.0;
    for (int c = 0; c < 7; ++c) v += W[r * 7 + c] * res[c];
    wr[r] = v;
  }
  double* o = rec + (int64_t)kPgRec * e;
  double en = 0.0;
  for (int r = 0; r < 7; ++r) en += wr[r] * wr[r];
  o[161] = en;
  if (energy_only) return;
  double Jri[49], Ad[49], J0[49], J[49];
  sim3_jr_inv(res, Jri);
  s_adjoint(Sj, Ad);
  mat7_mul(Jri, Ad, J0);   // J_i = Jr^-1(r) Ad(S_j), J_j = -J_i
  mat7_mul(W, J0, J);
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) {
      double h = 0.0;
      for (int k = 0; k < 7; ++k) h += J[k * 7 + r] * J[k * 7 + c];
      o[r * 7 + c] = h;          // J_i^T J_i
      o[49 + r * 7 + c] = h;     // J_j^T J_j
      o[98 + r * 7 + c] = -h;    // J_i^T J_j
    }
  for (int r = 0; r < 7; ++r) {
    double g = 0.0;
    for (int k = 0; k < 7; ++k) g += J[k * 7 + r] * wr[k];
    o[147 + r] = g;
    o[154 + r] = -g;
  }
}

// information -> whitening W = L^T (residuals.py:370-377): L = cholesky(information, lower)
// (scipy), or -- PSD but rank-deficient information, where the Cholesky meets a non-positive
// pivot -- the symmetric square root's factor L = V diag(sqrt(max(lambda, 0))) of the
// eigen-decomposition (np.linalg.eigh), computed here by cyclic Jacobi rotations.  Only
// W^T W = information (clamped) enters the energy and the normal equations, so the
// eigenvector basis (order, signs) does not matter.
__device__ void pg_eig_sqrt(const double* I, double* W) {
  double A[49], V[49];
  for (int k = 0; k < 49; ++k) { A[k] = 0.5 * (I[k] + I[(k % 7) * 7 + k / 7]); V[k] = (k % 8 == 0) ? 1.0 : 0.0; }
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int p = 0; p < 7; ++p)
      for (int q = 0; q < 7; ++q) {
        tot += A[p * 7 + q] * A[p * 7 + q];
        if (p != q) off += A[p * 7 + q] * A[p * 7 + q];
      }
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p < 6; ++p)
      for (int q = p + 1; q < 7; ++q) {
        const double apq = A[p * 7 + q];
        if (apq == 0.0) continue;
        const double theta = (A[q * 7 + q] - A[p * 7 + p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 7; ++k) {   // A <- A J (columns p, q)
          const double akp = A[k * 7 + p], akq = A[k * 7 + q];
          A[k * 7 + p] = c * akp - s * akq;
          A[k * 7 + q] = s * akp + c * akq;
        }
        for (int k = 0; k < 7; ++k) {   // A <- J^T A (rows p, q)
          const double apk = A[p * 7 + k], aqk = A[q * 7 + k];
          A[p * 7 + k] = c * apk - s * aqk;
          A[q * 7 + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 7; ++k) {   // V <- V J
          const double vkp = V[k * 7 + p], vkq = V[k * 7 + q];
          V[k * 7 + p] = c * vkp - s * vkq;
          V[k * 7 + q] = s * vkp + c * vkq;
        }
      }
  }
  // L = V diag(sqrt(max(lambda, 0))),  W = L^T: W[r][c] = sqrt(lambda_r) V[c][r]
  for (int r = 0; r < 7; ++r) {
    const double sl = sqrt(fmax(A[r * 7 + r], 0.0));
    for (int c = 0; c < 7; ++c) W[r * 7 + c] = sl * V[c * 7 + r];
  }
}

__global__ void k_pg_whiten(const double* __restrict__ relrec, int R, double* __restrict__ Wt,
                            int* __restrict__ status) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R) return;
  const double* I = relrec + (int64_t)VBA_PG_REL_REC * e + 8;
  double* W = Wt + 49 * (int64_t)e;
  double L[49];
  for (int k = 0; k < 49; ++k) L[k] = 0.0;
  for (int c = 0; c < 7; ++c) {
    double d = I[c * 7 + c];
    for (int k = 0; k < c; ++k) d -= L[c * 7 + k] * L[c * 7 + k];
    if (!(d > 0.0)) {
      pg_eig_sqrt(I, W);
      return;
    }
    const double lc = sqrt(d);
    L[c * 7 + c] = lc;
    for (int r = c + 1; r < 7; ++r) {
      double v = I[r * 7 + c];
      for (int k = 0; k < c; ++k) v -= L[r * 7 + k] * L[c * 7 + k];
      L[r * 7 + c] = v / lc;
    }
  }
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c) W[r * 7 + c] = L[c * 7 + r];
  (void)status;
}

// total energy: vision records then relative records (loopclosure.py:378-390), fixed order
__global__ void k_pg_energy(const double* __restrict__ rec, int n, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double e = 0.0;
  for (int k = 0; k < n; ++k) e += rec[(int64_t)kPgRec * k + 161];
  out[0] = e;
}

// ---------------------------------------------------------------------------
// P4: per loop source, Schur elimination of its disparities (solver.py:276-285 restricted to
// the source's pixels): u_n over the source's pose blocks (slot 0 = the source, then the
// distinct loop targets), h_n = H_dd (1 + lam) + ridge, F = sum u u^T / h, b = sum u g_d / h.
// ---------------------------------------------------------------------------
struct PgSrc {
  int32_t node;       // source node index
  int32_t eb, ee;     // its loop edges [eb, ee) (sorted by source)
  int32_t m;          // pose blocks
  int32_t slot[16];   // per edge (e - eb): pose slot of its target
  int64_t doff, npix, out;   // disparity offset, pixels, fill record offset (arena doubles)
};

__device__ __forceinline__ void pg_coupling(const PgSrc& S, const int64_t* voff, const double* rows, int n,
                                            double* u, double& h, double& g) {
  for (int k = 0; k < 7 * S.m; ++k) u[k] = 0.0;
  h = 0.0;
  g = 0.0;
  for (int e = S.eb; e < S.ee; ++e) {
    const double* r = rows + (int64_t)kPgRow * (voff[e] + n);
    const int sl = S.slot[e - S.eb];
    for (int c = 0; c < 2; ++c) {
      const double* q = r + 16 * c;
      const double jd = q[15];
      for (int k = 0; k < 7; ++k) {
        u[k] += q[k] * jd;
        u[7 * sl + k] += q[7 + k] * jd;
      }
      h += jd * jd;
      g += jd * q[14];
    }
  }
}

constexpr int kPgFillPart = 7 * kPgMaxPoses * (7 * kPgMaxPoses + 1) / 2 + 7 * kPgMaxPoses;   // doubles per partial

// partial fill-ins: CTA (range x, source y) over pixels [x kPgRange, ...): the D(D+1)/2 lower
// entries of F and the D entries of b to part[(y * nrng + x) * kPgFillPart]; the per-pixel
// H_dd / g_d of its pixels
__global__ void __launch_bounds__(256) k_pg_fill(const PgSrc* __restrict__ srcs, const int64_t* __restrict__ voff,
                                                 const double* __restrict__ rows, double lam, double ridge,
                                                 int nrng, double* __restrict__ part, double* __restrict__ hdd,
                                                 double* __restrict__ gd) {
  __shared__ double U[kPgChunk][7 * kPgMaxPoses + 2];
  const PgSrc S = srcs[blockIdx.y];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int D = 7 * S.m;
  const int nent = D * (D + 1) / 2;   // lower entries (a >= b), row-major
  constexpr int kEnt = (7 * kPgMaxPoses * (7 * kPgMaxPoses + 1) / 2 + 255) / 256;
  double acc[kEnt];
  double accg[1] = {0.0};
#pragma unroll
  for (int q = 0; q < kEnt; ++q) acc[q] = 0.0;
  const double damp = 1.0 + lam;
  const int64_t n0 = (int64_t)blockIdx.x * kPgRange, n1 = min(S.npix, n0 + kPgRange);
  for (int64_t c0 = n0; c0 < n1; c0 += kPgChunk) {
    const int cnt = (int)(n1 - c0 < kPgChunk ? n1 - c0 : kPgChunk);
    __syncthreads();
    if (tid < cnt) {
      double u[7 * kPgMaxPoses], h, g;
      pg_coupling(S, voff, rows, (int)(c0 + tid), u, h, g);
      hdd[S.doff + c0 + tid] = h;
      gd[S.doff + c0 + tid] = g;
      const double ih = 1.0 / (h * damp + ridge);
      for (int k = 0; k < D; ++k) U[tid][k] = u[k];
      U[tid][D] = ih;
      U[tid][D + 1] = g;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kEnt; ++q) {
      const int t = tid + q * nth;
      if (t >= nent) break;
      int a = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= t) ++a;
      while (a * (a + 1) / 2 > t) --a;
      const int b = t - a * (a + 1) / 2;
      for (int p = 0; p < cnt; ++p) acc[q] += U[p][a] * U[p][b] * U[p][D];
    }
    if (tid < D)
      for (int p = 0; p < cnt; ++p) accg[0] += U[p][tid] * U[p][D + 1] * U[p][D];
  }
  double* o = part + ((int64_t)blockIdx.y * nrng + blockIdx.x) * kPgFillPart;
#pragma unroll
  for (int q = 0; q < kEnt; ++q) {
    const int t = tid + q * nth;
    if (t >= nent) break;
    o[t] = acc[q];
  }
  if (tid < D) o[nent + tid] = accg[0];
}

// per loop source: the range partials summed in range order -> fill record: blocks (A, B),
// A >= B, full 7x7 row-major each, then b (D)
__global__ void __launch_bounds__(256) k_pg_fill_fin(const PgSrc* __restrict__ srcs, const double* __restrict__ part,
                                                     int nrng, double* __restrict__ arena) {
  const PgSrc S = srcs[blockIdx.x];
  const int D = 7 * S.m, nent = D * (D + 1) / 2;
  const double* p = part + (int64_t)blockIdx.x * nrng * kPgFillPart;
  double* o = arena + S.out;
  const int nr = (int)((S.npix + kPgRange - 1) / kPgRange);
  for (int t = threadIdx.x; t < nent + D; t += blockDim.x) {
    double acc = 0.0;
    for (int x = 0; x < nr; ++x) acc += p[(int64_t)x * kPgFillPart + t];
    if (t < nent) {
      int a = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= t) ++a;
      while (a * (a + 1) / 2 > t) --a;
      const int b = t - a * (a + 1) / 2;
      const int A = a / 7, B = b / 7, ra = a % 7, cb = b % 7;
      o[(A * (A + 1) / 2 + B) * 49 + ra * 7 + cb] = acc;
      if (A == B && ra != cb) o[(A * (A + 1) / 2 + B) * 49 + cb * 7 + ra] = acc;
    } else {
      o[(int64_t)S.m * (S.m + 1) / 2 * 49 + (t - nent)] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// P5 / P6: back-substitution (solver.py:290) + retraction (loopclosure.py:489-499)
// ---------------------------------------------------------------------------
__global__ void k_pg_backsub(const PgSrc* __restrict__ srcs, int nsrc, const int64_t* __restrict__ voff,
                             const double* __restrict__ rows, const int32_t* __restrict__ vj,
                             const double* __restrict__ dx, double lam, double ridge, const double* __restrict__ dcur,
                             double* __restrict__ dnxt, double* __restrict__ dxd,
                             unsigned long long* __restrict__ step_bits) {
  const PgSrc S = srcs[blockIdx.y];
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0;
  if (n < S.npix) {
    double u[7 * kPgMaxPoses], h, g;
    pg_coupling(S, voff, rows, n, u, h, g);
    // pose blocks: slot 0 the source, slot k the target of the edges mapped to it
    double acc = -g;
    for (int k = 0; k < 7; ++k) acc -= u[k] * dx[7 * S.node + k];
    for (int sl = 1; sl < S.m; ++sl) {
      int node = -1;
      for (int e = S.eb; e < S.ee; ++e)
        if (S.slot[e - S.eb] == sl) { node = vj[e]; break; }
      for (int k = 0; k < 7; ++k) acc -= u[7 * sl + k] * dx[7 * node + k];
    }
    const double d = acc / (h * (1.0 + lam) + ridge);
    const int64_t p = S.doff + n;
    dnxt[p] = fmax(dcur[p] + d, kDispFloor64);
    dxd[p] = d;
    mx = fabs(d);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(step_bits, (unsigned long long)__double_as_longlong(mx));
}

__global__ void k_pg_retract(const double* __restrict__ cur, double* __restrict__ nxt, const double* __restrict__ dx,
                             int K, unsigned long long* __restrict__ step_bits) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0;
  if (n < K) {
    const double* s = cur + 8 * n;
    double* o = nxt + 8 * n;
    if (n == 0) {   // the earliest keyframe is the gauge (loopclosure.py:403)
      for (int k = 0; k < 8; ++k) o[k] = s[k];
    } else {
      const double* d = dx + 7 * n;
      for (int k = 0; k < 7; ++k) mx = fmax(mx, fabs(d[k]));
      double E[8];
      s_exp(d, E);
      s_compose(s, E, o);   // SimTransform.retract = compose(exp(xi)) (geometry.py:326-327)
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(step_bits, (unsigned long long)__double_as_longlong(mx));
}

// dense H_pd export (reference layout: rows node*7 + a, columns = packed disparity index)
__global__ void k_pg_export_hpd(const PgSrc* __restrict__ srcs, const int64_t* __restrict__ voff,
                                const double* __restrict__ rows, const int32_t* __restrict__ vj, int64_t nd,
                                double* __restrict__ Hpd) {
  const PgSrc S = srcs[blockIdx.y];
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= S.npix) return;
  for (int e = S.eb; e < S.ee; ++e) {
    const double* r = rows + (int64_t)kPgRow * (voff[e] + n);
    const int j = vj[e];
    for (int k = 0; k < 7; ++k) {
      const double ci = r[k] * r[15] + r[16 + k] * r[31];
      const double cj = r[7 + k] * r[15] + r[23 + k] * r[31];
      Hpd[(int64_t)(7 * S.node + k) * nd + S.doff + n] += ci;
      Hpd[(int64_t)(7 * j + k) * nd + S.doff + n] += cj;
    }
  }
}

// dense reference path (use_schur=False, solver.py:291-304 through loopclosure.py:534): the
// disparity rows of the full [free poses | disparities] system, column-major lower triangle
// (ld = npad): row nf + p holds the couplings to the free pose columns of its source and
// targets (node 0, the gauge, has none), the damped diagonal h (1 + lam) + ridge, rhs -g_d
__global__ void k_pg_dense_disp(const PgSrc* __restrict__ srcs, const int64_t* __restrict__ voff,
                                const double* __restrict__ rows, const int32_t* __restrict__ vj, int nf, int64_t ld,
                                double lam, double ridge, double* __restrict__ D, double* __restrict__ rhs) {
  const PgSrc S = srcs[blockIdx.y];
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= S.npix) return;
  double u[7 * kPgMaxPoses], h, g;
  pg_coupling(S, voff, rows, n, u, h, g);
  const int64_t row = nf + S.doff + n;
  for (int sl = 0; sl < S.m; ++sl) {
    int node = S.node;
    if (sl > 0)
      for (int e = S.eb; e < S.ee; ++e)
        if (S.slot[e - S.eb] == sl) { node = vj[e]; break; }
    if (node == 0) continue;
    for (int k = 0; k < 7; ++k) D[(int64_t)(7 * (node - 1) + k) * ld + row] = u[7 * sl + k];
  }
  D[row * ld + row] = h * (1.0 + lam) + ridge;
  rhs[row] = -g;
}

__global__ void k_pg_dense_dxd(const double* __restrict__ x, int nf, int64_t nd, const double* __restrict__ dcur,
                               double* __restrict__ dnxt, double* __restrict__ dxd,
                               unsigned long long* __restrict__ step_bits) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0;
  if (p < nd) {
    const double d = x[nf + p];
    dnxt[p] = fmax(dcur[p] + d, kDispFloor64);
    dxd[p] = d;
    mx = fabs(d);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(step_bits, (unsigned long long)__double_as_longlong(mx));
}

__global__ void k_pg_scatter(const double* __restrict__ x, int npv, double* __restrict__ dx_full) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;   // free layout = nodes 1.. (node 0 frozen)
  if (k < npv) dx_full[k] = k < 7 ? 0.0 : x[k - 7];
}

// ---------------------------------------------------------------------------
// host context
// ---------------------------------------------------------------------------
static thread_local std::string pg_err;
static void pg_set_err(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  pg_err = buf;
  vba_set_error_string(buf);
}

#define PG_CUDA(x)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      pg_set_err("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));   \
      return VBA_E_CUDA;                                                            \
    }                                                                               \
  } while (0)

struct PgResult {
  double energy;
  unsigned long long step_bits;
  int status;
  int tc_bad;
  double tc[5];
};

struct PgCtx {
  vba_pg_problem P;
  vba_options O;
  int K = 0, V = 0, R = 0, nf = 0, npad = 0, nt = 0;
  int64_t nd = 0, nrows = 0;
  PgGeo geo;
  std::vector<void*> allocs;
  double* st[2] = {nullptr, nullptr};
  double* dp[2] = {nullptr, nullptr};
  int cur = 0;
  int32_t *d_vi = nullptr, *d_vj = nullptr, *d_ri = nullptr, *d_rj = nullptr, *d_pixedge = nullptr;
  int64_t *d_voff = nullptr, *d_doff = nullptr;
  std::vector<PgSrc> srcs;
  PgSrc* d_srcs = nullptr;
  double *d_rows = nullptr, *d_rows_t = nullptr, *d_arena = nullptr, *d_Wt = nullptr;
  double *d_hdd = nullptr, *d_gd = nullptr, *d_dxd = nullptr, *d_dx = nullptr;
  int vrng = 1, frng = 1;   // pixel ranges of the widest loop edge / loop source (k_pg_gram / k_pg_fill CTAs)
  // dense reference path (use_schur=False): the full system and its tile-DAG workspace, built on first use
  bool dn_ready = false;
  int dn_N = 0, dn_npad = 0, dn_nt = 0, n_dtasks = 0;
  double *d_D = nullptr, *d_drhs = nullptr, *d_dx2 = nullptr, *d_dLinv = nullptr, *d_dpart = nullptr;
  int* d_dflags = nullptr;
  void* d_dtasks = nullptr;
  double *d_gpart = nullptr, *d_fpart = nullptr;
  int64_t arena_rel = 0, arena_fill = 0, arena_len = 0;
  BlkPlan red, exp;
  bool exp_built = false;
  double *d_H = nullptr, *d_rhs = nullptr, *d_x = nullptr, *d_Ld = nullptr, *d_cpart = nullptr;
  int* d_cflags = nullptr;
  void* d_ctasks = nullptr;
  int n_ctasks = 0;
  void* d_tcws = nullptr;
  void* d_tctasks = nullptr;
  int n_tctasks = 0;
  bool use_tc = false, force_fp64 = false, tc_ran = false;
  int tc_gen = 1, tc_iters = 5;
  int* d_status = nullptr;
  PgResult* d_res = nullptr;
  PgResult* h_res = nullptr;
  bool have_step = false;
};

template <class T>
static int pg_alloc(PgCtx* c, T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  PG_CUDA(cudaMalloc((void**)p, n * sizeof(T)));
  c->allocs.push_back((void*)*p);
  return VBA_OK;
}
template <class T>
static int pg_upload(PgCtx* c, T** p, const std::vector<T>& h, cudaStream_t st) {
  PG_CUDA(plan_upload(c->allocs, p, h, st));
  return VBA_OK;
}

static void pg_destroy(PgCtx* c) {
  if (!c) return;
  for (void* p : c->allocs) cudaFree(p);
  if (c->h_res) cudaFreeHost(c->h_res);
  delete c;
}

static void qmat_host(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

// arena: [V vision records][R relative records][fill per source]
static void pg_add_records(PgCtx* c, BlkBuilder& B, const std::vector<int>& bidx, bool with_fill) {
  auto rec = [&](int i, int j, int64_t o) {
    B.add(bidx[i], bidx[i], o, 7, 7, 7, 1, false);
    B.add(bidx[j], bidx[j], o + 49, 7, 7, 7, 1, false);
    B.add(bidx[i], bidx[j], o + 98, 7, 7, 7, 1, false);
    B.addv(bidx[i], o + 147, 7, 1);
    B.addv(bidx[j], o + 154, 7, 1);
  };
  for (int e = 0; e < c->V; ++e) rec(c->P.h_vis_i[e], c->P.h_vis_j[e], (int64_t)kPgRec * e);
  for (int e = 0; e < c->R; ++e) rec(c->P.h_rel_i[e], c->P.h_rel_j[e], c->arena_rel + (int64_t)kPgRec * e);
  if (!with_fill) return;
  for (const PgSrc& S : c->srcs) {
    std::vector<int> node(S.m, -1);
    node[0] = S.node;
    for (int e = S.eb; e < S.ee; ++e) node[S.slot[e - S.eb]] = c->P.h_vis_j[e];
    for (int A = 0; A < S.m; ++A)
      for (int Bk = 0; Bk <= A; ++Bk) {
        const int64_t o = S.out + (int64_t)(A * (A + 1) / 2 + Bk) * 49;
        if (A == Bk) B.add(bidx[node[A]], bidx[node[A]], o, 7, 7, 7, -1, true);
        else if (node[A] == node[Bk]) B.add_both(bidx[node[A]], bidx[node[Bk]], o, 7, 7, 7, -1, true);
        else B.add(bidx[node[A]], bidx[node[Bk]], o, 7, 7, 7, -1, true);
      }
    const int64_t go = S.out + (int64_t)S.m * (S.m + 1) / 2 * 49;
    for (int A = 0; A < S.m; ++A) B.addv(bidx[node[A]], go + 7 * A, 7, -1);
  }
}

static int pg_plan(PgCtx* c, cudaStream_t st) {
  const vba_pg_problem& P = c->P;
  // loop sources (edges sorted by source node)
  for (int e = 1; e < c->V; ++e)
    if (P.h_vis_i[e] < P.h_vis_i[e - 1]) { pg_set_err("loop vision edges must be sorted by source"); return VBA_E_INVALID; }
  c->arena_rel = (int64_t)kPgRec * c->V;
  c->arena_fill = c->arena_rel + (int64_t)kPgRec * c->R;
  int64_t fo = c->arena_fill;
  for (int e = 0; e < c->V;) {
    PgSrc S{};
    S.node = P.h_vis_i[e];
    S.eb = e;
    while (e < c->V && P.h_vis_i[e] == S.node) ++e;
    S.ee = e;
    if (S.ee - S.eb > 16) { pg_set_err("more than 16 loop edges from one source"); return VBA_E_UNSUPPORTED; }
    std::vector<int> tgt;
    for (int q = S.eb; q < S.ee; ++q) {
      const int j = P.h_vis_j[q];
      auto it = std::find(tgt.begin(), tgt.end(), j);
      if (it == tgt.end()) { tgt.push_back(j); S.slot[q - S.eb] = (int)tgt.size(); }
      else S.slot[q - S.eb] = (int)(it - tgt.begin()) + 1;
      if (j == S.node) { pg_set_err("loop edge from a node to itself"); return VBA_E_INVALID; }
    }
    S.m = 1 + (int)tgt.size();
    if (S.m > kPgMaxPoses) { pg_set_err("loop source with more than %d pose blocks", kPgMaxPoses); return VBA_E_UNSUPPORTED; }
    S.doff = P.h_doff[S.node];
    S.npix = P.h_npix[S.node];
    S.out = fo;
    fo += (int64_t)S.m * (S.m + 1) / 2 * 49 + 7 * S.m;
    c->srcs.push_back(S);
  }
  c->arena_len = fo;
  // reduced system over the free nodes 1..K-1
  std::vector<int> bidx(c->K, -1);
  std::vector<int32_t> roff, rdim;
  for (int n = 1; n < c->K; ++n) {
    bidx[n] = n - 1;
    roff.push_back(7 * (n - 1));
    rdim.push_back(7);
  }
  c->nf = 7 * (c->K - 1);
  c->npad = (c->nf + 127) / 128 * 128;
  c->nt = c->npad / 128;
  BlkBuilder B(std::max(0, c->K - 1));
  pg_add_records(c, B, bidx, true);
  PG_CUDA(upload_blk_plan(c->allocs, B, roff, rdim, c->red, st));
  return VBA_OK;
}

static int pg_build_export(PgCtx* c, cudaStream_t st) {
  if (c->exp_built) return VBA_OK;
  std::vector<int> bidx(c->K);
  std::vector<int32_t> roff, rdim;
  for (int n = 0; n < c->K; ++n) {
    bidx[n] = n;
    roff.push_back(7 * n);
    rdim.push_back(7);
  }
  BlkBuilder B(c->K);
  pg_add_records(c, B, bidx, false);
  PG_CUDA(upload_blk_plan(c->allocs, B, roff, rdim, c->exp, st));
  c->exp_built = true;
  return VBA_OK;
}

static int pg_rows(PgCtx* c, const double* state, const double* disp, double* rows, cudaStream_t st) {
  if (c->nrows <= 0) return VBA_OK;
  const vba_pg_problem& P = c->P;
  k_pg_pixel<<<(unsigned)((c->nrows + 127) / 128), 128, 0, st>>>(c->d_pixedge, c->d_vi, c->d_vj, c->d_voff,
                                                                  c->d_doff, state, disp, P.pix, P.tgt, P.wts,
                                                                  c->nrows, P.fx, P.fy, P.cx, P.cy, c->geo, rows);
  launch_count();
  return VBA_OK;
}

// energy of (state, disp) into d_res->energy (vision records' e slots, then relative)
static int pg_energy_stage(PgCtx* c, const double* state, const double* disp, cudaStream_t st) {
  int rc = pg_rows(c, state, disp, c->d_rows_t, st);
  if (rc) return rc;
  if (c->V) {
    k_pg_gram<<<dim3(c->vrng, c->V), 128, 0, st>>>(c->d_voff, c->d_rows_t, 1, c->vrng, c->d_gpart);
    k_pg_gram_fin<<<c->V, 128, 0, st>>>(c->d_gpart, c->vrng, 1, c->d_arena);
    launch_count();
    launch_count();
  }
  if (c->R) {
    k_pg_rel<<<(c->R + 63) / 64, 64, 0, st>>>(c->P.rel, c->d_ri, c->d_rj, c->R, state, c->d_Wt, 1,
                                               c->d_arena + c->arena_rel);
    launch_count();
  }
  k_pg_energy<<<1, 32, 0, st>>>(c->d_arena, c->V + c->R, &c->d_res->energy);
  launch_count();
  return VBA_OK;
}

static int pg_linearize(PgCtx* c, cudaStream_t st) {
  const double* s = c->st[c->cur];
  int rc = pg_rows(c, s, c->dp[c->cur], c->d_rows, st);
  if (rc) return rc;
  if (c->V) {
    k_pg_gram<<<dim3(c->vrng, c->V), 128, 0, st>>>(c->d_voff, c->d_rows, 0, c->vrng, c->d_gpart);
    k_pg_gram_fin<<<c->V, 128, 0, st>>>(c->d_gpart, c->vrng, 0, c->d_arena);
    launch_count();
    launch_count();
  }
  if (c->R) {
    k_pg_rel<<<(c->R + 63) / 64, 64, 0, st>>>(c->P.rel, c->d_ri, c->d_rj, c->R, s, c->d_Wt, 0,
                                               c->d_arena + c->arena_rel);
    launch_count();
  }
  PG_CUDA(cudaGetLastError());
  return VBA_OK;
}

static int pg_reduce(PgCtx* c, double lam, cudaStream_t st) {
  PG_CUDA(cudaMemsetAsync(c->d_res, 0, sizeof(PgResult), st));
  if (!c->srcs.empty()) {
    k_pg_fill<<<dim3(c->frng, (unsigned)c->srcs.size()), 256, 0, st>>>(c->d_srcs, c->d_voff, c->d_rows, lam,
                                                                        c->O.ridge, c->frng, c->d_fpart, c->d_hdd,
                                                                        c->d_gd);
    k_pg_fill_fin<<<(unsigned)c->srcs.size(), 256, 0, st>>>(c->d_srcs, c->d_fpart, c->frng, c->d_arena);
    launch_count();
    launch_count();
  }
  if (c->nf > 0) {
    launch_assemble(c->red.bptr, c->red.bnff, c->red.cs, c->red.nbr, c->red.roff, c->red.rdim, c->d_arena, lam,
                    c->O.ridge, 1, c->d_H, c->npad, 0, st, c->red.blist, c->red.nblist);
    launch_assemble_vec(c->red.sptr, c->red.vs, c->red.nseg, c->red.soff, c->d_arena, -1.0, c->d_rhs, st);
  }
  return VBA_OK;
}

static int pg_step(PgCtx* c, double lam, cudaStream_t st) {
  int rc = pg_reduce(c, lam, st);
  if (rc) return rc;
  c->tc_ran = false;
  if (c->nf > 0) {
    if (c->use_tc && !c->force_fp64)
      c->tc_ran = chol_tc_solve(c->d_H, c->npad, c->nf, c->npad, c->d_rhs, c->d_x, c->d_tcws, c->d_tctasks,
                                c->n_tctasks, c->tc_iters, &c->d_res->tc_bad, c->tc_gen, st, c->d_res->tc) == 0;
    c->tc_gen += 2 * c->tc_iters;
    if (!c->tc_ran) {
      const char* ch = getenv("VBA_CHOL");
      if ((ch && std::strcmp(ch, "dag") == 0) ||
          chol_small_solve(c->d_H, c->npad, c->nf, c->d_rhs, c->d_x, &c->d_res->status, st))
        chol_dag_launch(c->d_H, c->npad, c->nt, c->d_rhs, c->d_x, c->d_Ld, c->d_cpart, c->d_cflags, c->d_ctasks,
                        c->n_ctasks, &c->d_res->status, st, nullptr);
    }
  }
  const int npv = 7 * c->K;
  k_pg_scatter<<<(npv + 127) / 128, 128, 0, st>>>(c->d_x, npv, c->d_dx);
  launch_count();
  const int nx = c->cur ^ 1;
  if (!c->srcs.empty()) {
    int64_t maxp = 0;
    for (const PgSrc& S : c->srcs) maxp = std::max(maxp, S.npix);
    if (maxp > 0) {
      dim3 g((unsigned)((maxp + 127) / 128), (unsigned)c->srcs.size());
      k_pg_backsub<<<g, 128, 0, st>>>(c->d_srcs, (int)c->srcs.size(), c->d_voff, c->d_rows, c->d_vj, c->d_dx, lam,
                                      c->O.ridge, c->dp[c->cur], c->dp[nx], c->d_dxd, &c->d_res->step_bits);
      launch_count();
    }
  }
  k_pg_retract<<<(c->K + 127) / 128, 128, 0, st>>>(c->st[c->cur], c->st[nx], c->d_dx, c->K, &c->d_res->step_bits);
  launch_count();
  c->have_step = true;
  return VBA_OK;
}

static int pg_ensure_dense(PgCtx* c, cudaStream_t st) {
  if (c->dn_ready) return VBA_OK;
  const int64_t N = (int64_t)c->nf + c->nd;
  if (N > 32768) {
    pg_set_err("use_schur=False: dense system of %lld unknowns exceeds the verification-path limit", (long long)N);
    return VBA_E_UNSUPPORTED;
  }
  c->dn_N = (int)N;
  c->dn_npad = (int)((N + 127) / 128 * 128);
  c->dn_nt = c->dn_npad / 128;
  const size_t np = (size_t)c->dn_npad;
  int rc;
  if ((rc = pg_alloc(c, &c->d_D, np * np)) || (rc = pg_alloc(c, &c->d_drhs, np)) || (rc = pg_alloc(c, &c->d_dx2, np)) ||
      (rc = pg_alloc(c, &c->d_dLinv, (size_t)c->dn_nt * 128 * 128)) ||
      (rc = pg_alloc(c, &c->d_dpart, (size_t)c->dn_nt * c->dn_nt * 128)) ||
      (rc = pg_alloc(c, &c->d_dflags, (size_t)2 * c->dn_nt * c->dn_nt + c->dn_nt + 1)))
    return rc;
  const int cap = chol_plan_tasks(c->dn_nt, nullptr, 0);
  std::vector<char> buf((size_t)std::max(cap, 1) * chol_task_bytes());
  c->n_dtasks = chol_plan_tasks(c->dn_nt, buf.data(), cap);
  if ((rc = pg_alloc(c, (char**)&c->d_dtasks, buf.size()))) return rc;
  PG_CUDA(cudaMemcpyAsync(c->d_dtasks, buf.data(), buf.size(), cudaMemcpyHostToDevice, st));
  c->dn_ready = true;
  return VBA_OK;
}

// the dense reference step: [damped H_ff | H_fd; H_df | damped diag(H_dd)] [dx_f; dx_d] = -[g_f; g_d]
static int pg_step_dense(PgCtx* c, double lam, cudaStream_t st) {
  int rc = pg_ensure_dense(c, st);
  if (rc) return rc;
  PG_CUDA(cudaMemsetAsync(c->d_res, 0, sizeof(PgResult), st));
  PG_CUDA(cudaMemsetAsync(c->d_D, 0, sizeof(double) * (size_t)c->dn_npad * c->dn_npad, st));
  PG_CUDA(cudaMemsetAsync(c->d_drhs, 0, sizeof(double) * c->dn_npad, st));
  launch_pad_identity(c->d_D, c->dn_npad, c->dn_N, c->dn_npad, c->d_drhs, st);
  if (c->nf > 0) {   // damped H_ff without the fill-in, and -g_f
    launch_assemble(c->red.bptr, c->red.bnff, c->red.cs, c->red.nbr, c->red.roff, c->red.rdim, c->d_arena, lam,
                    c->O.ridge, 1, c->d_D, c->dn_npad, 2, st, c->red.blist, c->red.nblist);
    launch_assemble_vec(c->red.sptr, c->red.vs, c->red.nseg, c->red.soff, c->d_arena, -1.0, c->d_drhs, st, 1);
  }
  int64_t maxp = 0;
  for (const PgSrc& S : c->srcs) maxp = std::max(maxp, S.npix);
  if (maxp > 0) {
    dim3 g((unsigned)((maxp + 127) / 128), (unsigned)c->srcs.size());
    k_pg_dense_disp<<<g, 128, 0, st>>>(c->d_srcs, c->d_voff, c->d_rows, c->d_vj, c->nf, c->dn_npad, lam, c->O.ridge,
                                       c->d_D, c->d_drhs);
    launch_count();
  }
  const char* ch = getenv("VBA_CHOL");
  if ((ch && std::strcmp(ch, "dag") == 0) ||
      chol_small_solve(c->d_D, c->dn_npad, c->dn_N, c->d_drhs, c->d_dx2, &c->d_res->status, st))
    chol_dag_launch(c->d_D, c->dn_npad, c->dn_nt, c->d_drhs, c->d_dx2, c->d_dLinv, c->d_dpart, c->d_dflags,
                    c->d_dtasks, c->n_dtasks, &c->d_res->status, st, nullptr);
  c->tc_ran = false;
  const int npv = 7 * c->K;
  k_pg_scatter<<<(npv + 127) / 128, 128, 0, st>>>(c->d_dx2, npv, c->d_dx);
  launch_count();
  const int nx = c->cur ^ 1;
  if (c->nd > 0) {
    k_pg_dense_dxd<<<(unsigned)((c->nd + 127) / 128), 128, 0, st>>>(c->d_dx2, c->nf, c->nd, c->dp[c->cur],
                                                                     c->dp[nx], c->d_dxd, &c->d_res->step_bits);
    launch_count();
  }
  k_pg_retract<<<(c->K + 127) / 128, 128, 0, st>>>(c->st[c->cur], c->st[nx], c->d_dx, c->K, &c->d_res->step_bits);
  launch_count();
  c->have_step = true;
  return VBA_OK;
}

static int pg_step_any(PgCtx* c, double lam, int use_schur, cudaStream_t st) {
  // the reference takes the Schur path only when there are disparities (solver.py:281)
  if (use_schur || c->nd == 0) return pg_step(c, lam, st);
  return pg_step_dense(c, lam, st);
}

static bool pg_tc_failed(PgCtx* c) { return c->tc_ran && (c->h_res->tc_bad != 0 || c->h_res->tc[4] != 1.0); }

// one LM trial: step, energy of the trial state; returns status/new cost/step norm
static int pg_trial(PgCtx* c, double lam, int* status, double* cost, double* step, cudaStream_t st) {
  int rc = pg_step_any(c, lam, c->O.use_schur, st);
  if (rc) return rc;
  const int nx = c->cur ^ 1;
  if ((rc = pg_energy_stage(c, c->st[nx], c->dp[nx], st))) return rc;
  PG_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(PgResult), cudaMemcpyDeviceToHost, st));
  PG_CUDA(cudaStreamSynchronize(st));
  if (pg_tc_failed(c)) {
    c->force_fp64 = true;
    rc = pg_trial(c, lam, status, cost, step, st);
    c->force_fp64 = false;
    return rc;
  }
  *status = c->h_res->status ? VBA_E_NOT_SPD : VBA_OK;
  *cost = c->h_res->energy;
  unsigned long long b = c->h_res->step_bits;
  std::memcpy(step, &b, sizeof(double));
  return VBA_OK;
}

}  // namespace vba

using namespace vba;

extern "C" {

int vba_pg_create(void** out, const vba_pg_problem* prob, const vba_options* opts, void* stream) {
  *out = nullptr;
  if (!prob || !opts) { pg_set_err("null problem/options"); return VBA_E_INVALID; }
  cudaStream_t st = (cudaStream_t)stream;
  PgCtx* c = new PgCtx();
  auto fail = [&](int rc) { pg_destroy(c); return rc; };
  c->P = *prob;
  c->O = *opts;
  c->K = prob->n_nodes;
  c->V = prob->n_vis;
  c->R = prob->n_rel;
  c->nd = prob->n_disp;
  c->nrows = prob->n_rows;
  if (c->K <= 0 || c->V < 0 || c->R < 0 || c->nd < 0 || c->nrows < 0) { pg_set_err("invalid sizes"); return fail(VBA_E_INVALID); }
  if (!(opts->ridge > 0) || !(opts->damping > 0)) { pg_set_err("invalid options"); return fail(VBA_E_INVALID); }
  {  // T_bc = T_cb^-1 (loopclosure.py:254-256)
    double qi[4] = {1, 0, 0, 0}, t[3] = {0, 0, 0};
    if (prob->has_Tcb) {
      const double* q = prob->Tcb;
      const double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      qi[0] = q[0] / n; qi[1] = -q[1] / n; qi[2] = -q[2] / n; qi[3] = -q[3] / n;
      if (qi[0] < 0) for (double& v : qi) v = -v;
      t[0] = prob->Tcb[4]; t[1] = prob->Tcb[5]; t[2] = prob->Tcb[6];
    }
    qmat_host(qi, c->geo.Rbc);
    for (int a = 0; a < 3; ++a)
      c->geo.pbc[a] = -(c->geo.Rbc[a * 3] * t[0] + c->geo.Rbc[a * 3 + 1] * t[1] + c->geo.Rbc[a * 3 + 2] * t[2]);
  }
  int rc = pg_plan(c, st);
  if (rc) return fail(rc);
  std::vector<int32_t> vi(prob->h_vis_i, prob->h_vis_i + c->V), vj(prob->h_vis_j, prob->h_vis_j + c->V);
  std::vector<int32_t> ri(prob->h_rel_i, prob->h_rel_i + c->R), rj(prob->h_rel_j, prob->h_rel_j + c->R);
  std::vector<int64_t> voff(prob->h_voff, prob->h_voff + c->V + 1), doff(prob->h_doff, prob->h_doff + c->K + 1);
  std::vector<int32_t> pe((size_t)std::max<int64_t>(1, c->nrows), 0);
  for (int e = 0; e < c->V; ++e)
    for (int64_t r = voff[e]; r < voff[e + 1]; ++r) pe[r] = e;
  for (int e = 0; e < c->V; ++e)
    if (voff[e + 1] - voff[e] != prob->h_npix[vi[e]]) {
      pg_set_err("loop vision rows must align with the source pixel snapshot");
      return fail(VBA_E_INVALID);
    }
  if ((rc = pg_upload(c, &c->d_vi, vi, st)) || (rc = pg_upload(c, &c->d_vj, vj, st)) ||
      (rc = pg_upload(c, &c->d_ri, ri, st)) || (rc = pg_upload(c, &c->d_rj, rj, st)) ||
      (rc = pg_upload(c, &c->d_voff, voff, st)) || (rc = pg_upload(c, &c->d_doff, doff, st)) ||
      (rc = pg_upload(c, &c->d_pixedge, pe, st)) || (rc = pg_upload(c, &c->d_srcs, c->srcs, st)))
    return fail(rc);
  for (int b = 0; b < 2; ++b)
    if ((rc = pg_alloc(c, &c->st[b], (size_t)8 * c->K)) || (rc = pg_alloc(c, &c->dp[b], (size_t)c->nd)))
      return fail(rc);
  for (int v = 0; v < c->V; ++v)
    c->vrng = std::max(c->vrng, (int)((voff[v + 1] - voff[v] + kPgRange - 1) / kPgRange));
  for (const PgSrc& S : c->srcs) c->frng = std::max(c->frng, (int)((S.npix + kPgRange - 1) / kPgRange));
  if ((rc = pg_alloc(c, &c->d_gpart, (size_t)120 * std::max(1, c->V) * c->vrng)) ||
      (rc = pg_alloc(c, &c->d_fpart, (size_t)kPgFillPart * std::max<size_t>(1, c->srcs.size()) * c->frng)))
    return fail(rc);
  if ((rc = pg_alloc(c, &c->d_rows, (size_t)kPgRow * c->nrows)) ||
      (rc = pg_alloc(c, &c->d_rows_t, (size_t)kPgRow * c->nrows)) || (rc = pg_alloc(c, &c->d_arena, (size_t)c->arena_len)) ||
      (rc = pg_alloc(c, &c->d_Wt, (size_t)49 * c->R)) || (rc = pg_alloc(c, &c->d_hdd, (size_t)c->nd)) ||
      (rc = pg_alloc(c, &c->d_gd, (size_t)c->nd)) || (rc = pg_alloc(c, &c->d_dxd, (size_t)c->nd)) ||
      (rc = pg_alloc(c, &c->d_dx, (size_t)7 * c->K)) || (rc = pg_alloc(c, &c->d_H, (size_t)c->npad * c->npad)) ||
      (rc = pg_alloc(c, &c->d_rhs, (size_t)c->npad)) || (rc = pg_alloc(c, &c->d_x, (size_t)c->npad)) ||
      (rc = pg_alloc(c, &c->d_Ld, (size_t)std::max(1, c->nt) * 128 * 128)) ||
      (rc = pg_alloc(c, &c->d_cpart, (size_t)std::max(1, c->nt * c->nt) * 128)) ||
      (rc = pg_alloc(c, &c->d_cflags, (size_t)2 * c->nt * c->nt + c->nt + 1)) || (rc = pg_alloc(c, &c->d_status, 1)) ||
      (rc = pg_alloc(c, &c->d_res, 1)))
    return fail(rc);
  if (cudaMallocHost((void**)&c->h_res, sizeof(PgResult)) != cudaSuccess) { pg_set_err("pinned alloc failed"); return fail(VBA_E_CUDA); }
  if (cudaMemcpyAsync(c->st[0], prob->state, sizeof(double) * 8 * c->K, cudaMemcpyDeviceToDevice, st) ||
      (c->nd && cudaMemcpyAsync(c->dp[0], prob->disp, sizeof(double) * c->nd, cudaMemcpyDeviceToDevice, st))) {
    pg_set_err("state upload failed");
    return fail(VBA_E_CUDA);
  }
  {  // reduced solve: fp64 tile DAG, tensor cores from 4 tiles up (as VI-BA)
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* ch = getenv("VBA_CHOL");
    c->use_tc = (ch && std::strcmp(ch, "tc") == 0) ? c->nt > 0
              : (ch && std::strcmp(ch, "fp64") == 0) ? false : c->nt >= 4;
    if (c->nt > sms) c->use_tc = false;
    const int cap = chol_plan_tasks(c->nt, nullptr, 0);
    std::vector<char> buf((size_t)std::max(cap, 1) * chol_task_bytes());
    c->n_ctasks = chol_plan_tasks(c->nt, buf.data(), cap);
    if ((rc = pg_alloc(c, (char**)&c->d_ctasks, buf.size()))) return fail(rc);
    PG_CUDA(cudaMemcpyAsync(c->d_ctasks, buf.data(), buf.size(), cudaMemcpyHostToDevice, st));
    if (c->use_tc) {
      const size_t wb = chol_tc_ws_bytes(c->npad);
      if ((rc = pg_alloc(c, (char**)&c->d_tcws, wb))) return fail(rc);
      cudaMemsetAsync(c->d_tcws, 0, wb, st);
      const int cap2 = chol_plan_tasks_tc(c->nt, nullptr, 0);
      std::vector<char> b2((size_t)std::max(cap2, 1) * chol_task_bytes());
      c->n_tctasks = chol_plan_tasks_tc(c->nt, b2.data(), cap2);
      if ((rc = pg_alloc(c, (char**)&c->d_tctasks, b2.size()))) return fail(rc);
      PG_CUDA(cudaMemcpyAsync(c->d_tctasks, b2.data(), b2.size(), cudaMemcpyHostToDevice, st));
    }
  }
  cudaMemsetAsync(c->d_arena, 0, sizeof(double) * std::max<int64_t>(1, c->arena_len), st);
  cudaMemsetAsync(c->d_H, 0, sizeof(double) * std::max<size_t>(1, (size_t)c->npad * c->npad), st);
  cudaMemsetAsync(c->d_rhs, 0, sizeof(double) * std::max(1, c->npad), st);
  cudaMemsetAsync(c->d_x, 0, sizeof(double) * std::max(1, c->npad), st);
  launch_pad_identity(c->d_H, c->npad, c->nf, c->npad, c->d_rhs, st);
  // whitening of every relative edge (constant over the solve)
  cudaMemsetAsync(c->d_status, 0, sizeof(int), st);
  if (c->R) {
    k_pg_whiten<<<(c->R + 63) / 64, 64, 0, st>>>(prob->rel, c->R, c->d_Wt, c->d_status);
    launch_count();
  }
  int hs = 0;
  if (cudaMemcpyAsync(&hs, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, st) ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    pg_set_err("create: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(VBA_E_CUDA);
  }
  if (hs) {
    pg_set_err("relative-pose whitening failed");
    return fail(VBA_E_UNSUPPORTED);
  }
  *out = c;
  return VBA_OK;
}

int vba_pg_destroy(void* ctx) {
  pg_destroy((PgCtx*)ctx);
  return VBA_OK;
}

int vba_pg_energy(void* ctx, void* stream, double* out) {
  PgCtx* c = (PgCtx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = pg_energy_stage(c, c->st[c->cur], c->dp[c->cur], st);
  if (rc) return rc;
  PG_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(PgResult), cudaMemcpyDeviceToHost, st));
  PG_CUDA(cudaStreamSynchronize(st));
  *out = c->h_res->energy;
  return VBA_OK;
}

int vba_pg_linearize(void* ctx, void* stream) { return pg_linearize((PgCtx*)ctx, (cudaStream_t)stream); }

int vba_pg_export_normal_eq(void* ctx, void* stream, double* H_pp, double* g_p, double* H_pd, double* H_dd,
                            double* g_d) {
  PgCtx* c = (PgCtx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = pg_build_export(c, st);
  if (rc) return rc;
  const int npv = 7 * c->K;
  if (H_pp) {
    PG_CUDA(cudaMemsetAsync(H_pp, 0, sizeof(double) * npv * npv, st));
    launch_assemble(c->exp.bptr, c->exp.bnff, c->exp.cs, c->exp.nbr, c->exp.roff, c->exp.rdim, c->d_arena, 0.0, 0.0,
                    0, H_pp, npv, 1, st);
  }
  if (g_p) launch_assemble_vec(c->exp.sptr, c->exp.vs, c->exp.nseg, c->exp.soff, c->d_arena, 1.0, g_p, st);
  if ((H_dd || g_d) && !c->srcs.empty()) {   // per-pixel sums (k_pg_fill at lam = 0 writes them)
    if ((rc = pg_reduce(c, 0.0, st))) return rc;
    if (H_dd) PG_CUDA(cudaMemcpyAsync(H_dd, c->d_hdd, sizeof(double) * c->nd, cudaMemcpyDeviceToDevice, st));
    if (g_d) PG_CUDA(cudaMemcpyAsync(g_d, c->d_gd, sizeof(double) * c->nd, cudaMemcpyDeviceToDevice, st));
  }
  if (H_pd && c->nd > 0) {
    PG_CUDA(cudaMemsetAsync(H_pd, 0, sizeof(double) * npv * c->nd, st));
    int64_t maxp = 0;
    for (const PgSrc& S : c->srcs) maxp = std::max(maxp, S.npix);
    dim3 g((unsigned)((maxp + 127) / 128), (unsigned)c->srcs.size());
    k_pg_export_hpd<<<g, 128, 0, st>>>(c->d_srcs, c->d_voff, c->d_rows, c->d_vj, c->nd, H_pd);
    launch_count();
  }
  PG_CUDA(cudaStreamSynchronize(st));
  return VBA_OK;
}

int vba_pg_solve_step(void* ctx, void* stream, double lam, int32_t use_schur) {
  PgCtx* c = (PgCtx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = pg_step_any(c, lam, use_schur, st);
  if (rc) return rc;
  PG_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(PgResult), cudaMemcpyDeviceToHost, st));
  PG_CUDA(cudaStreamSynchronize(st));
  if (pg_tc_failed(c)) {
    c->force_fp64 = true;
    rc = pg_step(c, lam, st);
    c->force_fp64 = false;
    if (rc) return rc;
    PG_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(PgResult), cudaMemcpyDeviceToHost, st));
    PG_CUDA(cudaStreamSynchronize(st));
  }
  return c->h_res->status ? VBA_E_NOT_SPD : VBA_OK;
}

int vba_pg_export_step(void* ctx, void* stream, double* dx_full, double* dx_d) {
  PgCtx* c = (PgCtx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->have_step) { pg_set_err("no step computed"); return VBA_E_INVALID; }
  if (dx_full) PG_CUDA(cudaMemcpyAsync(dx_full, c->d_dx, sizeof(double) * 7 * c->K, cudaMemcpyDeviceToDevice, st));
  if (dx_d && c->nd) PG_CUDA(cudaMemcpyAsync(dx_d, c->d_dxd, sizeof(double) * c->nd, cudaMemcpyDeviceToDevice, st));
  PG_CUDA(cudaStreamSynchronize(st));
  return VBA_OK;
}

// solve_pgba's LM loop (loopclosure.py:515-574), the accept test requiring a finite energy
int vba_pg_solve(void* ctx, void* stream, vba_report* rep, double* traj, int32_t cap) {
  PgCtx* c = (PgCtx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  const vba_options& o = c->O;
  std::memset(rep, 0, sizeof(*rep));
  double cost;
  int rc = vba_pg_energy(ctx, stream, &cost);
  if (rc) return rc;
  if (!std::isfinite(cost)) { pg_set_err("pose-graph energy is not finite"); return VBA_E_NONFINITE; }
  std::vector<double> tr{cost};
  auto finish = [&](int iters, int term, int warns, int trials) {
    rep->iterations = iters;
    rep->termination = term;
    rep->n_warnings = warns;
    rep->trials = trials;
    rep->initial_cost = tr[0];
    rep->final_cost = cost;
    rep->n_costs = (int)tr.size();
    for (int i = 0; i < (int)tr.size() && i < cap; ++i) traj[i] = tr[i];
    return VBA_OK;
  };
  double lam = o.damping;
  int term = 0, iters = 0, warns = 0, trials = 0;
  bool broke = false;
  for (int it = 0; it < o.max_iterations; ++it) {
    nvtxRangePushA("vba.pg.linearize");
    rc = pg_linearize(c, st);
    nvtxRangePop();
    if (rc) return rc;
    bool accepted = false;
    while (true) {
      int status;
      double nc, step;
      nvtxRangePushA("vba.pg.trial");
      rc = pg_trial(c, lam, &status, &nc, &step, st);
      nvtxRangePop();
      if (rc) return rc;
      ++trials;
      if (status == VBA_E_NOT_SPD) {
        ++warns;
        lam *= o.damping_up;
        if (lam > o.max_damping) return finish(iters, 3, warns, trials);
        continue;
      }
      if (std::isfinite(nc) && nc < cost) {
        cost = nc;
        tr.push_back(cost);
        lam = std::max(lam * o.damping_down, 1e-12);
        accepted = true;
        iters = it + 1;
        c->cur ^= 1;
        if (step < o.step_tol) term = 1;
        break;
      }
      lam *= o.damping_up;
      if (lam > o.max_damping) { term = 2; break; }
    }
    if (!accepted) { broke = true; break; }
    if (term == 1) { broke = true; break; }
    const double prev = tr[tr.size() - 2];
    if (prev > 0 && (prev - cost) / prev < o.rel_decrease_tol) { term = 1; broke = true; break; }
  }
  if (!broke) term = 0;
  PG_CUDA(cudaGetLastError());
  return finish(iters, term, warns, trials);
}

int vba_pg_download(void* ctx, void* stream) {
  PgCtx* c = (PgCtx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  PG_CUDA(cudaMemcpyAsync(c->P.state, c->st[c->cur], sizeof(double) * 8 * c->K, cudaMemcpyDeviceToDevice, st));
  if (c->nd) PG_CUDA(cudaMemcpyAsync(c->P.disp, c->dp[c->cur], sizeof(double) * c->nd, cudaMemcpyDeviceToDevice, st));
  return VBA_OK;
}

}  // extern "C"
