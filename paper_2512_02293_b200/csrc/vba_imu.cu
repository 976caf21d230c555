// vba_imu.cu — inertial (preintegration) factors in fp64 (sm_100a).
//
// Restates inertial_residual (residuals.py:274-354) and the inertial part of
// _linearize (solver.py:222-249) / total_energy (solver.py:127-130), paths
// relative to /root/reference/pkg/src/vislam/.  One 64-thread CTA per factor:
// lane 0 evaluates the residual and the raw Jacobian blocks (the sparse block
// structure of residuals.py:306-332), the CTA whitens the 34 columns
// [J_i | J_j | J_g | r] with the Cholesky factors of the delta covariance
// (residuals.py:334-347) and forms the normal-equation blocks with fixed-order
// dot products.
#include <cuda_runtime.h>

#include "vba_internal.cuh"

namespace vba {

// IMU record offsets (include/vba.h)
constexpr int kDT = 0, kDR = 1, kDP = 5, kDV = 8, kJR = 11, kJP = 20, kJV = 38, kC9 = 56, kCB = 137, kBH = 173;
constexpr int kCols = 34;   // J_i(15) J_j(15) J_g(3) r(1)

// ---------------------------------------------------------------------------
// once per solve: lower Cholesky factors of cov[0:9,0:9] and cov[9:15,9:15]
// (scipy.linalg.cholesky(lower=True), residuals.py:338-339); non-PD -> status
// ---------------------------------------------------------------------------
__device__ bool chol_lower(const double* A, int n, int lda, double* L) {
  for (int i = 0; i < n * n; ++i) L[i] = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = A[j * lda + j];
    for (int k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
    if (!(s > 0.0)) return false;
    const double d = sqrt(s);
    L[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A[i * lda + j];
      for (int k = 0; k < j; ++k) t -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = t / d;
    }
  }
  return true;
}

__global__ void k_imu_prep(const double* __restrict__ imu, int F, double* __restrict__ Lbuf, int* status) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const double* r = imu + (int64_t)f * VBA_IMU_REC;
  double* L = Lbuf + (int64_t)f * kImuL;
  const bool ok9 = chol_lower(r + kC9, 9, 9, L);
  const bool okb = chol_lower(r + kCB, 6, 6, L + 81);
  if (!(ok9 && okb)) atomicExch(status, 1);
}

void launch_imu_prep(const double* imu, int F, double* Lbuf, int* status, cudaStream_t st) {
  if (F <= 0) return;
  k_imu_prep<<<(F + 63) / 64, 64, 0, st>>>(imu, F, Lbuf, status);
  launch_count();
}

// ---------------------------------------------------------------------------
// factor evaluation.  Output record (ld = sdof), ibs doubles per factor:
//   Hii[s*s] Hjj[s*s] Hij[s*s] gi[s] gj[s] Hgg[4] Hig[s*2] Hjg[s*2] gg[2] energy
// ---------------------------------------------------------------------------
// Residual and whitened Jacobian columns [J_i | J_j | J_g | r] of one factor into J (shared
// memory, 15 x kCols); called by every thread of the CTA (it synchronises).  energy_only:
// the residual column only.
__device__ void imu_whitened_J(const double* __restrict__ rec, const double* __restrict__ Lg,
                               const double* si, const double* sj, const double* __restrict__ grav, int energy_only,
                               double (*J)[kCols + 1], double* L) {
  const int tid = threadIdx.x;
  for (int i = tid; i < 117; i += blockDim.x) L[i] = Lg[i];
  for (int i = tid; i < 15 * (kCols + 1); i += blockDim.x) (&J[0][0])[i] = 0.0;
  __syncthreads();
  // the residual and raw Jacobian blocks by two threads in different warps (they run in
  // parallel): warp 0 the rotation rows (the long serial chain: Exp, Log, Jr^-1 x 2, Jr),
  // warp 1 the position / velocity / bias rows
  if (tid == 0 || tid == 32) {
    const double dt = rec[kDT];
    double Ri[9];
    qmat(si, Ri);
    double db[6];
    for (int k = 0; k < 6; ++k) db[k] = si[10 + k] - rec[kBH + k];   // s_i.bias - b_hat (:291)
    if (tid == 0) {
      double Rj[9];
      qmat(sj, Rj);
      const double* Jr = rec + kJR;
      double ct[3];
      mat3_vec(Jr, db, ct);                                         // corr_rot_tangent (:294)
      double dR[9], Ect[9], C[9], T2[9], Mrot[9];
      qmat(rec + kDR, dR);
      so3_exp(ct, Ect);
      mat3_mul(dR, Ect, C);                                         // :295
      // Mrot = C^T R_i^T R_j
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          T2[a * 3 + b] = C[0 * 3 + a] * Ri[b * 3 + 0] + C[1 * 3 + a] * Ri[b * 3 + 1] + C[2 * 3 + a] * Ri[b * 3 + 2];
      mat3_mul(T2, Rj, Mrot);
      double qrot[4], rrot[3];
      q_from_mat(Mrot, qrot);
      qlog(qrot, rrot);                                             // r_rot (:296)
      for (int k = 0; k < 3; ++k) J[k][33] = rrot[k];
      if (!energy_only) {
        double Jri[9], Jli[9], mr[3] = {-rrot[0], -rrot[1], -rrot[2]}, Jrc[9];
        so3_jr_inv(rrot, Jri);                                      // :303
        so3_jr_inv(mr, Jli);                                        // :304
        so3_jr(ct, Jrc);
        double RjtRi[9], A1[9], A2[9], A3[9];
        mat3_Tmul(Rj, Ri, RjtRi);
        mat3_mul(Jri, RjtRi, A1);                                   // J_i[rot,θ] = -Jr^-1 R_j^T R_i
        mat3_mul(Jli, Jrc, A2);
        mat3_mul(A2, Jr, A3);                                       // J_i[rot,bg] = -Jl^-1 Jr(ct) J_rot
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            J[a][b] = -A1[a * 3 + b];
            J[a][15 + b] = Jri[a * 3 + b];                          // J_j[rot,θ]
            J[a][9 + b] = -A3[a * 3 + b];
          }
      }
    } else {
      double Rwg[9];
      qmat(grav, Rwg);
      const double G = grav[4];
      const double g[3] = {Rwg[2] * G, Rwg[5] * G, Rwg[8] * G};    // R_wg (0,0,G)  residuals.py:125-130
      const double* Jp = rec + kJP;
      const double* Jv = rec + kJV;
      double spos[3], svel[3], rpos[3], rvel[3];
      for (int k = 0; k < 3; ++k) {
        spos[k] = sj[4 + k] - si[4 + k] - si[7 + k] * dt - 0.5 * dt * dt * g[k];   // :297
        svel[k] = sj[7 + k] - si[7 + k] - dt * g[k];                              // :299
      }
      double Rs[3], Rv[3];
      mat3T_vec(Ri, spos, Rs);
      mat3T_vec(Ri, svel, Rv);
      for (int k = 0; k < 3; ++k) {
        double jp = 0.0, jv = 0.0;
        for (int m = 0; m < 6; ++m) { jp += Jp[k * 6 + m] * db[m]; jv += Jv[k * 6 + m] * db[m]; }
        rpos[k] = Rs[k] - (rec[kDP + k] + jp);                       // :298
        rvel[k] = Rv[k] - (rec[kDV + k] + jv);                       // :300
      }
      for (int k = 0; k < 3; ++k) {
        J[3 + k][33] = rpos[k];
        J[6 + k][33] = rvel[k];
      }
      for (int k = 0; k < 6; ++k) J[9 + k][33] = sj[10 + k] - si[10 + k];   // r_bias (:301)
      if (!energy_only) {
        double Hs[9], Hv[9], RwgH[9], hg[9], gI[3] = {0.0, 0.0, G}, RitRwgH[9];
        hat3(Rs, Hs);
        hat3(Rv, Hv);
        hat3(gI, hg);
        mat3_mul(Rwg, hg, RwgH);
        mat3_Tmul(Ri, RwgH, RitRwgH);                               // R_i^T R_wg [g_I]x
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            J[3 + a][b] = Hs[a * 3 + b];                            // J_i[pos,θ]
            J[3 + a][3 + b] = -Ri[b * 3 + a];                       // -R_i^T
            J[3 + a][15 + 3 + b] = Ri[b * 3 + a];                   // J_j[pos,p] = R_i^T
            J[3 + a][6 + b] = -dt * Ri[b * 3 + a];
            J[3 + a][30 + b] = 0.5 * dt * dt * RitRwgH[a * 3 + b];  // J_g[pos]
            J[6 + a][b] = Hv[a * 3 + b];                            // J_i[vel,θ]
            J[6 + a][6 + b] = -Ri[b * 3 + a];
            J[6 + a][15 + 6 + b] = Ri[b * 3 + a];
            J[6 + a][30 + b] = dt * RitRwgH[a * 3 + b];             // J_g[vel]
          }
        for (int a = 0; a < 3; ++a)
          for (int m = 0; m < 6; ++m) {
            J[3 + a][9 + m] = -Jp[a * 6 + m];
            J[6 + a][9 + m] = -Jv[a * 6 + m];
          }
        for (int k = 0; k < 6; ++k) {
          J[9 + k][9 + k] = -1.0;
          J[9 + k][15 + 9 + k] = 1.0;
        }
      }
    }
  }
  __syncthreads();
  // whitening: forward substitution per column (residuals.py:343-347)
  const int ncol0 = energy_only ? 33 : 0;
  for (int c = ncol0 + tid; c < kCols; c += blockDim.x) {
    for (int r = 0; r < 9; ++r) {
      double t = J[r][c];
      for (int m = 0; m < r; ++m) t -= L[r * 9 + m] * J[m][c];
      J[r][c] = t / L[r * 9 + r];
    }
    for (int r = 0; r < 6; ++r) {
      double t = J[9 + r][c];
      for (int m = 0; m < r; ++m) t -= L[81 + r * 6 + m] * J[9 + m][c];
      J[9 + r][c] = t / L[81 + r * 6 + r];
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(64) k_imu_factor(const double* __restrict__ imu, const double* __restrict__ Lbuf,
                                                   const int32_t* __restrict__ fi, const int32_t* __restrict__ fj,
                                                   int f0, const double* __restrict__ state,
                                                   const double* __restrict__ grav, int sdof, int ibs, int energy_only,
                                                   double* __restrict__ out) {
  __shared__ double J[15][kCols + 1];
  __shared__ double L[kImuL];
  const int f = f0 + blockIdx.x, tid = threadIdx.x;
  imu_whitened_J(imu + (int64_t)f * VBA_IMU_REC, Lbuf + (int64_t)f * kImuL, state + 16 * fi[f], state + 16 * fj[f],
                 grav, energy_only, J, L);
  double* o = out + (int64_t)f * ibs;
  const int s = sdof, s2 = sdof * sdof;
  const int oE = 3 * s2 + 6 * s + 6;
  if (energy_only) {
    if (tid == 0) {
      double e = 0.0;
      for (int r = 0; r < 15; ++r) e += J[r][33] * J[r][33];
      o[oE] = e;
    }
    return;
  }
  // normal-equation blocks (solver.py:226-249): column pairs (ca, cb) dot products over 15 rows
  const int nout = oE + 1;
  for (int it = tid; it < nout; it += blockDim.x) {
    int ca, cb;
    if (it < s2) { ca = it / s; cb = it % s; }                               // Hii
    else if (it < 2 * s2) { ca = 15 + (it - s2) / s; cb = 15 + (it - s2) % s; }   // Hjj
    else if (it < 3 * s2) { ca = (it - 2 * s2) / s; cb = 15 + (it - 2 * s2) % s; } // Hij
    else if (it < 3 * s2 + s) { ca = it - 3 * s2; cb = 33; }                 // gi
    else if (it < 3 * s2 + 2 * s) { ca = 15 + it - 3 * s2 - s; cb = 33; }    // gj
    else if (it < 3 * s2 + 2 * s + 4) { const int q = it - 3 * s2 - 2 * s; ca = 30 + q / 2; cb = 30 + q % 2; }  // Hgg
    else if (it < 3 * s2 + 4 * s + 4) { const int q = it - 3 * s2 - 2 * s - 4; ca = q / 2; cb = 30 + q % 2; }  // Hig
    else if (it < 3 * s2 + 6 * s + 4) { const int q = it - 3 * s2 - 4 * s - 4; ca = 15 + q / 2; cb = 30 + q % 2; }  // Hjg
    else if (it < 3 * s2 + 6 * s + 6) { ca = 30 + it - 3 * s2 - 6 * s - 4; cb = 33; }   // gg
    else { ca = 33; cb = 33; }                                                // energy
    double acc = 0.0;
    for (int r = 0; r < 15; ++r) acc += J[r][ca] * J[r][cb];
    o[it] = acc;
  }
}

void launch_imu_factor(const double* imu, const double* Lbuf, const int32_t* fi, const int32_t* fj, int f0, int F,
                       const DevState& s, const double* /*ts*/, int sdof, int ibs, int energy_only,
                       double* imu_blocks, cudaStream_t st) {
  if (F <= 0) return;
  k_imu_factor<<<F, 64, 0, st>>>(imu, Lbuf, fi, fj, f0, s.state, s.grav, sdof, ibs, energy_only, imu_blocks);
  launch_count();
}

}  // namespace vba

namespace vba {

// ---------------------------------------------------------------------------
// Stage-2 inertial-only initialisation (initialization.py:152-231): per factor, the
// whitened inertial Jacobian re-expressed in the stage-2 unknowns
//   [log-scale, gravity (2), shared bias (6), v_i (3), v_j (3)]
// (initialization.py:183-190), its 15x15 Gram and gradient, and the energy.
// Record: H[15*15] g[15] e (kInit2Rec doubles).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(64) k_init2_factor(const double* __restrict__ imu, const double* __restrict__ Lbuf,
                                                     const int32_t* __restrict__ fi, const int32_t* __restrict__ fj,
                                                     const double* __restrict__ state, const double* __restrict__ grav,
                                                     const double* __restrict__ pvis, const double* __restrict__ es_p,
                                                     int energy_only, double* __restrict__ out) {
  __shared__ double J[15][kCols + 1];
  __shared__ double L[kImuL];
  __shared__ double J2[15][17];
  const int f = blockIdx.x, tid = threadIdx.x;
  const int i = fi[f], j = fj[f];
  imu_whitened_J(imu + (int64_t)f * VBA_IMU_REC, Lbuf + (int64_t)f * kImuL, state + 16 * i, state + 16 * j, grav,
                 energy_only, J, L);
  double* o = out + (int64_t)f * kInit2Rec;
  if (energy_only) {
    if (tid == 0) {
      double e = 0.0;
      for (int r = 0; r < 15; ++r) e += J[r][33] * J[r][33];
      o[240] = e;
    }
    return;
  }
  const double es = es_p[0];
  if (tid < 15) {
    const int r = tid;
    double pi[3], pj[3];
    for (int k = 0; k < 3; ++k) {
      pi[k] = es * pvis[3 * i + k];
      pj[k] = es * pvis[3 * j + k];
    }
    double a = 0.0, b = 0.0;
    for (int k = 0; k < 3; ++k) {
      a += J[r][3 + k] * pi[k];
      b += J[r][15 + 3 + k] * pj[k];
    }
    J2[r][0] = a + b;                                   // log-scale
    J2[r][1] = J[r][30];                                // gravity tangent (J_g B)
    J2[r][2] = J[r][31];
    for (int m = 0; m < 6; ++m) J2[r][3 + m] = J[r][9 + m] + J[r][15 + 9 + m];   // shared bias
    for (int k = 0; k < 3; ++k) {
      J2[r][9 + k] = J[r][6 + k];                       // v_i
      J2[r][12 + k] = J[r][15 + 6 + k];                 // v_j
    }
    J2[r][15] = J[r][33];                               // residual
  }
  __syncthreads();
  for (int it = tid; it < 241; it += blockDim.x) {
    int ca, cb;
    if (it < 225) { ca = it / 15; cb = it % 15; }
    else if (it < 240) { ca = it - 225; cb = 15; }
    else { ca = 15; cb = 15; }
    double acc = 0.0;
    for (int r = 0; r < 15; ++r) acc += J2[r][ca] * J2[r][cb];
    o[it] = acc;
  }
}

void launch_init2_factor(const double* imu, const double* Lbuf, const int32_t* fi, const int32_t* fj, int F,
                         const double* state, const double* grav, const double* pvis, const double* es,
                         int energy_only, double* out, cudaStream_t st) {
  if (F <= 0) return;
  k_init2_factor<<<F, 64, 0, st>>>(imu, Lbuf, fi, fj, state, grav, pvis, es, energy_only, out);
  launch_count();
}

}  // namespace vba
