// IMU preintegration between keyframe timestamps on the GPU.
//
// Restates vislam/imu.py:77-167 (`preintegrate`): midpoint scheme (the sample held
// over [t_k, t_k+1] is the endpoint average), rotation at the interval midpoint for
// position and velocity, bias Jacobians J_rot / J_pos / J_vel, and the discrete
// error-state covariance cov9 <- A cov9 A^T + B Qd B^T (symmetrised each step), all
// in fp64.  The propagation is sequential within a keyframe pair and independent
// across pairs: one thread per pair, the 9x9 covariance kept as 3x3 blocks and the
// block-sparse A (identity, E_full^T, dt I, two 3x3 couplings) and B applied in
// closed form instead of as dense 9x9 products.
//
// Output record per pair (kPreintRec doubles): dt_total, delta_R quaternion (wxyz,
// w >= 0, as Rotation.from_matrix, geometry.py:125-149), delta_p, delta_v, J_rot
// (3x3), J_pos (3x6), J_vel (3x6), covariance (15x15, row-major).

#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "vba_internal.cuh"

namespace vba {

namespace {
constexpr double kSmallAngle = 1e-8;   // geometry.py:20

struct M3 {
  double m[9];
  __device__ double& operator()(int r, int c) { return m[3 * r + c]; }
  __device__ double operator()(int r, int c) const { return m[3 * r + c]; }
};
__device__ __forceinline__ M3 mzero() { M3 a; for (int i = 0; i < 9; ++i) a.m[i] = 0.0; return a; }
__device__ __forceinline__ M3 meye() { M3 a = mzero(); a.m[0] = a.m[4] = a.m[8] = 1.0; return a; }
__device__ __forceinline__ M3 mmul(const M3& a, const M3& b) {
  M3 c;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) c(r, k) = a(r, 0) * b(0, k) + a(r, 1) * b(1, k) + a(r, 2) * b(2, k);
  return c;
}
__device__ __forceinline__ M3 mmulT(const M3& a, const M3& b) {   // a b^T
  M3 c;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) c(r, k) = a(r, 0) * b(k, 0) + a(r, 1) * b(k, 1) + a(r, 2) * b(k, 2);
  return c;
}
__device__ __forceinline__ M3 madd(const M3& a, const M3& b, double s = 1.0) {
  M3 c;
  for (int i = 0; i < 9; ++i) c.m[i] = a.m[i] + s * b.m[i];
  return c;
}
__device__ __forceinline__ M3 mhat(const double* v) {   // geometry.py:23-30
  M3 k = mzero();
  k(0, 1) = -v[2]; k(0, 2) = v[1];
  k(1, 0) = v[2];  k(1, 2) = -v[0];
  k(2, 0) = -v[1]; k(2, 1) = v[0];
  return k;
}
// geometry.py:33-43
__device__ M3 so3_exp(const double* w) {
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const M3 K = mhat(w), K2 = mmul(K, K);
  if (th < kSmallAngle) return madd(madd(meye(), K), K2, 0.5);
  return madd(madd(meye(), K, sin(th) / th), K2, (1.0 - cos(th)) / (th * th));
}
// geometry.py:57-67
__device__ M3 so3_jr(const double* w) {
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const M3 K = mhat(w), K2 = mmul(K, K);
  if (th < kSmallAngle) return madd(madd(meye(), K, -0.5), K2, 1.0 / 6.0);
  const double t2 = th * th;
  return madd(madd(meye(), K, -(1.0 - cos(th)) / t2), K2, (th - sin(th)) / (t2 * th));
}
// geometry.py:94-98, 125-149
__device__ void quat_from_matrix(const M3& R, double* q) {
  const double t = R(0, 0) + R(1, 1) + R(2, 2);
  double w, x, y, z;
  if (t > 0.0) {
    const double s = sqrt(t + 1.0) * 2.0;
    w = 0.25 * s; x = (R(2, 1) - R(1, 2)) / s; y = (R(0, 2) - R(2, 0)) / s; z = (R(1, 0) - R(0, 1)) / s;
  } else {
    int i = 0;
    if (R(1, 1) > R(i, i)) i = 1;   // np.argmax: first maximum
    if (R(2, 2) > R(i, i)) i = 2;
    if (i == 0) {
      const double s = sqrt(1.0 + R(0, 0) - R(1, 1) - R(2, 2)) * 2.0;
      w = (R(2, 1) - R(1, 2)) / s; x = 0.25 * s; y = (R(0, 1) + R(1, 0)) / s; z = (R(0, 2) + R(2, 0)) / s;
    } else if (i == 1) {
      const double s = sqrt(1.0 + R(1, 1) - R(0, 0) - R(2, 2)) * 2.0;
      w = (R(0, 2) - R(2, 0)) / s; x = (R(0, 1) + R(1, 0)) / s; y = 0.25 * s; z = (R(1, 2) + R(2, 1)) / s;
    } else {
      const double s = sqrt(1.0 + R(2, 2) - R(0, 0) - R(1, 1)) * 2.0;
      w = (R(1, 0) - R(0, 1)) / s; x = (R(0, 2) + R(2, 0)) / s; y = (R(1, 2) + R(2, 1)) / s; z = 0.25 * s;
    }
  }
  const double n = sqrt(w * w + x * x + y * y + z * z);
  const double sg = w < 0.0 ? -1.0 : 1.0;
  q[0] = sg * w / n; q[1] = sg * x / n; q[2] = sg * y / n; q[3] = sg * z / n;
}
}  // namespace

// Phase 1 (one thread per sample interval, fully parallel): everything of a step that
// depends only on the samples -- dt, the bias-corrected midpoint accel, and the
// exponentials / right Jacobians of the full and half rotation increments
// (imu.py:107-117) plus the state-free factors of R_mid Ahat E_half^T and
// R_mid Ahat Jr_half (R_mid = dR E_half): P1 = E_half Ahat E_half^T, P2 = E_half Ahat
// Jr_half, so both are one 3x3 product from dR in the sequential pass, and the noise
// scalings.  Record layout: dt, a[3], Ef[9], Eh[9], Jf[9], Jh[9], P1[9], P2[9], qg, qa.
constexpr int kStepRec = 60;

__global__ void __launch_bounds__(128) k_preint_steps(const double* __restrict__ ts, const double* __restrict__ gyro,
                                                      const double* __restrict__ accel,
                                                      const int64_t* __restrict__ soff, int F, int64_t S,
                                                      const double* __restrict__ bias,
                                                      const double* __restrict__ noise, double* __restrict__ steps,
                                                      int* __restrict__ status) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0 && soff[F] != S) atomicOr(status, 4);
  if (s >= S) return;
  int lo = 0, hi = F;   // pair f with soff[f] <= s < soff[f+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (soff[mid] <= s) lo = mid; else hi = mid;
  }
  const int f = lo;
  if (s + 1 >= soff[f + 1]) return;   // last sample of its pair
  const double dt = ts[s + 1] - ts[s];
  if (!(dt > 0.0)) { atomicOr(status, 2); return; }   // imu.py:89-91
  double w[3], wf[3], wh[3];
  double* r = steps + kStepRec * s;
  r[0] = dt;
  for (int c = 0; c < 3; ++c) {
    const double bg = bias[6 * f + c], ba = bias[6 * f + 3 + c];
    w[c] = 0.5 * ((gyro[3 * s + c] - bg) + (gyro[3 * s + 3 + c] - bg));
    r[1 + c] = 0.5 * ((accel[3 * s + c] - ba) + (accel[3 * s + 3 + c] - ba));
    wf[c] = w[c] * dt;
    wh[c] = w[c] * (0.5 * dt);
  }
  const M3 Ef = so3_exp(wf), Eh = so3_exp(wh), Jf = so3_jr(wf), Jh = so3_jr(wh);
  const double av[3] = {r[1], r[2], r[3]};
  const M3 EA = mmul(Eh, mhat(av));
  const M3 P1 = mmulT(EA, Eh), P2 = mmul(EA, Jh);
  for (int i = 0; i < 9; ++i) {
    r[4 + i] = Ef.m[i]; r[13 + i] = Eh.m[i]; r[22 + i] = Jf.m[i]; r[31 + i] = Jh.m[i];
    r[40 + i] = P1.m[i]; r[49 + i] = P2.m[i];
  }
  r[58] = noise[0] * noise[0] / dt;   // Qd diagonal (imu.py:137)
  r[59] = noise[1] * noise[1] / dt;
}

// Phase 2: the sequential propagation, 16 lanes per keyframe pair (two pairs per warp).
// The covariance recursion cov9 <- A cov9 A^T + B Qd B^T splits by columns: column c of
// M = A cov9 needs only column c of cov9, row r of M A^T only row r of M.  Lane c (< 9)
// owns column c of cov9 and row c of the product, the two exchanged through shared
// memory; the bias Jacobians split the same way over their 3 columns (lanes 0-2).
// dR, dp, dv and the 3x3 step matrices are replicated per lane (cheap, deterministic).
// Step records are double-buffered in shared memory: each lane loads its part of step
// k+1 into registers at the top of step k and stores it to shared memory at the end, so
// the global-load latency hides behind the step's arithmetic.
constexpr int kPairsPerBlock = 8;
struct PairSmem {
  double rec[2][kStepRec];
  double M[81];    // M = A cov9, written by columns, read by rows
  double Cp[81];   // C' rows, read by columns for the symmetrisation
  double RJ[9];    // R_mid Ahat Jr_half of the current step
  double Rm[9];    // R_mid of the current step
};

__device__ __forceinline__ double at3(const double* p, int i, int j) { return p[3 * i + j]; }

__global__ void __launch_bounds__(16 * kPairsPerBlock) k_preint_propagate(const double* __restrict__ ts,
                                                                         const int64_t* __restrict__ soff, int F,
                                                                         int64_t n_samples,
                                                                         const double* __restrict__ steps,
                                                                         const double* __restrict__ noise,
                                                                         double* __restrict__ out,
                                                                         int* __restrict__ status) {
  __shared__ PairSmem sm_all[kPairsPerBlock];
  const int grp = threadIdx.x >> 4, c = threadIdx.x & 15;
  const int f = blockIdx.x * kPairsPerBlock + grp;
  if (f >= F) return;
  const unsigned mask = 0xFFFFu << (threadIdx.x & 16);
  PairSmem& sm = sm_all[grp];
  const int64_t s0 = soff[f], S = soff[f + 1] - s0;
  // a malformed soff must not send this pass outside the step records (the step pass, which
  // checks soff[F] == n_samples, is skipped when there are no samples at all)
  if (s0 < 0 || soff[f + 1] > n_samples || soff[f + 1] < s0) { if (c == 0) atomicOr(status, 4); return; }
  if (S < 2) { if (c == 0) atomicOr(status, 1); return; }   // imu.py:87-88
  const bool cov_lane = c < 9, jac_lane = c < 3;
  const int br = cov_lane ? c / 3 : 0, rr = cov_lane ? c % 3 : 0;   // lane's row block / row in block
  M3 dR = meye();
  double dp[3] = {0, 0, 0}, dv[3] = {0, 0, 0};
  double Cc[9];                                   // column c of cov9
  for (int i = 0; i < 9; ++i) Cc[i] = 0.0;
  double jr[3] = {0, 0, 0}, jpg[3] = {0, 0, 0}, jvg[3] = {0, 0, 0}, jpa[3] = {0, 0, 0}, jva[3] = {0, 0, 0};
  const double* st = steps + kStepRec * s0;
  for (int i = c; i < kStepRec; i += 16) sm.rec[0][i] = st[i];
  __syncwarp(mask);
  for (int64_t k = 0; k + 1 < S; ++k) {
    const double* r = sm.rec[k & 1];
    double pf[4] = {0.0, 0.0, 0.0, 0.0};          // step k+1, loaded now, stored at the end of step k
    if (k + 2 < S)
      for (int q = 0; q < 4; ++q)
        if (c + 16 * q < kStepRec) pf[q] = __ldg(st + kStepRec * (k + 1) + c + 16 * q);
    const double* Ef = r + 4;
    const double* Eh = r + 13;
    const double* Jf = r + 22;
    const double* Jh = r + 31;
    const double dt = r[0];
    const double a[3] = {r[1], r[2], r[3]};
    const double* P1 = r + 40;
    const double* P2 = r + 49;
    M3 Rm, RAE, RAJh;   // R_mid, R_mid Ahat E_half^T = dR P1, R_mid Ahat Jr_half = dR P2
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        Rm(i, j) = dR(i, 0) * at3(Eh, 0, j) + dR(i, 1) * at3(Eh, 1, j) + dR(i, 2) * at3(Eh, 2, j);
        RAE(i, j) = dR(i, 0) * at3(P1, 0, j) + dR(i, 1) * at3(P1, 1, j) + dR(i, 2) * at3(P1, 2, j);
        RAJh(i, j) = dR(i, 0) * at3(P2, 0, j) + dR(i, 1) * at3(P2, 1, j) + dR(i, 2) * at3(P2, 2, j);
      }
    if (c == 0)
      for (int i = 0; i < 9; ++i) { sm.RJ[i] = RAJh.m[i]; sm.Rm[i] = Rm.m[i]; }
    const double hx = -0.5 * dt * dt, hy = -dt;   // X = hx * RAE, Y = hy * RAE
    if (cov_lane) {                               // column c of M = A cov9 (imu.py:124-128)
      for (int i = 0; i < 3; ++i) {
        const double e0 = at3(Ef, 0, i) * Cc[0] + at3(Ef, 1, i) * Cc[1] + at3(Ef, 2, i) * Cc[2];
        const double x0 = RAE(i, 0) * Cc[0] + RAE(i, 1) * Cc[1] + RAE(i, 2) * Cc[2];
        sm.M[9 * i + c] = e0;
        sm.M[9 * (3 + i) + c] = hx * x0 + Cc[3 + i] + dt * Cc[6 + i];
        sm.M[9 * (6 + i) + c] = hy * x0 + Cc[6 + i];
      }
    }
    __syncwarp(mask);
    if (cov_lane) {                               // row c of C' = M A^T + B Qd B^T (imu.py:130-138)
      double mr[9], cp[9];
      for (int j = 0; j < 9; ++j) mr[j] = sm.M[9 * c + j];
      for (int j = 0; j < 3; ++j) {
        const double x0 = mr[0] * RAE(j, 0) + mr[1] * RAE(j, 1) + mr[2] * RAE(j, 2);
        cp[j] = mr[0] * at3(Ef, 0, j) + mr[1] * at3(Ef, 1, j) + mr[2] * at3(Ef, 2, j);
        cp[3 + j] = hx * x0 + mr[3 + j] + dt * mr[6 + j];
        cp[6 + j] = hy * x0 + mr[6 + j];
      }
      // B rows: gyro part s_b * G_b (G_0 = Jr_full, G_1 = G_2 = R_mid Ahat Jr_half),
      // accel part t_b * R_mid (t_0 = 0), b = row block
      const double s1 = 0.25 * dt * dt * dt, s2 = 0.5 * dt * dt, t1 = -0.5 * dt * dt, t2 = -dt;
      const double qg = r[58], qa = r[59];
      const double sr = br == 0 ? -dt : (br == 1 ? s1 : s2), tr = br == 0 ? 0.0 : (br == 1 ? t1 : t2);
      const double* gp = br == 0 ? Jf : sm.RJ;
      const double g0 = sr * gp[3 * rr], g1 = sr * gp[3 * rr + 1], g2 = sr * gp[3 * rr + 2];
      const double a0 = tr * sm.Rm[3 * rr], a1 = tr * sm.Rm[3 * rr + 1], a2 = tr * sm.Rm[3 * rr + 2];
      for (int j = 0; j < 9; ++j) {
        const int bj = j / 3, rj = j % 3;
        const double sj = bj == 0 ? -dt : (bj == 1 ? s1 : s2), tj = bj == 0 ? 0.0 : (bj == 1 ? t1 : t2);
        const double* gq = bj == 0 ? Jf : sm.RJ;
        const double gg = g0 * (sj * gq[3 * rj]) + g1 * (sj * gq[3 * rj + 1]) + g2 * (sj * gq[3 * rj + 2]);
        const double aa = a0 * (tj * sm.Rm[3 * rj]) + a1 * (tj * sm.Rm[3 * rj + 1]) + a2 * (tj * sm.Rm[3 * rj + 2]);
        cp[j] = cp[j] + qg * gg + qa * aa;
        sm.Cp[9 * c + j] = cp[j];
      }
      __syncwarp(mask & 0x01FF01FFu);
      for (int i = 0; i < 9; ++i) Cc[i] = 0.5 * (sm.Cp[9 * i + c] + cp[i]);   // symmetrise (imu.py:139)
    }
    if (jac_lane) {                               // bias Jacobian column c (imu.py:120, 142-146)
      double jm[3], rj[3], jn[3];
      for (int i = 0; i < 3; ++i)
        jm[i] = at3(Eh, 0, i) * jr[0] + at3(Eh, 1, i) * jr[1] + at3(Eh, 2, i) * jr[2] - 0.5 * dt * at3(Jh, i, c);
      const double ax[3] = {a[1] * jm[2] - a[2] * jm[1], a[2] * jm[0] - a[0] * jm[2], a[0] * jm[1] - a[1] * jm[0]};
      for (int i = 0; i < 3; ++i) rj[i] = Rm(i, 0) * ax[0] + Rm(i, 1) * ax[1] + Rm(i, 2) * ax[2];   // R_mid Ahat J_mid
      for (int i = 0; i < 3; ++i)
        jn[i] = at3(Ef, 0, i) * jr[0] + at3(Ef, 1, i) * jr[1] + at3(Ef, 2, i) * jr[2] - dt * at3(Jf, i, c);
      for (int i = 0; i < 3; ++i) {
        const double rmc = sm.Rm[3 * i + c];
        jpg[i] += dt * jvg[i] - 0.5 * dt * dt * rj[i];
        jpa[i] += dt * jva[i] - 0.5 * dt * dt * rmc;
        jvg[i] += -dt * rj[i];
        jva[i] += -dt * rmc;
        jr[i] = jn[i];
      }
    }
    for (int i = 0; i < 3; ++i) {                 // imu.py:148-150
      const double ai = Rm(i, 0) * a[0] + Rm(i, 1) * a[1] + Rm(i, 2) * a[2];
      dp[i] = dp[i] + dv[i] * dt + 0.5 * dt * dt * ai;
      dv[i] = dv[i] + dt * ai;
    }
    M3 dn;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) dn(i, j) = dR(i, 0) * at3(Ef, 0, j) + dR(i, 1) * at3(Ef, 1, j) + dR(i, 2) * at3(Ef, 2, j);
    dR = dn;
    if (k + 2 < S)
      for (int q = 0; q < 4; ++q)
        if (c + 16 * q < kStepRec) sm.rec[(k + 1) & 1][c + 16 * q] = pf[q];
    __syncwarp(mask);   // rec[k+1] landed; M, Cp, RJ, Rm free for the next step
  }
  double* o = out + (int64_t)kPreintRec * f;
  double* cv = o + 56;
  const double dtt = ts[s0 + S - 1] - ts[s0];
  if (c == 0) {
    o[0] = dtt;
    quat_from_matrix(dR, o + 1);
    for (int i = 0; i < 3; ++i) { o[5 + i] = dp[i]; o[8 + i] = dv[i]; }
  }
  if (jac_lane)
    for (int i = 0; i < 3; ++i) {
      o[11 + 3 * i + c] = jr[i];
      o[20 + 6 * i + c] = jpg[i]; o[20 + 6 * i + 3 + c] = jpa[i];
      o[38 + 6 * i + c] = jvg[i]; o[38 + 6 * i + 3 + c] = jva[i];
    }
  for (int r = 0; r < 15; ++r) {                  // lane c writes column c (cov9 or bias-walk block)
    double v = 0.0;
    if (c < 9) v = r < 9 ? Cc[r] : 0.0;
    if (c < 15 && c >= 9 && r == c) v = (c < 12 ? noise[2] * noise[2] : noise[3] * noise[3]) * dtt;   // imu.py:152-156
    if (c < 15) cv[15 * r + c] = v;
  }
}

// Phase 2, log-depth variant (default): the recursion of a pair is an affine map of the
// state (dp, dv, cov9, bias Jacobians) once the rotation before each step is known, and such
// maps compose associatively.  One warp per pair: lane L takes a contiguous chunk of steps;
//   1. rotation: each lane multiplies its chunk's Exp(w dt) factors, a warp scan of 3x3
//      products (shuffles) gives every chunk its starting dR;
//   2. each lane composes its chunk's steps into one aggregate map (below) from the true dR;
//   3. a 5-level tree combines the 32 aggregates in chunk order; lane 0 writes the record.
// Aggregate (per lane, in shared memory, element e of lane L at e * 32 + L):
//   cov:  Phi = [[R,0,0],[X,I,T I],[Y,0,I]] (error-state transition), C (accumulated noise):
//         (Phi2, C2) o (Phi1, C1) = (Phi2 Phi1, Phi2 C1 Phi2^T + C2)
//   bias Jacobians (gyro, state [J_rot; J_vel; J_pos]): M = [[R,0,0],[JX,I,0],[JY,T I,I]] and
//         offsets O = [OR; OV; OP]:  (M2, O2) o (M1, O1) = (M2 M1, M2 O1 + O2)
//   dp/dv and the accel Jacobians: dv = dv0 + V, dp = dp0 + T dv0 + P (and J_vel/J_pos accel
//         columns alike with VA, PA).
// A step is the aggregate of one interval (R = Ef^T, X = -dt^2/2 RAE, Y = -dt RAE, C = B Qd B^T,
// ...), combined onto the running one, so the step update and the tree share one function.
// fp64 throughout; the reassociation moves results by ~1e-16 relative (parity tests: 1e-12).
namespace {
constexpr int kAR = 0, kAX = 9, kAY = 18, kAT = 27, kAC = 28, kJX = 109, kJY = 118, kOR = 127, kOV = 136,
              kOP = 145, kAP = 154, kAV = 157, kPA = 160, kVA = 169, kAggN = 178;
struct AggRef {   // one lane's aggregate in shared memory
  double* b;
  __device__ double& operator[](int e) const { return b[e * 32]; }
};
// 3x3 helpers on strided aggregate storage (row-major 3x3 at element offset e)
__device__ __forceinline__ void m3_load(const AggRef& a, int e, double* m) {
  for (int i = 0; i < 9; ++i) m[i] = a[e + i];
}
__device__ __forceinline__ void m3_store(const AggRef& a, int e, const double* m) {
  for (int i = 0; i < 9; ++i) a[e + i] = m[i];
}
__device__ __forceinline__ void mm3(const double* A, const double* B, double* C) {   // C = A B
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) C[3 * r + c] = A[3 * r] * B[c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
}
__device__ __forceinline__ void mm3T(const double* A, const double* B, double* C) {   // C = A B^T
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = A[3 * r] * B[3 * c] + A[3 * r + 1] * B[3 * c + 1] + A[3 * r + 2] * B[3 * c + 2];
}
// e1 (earlier, in/out) := e2 (later) o e1
__device__ void agg_combine(const AggRef& e2, const AggRef& e1) {
  double R1[9], R2[9], X1[9], X2[9], Y1[9], Y2[9], t[9], u[9];
  const double T1 = e1[kAT], T2 = e2[kAT];
  m3_load(e1, kAR, R1); m3_load(e2, kAR, R2);
  m3_load(e2, kAX, X2); m3_load(e2, kAY, Y2);
  // covariance: C = Phi2 C1 Phi2^T + C2 by 3x3 blocks, B = Phi2 C1 first
  double B[3][3][9];
  {
    double Cb[3][9];
    for (int j = 0; j < 3; ++j) {
      for (int bi = 0; bi < 3; ++bi)
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) Cb[bi][3 * r + c] = e1[kAC + 9 * (3 * bi + r) + 3 * j + c];
      // column block j of C1: Cb[bi] = C1_{bi, j}
      mm3(R2, Cb[0], B[0][j]);
      mm3(X2, Cb[0], t);
      mm3(Y2, Cb[0], u);
      for (int q = 0; q < 9; ++q) {
        B[1][j][q] = t[q] + Cb[1][q] + T2 * Cb[2][q];
        B[2][j][q] = u[q] + Cb[2][q];
      }
    }
  }
  for (int i = 0; i < 3; ++i) {   // row block i of B Phi2^T:  [B_i0 R2^T, B_i0 X2^T + B_i1 + T2 B_i2, B_i0 Y2^T + B_i2]
    double D0[9], D1[9], D2[9];
    mm3T(B[i][0], R2, D0);
    mm3T(B[i][0], X2, D1);
    mm3T(B[i][0], Y2, D2);
    for (int q = 0; q < 9; ++q) {
      D1[q] += B[i][1][q] + T2 * B[i][2][q];
      D2[q] += B[i][2][q];
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        const int row = 9 * (3 * i + r);
        e1[kAC + row + c] = D0[3 * r + c] + e2[kAC + row + c];
        e1[kAC + row + 3 + c] = D1[3 * r + c] + e2[kAC + row + 3 + c];
        e1[kAC + row + 6 + c] = D2[3 * r + c] + e2[kAC + row + 6 + c];
      }
  }
  // symmetrise (imu.py:139: the sequential recursion does it every step)
  for (int r = 0; r < 9; ++r)
    for (int c = r + 1; c < 9; ++c) {
      const double v = 0.5 * (e1[kAC + 9 * r + c] + e1[kAC + 9 * c + r]);
      e1[kAC + 9 * r + c] = v;
      e1[kAC + 9 * c + r] = v;
    }
  // covariance transition: X = X2 R1 + X1 + T2 Y1, Y = Y2 R1 + Y1
  m3_load(e1, kAX, X1); m3_load(e1, kAY, Y1);
  mm3(X2, R1, t);
  for (int q = 0; q < 9; ++q) t[q] += X1[q] + T2 * Y1[q];
  m3_store(e1, kAX, t);
  mm3(Y2, R1, t);
  for (int q = 0; q < 9; ++q) t[q] += Y1[q];
  m3_store(e1, kAY, t);
  // Jacobian maps: offsets first (they read the earlier JX1 .. through O1 only)
  double OR1[9], OV1[9], OP1[9], JX2[9], JY2[9];
  m3_load(e1, kOR, OR1); m3_load(e1, kOV, OV1); m3_load(e1, kOP, OP1);
  m3_load(e2, kJX, JX2); m3_load(e2, kJY, JY2);
  mm3(R2, OR1, t);
  for (int q = 0; q < 9; ++q) t[q] += e2[kOR + q];
  m3_store(e1, kOR, t);
  mm3(JX2, OR1, t);
  for (int q = 0; q < 9; ++q) t[q] += OV1[q] + e2[kOV + q];
  m3_store(e1, kOV, t);
  mm3(JY2, OR1, t);
  for (int q = 0; q < 9; ++q) t[q] += T2 * OV1[q] + OP1[q] + e2[kOP + q];
  m3_store(e1, kOP, t);
  // M = M2 M1: JX = JX2 R1 + JX1, JY = JY2 R1 + T2 JX1 + JY1
  double JX1[9], JY1[9];
  m3_load(e1, kJX, JX1); m3_load(e1, kJY, JY1);
  mm3(JX2, R1, t);
  for (int q = 0; q < 9; ++q) t[q] += JX1[q];
  m3_store(e1, kJX, t);
  mm3(JY2, R1, t);
  for (int q = 0; q < 9; ++q) t[q] += T2 * JX1[q] + JY1[q];
  m3_store(e1, kJY, t);
  // dp/dv and the accel Jacobians
  for (int q = 0; q < 3; ++q) {
    const double v1 = e1[kAV + q];
    e1[kAP + q] = e1[kAP + q] + e2[kAP + q] + T2 * v1;
    e1[kAV + q] = v1 + e2[kAV + q];
  }
  for (int q = 0; q < 9; ++q) {
    const double v1 = e1[kVA + q];
    e1[kPA + q] = e1[kPA + q] + e2[kPA + q] + T2 * v1;
    e1[kVA + q] = v1 + e2[kVA + q];
  }
  mm3(R2, R1, t);
  m3_store(e1, kAR, t);
  e1[kAT] = T1 + T2;
}
__device__ void agg_identity(const AggRef& a) {
  for (int e = 0; e < kAggN; ++e) a[e] = 0.0;
  a[kAR] = a[kAR + 4] = a[kAR + 8] = 1.0;
}
}  // namespace

constexpr int kScanWarps = 2;   // pairs per CTA
__global__ void __launch_bounds__(32 * kScanWarps) k_preint_scan(const double* __restrict__ ts,
                                                                 const int64_t* __restrict__ soff, int F,
                                                                 int64_t n_samples,
                                                                 const double* __restrict__ steps,
                                                                 const double* __restrict__ noise,
                                                                 double* __restrict__ out, int* __restrict__ status) {
  extern __shared__ double scan_sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * kScanWarps + w;
  if (f >= F) return;
  double* base = scan_sm + (size_t)w * 2 * kAggN * 32;
  const AggRef run{base + lane}, stp{base + kAggN * 32 + lane};
  const int64_t s0 = soff[f], S = soff[f + 1] - s0;
  if (s0 < 0 || soff[f + 1] > n_samples || soff[f + 1] < s0) { if (lane == 0) atomicOr(status, 4); return; }
  if (S < 2) { if (lane == 0) atomicOr(status, 1); return; }
  const int64_t n = S - 1, ch = (n + 31) / 32, k0 = lane * ch, k1 = k0 + ch < n ? k0 + ch : n;
  const double* st = steps + kStepRec * s0;
  // 1. rotation prefix: Pr = product of this chunk's Ef, then an inclusive warp scan
  double Pr[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[9];
  for (int64_t k = k0; k < k1; ++k) {
    mm3(Pr, st + kStepRec * k + 4, t);
    for (int q = 0; q < 9; ++q) Pr[q] = t[q];
  }
  for (int d = 1; d < 32; d <<= 1) {
    double o[9];
    for (int q = 0; q < 9; ++q) o[q] = __shfl_up_sync(0xffffffffu, Pr[q], d);
    if (lane >= d) {
      mm3(o, Pr, t);
      for (int q = 0; q < 9; ++q) Pr[q] = t[q];
    }
  }
  double dR[9];   // rotation before this chunk (exclusive scan)
  for (int q = 0; q < 9; ++q) {
    const double v = __shfl_up_sync(0xffffffffu, Pr[q], 1);
    dR[q] = lane == 0 ? (q % 4 == 0 ? 1.0 : 0.0) : v;
  }
  double dRtot[9];
  for (int q = 0; q < 9; ++q) dRtot[q] = __shfl_sync(0xffffffffu, Pr[q], 31);
  // 2. this chunk's aggregate
  agg_identity(run);
  for (int64_t k = k0; k < k1; ++k) {
    const double* r = st + kStepRec * k;
    const double dt = r[0];
    const double* Ef = r + 4;
    const double* Eh = r + 13;
    const double* Jf = r + 22;
    const double* Jh = r + 31;
    double Rm[9], RAE[9], RJ[9], E[9];
    mm3(dR, Eh, Rm);
    mm3(dR, r + 40, RAE);
    mm3(dR, r + 49, RJ);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) E[3 * i + j] = Ef[3 * j + i];
    m3_store(stp, kAR, E);
    for (int q = 0; q < 9; ++q) {
      stp[kAX + q] = -0.5 * dt * dt * RAE[q];
      stp[kAY + q] = -dt * RAE[q];
    }
    stp[kAT] = dt;
    // B Qd B^T: row c = (block br, row rr); gyro rows s_b G_b, accel rows t_b Rm (imu.py:130-138)
    const double qg = r[58], qa = r[59];
    const double s1 = 0.25 * dt * dt * dt, s2 = 0.5 * dt * dt, t1 = -0.5 * dt * dt, t2 = -dt;
    for (int c = 0; c < 9; ++c) {
      const int br = c / 3, rr = c % 3;
      const double sr = br == 0 ? -dt : (br == 1 ? s1 : s2), tr = br == 0 ? 0.0 : (br == 1 ? t1 : t2);
      const double* gp = br == 0 ? Jf : RJ;
      const double g0 = sr * gp[3 * rr], g1 = sr * gp[3 * rr + 1], g2 = sr * gp[3 * rr + 2];
      const double a0 = tr * Rm[3 * rr], a1 = tr * Rm[3 * rr + 1], a2 = tr * Rm[3 * rr + 2];
      for (int j = 0; j < 9; ++j) {
        const int bj = j / 3, rj = j % 3;
        const double sj = bj == 0 ? -dt : (bj == 1 ? s1 : s2), tj = bj == 0 ? 0.0 : (bj == 1 ? t1 : t2);
        const double* gq = bj == 0 ? Jf : RJ;
        const double gg = g0 * (sj * gq[3 * rj]) + g1 * (sj * gq[3 * rj + 1]) + g2 * (sj * gq[3 * rj + 2]);
        const double aa = a0 * (tj * Rm[3 * rj]) + a1 * (tj * Rm[3 * rj + 1]) + a2 * (tj * Rm[3 * rj + 2]);
        stp[kAC + 9 * c + j] = qg * gg + qa * aa;
      }
    }
    // Jacobian step map: G = Rm [a]x Eh^T, h = Rm [a]x Jh (imu.py:120, 142-146)
    const double a[3] = {r[1], r[2], r[3]};
    double AxEt[9], Axh[9], G[9], h[9];
    for (int c = 0; c < 3; ++c) {   // column c of [a]x Eh^T and [a]x Jh
      const double e0 = Eh[3 * c], e1 = Eh[3 * c + 1], e2 = Eh[3 * c + 2];   // (Eh^T)[:, c] = row c of Eh
      AxEt[c] = a[1] * e2 - a[2] * e1; AxEt[3 + c] = a[2] * e0 - a[0] * e2; AxEt[6 + c] = a[0] * e1 - a[1] * e0;
      const double j0 = Jh[c], j1 = Jh[3 + c], j2 = Jh[6 + c];
      Axh[c] = a[1] * j2 - a[2] * j1; Axh[3 + c] = a[2] * j0 - a[0] * j2; Axh[6 + c] = a[0] * j1 - a[1] * j0;
    }
    mm3(Rm, AxEt, G);
    mm3(Rm, Axh, h);
    for (int q = 0; q < 9; ++q) {
      stp[kJX + q] = -dt * G[q];
      stp[kJY + q] = -0.5 * dt * dt * G[q];
      stp[kOR + q] = -dt * Jf[q];
      stp[kOV + q] = 0.5 * dt * dt * h[q];
      stp[kOP + q] = 0.25 * dt * dt * dt * h[q];
      stp[kPA + q] = -0.5 * dt * dt * Rm[q];
      stp[kVA + q] = -dt * Rm[q];
    }
    for (int i = 0; i < 3; ++i) {
      const double ai = Rm[3 * i] * a[0] + Rm[3 * i + 1] * a[1] + Rm[3 * i + 2] * a[2];
      stp[kAP + i] = 0.5 * dt * dt * ai;
      stp[kAV + i] = dt * ai;
    }
    agg_combine(stp, run);
    mm3(dR, Ef, t);
    for (int q = 0; q < 9; ++q) dR[q] = t[q];
  }
  // 3. ordered tree over the chunks
  for (int d = 1; d < 32; d <<= 1) {
    __syncwarp();
    if ((lane & (2 * d - 1)) == 0 && lane + d < 32) agg_combine(AggRef{base + lane + d}, run);
  }
  __syncwarp();
  if (lane != 0) return;
  double* o = out + (int64_t)kPreintRec * f;
  const double dtt = ts[s0 + S - 1] - ts[s0];
  o[0] = dtt;
  M3 R;
  for (int q = 0; q < 9; ++q) R.m[q] = dRtot[q];
  quat_from_matrix(R, o + 1);
  for (int i = 0; i < 3; ++i) { o[5 + i] = run[kAP + i]; o[8 + i] = run[kAV + i]; }
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) {
      o[11 + 3 * i + c] = run[kOR + 3 * i + c];
      o[20 + 6 * i + c] = run[kOP + 3 * i + c];
      o[20 + 6 * i + 3 + c] = run[kPA + 3 * i + c];
      o[38 + 6 * i + c] = run[kOV + 3 * i + c];
      o[38 + 6 * i + 3 + c] = run[kVA + 3 * i + c];
    }
  double* cv = o + 56;
  for (int r = 0; r < 15; ++r)
    for (int c = 0; c < 15; ++c) {
      double v = 0.0;
      if (r < 9 && c < 9) v = run[kAC + 9 * r + c];
      else if (r == c) v = (c < 12 ? noise[2] * noise[2] : noise[3] * noise[3]) * dtt;   // imu.py:152-156
      cv[15 * r + c] = v;
    }
}

// Preintegration record -> IMU factor record of the solver (include/vba.h VBA_IMU_REC):
// the first 56 doubles are shared, then cov[0:9,0:9], cov[9:15,9:15], the bias
// linearisation point.  One thread per output double.
__global__ void k_preint_pack(const double* __restrict__ rec, const double* __restrict__ bias, int F,
                              double* __restrict__ imu) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)F * kImuRec) return;
  const int f = (int)(t / kImuRec), i = (int)(t % kImuRec);
  const double* r = rec + (int64_t)kPreintRec * f;
  double v = 0.0;
  if (i < 56) v = r[i];
  else if (i < 137) v = r[56 + ((i - 56) / 9) * 15 + (i - 56) % 9];
  else if (i < 173) v = r[56 + (9 + (i - 137) / 6) * 15 + 9 + (i - 137) % 6];
  else if (i < 179) v = bias[6 * f + (i - 173)];
  imu[t] = v;
}

void launch_preint_pack(const double* rec, const double* bias, int F, double* imu, cudaStream_t st) {
  if (F <= 0) return;
  const int64_t n = (int64_t)F * kImuRec;
  k_preint_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rec, bias, F, imu);
  launch_count();
}

size_t preint_scratch_bytes(int64_t S) { return sizeof(double) * kStepRec * (size_t)(S > 0 ? S : 1); }

void launch_preintegrate(const double* ts, const double* gyro, const double* accel, int64_t S, const int64_t* soff,
                         int F, const double* bias, const double* noise, double* scratch, double* out, int* status,
                         cudaStream_t st) {
  if (F <= 0) return;
  if (S > 0) {
    k_preint_steps<<<(unsigned)((S + 127) / 128), 128, 0, st>>>(ts, gyro, accel, soff, F, S, bias, noise, scratch,
                                                                status);
    launch_count();
  }
  // the log-depth scan wins from ~64 intervals per pair (256 x 200: 0.14 vs 0.30 ms); with
  // short pairs the 32-chunk tree costs more than the sequential steps it replaces (1024 x 40:
  // 0.22 vs 0.11 ms).  VBA_PREINT=seq / scan forces either.
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_preint_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * 2 * kAggN * 32 * kScanWarps));
    attr = true;
  }
  const char* e = getenv("VBA_PREINT");   // read per call (tests switch it)
  const int force = !e ? -1 : (e[0] == 's' && e[1] == 'e') ? 1 : (e[0] == 's' && e[1] == 'c') ? 0 : -1;
  const bool seq = force >= 0 ? force == 1 : S < (int64_t)64 * F;
  if (seq)
    k_preint_propagate<<<(F + kPairsPerBlock - 1) / kPairsPerBlock, 16 * kPairsPerBlock, 0, st>>>(
        ts, soff, F, S, scratch, noise, out, status);
  else
    k_preint_scan<<<(F + kScanWarps - 1) / kScanWarps, 32 * kScanWarps,
                    sizeof(double) * 2 * kAggN * 32 * kScanWarps, st>>>(ts, soff, F, S, scratch, noise, out, status);
  launch_count();
}

}  // namespace vba
