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
__device__ __forceinline__ M3 mTmul(const M3& a, const M3& b) {   // a^T b
  M3 c;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) c(r, k) = a(0, r) * b(0, k) + a(1, r) * b(1, k) + a(2, r) * b(2, k);
  return c;
}
__device__ __forceinline__ M3 madd(const M3& a, const M3& b, double s = 1.0) {
  M3 c;
  for (int i = 0; i < 9; ++i) c.m[i] = a.m[i] + s * b.m[i];
  return c;
}
__device__ __forceinline__ M3 mscale(const M3& a, double s) {
  M3 c;
  for (int i = 0; i < 9; ++i) c.m[i] = s * a.m[i];
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

__global__ void __launch_bounds__(64) k_preintegrate(const double* __restrict__ ts, const double* __restrict__ gyro,
                                                     const double* __restrict__ accel,
                                                     const int64_t* __restrict__ soff, int F,
                                                     const double* __restrict__ bias, const double* __restrict__ noise,
                                                     double* __restrict__ out, int* __restrict__ status) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int64_t s0 = soff[f], S = soff[f + 1] - s0;
  double* o = out + (int64_t)kPreintRec * f;
  if (S < 2) { atomicOr(status, 1); return; }                    // imu.py:87-88
  for (int64_t k = 0; k + 1 < S; ++k)
    if (!(ts[s0 + k + 1] - ts[s0 + k] > 0.0)) { atomicOr(status, 2); return; }   // imu.py:89-91
  const double bg[3] = {bias[6 * f + 0], bias[6 * f + 1], bias[6 * f + 2]};
  const double ba[3] = {bias[6 * f + 3], bias[6 * f + 4], bias[6 * f + 5]};
  const double sg2 = noise[0] * noise[0], sa2 = noise[1] * noise[1];
  M3 dR = meye(), Jr = mzero(), Jvg = mzero(), Jva = mzero(), Jpg = mzero(), Jpa = mzero();
  double dv[3] = {0, 0, 0}, dp[3] = {0, 0, 0};
  M3 C[3][3];   // cov9 as 3x3 blocks (theta, p, v)
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[i][j] = mzero();
  for (int64_t k = 0; k + 1 < S; ++k) {                          // imu.py:106-150
    const int64_t a0 = s0 + k, a1 = a0 + 1;
    const double dt = ts[a1] - ts[a0];
    double w[3], a[3], wf[3], wh[3];
    for (int c = 0; c < 3; ++c) {
      w[c] = 0.5 * ((gyro[3 * a0 + c] - bg[c]) + (gyro[3 * a1 + c] - bg[c]));
      a[c] = 0.5 * ((accel[3 * a0 + c] - ba[c]) + (accel[3 * a1 + c] - ba[c]));
      wf[c] = w[c] * dt;
      wh[c] = w[c] * (0.5 * dt);
    }
    const M3 Ef = so3_exp(wf), Eh = so3_exp(wh), Jf = so3_jr(wf), Jh = so3_jr(wh);
    const M3 Rm = mmul(dR, Eh);
    double ai[3];
    for (int r = 0; r < 3; ++r) ai[r] = Rm(r, 0) * a[0] + Rm(r, 1) * a[1] + Rm(r, 2) * a[2];
    const M3 RA = mmul(Rm, mhat(a));
    const M3 Jmid = madd(mTmul(Eh, Jr), Jh, -0.5 * dt);           // imu.py:120
    const M3 RAJmid = mmul(RA, Jmid);
    const M3 RAE = mmulT(RA, Eh);                                 // R_mid Ahat E_half^T
    const M3 RAJh = mmul(RA, Jh);
    const M3 X = mscale(RAE, -0.5 * dt * dt), Y = mscale(RAE, -dt);   // A[3:6,0:3], A[6:9,0:3]
    // M = A C  (imu.py:124-128: A = I with the blocks above, E_full^T and dt I)
    M3 Mb[3][3];
    for (int j = 0; j < 3; ++j) {
      Mb[0][j] = mTmul(Ef, C[0][j]);
      Mb[1][j] = madd(madd(mmul(X, C[0][j]), C[1][j]), C[2][j], dt);
      Mb[2][j] = madd(mmul(Y, C[0][j]), C[2][j]);
    }
    // C' = M A^T + B Qd B^T  (imu.py:130-138)
    M3 Bg[3], Bav[3];
    Bg[0] = mscale(Jf, -dt);
    Bg[1] = mscale(RAJh, 0.25 * dt * dt * dt);
    Bg[2] = mscale(RAJh, 0.5 * dt * dt);
    Bav[0] = mzero();
    Bav[1] = mscale(Rm, -0.5 * dt * dt);
    Bav[2] = mscale(Rm, -dt);
    const double qg = sg2 / dt, qa = sa2 / dt;
    M3 Cn[3][3];
    for (int i = 0; i < 3; ++i) {
      Cn[i][0] = mmul(Mb[i][0], Ef);
      Cn[i][1] = madd(madd(mmulT(Mb[i][0], X), Mb[i][1]), Mb[i][2], dt);
      Cn[i][2] = madd(mmulT(Mb[i][0], Y), Mb[i][2]);
      for (int j = 0; j < 3; ++j) {
        Cn[i][j] = madd(Cn[i][j], mmulT(Bg[i], Bg[j]), qg);
        if (i > 0 && j > 0) Cn[i][j] = madd(Cn[i][j], mmulT(Bav[i], Bav[j]), qa);
      }
    }
    for (int i = 0; i < 3; ++i)                                   // symmetrise (imu.py:139)
      for (int j = 0; j < 3; ++j)
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) C[i][j](r, c) = 0.5 * (Cn[i][j](r, c) + Cn[j][i](c, r));
    // bias Jacobians, position before velocity (imu.py:142-146)
    Jpg = madd(madd(Jpg, Jvg, dt), RAJmid, -0.5 * dt * dt);
    Jpa = madd(madd(Jpa, Jva, dt), Rm, -0.5 * dt * dt);
    Jvg = madd(Jvg, RAJmid, -dt);
    Jva = madd(Jva, Rm, -dt);
    Jr = madd(mTmul(Ef, Jr), Jf, -dt);
    for (int c = 0; c < 3; ++c) {                                  // imu.py:148-150
      dp[c] = dp[c] + dv[c] * dt + 0.5 * dt * dt * ai[c];
      dv[c] = dv[c] + dt * ai[c];
    }
    dR = mmul(dR, Ef);
  }
  const double dtt = ts[s0 + S - 1] - ts[s0];
  o[0] = dtt;
  quat_from_matrix(dR, o + 1);
  for (int c = 0; c < 3; ++c) { o[5 + c] = dp[c]; o[8 + c] = dv[c]; }
  for (int i = 0; i < 9; ++i) o[11 + i] = Jr.m[i];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      o[20 + 6 * r + c] = Jpg(r, c); o[20 + 6 * r + 3 + c] = Jpa(r, c);
      o[38 + 6 * r + c] = Jvg(r, c); o[38 + 6 * r + 3 + c] = Jva(r, c);
    }
  double* cv = o + 56;
  for (int i = 0; i < 225; ++i) cv[i] = 0.0;
  for (int bi = 0; bi < 3; ++bi)
    for (int bj = 0; bj < 3; ++bj)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) cv[(3 * bi + r) * 15 + 3 * bj + c] = C[bi][bj](r, c);
  for (int d = 0; d < 3; ++d) {                                    // imu.py:152-156
    cv[(9 + d) * 15 + 9 + d] = noise[2] * noise[2] * dtt;
    cv[(12 + d) * 15 + 12 + d] = noise[3] * noise[3] * dtt;
  }
}

void launch_preintegrate(const double* ts, const double* gyro, const double* accel, const int64_t* soff, int F,
                         const double* bias, const double* noise, double* out, int* status, cudaStream_t st) {
  if (F <= 0) return;
  k_preintegrate<<<(F + 63) / 64, 64, 0, st>>>(ts, gyro, accel, soff, F, bias, noise, out, status);
  launch_count();
}

}  // namespace vba
