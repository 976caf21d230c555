// vba_init.cu — stage-2 inertial-only initialisation on the GPU.
//
// Replaces vislam.initialization.init_inertial_only (/root/reference/pkg/src/vislam/
// initialization.py:152-231): with the vision rotations and (unscaled) positions frozen, a
// damped Gauss-Newton over x = [log-scale s, gravity tangent (2), one shared bias (6),
// per-keyframe velocities (3K)] on the inertial residuals of the scale-adjusted states
// (positions exp(s) p_vision, initialization.py:137-149).
//
//   k_init2_factor   (vba_imu.cu) per factor: the whitened inertial Jacobian (the VI-BA
//                    factor kernel's own residual / Jacobian / whitening), re-expressed in the
//                    stage-2 unknowns, its 15x15 Gram, gradient and energy
//   k_init2_assemble dense H, g (9+3K), fixed factor order (initialization.py:179-190)
//   k_init2_solve    one CTA: (H + diag(H) lam + 1e-10 I) dx = -g by LU with partial pivoting
//                    (np.linalg.solve's algorithm); an exactly zero pivot = LinAlgError
//   k_init2_update   trial state: s + dx_0, R_wg Exp(B dx_1:3), bias + dx_3:9, v + dx_9:
// The LM driver (host) follows initialization.py:174-229 line by line.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "vba_internal.cuh"

namespace vba {

constexpr int kInit2SmemDim = 160;   // k_init2_solve keeps A (+ b) in shared memory up to this size

// virtual keyframe states [K,16] of the stage-2 estimate: q (vision), exp(s) p, v, shared bias
__global__ void k_init2_states(const double* __restrict__ q, const double* __restrict__ p, const double* __restrict__ v,
                               const double* __restrict__ x, int K, double* __restrict__ state,
                               double* __restrict__ es_out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const double es = exp(x[0]);   // float(np.exp(s)) (initialization.py:139)
  if (k == 0) es_out[0] = es;
  if (k >= K) return;
  double* o = state + 16 * k;
  for (int a = 0; a < 4; ++a) o[a] = q[4 * k + a];
  for (int a = 0; a < 3; ++a) o[4 + a] = es * p[3 * k + a];
  for (int a = 0; a < 3; ++a) o[7 + a] = v[3 * k + a];
  for (int a = 0; a < 6; ++a) o[10 + a] = x[3 + a];
}

__global__ void k_init2_assemble(const double* __restrict__ rec, const int32_t* __restrict__ fi,
                                 const int32_t* __restrict__ fj, int F, int dim, double* __restrict__ H,
                                 double* __restrict__ g) {
  const int a = blockIdx.x;
  auto loc = [](int col, int i, int j) {
    if (col < 9) return col;
    const int kf = (col - 9) / 3, c = (col - 9) % 3;
    if (kf == i) return 9 + c;
    if (kf == j) return 12 + c;
    return -1;
  };
  for (int b = threadIdx.x; b < dim; b += blockDim.x) {
    double v = 0.0;
    for (int f = 0; f < F; ++f) {   // H += J^T J per factor, in factor order
      const int la = loc(a, fi[f], fj[f]), lb = loc(b, fi[f], fj[f]);
      if (la >= 0 && lb >= 0) v += rec[(int64_t)f * kInit2Rec + la * 15 + lb];
    }
    H[(int64_t)a * dim + b] = v;
  }
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int f = 0; f < F; ++f) {
      const int la = loc(a, fi[f], fj[f]);
      if (la >= 0) v += rec[(int64_t)f * kInit2Rec + 225 + la];
    }
    g[a] = v;
  }
}

__global__ void k_init2_energy(const double* __restrict__ rec, int F, double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double e = 0.0;
  for (int f = 0; f < F; ++f) e += rec[(int64_t)f * kInit2Rec + 240];
  out[0] = e;
}

// (H + diag(H) lam + 1e-10 I) dx = -g (initialization.py:194-196), LU with partial pivoting in
// A (dim x dim row-major scratch); status 1 on an exactly zero pivot (numpy's LinAlgError)
__global__ void __launch_bounds__(256) k_init2_solve(const double* __restrict__ H, const double* __restrict__ g,
                                                     int dim, double lam, double* __restrict__ Ag,
                                                     double* __restrict__ dx, int* __restrict__ status) {
  // the working matrix lives in shared memory when it fits (dim <= 160), else in Ag
  extern __shared__ double A_s[];
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5;
  double* A = dim <= kInit2SmemDim ? A_s : Ag;
  double* b = dim <= kInit2SmemDim ? A_s + dim * dim : dx;
  __shared__ int piv;
  for (int t = tid; t < dim * dim; t += nth) {
    const int r = t / dim, c = t % dim;
    double v = H[t];
    if (r == c) v = v + H[t] * lam + 1e-10;
    A[t] = v;
  }
  for (int r = tid; r < dim; r += nth) b[r] = -g[r];
  if (tid == 0) *status = 0;
  __syncthreads();
  const int nw = nth / 32;
  for (int k = 0; k < dim; ++k) {
    // pivot: first maximum of |A[r][k]|, r >= k (idamax), by warp 0 alone (dim <= a few
    // hundred: a lane-strided scan and one warp tree, no cross-warp stage)
    if (warp == 0) {
      double best = -1.0;
      int bi = dim;
      for (int r = k + lane; r < dim; r += 32) {
        const double v = fabs(A[r * dim + k]);
        if (v > best) { best = v; bi = r; }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) piv = best > 0.0 ? bi : -1;   // exactly zero column: numpy's LinAlgError
    }
    __syncthreads();
    const int p = piv;   // (shared: a global status read here cost a memory round trip per column)
    if (p < 0) {
      if (tid == 0) *status = 1;
      return;
    }
    if (p != k) {
      for (int c = tid; c < dim; c += nth) {
        const double t = A[k * dim + c];
        A[k * dim + c] = A[p * dim + c];
        A[p * dim + c] = t;
      }
      if (tid == 0) {
        const double t = b[k];
        b[k] = b[p];
        b[p] = t;
      }
      __syncthreads();
    }
    // multiplier and rank-1 update of row r by one warp (lanes over columns): each element
    // one fma per k, in k order -- the same arithmetic as the row-serial form
    const double inv = 1.0 / A[k * dim + k];
    for (int r = k + 1 + warp; r < dim; r += nw) {
      const double l = A[r * dim + k] * inv;
      for (int c = k + 1 + lane; c < dim; c += 32) A[r * dim + c] -= l * A[k * dim + c];
      __syncwarp();   // every lane has read A[r][k]
      if (lane == 0) {
        A[r * dim + k] = l;
        b[r] -= l * b[k];
      }
    }
    __syncthreads();
  }
  // back substitution: warp 0, row dot products as warp trees (fixed order)
  if (warp == 0) {
    for (int k = dim - 1; k >= 0; --k) {
      double v = 0.0;
      for (int c = k + 1 + lane; c < dim; c += 32) v += A[k * dim + c] * b[c];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) b[k] = (b[k] - v) / A[k * dim + k];
      __syncwarp();
    }
  }
  __syncthreads();
  if (b != dx)
    for (int r = tid; r < dim; r += nth) dx[r] = b[r];
}

// trial estimate from dx (initialization.py:197-201): x = [s, 0, 0, bias(6)], gravity, velocities
__global__ void k_init2_update(const double* __restrict__ x, const double* __restrict__ grav,
                               const double* __restrict__ v, const double* __restrict__ dx, int K,
                               double* __restrict__ xn, double* __restrict__ gn, double* __restrict__ vn) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) {
    xn[0] = x[0] + dx[0];
    xn[1] = xn[2] = 0.0;
    for (int a = 0; a < 6; ++a) xn[3 + a] = x[3 + a] + dx[3 + a];
    const double w[3] = {dx[1], dx[2], 0.0};   // GRAVITY_TANGENT_BASIS @ dx[1:3] (residuals.py:141)
    double qe[4], qn[4];
    qexp(w, qe);
    qmul(grav, qe, qn);
    qcanon(qn);
    for (int a = 0; a < 4; ++a) gn[a] = qn[a];
    gn[4] = grav[4];
  }
  if (k < K)
    for (int a = 0; a < 3; ++a) vn[3 * k + a] = v[3 * k + a] + dx[9 + 3 * k + a];
}

}  // namespace vba

using namespace vba;

extern "C" {

int vba_init_inertial(const vba_init_problem* P, const vba_init_options* O, void* stream, vba_init_result* R,
                      double* cost_trajectory, int32_t cap, double* v_out) {
  cudaStream_t st = (cudaStream_t)stream;
  std::memset(R, 0, sizeof(*R));
  const int K = P->n_kf, F = P->n_imu;
  if (K < 2 || F < 1) {
    vba_set_error_string("need at least two keyframes with inertial edges");
    return VBA_E_INVALID;
  }
  const int dim = 9 + 3 * K;
  // one device allocation per call, carved into the buffers below (256-B aligned)
  size_t need = 0;
  const size_t sizes[] = {sizeof(double) * kImuL * F, sizeof(double) * 16 * K, sizeof(double) * kInit2Rec * F,
                          sizeof(double) * dim * dim, sizeof(double) * dim, sizeof(double) * dim * dim,
                          sizeof(double) * dim, sizeof(double), sizeof(double), sizeof(int) * 2,
                          sizeof(int32_t) * F, sizeof(int32_t) * F, sizeof(double) * 9, sizeof(double) * 5,
                          sizeof(double) * 3 * K, sizeof(double) * 9, sizeof(double) * 5, sizeof(double) * 3 * K};
  for (size_t z : sizes) need += (z + 255) / 256 * 256;
  char* arena = nullptr;
  size_t used = 0;
  {   // keep the default pool's freed blocks cached (release threshold 0 hands them back to the
      // driver at every synchronisation, and the next call's allocation re-maps them)
    static bool kept = false;
    int dev = 0;
    cudaMemPool_t pool;
    if (!kept && cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~(uint64_t)0;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      kept = true;
    }
  }
  if (cudaMallocAsync((void**)&arena, need, st) != cudaSuccess) arena = nullptr;
  auto alloc = [&](void** p, size_t bytes) {
    if (!arena) return false;
    *p = arena + used;
    used += (bytes + 255) / 256 * 256;
    return used <= need;
  };
  auto cleanup = [&]() {
    if (arena) cudaFreeAsync(arena, st);
  };
  double *L, *state, *rec, *H, *g, *A, *dx, *x[2], *gr[2], *v[2], *es, *cost;
  int32_t *fi, *fj;
  int* status;
  bool ok = alloc((void**)&L, sizeof(double) * kImuL * F) && alloc((void**)&state, sizeof(double) * 16 * K) &&
            alloc((void**)&rec, sizeof(double) * kInit2Rec * F) && alloc((void**)&H, sizeof(double) * dim * dim) &&
            alloc((void**)&g, sizeof(double) * dim) && alloc((void**)&A, sizeof(double) * dim * dim) &&
            alloc((void**)&dx, sizeof(double) * dim) && alloc((void**)&es, sizeof(double)) &&
            alloc((void**)&cost, sizeof(double)) && alloc((void**)&status, sizeof(int) * 2) &&
            alloc((void**)&fi, sizeof(int32_t) * F) && alloc((void**)&fj, sizeof(int32_t) * F);
  for (int b = 0; b < 2 && ok; ++b)
    ok = alloc((void**)&x[b], sizeof(double) * 9) && alloc((void**)&gr[b], sizeof(double) * 5) &&
         alloc((void**)&v[b], sizeof(double) * 3 * K);
  if (!ok) {
    cleanup();
    vba_set_error_string("vba_init_inertial: allocation failed");
    return VBA_E_CUDA;
  }
  const size_t solve_smem = dim <= kInit2SmemDim ? sizeof(double) * ((size_t)dim * dim + dim) : 0;
  if (solve_smem > 48 * 1024)
    cudaFuncSetAttribute(k_init2_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem);
  double hx[9] = {0, 0, 0, P->bias0[0], P->bias0[1], P->bias0[2], P->bias0[3], P->bias0[4], P->bias0[5]};
  double hg[5] = {P->grav_q[0], P->grav_q[1], P->grav_q[2], P->grav_q[3], P->grav_G};
  cudaMemcpyAsync(x[0], hx, sizeof(hx), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(gr[0], hg, sizeof(hg), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(v[0], P->v0, sizeof(double) * 3 * K, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(fi, P->h_imu_i, sizeof(int32_t) * F, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(fj, P->h_imu_j, sizeof(int32_t) * F, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(status, 0, sizeof(int) * 2, st);
  launch_imu_prep(P->imu, F, L, status + 1, st);
  int hs[2] = {0, 0};
  double hcost = 0.0;
  auto sync_err = [&](const char* what) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      char b[256];
      snprintf(b, sizeof(b), "vba_init_inertial %s: %s", what, cudaGetErrorString(e));
      vba_set_error_string(b);
      return true;
    }
    return false;
  };
  cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st);
  if (sync_err("prep")) { cleanup(); return VBA_E_CUDA; }
  if (hs[1]) { cleanup(); vba_set_error_string("non-PSD preintegration covariance"); return VBA_E_COV; }
  int cur = 0;
  // energy of estimate b (initialization.py:137-149)
  auto energy = [&](int b) {
    k_init2_states<<<(K + 127) / 128, 128, 0, st>>>(P->q, P->p, v[b], x[b], K, state, es);
    launch_init2_factor(P->imu, L, fi, fj, F, state, gr[b], P->p, es, 1, rec, st);
    k_init2_energy<<<1, 32, 0, st>>>(rec, F, cost);
    cudaMemcpyAsync(&hcost, cost, sizeof(double), cudaMemcpyDeviceToHost, st);
    return !sync_err("energy");
  };
  if (!energy(cur)) { cleanup(); return VBA_E_CUDA; }
  double c0 = hcost;
  std::vector<double> traj{c0};
  double lam = O->damping;
  int term = 0, iters = 0;   // 0 max_iterations, 1 converged, 2 no_decrease_at_max_damping
  for (int it = 0; it < O->max_iterations; ++it) {
    k_init2_states<<<(K + 127) / 128, 128, 0, st>>>(P->q, P->p, v[cur], x[cur], K, state, es);
    launch_init2_factor(P->imu, L, fi, fj, F, state, gr[cur], P->p, es, 0, rec, st);
    k_init2_assemble<<<dim, 128, 0, st>>>(rec, fi, fj, F, dim, H, g);
    bool accepted = false;
    while (lam <= 1e8) {
      k_init2_solve<<<1, 256, solve_smem, st>>>(H, g, dim, lam, A, dx, status);
      cudaMemcpyAsync(hs, status, sizeof(int), cudaMemcpyDeviceToHost, st);
      if (sync_err("solve")) { cleanup(); return VBA_E_CUDA; }
      if (hs[0]) break;   // np.linalg.LinAlgError (initialization.py:195-196)
      const int nx = cur ^ 1;
      k_init2_update<<<(K + 127) / 128, 128, 0, st>>>(x[cur], gr[cur], v[cur], dx, K, x[nx], gr[nx], v[nx]);
      if (!energy(nx)) { cleanup(); return VBA_E_CUDA; }
      const double cn = hcost;
      if (cn < traj.back()) {
        const double rel = (traj.back() - cn) / std::max(traj.back(), 1e-30);
        cur = nx;
        traj.push_back(cn);
        lam = std::max(lam * 0.5, 1e-12);
        accepted = true;
        ++iters;
        if (rel < 1e-10) term = 1;
        break;
      }
      lam *= 10.0;
    }
    if (!accepted) { term = 2; break; }
    if (term == 1) break;
  }
  double hxo[9], hgo[5];
  cudaMemcpyAsync(hxo, x[cur], sizeof(hxo), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hgo, gr[cur], sizeof(hgo), cudaMemcpyDeviceToHost, st);
  if (v_out) cudaMemcpyAsync(v_out, v[cur], sizeof(double) * 3 * K, cudaMemcpyDeviceToDevice, st);
  if (sync_err("result")) { cleanup(); return VBA_E_CUDA; }
  R->log_scale = hxo[0];
  for (int a = 0; a < 4; ++a) R->grav_q[a] = hgo[a];
  for (int a = 0; a < 6; ++a) R->bias[a] = hxo[3 + a];
  R->iterations = iters;
  R->termination = term;
  R->n_costs = (int)traj.size();
  R->initial_cost = traj.front();
  R->final_cost = traj.back();
  for (int i = 0; i < (int)traj.size() && i < cap; ++i) cost_trajectory[i] = traj[i];
  cleanup();
  return VBA_OK;
}

}  // extern "C"
