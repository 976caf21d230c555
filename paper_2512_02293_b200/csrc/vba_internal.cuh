// vba_internal.cuh — shared device structs, fp64 Lie-group helpers and launchers.
//
// Numerical conventions restated from the reference (paths relative to
// /root/reference/pkg/src/vislam/):
//   quaternions wxyz, canonical w >= 0, renormalised on every product (geometry.py:94-107)
//   small-angle cutoff 1e-8 for exp / Jr / Jr^-1 / log (geometry.py:20,38,62,75,117,163)
//   right rotation perturbation, additive world translation (geometry.py:221-223)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vba.h"

namespace vba {

#ifndef VBA_TP
#define VBA_TP 4                          // pixel pairs per thread of the per-pixel kernels
#endif
constexpr int kTilePx = 2 * VBA_TP * 128;   // pixels per per-pixel work tile (128-thread CTAs)
constexpr double kSmallAngle = 1e-8;
constexpr float kDispFloor = 1e-4f;      // solver.py:32
constexpr double kDispFloor64 = 1e-4;    // solver.py:32 (the fp64 master update)
constexpr int kPartWarps = 4;            // warps of the K1 CTA, one fp32 32-vector each
constexpr int kPartStride = 32 * kPartWarps;   // floats per K1 (tile, edge) partial record
constexpr int kVisBlock = 120;           // doubles per edge pose-space block record
constexpr int kGeo64 = 24;               // doubles per EdgeGeo64 record
constexpr int kImuL = 120;               // doubles per IMU whitening-factor record (81 + 36 + pad)

// Per-edge camera-frame constants for the per-pixel loops (fp32):
// X_h = ray + (M - I) ray + d t, with M = A R_i R_bc the camera-i -> camera-j rotation.
struct __align__(16) EdgeGeo32 {
  float M[9];   // M - I

  float t[3];
  float pad[4];
};

// Global extrinsic constants: R_bc^T and c2 = R_bc^T p_bc (residuals.py:187-204).
struct Extr {
  double RbcT[9];
  double Rbc[9];
  double pbc[3];
  double c2[3];
};

// Work tile of the per-pixel kernels: `cnt` padded pixels of source keyframe `src`
// starting at pixel `n0`, looping over that source's out-edges [eb, ee).
struct PixTile {
  int32_t src, n0, cnt, eb, ee;
  int32_t pad;    // K1 chunks: 1 = half of a split tile (H_dd / g_d added atomically)
  int64_t poff;   // first K1 partial record of this tile (one per out-edge)
};

// One streamed (tile, edge) item of K1 / K2: its flow / weight rows start at
// float offset `foff` (= 2 (eoff[e] + n0)) and span `bytes` per array.
struct StreamItem {
  int64_t foff;
  int32_t bytes, edge;
};

// Work tile of the Schur Gram kernel (one source keyframe, a pixel range).
struct GramTile {
  int32_t src, n0, n1, eb, ee, nsplit;
  int32_t u0, u1;   // unit slice of the DMMA Gram (u1 > u0: sources with more than 31 out-edges)
  int64_t out;      // offset (doubles) of this tile's partial Gram output (shared by a range's slices)
};

// Assembly contribution: value(r,c) = sign * buf[off + (trans ? c*ld + r : r*ld + c)]
struct Contrib {
  int64_t off;
  int32_t ld;
  int16_t rows, cols;
  int8_t trans, sign;
  int8_t pad[6];
};

struct Vec {
  int64_t off;
  int32_t len;
  int32_t sign;
};

// ---------------------------------------------------------------------------
// fp64 SO(3) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C[i * 3 + j] = A[i * 3 + 0] * B[0 * 3 + j] + A[i * 3 + 1] * B[1 * 3 + j] + A[i * 3 + 2] * B[2 * 3 + j];
}
__device__ __forceinline__ void mat3_mulT(const double* A, const double* B, double* C) {  // A B^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C[i * 3 + j] = A[i * 3 + 0] * B[j * 3 + 0] + A[i * 3 + 1] * B[j * 3 + 1] + A[i * 3 + 2] * B[j * 3 + 2];
}
__device__ __forceinline__ void mat3_Tmul(const double* A, const double* B, double* C) {  // A^T B
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C[i * 3 + j] = A[0 * 3 + i] * B[0 * 3 + j] + A[1 * 3 + i] * B[1 * 3 + j] + A[2 * 3 + i] * B[2 * 3 + j];
}
__device__ __forceinline__ void mat3_vec(const double* A, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < 3; ++i) y[i] = A[i * 3 + 0] * x[0] + A[i * 3 + 1] * x[1] + A[i * 3 + 2] * x[2];
}
__device__ __forceinline__ void mat3T_vec(const double* A, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < 3; ++i) y[i] = A[0 * 3 + i] * x[0] + A[1 * 3 + i] * x[1] + A[2 * 3 + i] * x[2];
}
__device__ __forceinline__ void hat3(const double* v, double* H) {
  H[0] = 0.0;   H[1] = -v[2]; H[2] = v[1];
  H[3] = v[2];  H[4] = 0.0;   H[5] = -v[0];
  H[6] = -v[1]; H[7] = v[0];  H[8] = 0.0;
}
__device__ __forceinline__ void qmat(const double* q, double* R) {  // geometry.py:151-157
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}
__device__ __forceinline__ void qcanon(double* q) {  // geometry.py:94-98
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double s = (q[0] / n < 0.0) ? -1.0 : 1.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = s * (q[k] / n);
}
__device__ __forceinline__ void qmul(const double* a, const double* b, double* o) {  // geometry.py:83-91
  o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}
__device__ __forceinline__ void qexp(const double* w, double* q) {  // geometry.py:113-123
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  if (th < kSmallAngle) {
    q[0] = 1.0; q[1] = 0.5 * w[0]; q[2] = 0.5 * w[1]; q[3] = 0.5 * w[2];
  } else {
    double s, c;
    sincos(0.5 * th, &s, &c);
    q[0] = c; q[1] = s * (w[0] / th); q[2] = s * (w[1] / th); q[3] = s * (w[2] / th);
  }
  qcanon(q);
}
__device__ __forceinline__ void so3_exp(const double* w, double* R) {  // geometry.py:33-43
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9], K2[9];
  hat3(w, K);
  mat3_mul(K, K, K2);
  double a, b;
  if (th < kSmallAngle) { a = 1.0; b = 0.5; }
  else { a = sin(th) / th; b = (1.0 - cos(th)) / (th * th); }
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = ((k % 4) == 0 ? 1.0 : 0.0) + a * K[k] + b * K2[k];
}
__device__ __forceinline__ void so3_jr(const double* w, double* J) {  // geometry.py:57-67
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9], K2[9];
  hat3(w, K);
  mat3_mul(K, K, K2);
  double a, b;
  if (th < kSmallAngle) { a = 0.5; b = 1.0 / 6.0; }
  else { const double t2 = th * th; a = (1.0 - cos(th)) / t2; b = (th - sin(th)) / (t2 * th); }
#pragma unroll
  for (int k = 0; k < 9; ++k) J[k] = ((k % 4) == 0 ? 1.0 : 0.0) - a * K[k] + b * K2[k];
}
__device__ __forceinline__ void so3_jr_inv(const double* w, double* J) {  // geometry.py:70-80
  const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double K[9], K2[9];
  hat3(w, K);
  mat3_mul(K, K, K2);
  double b;
  if (th < kSmallAngle) b = 1.0 / 12.0;
  else b = (1.0 / (th * th)) * (1.0 - th * (1.0 / tan(0.5 * th)) / 2.0);
#pragma unroll
  for (int k = 0; k < 9; ++k) J[k] = ((k % 4) == 0 ? 1.0 : 0.0) + 0.5 * K[k] + b * K2[k];
}
__device__ __forceinline__ void q_from_mat(const double* R, double* q) {  // geometry.py:125-149
  const double t = R[0] + R[4] + R[8];
  if (t > 0.0) {
    const double s = sqrt(t + 1.0) * 2.0;
    q[0] = 0.25 * s; q[1] = (R[7] - R[5]) / s; q[2] = (R[2] - R[6]) / s; q[3] = (R[3] - R[1]) / s;
  } else {
    int i = 0;
    if (R[4] > R[0]) i = 1;
    if (R[8] > R[i * 4]) i = 2;
    if (i == 0) {
      const double s = sqrt(1.0 + R[0] - R[4] - R[8]) * 2.0;
      q[0] = (R[7] - R[5]) / s; q[1] = 0.25 * s; q[2] = (R[1] + R[3]) / s; q[3] = (R[2] + R[6]) / s;
    } else if (i == 1) {
      const double s = sqrt(1.0 + R[4] - R[0] - R[8]) * 2.0;
      q[0] = (R[2] - R[6]) / s; q[1] = (R[1] + R[3]) / s; q[2] = 0.25 * s; q[3] = (R[5] + R[7]) / s;
    } else {
      const double s = sqrt(1.0 + R[8] - R[0] - R[4]) * 2.0;
      q[0] = (R[3] - R[1]) / s; q[1] = (R[2] + R[6]) / s; q[2] = (R[5] + R[7]) / s; q[3] = 0.25 * s;
    }
  }
  qcanon(q);
}
__device__ __forceinline__ void qlog(const double* q, double* w) {  // geometry.py:159-167
  const double n = sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (n < kSmallAngle) {
    const double s = 2.0 / q[0];
    w[0] = s * q[1]; w[1] = s * q[2]; w[2] = s * q[3];
  } else {
    const double s = 2.0 * atan2(n, q[0]) / n;
    w[0] = s * q[1]; w[1] = s * q[2]; w[2] = s * q[3];
  }
}

// G matrices of the factorised vision Jacobian:
//   J_i = K G_i,  J_j = -K G_j,  K = [P[X_j]x | -P]
//   G_i = [[A R_i, 0], [-[c1]x A R_i, A]],  G_j = [[R_bc^T, 0], [-[c2]x R_bc^T, A]]
__device__ __forceinline__ void build_G(const double* R3, const double* c, const double* A, double* G) {
  double H[9], HR[9];
  hat3(c, H);
  mat3_mul(H, R3, HR);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      G[r * 6 + k] = R3[r * 3 + k];
      G[r * 6 + 3 + k] = 0.0;
      G[(3 + r) * 6 + k] = -HR[r * 3 + k];
      G[(3 + r) * 6 + 3 + k] = A[r * 3 + k];
    }
}

// warp-level reduce-scatter of 32 per-lane values: afterwards lane l holds
// sum over the warp of v[l] (31 shuffles instead of 160 for a naive butterfly).
__device__ __forceinline__ float warp_reduce_scatter32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float keep = up ? v[i + o] : v[i];
      const float send = up ? v[i] : v[i + o];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

}  // namespace vba

// ---------------------------------------------------------------------------
// launchers (defined in the .cu files, used by the host runtime)
// ---------------------------------------------------------------------------
namespace vba {

struct DevState {      // one side of the double-buffered solver state
  double* state;       // [K,16]
  float* disp;         // [n_disp_pad] fp32 copy read by the per-pixel kernels
  double* disp64;      // [n_disp_pad] master disparities: updated in fp64 (solver.py:336-338)
  double* grav;        // [5]
  EdgeGeo32* geo32;    // [E]
  double* geo64;       // [E, kGeo64]
};

void launch_edge_prep(const DevState& s, const int32_t* ei, const int32_t* ej, int E, const Extr& x,
                      cudaStream_t st);
// Streamed K1 / K2: CTA b processes tiles sids[soff[b] .. soff[b+1]) whose (tile, edge)
// items are items[ioff[b] .. ioff[b+1]); ncta = vision_stream_ctas()
int vision_stream_ctas();
void launch_ray_table(float* tab, int W, int rows, const double* grid, const double* intr, cudaStream_t st);
void launch_count_nz_blocks(const float* wts, const int64_t* row0, const int32_t* cnt, int n, int grid_w,
                            int32_t* out, cudaStream_t st);
void launch_vision_linearize(int pixel_mode, const PixTile* tiles, const int32_t* soff, const int32_t* sids,
                             const StreamItem* items, const int32_t* ioff, int ncta, const DevState& s, const float* pix, const float* tgt, const float* wts,
                             const int64_t* eoff, const int64_t* doff, int grid_w, const double* grid,
                             const double* intr, double* partials, float* Hdd, float* gd, cudaStream_t st);
void launch_vision_energy(int pixel_mode, const PixTile* tiles, const int32_t* soff, const int32_t* sids,
                          const StreamItem* items, const int32_t* ioff, int ncta, const DevState& s, const float* pix, const float* tgt, const float* wts,
                          const int64_t* eoff, const int64_t* doff, int grid_w, const double* grid,
                          const double* intr, double* tile_energy, cudaStream_t st);
// edges [e0, e0 + n)
void launch_edge_finalize(const int32_t* esrc_tile0, const int32_t* esrc_tile1, const PixTile* tiles,
                          const int32_t* edge_i, int e0, int n, const double* partials, const DevState& s,
                          const Extr& x, double* visblocks, double* edge_energy, cudaStream_t st);
void launch_gram(int pixel_mode, const GramTile* gt, int ngt, int block, size_t smem, int kmax,
                 const DevState& s, const float* pix, const float* wts, const int64_t* eoff,
                 const int64_t* doff, int grid_w, const double* grid, const double* intr,
                 const float* Hdd, const float* gd, double lam, double ridge, double* gram_part,
                 cudaStream_t st, const int32_t* order = nullptr);
void launch_fill_transform(const int32_t* src_list, int nsrc, const int32_t* src_eb, const int32_t* src_ee,
                           const int32_t* src_gt0, const int32_t* src_gt1, const GramTile* gt, const int64_t* foff,
                           const double* part, const DevState& s, const Extr& x, double* fill, int kmax,
                           cudaStream_t st);
void launch_step_edges(const int32_t* ei, const int32_t* ej, int E, const DevState& s, const Extr& x,
                       const double* dx_full, int sdof, float* ustep, cudaStream_t st);
size_t gram_smem_bytes(int kmax, int nsplit, int npairs, int k);
size_t gram_tc_smem_bytes(int kmax);
int gram_units(int k);
int gram_slice_units();
void launch_copy_segments(const vba_copy_seg* segs, int n, cudaStream_t st);
void launch_gram_tc(int pixel_mode, const GramTile* gt, int ngt, size_t smem, int kmax, const DevState& s,
                    const float* pix, const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w,
                    const double* grid, const double* intr, const float* Hdd, const float* gd, double lam,
                    double ridge, double* gram_part, cudaStream_t st, const int32_t* order);
void launch_backsub(int pixel_mode, const PixTile* tiles, int ntiles, const DevState& cur, const DevState& nxt,
                    const float* pix, const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w,
                    const double* grid, const double* intr, const float* Hdd, const float* gd,
                    const float* ustep, double lam, double ridge, double* dxd_out,
                    unsigned long long* step_max_bits, cudaStream_t st);
void launch_retract(const DevState& cur, const DevState& nxt, const double* dx_full, const int32_t* frozen,
                    int K, int sdof, int ngrav, int n_state, unsigned long long* step_max_bits,
                    int npv, cudaStream_t st);
void launch_energy_reduce(const double* tile_energy, int ntiles, const double* imu_blocks, int F, int ibs,
                          int energy_off, double* out3, cudaStream_t st);
// IMU
void launch_imu_prep(const double* imu, int F, double* Lbuf, int* status, cudaStream_t st);
// factors [f0, f0 + F)
void launch_imu_factor(const double* imu, const double* Lbuf, const int32_t* fi, const int32_t* fj, int f0, int F,
                       const DevState& s, const double* ts, int sdof, int ibs, int energy_only,
                       double* imu_blocks, cudaStream_t st);
// stage-2 inertial-only initialisation (vba_imu.cu / vba_init.cu)
constexpr int kInit2Rec = 248;   // H 15x15, g 15, e (+pad)
void launch_init2_factor(const double* imu, const double* Lbuf, const int32_t* fi, const int32_t* fj, int F,
                         const double* state, const double* grav, const double* pvis, const double* es,
                         int energy_only, double* out, cudaStream_t st);
// dense
void launch_assemble(const int32_t* blk_ptr, const int32_t* blk_nff, const Contrib* contribs, int nblk_rows,
                     const int32_t* roff, const int32_t* rdim, const double* arena, double lam, double ridge,
                     int add_ridge, double* H, int64_t ld, int sym, cudaStream_t st, const int32_t* blist = nullptr,
                     int nblist = 0);
void launch_assemble_vec(const int32_t* seg_ptr, const Vec* vecs, int nseg, const int32_t* seg_off,
                         const double* arena, double scale, double* g, cudaStream_t st, int skip_fill = 0);
void launch_pad_identity(double* H, int64_t ld, int n, int npad, double* rhs, cudaStream_t st);
void launch_export_sym(const double* H, int64_t ld, int n, double* out, const double* rhs, double scale, double* g,
                       cudaStream_t st);
// tile-task DAG Cholesky (vba_chol.cu): plan writes up to `cap` task records into `out`
// (opaque, chol_task_bytes() each) and returns the task count
int chol_plan_tasks(int nt, void* out, int cap);
size_t chol_task_bytes();
// one-CTA fp64 Cholesky solve of the lower triangle of A (column-major, ld) for n <= 232
// (vba_small.cu); returns non-zero (nothing launched) for larger systems
int chol_small_solve(const double* A, int64_t ld, int n, const double* rhs, double* x, int* status, cudaStream_t st);
int chol_dag_launch(double* A, int64_t ld, int nt, double* rhs, double* x, double* Linv, double* part, int* flags,
                    const void* tasks, int ntasks, int* status, cudaStream_t st,
                    unsigned long long* trace = nullptr);
// Mixed-precision (tcgen05 3xTF32 factor + fp64 iterative refinement) SPD solve,
// vba_chol.cu.  out2[0] = max |correction| of the last refinement pass, out2[1] = max |x|,
// out2[2] = refinement passes run.
size_t chol_tc_ws_bytes(int npad);
int chol_plan_tasks_tc(int nt, void* out, int cap);
int chol_tc_solve(const double* H, int64_t ld, int n, int npad, const double* b, double* x, void* ws,
                  const void* tasks, int ntasks, int iters, int* status, int gen, cudaStream_t st, double* out2,
                  unsigned long long* trace = nullptr, cudaEvent_t* ev3 = nullptr);
void chol_trace_print(const char* tag, const unsigned long long* d_trace, const void* d_tasks, int ntasks, int nt);
// copy the task list back (for trace decoding): type,i,j,k per task
void chol_task_fields(const void* tasks, int n, int* out4);
void chol_task_fields5(const void* tasks, int n, int* out5);
void launch_scatter_dx(const double* x, const int32_t* free_map, int npv, double* dx_full, cudaStream_t st);
// pose-disparity coupling writer: reference-layout export (colmap == NULL, rows k*sdof+a) or the
// free-layout full dense system of the use_schur=False path (rows colmap[k]+a, plus the damped
// disparity diagonal and right-hand side when Hdd != NULL).  Entry (row, base+col) at H[row*ld + base+col].
struct HpdOut {
  double* H;
  int64_t ld, base;
  int sdof;
  const int32_t* colmap;
  const float* Hdd;
  const float* gd;
  double* rhs;
  double lam, ridge;
};
void launch_export_hpd(int mode, const int32_t* seb, const int32_t* see, const int64_t* doff, const int64_t* roff,
                       const int32_t* npix, int maxpix, const int32_t* ej, int K, const DevState& s, const Extr& x,
                       const float* pix, const float* wts, const int64_t* eoff, int grid_w, const double* grid,
                       const double* intr, const HpdOut& out, cudaStream_t st);
void launch_dense_dxd(const double* x, int nf, const int64_t* doff, const int64_t* roff, const int32_t* npix,
                      int maxpix, int K, const DevState& cur, const DevState& nxt, double* dxd,
                      unsigned long long* step_bits, cudaStream_t st);
void launch_unpad(const float* src, const int64_t* doff, const int64_t* roff, const int32_t* npix, int maxpix, int K,
                  double* dst, cudaStream_t st);
void launch_unpad(const double* src, const int64_t* doff, const int64_t* roff, const int32_t* npix, int maxpix, int K,
                  double* dst, cudaStream_t st);
// fp32 <-> fp64 disparity copies (master state <-> kernel copy / caller arrays)
void launch_widen(const float* src, double* dst, int64_t n, cudaStream_t st);
void launch_narrow(const double* src, float* dst, int64_t n, cudaStream_t st);
// The tensor-core reduced solve stops refining once a pass corrects x by <= kTcRefineTol
// max|x| AND the geometric-tail bound of the remaining error, rel * rho / (1 - rho) with the
// measured per-pass contraction rho, is <= kTcErrTol (k_tc_check); with the factor's usual
// contraction (~1e-3) that is 3 passes and <= 1e-7 relative error, far inside the 1e-5 update
// parity.  A solve that does not meet both within its pass budget is redone on the fp64 path.
constexpr double kTcRefineTol = 1e-5;
constexpr double kTcErrTol = 1e-7;

// IMU preintegration (vba_preint.cu): record per keyframe pair, see include/vba.h.
constexpr int kPreintRec = 281;
size_t preint_scratch_bytes(int64_t S);
constexpr int kImuRec = 180;   // VBA_IMU_REC
void launch_preint_pack(const double* rec, const double* bias, int F, double* imu, cudaStream_t st);
void launch_preintegrate(const double* ts, const double* gyro, const double* accel, int64_t S, const int64_t* soff,
                         int F, const double* bias, const double* noise, double* scratch, double* out, int* status,
                         cudaStream_t st);
void launch_count();   // instrumentation hook
void vba_set_error_string(const char* msg);   // vba_last_error() of every C entry point
int64_t launch_total();

}  // namespace vba
