/*
 * vba.h — C ABI of the B200-native dense visual-inertial bundle adjustment.
 *
 * Drop-in boundary for the reference's VI-BA path
 * (/root/reference/pkg/src/vislam/solver.py).  The reference has no native
 * FFI — it is pure Python/numpy — so each entry point below replaces one
 * reference *function*; a maintainer binds them with ctypes.
 *
 *   vba_solve            <- solve_vi_ba        solver.py:344-411
 *   vba_energy           <- total_energy       solver.py:118-131
 *   vba_linearize        <- _linearize         solver.py:173-251
 *   vba_export_normal_eq <- (_linearize's dense outputs H_pp,H_pd,H_dd,g_p,g_d)
 *   vba_solve_step       <- _solve_step        solver.py:254-308
 *   vba_export_reduced   <- (_solve_step's H_red, g_red)     solver.py:272-285
 *   vba_apply_step       <- _snapshot + _apply_step  solver.py:311-341
 *   vba_restore          <- _restore           solver.py:318-323
 *   vba_trial            <- one LM trial (solve, apply, energy) solver.py:370-383
 *   vba_accept           <- accepted step bookkeeping       solver.py:383-393
 *
 * Conventions: plain pointers and sizes only; every pointer in vba_problem is
 * a DEVICE pointer owned by the caller except the h_* topology arrays, which
 * are host pointers read only inside vba_create.  All calls are
 * stream-ordered on the caller's cudaStream_t (passed as void*); the calls
 * that return host scalars synchronise that stream.  No C++ exception
 * crosses the ABI; errors are integer status codes (vba_last_error() gives
 * the message).  A context is bound to one device and is not thread-safe.
 */
#ifndef VBA_H
#define VBA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VBA_API __attribute__((visibility("default")))
#else
#define VBA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define VBA_OK 0
#define VBA_E_INVALID 1  /* invalid problem/options -> reference raises ValueError */
#define VBA_E_CUDA 2     /* CUDA runtime failure */
#define VBA_E_NOT_SPD 3  /* reduced system not positive definite -> reference's
                            RuntimeError("singular reduced pose system"), solver.py:287-289 */
#define VBA_E_COV 4      /* preintegration covariance not PD -> ValueError, residuals.py:337-341 */
#define VBA_E_UNSUPPORTED 5

#define VBA_PIX_GRID 0   /* pixel n of a keyframe = (ox + sx*(n % w), oy + sy*(n / w)) */
#define VBA_PIX_KF 1     /* explicit per-keyframe coordinates (padded keyframe layout) */
#define VBA_PIX_EDGE 2   /* explicit per-edge coordinates (padded edge-row layout) */

/* Packed IMU factor record (fp64), one per preintegrated delta:
 *  [0] dt  [1..4] dR quat wxyz  [5..7] dp  [8..10] dv  [11..19] J_rot 3x3 row-major
 *  [20..37] J_pos 3x6  [38..55] J_vel 3x6  [56..136] cov[0:9,0:9]  [137..172] cov[9:15,9:15]
 *  [173..178] bias linearisation point (gyro, accel)                                  */
#define VBA_IMU_REC 180

typedef struct vba_problem {
  /* sizes */
  int32_t n_kf;          /* K */
  int32_t n_edges;       /* E (vision edges on this rank) */
  int32_t n_imu;         /* F (inertial factors on this rank) */
  int32_t pixel_mode;    /* VBA_PIX_* */
  int64_t n_disp_pad;    /* disparity slots, per-keyframe segments padded to 4 */
  int64_t n_rows_pad;    /* edge rows, per-edge segments padded to 4 */
  int32_t grid_w;        /* VBA_PIX_GRID: columns */
  int32_t has_Tcb;
  double grid_ox, grid_oy, grid_sx, grid_sy;
  double fx, fy, cx, cy;
  double Tcb[7];         /* camera-from-body extrinsic T_cb: quat wxyz, translation */
  /* device arrays (caller-owned) */
  double* state;         /* [K,16]: q wxyz, p, v, b_g, b_a — read at create, updated by solve */
  const double* ts;      /* [K] timestamps */
  float* disp;           /* [n_disp_pad] disparities — read at create, updated by solve */
  const float* pix;      /* [n_disp_pad,2] (VBA_PIX_KF) or [n_rows_pad,2] (VBA_PIX_EDGE) or NULL */
  const float* tgt;      /* [n_rows_pad,2] flow targets relative to the source pixel: u* - u
                            (the reference's VisionEdge.targets minus VisionEdge.pixels) */
  const float* wts;      /* [n_rows_pad,2] confidence weights (>= 0) */
  const double* imu;     /* [F, VBA_IMU_REC] */
  double* grav;          /* [5]: R_wg quat wxyz, magnitude */
  /* host topology (read in vba_create only) */
  const int64_t* h_doff;   /* [K+1] padded disparity offsets */
  const int32_t* h_npix;   /* [K]   real pixel count per keyframe */
  const int32_t* h_edge_i; /* [E]   source keyframe index (edges sorted by source) */
  const int32_t* h_edge_j; /* [E]   target keyframe index */
  const int64_t* h_eoff;   /* [E]   padded row offset of each edge */
  const int32_t* h_imu_i;  /* [F] */
  const int32_t* h_imu_j;  /* [F] */
  const int32_t* h_frozen; /* [K] 1 = frozen (gauge) keyframe */
  /* optional device array (may be NULL): fp64 master disparities [n_disp_pad].  The solver
   * keeps the disparity state in fp64 and updates it as max(d + dx_d, 1e-4) in fp64
   * (solver.py:336-338); the per-pixel kernels read its fp32 copy.  When given it seeds the
   * state at create / vba_load_state (disp is then ignored) and vba_download writes it;
   * when NULL the state is seeded from the fp32 disp. */
  double* disp64;
  /* edge sharding across ranks (one process per GPU).  shard_world <= 1:
   * a single-GPU solve.  Otherwise every rank passes the FULL problem and the same keyframe
   * bounds h_shard_kbounds[shard_world + 1] (host, read in vba_create): rank r owns the
   * source keyframes [kb[r], kb[r+1]) -- their out-edges, pixel tiles, Schur fill-in and
   * disparities -- and the IMU factors (i, j) with i in that range (factors must be sorted
   * by i).  Ranks exchange their per-edge / per-factor / per-source blocks with the gather
   * hook (vba_set_gather) and every rank assembles and solves the identical reduced system,
   * so an N-rank solve is bitwise the 1-rank solve. */
  int32_t shard_world;
  int32_t shard_rank;
  const int32_t* h_shard_kbounds;
} vba_problem;

typedef struct vba_options {       /* SolveOptions, solver.py:82-105 */
  int32_t max_iterations;
  double damping, damping_up, damping_down;
  double rel_decrease_tol, step_tol, max_damping;
  int32_t optimize_gravity;
  int32_t optimize_velocity_bias;
  int32_t use_schur;
  double ridge;
} vba_options;

typedef struct vba_report {        /* SolveReport, solver.py:108-115 */
  int32_t iterations;
  int32_t termination;             /* 0 max_iterations, 1 converged,
                                      2 no_decrease_at_max_damping, 3 singular */
  int32_t n_costs;                 /* entries written to cost_trajectory */
  int32_t n_warnings;              /* singular-system retries */
  int32_t trials;                  /* LM trials run */
  double initial_cost, final_cost;
} vba_report;

typedef struct vba_trial_result {
  int32_t status;                  /* VBA_OK or VBA_E_NOT_SPD */
  double new_cost;
  double step_inf;                 /* max(|dx_full|, |dx_d|) */
} vba_trial_result;

/* Collective hook for edge-sharded multi-GPU solves: sum (op 0) or max (op 1)
 * of `count` doubles at device pointer `buf` across ranks, stream-ordered.
 * Supplied by the host (torch.distributed / NCCL); NULL for one GPU. */
typedef int (*vba_allreduce_fn)(void* user, double* buf, int64_t count, int32_t op,
                                void* stream);
/* Gather hook of a sharded solve: rank r holds buf[offsets[r] .. offsets[r+1]) (doubles,
 * device memory); on return every rank holds all of buf[offsets[0] .. offsets[world]).
 * Stream-ordered on `stream`.  Returns 0 on success. */
typedef int (*vba_allgather_fn)(void* user, double* buf, const int64_t* offsets, int32_t world, void* stream);

VBA_API const char* vba_last_error(void);
VBA_API int vba_version(void);

VBA_API int vba_create(void** ctx, const vba_problem* prob, const vba_options* opts, void* stream);
VBA_API int vba_destroy(void* ctx);
VBA_API int vba_set_collective(void* ctx, vba_allreduce_fn fn, void* user);
VBA_API int vba_set_gather(void* ctx, vba_allgather_fn fn, void* user);
/* free-variable count of the reduced system (solver.py:254-257) */
VBA_API int64_t vba_reduced_dim(void* ctx);

VBA_API int vba_energy(void* ctx, void* stream, double* out_total, double* out_vision,
               double* out_inertial);
VBA_API int vba_linearize(void* ctx, void* stream);
/* Dense (reference-layout) normal equations of the last linearisation.  All
 * outputs are device pointers in the reference's column layout
 * (solver.py:139-170): H_pp [npv,npv] row-major, g_p [npv], H_dd/g_d [n_disp]
 * in the *unpadded* keyframe order, H_pd [npv, n_disp] row-major (may be NULL). */
VBA_API int vba_export_normal_eq(void* ctx, void* stream, double* H_pp, double* g_p, double* H_pd,
                         double* H_dd, double* g_d);
VBA_API int vba_solve_step(void* ctx, void* stream, double lam, int32_t use_schur);
/* Reduced (Schur) system of the last linearisation at damping lam, before the solve:
 * H_red = Hf_d - Hfd D^-1 Hfd^T [nfree, nfree] row-major (full symmetric) and
 * g_red = g_f - Hfd D^-1 g_d [nfree] (solver.py:272-285), device pointers;
 * nfree = vba_reduced_dim().  Synchronises the stream. */
VBA_API int vba_export_reduced(void* ctx, void* stream, double lam, double* H_red, double* g_red);
/* dx_full [npv] (zeros at frozen states) and dx_d [n_disp] unpadded, device pointers */
VBA_API int vba_export_step(void* ctx, void* stream, double* dx_full, double* dx_d);
VBA_API int vba_apply_step(void* ctx, void* stream);
VBA_API int vba_restore(void* ctx, void* stream);
VBA_API int vba_accept(void* ctx, void* stream);
VBA_API int vba_trial(void* ctx, void* stream, double lam, int32_t use_schur, vba_trial_result* out);
VBA_API int vba_solve(void* ctx, void* stream, vba_report* report, double* cost_trajectory,
              int32_t traj_capacity);
/* re-seed the current state from the caller's problem arrays (state, disp, grav) */
VBA_API int vba_load_state(void* ctx, void* stream);
/* (new, streaming) bind another window's per-edge-pixel inputs of the same topology:
 * flow targets and weights (device pointers, the layout of vba_problem.tgt / .wts).
 * refresh_imu != 0 re-derives the IMU whitening factors from vba_problem.imu (its
 * contents may have changed); returns VBA_E_COV for a non-PSD covariance.  The
 * static per-pixel schedule built at create is kept (valid for any weights). */
VBA_API int vba_bind_inputs(void* ctx, void* stream, const float* tgt, const float* wts, int32_t refresh_imu);
/* enable per-stage CUDA-event timing of vba_solve / vba_trial (resets the counters) */
VBA_API int vba_set_profiling(void* ctx, int32_t on);
/* copy the current (accepted) state back to the caller's problem arrays */
VBA_API int vba_download(void* ctx, void* stream);
/* kernel launches issued by this context since creation (instrumentation) */
VBA_API int64_t vba_launch_count(void* ctx);
/* accumulated per-stage device time since vba_set_profiling, ms:
 * [0] linearise  [1] Schur Gram + fill transform  [2] assembly + Cholesky
 * [3] back-substitution + retraction  [4] trial energy  [5] vision linearisation
 * kernel alone  [6] number of samples in [5]   (out must hold 7 doubles) */
VBA_API int vba_stage_times(void* ctx, double* out5);
/* tensor-core reduced solve timing since vba_set_profiling, ms: [0] tile-DAG
 * factorisation kernel, [1] refinement passes (triangular solves + fp64
 * residuals), [2] number of solves timed, [3] reduced dimension n */
VBA_API int vba_solve_times(void* ctx, double* out4);
/* solver statistics: [0] tensor-core reduced solve enabled, [1] steps that fell
 * back to the fp64 factorisation, [2] tensor-core solves, [3] refinement passes
 * summed over them */
VBA_API int vba_stats(void* ctx, int64_t* out4);

/* Which Schur fill-in Gram the context runs (solver.py:282-285): 1 = tcgen05 kind::tf32
 * 3-product kernel (windows with >= 256 pixels per source keyframe), 0 = fp64 DMMA kernel;
 * the environment variable VBA_GRAM=tc|dmma, read by vba_create, forces either. */
VBA_API int vba_gram_kind(void* ctx);

/* Task list of the tensor-core Cholesky DAG for nt 128-row tiles (host only, no GPU):
 * writes min(count, cap) tasks as 5 ints each -- type (1 TRSM of column 0, 6 the chain task,
 * 7 a left-looking tile task, 8 a CONV task), i, j, k (TILE: columns accumulated), mode
 * (TILE: 0 SYRK target, 1 followed by its TRSM, 2 the chain's TRSM operand) -- in claim order
 * and returns the count.  Exposed so the host tests can check the DAG's invariants (every tile
 * produced once, every dependency earlier in claim order or on the chain). */
VBA_API int vba_chol_plan(int32_t nt, int32_t* out5, int32_t cap);

/* Standalone SPD solve H x = b of a dense fp64 n x n system (column-major,
 * lower triangle read; device pointers), replacing np.linalg.solve(Hred, -gred)
 * of solver.py:287.  mode 0: tcgen05 split-fp16 (3-product) Cholesky + fp64 iterative
 * refinement (falls back to mode 1 when its checks fail), mode 1: fp64 Cholesky (one-CTA
 * shared-memory solve up to n = 232, else the DMMA tile DAG; VBA_CHOL=dag forces the DAG), mode 2: tensor-core result unconditionally (diagnostics;
 * info[0] on entry = refinement passes, 0 -> 4).  On return info[0] = 1 if the
 * tensor-core result was used, info[1] = tensor-core pivot failure.  Returns VBA_E_NOT_SPD on a
 * non-positive fp64 pivot.  Synchronises `stream`. */
VBA_API int vba_spd_solve(const double* H, int64_t n, const double* b, double* x, int32_t mode,
                          void* stream, int32_t* info);

/* IMU preintegration of F keyframe pairs, replacing vislam/imu.py:77-167
 * (`preintegrate`, called per pair by the tracking frontend).  Pair f owns the
 * samples soff[f] .. soff[f+1]-1 of ts [S = n_samples = soff[F]] (seconds), gyro [S,3] and accel [S,3];
 * bias [F,6] = (b_g, b_a); noise [4] = (gyro, accel, gyro random walk, accel random
 * walk) densities.  Writes out [F, VBA_PREINT_REC] = dt_total, delta_R quaternion
 * (w,x,y,z; w >= 0), delta_p (3), delta_v (3), J_rot (3x3), J_pos (3x6), J_vel (3x6),
 * covariance (15x15), row-major, fp64.  All pointers are device pointers; `scratch`
 * holds vba_preint_scratch_bytes(n_samples) bytes (caller-owned, reusable).  Returns
 * VBA_E_INVALID (the reference's ValueError) for a pair with fewer than two samples
 * or non-increasing timestamps.  Synchronises `stream`. */
#define VBA_PREINT_REC 281
VBA_API int64_t vba_preint_scratch_bytes(int64_t n_samples);
VBA_API int vba_preintegrate(const double* ts, const double* gyro, const double* accel, int64_t n_samples,
                             const int64_t* soff, int32_t n_pairs, const double* bias, const double* noise,
                             void* scratch, double* out, void* stream);

/* Device-resident hand-off from preintegration to the solver: converts F records of
 * vba_preintegrate (`rec` [F, VBA_PREINT_REC]) plus their bias linearisation points
 * (`bias` [F,6]) into IMU factor records `imu` [F, VBA_IMU_REC] (the host packing of
 * PreintegratedDelta, residuals.py:274-354 inputs), e.g. straight into the buffer bound
 * as vba_problem.imu before vba_bind_inputs(..., refresh_imu = 1).  Stream-ordered, no
 * synchronisation. */
VBA_API int vba_preint_factor_records(const double* rec, const double* bias, int32_t n_pairs, double* imu,
                                      void* stream);

/* Batched device-to-device segment copy (the device-resident tracking window's gather
 * of per-keyframe / per-edge buffers into the solver's packed layout and the scatter of
 * solved disparities back, frontend.py:341-482 without host round trips): `segs` is a
 * DEVICE array of n records {src, dst, bytes}; one launch for all of them.
 * Stream-ordered, no synchronisation. */
typedef struct vba_copy_seg {
  const void* src;
  void* dst;
  int64_t bytes;
} vba_copy_seg;
VBA_API int vba_copy_segments(const vba_copy_seg* segs, int32_t n, void* stream);

/* ------------------------------------------------------------------------
 * Sim(3) pose-graph BA (PGBA), replacing vislam.loopclosure.solve_pgba
 * (loopclosure.py:502-574) and its callees: total_pg_energy (:378-390),
 * _linearize_pg (:425-475), sim3_vision_residual (:225-307),
 * relative_pose_residual (residuals.py:364-380), _pg_apply (:489-499), with the
 * shared damped Schur step solver._solve_step (loopclosure.py:27,534).
 * Nodes are sorted by kid; node 0 is the gauge.  fp64 throughout.
 * ------------------------------------------------------------------------ */
#define VBA_E_NONFINITE 6  /* non-finite initial energy -> RuntimeError (loopclosure.py:520-521) */
#define VBA_PG_REL_REC 64  /* relative edge record: measurement q wxyz (4), t (3), scale (1),
                              information 7x7 row-major (49), padding */

typedef struct vba_pg_problem {
  int32_t n_nodes;        /* K */
  int32_t n_vis;          /* V loop edges with dense correspondences (sorted by source node) */
  int32_t n_rel;          /* R relative edges: loops without vision, then the chain */
  int32_t has_Tcb;
  int64_t n_disp;         /* disparity variables: the pixels of vision-loop source nodes */
  int64_t n_rows;         /* loop-edge rows (= the source's pixels, per edge) */
  double fx, fy, cx, cy;
  double Tcb[7];
  /* device arrays (caller-owned) */
  double* state;          /* [K,8]: q wxyz, t, scale -- read at create, written by vba_pg_download */
  double* disp;           /* [n_disp] -- read at create, written by vba_pg_download */
  const double* pix;      /* [n_disp,2] source pixel coordinates */
  const double* tgt;      /* [n_rows,2] loop correspondences u* (in the target frame) */
  const double* wts;      /* [n_rows,2] confidence weights */
  const double* rel;      /* [R, VBA_PG_REL_REC] */
  /* host topology (read in vba_pg_create only) */
  const int64_t* h_doff;  /* [K+1] disparity offsets (0 pixels for non-source nodes) */
  const int32_t* h_npix;  /* [K] */
  const int32_t* h_vis_i; /* [V] source node */
  const int32_t* h_vis_j; /* [V] target node */
  const int64_t* h_voff;  /* [V+1] row offsets */
  const int32_t* h_rel_i; /* [R] */
  const int32_t* h_rel_j; /* [R] */
} vba_pg_problem;

VBA_API int vba_pg_create(void** ctx, const vba_pg_problem* prob, const vba_options* opts, void* stream);
VBA_API int vba_pg_destroy(void* ctx);
VBA_API int vba_pg_energy(void* ctx, void* stream, double* out_total);                 /* total_pg_energy */
VBA_API int vba_pg_linearize(void* ctx, void* stream);                                 /* _linearize_pg */
/* reference-layout normal equations (H_pp [7K,7K], g_p [7K], H_pd [7K, n_disp] row-major,
 * H_dd/g_d [n_disp]) of the last linearisation; device pointers, any may be NULL */
VBA_API int vba_pg_export_normal_eq(void* ctx, void* stream, double* H_pp, double* g_p, double* H_pd,
                                    double* H_dd, double* g_d);
VBA_API int vba_pg_solve_step(void* ctx, void* stream, double lam, int32_t use_schur);  /* _solve_step */
VBA_API int vba_pg_export_step(void* ctx, void* stream, double* dx_full, double* dx_d);
VBA_API int vba_pg_solve(void* ctx, void* stream, vba_report* report, double* cost_trajectory,
                         int32_t traj_capacity);                                         /* solve_pgba */
VBA_API int vba_pg_download(void* ctx, void* stream);

/* ------------------------------------------------------------------------
 * Stage-2 inertial-only initialisation, replacing vislam.initialization.
 * init_inertial_only (initialization.py:152-231): damped Gauss-Newton over
 * [log-scale, gravity tangent (2), one shared bias (6), velocities (3K)] on the
 * inertial residuals of the vision poses with positions scaled by exp(s).
 * ------------------------------------------------------------------------ */
typedef struct vba_init_problem {
  int32_t n_kf, n_imu;
  const double* q;         /* [K,4] device: vision rotations (fixed) */
  const double* p;         /* [K,3] device: vision positions (unscaled) */
  const double* v0;        /* [K,3] device: velocity seeds (initialization.py:121-134) */
  const double* imu;       /* [F, VBA_IMU_REC] device */
  const int32_t* h_imu_i;  /* [F] host, keyframe indices */
  const int32_t* h_imu_j;
  double grav_q[4], grav_G;   /* initial gravity model */
  double bias0[6];            /* initial shared bias (gyro, accel) */
} vba_init_problem;

typedef struct vba_init_options {
  int32_t max_iterations;     /* InitConfig.max_iterations_inertial */
  double damping;             /* InitConfig.damping */
} vba_init_options;

typedef struct vba_init_result {
  double log_scale;
  double grav_q[4];
  double bias[6];
  int32_t iterations;
  int32_t termination;        /* 0 max_iterations, 1 converged, 2 no_decrease_at_max_damping */
  int32_t n_costs;
  double initial_cost, final_cost;
} vba_init_result;

/* writes the solved velocities to v_out [K,3] (device) and cap costs to cost_trajectory (host) */
VBA_API int vba_init_inertial(const vba_init_problem* prob, const vba_init_options* opts, void* stream,
                              vba_init_result* result, double* cost_trajectory, int32_t cap, double* v_out);

#ifdef __cplusplus
}
#endif
#endif /* VBA_H */
