// vba_host.cu — native runtime of the B200 VI-BA: planner, device workspace,
// C ABI (include/vba.h) and the Levenberg–Marquardt driver.
//
// The driver restates solve_vi_ba (solver.py:344-411 in
// /root/reference/pkg/src/vislam/) with device-resident, double-buffered
// state: a trial writes the "next" buffers, acceptance swaps them in, and a
// rejection simply discards them (the reference's _snapshot/_restore,
// solver.py:311-323).  Exactly one device->host transfer (energy, step norm,
// factorisation status) happens per LM trial, mirroring the accept test at
// solver.py:383.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX ranges (profilers pick them up; no-ops otherwise)

#include "vba_internal.cuh"
#include "vba_plan.h"

namespace vba {

static thread_local std::string g_err;
void vba_set_error_string(const char* msg) { g_err = msg; }
static void set_err(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

#define VBA_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      set_err("%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return VBA_E_CUDA;                                                                \
    }                                                                                   \
  } while (0)

constexpr int kTileRt = kTilePx;   // pixels per per-pixel work tile (vba_internal.cuh)
constexpr int kGramBlock = 512;
constexpr int kMaxOutDegree = 63;   // Gram: 31 in one CTA, up to 63 in unit slices (k_gram<.., 63>)
constexpr int NBc = 128;         // Cholesky tile (vba_chol.cu)
constexpr int kTcMinTiles = 4;   // tensor-core reduced solve from this many 128-tiles up (n >= 385; config 3: 8.2 -> 4.5 ms)

struct Result {       // device -> host once per trial
  double energy[3];
  unsigned long long step_bits;
  int status;         // fp64 factorisation: non-positive pivot
  int tc_bad;         // tensor-core factorisation: non-positive pivot
  double tc[5];       // tensor-core solve: last correction, max |x|, passes, previous rel. correction, accepted
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
};

struct Ctx {
  vba_problem P;
  vba_options O;
  int K = 0, E = 0, F = 0, sdof = 15, ngrav = 0, npv = 0, n_state = 0;
  int nfree = 0, npad = 0, nt = 0, nfk = 0;
  int64_t n_disp = 0, n_rows = 0;
  Extr extr;
  double grid[4];
  double intr[4];
  // host plan
  std::vector<PixTile> tiles;
  std::vector<PixTile> chunks;      // K1/K2 work units (tiles or edge halves of tiles)
  bool k1_split = false;
  std::vector<int32_t> soff, sids, ioff;
  std::vector<StreamItem> sitems;   // K1/K2 static LPT schedule: CTA b owns sids[soff[b] .. soff[b+1])
  int ncta = 0;
  std::vector<int32_t> t0s, t1s, seb, see;
  std::vector<GramTile> gtiles;
  std::vector<int32_t> gsrc, g0, g1, gorder, gsrc_lpt;   // Gram tile / fill-in source launch orders (largest first)
  std::vector<int64_t> goff, foff;
  int kmax = 0;
  size_t gram_smem = 0;
  bool gram_tc = false;   // K4 on tcgen05 (3xTF32) instead of the fp64 DMMA kernel
  int64_t n_part = 0, gram_part_len = 0, gram_len = 0, fill_len = 0;
  int ibs = 0;
  int64_t arena_vis = 0, arena_imu = 0, arena_fill = 0, arena_len = 0;
  std::vector<int32_t> kf_col;   // column offset of each keyframe in the reduced system, -1 frozen
  std::vector<int32_t> fmap;     // npv -> free index or -1
  // device
  std::vector<void*> allocs;
  DevState S[2];
  int cur = 0;
  int32_t *d_ei = nullptr, *d_ej = nullptr, *d_fi = nullptr, *d_fj = nullptr, *d_frozen = nullptr;
  int64_t *d_eoff = nullptr, *d_doff = nullptr;
  PixTile* d_tiles = nullptr;
  int32_t *d_soff = nullptr, *d_sids = nullptr, *d_ioff = nullptr;
  StreamItem* d_sitems = nullptr;
  PixTile* d_chunks = nullptr;
  int32_t *d_t0s = nullptr, *d_t1s = nullptr, *d_seb = nullptr, *d_see = nullptr;
  GramTile* d_gtiles = nullptr;
  int32_t *d_gsrc = nullptr, *d_g0 = nullptr, *d_g1 = nullptr, *d_gorder = nullptr, *d_gsrc_lpt = nullptr;
  int64_t *d_goff = nullptr, *d_foff = nullptr;
  double *d_part = nullptr, *d_tile_e = nullptr, *d_arena = nullptr, *d_gram_part = nullptr, *d_gram = nullptr;
  float *d_Hdd = nullptr, *d_gd = nullptr, *d_ustep = nullptr;
  double* d_dxd = nullptr;
  double *d_L = nullptr;
  int* d_imu_status = nullptr;
  // reduced system
  using Plan = BlkPlan;
  Plan red, exp;
  bool exp_built = false;
  double *d_H = nullptr, *d_rhs = nullptr, *d_x = nullptr, *d_Ld = nullptr, *d_dx = nullptr;
  double* d_cpart = nullptr;       // Cholesky backward-substitution partials
  int* d_cflags = nullptr;         // Cholesky DAG counters
  void* d_ctasks = nullptr;        // Cholesky task list
  int n_ctasks = 0;
  float* d_raytab = nullptr;       // VBA_PIX_GRID: per-column / per-row rays (replaces P.pix)
  const float* pix = nullptr;      // pixel argument of the per-pixel kernels
  void* d_tcws = nullptr;          // tensor-core (3xTF32 + fp64 refinement) solve workspace
  void* d_tctasks = nullptr;       // its task DAG (DIAG-fused critical chain)
  int n_tctasks = 0;
  bool use_tc = false;             // VBA_CHOL=tc: tensor-core reduced solve
  bool use_small = false;          // one-CTA fp64 solve (n <= 232; VBA_CHOL=dag forces the tile DAG)
  bool force_fp64 = false;         // this step: fp64 DAG (tensor-core solve failed its checks)
  bool tc_ran = false;             // the last step's reduced solve ran on the tensor cores
  int tc_gen = 1;
  int tc_iters = 5;   // refinement passes at most (early exit once converged; fp64 fallback beyond)
  int64_t tc_fallbacks = 0;
  int64_t tc_solves = 0, tc_passes = 0;
  int32_t* d_fmap = nullptr;
  Result* d_res = nullptr;
  Result* h_res = nullptr;
  vba_allreduce_fn coll = nullptr;
  void* coll_user = nullptr;
  // edge sharding (vba_problem.shard_*): this rank owns source keyframes [own_k0, own_k1)
  int world = 1, rank = 0, own_k0 = 0, own_k1 = 0;
  std::vector<int32_t> kb;                          // [world+1] keyframe bounds
  int oe0 = 0, oe1 = 0, of0 = 0, of1 = 0, ot0 = 0, ot1 = 0, oc0 = 0, oc1 = 0;   // owned edges/factors/tiles/chunks
  std::vector<int64_t> g_vis, g_imu, g_fill, g_te, g_disp;   // [world+1] gather offsets (doubles)
  std::vector<int32_t> gorder_own, gsrc_own;        // owned Gram tiles (launch order) / fill sources
  int32_t *d_gorder_own = nullptr, *d_gsrc_own = nullptr;
  vba_allgather_fn gat = nullptr;
  void* gat_user = nullptr;
  bool have_step = false;
  double last_lam = 0.0;
  // reference (unpadded) disparity layout, built on first export
  int32_t* d_npix = nullptr;
  int64_t* d_roff_real = nullptr;
  int maxpix = 0;
  int64_t n_real = 0;
  // dense (use_schur=False) verification path, built on first use
  bool dn_ready = false;
  int dn_N = 0, dn_npad = 0, dn_nt = 0, n_dtasks = 0;
  double *d_D = nullptr, *d_drhs = nullptr, *d_dx2 = nullptr, *d_dLinv = nullptr, *d_dpart = nullptr;
  int* d_dflags = nullptr;
  void* d_dtasks = nullptr;
  int32_t* d_kfcol = nullptr;
  unsigned long long* d_trace = nullptr;   // VBA_CHOL_TRACE: per-task timestamps of the Cholesky DAG
  // profiling
  bool prof = false;
  cudaEvent_t ev[10] = {};
  cudaEvent_t sev[3] = {};          // tensor-core solve: factor start, factor end, refinement end
  bool sev_pending = false;
  double solve_ms[2] = {0, 0};      // factorisation kernel, refinement passes
  int64_t solve_samples = 0;
  double stage_ms[6] = {0, 0, 0, 0, 0, 0};
  int64_t k1_launches = 0;
  bool lin_pending = false;
};

template <class T>
static int dalloc(Ctx* c, T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  VBA_CUDA(cudaMalloc((void**)p, n * sizeof(T)));
  c->allocs.push_back((void*)*p);
  return VBA_OK;
}
template <class T>
static int dupload(Ctx* c, T** p, const std::vector<T>& h, cudaStream_t st) {
  int rc = dalloc(c, p, h.size());
  if (rc) return rc;
  if (!h.empty()) VBA_CUDA(cudaMemcpyAsync(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return VBA_OK;
}

static void qmat_h(const double* q, double* R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

// T_bc = T_cb^{-1}; R_bc^T, c2 = R_bc^T p_bc  (residuals.py:187-192, geometry.py:217-219)
static void make_extr(const vba_problem& P, Extr& x) {
  double qi[4] = {1, 0, 0, 0}, t[3] = {0, 0, 0};
  if (P.has_Tcb) {
    const double* q = P.Tcb;
    double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    qi[0] = q[0] / n; qi[1] = -q[1] / n; qi[2] = -q[2] / n; qi[3] = -q[3] / n;
    if (qi[0] < 0) for (double& v : qi) v = -v;
    t[0] = P.Tcb[4]; t[1] = P.Tcb[5]; t[2] = P.Tcb[6];
  }
  qmat_h(qi, x.Rbc);
  for (int a = 0; a < 3; ++a) {
    x.pbc[a] = -(x.Rbc[a * 3 + 0] * t[0] + x.Rbc[a * 3 + 1] * t[1] + x.Rbc[a * 3 + 2] * t[2]);
    for (int b = 0; b < 3; ++b) x.RbcT[a * 3 + b] = x.Rbc[b * 3 + a];
  }
  for (int a = 0; a < 3; ++a)
    x.c2[a] = x.RbcT[a * 3 + 0] * x.pbc[0] + x.RbcT[a * 3 + 1] * x.pbc[1] + x.RbcT[a * 3 + 2] * x.pbc[2];
}

static int upload_plan(Ctx* c, BlkBuilder& B, const std::vector<int32_t>& roff, const std::vector<int32_t>& rdim,
                       Ctx::Plan& pl, cudaStream_t st) {
  const cudaError_t e = upload_blk_plan(c->allocs, B, roff, rdim, pl, st);
  if (e != cudaSuccess) { set_err("plan upload: %s", cudaGetErrorString(e)); return VBA_E_CUDA; }
  return VBA_OK;
}

// Block indices: `bidx[n]` block of keyframe n (-1 = excluded), gravity block `gb` (-1 = none).
static void add_all(Ctx* c, BlkBuilder& B, const std::vector<int>& bidx, int gb, bool with_fill) {
  const int s = c->sdof;
  const std::vector<int32_t>& ei = c->seb;  (void)ei;
  // vision edges: [Hii 36][Hjj 36][Hij 36][gi 6][gj 6]
  for (int e = 0; e < c->E; ++e) {
    const int i = bidx[c->P.h_edge_i[e]], j = bidx[c->P.h_edge_j[e]];
    const int64_t o = c->arena_vis + (int64_t)kVisBlock * e;
    B.add(i, i, o, 6, 6, 6, 1, false);
    B.add(j, j, o + 36, 6, 6, 6, 1, false);
    if (c->P.h_edge_i[e] == c->P.h_edge_j[e]) B.add_both(i, j, o + 72, 6, 6, 6, 1, false);
    else B.add(i, j, o + 72, 6, 6, 6, 1, false);
    B.addv(i, o + 108, 6, 1);
    B.addv(j, o + 114, 6, 1);
  }
  // IMU factors: [Hii][Hjj][Hij][gi][gj][Hgg 4][Hig s*2][Hjg s*2][gg 2][E]
  for (int f = 0; f < c->F; ++f) {
    const int i = bidx[c->P.h_imu_i[f]], j = bidx[c->P.h_imu_j[f]];
    const int64_t o = c->arena_imu + (int64_t)c->ibs * f;
    const int s2 = s * s;
    B.add(i, i, o, s, s, s, 1, false);
    B.add(j, j, o + s2, s, s, s, 1, false);
    if (c->P.h_imu_i[f] == c->P.h_imu_j[f]) B.add_both(i, j, o + 2 * s2, s, s, s, 1, false);
    else B.add(i, j, o + 2 * s2, s, s, s, 1, false);
    B.addv(i, o + 3 * s2, s, 1);
    B.addv(j, o + 3 * s2 + s, s, 1);
    if (gb >= 0) {
      B.add(gb, gb, o + 3 * s2 + 2 * s, 2, 2, 2, 1, false);
      B.add(i, gb, o + 3 * s2 + 2 * s + 4, 2, s, 2, 1, false);
      B.add(j, gb, o + 3 * s2 + 4 * s + 4, 2, s, 2, 1, false);
      B.addv(gb, o + 3 * s2 + 6 * s + 4, 2, 1);
    }
  }
  if (!with_fill) return;
  // fill-in per source: [F_ii][F_ij k][F_jj npairs][gr_i][gr_j k], subtracted
  for (size_t q = 0; q < c->gsrc.size(); ++q) {
    const int src = c->gsrc[q];
    const int eb = c->seb[src], k = c->see[src] - eb, np = k * (k + 1) / 2;
    const int64_t o = c->arena_fill + c->foff[src];
    const int bi = bidx[src];
    B.add(bi, bi, o, 6, 6, 6, -1, true);
    for (int e = 0; e < k; ++e) {
      const int kj = c->P.h_edge_j[eb + e];
      if (kj == src) B.add_both(bi, bidx[kj], o + 36 + 36 * e, 6, 6, 6, -1, true);
      else B.add(bi, bidx[kj], o + 36 + 36 * e, 6, 6, 6, -1, true);
    }
    for (int e1 = 0; e1 < k; ++e1)
      for (int e2 = 0; e2 <= e1; ++e2) {
        const int p = e1 * (e1 + 1) / 2 + e2;
        const int k1 = c->P.h_edge_j[eb + e1], k2 = c->P.h_edge_j[eb + e2];
        const int64_t off = o + 36 + 36 * k + 36 * p;
        if (k1 == k2 && e1 != e2) B.add_both(bidx[k1], bidx[k2], off, 6, 6, 6, -1, true);
        else B.add(bidx[k1], bidx[k2], off, 6, 6, 6, -1, true);
      }
    const int64_t go = o + 36 + 36 * k + 36 * np;
    B.addv(bi, go, 6, -1);
    for (int e = 0; e < k; ++e) B.addv(bidx[c->P.h_edge_j[eb + e]], go + 6 + 6 * e, 6, -1);
  }
}

static int build_plans(Ctx* c, cudaStream_t st) {
  const vba_problem& P = c->P;
  const int K = c->K, E = c->E;
  // --- sources and per-pixel tiles
  c->seb.assign(K, 0);
  c->see.assign(K, 0);
  for (int e = 0; e < E; ++e) {
    const int i = P.h_edge_i[e], j = P.h_edge_j[e];
    if (i < 0 || i >= K || j < 0 || j >= K) { set_err("edge %d references keyframe out of range", e); return VBA_E_INVALID; }
    if (e > 0 && i < P.h_edge_i[e - 1]) { set_err("vision edges must be sorted by source keyframe"); return VBA_E_INVALID; }
    if (P.h_eoff[e] % 4 != 0) { set_err("edge row offsets must be multiples of 4"); return VBA_E_INVALID; }
  }
  for (int n = 0; n < K; ++n) { c->seb[n] = 0; c->see[n] = 0; }
  {
    int e = 0;
    for (int n = 0; n < K; ++n) {
      c->seb[n] = e;
      while (e < E && P.h_edge_i[e] == n) ++e;
      c->see[n] = e;
    }
  }
  c->t0s.assign(K, 0);
  c->t1s.assign(K, 0);
  int64_t poff = 0;
  c->kmax = 0;
  for (int n = 0; n < K; ++n) {
    const int64_t npad = P.h_doff[n + 1] - P.h_doff[n];
    if (npad % 4 != 0) { set_err("keyframe disparity segments must be padded to 4"); return VBA_E_INVALID; }
    const int k = c->see[n] - c->seb[n];
    if (k > kMaxOutDegree) {
      set_err("keyframe %d has out-degree %d > %d (the Schur Gram stages at most 6*%d+1 coupling columns)", n, k,
              kMaxOutDegree, kMaxOutDegree);
      return VBA_E_UNSUPPORTED;
    }
    c->kmax = std::max(c->kmax, k);
    c->t0s[n] = (int)c->tiles.size();
    for (int64_t n0 = 0; n0 < npad; n0 += kTileRt) {
      PixTile t{};
      t.src = n;
      t.n0 = (int)n0;
      t.cnt = (int)std::min<int64_t>(kTileRt, npad - n0);
      t.eb = c->seb[n];
      t.ee = c->see[n];
      t.poff = poff;
      poff += k;
      c->tiles.push_back(t);
    }
    c->t1s[n] = (int)c->tiles.size();
  }
  c->n_part = poff;
  {  // K1/K2 schedule.  Work units ("chunks") are tiles with out-edges, split into two
     // halves of their edge list when there are too few tiles per CTA to balance
     // (then H_dd / g_d get the two partial sums by atomic adds onto zero: two
     // addends, so the result is order-independent); longest first, each to the
     // least-loaded CTA (LPT).
    const int G = vision_stream_ctas();
    int nt_edges = 0;
    for (const PixTile& T : c->tiles) nt_edges += T.ee > T.eb;
    const bool split = nt_edges < 8 * G;
    c->chunks.clear();
    c->k1_split = false;
    for (const PixTile& T : c->tiles) {
      const int k = T.ee - T.eb;
      if (k <= 0) continue;
      if (split && k >= 2) {
        PixTile a = T, b = T;
        a.ee = T.eb + (k + 1) / 2;
        b.eb = a.ee;
        b.poff = T.poff + (b.eb - T.eb);
        a.pad = b.pad = 1;   // partial H_dd / g_d: accumulate atomically
        c->chunks.push_back(a);
        c->chunks.push_back(b);
        c->k1_split = true;
      } else {
        PixTile a = T;
        a.pad = 0;
        c->chunks.push_back(a);
      }
    }
    // Cost of an item = a fixed per-item part + its 64-pixel blocks holding any non-zero
    // weight (K1 skips all-zero blocks, so invisible regions are nearly free); counted once
    // per solve on the device from the caller's weights (tiles x out-edges = the K1 partials).
    std::vector<int32_t> nzb((size_t)std::max<int64_t>(c->n_part, 1), kTileRt / 64);
    if (c->n_part > 0 && c->P.wts) {
      std::vector<int64_t> prow((size_t)c->n_part);
      std::vector<int32_t> pcnt((size_t)c->n_part);
      for (const PixTile& T : c->tiles)
        for (int e = T.eb; e < T.ee; ++e) {
          prow[T.poff + (e - T.eb)] = P.h_eoff[e] + T.n0;
          pcnt[T.poff + (e - T.eb)] = T.cnt;
        }
      int64_t* d_prow = nullptr;
      int32_t *d_pcnt = nullptr, *d_nz = nullptr;
      if (cudaMalloc(&d_prow, sizeof(int64_t) * prow.size()) || cudaMalloc(&d_pcnt, sizeof(int32_t) * pcnt.size()) ||
          cudaMalloc(&d_nz, sizeof(int32_t) * pcnt.size())) {
        cudaFree(d_prow); cudaFree(d_pcnt); cudaFree(d_nz);
        set_err("planner allocation failed");
        return VBA_E_CUDA;
      }
      cudaMemcpyAsync(d_prow, prow.data(), sizeof(int64_t) * prow.size(), cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(d_pcnt, pcnt.data(), sizeof(int32_t) * pcnt.size(), cudaMemcpyHostToDevice, st);
      launch_count_nz_blocks(c->P.wts, d_prow, d_pcnt, (int)pcnt.size(),
                             P.pixel_mode == VBA_PIX_GRID ? P.grid_w : 0, d_nz, st);
      cudaMemcpyAsync(nzb.data(), d_nz, sizeof(int32_t) * pcnt.size(), cudaMemcpyDeviceToHost, st);
      const cudaError_t err = cudaStreamSynchronize(st);
      cudaFree(d_prow); cudaFree(d_pcnt); cudaFree(d_nz);
      if (err != cudaSuccess) { set_err("planner: %s", cudaGetErrorString(err)); return VBA_E_CUDA; }
    }
    std::vector<int32_t> order(c->chunks.size());
    for (int t = 0; t < (int)order.size(); ++t) order[t] = t;
    auto work = [&](int t) {   // per item: ~10 blocks' worth of fixed cost + the non-zero blocks
      const PixTile& T = c->chunks[t];
      int64_t w = 2 * kTileRt / 64;   // per-chunk setup
      for (int e = T.eb; e < T.ee; ++e) w += 10 + nzb[T.poff + (e - T.eb)];
      return w;
    };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return work(a) > work(b); });
    // a sharded rank streams only the chunks of its own source keyframes (the chunk list,
    // and with it every partial's slot, is the global one on every rank)
    order.erase(std::remove_if(order.begin(), order.end(),
                               [&](int t) { return c->chunks[t].src < c->own_k0 || c->chunks[t].src >= c->own_k1; }),
                order.end());
    c->ncta = std::min<int>(G, (int)order.size());
    std::vector<std::vector<int32_t>> bins(c->ncta);
    std::vector<std::pair<int64_t, int>> heap;
    for (int b = 0; b < c->ncta; ++b) heap.push_back({0, b});
    auto cmp = [](const std::pair<int64_t, int>& x, const std::pair<int64_t, int>& y) { return x > y; };
    std::make_heap(heap.begin(), heap.end(), cmp);
    for (int t : order) {
      std::pop_heap(heap.begin(), heap.end(), cmp);
      heap.back().first += work(t);
      bins[heap.back().second].push_back(t);
      std::push_heap(heap.begin(), heap.end(), cmp);
    }
    c->soff.assign(1, 0);
    c->sids.clear();
    c->ioff.assign(1, 0);
    c->sitems.clear();
    for (auto& bn : bins) {
      c->sids.insert(c->sids.end(), bn.begin(), bn.end());
      c->soff.push_back((int32_t)c->sids.size());
      for (int t : bn) {
        const PixTile& T = c->chunks[t];
        for (int e = T.eb; e < T.ee; ++e)
          c->sitems.push_back(StreamItem{2 * (P.h_eoff[e] + T.n0), 8 * T.cnt, e});
      }
      c->ioff.push_back((int32_t)c->sitems.size());
    }
    if (c->sids.empty()) c->sids.push_back(0);
    if (c->sitems.empty()) c->sitems.push_back(StreamItem{0, 0, 0});
    if (c->chunks.empty()) c->chunks.push_back(PixTile{});
  }
  // --- Gram tiles
  int nsrc = 0;
  int64_t work_px = 0;
  for (int n = 0; n < K; ++n)
    if (c->see[n] > c->seb[n] && P.h_npix[n] > 0) { ++nsrc; work_px += P.h_npix[n]; }
  // ~7 waves of CTAs on 148 SMs (wave quantisation of the 1-CTA-per-SM Gram kernel)
  const int target = getenv("VBA_GRAM_TARGET") ? atoi(getenv("VBA_GRAM_TARGET")) : 1024;
  c->goff.assign(K, 0);
  c->foff.assign(K, 0);
  c->g0.assign(K, 0);
  c->g1.assign(K, 0);
  int64_t gpo = 0, go = 0, fo = 0;
  c->gram_smem = 0;
  for (int n = 0; n < K; ++n) {
    const int k = c->see[n] - c->seb[n];
    const int npix = P.h_npix[n];
    c->g0[n] = c->g1[n] = (int)c->gtiles.size();
    if (k == 0 || npix == 0) continue;
    c->gsrc.push_back(n);
    const int np = k * (k + 1) / 2;
    int nsplit = std::max(1, std::min(16, kGramBlock / np));
    while (nsplit > 1 && gram_smem_bytes(c->kmax, nsplit, np, k) > 200 * 1024) --nsplit;
    c->gram_smem = std::max(c->gram_smem, gram_smem_bytes(c->kmax, nsplit, np, k));
    int R = std::max(1, (int)((target + nsrc - 1) / nsrc));
    R = std::min(R, std::max(1, npix / 256));
    // more than 31 out-edges: one pixel range (k_fill_transform reads its record in place),
    // its 2x2 tile units in slices of gram_slice_units() per CTA (the DMMA Gram)
    const bool big = k > 31;
    if (big) R = 1;
    const int U = big ? gram_units(k) : 0, su = gram_slice_units();
    const int chunk = ((npix + R - 1) / R + 31) / 32 * 32;   // whole k_gram staging chunks (kGramPC)
    for (int a = 0; a < npix; a += chunk) {
      for (int u0 = 0; u0 < (big ? U : 1); u0 += su) {
        GramTile g{};
        g.src = n;
        g.n0 = a;
        g.n1 = std::min(npix, a + chunk);
        g.eb = c->seb[n];
        g.ee = c->see[n];
        g.nsplit = nsplit;
        g.u0 = big ? u0 : 0;
        g.u1 = big ? std::min(U, u0 + su) : 0;
        g.out = gpo;
        c->gtiles.push_back(g);
      }
      gpo += (int64_t)np * 36 + 6 * k;
    }
    c->g1[n] = (int)c->gtiles.size();
    c->goff[n] = go;
    go += (int64_t)np * 36 + 6 * k;
    c->foff[n] = fo;
    fo += (int64_t)(1 + k + np) * 36 + 6 * (1 + k);
  }
  // K4 path: the tensor-core Gram (3xTF32, fp32 accumulation per pixel range) for windows
  // with >= 256 pixels per source keyframe, the exact fp64 DMMA Gram for the small ones
  // (where it costs little and ill-conditioned windows keep every bit); VBA_GRAM=tc|dmma forces
  {
    const char* gm = getenv("VBA_GRAM");
    c->gram_tc = gm ? (strcmp(gm, "tc") == 0) : (nsrc > 0 && work_px >= 256 * (int64_t)nsrc);
    if (c->kmax > 31) c->gram_tc = false;   // the tensor-core Gram holds 31 out-edges per CTA
    if (c->gram_tc) c->gram_smem = gram_tc_smem_bytes(c->kmax);
  }
  if (c->gram_smem > 227 * 1024) { set_err("Gram kernel shared memory too large"); return VBA_E_UNSUPPORTED; }
  // Gram launch order: longest tiles (pixels x edge pairs) first, so the last of the ~7
  // waves of one-CTA-per-SM tiles are the short ones.  Only the launch order changes: each
  // tile keeps its output slot and the partials are summed in tile-index order (bitwise).
  c->gorder.resize(c->gtiles.size());
  for (size_t t = 0; t < c->gtiles.size(); ++t) c->gorder[t] = (int32_t)t;
  auto tile_work = [&](int32_t t) {
    const GramTile& g = c->gtiles[t];
    const int64_t k = g.ee - g.eb;
    return (int64_t)(g.n1 - g.n0) * k * (k + 1);
  };
  std::stable_sort(c->gorder.begin(), c->gorder.end(),
                   [&](int32_t x, int32_t y) { return tile_work(x) > tile_work(y); });
  c->gsrc_lpt = c->gsrc;   // k_fill_transform: one CTA per source, most out-edges first
  std::stable_sort(c->gsrc_lpt.begin(), c->gsrc_lpt.end(), [&](int32_t x, int32_t y) {
    return c->see[x] - c->seb[x] > c->see[y] - c->seb[y];
  });
  c->gram_part_len = gpo;
  c->gram_len = go;
  c->fill_len = fo;
  for (int32_t t : c->gorder)
    if (c->gtiles[t].src >= c->own_k0 && c->gtiles[t].src < c->own_k1) c->gorder_own.push_back(t);
  for (int32_t n : c->gsrc_lpt)
    if (n >= c->own_k0 && n < c->own_k1) c->gsrc_own.push_back(n);
  // --- arena layout
  const int s = c->sdof;
  c->ibs = ((3 * s * s + 6 * s + 7) + 7) / 8 * 8;
  c->arena_vis = 0;
  c->arena_imu = (int64_t)kVisBlock * E;
  c->arena_fill = c->arena_imu + (int64_t)c->ibs * c->F;
  c->arena_len = c->arena_fill + c->fill_len;
  {  // sharding: owned ranges and the per-rank slices every gather moves
    auto edge_at = [&](int n) { return n < K ? c->seb[n] : E; };
    auto tile_at = [&](int n) { return n < K ? c->t0s[n] : (int)c->tiles.size(); };
    std::vector<int32_t> chunk_at(K + 1, 0), fac_at(K + 1, 0);
    std::vector<int64_t> fill_at(K + 1, 0);
    {
      size_t q = 0;
      for (int n = 0; n <= K; ++n) {
        while (q < c->chunks.size() && c->chunks[q].ee > c->chunks[q].eb && c->chunks[q].src < n) ++q;
        chunk_at[n] = (int32_t)q;
      }
      int f = 0;
      for (int n = 0; n <= K; ++n) {
        while (f < c->F && P.h_imu_i[f] < n) ++f;
        fac_at[n] = f;
      }
    }
    // fill offsets per source are cumulative in source order (foff[n] for sources with a Gram)
    {
      int64_t acc = 0;
      for (int n = 0; n < K; ++n) {
        fill_at[n] = acc;
        const int k = c->see[n] - c->seb[n];
        if (k > 0 && P.h_npix[n] > 0) acc += (int64_t)(1 + k + k * (k + 1) / 2) * 36 + 6 * (1 + k);
      }
      fill_at[K] = acc;
    }
    c->oe0 = edge_at(c->own_k0); c->oe1 = edge_at(c->own_k1);
    c->ot0 = tile_at(c->own_k0); c->ot1 = tile_at(c->own_k1);
    c->oc0 = chunk_at[c->own_k0]; c->oc1 = chunk_at[c->own_k1];
    c->of0 = fac_at[c->own_k0]; c->of1 = fac_at[c->own_k1];
    for (int r = 0; r <= c->world; ++r) {
      const int n = c->kb[r];
      c->g_vis.push_back(c->arena_vis + (int64_t)kVisBlock * edge_at(n));
      c->g_imu.push_back(c->arena_imu + (int64_t)c->ibs * fac_at[n]);
      c->g_fill.push_back(c->arena_fill + fill_at[n]);
      c->g_te.push_back((int64_t)kPartWarps * chunk_at[n]);
      c->g_disp.push_back(P.h_doff[n]);
    }
  }
  // --- reduced-system layout (free keyframes, then gravity)
  std::vector<int> bidx(K, -1);
  std::vector<int32_t> roff, rdim;
  c->kf_col.assign(K, -1);
  int col = 0, nb = 0;
  for (int n = 0; n < K; ++n) {
    if (P.h_frozen[n]) continue;
    bidx[n] = nb++;
    c->kf_col[n] = col;
    roff.push_back(col);
    rdim.push_back(s);
    col += s;
  }
  c->nfk = nb;
  int gb = -1;
  if (c->ngrav) {
    gb = nb++;
    roff.push_back(col);
    rdim.push_back(2);
    col += 2;
  }
  c->nfree = col;
  c->npad = (col + NBc - 1) / NBc * NBc;
  c->nt = c->npad / NBc;
  c->fmap.assign(c->npv, -1);
  for (int n = 0; n < K; ++n)
    if (c->kf_col[n] >= 0)
      for (int r = 0; r < s; ++r) c->fmap[n * s + r] = c->kf_col[n] + r;
  if (c->ngrav)
    for (int r = 0; r < 2; ++r) c->fmap[c->n_state + r] = c->nfree - 2 + r;
  BlkBuilder B(nb);
  add_all(c, B, bidx, gb, true);
  return upload_plan(c, B, roff, rdim, c->red, st);
}

static int build_export_plan(Ctx* c, cudaStream_t st) {
  if (c->exp_built) return VBA_OK;
  const int K = c->K, s = c->sdof;
  std::vector<int> bidx(K);
  std::vector<int32_t> roff, rdim;
  for (int n = 0; n < K; ++n) {
    bidx[n] = n;
    roff.push_back(n * s);
    rdim.push_back(s);
  }
  int gb = -1;
  if (c->ngrav) {
    gb = K;
    roff.push_back(K * s);
    rdim.push_back(2);
  }
  BlkBuilder B(K + (c->ngrav ? 1 : 0));
  add_all(c, B, bidx, gb, false);
  int rc = upload_plan(c, B, roff, rdim, c->exp, st);
  if (rc) return rc;
  c->exp_built = true;
  return VBA_OK;
}

// ---------------------------------------------------------------------------
// stages
// ---------------------------------------------------------------------------
static DevState& CUR(Ctx* c) { return c->S[c->cur]; }
static DevState& NXT(Ctx* c) { return c->S[c->cur ^ 1]; }

// optional per-stage CUDA-event timing (vba_set_profiling), events on the launch stream:
//   7 | 0 edge prep | 8 K1 kernel | 9 finalize + IMU | 1     (linearisation)
//   2 gram+fill | 3 assemble+chol | 4 backsub+retract | 5 energy | 6     (trial)
// stage_ms: [0] linearise (all) [1] gram+fill [2] assemble+chol [3] backsub+retract
//           [4] energy [5] K1 kernel alone;  k1_launches counts [5]'s samples.
static void mark(Ctx* c, int i, cudaStream_t st) {
  if (c->prof) cudaEventRecord(c->ev[i], st);
}
static void prof_collect(Ctx* c, bool with_lin) {
  if (!c->prof) return;
  float ms;
  if (with_lin && cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]) == cudaSuccess) c->stage_ms[0] += ms;
  if (with_lin && cudaEventElapsedTime(&ms, c->ev[8], c->ev[9]) == cudaSuccess) {
    c->stage_ms[5] += ms;
    c->k1_launches += 1;
  }
  for (int s = 0; s < 4; ++s)
    if (cudaEventElapsedTime(&ms, c->ev[2 + s], c->ev[3 + s]) == cudaSuccess) c->stage_ms[1 + s] += ms;
  if (c->sev_pending) {
    float f = 0.f, r = 0.f;
    if (cudaEventElapsedTime(&f, c->sev[0], c->sev[1]) == cudaSuccess &&
        cudaEventElapsedTime(&r, c->sev[1], c->sev[2]) == cudaSuccess) {
      c->solve_ms[0] += f;
      c->solve_ms[1] += r;
      c->solve_samples += 1;
    }
    c->sev_pending = false;
  }
}

// sharded solve: every rank receives the other ranks' slices of buf (offsets per rank)
static int gather(Ctx* c, double* buf, const std::vector<int64_t>& off, cudaStream_t st, const char* what) {
  if (c->world <= 1) return VBA_OK;
  if (!c->gat) { set_err("sharded solve without a gather hook (vba_set_gather)"); return VBA_E_INVALID; }
  if (c->gat(c->gat_user, buf, off.data(), c->world, st)) { set_err("gather(%s) failed", what); return VBA_E_CUDA; }
  return VBA_OK;
}

// seed a state buffer's disparities from the caller: the fp64 master from vba_problem.disp64
// when given (its fp32 copy derived), else from the fp32 vba_problem.disp (widened)
static int load_disparities(Ctx* c, DevState& s, cudaStream_t st) {
  if (!c->n_disp) return 0;
  if (c->P.disp64) {
    if (cudaMemcpyAsync(s.disp64, c->P.disp64, sizeof(double) * c->n_disp, cudaMemcpyDeviceToDevice, st)) return 1;
    launch_narrow(s.disp64, s.disp, c->n_disp, st);
  } else {
    if (cudaMemcpyAsync(s.disp, c->P.disp, sizeof(float) * c->n_disp, cudaMemcpyDeviceToDevice, st)) return 1;
    launch_widen(s.disp, s.disp64, c->n_disp, st);
  }
  return cudaGetLastError() != cudaSuccess;
}

static int stage_energy(Ctx* c, DevState& s, cudaStream_t st) {
  launch_edge_prep(s, c->d_ei, c->d_ej, c->E, c->extr, st);
  launch_vision_energy(c->P.pixel_mode, c->d_chunks, c->d_soff, c->d_sids, c->d_sitems, c->d_ioff, c->ncta, s, c->pix, c->P.tgt, c->P.wts,
                       c->d_eoff, c->d_doff, c->P.grid_w, c->grid, c->intr, c->d_tile_e, st);
  launch_imu_factor(c->P.imu, c->d_L, c->d_fi, c->d_fj, c->of0, c->of1 - c->of0, s, c->P.ts, c->sdof, c->ibs, 1,
                    c->d_arena + c->arena_imu, st);
  int rc;
  if ((rc = gather(c, c->d_tile_e, c->g_te, st, "energy partials")) ||
      (rc = gather(c, c->d_arena, c->g_imu, st, "IMU factors")))
    return rc;
  const int oE = 3 * c->sdof * c->sdof + 6 * c->sdof + 6;
  launch_energy_reduce(c->d_tile_e, (int)c->chunks.size() * kPartWarps, c->d_arena + c->arena_imu, c->F, c->ibs, oE,
                       c->d_res->energy, st);
  return VBA_OK;
}

static int stage_linearize(Ctx* c, cudaStream_t st) {
  DevState& s = CUR(c);
  mark(c, 0, st);
  c->lin_pending = true;
  if (c->k1_split) {   // split chunks add their partial H_dd / g_d onto zero
    cudaMemsetAsync(c->d_Hdd, 0, sizeof(float) * std::max<int64_t>(1, c->n_disp), st);
    cudaMemsetAsync(c->d_gd, 0, sizeof(float) * std::max<int64_t>(1, c->n_disp), st);
  }
  launch_edge_prep(s, c->d_ei, c->d_ej, c->E, c->extr, st);
  mark(c, 8, st);
  launch_vision_linearize(c->P.pixel_mode, c->d_chunks, c->d_soff, c->d_sids, c->d_sitems, c->d_ioff, c->ncta, s, c->pix, c->P.tgt, c->P.wts,
                          c->d_eoff, c->d_doff, c->P.grid_w, c->grid, c->intr, c->d_part, c->d_Hdd, c->d_gd, st);
  mark(c, 9, st);
  launch_edge_finalize(c->d_t0s, c->d_t1s, c->d_tiles, c->d_ei, c->oe0, c->oe1 - c->oe0, c->d_part, s, c->extr,
                       c->d_arena + c->arena_vis, nullptr, st);
  launch_imu_factor(c->P.imu, c->d_L, c->d_fi, c->d_fj, c->of0, c->of1 - c->of0, s, c->P.ts, c->sdof, c->ibs, 0,
                    c->d_arena + c->arena_imu, st);
  int rc;
  if ((rc = gather(c, c->d_arena, c->g_vis, st, "vision blocks")) ||
      (rc = gather(c, c->d_arena, c->g_imu, st, "IMU blocks")))
    return rc;
  mark(c, 1, st);
  return VBA_OK;
}

// Schur fill-in + freeze/damp assembly of the reduced system H_red (lower triangle of
// d_H, column-major) and its right-hand side -g_red (d_rhs), all-reduced across ranks
// for a sharded solve (solver.py:272-285)
static int stage_reduce(Ctx* c, double lam, cudaStream_t st) {
  DevState& s = CUR(c);
  mark(c, 2, st);
  VBA_CUDA(cudaMemsetAsync(c->d_res, 0, sizeof(Result), st));
  if (!c->gorder_own.empty()) {
    if (c->gram_tc)
      launch_gram_tc(c->P.pixel_mode, c->d_gtiles, (int)c->gorder_own.size(), c->gram_smem, c->kmax, s, c->pix,
                     c->P.wts, c->d_eoff, c->d_doff, c->P.grid_w, c->grid, c->intr, c->d_Hdd, c->d_gd, lam,
                     c->O.ridge, c->d_gram_part, st, c->d_gorder_own);
    else
      launch_gram(c->P.pixel_mode, c->d_gtiles, (int)c->gorder_own.size(), kGramBlock, c->gram_smem, c->kmax, s,
                  c->pix, c->P.wts, c->d_eoff, c->d_doff, c->P.grid_w, c->grid, c->intr, c->d_Hdd, c->d_gd, lam,
                  c->O.ridge, c->d_gram_part, st, c->d_gorder_own);
    launch_fill_transform(c->d_gsrc_own, (int)c->gsrc_own.size(), c->d_seb, c->d_see, c->d_g0, c->d_g1,
                          c->d_gtiles, c->d_foff, c->d_gram_part, s, c->extr, c->d_arena + c->arena_fill, c->kmax,
                          st);
  }
  int rc = gather(c, c->d_arena, c->g_fill, st, "fill-in blocks");
  if (rc) return rc;
  mark(c, 3, st);
  if (c->nfree > 0) {
    // every rank now holds the whole arena: the identical assembly (blocks with contributions
    // only; the others stay at the zeros of vba_create), lower triangle read by the solves
    launch_assemble(c->red.bptr, c->red.bnff, c->red.cs, c->red.nbr, c->red.roff, c->red.rdim, c->d_arena, lam,
                    c->O.ridge, 1, c->d_H, c->npad, 0, st, c->red.blist, c->red.nblist);
    // right-hand side -g_red: the step solves H_red dx = -g_red (solver.py:287)
    launch_assemble_vec(c->red.sptr, c->red.vs, c->red.nseg, c->red.soff, c->d_arena, -1.0, c->d_rhs, st);
  }
  return VBA_OK;
}

// reduced system + Cholesky + back-substitution into the NEXT buffers
static int stage_step(Ctx* c, double lam, cudaStream_t st) {
  DevState& s = CUR(c);
  DevState& n = NXT(c);
  int rc = stage_reduce(c, lam, st);
  if (rc) return rc;
  if (c->nfree > 0) {
    if (getenv("VBA_CHOL_TRACE") && !c->d_trace) {
      if (dalloc(c, &c->d_trace, (size_t)4 * std::max(1, c->n_ctasks) + 16 * (size_t)std::max(1, c->nt)))
        return VBA_E_CUDA;
    }
    bool tc_ran = false;
    if (c->use_tc && !c->force_fp64 && !c->d_trace) {
      // returns non-zero (before any refinement) when the system is too large for its
      // co-resident triangular solves: solved on the fp64 DAG below instead
      tc_ran = chol_tc_solve(c->d_H, c->npad, c->nfree, c->npad, c->d_rhs, c->d_x, c->d_tcws, c->d_tctasks,
                             c->n_tctasks, c->tc_iters, &c->d_res->tc_bad, c->tc_gen, st, c->d_res->tc, nullptr,
                             c->prof ? c->sev : nullptr) == 0;
      c->sev_pending = c->prof && tc_ran;
      c->tc_gen += 2 * c->tc_iters;
    }
    c->tc_ran = tc_ran;
    if (!tc_ran) {
      // small systems: the one-CTA solve (vba_small.cu); else the fp64 tile DAG
      if (!c->use_small || c->d_trace ||
          chol_small_solve(c->d_H, c->npad, c->nfree, c->d_rhs, c->d_x, &c->d_res->status, st))
        chol_dag_launch(c->d_H, c->npad, c->nt, c->d_rhs, c->d_x, c->d_Ld, c->d_cpart, c->d_cflags, c->d_ctasks,
                        c->n_ctasks, &c->d_res->status, st, c->d_trace);
    }
  }
  mark(c, 4, st);
  launch_scatter_dx(c->d_x, c->d_fmap, c->npv, c->d_dx, st);
  launch_step_edges(c->d_ei, c->d_ej, c->E, s, c->extr, c->d_dx, c->sdof, c->d_ustep, st);
  launch_backsub(c->P.pixel_mode, c->d_tiles + c->ot0, c->ot1 - c->ot0, s, n, c->pix, c->P.wts, c->d_eoff,
                 c->d_doff, c->P.grid_w, c->grid, c->intr, c->d_Hdd, c->d_gd, c->d_ustep, lam, c->O.ridge,
                 c->d_dxd, &c->d_res->step_bits, st);
  launch_retract(s, n, c->d_dx, c->d_frozen, c->K, c->sdof, c->ngrav, c->n_state, &c->d_res->step_bits, c->npv, st);
  c->have_step = true;
  c->last_lam = lam;
  return VBA_OK;
}

// ---------------------------------------------------------------------------
// dense reference path (use_schur=False, solver.py:291-304): the full
// [free poses | disparities] system is materialised and factorised with the
// same DAG Cholesky.  Meant for small verification problems, like the reference's.
// ---------------------------------------------------------------------------
static int ensure_real_layout(Ctx* c, cudaStream_t st) {
  if (c->d_npix) return VBA_OK;
  std::vector<int32_t> np(c->P.h_npix, c->P.h_npix + c->K);
  std::vector<int64_t> ro(c->K + 1, 0);
  c->maxpix = 0;
  for (int n = 0; n < c->K; ++n) {
    ro[n + 1] = ro[n] + np[n];
    c->maxpix = std::max(c->maxpix, np[n]);
  }
  c->n_real = ro[c->K];
  int rc;
  if ((rc = dupload(c, &c->d_npix, np, st)) || (rc = dupload(c, &c->d_roff_real, ro, st))) return rc;
  return VBA_OK;
}


static int ensure_dense(Ctx* c, cudaStream_t st) {
  if (c->dn_ready) return VBA_OK;
  int rc = ensure_real_layout(c, st);
  if (rc) return rc;
  const int64_t N = c->nfree + c->n_real;
  if (N > 32768) {
    set_err("use_schur=False: dense system of %lld unknowns exceeds the verification-path limit", (long long)N);
    return VBA_E_UNSUPPORTED;
  }
  c->dn_N = (int)N;
  c->dn_npad = (int)((N + NBc - 1) / NBc * NBc);
  c->dn_nt = c->dn_npad / NBc;
  const size_t np = (size_t)c->dn_npad;
  if ((rc = dalloc(c, &c->d_D, np * np)) || (rc = dalloc(c, &c->d_drhs, np)) || (rc = dalloc(c, &c->d_dx2, np)) ||
      (rc = dalloc(c, &c->d_dLinv, (size_t)c->dn_nt * NBc * NBc)) ||
      (rc = dalloc(c, &c->d_dpart, (size_t)c->dn_nt * c->dn_nt * NBc)) ||
      (rc = dalloc(c, &c->d_dflags, (size_t)2 * c->dn_nt * c->dn_nt + c->dn_nt + 1)) ||
      (rc = dupload(c, &c->d_kfcol, c->kf_col, st)))
    return rc;
  const int cap = chol_plan_tasks(c->dn_nt, nullptr, 0);
  std::vector<char> buf((size_t)std::max(cap, 1) * chol_task_bytes());
  c->n_dtasks = chol_plan_tasks(c->dn_nt, buf.data(), cap);
  if ((rc = dalloc(c, (char**)&c->d_dtasks, buf.size()))) return rc;
  VBA_CUDA(cudaMemcpyAsync(c->d_dtasks, buf.data(), buf.size(), cudaMemcpyHostToDevice, st));
  c->dn_ready = true;
  return VBA_OK;
}

static int stage_step_dense(Ctx* c, double lam, cudaStream_t st) {
  if (c->world > 1) { set_err("use_schur=False is single-GPU only"); return VBA_E_UNSUPPORTED; }
  int rc = ensure_dense(c, st);
  if (rc) return rc;
  DevState& s = CUR(c);
  DevState& n = NXT(c);
  mark(c, 2, st);
  VBA_CUDA(cudaMemsetAsync(c->d_res, 0, sizeof(Result), st));
  VBA_CUDA(cudaMemsetAsync(c->d_D, 0, sizeof(double) * (size_t)c->dn_npad * c->dn_npad, st));
  VBA_CUDA(cudaMemsetAsync(c->d_drhs, 0, sizeof(double) * c->dn_npad, st));
  launch_pad_identity(c->d_D, c->dn_npad, c->dn_N, c->dn_npad, c->d_drhs, st);
  mark(c, 3, st);
  if (c->nfree > 0) {   // damped H_ff (no fill-in) and -g_f
    launch_assemble(c->red.bptr, c->red.bnff, c->red.cs, c->red.nbr, c->red.roff, c->red.rdim, c->d_arena, lam,
                    c->O.ridge, 1, c->d_D, c->dn_npad, 2, st);
    launch_assemble_vec(c->red.sptr, c->red.vs, c->red.nseg, c->red.soff, c->d_arena, -1.0, c->d_drhs, st, 1);
  }
  HpdOut o{c->d_D, c->dn_npad, c->nfree, c->sdof, c->d_kfcol, c->d_Hdd, c->d_gd, c->d_drhs, lam, c->O.ridge};
  launch_export_hpd(c->P.pixel_mode, c->d_seb, c->d_see, c->d_doff, c->d_roff_real, c->d_npix, c->maxpix, c->d_ej,
                    c->K, s, c->extr, c->pix, c->P.wts, c->d_eoff, c->P.grid_w, c->grid, c->intr, o, st);
  if (!c->use_small || chol_small_solve(c->d_D, c->dn_npad, c->dn_N, c->d_drhs, c->d_dx2, &c->d_res->status, st))
    chol_dag_launch(c->d_D, c->dn_npad, c->dn_nt, c->d_drhs, c->d_dx2, c->d_dLinv, c->d_dpart, c->d_dflags,
                    c->d_dtasks, c->n_dtasks, &c->d_res->status, st);
  mark(c, 4, st);
  launch_scatter_dx(c->d_dx2, c->d_fmap, c->npv, c->d_dx, st);
  if (c->n_disp) {   // padding slots keep their values; real pixels are rewritten below
    VBA_CUDA(cudaMemcpyAsync(n.disp, s.disp, sizeof(float) * c->n_disp, cudaMemcpyDeviceToDevice, st));
    VBA_CUDA(cudaMemcpyAsync(n.disp64, s.disp64, sizeof(double) * c->n_disp, cudaMemcpyDeviceToDevice, st));
  }
  launch_dense_dxd(c->d_dx2, c->nfree, c->d_doff, c->d_roff_real, c->d_npix, c->maxpix, c->K, s, n, c->d_dxd,
                   &c->d_res->step_bits, st);
  launch_retract(s, n, c->d_dx, c->d_frozen, c->K, c->sdof, c->ngrav, c->n_state, &c->d_res->step_bits, c->npv, st);
  c->have_step = true;
  c->last_lam = lam;
  return VBA_OK;
}

static int stage_step_any(Ctx* c, double lam, int use_schur, cudaStream_t st) {
  // the reference takes the Schur path only when there are disparities (solver.py:281)
  if (use_schur || c->n_disp == 0) return stage_step(c, lam, st);
  return stage_step_dense(c, lam, st);
}

// The tensor-core solve is accepted when its fp32 factor had positive pivots and
// the last fp64 refinement pass moved x by <= kTcRefineTol max|x|.
static bool tc_failed(Ctx* c, int use_schur) {
  if (!c->tc_ran || c->nfree == 0 || !(use_schur || c->n_disp == 0)) return false;
  const Result& r = *c->h_res;
  ++c->tc_solves;
  c->tc_passes += (int64_t)r.tc[2];
  if (getenv("VBA_TC_REFINE_TRACE"))   // passes, previous pass's and last pass's relative corrections
    fprintf(stderr, "tc refine: passes %.0f rel_prev %.3e rel_last %.3e accepted %.0f\n", r.tc[2], r.tc[3],
            r.tc[1] > 0 ? r.tc[0] / r.tc[1] : 0.0, r.tc[4]);
  return r.tc_bad != 0 || r.tc[4] != 1.0;
}

static int run_trial(Ctx* c, double lam, int use_schur, vba_trial_result* out, cudaStream_t st) {
  int rc = stage_step_any(c, lam, use_schur, st);
  if (rc) return rc;
  mark(c, 5, st);
  rc = stage_energy(c, NXT(c), st);
  if (rc) return rc;
  mark(c, 6, st);
  if (c->world > 1) {   // each rank saw only its own pixels' dx_d: max of the step norm
    if (!c->coll) { set_err("sharded solve without a collective hook (vba_set_collective)"); return VBA_E_INVALID; }
    if (c->coll(c->coll_user, (double*)&c->d_res->step_bits, 1, 1, st)) { set_err("allreduce(step) failed"); return VBA_E_CUDA; }
  }
  VBA_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(Result), cudaMemcpyDeviceToHost, st));
  VBA_CUDA(cudaStreamSynchronize(st));
  if (tc_failed(c, use_schur)) {   // tensor-core solve failed its own checks: redo the step in fp64
    ++c->tc_fallbacks;
    c->force_fp64 = true;
    rc = run_trial(c, lam, use_schur, out, st);
    c->force_fp64 = false;
    return rc;
  }
  prof_collect(c, c->lin_pending);
  c->lin_pending = false;
  if (c->d_trace && use_schur) {   // Cholesky DAG task timing summary (diagnostics)
    std::vector<unsigned long long> tr((size_t)4 * c->n_ctasks);
    std::vector<char> tb((size_t)c->n_ctasks * chol_task_bytes());
    std::vector<int> f4((size_t)4 * c->n_ctasks);
    cudaMemcpy(tr.data(), c->d_trace, tr.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(tb.data(), c->d_ctasks, tb.size(), cudaMemcpyDeviceToHost);
    chol_task_fields(tb.data(), c->n_ctasks, f4.data());
    unsigned long long t0 = ~0ull, t1 = 0;
    double busy[5] = {0, 0, 0, 0, 0}, wait[5] = {0, 0, 0, 0, 0};
    int cnt[5] = {0, 0, 0, 0, 0};
    for (int q = 0; q < c->n_ctasks; ++q) {
      t0 = std::min(t0, tr[4 * q]);
      t1 = std::max(t1, tr[4 * q + 2]);
      const int ty = f4[4 * q];
      busy[ty] += (double)(tr[4 * q + 2] - tr[4 * q + 1]) * 1e-3;
      wait[ty] += (double)(tr[4 * q + 1] - tr[4 * q]) * 1e-3;
      cnt[ty] += 1;
    }
    const char* nm[5] = {"POTRF", "TRSM", "GEMM", "BUPD", "BSOL"};
    fprintf(stderr, "[chol trace] nt=%d tasks=%d span %.1f us\n", c->nt, c->n_ctasks, (double)(t1 - t0) * 1e-3);
    {  // POTRF phase stamps: [0] start [1+2p] factor32 done [2+2p] panel done [9] end
      std::vector<unsigned long long> ph((size_t)16 * c->nt);
      cudaMemcpy(ph.data(), c->d_trace + 4 * (size_t)c->n_ctasks, ph.size() * 8, cudaMemcpyDeviceToHost);
      double f = 0, u = 0, inv = 0;
      for (int k = 0; k < c->nt; ++k) {
        const unsigned long long* q = &ph[16 * (size_t)k];
        unsigned long long prev = q[0];
        for (int p = 0; p < 4; ++p) {
          f += (double)(q[1 + 2 * p] - prev) * 1e-3;
          u += (double)(q[2 + 2 * p] - q[1 + 2 * p]) * 1e-3;
          prev = q[2 + 2 * p];
        }
        inv += (double)(q[9] - q[8]) * 1e-3;
      }
      fprintf(stderr, "  POTRF phases (avg us): factor32 x4 %.2f | trsm+syrk %.2f | inverse+y %.2f\n", f / c->nt,
              u / c->nt, inv / c->nt);
    }
    for (int ty = 0; ty < 5; ++ty)
      if (cnt[ty])
        fprintf(stderr, "  %-5s n=%6d  avg busy %8.2f us  avg wait %8.2f us\n", nm[ty], cnt[ty], busy[ty] / cnt[ty],
                wait[ty] / cnt[ty]);
  }
  out->status = c->h_res->status ? VBA_E_NOT_SPD : VBA_OK;
  out->new_cost = c->h_res->energy[0];
  double si;
  unsigned long long b = c->h_res->step_bits;
  std::memcpy(&si, &b, sizeof(double));
  out->step_inf = si;
  return VBA_OK;
}

}  // namespace vba

using namespace vba;

extern "C" {

const char* vba_last_error(void) { return g_err.c_str(); }
int vba_version(void) { return 1; }

int vba_create(void** out, const vba_problem* prob, const vba_options* opts, void* stream) {
  *out = nullptr;
  if (!prob || !opts) { set_err("null problem/options"); return VBA_E_INVALID; }
  cudaStream_t st = (cudaStream_t)stream;
  Ctx* c = new Ctx();
  c->P = *prob;
  c->O = *opts;
  c->K = prob->n_kf;
  c->E = prob->n_edges;
  c->F = prob->n_imu;
  c->sdof = opts->optimize_velocity_bias ? 15 : 6;
  c->ngrav = opts->optimize_gravity ? 2 : 0;
  c->n_state = c->K * c->sdof;
  c->npv = c->n_state + c->ngrav;
  c->n_disp = prob->n_disp_pad;
  c->n_rows = prob->n_rows_pad;
  c->grid[0] = prob->grid_ox; c->grid[1] = prob->grid_oy; c->grid[2] = prob->grid_sx; c->grid[3] = prob->grid_sy;
  c->intr[0] = prob->fx; c->intr[1] = prob->fy; c->intr[2] = prob->cx; c->intr[3] = prob->cy;
  auto fail = [&](int rc) { vba_destroy(c); return rc; };
  if (c->K <= 0 || c->E < 0 || c->F < 0) { set_err("invalid sizes"); return fail(VBA_E_INVALID); }
  if (prob->pixel_mode < 0 || prob->pixel_mode > 2 || (prob->pixel_mode == VBA_PIX_GRID && prob->grid_w <= 0) ||
      (prob->pixel_mode != VBA_PIX_GRID && !prob->pix)) {
    set_err("invalid pixel mode");
    return fail(VBA_E_INVALID);
  }
  if (!(opts->ridge > 0) || !(opts->damping > 0)) { set_err("invalid options"); return fail(VBA_E_INVALID); }
  make_extr(*prob, c->extr);
  c->own_k1 = c->K;
  if (prob->shard_world > 1) {
    c->world = prob->shard_world;
    c->rank = prob->shard_rank;
    if (c->rank < 0 || c->rank >= c->world || !prob->h_shard_kbounds) {
      set_err("invalid shard spec");
      return fail(VBA_E_INVALID);
    }
    c->kb.assign(prob->h_shard_kbounds, prob->h_shard_kbounds + c->world + 1);
    for (int r = 0; r < c->world; ++r)
      if (c->kb[r] > c->kb[r + 1]) { set_err("shard bounds must be nondecreasing"); return fail(VBA_E_INVALID); }
    if (c->kb[0] != 0 || c->kb[c->world] != c->K) { set_err("shard bounds must cover [0, K)"); return fail(VBA_E_INVALID); }
    for (int f = 1; f < c->F; ++f)
      if (prob->h_imu_i[f] < prob->h_imu_i[f - 1]) {
        set_err("a sharded solve needs IMU factors sorted by their first keyframe");
        return fail(VBA_E_UNSUPPORTED);
      }
    c->own_k0 = c->kb[c->rank];
    c->own_k1 = c->kb[c->rank + 1];
  } else {
    c->kb = {0, c->K};
  }
  int rc = build_plans(c, st);
  if (rc) return fail(rc);
  // topology to device
  std::vector<int32_t> ei(prob->h_edge_i, prob->h_edge_i + c->E), ej(prob->h_edge_j, prob->h_edge_j + c->E);
  std::vector<int32_t> fi(prob->h_imu_i, prob->h_imu_i + c->F), fj(prob->h_imu_j, prob->h_imu_j + c->F);
  std::vector<int32_t> fr(prob->h_frozen, prob->h_frozen + c->K);
  std::vector<int64_t> eoff(prob->h_eoff, prob->h_eoff + c->E), doff(prob->h_doff, prob->h_doff + c->K + 1);
  if ((rc = dupload(c, &c->d_ei, ei, st)) || (rc = dupload(c, &c->d_ej, ej, st)) ||
      (rc = dupload(c, &c->d_fi, fi, st)) || (rc = dupload(c, &c->d_fj, fj, st)) ||
      (rc = dupload(c, &c->d_frozen, fr, st)) || (rc = dupload(c, &c->d_eoff, eoff, st)) ||
      (rc = dupload(c, &c->d_doff, doff, st)) || (rc = dupload(c, &c->d_tiles, c->tiles, st)) ||
      (rc = dupload(c, &c->d_soff, c->soff, st)) || (rc = dupload(c, &c->d_sids, c->sids, st)) ||
      (rc = dupload(c, &c->d_ioff, c->ioff, st)) || (rc = dupload(c, &c->d_sitems, c->sitems, st)) ||
      (rc = dupload(c, &c->d_chunks, c->chunks, st)) ||
      (rc = dupload(c, &c->d_t0s, c->t0s, st)) || (rc = dupload(c, &c->d_t1s, c->t1s, st)) ||
      (rc = dupload(c, &c->d_seb, c->seb, st)) || (rc = dupload(c, &c->d_see, c->see, st)) ||
      (rc = dupload(c, &c->d_gtiles, c->gtiles, st)) || (rc = dupload(c, &c->d_gsrc, c->gsrc, st)) ||
      (rc = dupload(c, &c->d_gorder, c->gorder, st)) || (rc = dupload(c, &c->d_gsrc_lpt, c->gsrc_lpt, st)) ||
      (rc = dupload(c, &c->d_g0, c->g0, st)) || (rc = dupload(c, &c->d_g1, c->g1, st)) ||
      (rc = dupload(c, &c->d_goff, c->goff, st)) || (rc = dupload(c, &c->d_foff, c->foff, st)) ||
      (rc = dupload(c, &c->d_fmap, c->fmap, st)) || (rc = dupload(c, &c->d_gorder_own, c->gorder_own, st)) ||
      (rc = dupload(c, &c->d_gsrc_own, c->gsrc_own, st)))
    return fail(rc);
  // state double buffers
  for (int b = 0; b < 2; ++b) {
    DevState& s = c->S[b];
    if ((rc = dalloc(c, &s.state, (size_t)16 * c->K)) || (rc = dalloc(c, &s.disp, (size_t)c->n_disp)) ||
        (rc = dalloc(c, &s.disp64, (size_t)c->n_disp)) ||
        (rc = dalloc(c, &s.grav, 5)) || (rc = dalloc(c, &s.geo32, (size_t)c->E)) ||
        (rc = dalloc(c, &s.geo64, (size_t)kGeo64 * c->E)))
      return fail(rc);
  }
  if (cudaMemcpyAsync(c->S[0].state, prob->state, sizeof(double) * 16 * c->K, cudaMemcpyDeviceToDevice, st) ||
      cudaMemcpyAsync(c->S[0].grav, prob->grav, sizeof(double) * 5, cudaMemcpyDeviceToDevice, st) ||
      load_disparities(c, c->S[0], st)) {
    set_err("state upload failed");
    return fail(VBA_E_CUDA);
  }
  // workspace
  if ((rc = dalloc(c, &c->d_part, (size_t)c->n_part * kPartStride / 2)) ||
      (rc = dalloc(c, &c->d_tile_e, c->chunks.size() * kPartWarps)) || (rc = dalloc(c, &c->d_arena, (size_t)c->arena_len)) ||
      (rc = dalloc(c, &c->d_gram_part, (size_t)c->gram_part_len)) ||
      (rc = dalloc(c, &c->d_gram, (size_t)1)) || (rc = dalloc(c, &c->d_Hdd, (size_t)c->n_disp)) ||
      (rc = dalloc(c, &c->d_gd, (size_t)c->n_disp)) || (rc = dalloc(c, &c->d_ustep, (size_t)8 * c->E)) ||
      (rc = dalloc(c, &c->d_dxd, (size_t)c->n_disp)) || (rc = dalloc(c, &c->d_L, (size_t)kImuL * c->F)) ||
      (rc = dalloc(c, &c->d_imu_status, 1)) || (rc = dalloc(c, &c->d_H, (size_t)c->npad * c->npad)) ||
      (rc = dalloc(c, &c->d_rhs, (size_t)c->npad)) || (rc = dalloc(c, &c->d_x, (size_t)c->npad)) ||
      (rc = dalloc(c, &c->d_Ld, (size_t)std::max(1, c->nt) * NBc * NBc)) ||
      (rc = dalloc(c, &c->d_cpart, (size_t)std::max(1, c->nt * c->nt) * NBc)) ||
      (rc = dalloc(c, &c->d_cflags, (size_t)2 * c->nt * c->nt + c->nt + 1)) ||
      (rc = dalloc(c, &c->d_dx, (size_t)c->npv)) || (rc = dalloc(c, &c->d_res, 1)))
    return fail(rc);
  if (cudaMallocHost((void**)&c->h_res, sizeof(Result)) != cudaSuccess) { set_err("pinned alloc failed"); return fail(VBA_E_CUDA); }
  c->pix = prob->pix;
  if (prob->pixel_mode == VBA_PIX_GRID) {   // ray table: columns, then rows up to the longest segment
    int64_t maxpad = 0;
    for (int n = 0; n < c->K; ++n) maxpad = std::max<int64_t>(maxpad, prob->h_doff[n + 1] - prob->h_doff[n]);
    const int rows = (int)((maxpad + prob->grid_w - 1) / prob->grid_w) + 1;
    if ((rc = dalloc(c, &c->d_raytab, (size_t)prob->grid_w + rows))) return fail(rc);
    launch_ray_table(c->d_raytab, prob->grid_w, rows, c->grid, c->intr, st);
    c->pix = c->d_raytab;
  }
  {
    // tensor-core reduced solve for large reduced systems (its fixed costs -- refinement
    // passes, extra launches -- lose to the fp64 DAG below ~32 tiles, n ~ 4000);
    // VBA_CHOL=tc / fp64 forces either
    const char* ch = getenv("VBA_CHOL");
    if (ch && std::strcmp(ch, "tc") == 0) c->use_tc = c->nt > 0;
    else if (ch && std::strcmp(ch, "fp64") == 0) c->use_tc = false;
    else c->use_tc = c->nt >= kTcMinTiles;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // the tensor-core solve's triangular sweeps keep one CTA per 128-row tile resident:
    // larger systems (n > 128 * SMs = 18944 on B200) are solved on the fp64 tile DAG
    if (c->nt > sms) c->use_tc = false;
    c->use_small = !c->use_tc && !(ch && std::strcmp(ch, "dag") == 0);
    const char* it = getenv("VBA_TC_ITERS");
    if (it) c->tc_iters = std::max(1, atoi(it));
  }
  if (c->use_tc) {
    const size_t wb = chol_tc_ws_bytes(c->npad);
    if ((rc = dalloc(c, (char**)&c->d_tcws, wb))) return fail(rc);
    cudaMemsetAsync(c->d_tcws, 0, wb, st);
    const int cap = chol_plan_tasks_tc(c->nt, nullptr, 0);
    std::vector<char> buf((size_t)std::max(cap, 1) * chol_task_bytes());
    c->n_tctasks = chol_plan_tasks_tc(c->nt, buf.data(), cap);
    if ((rc = dalloc(c, (char**)&c->d_tctasks, buf.size()))) return fail(rc);
    if (cudaMemcpyAsync(c->d_tctasks, buf.data(), buf.size(), cudaMemcpyHostToDevice, st) != cudaSuccess) {
      set_err("task upload failed");
      return fail(VBA_E_CUDA);
    }
  }
  {  // Cholesky task DAG (dense, lookahead 1)
    const int cap = chol_plan_tasks(c->nt, nullptr, 0);
    std::vector<char> buf((size_t)std::max(cap, 1) * chol_task_bytes());
    c->n_ctasks = chol_plan_tasks(c->nt, buf.data(), cap);
    if ((rc = dalloc(c, (char**)&c->d_ctasks, buf.size()))) return fail(rc);
    if (cudaMemcpyAsync(c->d_ctasks, buf.data(), buf.size(), cudaMemcpyHostToDevice, st) != cudaSuccess) {
      set_err("task upload failed");
      return fail(VBA_E_CUDA);
    }
  }
  cudaMemsetAsync(c->d_arena, 0, sizeof(double) * std::max<int64_t>(1, c->arena_len), st);
  cudaMemsetAsync(c->d_Hdd, 0, sizeof(float) * std::max<int64_t>(1, c->n_disp), st);   // edge-less tiles stay 0
  cudaMemsetAsync(c->d_tile_e, 0, sizeof(double) * std::max<size_t>(1, c->chunks.size() * kPartWarps), st);
  cudaMemsetAsync(c->d_gd, 0, sizeof(float) * std::max<int64_t>(1, c->n_disp), st);
  cudaMemsetAsync(c->d_x, 0, sizeof(double) * std::max(1, c->npad), st);
  cudaMemsetAsync(c->d_rhs, 0, sizeof(double) * std::max(1, c->npad), st);
  cudaMemsetAsync(c->d_H, 0, sizeof(double) * std::max<size_t>(1, (size_t)c->npad * c->npad), st);
  launch_pad_identity(c->d_H, c->npad, c->nfree, c->npad, c->d_rhs, st);
  // IMU whitening factors (constant over the solve)
  cudaMemsetAsync(c->d_imu_status, 0, sizeof(int), st);
  launch_imu_prep(prob->imu, c->F, c->d_L, c->d_imu_status, st);
  int hs = 0;
  if (cudaMemcpyAsync(&hs, c->d_imu_status, sizeof(int), cudaMemcpyDeviceToHost, st) ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_err("create: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(VBA_E_CUDA);
  }
  if (hs) { set_err("non-PSD preintegration covariance"); return fail(VBA_E_COV); }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_err("create: %s", cudaGetErrorString(e)); return fail(VBA_E_CUDA); }
  *out = c;
  return VBA_OK;
}

int vba_destroy(void* ctx) {
  Ctx* c = (Ctx*)ctx;
  if (!c) return VBA_OK;
  for (void* p : c->allocs) cudaFree(p);
  if (c->h_res) cudaFreeHost(c->h_res);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->sev)
    if (e) cudaEventDestroy(e);
  delete c;
  return VBA_OK;
}

int vba_set_collective(void* ctx, vba_allreduce_fn fn, void* user) {
  Ctx* c = (Ctx*)ctx;
  c->coll = fn;
  c->coll_user = user;
  return VBA_OK;
}

int vba_set_gather(void* ctx, vba_allgather_fn fn, void* user) {
  Ctx* c = (Ctx*)ctx;
  c->gat = fn;
  c->gat_user = user;
  return VBA_OK;
}

int64_t vba_reduced_dim(void* ctx) { return ((Ctx*)ctx)->nfree; }
int64_t vba_launch_count(void* /*ctx*/) { return launch_total(); }

int vba_stats(void* ctx, int64_t* out4) {
  Ctx* c = (Ctx*)ctx;
  out4[0] = c->use_tc ? 1 : 0;
  out4[1] = c->tc_fallbacks;
  out4[2] = c->tc_solves;
  out4[3] = c->tc_passes;
  return VBA_OK;
}

int vba_gram_kind(void* ctx) { return ((Ctx*)ctx)->gram_tc ? 1 : 0; }

int vba_chol_plan(int32_t nt, int32_t* out5, int32_t cap) {
  if (nt < 0 || cap < 0 || (cap > 0 && !out5)) { set_err("vba_chol_plan: bad arguments"); return VBA_E_INVALID; }
  const int n = chol_plan_tasks_tc(nt, nullptr, 0);
  std::vector<char> tb((size_t)std::max(n, 1) * chol_task_bytes());
  chol_plan_tasks_tc(nt, tb.data(), n);
  std::vector<int> f((size_t)5 * std::max(n, 1));
  chol_task_fields5(tb.data(), n, f.data());
  for (int q = 0; q < n && q < cap; ++q)
    for (int u = 0; u < 5; ++u) out5[5 * q + u] = f[5 * (size_t)q + u];
  return n;
}

// Standalone SPD solve (np.linalg.solve of solver.py:287 on a damped reduced system).
int vba_spd_solve(const double* H, int64_t n, const double* b, double* x, int32_t mode, void* stream,
                  int32_t* info) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0 || n > (int64_t)1 << 16) { set_err("vba_spd_solve: n out of range"); return VBA_E_INVALID; }
  const int npad = (int)((n + NBc - 1) / NBc * NBc), nt = npad / NBc;
  const int cap = chol_plan_tasks(nt, nullptr, 0);
  std::vector<char> tb((size_t)cap * chol_task_bytes());
  const int ntasks = chol_plan_tasks(nt, tb.data(), cap);
  const int cap2 = chol_plan_tasks_tc(nt, nullptr, 0);
  std::vector<char> tb2((size_t)cap2 * chol_task_bytes());
  const int ntasks2 = chol_plan_tasks_tc(nt, tb2.data(), cap2);
  const size_t tcb = mode != 1 ? chol_tc_ws_bytes(npad) : 0;
  double *Hp = nullptr, *bp = nullptr, *xp = nullptr, *Ld = nullptr, *part = nullptr, *tc2 = nullptr;
  int *flags = nullptr, *stat = nullptr;
  void *tasks = nullptr, *tasks2 = nullptr, *ws = nullptr;
  auto cleanup = [&]() {
    cudaFree(Hp); cudaFree(bp); cudaFree(xp); cudaFree(Ld); cudaFree(part); cudaFree(tc2);
    cudaFree(flags); cudaFree(stat); cudaFree(tasks); cudaFree(tasks2); cudaFree(ws);
  };
  if (cudaMalloc(&Hp, sizeof(double) * (size_t)npad * npad) || cudaMalloc(&bp, sizeof(double) * npad) ||
      cudaMalloc(&xp, sizeof(double) * npad) || cudaMalloc(&Ld, sizeof(double) * (size_t)nt * NBc * NBc) ||
      cudaMalloc(&part, sizeof(double) * (size_t)nt * nt * NBc) || cudaMalloc(&tc2, sizeof(double) * 5) ||
      cudaMalloc(&flags, sizeof(int) * ((size_t)2 * nt * nt + nt + 1)) || cudaMalloc(&stat, sizeof(int) * 2) ||
      cudaMalloc(&tasks, tb.size()) || cudaMalloc(&tasks2, tb2.size()) || (tcb && cudaMalloc(&ws, tcb))) {
    cleanup();
    set_err("vba_spd_solve: allocation failed");
    return VBA_E_CUDA;
  }
  cudaMemsetAsync(Hp, 0, sizeof(double) * (size_t)npad * npad, st);
  cudaMemsetAsync(bp, 0, sizeof(double) * npad, st);
  cudaMemsetAsync(stat, 0, sizeof(int) * 2, st);
  cudaMemsetAsync(tc2, 0, sizeof(double) * 5, st);
  if (tcb) cudaMemsetAsync(ws, 0, tcb, st);
  cudaMemcpy2DAsync(Hp, sizeof(double) * npad, H, sizeof(double) * n, sizeof(double) * n, n,
                    cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(bp, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(tasks, tb.data(), tb.size(), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(tasks2, tb2.data(), tb2.size(), cudaMemcpyHostToDevice, st);
  launch_pad_identity(Hp, npad, (int)n, npad, bp, st);
  int hs[2] = {0, 0};
  double h2[5] = {0, 0, 0, 0, 0};
  int used_tc = 0;
  if (mode == 0 || mode == 2) {   // 2: tensor-core result without the fallback (diagnostics)
    const int iters = info && info[0] > 0 ? info[0] : 8;
    unsigned long long* tr = nullptr;
    if (getenv("VBA_CHOL_TRACE")) { cudaMalloc(&tr, sizeof(unsigned long long) * (4 * (size_t)ntasks2 + 16 * (size_t)nt)); cudaMemsetAsync(tr, 0, sizeof(unsigned long long) * (4 * (size_t)ntasks2 + 16 * (size_t)nt), st); }
    const int tcrc = chol_tc_solve(Hp, npad, (int)n, npad, bp, xp, ws, tasks2, ntasks2, iters, stat + 1, 1, st, tc2, tr);
    if (tr) { cudaStreamSynchronize(st); chol_trace_print("tc", tr, tasks2, ntasks2, nt); cudaFree(tr); }
    cudaMemcpyAsync(hs, stat, sizeof(hs), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h2, tc2, sizeof(h2), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) { cleanup(); set_err("vba_spd_solve: %s", cudaGetErrorString(cudaGetLastError())); return VBA_E_CUDA; }
    used_tc = tcrc == 0 && (mode == 2 || (hs[1] == 0 && h2[4] == 1.0)) ? 1 : 0;
  }
  if (!used_tc) {
    const char* ch = getenv("VBA_CHOL");
    if ((ch && std::strcmp(ch, "dag") == 0) || chol_small_solve(Hp, npad, (int)n, bp, xp, stat, st))
      chol_dag_launch(Hp, npad, nt, bp, xp, Ld, part, flags, tasks, ntasks, stat, st);
    cudaMemcpyAsync(hs, stat, sizeof(hs), cudaMemcpyDeviceToHost, st);
  }
  cudaMemcpyAsync(x, xp, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { cleanup(); set_err("vba_spd_solve: %s", cudaGetErrorString(cudaGetLastError())); return VBA_E_CUDA; }
  if (info) { info[0] = used_tc; info[1] = hs[1]; }
  cleanup();
  return hs[0] ? VBA_E_NOT_SPD : VBA_OK;
}

int64_t vba_preint_scratch_bytes(int64_t n_samples) {
  return n_samples < 0 ? -1 : (int64_t)(preint_scratch_bytes(n_samples) + 256);
}

int vba_preintegrate(const double* ts, const double* gyro, const double* accel, int64_t n_samples,
                     const int64_t* soff, int32_t n_pairs, const double* bias, const double* noise, void* scratch,
                     double* out, void* stream) {
  static_assert(VBA_PREINT_REC == kPreintRec, "preintegration record size");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_pairs < 0 || n_samples < 0) { set_err("vba_preintegrate: negative size"); return VBA_E_INVALID; }
  if (n_pairs == 0) return VBA_OK;
  if ((n_samples && (!ts || !gyro || !accel)) || !soff || !bias || !noise || !out || !scratch) {
    set_err("vba_preintegrate: null buffer");
    return VBA_E_INVALID;
  }
  int* stat = (int*)scratch;                            // status word, then the step records
  double* steps = (double*)((char*)scratch + 256);
  VBA_CUDA(cudaMemsetAsync(stat, 0, sizeof(int), st));
  launch_preintegrate(ts, gyro, accel, n_samples, soff, n_pairs, bias, noise, steps, out, stat, st);
  int hs = 0;
  VBA_CUDA(cudaMemcpyAsync(&hs, stat, sizeof(int), cudaMemcpyDeviceToHost, st));
  VBA_CUDA(cudaStreamSynchronize(st));
  if (hs & 1) { set_err("Need at least two IMU samples to preintegrate"); return VBA_E_INVALID; }
  if (hs & 2) { set_err("IMU timestamps must be strictly increasing"); return VBA_E_INVALID; }
  if (hs & 4) { set_err("vba_preintegrate: malformed soff (soff[n_pairs] != n_samples or out of range)"); return VBA_E_INVALID; }
  return VBA_OK;
}

int vba_preint_factor_records(const double* rec, const double* bias, int32_t n_pairs, double* imu, void* stream) {
  static_assert(VBA_IMU_REC == kImuRec, "IMU record size");
  if (n_pairs < 0 || (n_pairs > 0 && (!rec || !bias || !imu))) {
    set_err("vba_preint_factor_records: invalid arguments");
    return VBA_E_INVALID;
  }
  if (n_pairs == 0) return VBA_OK;
  launch_preint_pack(rec, bias, n_pairs, imu, (cudaStream_t)stream);
  VBA_CUDA(cudaGetLastError());
  return VBA_OK;
}

int vba_copy_segments(const vba_copy_seg* segs, int32_t n, void* stream) {
  if (n < 0 || (n > 0 && !segs)) {
    set_err("vba_copy_segments: invalid arguments");
    return VBA_E_INVALID;
  }
  if (n == 0) return VBA_OK;
  launch_copy_segments(segs, n, (cudaStream_t)stream);
  VBA_CUDA(cudaGetLastError());
  return VBA_OK;
}

int vba_energy(void* ctx, void* stream, double* tot, double* vis, double* ine) {
  Ctx* c = (Ctx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = stage_energy(c, CUR(c), st);
  if (rc) return rc;
  VBA_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(Result), cudaMemcpyDeviceToHost, st));
  VBA_CUDA(cudaStreamSynchronize(st));
  if (tot) *tot = c->h_res->energy[0];
  if (vis) *vis = c->h_res->energy[1];
  if (ine) *ine = c->h_res->energy[2];
  return VBA_OK;
}

int vba_linearize(void* ctx, void* stream) {
  Ctx* c = (Ctx*)ctx;
  int rc = stage_linearize(c, (cudaStream_t)stream);
  if (rc) return rc;
  VBA_CUDA(cudaGetLastError());
  return VBA_OK;
}

int vba_solve_step(void* ctx, void* stream, double lam, int32_t use_schur) {
  Ctx* c = (Ctx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = stage_step_any(c, lam, use_schur, st);
  if (rc) return rc;
  VBA_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(Result), cudaMemcpyDeviceToHost, st));
  VBA_CUDA(cudaStreamSynchronize(st));
  if (tc_failed(c, use_schur)) {
    ++c->tc_fallbacks;
    c->force_fp64 = true;
    rc = stage_step_any(c, lam, use_schur, st);
    c->force_fp64 = false;
    if (rc) return rc;
    VBA_CUDA(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(Result), cudaMemcpyDeviceToHost, st));
    VBA_CUDA(cudaStreamSynchronize(st));
  }
  return c->h_res->status ? VBA_E_NOT_SPD : VBA_OK;
}

int vba_apply_step(void* ctx, void* /*stream*/) {
  Ctx* c = (Ctx*)ctx;
  if (!c->have_step) { set_err("no step computed"); return VBA_E_INVALID; }
  c->cur ^= 1;   // the next buffers already hold the retracted state; the old ones are the snapshot
  return VBA_OK;
}

int vba_restore(void* ctx, void* /*stream*/) {
  Ctx* c = (Ctx*)ctx;
  c->cur ^= 1;
  return VBA_OK;
}

int vba_accept(void* ctx, void* /*stream*/) {
  ((Ctx*)ctx)->cur ^= 1;
  return VBA_OK;
}

int vba_trial(void* ctx, void* stream, double lam, int32_t use_schur, vba_trial_result* out) {
  Ctx* c = (Ctx*)ctx;
  return run_trial(c, lam, use_schur, out, (cudaStream_t)stream);
}

int vba_solve(void* ctx, void* stream, vba_report* rep, double* traj, int32_t cap) {
  Ctx* c = (Ctx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  const vba_options& o = c->O;
  std::memset(rep, 0, sizeof(*rep));
  double cost;
  int rc = vba_energy(ctx, stream, &cost, nullptr, nullptr);
  if (rc) return rc;
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
  if (o.max_iterations == 0) return finish(0, 0, 0, 0);
  double lam = o.damping;
  int term = 0, iters = 0, warns = 0, trials = 0;
  bool broke = false;
  for (int it = 0; it < o.max_iterations; ++it) {
    nvtxRangePushA("vba.linearize");
    rc = stage_linearize(c, st);
    nvtxRangePop();
    if (rc) return rc;
    bool accepted = false;
    while (true) {
      vba_trial_result r;
      nvtxRangePushA("vba.trial");
      rc = run_trial(c, lam, o.use_schur, &r, st);
      nvtxRangePop();
      if (rc) return rc;
      ++trials;
      if (r.status == VBA_E_NOT_SPD) {   // solver.py:373-379
        ++warns;
        lam *= o.damping_up;
        if (lam > o.max_damping) return finish(iters, 3, warns, trials);
        continue;
      }
      if (r.new_cost < cost) {             // solver.py:383-393
        cost = r.new_cost;
        tr.push_back(cost);
        lam = std::max(lam * o.damping_down, 1e-12);
        accepted = true;
        iters = it + 1;
        c->cur ^= 1;
        if (r.step_inf < o.step_tol) term = 1;
        break;
      }
      lam *= o.damping_up;                 // solver.py:394-398
      if (lam > o.max_damping) { term = 2; break; }
    }
    if (!accepted) { broke = true; break; }
    if (term == 1) { broke = true; break; }
    const double prev = tr[tr.size() - 2];
    if (prev > 0 && (prev - cost) / prev < o.rel_decrease_tol) { term = 1; broke = true; break; }
  }
  if (!broke) term = 0;
  VBA_CUDA(cudaGetLastError());
  return finish(iters, term, warns, trials);
}

int vba_download(void* ctx, void* stream) {
  Ctx* c = (Ctx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  DevState& s = CUR(c);
  VBA_CUDA(cudaMemcpyAsync(c->P.state, s.state, sizeof(double) * 16 * c->K, cudaMemcpyDeviceToDevice, st));
  if (c->n_disp && c->world > 1) {   // each rank updated only its own keyframes' disparities
    int rc = gather(c, s.disp64, c->g_disp, st, "disparities");
    if (rc) return rc;
    launch_narrow(s.disp64, s.disp, c->n_disp, st);
  }
  if (c->n_disp) {
    VBA_CUDA(cudaMemcpyAsync(c->P.disp, s.disp, sizeof(float) * c->n_disp, cudaMemcpyDeviceToDevice, st));
    if (c->P.disp64)
      VBA_CUDA(cudaMemcpyAsync(c->P.disp64, s.disp64, sizeof(double) * c->n_disp, cudaMemcpyDeviceToDevice, st));
  }
  VBA_CUDA(cudaMemcpyAsync(c->P.grav, s.grav, sizeof(double) * 5, cudaMemcpyDeviceToDevice, st));
  return VBA_OK;
}

int vba_export_normal_eq(void* ctx, void* stream, double* H_pp, double* g_p, double* H_pd, double* H_dd,
                         double* g_d) {
  Ctx* c = (Ctx*)ctx;
  if (c->world > 1) { set_err("vba_export_normal_eq: not available on a sharded context"); return VBA_E_UNSUPPORTED; }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = build_export_plan(c, st);
  if (rc) return rc;
  if ((rc = ensure_real_layout(c, st))) return rc;
  DevState& s = CUR(c);
  if (H_pp) {
    VBA_CUDA(cudaMemsetAsync(H_pp, 0, sizeof(double) * c->npv * c->npv, st));
    launch_assemble(c->exp.bptr, c->exp.bnff, c->exp.cs, c->exp.nbr, c->exp.roff, c->exp.rdim, c->d_arena, 0.0,
                    0.0, 0, H_pp, c->npv, 1, st);
  }
  if (g_p) launch_assemble_vec(c->exp.sptr, c->exp.vs, c->exp.nseg, c->exp.soff, c->d_arena, 1.0, g_p, st);
  if (H_dd) launch_unpad(c->d_Hdd, c->d_doff, c->d_roff_real, c->d_npix, c->maxpix, c->K, H_dd, st);
  if (g_d) launch_unpad(c->d_gd, c->d_doff, c->d_roff_real, c->d_npix, c->maxpix, c->K, g_d, st);
  if (H_pd) {
    VBA_CUDA(cudaMemsetAsync(H_pd, 0, sizeof(double) * c->npv * std::max<int64_t>(1, c->n_real), st));
    HpdOut o{H_pd, c->n_real, 0, c->sdof, nullptr, nullptr, nullptr, nullptr, 0.0, 0.0};
    launch_export_hpd(c->P.pixel_mode, c->d_seb, c->d_see, c->d_doff, c->d_roff_real, c->d_npix, c->maxpix, c->d_ej,
                      c->K, s, c->extr, c->pix, c->P.wts, c->d_eoff, c->P.grid_w, c->grid, c->intr, o, st);
  }
  VBA_CUDA(cudaStreamSynchronize(st));
  return VBA_OK;
}

int vba_export_reduced(void* ctx, void* stream, double lam, double* H_red, double* g_red) {
  Ctx* c = (Ctx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = stage_reduce(c, lam, st);
  if (rc) return rc;
  launch_export_sym(c->d_H, c->npad, c->nfree, H_red, c->d_rhs, -1.0, g_red, st);
  VBA_CUDA(cudaStreamSynchronize(st));
  return VBA_OK;
}

int vba_export_step(void* ctx, void* stream, double* dx_full, double* dx_d) {
  Ctx* c = (Ctx*)ctx;
  if (c->world > 1 && dx_d) { set_err("vba_export_step: dx_d is rank-local on a sharded context"); return VBA_E_UNSUPPORTED; }
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->have_step) { set_err("no step computed"); return VBA_E_INVALID; }
  int rc = ensure_real_layout(c, st);
  if (rc) return rc;
  if (dx_full) VBA_CUDA(cudaMemcpyAsync(dx_full, c->d_dx, sizeof(double) * c->npv, cudaMemcpyDeviceToDevice, st));
  if (dx_d) launch_unpad(c->d_dxd, c->d_doff, c->d_roff_real, c->d_npix, c->maxpix, c->K, dx_d, st);
  VBA_CUDA(cudaStreamSynchronize(st));
  return VBA_OK;
}

int vba_set_profiling(void* ctx, int32_t on) {
  Ctx* c = (Ctx*)ctx;
  if (on && !c->ev[0]) {
    for (auto& e : c->ev) VBA_CUDA(cudaEventCreate(&e));
    for (auto& e : c->sev) VBA_CUDA(cudaEventCreate(&e));
  }
  c->prof = on != 0;
  for (double& v : c->stage_ms) v = 0.0;
  c->k1_launches = 0;
  c->solve_ms[0] = c->solve_ms[1] = 0.0;
  c->solve_samples = 0;
  c->sev_pending = false;
  return VBA_OK;
}

int vba_solve_times(void* ctx, double* out4) {
  Ctx* c = (Ctx*)ctx;
  out4[0] = c->solve_ms[0];
  out4[1] = c->solve_ms[1];
  out4[2] = (double)c->solve_samples;
  out4[3] = (double)c->nfree;
  return VBA_OK;
}

int vba_stage_times(void* ctx, double* out7) {
  Ctx* c = (Ctx*)ctx;
  for (int i = 0; i < 6; ++i) out7[i] = c->stage_ms[i];
  out7[6] = (double)c->k1_launches;
  return VBA_OK;
}

int vba_bind_inputs(void* ctx, void* stream, const float* tgt, const float* wts, int32_t refresh_imu) {
  Ctx* c = (Ctx*)ctx;
  if (!c || !tgt || !wts) { set_err("vba_bind_inputs: null argument"); return VBA_E_INVALID; }
  cudaStream_t st = (cudaStream_t)stream;
  c->P.tgt = tgt;
  c->P.wts = wts;
  if (refresh_imu && c->F > 0) {
    cudaMemsetAsync(c->d_imu_status, 0, sizeof(int), st);
    launch_imu_prep(c->P.imu, c->F, c->d_L, c->d_imu_status, st);
    int hs = 0;
    VBA_CUDA(cudaMemcpyAsync(&hs, c->d_imu_status, sizeof(int), cudaMemcpyDeviceToHost, st));
    VBA_CUDA(cudaStreamSynchronize(st));
    if (hs) { set_err("non-PSD preintegration covariance"); return VBA_E_COV; }
  }
  return VBA_OK;
}

int vba_load_state(void* ctx, void* stream) {
  Ctx* c = (Ctx*)ctx;
  cudaStream_t st = (cudaStream_t)stream;
  DevState& s = CUR(c);
  VBA_CUDA(cudaMemcpyAsync(s.state, c->P.state, sizeof(double) * 16 * c->K, cudaMemcpyDeviceToDevice, st));
  if (load_disparities(c, s, st)) { set_err("load_state: %s", cudaGetErrorString(cudaGetLastError())); return VBA_E_CUDA; }
  VBA_CUDA(cudaMemcpyAsync(s.grav, c->P.grav, sizeof(double) * 5, cudaMemcpyDeviceToDevice, st));
  c->have_step = false;
  return VBA_OK;
}

}  // extern "C"
