// vba_vision.cu — per-pixel vision kernels of the dense VI-BA (sm_100a).
//
// Restates the vision factor of residuals.py:172-263 and the vision part of
// solver.py:173-220 / 276-290 (paths relative to /root/reference/pkg/src/vislam/)
// in the factorised form documented in DESIGN.md §4.1:
//
//   X_h = M ray + d t            (= d * X_j, camera-j point scaled by the disparity)
//   J_i = K G_i,  J_j = -K G_j,  J_d = -P t / d
//   K   = [P [X_j]x | -P]  (2x6),  rows K0 = fx k0', K1 = fy k1'
//
// so each edge-pixel accumulates ONE 6x6 symmetric K-space Gram, a 6-vector
// gradient and two per-pixel scalars; the 6x6 -> pose-space transforms happen
// once per edge in fp64 (k_edge_finalize).  Per-pixel math is fp32, sums over
// <= 256 edge-pixels are fp32 (8 sequential + 5-level tree), everything
// beyond is fp64 with a fixed reduction order (bitwise deterministic).
#include <cuda_runtime.h>

#include "vba_internal.cuh"
#include "vba_tc.cuh"

namespace vba {

static int64_t g_launches = 0;
void launch_count() { ++g_launches; }
int64_t launch_total() { return g_launches; }

constexpr int kPixBlock = 128;   // threads of the per-pixel kernels
constexpr int kTP = VBA_TP;      // pixel pairs per thread
constexpr int kTile = 2 * kTP * kPixBlock;
static_assert(kTile == kTilePx, "tile size shared with the host planner");
constexpr int kGramPC = 32;      // pixels per Gram staging chunk
constexpr int kGramStride = 12;  // floats per (pixel, edge) in the Gram stage: u[6] v[6]

struct GridP { double ox, oy, sx, sy; };

// Gram stage pixel stride (floats): a multiple of 4 with an odd quad count, so
// quarter-warp float4 accesses of consecutive pixels hit distinct bank groups.
__host__ __device__ __forceinline__ int gram_px_stride(int kmax) {
  const int s = kGramStride * kmax;
  return ((s / 4) & 1) ? s : s + 4;
}

// dynamic shared memory of the DMMA Gram kernel: U and V, (6 kmax + 1 -> 8) columns x (PC + 4) pixels, fp64
size_t gram_smem_bytes(int kmax, int /*nsplit*/, int /*npairs*/, int /*k*/) {
  return (size_t)2 * ((6 * kmax + 1 + 7) / 8 * 8) * (kGramPC + 4) * sizeof(double);   // W, double-buffered
}
struct IntrP { double fx, fy, cx, cy; };

// ray (fp64 -> fp32) of pixel n of a keyframe segment
template <int MODE>
__device__ __forceinline__ void load_rays(const float* __restrict__ pix, int64_t kbase, int n, int grid_w,
                                          const GridP& gp, const IntrP& in, float& rx0, float& ry0,
                                          float& rx1, float& ry1) {
  double u0, v0, u1, v1;
  if (MODE == VBA_PIX_GRID) {
    // `pix` is the ray table of the grid (k_ray_table: the same fp64 expression as
    // below, evaluated once per column / row): [grid_w column rays | row rays]
    const int c0 = n % grid_w, r0 = n / grid_w;
    const int c1 = (n + 1) % grid_w, r1 = (n + 1) / grid_w;
    rx0 = __ldg(pix + c0); ry0 = __ldg(pix + grid_w + r0);
    rx1 = __ldg(pix + c1); ry1 = __ldg(pix + grid_w + r1);
    return;
  } else {
    const float4 p = __ldg(reinterpret_cast<const float4*>(pix + 2 * (kbase + n)));
    u0 = p.x; v0 = p.y; u1 = p.z; v1 = p.w;
  }
  rx0 = (float)((u0 - in.cx) / in.fx); ry0 = (float)((v0 - in.cy) / in.fy);
  rx1 = (float)((u1 - in.cx) / in.fx); ry1 = (float)((v1 - in.cy) / in.fy);
}

// Ray table of a regular pixel grid: column c -> (float)((ox + sx c - cx) / fx),
// row r -> (float)((oy + sy r - cy) / fy), in fp64 then rounded (the per-pixel
// kernels read it instead of recomputing the fp64 division per pixel).
__global__ void k_ray_table(float* __restrict__ tab, int W, int rows, GridP gp, IntrP in) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W) {
    const double u = gp.ox + gp.sx * i;
    tab[i] = (float)((u - in.cx) / in.fx);
  } else if (i < W + rows) {
    const double v = gp.oy + gp.sy * (i - W);
    tab[i] = (float)((v - in.cy) / in.fy);
  }
}
void launch_ray_table(float* tab, int W, int rows, const double* grid, const double* intr, cudaStream_t st) {
  GridP gp{grid[0], grid[1], grid[2], grid[3]};
  IntrP in{intr[0], intr[1], intr[2], intr[3]};
  k_ray_table<<<(W + rows + 255) / 256, 256, 0, st>>>(tab, W, rows, gp, in);
  launch_count();
}

// 1/x on the MUFU (<= 1 ulp); every per-pixel kernel projects with it so K1,
// the Gram and the back-substitution see bitwise identical geometry
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// one Newton step on top: r (2 - x r), ~correctly rounded; the packed pixel-pair
// kernels apply the same two FMAs with FFMA2 (bitwise equal)
__device__ __forceinline__ float rcp_nr(float x) {
  const float r = rcp_approx(x);
  return fmaf(r, fmaf(-x, r, 1.0f), r);
}

struct PxGeom {  // per edge-pixel projection at the current estimate
  float x, y, dx, dy, iz, izh;
  bool valid;
};

// Displacement form of the reprojection.  With X_h = d X_j = ray + D,
// D = (M - I) ray + d t (ray.z = 1):
//   x = (rx + Dx) / (1 + Dz),   x - rx = (Dx - rx Dz) / (1 + Dz)
// so the residual  r = u* - (cx + fx x) = flow - fx (x - rx)  only involves
// the displacement, whose fp32 rounding error scales with the flow instead of
// the absolute pixel coordinate (flow = u* - u is stored per row).
__device__ __forceinline__ PxGeom project(const EdgeGeo32& g, float rx, float ry, float d) {
  const float Dx = fmaf(d, g.t[0], fmaf(g.M[0], rx, fmaf(g.M[1], ry, g.M[2])));
  const float Dy = fmaf(d, g.t[1], fmaf(g.M[3], rx, fmaf(g.M[4], ry, g.M[5])));
  const float Dz = fmaf(d, g.t[2], fmaf(g.M[6], rx, fmaf(g.M[7], ry, g.M[8])));
  const float Xz = 1.0f + Dz;
  PxGeom o;
  o.valid = Xz > 1e-6f * d;                // z_j = Xz / d > 1e-6  (residuals.py:206-209)
  o.izh = o.valid ? rcp_nr(Xz) : 0.0f;      // invalid pixels: finite zeros, weight 0
  o.dx = fmaf(-rx, Dz, Dx) * o.izh;
  o.dy = fmaf(-ry, Dz, Dy) * o.izh;
  o.x = rx + o.dx;
  o.y = ry + o.dy;
  o.iz = d * o.izh;
  return o;
}

static_assert(sizeof(EdgeGeo32) == 64, "EdgeGeo32 records are 4 float4");
template <bool SMEM = false>
__device__ __forceinline__ EdgeGeo32 load_geo(const EdgeGeo32* __restrict__ geo, int e) {
  const float4* p = reinterpret_cast<const float4*>(geo + e);
  const float4 a = SMEM ? p[0] : __ldg(p), b = SMEM ? p[1] : __ldg(p + 1), c = SMEM ? p[2] : __ldg(p + 2);
  EdgeGeo32 g;
  g.M[0] = a.x; g.M[1] = a.y; g.M[2] = a.z; g.M[3] = a.w;
  g.M[4] = b.x; g.M[5] = b.y; g.M[6] = b.z; g.M[7] = b.w;
  g.M[8] = c.x; g.t[0] = c.y; g.t[1] = c.z; g.t[2] = c.w;
  return g;
}

// ---------------------------------------------------------------------------
// per-edge geometry (fp64 -> fp32 constants), one thread per edge
// ---------------------------------------------------------------------------
__global__ void k_edge_prep(const double* __restrict__ state, const int32_t* __restrict__ ei,
                            const int32_t* __restrict__ ej, int E, Extr x, EdgeGeo32* __restrict__ g32,
                            double* __restrict__ g64) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double* si = state + 16 * ei[e];
  const double* sj = state + 16 * ej[e];
  double Ri[9], Rj[9], A[9], ARi[9], M[9];
  qmat(si, Ri);
  qmat(sj, Rj);
  mat3_mulT(x.RbcT, Rj, A);            // A = R_bc^T R_j^T            (residuals.py:202)
  mat3_mul(A, Ri, ARi);
  mat3_mul(ARi, x.Rbc, M);             // camera i -> camera j rotation
  double dp[3] = {si[4] - sj[4], si[5] - sj[5], si[6] - sj[6]};
  double t1[3], t2[3], t3[3];
  mat3_vec(ARi, x.pbc, t1);
  mat3_vec(A, dp, t2);
  mat3_vec(x.RbcT, x.pbc, t3);
  EdgeGeo32 o;
#pragma unroll
  for (int k = 0; k < 9; ++k) o.M[k] = (float)(M[k] - ((k % 4) == 0 ? 1.0 : 0.0));   // M - I, exact small part
#pragma unroll
  for (int k = 0; k < 3; ++k) o.t[k] = (float)(t1[k] + t2[k] - t3[k]);
  o.pad[0] = o.pad[1] = o.pad[2] = o.pad[3] = 0.f;
  g32[e] = o;
  double* q = g64 + (int64_t)kGeo64 * e;
#pragma unroll
  for (int k = 0; k < 9; ++k) { q[k] = ARi[k]; q[9 + k] = A[k]; }
#pragma unroll
  for (int k = 0; k < 3; ++k) q[18 + k] = -t2[k] + t3[k];   // c1 = A(p_j - p_i) + R_bc^T p_bc
}

void launch_edge_prep(const DevState& s, const int32_t* ei, const int32_t* ej, int E, const Extr& x,
                      cudaStream_t st) {
  if (E <= 0) return;
  k_edge_prep<<<(E + 127) / 128, 128, 0, st>>>(s.state, ei, ej, E, x, s.geo32, s.geo64);
  launch_count();
}

// ---------------------------------------------------------------------------
// K1 (linearisation) and K2 (energy): streamed per-pixel kernels.
//
// Work item = (source tile, out-edge): 1024 pixels of one source keyframe
// against one edge.  A persistent grid (SMs x resident CTAs) pulls source
// tiles from an LPT-ordered list (most edge-pixels first) through a global
// counter; inside a CTA, thread 0 streams each item's flow and weight rows
// (2 x 8 KB, contiguous per edge) into a kStages-deep shared-memory ring with
// cp.async.bulk + mbarrier complete_tx, running ahead of the arithmetic across
// edge and tile boundaries, so HBM reads never wait on compute.  Per-pixel
// math is fp32 on pixel pairs with packed FFMA2 (sm_100a), the same operation
// order as project() (bitwise equal to the scalar kernels).
//
// K1 writes per (tile, edge) a 32-double partial: 21 upper-triangular entries
// of S = sum w K^T K and 6 of s = sum w K^T r (slots 27..31 zero), and per
// pixel H_dd, g_d (sum over out-edges).  K2 writes one fp64 energy per tile.
// ---------------------------------------------------------------------------
constexpr int kStages = 3;
constexpr int kPairs = kTile / 2;   // float4 (= 2 pixels) per row of a stage
static_assert(kPixBlock / 32 == kPartWarps, "K1 partial records hold one vector per warp");
constexpr int kSchedCap = 24;       // tile records of one CTA staged in shared memory
constexpr int kItemCap = 160;       // stream items of one CTA staged in shared memory
constexpr int kRedS = 36;           // row stride (floats) of the warp transpose: 4c mod 32 distinct per quarter-warp

struct StreamSmem {
  float4 flow[kStages][kPairs];
  float4 wts[kStages][kPairs];
  EdgeGeo32 geo[kStages];
  float xr[kPixBlock / 32][28 * kRedS];   // per-warp transpose of the 27 per-lane sums
  StreamItem it[kItemCap];
  PixTile tl[kSchedCap];
  int tid[kSchedCap];
  unsigned long long full[kStages];
  unsigned int rel[kStages];              // warp releases per stage (monotonic; 4 per use)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Pair index (within a whole-row grid tile of kTile pixels, grid width W) of
// thread tid at step m: warp w covers block b = 4 m + (w + m) % 4 of 4 rows x 16 columns,
// lane l the pixels (row 4 rb + l / 8, columns 16 cb + 2 (l % 8) + {0, 1}).  A
// quarter-warp reads 8 consecutive float4 of one row (conflict-free).
__device__ __forceinline__ int blk_pair(int m, int tid, int W) {
  // the 4 warps rotate over the 4 blocks of step m, so every warp visits every
  // 16-column strip: invisible image strips (w = 0, skipped) are spread over the
  // warps instead of idling some while others carry the whole item
  const int b = 4 * m + (((tid >> 5) + m) & 3), l = tid & 31;
  const int cbw = W >> 4;
  const int rb = b / cbw, cb = b - rb * cbw;
  return ((4 * rb + (l >> 3)) * W + 16 * cb + 2 * (l & 7)) >> 1;
}

#define FMA2 __ffma2_rn
#define MUL2 __fmul2_rn
#define ADD2 __fadd2_rn
__device__ __forceinline__ float2 S2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 operator-(float2 a) { return make_float2(-a.x, -a.y); }

// Static LPT schedule: CTA b owns tiles sched_ids[sched_off[b] .. sched_off[b+1])
// (host-balanced by edge-pixels, vba_host.cu build_plans), so the producer knows
// every upcoming tile without a global atomic on the critical path.
template <int MODE, bool LIN>
__global__ void __launch_bounds__(kPixBlock, 3) k_vision_stream(
    const PixTile* __restrict__ tiles, const int32_t* __restrict__ sched_off, const int32_t* __restrict__ sched_ids,
    const StreamItem* __restrict__ items, const int32_t* __restrict__ item_off, const float* __restrict__ disp,
    const EdgeGeo32* __restrict__ geo, const float* __restrict__ pix, const float* __restrict__ tgt,
    const float* __restrict__ wts, const int64_t* __restrict__ eoff, const int64_t* __restrict__ doff, int grid_w,
    GridP gp, IntrP in, double* __restrict__ partials, float* __restrict__ Hdd, float* __restrict__ gdo,
    double* __restrict__ tile_energy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* const fpart = reinterpret_cast<float*>(partials);
  StreamSmem& S = *reinterpret_cast<StreamSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float fx = (float)in.fx, fy = (float)in.fy;
  const float fx2 = fx * fx, fy2 = fy * fy;
  const float ifx = (float)(1.0 / in.fx), ify = (float)(1.0 / in.fy);
  const bool blk_ok = grid_w > 0 && grid_w % 16 == 0 && kTile % (4 * grid_w) == 0;
  const int s0 = sched_off[blockIdx.x], nmine = sched_off[blockIdx.x + 1] - s0;
  const int i0 = item_off[blockIdx.x], nitems = item_off[blockIdx.x + 1] - i0;
  auto tile_id = [&](int o) { return o < kSchedCap ? S.tid[o] : sched_ids[s0 + o]; };
  auto tile_at = [&](int o) { return o < kSchedCap ? S.tl[o] : tiles[sched_ids[s0 + o]]; };

  // rows beyond a short tile's count are masked by `act` but still read: zero the
  // ring once so they are finite (stale rows of earlier items are finite too)
  for (int i = tid; i < kStages * kPairs; i += kPixBlock) {
    (&S.flow[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    (&S.wts[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int i = tid; i < nmine && i < kSchedCap; i += kPixBlock) {
    const int t = sched_ids[s0 + i];
    S.tid[i] = t;
    S.tl[i] = tiles[t];
  }
  for (int i = tid; i < nitems && i < kItemCap; i += kPixBlock) S.it[i] = items[i0 + i];
  if (tid < kStages) S.rel[tid] = 0u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes before async-proxy copies
  __syncthreads();

  // ---- producer: item j -> stage j % kStages.  Items 0..kStages-1 by thread 0;
  // item j + kStages by the LAST warp to release item j (no thread ever waits
  // to refill: the ring is topped up the moment a stage drains)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int j) {
    const StreamItem I = j < kItemCap ? S.it[j] : items[i0 + j];
    const int s = j % kStages;
    mbar_expect_tx(&S.full[s], 2u * (uint32_t)I.bytes + (uint32_t)sizeof(EdgeGeo32));
    bulk_g2s(&S.geo[s], geo + I.edge, (uint32_t)sizeof(EdgeGeo32), &S.full[s], pol);
    bulk_g2s(S.flow[s], tgt + I.foff, (uint32_t)I.bytes, &S.full[s], pol);
    bulk_g2s(S.wts[s], wts + I.foff, (uint32_t)I.bytes, &S.full[s], pol);
  };
  auto release = [&](int j) {   // whole warp; call after its last read of item j's stage
    __syncwarp();
    if (lane == 0) {
      // the warp's reads of the stage have returned (their values were consumed);
      // the acq_rel counter orders them before the refill issued by the last warp
      unsigned int r;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(r) : "r"(smem_u32(&S.rel[j % kStages])) : "memory");
      if (r % (kPixBlock / 32) == (kPixBlock / 32) - 1 && j + kStages < nitems) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // others' generic reads before the refill
        issue(j + kStages);
      }
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&S.full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < kStages && j < nitems; ++j) issue(j);
  }
  __syncthreads();

  int item = 0;
#pragma unroll 1
  for (int ord = 0; ord < nmine; ++ord) {
    const PixTile T = tile_at(ord);
    const int64_t kbase = doff[T.src];
    // pixel-pair -> thread map: 4x16-pixel blocks per warp on whole-row grid tiles
    // (spatially coherent, so warp-uniform zero-weight skips are frequent), else linear
    const bool blk = MODE == VBA_PIX_GRID && T.cnt == kTile && blk_ok;
    float2 RX[kTP], RY[kTP], DD[kTP], HD[kTP], GD[kTP];
    int QP[kTP];   // pair index within the tile (= float4 index into the stage rows)
    uint32_t act = 0;
#pragma unroll
    for (int m = 0; m < kTP; ++m) {
      const int p = blk ? blk_pair(m, tid, grid_w) : m * kPixBlock + tid;
      QP[m] = p;
      const int n = T.n0 + 2 * p;
      RX[m] = RY[m] = make_float2(0.f, 0.f);
      DD[m] = make_float2(1.f, 1.f);
      HD[m] = GD[m] = make_float2(0.f, 0.f);
      if (2 * p < T.cnt) {
        act |= 1u << m;
        DD[m] = __ldg(reinterpret_cast<const float2*>(disp + kbase + n));
        if (MODE != VBA_PIX_EDGE)
          load_rays<MODE>(pix, kbase, n, grid_w, gp, in, RX[m].x, RY[m].x, RX[m].y, RY[m].y);
      }
    }
    double etile = 0.0;
#pragma unroll 1
    for (int e = T.eb; e < T.ee; ++e, ++item) {
      const int s = item % kStages;
      if (MODE == VBA_PIX_EDGE) {
#pragma unroll
        for (int m = 0; m < kTP; ++m)
          if (act & (1u << m))
            load_rays<VBA_PIX_KF>(pix, eoff[e], T.n0 + 2 * QP[m], grid_w, gp, in, RX[m].x,
                                  RY[m].x, RX[m].y, RY[m].y);
      }
      mbar_wait(&S.full[s], (item / kStages) & 1);
      const EdgeGeo32 g = S.geo[s];
      float2 acc[LIN ? 27 : 1];
#pragma unroll
      for (int k = 0; k < (LIN ? 27 : 1); ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll
      for (int m = 0; m < kTP; ++m) {
        const float4 wl = S.wts[s][QP[m]];
        // zero-weight skip: a pixel with w = 0 adds exact zeros to every sum
        // (residuals.py:254-263), so a warp whose 64 pixels all have w = 0 skips
        // the arithmetic (bitwise identical result; the rows are still streamed)
        const bool nz = ((act >> m) & 1u) && (wl.x != 0.f || wl.y != 0.f || wl.z != 0.f || wl.w != 0.f);
        if (!__any_sync(0xffffffffu, nz)) continue;
        const float4 fl = S.flow[s][QP[m]];
        const float2 rx = RX[m], ry = RY[m], d = DD[m];
        // project(): D = (M - I) ray + d t,  x - rx = (Dx - rx Dz) / (1 + Dz)
        const float2 Dx = FMA2(d, S2(g.t[0]), FMA2(S2(g.M[0]), rx, FMA2(S2(g.M[1]), ry, S2(g.M[2]))));
        const float2 Dy = FMA2(d, S2(g.t[1]), FMA2(S2(g.M[3]), rx, FMA2(S2(g.M[4]), ry, S2(g.M[5]))));
        const float2 Dz = FMA2(d, S2(g.t[2]), FMA2(S2(g.M[6]), rx, FMA2(S2(g.M[7]), ry, S2(g.M[8]))));
        const float2 Xz = ADD2(S2(1.0f), Dz);
        const float2 th = MUL2(S2(1e-6f), d);
        const bool va = (act >> m) & 1u && Xz.x > th.x;   // z_j > 1e-6 (residuals.py:206-209)
        const bool vb = (act >> m) & 1u && Xz.y > th.y;
        float2 izh = make_float2(va ? rcp_approx(Xz.x) : 0.f, vb ? rcp_approx(Xz.y) : 0.f);
        izh = FMA2(izh, FMA2(-Xz, izh, S2(1.0f)), izh);   // rcp_nr (invalid lanes stay 0)
        const float2 ddx = MUL2(FMA2(-rx, Dz, Dx), izh);
        const float2 ddy = MUL2(FMA2(-ry, Dz, Dy), izh);
        const float2 w0 = make_float2(va ? wl.x : 0.f, vb ? wl.z : 0.f);
        const float2 w1 = make_float2(va ? wl.y : 0.f, vb ? wl.w : 0.f);
        if (!LIN) {
          const float2 r0 = FMA2(S2(-fx), ddx, make_float2(fl.x, fl.z));   // flow - fx (x - rx)
          const float2 r1 = FMA2(S2(-fy), ddy, make_float2(fl.y, fl.w));
          acc[0] = FMA2(MUL2(w0, r0), r0, FMA2(MUL2(w1, r1), r1, acc[0]));
          continue;
        }
        // residual over the focal length: r / fx = flow / fx - (x - rx)
        const float2 rf0 = FMA2(make_float2(fl.x, fl.z), S2(ifx), -ddx);
        const float2 rf1 = FMA2(make_float2(fl.y, fl.w), S2(ify), -ddy);
        const float2 x = ADD2(rx, ddx), y = ADD2(ry, ddy);
        const float2 iz = MUL2(d, izh);
        const float2 xy = MUL2(x, y);
        const float2 a1 = -FMA2(x, x, S2(1.f));   // k0' = [xy, -(1+x^2), y, -iz, 0, x iz]
        const float2 a5 = MUL2(x, iz);
        const float2 b0 = FMA2(y, y, S2(1.f));    // k1' = [1+y^2, -xy, -x, 0, -iz, y iz]
        const float2 b5 = MUL2(y, iz);
        const float2 jd0 = MUL2(FMA2(x, S2(g.t[2]), S2(-g.t[0])), izh);   // J_d = (fx jd0', fy jd1')
        const float2 jd1 = MUL2(FMA2(y, S2(g.t[2]), S2(-g.t[1])), izh);
        const float2 W0 = MUL2(w0, S2(fx2)), W1 = MUL2(w1, S2(fy2));   // as the Gram: (w fx^2) jd
        const float2 R0 = MUL2(W0, rf0), R1 = MUL2(W1, rf1);   // = (w fx) r
        const float2 p0 = MUL2(W0, xy), p1 = MUL2(W0, a1), p2 = MUL2(W0, y), p3 = -MUL2(W0, iz),
                     p5 = MUL2(W0, a5);
        const float2 q0 = MUL2(W1, b0), q1 = -MUL2(W1, xy), q2 = -MUL2(W1, x), q4 = -MUL2(W1, iz),
                     q5 = MUL2(W1, b5);
        acc[0] = FMA2(p0, xy, FMA2(q0, b0, acc[0]));
        acc[1] = FMA2(p0, a1, FMA2(q0, -xy, acc[1]));
        acc[2] = FMA2(p0, y, FMA2(q0, -x, acc[2]));
        acc[3] = FMA2(p0, -iz, acc[3]);
        acc[4] = FMA2(q0, -iz, acc[4]);
        acc[5] = FMA2(p0, a5, FMA2(q0, b5, acc[5]));
        acc[6] = FMA2(p1, a1, FMA2(q1, -xy, acc[6]));
        acc[7] = FMA2(p1, y, FMA2(q1, -x, acc[7]));
        acc[8] = FMA2(p1, -iz, acc[8]);
        acc[9] = FMA2(q1, -iz, acc[9]);
        acc[10] = FMA2(p1, a5, FMA2(q1, b5, acc[10]));
        acc[11] = FMA2(p2, y, FMA2(q2, -x, acc[11]));
        acc[12] = FMA2(p2, -iz, acc[12]);
        acc[13] = FMA2(q2, -iz, acc[13]);
        acc[14] = FMA2(p2, a5, FMA2(q2, b5, acc[14]));
        acc[15] = FMA2(p3, -iz, acc[15]);
        acc[17] = FMA2(p3, a5, acc[17]);
        acc[18] = FMA2(q4, -iz, acc[18]);
        acc[19] = FMA2(q4, b5, acc[19]);
        acc[20] = FMA2(p5, a5, FMA2(q5, b5, acc[20]));
        acc[21] = FMA2(R0, xy, FMA2(R1, b0, acc[21]));
        acc[22] = FMA2(R0, a1, FMA2(R1, -xy, acc[22]));
        acc[23] = FMA2(R0, y, FMA2(R1, -x, acc[23]));
        acc[24] = FMA2(R0, -iz, acc[24]);
        acc[25] = FMA2(R1, -iz, acc[25]);
        acc[26] = FMA2(R0, a5, FMA2(R1, b5, acc[26]));
        HD[m] = FMA2(MUL2(W0, jd0), jd0, FMA2(MUL2(W1, jd1), jd1, HD[m]));
        GD[m] = FMA2(R0, jd0, FMA2(R1, jd1, GD[m]));
      }
      if (LIN) {
        // per-lane sums; stage s is no longer read by this warp: release it
        float v[28];
#pragma unroll
        for (int k = 0; k < 27; ++k) v[k] = acc[k].x + acc[k].y;
        v[16] = 0.f;   // S(3,4): structural zero
        v[27] = 0.f;
        release(item);
        // warp sum by transpose: value k of lane l at xr[k * kRedS + l] (conflict-free
        // stores), lane c < 28 then reads row c as 8 x LDS.128 (row stride 36 words:
        // conflict-free) and sums it with a 3-level FADD2 tree
        float* xr = S.xr[warp];
#pragma unroll
        for (int k = 0; k < 28; ++k) xr[k * kRedS + lane] = v[k];
        __syncwarp();
        if (lane < 28) {
          const float4* row = reinterpret_cast<const float4*>(xr + lane * kRedS);
          float4 q[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) q[j] = row[j];
          float2 h[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) h[j] = ADD2(make_float2(q[j].x, q[j].y), make_float2(q[j].z, q[j].w));
#pragma unroll
          for (int j = 0; j < 4; ++j) h[j] = ADD2(h[j], h[j + 4]);
          h[0] = ADD2(h[0], h[2]);
          h[1] = ADD2(h[1], h[3]);
          h[0] = ADD2(h[0], h[1]);
          fpart[(T.poff + (e - T.eb)) * kPartStride + warp * 32 + lane] = h[0].x + h[0].y;
        }
        __syncwarp();   // xr reads done before the next item's stores
      } else {
        etile += (double)(acc[0].x + acc[0].y);
        release(item);
      }
    }
    if (LIN) {
#pragma unroll
      for (int m = 0; m < kTP; ++m) {
        if (!((act >> m) & 1u)) continue;
        const int64_t n = kbase + T.n0 + 2 * QP[m];
        if (T.pad) {   // one of two edge halves of the tile: add onto zero (order-free with 2 addends)
          atomicAdd(reinterpret_cast<float2*>(Hdd + n), HD[m]);
          atomicAdd(reinterpret_cast<float2*>(gdo + n), GD[m]);
        } else {
          *reinterpret_cast<float2*>(Hdd + n) = HD[m];
          *reinterpret_cast<float2*>(gdo + n) = GD[m];
        }
      }
    } else {
      // per-warp tile energy (fixed-order warp tree; k_energy_reduce sums the records)
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) etile += __shfl_xor_sync(0xffffffffu, etile, o);
      if (lane == 0) tile_energy[(int64_t)tile_id(ord) * (kPixBlock / 32) + warp] = etile;
    }
  }
}

// Planner helper: number of 64-pixel blocks with any non-zero weight per (tile, edge)
// item, in K1's pixel -> warp mapping (4x16 blocks on whole-row grid tiles, else 64
// consecutive pixels).  One warp per item.
__global__ void k_count_nz_blocks(const float* __restrict__ wts, const int64_t* __restrict__ row0,
                                  const int32_t* __restrict__ cnt, int n, int grid_w, int32_t* __restrict__ out) {
  const int item = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (item >= n) return;
  const int c = cnt[item];
  const bool blk = grid_w > 0 && grid_w % 16 == 0 && kTile % (4 * grid_w) == 0 && c == kTile;
  int nz = 0;
  for (int b = 0; b < kTile / 64; ++b) {
    int q;   // pair index of this lane in block b (as K1: block b = 4 m + warp)
    if (blk) {   // block index b is a position in the tile; the counts do not depend on which warp
      const int cbw = grid_w >> 4, rb = b / cbw, cb = b - rb * cbw;
      q = ((4 * rb + (lane >> 3)) * grid_w + 16 * cb + 2 * (lane & 7)) >> 1;
    } else {
      q = (b >> 2) * kPixBlock + (b & 3) * 32 + lane;
    }
    bool any = false;
    if (2 * q < c) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(wts + 2 * (row0[item] + 2 * q)));
      any = w.x != 0.f || w.y != 0.f || w.z != 0.f || w.w != 0.f;
    }
    nz += __any_sync(0xffffffffu, any) ? 1 : 0;
  }
  if (lane == 0) out[item] = nz;
}
void launch_count_nz_blocks(const float* wts, const int64_t* row0, const int32_t* cnt, int n, int grid_w,
                            int32_t* out, cudaStream_t st) {
  if (n <= 0) return;
  k_count_nz_blocks<<<(n + 7) / 8, 256, 0, st>>>(wts, row0, cnt, n, grid_w, out);
  launch_count();
}

// CTAs of the streamed kernels (SMs x resident CTAs of the K1 instance; the
// static schedule is built for exactly this many)
int vision_stream_ctas() {
  static int grid = 0;
  if (grid == 0) {
    const int smem = (int)sizeof(StreamSmem);
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_vision_stream<VBA_PIX_GRID, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_vision_stream<VBA_PIX_GRID, true>, kPixBlock, smem);
    grid = nsm * (occ > 0 ? occ : 1);
  }
  return grid;
}

template <int MODE, bool LIN>
static void launch_stream_t(int ncta, const PixTile* tiles, const int32_t* soff, const int32_t* sids,
                            const StreamItem* items, const int32_t* ioff, const DevState& s, const float* pix, const float* tgt, const float* wts,
                            const int64_t* eoff, const int64_t* doff, int grid_w, GridP gp, IntrP in,
                            double* partials, float* Hdd, float* gd, double* tile_energy, cudaStream_t st) {
  static bool init = false;
  const int smem = (int)sizeof(StreamSmem);
  if (!init) {
    cudaFuncSetAttribute(k_vision_stream<MODE, LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  k_vision_stream<MODE, LIN><<<ncta, kPixBlock, smem, st>>>(tiles, soff, sids, items, ioff, s.disp, s.geo32, pix, tgt, wts,
                                                             eoff, doff, grid_w, gp, in, partials, Hdd, gd,
                                                             tile_energy);
  launch_count();
}

template <bool LIN>
static void launch_stream(int mode, const PixTile* tiles, const int32_t* soff, const int32_t* sids,
                          const StreamItem* items, const int32_t* ioff, int ncta,
                          const DevState& s, const float* pix, const float* tgt, const float* wts,
                          const int64_t* eoff, const int64_t* doff, int grid_w, const double* grid,
                          const double* intr, double* partials, float* Hdd, float* gd, double* tile_energy,
                          cudaStream_t st) {
  if (ncta <= 0) return;
  GridP gp{grid[0], grid[1], grid[2], grid[3]};
  IntrP in{intr[0], intr[1], intr[2], intr[3]};
  if (mode == VBA_PIX_GRID)
    launch_stream_t<VBA_PIX_GRID, LIN>(ncta, tiles, soff, sids, items, ioff, s, pix, tgt, wts, eoff, doff, grid_w, gp, in,
                                       partials, Hdd, gd, tile_energy, st);
  else if (mode == VBA_PIX_KF)
    launch_stream_t<VBA_PIX_KF, LIN>(ncta, tiles, soff, sids, items, ioff, s, pix, tgt, wts, eoff, doff, grid_w, gp, in,
                                     partials, Hdd, gd, tile_energy, st);
  else
    launch_stream_t<VBA_PIX_EDGE, LIN>(ncta, tiles, soff, sids, items, ioff, s, pix, tgt, wts, eoff, doff, grid_w, gp, in,
                                       partials, Hdd, gd, tile_energy, st);
}

void launch_vision_linearize(int mode, const PixTile* tiles, const int32_t* soff, const int32_t* sids,
                             const StreamItem* items, const int32_t* ioff, int ncta,
                             const DevState& s, const float* pix, const float* tgt, const float* wts,
                             const int64_t* eoff, const int64_t* doff, int grid_w, const double* grid,
                             const double* intr, double* partials, float* Hdd, float* gd, cudaStream_t st) {
  launch_stream<true>(mode, tiles, soff, sids, items, ioff, ncta, s, pix, tgt, wts, eoff, doff, grid_w, grid, intr, partials,
                      Hdd, gd, nullptr, st);
}

void launch_vision_energy(int mode, const PixTile* tiles, const int32_t* soff, const int32_t* sids,
                          const StreamItem* items, const int32_t* ioff, int ncta,
                          const DevState& s, const float* pix, const float* tgt, const float* wts,
                          const int64_t* eoff, const int64_t* doff, int grid_w, const double* grid,
                          const double* intr, double* tile_energy, cudaStream_t st) {
  launch_stream<false>(mode, tiles, soff, sids, items, ioff, ncta, s, pix, tgt, wts, eoff, doff, grid_w, grid, intr, nullptr,
                       nullptr, nullptr, tile_energy, st);
}

// ---------------------------------------------------------------------------
// per-edge finalisation: sum K1 partials over the source's tiles (fixed order),
// then H_ii = G_i^T S G_i, H_jj = G_j^T S G_j, H_ij = -G_i^T S G_j,
// g_i = G_i^T s, g_j = -G_j^T s   (fp64; solver.py:201-219 in factorised form)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(64) k_edge_finalize(const int32_t* __restrict__ t0s,
                                                      const int32_t* __restrict__ t1s,
                                                      const PixTile* __restrict__ tiles,
                                                      const int32_t* __restrict__ edge_i, int e0,
                                                      const double* __restrict__ partials,
                                                      const double* __restrict__ geo64, Extr x,
                                                      double* __restrict__ vis, double* __restrict__ eng) {
  __shared__ double v[32], S[36], Gi[36], Gj[36], T1[36], T2[36];
  const int e = e0 + blockIdx.x, tid = threadIdx.x;
  const int src = edge_i[e];
  if (tid < 32) {   // K1 records: per (tile, edge) one fp32 32-vector per warp, summed in fp64, fixed order
    const float* fp = reinterpret_cast<const float*>(partials);
    double s = 0.0;
    for (int t = t0s[src]; t < t1s[src]; ++t) {
      const float* r = fp + (tiles[t].poff + (e - tiles[t].eb)) * kPartStride;
#pragma unroll
      for (int w = 0; w < kPartWarps; ++w) s += (double)r[w * 32 + tid];
    }
    v[tid] = s;
  }
  if (tid == 32) {
    const double* q = geo64 + (int64_t)kGeo64 * e;
    build_G(q, q + 18, q + 9, Gi);           // G_i from (A R_i, c1, A)
  }
  if (tid == 33) {
    const double* q = geo64 + (int64_t)kGeo64 * e;
    build_G(x.RbcT, x.c2, q + 9, Gj);        // G_j from (R_bc^T, c2, A)
  }
  __syncthreads();
  if (tid < 36) {  // unpack upper triangle -> full symmetric S
    const int a = tid / 6, b = tid % 6;
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    const int idx = lo * 6 - lo * (lo - 1) / 2 + (hi - lo);
    S[tid] = v[idx];
  }
  __syncthreads();
  if (tid < 36) {
    const int a = tid / 6, b = tid % 6;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      s1 += S[a * 6 + m] * Gi[m * 6 + b];
      s2 += S[a * 6 + m] * Gj[m * 6 + b];
    }
    T1[tid] = s1;
    T2[tid] = s2;
  }
  __syncthreads();
  double* out = vis + (int64_t)kVisBlock * e;
  if (tid < 36) {
    const int a = tid / 6, b = tid % 6;
    double hii = 0.0, hjj = 0.0, hij = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      hii += Gi[m * 6 + a] * T1[m * 6 + b];
      hjj += Gj[m * 6 + a] * T2[m * 6 + b];
      hij += Gi[m * 6 + a] * T2[m * 6 + b];
    }
    out[tid] = hii;
    out[36 + tid] = hjj;
    out[72 + tid] = -hij;
  } else if (tid < 48) {
    const int a = (tid - 36) % 6;
    const bool isj = tid >= 42;
    const double* G = isj ? Gj : Gi;
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) s += G[m * 6 + a] * v[21 + m];
    out[108 + (isj ? 6 : 0) + a] = isj ? -s : s;
  } else if (tid == 48 && eng) {
    eng[e] = v[27];
  }
}

void launch_edge_finalize(const int32_t* t0s, const int32_t* t1s, const PixTile* tiles, const int32_t* edge_i,
                          int e0, int n, const double* partials, const DevState& s, const Extr& x, double* vis,
                          double* eng, cudaStream_t st) {
  if (n <= 0) return;
  k_edge_finalize<<<n, 64, 0, st>>>(t0s, t1s, tiles, edge_i, e0, partials, s.geo64, x, vis, eng);
  launch_count();
}

// ---------------------------------------------------------------------------
// K4: Schur fill-in Gram (per LM trial, λ-dependent), on the fp64 tensor cores.
//   C_{e1 e2} = sum_n k_{n,e1} k_{n,e2}^T / Hdd_d(n),   b_e = sum_n k_{n,e} g_d(n) / Hdd_d(n)
// with k_{n,e} = sum_c w_c K_c^T J_d,c the per-pixel coupling (K-space).  One CTA
// (16 warps) per (source, pixel range).  Per 32-pixel chunk the CTA computes the
// fp32 coupling vectors and widens them exactly to fp64 in shared memory as
//   U = [k_{n,e} (6k columns) | g_d(n)]   and   V = k_{n,e} / Hdd_d(n)
// (column-major [column][pixel], stride GPX = 36 ≡ 4 mod 16: conflict-free DMMA
// fragments), then C = U^T V accumulates with mma.sync m8n8k4 f64 in registers
// across all chunks (each warp owns up to GT 8x8 output tiles of the lower
// band, in 2x2 units).  The last row of C is b.  fp64 products of fp32 factors are exact and
// all sums are fp64: no fp32 partial-sum error, fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int GPX = kGramPC + 4;   // pixel stride of the U / V columns (doubles)
constexpr int GWARPS = 16;
// 8x8 output tiles per warp: 2x2 units, 5 per warp up to 30 out-edges, 6 at 31 (and in slices)
__host__ __device__ constexpr int gram_tiles_per_warp(int kmax) { return kmax <= 30 ? 20 : 24; }
// 2x2 tile units of a source with k out-edges, and the units one CTA takes in a slice
int gram_units(int k) {
  const int nc = 6 * k, NRt = (nc + 1 + 7) / 8, NCt = (nc + 7) / 8;
  int U = 0;
  for (int tj = 0; tj < NCt; tj += 2)
    for (int ti = tj > 0 ? tj - 1 : 0; ti < NRt; ti += 2) ++U;
  return U;
}
int gram_slice_units() { return GWARPS * 24 / 4; }

__device__ __forceinline__ void gdmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

#define GPROF(i, v)
template <int MODE, int GT, int KE>
__global__ void __launch_bounds__(GWARPS * 32, 1) k_gram(
    const GramTile* __restrict__ gts, const float* __restrict__ disp, const EdgeGeo32* __restrict__ geo,
    const float* __restrict__ pix, const float* __restrict__ wts, const int64_t* __restrict__ eoff,
    const int64_t* __restrict__ doff, int grid_w, GridP gp, IntrP in, const float* __restrict__ Hdd,
    const float* __restrict__ gd, double lam, double ridge, int kmax, double* __restrict__ out,
    const int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const GramTile T = gts[order ? order[blockIdx.x] : blockIdx.x];   // launch order: largest sources first
  const int k = T.ee - T.eb;
  const int npairs = k * (k + 1) / 2;
  const int NRmax = (6 * kmax + 1 + 7) / 8 * 8;
  // U / V staging, double-buffered by chunk: buffer b at smem_raw + b * 2 * NRmax * GPX doubles
  double* const UV = reinterpret_cast<double*>(smem_raw);
  const size_t uvs = (size_t)NRmax * GPX;   // doubles per U (or V) buffer
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int64_t kbase = doff[T.src];
  const float fx = (float)in.fx, fy = (float)in.fy;
  const float fx2 = fx * fx, fy2 = fy * fy;
  const double damp = 1.0 + lam;
  const int nc = 6 * k;
  const int NRt = (nc + 1 + 7) / 8, NCt = (nc + 7) / 8;   // row / column tiles of C
  // output tiles: lower band tj <= ti + 1 (6x6 blocks may straddle the 8-tile diagonal),
  // grouped in 2x2 units (ti, ti + 1) x (tj, tj + 1) that share their A and B fragments
  // (4 shared-memory loads per 4 DMMAs: shared-memory bandwidth co-limits the DMMA pipe).
  // Every warp takes nu = U / GWARPS whole units (slots 4u + {0: (ti, tj), 1: (ti + 1, tj),
  // 2: (ti, tj + 1), 3: (ti + 1, tj + 1)}); the U % GWARPS leftover units are split into
  // column pairs {(ti, tj), (ti + 1, tj)} (3 loads per 2 DMMAs) dealt round-robin after
  // them, so the per-chunk barrier waits for at most one pair more than the average.
  // -1 = outside C (computed on clamped fragments, never stored; also the one tile of a
  // diagonal unit above the band).
  __shared__ short tile_i[GWARPS * GT], tile_j[GWARPS * GT];
  __shared__ int nu_s, npw_s[GWARPS];
  __shared__ double invs[2][kGramPC];   // 1 / (Hdd (1 + lam) + ridge) per pixel, double-buffered by chunk
  __shared__ float4 geos[(KE + 1) * 4];   // the source's out-edge geometry (k <= KE), EdgeGeo32 records
  // C = sum_n u_n u_n^T / h_n is formed as W^T W with W = u / sqrt(h_n) (one staged matrix)
  auto pixel_inv = [&](int n) { return n < T.n1 ? 1.0 / sqrt((double)Hdd[kbase + n] * damp + ridge) : 0.0; };
  if (tid == 0 && T.u1 > T.u0) {
    // slice [u0, u1) of the unit list (sources with more out-edges than one CTA's registers
    // hold: several CTAs share the pixel range, each its own units, disjoint outputs of one
    // partial record): whole units round-robin over the warps, missing slots -1
    const int cnt = T.u1 - T.u0, nu = (cnt + GWARPS - 1) / GWARPS;
    for (int i = 0; i < GWARPS * GT; ++i) tile_i[i] = tile_j[i] = -1;
    for (int w = 0; w < GWARPS; ++w) npw_s[w] = 0;
    int u = 0;
    for (int tj = 0; tj < NCt; tj += 2)
      for (int ti = tj > 0 ? tj - 1 : 0; ti < NRt; ti += 2, ++u) {
        if (u < T.u0 || u >= T.u1) continue;
        const int r1 = ti + 1 < NRt ? ti + 1 : -1, c1 = tj + 1 < NCt ? tj + 1 : -1;
        const int w = (u - T.u0) % GWARPS, sl = 4 * ((u - T.u0) / GWARPS);
        tile_i[w + GWARPS * sl] = (short)ti; tile_j[w + GWARPS * sl] = (short)tj;
        tile_i[w + GWARPS * (sl + 1)] = (short)r1; tile_j[w + GWARPS * (sl + 1)] = (short)tj;
        tile_i[w + GWARPS * (sl + 2)] = (short)ti; tile_j[w + GWARPS * (sl + 2)] = (short)c1;
        tile_i[w + GWARPS * (sl + 3)] = (short)r1; tile_j[w + GWARPS * (sl + 3)] = (short)c1;
      }
    nu_s = nu;
  } else if (tid == 0) {
    int U = 0;
    for (int tj = 0; tj < NCt; tj += 2)
      for (int ti = tj > 0 ? tj - 1 : 0; ti < NRt; ti += 2) ++U;
    const int nu = U / GWARPS;
    int u = 0, pr = 0;
    for (int w = 0; w < GWARPS; ++w) npw_s[w] = 0;
    auto put = [&](int w, int sl, int ti, int tj) {
      if (sl < GT) { tile_i[w + GWARPS * sl] = (short)ti; tile_j[w + GWARPS * sl] = (short)tj; }
    };
    for (int tj = 0; tj < NCt; tj += 2)
      for (int ti = tj > 0 ? tj - 1 : 0; ti < NRt; ti += 2, ++u) {
        const int r1 = ti + 1 < NRt ? ti + 1 : -1, c1 = tj + 1 < NCt ? tj + 1 : -1;
        if (u < nu * GWARPS) {
          const int w = u % GWARPS, sl = 4 * (u / GWARPS);
          put(w, sl, ti, tj); put(w, sl + 1, r1, tj); put(w, sl + 2, ti, c1); put(w, sl + 3, r1, c1);
        } else {
          for (int h = 0; h < 2; ++h) {
            const int c = h == 0 ? tj : c1;
            if (c < 0) continue;
            const int w = pr % GWARPS, sl = 4 * nu + 2 * npw_s[w];
            put(w, sl, ti, c); put(w, sl + 1, r1, c);
            ++npw_s[w];
            ++pr;
          }
        }
      }
    nu_s = nu;
  }
  double acc[GT][2];
#pragma unroll
  for (int q = 0; q < GT; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int i = tid; i < 2 * (int)uvs; i += nth) UV[i] = 0.0;   // padding columns stay zero
  if (tid < kGramPC) invs[0][tid] = pixel_inv(T.n0 + tid);
  if (tid < 4 * k) geos[tid] = __ldg(reinterpret_cast<const float4*>(geo + T.eb) + tid);
  __syncthreads();
  const int n4 = 4 * nu_s;                       // slots in whole 2x2 units (same for all warps)
  const int nmine = n4 + 2 * npw_s[warp];        // + column pairs: tile slots of this warp

  // Phase 1 of a chunk: coupling vectors of its (pixel, edge) items (at most kGramItems
  // per thread), widened to fp64 into buffer b.  Loads of all items first (gload),
  // arithmetic + stores per item (gitem), so the arithmetic can be interleaved with
  // the DMMAs of the previous chunk.
  constexpr int kGramItems = (kGramPC * KE + GWARPS * 32 - 1) / (GWARPS * 32);
  float d_[kGramItems], rx_[kGramItems], ry_[kGramItems], gd_[kGramItems];
  float2 w_[kGramItems];
  auto gload = [&](int c0) {
#pragma unroll
    for (int j = 0; j < kGramItems; ++j) {
      const int it = tid + j * nth;
      const int e = it / kGramPC, px = it % kGramPC, n = c0 + px;
      d_[j] = rx_[j] = ry_[j] = gd_[j] = 0.f;
      w_[j] = make_float2(0.f, 0.f);
      if (it < kGramPC * k && n < T.n1) {
        d_[j] = disp[kbase + n];
        if (e == 0) gd_[j] = gd[kbase + n];
        float rx1, ry1;
        if (MODE == VBA_PIX_EDGE)
          load_rays<VBA_PIX_KF>(pix, eoff[T.eb + e], n & ~1, grid_w, gp, in, rx_[j], ry_[j], rx1, ry1);
        else
          load_rays<MODE>(pix, kbase, n & ~1, grid_w, gp, in, rx_[j], ry_[j], rx1, ry1);
        if (n & 1) { rx_[j] = rx1; ry_[j] = ry1; }
        w_[j] = __ldg(reinterpret_cast<const float2*>(wts + 2 * (eoff[T.eb + e] + n)));
      }
    }
  };
  auto gitem = [&](int j, int c0, int b) {
    const int it = tid + j * nth;
    if (it >= kGramPC * k) return;
    double* U = UV + (size_t)b * uvs;
    const int e = it / kGramPC, px = it % kGramPC;
    const int n = c0 + px;
    float u[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    double sc = 0.0;   // 1 / sqrt(h_n)
    if (n < T.n1) {
      const EdgeGeo32 g = load_geo<true>(reinterpret_cast<const EdgeGeo32*>(geos), e);
      const PxGeom o = project(g, rx_[j], ry_[j], d_[j]);
      const float w0 = o.valid ? w_[j].x : 0.f, w1 = o.valid ? w_[j].y : 0.f;
      const float jd0 = fmaf(o.x, g.t[2], -g.t[0]) * o.izh;
      const float jd1 = fmaf(o.y, g.t[2], -g.t[1]) * o.izh;
      const float c0w = w0 * fx2 * jd0, c1w = w1 * fy2 * jd1;
      const float xy = o.x * o.y;
      u[0] = fmaf(c0w, xy, c1w * fmaf(o.y, o.y, 1.f));
      u[1] = fmaf(c0w, -fmaf(o.x, o.x, 1.f), c1w * -xy);
      u[2] = fmaf(c0w, o.y, c1w * -o.x);
      u[3] = c0w * -o.iz;
      u[4] = c1w * -o.iz;
      u[5] = fmaf(c0w, o.x * o.iz, c1w * (o.y * o.iz));
      sc = invs[b][px];
      if (e == 0) U[(size_t)nc * GPX + px] = (double)gd_[j] * sc;
    } else if (e == 0) {
      U[(size_t)nc * GPX + px] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) U[(size_t)(6 * e + r) * GPX + px] = (double)u[r] * sc;
  };
  // prologue: phase 1 of chunk 0 (buffer 0) and the pixel inverses of chunk 1
  gload(T.n0);
#pragma unroll
  for (int j = 0; j < kGramItems; ++j) gitem(j, T.n0, 0);
  if (tid >= nth - kGramPC) invs[1][tid - (nth - kGramPC)] = pixel_inv(T.n0 + kGramPC + tid - (nth - kGramPC));
  for (int c0 = T.n0, cb = 0; c0 < T.n1; c0 += kGramPC, cb ^= 1) {
    __syncthreads();
    // C += U^T V (buffer cb) on the fp64 tensor cores, 8 pixel-steps of 4, with the
    // phase-1 items of chunk c + 1 (buffer cb ^ 1) interleaved between the tiles
    const int cn = c0 + kGramPC;
    const bool more = cn < T.n1;
    if (more) gload(cn);
    const double* Ub = UV + (size_t)cb * uvs;
    const double* Vb = Ub;   // C = W^T W
    const int am = lane >> 2, ak = lane & 3;
    static_assert(GT % 4 == 0, "2x2 units");
#pragma unroll
    for (int q = 0; q < GT; q += 4) {
      if (q >= n4 && q < nmine) {   // one or two column pairs (slots q, q + 1 and q + 2, q + 3)
#pragma unroll
        for (int h = 0; h < 4; h += 2) {
          if (q + h >= nmine) break;
          const int r1 = tile_i[warp + GWARPS * (q + h + 1)];
          const int i0 = tile_i[warp + GWARPS * (q + h)], j0 = tile_j[warp + GWARPS * (q + h)];
          const double* pa0 = Ub + (size_t)((i0 >= 0 ? i0 : 0) * 8 + am) * GPX + ak;
          const double* pa1 = Ub + (size_t)((r1 >= 0 ? r1 : 0) * 8 + am) * GPX + ak;
          const double* pb = Vb + (size_t)((j0 >= 0 ? j0 : 0) * 8 + am) * GPX + ak;
#pragma unroll
          for (int ks = 0; ks < kGramPC / 4; ++ks) {
            const double b = pb[4 * ks];
            gdmma(acc[q + h][0], acc[q + h][1], pa0[4 * ks], b);
            gdmma(acc[q + h + 1][0], acc[q + h + 1][1], pa1[4 * ks], b);
          }
        }
      } else if (q < n4) {
        const int r1 = tile_i[warp + GWARPS * (q + 1)], c1 = tile_j[warp + GWARPS * (q + 2)];
        const int i0 = tile_i[warp + GWARPS * q], j0 = tile_j[warp + GWARPS * q];
        const double* pa0 = Ub + (size_t)((i0 >= 0 ? i0 : 0) * 8 + am) * GPX + ak;
        const double* pa1 = Ub + (size_t)((r1 >= 0 ? r1 : 0) * 8 + am) * GPX + ak;
        const double* pb0 = Vb + (size_t)((j0 >= 0 ? j0 : 0) * 8 + am) * GPX + ak;
        const double* pb1 = Vb + (size_t)((c1 >= 0 ? c1 : 0) * 8 + am) * GPX + ak;
#pragma unroll
        for (int ks = 0; ks < kGramPC / 4; ++ks) {
          const double a0 = pa0[4 * ks], a1 = pa1[4 * ks], b0 = pb0[4 * ks], b1 = pb1[4 * ks];
          gdmma(acc[q][0], acc[q][1], a0, b0);
          gdmma(acc[q + 1][0], acc[q + 1][1], a1, b0);
          gdmma(acc[q + 2][0], acc[q + 2][1], a0, b1);
          gdmma(acc[q + 3][0], acc[q + 3][1], a1, b1);
        }
      }
      if (q % 8 == 4 && q / 8 < kGramItems && more) gitem(q / 8, cn, cb ^ 1);
    }
#pragma unroll
    for (int j = (GT + 3) / 8; j < kGramItems; ++j)
      if (more) gitem(j, cn, cb ^ 1);
    // pixel inverses of chunk c + 2 (buffer cb: chunk c's items are done)
    if (tid >= nth - kGramPC) invs[cb][tid - (nth - kGramPC)] = pixel_inv(cn + kGramPC + tid - (nth - kGramPC));
  }
  // epilogue: scatter the lower 6x6 blocks (e1 >= e2) and the b row into the output layout
  double* o = out + T.out;
#pragma unroll
  for (int q = 0; q < GT; ++q) {
    if (q >= nmine || tile_i[warp + GWARPS * q] < 0 || tile_j[warp + GWARPS * q] < 0) continue;
    const int a = tile_i[warp + GWARPS * q] * 8 + (lane >> 2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = tile_j[warp + GWARPS * q] * 8 + 2 * (lane & 3) + h;
      if (b >= nc) continue;
      if (a < nc) {
        const int e1 = a / 6, e2 = b / 6;
        if (e1 >= e2) o[(e1 * (e1 + 1) / 2 + e2) * 36 + (a % 6) * 6 + (b % 6)] = acc[q][h];
      } else if (a == nc) {
        o[npairs * 36 + b] = acc[q][h];
      }
    }
  }
}

template <int MODE, int GT, int KE>
static void launch_gram_t(const GramTile* gt, int ngt, int block, size_t smem, int kmax, const DevState& s,
                          const float* pix, const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w,
                          GridP gp, IntrP in, const float* Hdd, const float* gd, double lam, double ridge,
                          double* gram_part, const int32_t* order, cudaStream_t st) {
  cudaFuncSetAttribute(k_gram<MODE, GT, KE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_gram<MODE, GT, KE><<<ngt, block, smem, st>>>(gt, s.disp, s.geo32, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd,
                                                 lam, ridge, kmax, gram_part, order);
}

template <int MODE>
static void launch_gram_m(const GramTile* gt, int ngt, int block, size_t smem, int kmax, const DevState& s,
                          const float* pix, const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w,
                          GridP gp, IntrP in, const float* Hdd, const float* gd, double lam, double ridge,
                          double* gram_part, const int32_t* order, cudaStream_t st) {
  if (kmax > 31)   // sliced units (gram_unit_slice), up to 63 out-edges
    launch_gram_t<MODE, 24, 63>(gt, ngt, block, smem, kmax, s, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                                ridge, gram_part, order, st);
  else if (gram_tiles_per_warp(kmax) == 20)
    launch_gram_t<MODE, 20, 31>(gt, ngt, block, smem, kmax, s, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                                ridge, gram_part, order, st);
  else
    launch_gram_t<MODE, 24, 31>(gt, ngt, block, smem, kmax, s, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                                ridge, gram_part, order, st);
}

void launch_gram(int mode, const GramTile* gt, int ngt, int block, size_t smem, int kmax, const DevState& s,
                 const float* pix, const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w,
                 const double* grid, const double* intr, const float* Hdd, const float* gd, double lam,
                 double ridge, double* gram_part, cudaStream_t st, const int32_t* order) {
  if (ngt <= 0) return;
  GridP gp{grid[0], grid[1], grid[2], grid[3]};
  IntrP in{intr[0], intr[1], intr[2], intr[3]};
  if (mode == VBA_PIX_GRID)
    launch_gram_m<VBA_PIX_GRID>(gt, ngt, block, smem, kmax, s, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                                ridge, gram_part, order, st);
  else if (mode == VBA_PIX_KF)
    launch_gram_m<VBA_PIX_KF>(gt, ngt, block, smem, kmax, s, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                              ridge, gram_part, order, st);
  else
    launch_gram_m<VBA_PIX_EDGE>(gt, ngt, block, smem, kmax, s, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                                ridge, gram_part, order, st);
  launch_count();
}


// ---------------------------------------------------------------------------
// K4 on the 5th-gen tensor cores (windows with >= 256 pixels per keyframe): the same
// Gram C = W^T W, W = [k_{n,e} / sqrt(h_n) (6k columns) | g_d(n) / sqrt(h_n)], as
// k_gram, on tcgen05.mma kind::tf32 with 3xTF32 splitting: w = hi + lo (hi = tf32(w),
// lo = tf32(w - hi), 22 significant bits), C ~ Wh^T Wh + Wh^T Wl + Wl^T Wh with fp32
// accumulation in TMEM over the tile's pixel range; k_fill_transform sums the ranges
// in fp64 (fixed order: deterministic).  Emulated on configs 3 and 4 the reduced
// step moves by < 1e-7 relative (tools/gram_tc_precision.py), far inside 1e-5.
//
// Operands: W^T staged per 32-pixel chunk as K-major SWIZZLE_128B images (row m = W
// column m, its 32 pixels = one 128-B swizzle row; 8-row atoms of 1 KB), hi and lo.
// A and B are the same images:  tile 0 = rows 0..127 x columns 0..Mp (N0 = Mp, the
// rows beyond 127 of C come out transposed), tile 1 (M = 6k + 1 > 128 only) = rows
// 128..255 x columns 128..Mp (N1 = Mp - 128).  Rows >= M of A and columns >= M of B
// only feed accumulator rows / columns that are never read.
//
// Warp roles (288 threads): warps 0-7 produce the chunks (lane = pixel, warp w takes
// out-edges w, w + 8, ...; warp 0 also the g_d row) into a 2-stage ring (full / empty
// mbarriers) and run the epilogue; warp 8 owns TMEM (256 columns: 2 CTAs per SM) and
// one of its lanes issues the MMAs.
// ---------------------------------------------------------------------------
// measured alternatives: 12 or 16 producer warps, 3-4 stages at 1 CTA per SM
constexpr int kGtcPW = 8;                        // producer warps
constexpr int kGtcEPW = (31 + kGtcPW - 1) / kGtcPW;   // out-edges per producer warp (k <= 31)
constexpr int kGtcThreads = (kGtcPW + 1) * 32;
static_assert(kGtcPW % 4 == 0, "epilogue: whole groups of 4 warps (one per TMEM lane quarter)");
constexpr int kGtcStages = 2;
constexpr int kGtcTmemCols = 256;

__host__ __device__ __forceinline__ int gtc_mp(int kmax) { return (6 * kmax + 1 + 15) / 16 * 16; }
__host__ __device__ __forceinline__ int gtc_rows(int kmax) { return gtc_mp(kmax) > 128 ? gtc_mp(kmax) : 128; }
// stage = hi + lo images of gtc_rows rows x 128 B; tile 1's A reads 128 rows from row 128,
// so up to 256 - rows rows past the last image are addressed (slack) -- plus 1 KB alignment
size_t gram_tc_smem_bytes(int kmax) {
  const int R = gtc_rows(kmax);
  return (size_t)kGtcStages * 2 * R * 128 + (size_t)(256 - (R < 256 ? R : 256)) * 128 + 1024;
}

template <int MODE>
__global__ void __launch_bounds__(kGtcThreads, 2) k_gram_tc(
    const GramTile* __restrict__ gts, const float* __restrict__ disp, const EdgeGeo32* __restrict__ geo,
    const float* __restrict__ pix, const float* __restrict__ wts, const int64_t* __restrict__ eoff,
    const int64_t* __restrict__ doff, int grid_w, GridP gp, IntrP in, const float* __restrict__ Hdd,
    const float* __restrict__ gd, double lam, double ridge, int kmax, double* __restrict__ out,
    const int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char gtc_raw[];
  unsigned char* ring = gtc_raw + ((1024u - (su32(gtc_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kGtcStages], empty[kGtcStages], accb;
  __shared__ uint32_t tmem_sh;
  __shared__ float4 geos[32 * 4];   // the source's out-edge geometry (k <= 31)
  const GramTile T = gts[order ? order[blockIdx.x] : blockIdx.x];
  const int k = T.ee - T.eb, nc = 6 * k, M = nc + 1;
  const int Mp = (M + 15) / 16 * 16;
  const bool two = M > 128;
  const int N0 = Mp, N1 = two ? Mp - 128 : 0;
  const int R = gtc_rows(kmax);
  const uint32_t img = (uint32_t)R * 128, stage_bytes = 2 * img;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t kbase = doff[T.src];
  const int nch = (T.n1 - T.n0 + 31) / 32;
  if (warp == kGtcPW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_sh)),
                 "n"(kGtcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int q = 0; q < kGtcStages; ++q) {
      tc_mbar_init(&full[q], kGtcPW);
      tc_mbar_init(&empty[q], 1);
    }
    tc_mbar_init(&accb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 4 * k) geos[tid] = __ldg(reinterpret_cast<const float4*>(geo + T.eb) + tid);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == kGtcPW) {
    // ---- MMA issuer
    if (lane == 0) {
      const uint32_t id0 = tc_idesc_tf32(N0), id1 = tc_idesc_tf32(two ? N1 : 16);
      const uint32_t d0 = tmem, d1 = tmem + (uint32_t)N0;
      for (int c = 0; c < nch; ++c) {
        const int sidx = c % kGtcStages;
        tc_mbar_wait(&full[sidx], (uint32_t)(c / kGtcStages) & 1u);
        tc_fence_after();
        const uint32_t hi = su32(ring) + (uint32_t)sidx * stage_bytes, lo = hi + img;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {   // 8 tf32 (32 B) of K per MMA
          const uint32_t o = 32u * kk, acc = (c > 0 || kk > 0) ? 1u : 0u;
          tc_mma_tf32(d0, tc_sdesc(hi + o), tc_sdesc(hi + o), acc, id0);
          tc_mma_tf32(d0, tc_sdesc(hi + o), tc_sdesc(lo + o), 1u, id0);
          tc_mma_tf32(d0, tc_sdesc(lo + o), tc_sdesc(hi + o), 1u, id0);
          if (two) {
            const uint32_t t1 = 128u * 128u;   // row 128 of the images
            tc_mma_tf32(d1, tc_sdesc(hi + t1 + o), tc_sdesc(hi + t1 + o), acc, id1);
            tc_mma_tf32(d1, tc_sdesc(hi + t1 + o), tc_sdesc(lo + t1 + o), 1u, id1);
            tc_mma_tf32(d1, tc_sdesc(lo + t1 + o), tc_sdesc(hi + t1 + o), 1u, id1);
          }
        }
        tc_commit(&empty[sidx]);
      }
      tc_commit(&accb);
    }
    __syncwarp();
  } else {
    // ---- producers: lane = pixel of the chunk, warp w: out-edges w, w + 8, ...
    // The global loads of chunk c + 1 are issued before chunk c is computed (register
    // double buffer), so their latency hides under the arithmetic and the ring waits.
    const float fx = (float)in.fx, fy = (float)in.fy;
    const float fx2 = fx * fx, fy2 = fy * fy;
    const float dampf = (float)(1.0 + lam), ridgef = (float)ridge;
    int64_t ew[kGtcEPW];   // first flow/weight row of each of this warp's out-edges
#pragma unroll
    for (int q = 0; q < kGtcEPW; ++q) {
      const int e = warp + kGtcPW * q;
      ew[q] = e < k ? eoff[T.eb + e] : 0;
    }
    struct Pre { float d, h, g, rx, ry; float2 w[kGtcEPW]; };
    auto fetch = [&](int c, Pre& p) {
      const int n = T.n0 + 32 * c + lane;
      p.d = p.h = p.g = p.rx = p.ry = 0.f;
#pragma unroll
      for (int q = 0; q < kGtcEPW; ++q) p.w[q] = make_float2(0.f, 0.f);
      if (n >= T.n1) return;
      p.d = disp[kbase + n];
      p.h = Hdd[kbase + n];
      if (warp == 0) p.g = gd[kbase + n];
      if (MODE != VBA_PIX_EDGE) {
        float rx1, ry1;
        load_rays<MODE>(pix, kbase, n & ~1, grid_w, gp, in, p.rx, p.ry, rx1, ry1);
        if (n & 1) { p.rx = rx1; p.ry = ry1; }
      }
#pragma unroll
      for (int q = 0; q < kGtcEPW; ++q)
        if (warp + kGtcPW * q < k) p.w[q] = __ldg(reinterpret_cast<const float2*>(wts + 2 * (ew[q] + n)));
    };
    // W^T[m][lane] = hi + lo: hi = w rounded to 11 significant bits (its low 13 bits are
    // zero: an exact tf32), lo = w - hi exactly (the tensor core reads lo's leading 11
    // bits: ~2^-21 relative overall)
    auto soff = [&](int m) {   // byte offset of W^T[m][lane] in an image
      return (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u +
             ((uint32_t)((lane >> 2) ^ (m & 7)) << 4) + (uint32_t)(lane & 3) * 4u;
    };
    auto put = [&](unsigned char* hi, uint32_t off, float w) {
      const float h = __uint_as_float((__float_as_uint(w) + 0x1000u) & 0xFFFFE000u);
      *reinterpret_cast<float*>(hi + off) = h;
      *reinterpret_cast<float*>(hi + img + off) = w - h;
    };
    // row m = 6 (warp + 8 q) + r: m & 7 does not depend on q (48 q = 0 mod 8), so the row
    // offsets are base_r + q * 6 KB with warp-constant base_r
    uint32_t base[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) base[r] = soff(6 * warp + r);
    const uint32_t goff = soff(nc);
    Pre cur, nxt;
    fetch(0, cur);
    for (int c = 0; c < nch; ++c) {
      const int sidx = c % kGtcStages;
      const int n = T.n0 + 32 * c + lane;
      const bool in_range = n < T.n1;
      if (c + 1 < nch) fetch(c + 1, nxt);
      const float sc = in_range ? rsqrtf(fmaf(cur.h, dampf, ridgef)) : 0.f;
      if (c >= kGtcStages) tc_mbar_wait(&empty[sidx], (uint32_t)(c / kGtcStages - 1) & 1u);
      unsigned char* hi = ring + (size_t)sidx * stage_bytes;
#pragma unroll
      for (int q = 0; q < kGtcEPW; ++q) {
        const int e = warp + kGtcPW * q;
        if (e >= k) break;   // warp-uniform
        float u[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (in_range) {
          float erx = cur.rx, ery = cur.ry;
          if (MODE == VBA_PIX_EDGE) {
            float rx1, ry1;
            load_rays<VBA_PIX_KF>(pix, ew[q], n & ~1, grid_w, gp, in, erx, ery, rx1, ry1);
            if (n & 1) { erx = rx1; ery = ry1; }
          }
          const EdgeGeo32 ge = load_geo<true>(reinterpret_cast<const EdgeGeo32*>(geos), e);
          const PxGeom o = project(ge, erx, ery, cur.d);
          const float w0 = o.valid ? cur.w[q].x : 0.f, w1 = o.valid ? cur.w[q].y : 0.f;
          const float jd0 = fmaf(o.x, ge.t[2], -ge.t[0]) * o.izh;
          const float jd1 = fmaf(o.y, ge.t[2], -ge.t[1]) * o.izh;
          const float c0w = w0 * fx2 * jd0 * sc, c1w = w1 * fy2 * jd1 * sc;
          const float xy = o.x * o.y;
          u[0] = fmaf(c0w, xy, c1w * fmaf(o.y, o.y, 1.f));
          u[1] = fmaf(c0w, -fmaf(o.x, o.x, 1.f), c1w * -xy);
          u[2] = fmaf(c0w, o.y, c1w * -o.x);
          u[3] = c0w * -o.iz;
          u[4] = c1w * -o.iz;
          u[5] = fmaf(c0w, o.x * o.iz, c1w * (o.y * o.iz));
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) put(hi, base[r] + 6144u * q, u[r]);
      }
      if (warp == 0) put(hi, goff, cur.g * sc);
      proxy_fence_shared();   // generic image writes -> tcgen05 reads
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&full[sidx]);
      cur = nxt;
    }
    // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 (accumulator rows),
    // column chunks of 32 split between warps w and w + 4; the lower 6x6 blocks
    // (e1 >= e2) and the b row are scattered into the partial's fp64 layout
    tc_mbar_wait(&accb, 0u);
    tc_fence_after();
    double* o = out + T.out;
    const int npairs = k * (k + 1) / 2;
    const int qr = warp & 3, half = warp >> 2, nhalf = kGtcPW / 4;
    auto cidx = [&](int a, int b) { const int e1 = a / 6, e2 = b / 6;
                                    return (e1 * (e1 + 1) / 2 + e2) * 36 + (a % 6) * 6 + (b % 6); };
    const int a0 = 32 * qr + lane;   // tile-0 row
    for (int cb = 32 * half; cb < N0; cb += 32 * nhalf) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * qr) << 16) + (uint32_t)cb, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int a = a0, b = cb + j;
        if (b >= M) continue;
        const double x = (double)v[j];
        if (a < nc) {
          if (b < nc) {
            if (b / 6 <= a / 6) o[cidx(a, b)] = x;
            if (b >= 128 && a / 6 <= b / 6) o[cidx(b, a)] = x;
          } else if (nc >= 128) {   // b == nc: row nc lies in tile 1, this is its column a
            o[npairs * 36 + a] = x;
          }
        } else if (a == nc && b < nc) {
          o[npairs * 36 + b] = x;
        }
      }
    }
    if (two) {
      const int a = 128 + a0;
      for (int cb = 32 * half; cb < N1; cb += 32 * nhalf) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * qr) << 16) + (uint32_t)(N0 + cb), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int b = 128 + cb + j;
          if (a >= M || b >= nc) continue;
          const double x = (double)v[j];
          if (a < nc) {
            if (b / 6 <= a / 6) o[cidx(a, b)] = x;
          } else {
            o[npairs * 36 + b] = x;
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == kGtcPW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kGtcTmemCols));
  }
}

void launch_gram_tc(int mode, const GramTile* gt, int ngt, size_t smem, int kmax, const DevState& s, const float* pix,
                    const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w, const double* grid,
                    const double* intr, const float* Hdd, const float* gd, double lam, double ridge,
                    double* gram_part, cudaStream_t st, const int32_t* order) {
  if (ngt <= 0) return;
  GridP gp{grid[0], grid[1], grid[2], grid[3]};
  IntrP in{intr[0], intr[1], intr[2], intr[3]};
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<ngt, kGtcThreads, smem, st>>>(gt, s.disp, s.geo32, pix, wts, eoff, doff, grid_w, gp, in, Hdd, gd, lam,
                                          ridge, kmax, gram_part, order);
  };
  if (mode == VBA_PIX_GRID) go(k_gram_tc<VBA_PIX_GRID>);
  else if (mode == VBA_PIX_KF) go(k_gram_tc<VBA_PIX_KF>);
  else go(k_gram_tc<VBA_PIX_EDGE>);
  launch_count();
}

// ---------------------------------------------------------------------------
// fill-in transform (fp64, one CTA per source): K-space Gram -> pose-space blocks
//   F_ii = sum_{e1,e2} G_{e1,i}^T C_{e1e2} G_{e2,i},  F_{i,j(e)} = -sum_{e1} G_{e1,i}^T C_{e1 e} G_{e,j}
//   F_{j(e1),j(e2)} = G_{e1,j}^T C_{e1e2} G_{e2,j},   gr_i = sum_e G_{e,i}^T b_e,  gr_{j(e)} = -G_{e,j}^T b_e
// layout: [F_ii 36][F_ij k*36][F_jj npairs*36][gr_i 6][gr_j k*6]
// ---------------------------------------------------------------------------
__device__ __forceinline__ double cblk(const double* C, int e1, int e2, int m, int b) {
  // C(e1,e2)[m][b] with only e1 >= e2 stored
  if (e1 >= e2) return C[(e1 * (e1 + 1) / 2 + e2) * 36 + m * 6 + b];
  return C[(e2 * (e2 + 1) / 2 + e1) * 36 + b * 6 + m];
}

// The source's Gram C (and b) is the fixed-order sum of its pixel-range partials,
// formed while staging it into shared memory (no separate reduction pass).
__global__ void k_fill_transform(const int32_t* __restrict__ srcs, const int32_t* __restrict__ seb,
                                 const int32_t* __restrict__ see, const int32_t* __restrict__ g0,
                                 const int32_t* __restrict__ g1, const GramTile* __restrict__ gt,
                                 const int64_t* __restrict__ foff, const double* __restrict__ part, int kmax,
                                 const double* __restrict__ geo64, Extr x, double* __restrict__ fill) {
  extern __shared__ double sm[];
  const int s = srcs[blockIdx.x];
  const int eb = seb[s], k = see[s] - eb;
  const int npairs = k * (k + 1) / 2;
  double* Gi = sm;
  double* Gj = Gi + kmax * 36;
  double* D = Gj + kmax * 36;
  double* Cs = D + kmax * 36;
  const double* C = Cs;
  if (k > 31) {   // one pixel range (its unit slices share the record): read it in place
    C = part + gt[g0[s]].out;
  } else {
    // four elements per thread per pass, their loads issued together (one element at a time
    // left one dependent global load in flight per thread: the staging dominated the kernel)
    const int len = npairs * 36 + 6 * k, t0 = g0[s], t1 = g1[s];
    const double* p0 = part + gt[t0].out;
    const int nth4 = 4 * blockDim.x;
    for (int i0 = threadIdx.x; i0 < len; i0 += nth4) {
      double acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * blockDim.x;
        acc[u] = i < len ? p0[i] : 0.0;
      }
      for (int t = t0 + 1; t < t1; ++t) {
        const double* pt = part + gt[t].out;
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * blockDim.x;
          v[u] = i < len ? pt[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += v[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < len) Cs[i] = acc[u];
      }
    }
  }
  const double* b = C + npairs * 36;
  double* o = fill + foff[s];
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int e = tid; e < k; e += nth) {
    const double* q = geo64 + (int64_t)kGeo64 * (eb + e);
    build_G(q, q + 18, q + 9, Gi + e * 36);
    build_G(x.RbcT, x.c2, q + 9, Gj + e * 36);
  }
  __syncthreads();
  // D_{e2} = sum_{e1} G_{e1,i}^T C(e1,e2): a thread per (e2, row a) computes the row's 6 entries
  for (int it = tid; it < k * 6; it += nth) {
    const int e2 = it / 6, a = it % 6;
    double r[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int e1 = 0; e1 < k; ++e1) {
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        const double g = Gi[e1 * 36 + m * 6 + a];
#pragma unroll
        for (int bc = 0; bc < 6; ++bc) r[bc] = fma(g, cblk(C, e1, e2, m, bc), r[bc]);
      }
    }
#pragma unroll
    for (int bc = 0; bc < 6; ++bc) D[e2 * 36 + a * 6 + bc] = r[bc];
  }
  __syncthreads();
  if (tid < 36) {
    const int a = tid / 6, bc = tid % 6;
    double acc = 0.0;
    for (int e = 0; e < k; ++e)
#pragma unroll
      for (int m = 0; m < 6; ++m) acc += D[e * 36 + a * 6 + m] * Gi[e * 36 + m * 6 + bc];
    o[tid] = acc;
  }
  for (int it = tid; it < k * 36; it += nth) {
    const int e = it / 36, a = (it % 36) / 6, bc = it % 6;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) acc += D[e * 36 + a * 6 + m] * Gj[e * 36 + m * 6 + bc];
    o[36 + it] = -acc;
  }
  // F_{j(e1) j(e2)} = G_{e1,j}^T C(e1,e2) G_{e2,j}: a thread per (pair, row a): row a of
  // T = G1^T C (6 x 6 MACs), then row a of T G2
  for (int it = tid; it < npairs * 6; it += nth) {
    const int p = it / 6, a = it % 6;
    int e1 = (int)((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
    while ((e1 + 1) * (e1 + 2) / 2 <= p) ++e1;
    while (e1 * (e1 + 1) / 2 > p) --e1;
    const int e2 = p - e1 * (e1 + 1) / 2;
    const double* Cb = C + p * 36;
    const double* G1 = Gj + e1 * 36;
    const double* G2 = Gj + e2 * 36;
    double t[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      const double g = G1[m * 6 + a];
#pragma unroll
      for (int l = 0; l < 6; ++l) t[l] = fma(g, Cb[m * 6 + l], t[l]);
    }
    double f[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < 6; ++l)
#pragma unroll
      for (int bc = 0; bc < 6; ++bc) f[bc] = fma(t[l], G2[l * 6 + bc], f[bc]);
#pragma unroll
    for (int bc = 0; bc < 6; ++bc) o[36 + k * 36 + p * 36 + a * 6 + bc] = f[bc];
  }
  const int goffs = 36 + k * 36 + npairs * 36;
  if (tid < 6) {
    double acc = 0.0;
    for (int e = 0; e < k; ++e)
#pragma unroll
      for (int m = 0; m < 6; ++m) acc += Gi[e * 36 + m * 6 + tid] * b[e * 6 + m];
    o[goffs + tid] = acc;
  }
  for (int it = tid; it < k * 6; it += nth) {
    const int e = it / 6, a = it % 6;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m) acc += Gj[e * 36 + m * 6 + a] * b[e * 6 + m];
    o[goffs + 6 + it] = -acc;
  }
}

void launch_fill_transform(const int32_t* srcs, int nsrc, const int32_t* seb, const int32_t* see,
                           const int32_t* g0, const int32_t* g1, const GramTile* gt, const int64_t* foff,
                           const double* part, const DevState& s, const Extr& x, double* fill, int kmax,
                           cudaStream_t st) {
  if (nsrc <= 0) return;
  const int ks = kmax < 31 ? kmax : 31;   // sources with more out-edges read their Gram in place
  const size_t smem = ((size_t)3 * kmax * 36 + (size_t)ks * (ks + 1) / 2 * 36 + 6 * ks) * sizeof(double);
  cudaFuncSetAttribute(k_fill_transform, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_fill_transform<<<nsrc, 512, smem, st>>>(srcs, seb, see, g0, g1, gt, foff, part, kmax, s.geo64, x, fill);
  launch_count();
}

// ---------------------------------------------------------------------------
// per-edge K-space step  u_e = G_{e,i} dx_i - G_{e,j} dx_j  (fp64 -> fp32)
// ---------------------------------------------------------------------------
__global__ void k_step_edges(const int32_t* __restrict__ ei, const int32_t* __restrict__ ej, int E,
                             const double* __restrict__ geo64, Extr x, const double* __restrict__ dx_full,
                             int sdof, float* __restrict__ ustep) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double* q = geo64 + (int64_t)kGeo64 * e;
  double Gi[36], Gj[36];
  build_G(q, q + 18, q + 9, Gi);
  build_G(x.RbcT, x.c2, q + 9, Gj);
  const double* di = dx_full + (int64_t)sdof * ei[e];
  const double* dj = dx_full + (int64_t)sdof * ej[e];
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 6; ++c) acc += Gi[r * 6 + c] * di[c] - Gj[r * 6 + c] * dj[c];
    ustep[e * 8 + r] = (float)acc;
  }
  ustep[e * 8 + 6] = 0.f;
  ustep[e * 8 + 7] = 0.f;
}

void launch_step_edges(const int32_t* ei, const int32_t* ej, int E, const DevState& s, const Extr& x,
                       const double* dx_full, int sdof, float* ustep, cudaStream_t st) {
  if (E <= 0) return;
  k_step_edges<<<(E + 127) / 128, 128, 0, st>>>(ei, ej, E, s.geo64, x, dx_full, sdof, ustep);
  launch_count();
}

// ---------------------------------------------------------------------------
// K6: disparity back-substitution + update (solver.py:290, 336-338)
//   dx_d = (-g_d - sum_e k_{n,e} . u_e) / Hdd_d,   d' = max(d + dx_d, 1e-4)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kPixBlock, 4) k_backsub(
    const PixTile* __restrict__ tiles, const float* __restrict__ disp, const EdgeGeo32* __restrict__ geo,
    const float* __restrict__ pix, const float* __restrict__ wts, const int64_t* __restrict__ eoff,
    const int64_t* __restrict__ doff, int grid_w, GridP gp, IntrP in, const float* __restrict__ Hdd,
    const float* __restrict__ gd, const float* __restrict__ ustep, double lam, double ridge,
    const double* __restrict__ disp64, float* __restrict__ disp_out, double* __restrict__ disp64_out,
    double* __restrict__ dxd_out, unsigned long long* __restrict__ step_bits) {
  const PixTile T = tiles[blockIdx.x];
  const int tid = threadIdx.x;
  const int64_t kbase = doff[T.src];
  const float fx2 = (float)in.fx * (float)in.fx, fy2 = (float)in.fy * (float)in.fy;
  float rx[2 * kTP], ry[2 * kTP], dd[2 * kTP], acc[2 * kTP];
  bool act[kTP];
#pragma unroll
  for (int m = 0; m < kTP; ++m) {
    const int p = m * kPixBlock + tid;
    const int n = T.n0 + 2 * p;
    act[m] = 2 * p < T.cnt;
    rx[2 * m] = ry[2 * m] = rx[2 * m + 1] = ry[2 * m + 1] = 0.f;
    dd[2 * m] = dd[2 * m + 1] = 1.f;
    acc[2 * m] = acc[2 * m + 1] = 0.f;
    if (act[m]) {
      const float2 d2 = __ldg(reinterpret_cast<const float2*>(disp + kbase + n));
      dd[2 * m] = d2.x;
      dd[2 * m + 1] = d2.y;
      if (MODE != VBA_PIX_EDGE)
        load_rays<MODE>(pix, kbase, n, grid_w, gp, in, rx[2 * m], ry[2 * m], rx[2 * m + 1], ry[2 * m + 1]);
    }
  }
  // the tile's out-edge geometry and K-space steps, staged once (read every edge by all threads)
  __shared__ float4 sgeo[64 * 4];
  __shared__ float4 sstep[64 * 2];
  // the weight rows of each out-edge (8 B per pixel, contiguous) stream through a 3-stage ring
  // of bulk copies issued by thread 0, kBsStages edges ahead of the arithmetic
  constexpr int kBsStages = 3;
  __shared__ __align__(16) float4 wring[kBsStages][kTile / 2];
  __shared__ __align__(8) unsigned long long wfull[kBsStages];
  const int ne = T.ee - T.eb;
  const uint32_t wbytes = (uint32_t)T.cnt * 8u;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int q) {   // edge T.eb + q -> stage q % kBsStages
    const int sidx = q % kBsStages;
    mbar_expect_tx(&wfull[sidx], wbytes);
    bulk_g2s(wring[sidx], wts + 2 * (eoff[T.eb + q] + T.n0), wbytes, &wfull[sidx], pol);
  };
  for (int i = tid; i < 4 * ne; i += kPixBlock) sgeo[i] = __ldg(reinterpret_cast<const float4*>(geo + T.eb) + i);
  for (int i = tid; i < 2 * ne; i += kPixBlock) sstep[i] = __ldg(reinterpret_cast<const float4*>(ustep + 8 * T.eb) + i);
  if (tid == 0) {
    for (int q = 0; q < kBsStages; ++q) mbar_init(&wfull[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kBsStages && q < ne; ++q) issue(q);
  }
  __syncthreads();
  for (int e = T.eb; e < T.ee; ++e) {
    const int q = e - T.eb, sidx = q % kBsStages;
    const EdgeGeo32 g = load_geo<true>(reinterpret_cast<const EdgeGeo32*>(sgeo), q);
    const float4 ua = sstep[2 * q];
    const float2 ub = make_float2(sstep[2 * q + 1].x, sstep[2 * q + 1].y);
    const int64_t rbase = eoff[e] + T.n0;
    mbar_wait(&wfull[sidx], (uint32_t)(q / kBsStages) & 1u);
    float4 wc[kTP];
#pragma unroll
    for (int m = 0; m < kTP; ++m) wc[m] = act[m] ? wring[sidx][m * kPixBlock + tid] : make_float4(0.f, 0.f, 0.f, 0.f);
    // the stage is consumed (values in registers): refill it once every thread has read it
    // (a CTA barrier measured faster here than K1's per-warp release counter)
    __syncthreads();
    if (tid == 0 && q + kBsStages < ne) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(q + kBsStages);
    }
#pragma unroll
    for (int m = 0; m < kTP; ++m) {
      const int p = m * kPixBlock + tid;
      const float4 ww = wc[m];
      if (act[m]) {
        if (MODE == VBA_PIX_EDGE)
          load_rays<VBA_PIX_KF>(pix, rbase - T.n0, T.n0 + 2 * p, grid_w, gp, in, rx[2 * m], ry[2 * m],
                                rx[2 * m + 1], ry[2 * m + 1]);
      }
      // the pixel pair in packed fp32 (FFMA2/FMUL2), the same operations as project() and
      // the scalar coupling per lane
      const float2 rxp = make_float2(rx[2 * m], rx[2 * m + 1]), ryp = make_float2(ry[2 * m], ry[2 * m + 1]);
      const float2 d = make_float2(dd[2 * m], dd[2 * m + 1]);
      const float2 Dx = FMA2(d, S2(g.t[0]), FMA2(S2(g.M[0]), rxp, FMA2(S2(g.M[1]), ryp, S2(g.M[2]))));
      const float2 Dy = FMA2(d, S2(g.t[1]), FMA2(S2(g.M[3]), rxp, FMA2(S2(g.M[4]), ryp, S2(g.M[5]))));
      const float2 Dz = FMA2(d, S2(g.t[2]), FMA2(S2(g.M[6]), rxp, FMA2(S2(g.M[7]), ryp, S2(g.M[8]))));
      const float2 Xz = ADD2(S2(1.0f), Dz);
      const float2 th = MUL2(S2(1e-6f), d);
      const bool va = Xz.x > th.x, vb = Xz.y > th.y;
      float2 izh = make_float2(va ? rcp_approx(Xz.x) : 0.f, vb ? rcp_approx(Xz.y) : 0.f);
      izh = FMA2(izh, FMA2(-Xz, izh, S2(1.0f)), izh);
      const float2 ddx = MUL2(FMA2(-rxp, Dz, Dx), izh);
      const float2 ddy = MUL2(FMA2(-ryp, Dz, Dy), izh);
      const float2 x = ADD2(rxp, ddx), y = ADD2(ryp, ddy), iz = MUL2(d, izh);
      const float2 w0 = make_float2(va ? ww.x : 0.f, vb ? ww.z : 0.f);
      const float2 w1 = make_float2(va ? ww.y : 0.f, vb ? ww.w : 0.f);
      const float2 jd0 = MUL2(FMA2(x, S2(g.t[2]), S2(-g.t[0])), izh);
      const float2 jd1 = MUL2(FMA2(y, S2(g.t[2]), S2(-g.t[1])), izh);
      const float2 c0w = MUL2(MUL2(w0, S2(fx2)), jd0), c1w = MUL2(MUL2(w1, S2(fy2)), jd1);
      const float2 xy = MUL2(x, y);
      // k_{n,e} . u_e
      float2 sv = MUL2(S2(ua.x), FMA2(c0w, xy, MUL2(c1w, FMA2(y, y, S2(1.f)))));
      sv = FMA2(S2(ua.y), FMA2(c0w, -FMA2(x, x, S2(1.f)), MUL2(c1w, -xy)), sv);
      sv = FMA2(S2(ua.z), FMA2(c0w, y, MUL2(c1w, -x)), sv);
      sv = FMA2(S2(ua.w), MUL2(c0w, -iz), sv);
      sv = FMA2(S2(ub.x), MUL2(c1w, -iz), sv);
      sv = FMA2(S2(ub.y), FMA2(c0w, MUL2(x, iz), MUL2(c1w, MUL2(y, iz))), sv);
      acc[2 * m] += sv.x;
      acc[2 * m + 1] += sv.y;
    }
  }
  double mx = 0.0;
  const double damp = 1.0 + lam;
#pragma unroll
  for (int m = 0; m < kTP; ++m) {
    if (!act[m]) continue;
    const int64_t n = kbase + T.n0 + 2 * (m * kPixBlock + tid);
    const float2 h2 = *reinterpret_cast<const float2*>(Hdd + n);
    const float2 g2 = *reinterpret_cast<const float2*>(gd + n);
    const double dx0 = (-(double)g2.x - (double)acc[2 * m]) / ((double)h2.x * damp + ridge);
    const double dx1 = (-(double)g2.y - (double)acc[2 * m + 1]) / ((double)h2.y * damp + ridge);
    // fp64 master update d' = max(d + dx_d, 1e-4) (solver.py:336-338); the kernels read its fp32 copy
    const double2 d64 = *reinterpret_cast<const double2*>(disp64 + n);
    const double n0v = fmax(d64.x + dx0, kDispFloor64), n1v = fmax(d64.y + dx1, kDispFloor64);
    *reinterpret_cast<double2*>(disp64_out + n) = make_double2(n0v, n1v);
    *reinterpret_cast<float2*>(disp_out + n) = make_float2((float)n0v, (float)n1v);
    if (dxd_out) *reinterpret_cast<double2*>(dxd_out + n) = make_double2(dx0, dx1);
    mx = fmax(mx, fmax(fabs(dx0), fabs(dx1)));
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0 && mx > 0.0)
    atomicMax(step_bits, (unsigned long long)__double_as_longlong(mx));   // max is order-independent
}

void launch_backsub(int mode, const PixTile* tiles, int ntiles, const DevState& cur, const DevState& nxt,
                    const float* pix, const float* wts, const int64_t* eoff, const int64_t* doff, int grid_w,
                    const double* grid, const double* intr, const float* Hdd, const float* gd, const float* ustep,
                    double lam, double ridge, double* dxd_out, unsigned long long* step_bits, cudaStream_t st) {
  if (ntiles <= 0) return;
  GridP gp{grid[0], grid[1], grid[2], grid[3]};
  IntrP in{intr[0], intr[1], intr[2], intr[3]};
  if (mode == VBA_PIX_GRID)
    k_backsub<VBA_PIX_GRID><<<ntiles, kPixBlock, 0, st>>>(tiles, cur.disp, cur.geo32, pix, wts, eoff, doff, grid_w,
                                                          gp, in, Hdd, gd, ustep, lam, ridge, cur.disp64, nxt.disp, nxt.disp64, dxd_out,
                                                          step_bits);
  else if (mode == VBA_PIX_KF)
    k_backsub<VBA_PIX_KF><<<ntiles, kPixBlock, 0, st>>>(tiles, cur.disp, cur.geo32, pix, wts, eoff, doff, grid_w,
                                                        gp, in, Hdd, gd, ustep, lam, ridge, cur.disp64, nxt.disp, nxt.disp64, dxd_out,
                                                        step_bits);
  else
    k_backsub<VBA_PIX_EDGE><<<ntiles, kPixBlock, 0, st>>>(tiles, cur.disp, cur.geo32, pix, wts, eoff, doff, grid_w,
                                                          gp, in, Hdd, gd, ustep, lam, ridge, cur.disp64, nxt.disp, nxt.disp64, dxd_out,
                                                          step_bits);
  launch_count();
}

// ---------------------------------------------------------------------------
// retraction of keyframe states and gravity (solver.py:326-341, residuals.py:44-52,
// geometry.py:221-223, residuals.py:132-134); frozen keyframes copied bitwise.
// ---------------------------------------------------------------------------
__global__ void k_retract(const double* __restrict__ cur, double* __restrict__ nxt, const double* __restrict__ dx,
                          const int32_t* __restrict__ frozen, int K, int sdof, int ngrav, int n_state,
                          const double* __restrict__ gcur, double* __restrict__ gnxt,
                          unsigned long long* __restrict__ step_bits, int npv) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  // max |dx_full| over this thread's slice (sdof entries; the last thread also the
  // gravity columns), then a warp max and one integer atomicMax per warp (the bit
  // patterns of non-negative doubles order like the values: order-independent)
  double mx = 0.0;
  if (n < K)
    for (int k = 0; k < sdof; ++k) mx = fmax(mx, fabs(dx[(int64_t)sdof * n + k]));
  if (n == K)
    for (int i = n_state; i < npv; ++i) mx = fmax(mx, fabs(dx[i]));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(step_bits, (unsigned long long)__double_as_longlong(mx));
  if (n < K) {
    const double* s = cur + 16 * n;
    double* o = nxt + 16 * n;
    const double* d = dx + (int64_t)sdof * n;
    if (frozen[n]) {
#pragma unroll
      for (int k = 0; k < 16; ++k) o[k] = s[k];
    } else {
      double qe[4], qn[4];
      qexp(d, qe);
      qmul(s, qe, qn);
      qcanon(qn);
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = qn[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) o[4 + k] = s[4 + k] + d[3 + k];
      if (sdof == 15) {
#pragma unroll
        for (int k = 0; k < 9; ++k) o[7 + k] = s[7 + k] + d[6 + k];
      } else {
#pragma unroll
        for (int k = 0; k < 9; ++k) o[7 + k] = s[7 + k];
      }
    }
  }
  if (n == K) {  // gravity
    for (int k = 0; k < 5; ++k) gnxt[k] = gcur[k];
    if (ngrav) {
      const double w[3] = {dx[n_state], dx[n_state + 1], 0.0};   // GRAVITY_TANGENT_BASIS @ dg
      double qe[4], qn[4];
      qexp(w, qe);
      qmul(gcur, qe, qn);
      qcanon(qn);
      for (int k = 0; k < 4; ++k) gnxt[k] = qn[k];
    }
  }
}

void launch_retract(const DevState& cur, const DevState& nxt, const double* dx_full, const int32_t* frozen, int K,
                    int sdof, int ngrav, int n_state, unsigned long long* step_bits, int npv, cudaStream_t st) {
  k_retract<<<(K + 1 + 127) / 128, 128, 0, st>>>(cur.state, nxt.state, dx_full, frozen, K, sdof, ngrav, n_state,
                                                 cur.grav, nxt.grav, step_bits, npv);
  launch_count();
}

// ---------------------------------------------------------------------------
// export of the dense pose-disparity coupling H_pd (reference layout,
// solver.py:209-213): column = real disparity index, rows = 6 pose columns of
// the source and of every edge target.  Test/diagnostic path only.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void k_export_hpd(const int32_t* __restrict__ seb, const int32_t* __restrict__ see,
                             const int64_t* __restrict__ doff, const int64_t* __restrict__ roff,
                             const int32_t* __restrict__ npix, const int32_t* __restrict__ ej, int K,
                             const float* __restrict__ disp, const EdgeGeo32* __restrict__ geo,
                             const double* __restrict__ geo64, Extr x, const float* __restrict__ pix,
                             const float* __restrict__ wts, const int64_t* __restrict__ eoff, int grid_w, GridP gp,
                             IntrP in, HpdOut out) {
  const int src = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (src >= K || n >= npix[src]) return;
  const int64_t kbase = doff[src];
  const int64_t col = out.base + roff[src] + n;
  const float fx2 = (float)in.fx * (float)in.fx, fy2 = (float)in.fy * (float)in.fy;
  const float d = disp[kbase + n];
  // pose row of keyframe k, entry a: reference layout k*sdof + a, or the free layout (frozen -> skip)
  auto prow = [&](int k, int a) -> int64_t {
    if (!out.colmap) return (int64_t)k * out.sdof + a;
    return out.colmap[k] < 0 ? -1 : (int64_t)out.colmap[k] + a;
  };
  double hi[6] = {0, 0, 0, 0, 0, 0};
  for (int e = seb[src]; e < see[src]; ++e) {
    float rx, ry, rx1, ry1;
    if (MODE == VBA_PIX_EDGE) load_rays<VBA_PIX_KF>(pix, eoff[e], n & ~1, grid_w, gp, in, rx, ry, rx1, ry1);
    else load_rays<MODE>(pix, kbase, n & ~1, grid_w, gp, in, rx, ry, rx1, ry1);
    if (n & 1) { rx = rx1; ry = ry1; }
    const EdgeGeo32 g = load_geo(geo, e);
    const PxGeom o = project(g, rx, ry, d);
    const float2 w = __ldg(reinterpret_cast<const float2*>(wts + 2 * (eoff[e] + n)));
    const float w0 = o.valid ? w.x : 0.f, w1 = o.valid ? w.y : 0.f;
    const float jd0 = fmaf(o.x, g.t[2], -g.t[0]) * o.izh;
    const float jd1 = fmaf(o.y, g.t[2], -g.t[1]) * o.izh;
    const float c0w = w0 * fx2 * jd0, c1w = w1 * fy2 * jd1;
    const float xy = o.x * o.y;
    float u[6];
    u[0] = fmaf(c0w, xy, c1w * fmaf(o.y, o.y, 1.f));
    u[1] = fmaf(c0w, -fmaf(o.x, o.x, 1.f), c1w * -xy);
    u[2] = fmaf(c0w, o.y, c1w * -o.x);
    u[3] = c0w * -o.iz;
    u[4] = c1w * -o.iz;
    u[5] = fmaf(c0w, o.x * o.iz, c1w * (o.y * o.iz));
    double Gi[36], Gj[36];
    const double* q = geo64 + (int64_t)kGeo64 * e;
    build_G(q, q + 18, q + 9, Gi);
    build_G(x.RbcT, x.c2, q + 9, Gj);
    const int j = ej[e];
    for (int a = 0; a < 6; ++a) {
      double si = 0.0, sj = 0.0;
      for (int m = 0; m < 6; ++m) {
        si += Gi[m * 6 + a] * (double)u[m];
        sj += Gj[m * 6 + a] * (double)u[m];
      }
      hi[a] += si;
      const int64_t r = prow(j, a);
      if (r >= 0) out.H[r * out.ld + col] -= sj;
    }
  }
  for (int a = 0; a < 6; ++a) {
    const int64_t r = prow(src, a);
    if (r >= 0) out.H[r * out.ld + col] += hi[a];
  }
  if (out.Hdd) {   // dense system: damped disparity diagonal and right-hand side (solver.py:292-301)
    out.H[col * out.ld + col] = (double)out.Hdd[kbase + n] * (1.0 + out.lam) + out.ridge;
    out.rhs[col] = -(double)out.gd[kbase + n];
  }
}

void launch_export_hpd(int mode, const int32_t* seb, const int32_t* see, const int64_t* doff, const int64_t* roff,
                       const int32_t* npix, int maxpix, const int32_t* ej, int K, const DevState& s, const Extr& x,
                       const float* pix, const float* wts, const int64_t* eoff, int grid_w, const double* grid,
                       const double* intr, const HpdOut& out, cudaStream_t st) {
  if (K <= 0 || maxpix <= 0) return;
  GridP gp{grid[0], grid[1], grid[2], grid[3]};
  IntrP in{intr[0], intr[1], intr[2], intr[3]};
  dim3 grd((maxpix + 127) / 128, K);   // one source per grid row; a pixel's edges are serial in its thread
  if (mode == VBA_PIX_GRID)
    k_export_hpd<VBA_PIX_GRID><<<grd, 128, 0, st>>>(seb, see, doff, roff, npix, ej, K, s.disp, s.geo32, s.geo64, x,
                                                    pix, wts, eoff, grid_w, gp, in, out);
  else if (mode == VBA_PIX_KF)
    k_export_hpd<VBA_PIX_KF><<<grd, 128, 0, st>>>(seb, see, doff, roff, npix, ej, K, s.disp, s.geo32, s.geo64, x,
                                                  pix, wts, eoff, grid_w, gp, in, out);
  else
    k_export_hpd<VBA_PIX_EDGE><<<grd, 128, 0, st>>>(seb, see, doff, roff, npix, ej, K, s.disp, s.geo32, s.geo64, x,
                                                    pix, wts, eoff, grid_w, gp, in, out);
  launch_count();
}

// padded per-keyframe fp32 / fp64 array -> reference-order fp64 array
template <class T>
__global__ void k_unpad(const T* __restrict__ src, const int64_t* __restrict__ doff,
                        const int64_t* __restrict__ roff, const int32_t* __restrict__ npix, int K,
                        double* __restrict__ dst) {
  const int k = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K || n >= npix[k]) return;
  dst[roff[k] + n] = (double)src[doff[k] + n];
}

void launch_unpad(const float* src, const int64_t* doff, const int64_t* roff, const int32_t* npix, int maxpix, int K,
                  double* dst, cudaStream_t st) {
  if (K <= 0 || maxpix <= 0) return;
  dim3 grd((maxpix + 255) / 256, K);
  k_unpad<float><<<grd, 256, 0, st>>>(src, doff, roff, npix, K, dst);
  launch_count();
}

void launch_unpad(const double* src, const int64_t* doff, const int64_t* roff, const int32_t* npix, int maxpix,
                  int K, double* dst, cudaStream_t st) {
  if (K <= 0 || maxpix <= 0) return;
  dim3 grd((maxpix + 255) / 256, K);
  k_unpad<double><<<grd, 256, 0, st>>>(src, doff, roff, npix, K, dst);
  launch_count();
}

// energy = sum over vision tiles (fixed order) + sum over IMU factors (fixed order)
__global__ void k_energy_reduce(const double* __restrict__ te, int nt, const double* __restrict__ ib, int F,
                                int ibs, int eoff, double* __restrict__ out) {
  // both sums as strided per-thread partials + fixed-order warp / block trees (deterministic)
  __shared__ double red[2][32];
  double v = 0.0, u = 0.0;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) v += te[i];
  for (int f = threadIdx.x; f < F; f += blockDim.x) u += ib[(int64_t)f * ibs + eoff];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    u += __shfl_xor_sync(0xffffffffu, u, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = v;
    red[1][threadIdx.x >> 5] = u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, si = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      s += red[0][w];
      si += red[1][w];
    }
    out[0] = s + si;
    out[1] = s;
    out[2] = si;
  }
}

void launch_energy_reduce(const double* te, int nt, const double* ib, int F, int ibs, int eoff, double* out3,
                          cudaStream_t st) {
  k_energy_reduce<<<1, 1024, 0, st>>>(te, nt, ib, F, ibs, eoff, out3);
  launch_count();
}

}  // namespace vba
