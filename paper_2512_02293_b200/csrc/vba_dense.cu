// vba_dense.cu — reduced-system assembly and the dense fp64 Cholesky solve (sm_100a).
//
// Replaces the freeze / damp / Schur / np.linalg.solve sequence of
// solver.py:254-290 (/root/reference/pkg/src/vislam/):
//   H_red = damp(H_ff) - F,  g_red = g_f - g_F,  H_red dx_f = -g_red
// The assembly gathers per-block contribution lists (built once per solve by
// the host planner) in a fixed order, so the result is bitwise deterministic.
// The solve is a right-looking blocked Cholesky (64x64 tiles, fp64 FMA) on a
// column-major, tile-padded matrix with the right-hand side carried as an
// augmented column (forward substitution during the factorisation), followed
// by a tiled backward substitution.  A non-positive pivot sets *status
// (host maps it to the reference's "singular reduced pose system" retry).
#include <cuda_runtime.h>

#include "vba_internal.cuh"

namespace vba {

// ---------------------------------------------------------------------------
// assembly: one CTA per lower block (a >= b) of the block matrix
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_assemble(const int32_t* __restrict__ bptr, const int32_t* __restrict__ bnff,
                                                  const Contrib* __restrict__ cs, int nbr,
                                                  const int32_t* __restrict__ roff, const int32_t* __restrict__ rdim,
                                                  const double* __restrict__ arena, double lam, double ridge,
                                                  int add_ridge, double* __restrict__ H, int64_t ld, int sym,
                                                  const int32_t* __restrict__ blist) {
  const int64_t id = blist ? blist[blockIdx.x] : blockIdx.x;   // blist: blocks with contributions
  // block (a, b) of the packed lower index, decoded once per CTA (an fp64 sqrt per thread
  // was a fifth of the kernel's instructions)
  __shared__ int ab[2];
  if (threadIdx.x == 0) {
    int a0 = (int)((sqrtf(8.f * (float)id + 1.f) - 1.f) * 0.5f);
    while ((int64_t)(a0 + 1) * (a0 + 2) / 2 <= id) ++a0;
    while ((int64_t)a0 * (a0 + 1) / 2 > id) --a0;
    ab[0] = a0;
    ab[1] = (int)(id - (int64_t)a0 * (a0 + 1) / 2);
  }
  __syncthreads();
  const int a = ab[0], b = ab[1];
  const int ra = rdim[a], cb = rdim[b];
  // sym bit 0: also write the upper triangle; bit 1: skip the Schur fill-in contributions
  const int p0 = bptr[id], pf = p0 + bnff[id], p1 = (sym & 2) ? pf : bptr[id + 1];
  const double damp = 1.0 + lam;
  for (int t = threadIdx.x; t < ra * cb; t += blockDim.x) {
    const int r = t % ra, c = t / ra;
    double v = 0.0;
    for (int p = p0; p < pf; ++p) {
      const Contrib C = cs[p];
      if (r < C.rows && c < C.cols)
        v += (double)C.sign * arena[C.off + (C.trans ? (int64_t)c * C.ld + r : (int64_t)r * C.ld + c)];
    }
    if (a == b && r == c) {
      v = v * damp;
      if (add_ridge) v += ridge;
    }
    for (int p = pf; p < p1; ++p) {
      const Contrib C = cs[p];
      if (r < C.rows && c < C.cols)
        v += (double)C.sign * arena[C.off + (C.trans ? (int64_t)c * C.ld + r : (int64_t)r * C.ld + c)];
    }
    const int64_t gr = roff[a] + r, gc = roff[b] + c;
    H[gc * ld + gr] = v;
    if (sym & 1) H[gr * ld + gc] = v;
  }
}

void launch_assemble(const int32_t* bptr, const int32_t* bnff, const Contrib* cs, int nbr, const int32_t* roff,
                     const int32_t* rdim, const double* arena, double lam, double ridge, int add_ridge, double* H,
                     int64_t ld, int sym, cudaStream_t st, const int32_t* blist, int nblist) {
  const int64_t nblk = blist ? (int64_t)nblist : (int64_t)nbr * (nbr + 1) / 2;
  if (nblk <= 0) return;
  k_assemble<<<(unsigned)nblk, 128, 0, st>>>(bptr, bnff, cs, nbr, roff, rdim, arena, lam, ridge, add_ridge, H, ld,
                                             sym, blist);
  launch_count();
}

__global__ void k_assemble_vec(const int32_t* __restrict__ sptr, const Vec* __restrict__ vs,
                               const int32_t* __restrict__ soff, const int32_t* __restrict__ sdim,
                               const double* __restrict__ arena, double scale, int skip_fill,
                               double* __restrict__ g) {
  const int a = blockIdx.x, r = threadIdx.x;
  if (r >= sdim[a]) return;
  double v = 0.0;
  for (int p = sptr[a]; p < sptr[a + 1]; ++p) {
    const Vec V = vs[p];
    if (skip_fill && V.sign < 0) continue;   // fill-in contributions are the negative ones
    if (r < V.len) v += (double)V.sign * arena[V.off + r];
  }
  g[soff[a] + r] = scale * v;
}

void launch_assemble_vec(const int32_t* sptr, const Vec* vs, int nseg, const int32_t* soff, const double* arena,
                         double scale, double* g, cudaStream_t st, int skip_fill) {
  // soff[nseg .. 2*nseg) holds the segment dims
  if (nseg <= 0) return;
  k_assemble_vec<<<nseg, 32, 0, st>>>(sptr, vs, soff, soff + nseg, arena, scale, skip_fill, g);
  launch_count();
}

// dense (use_schur=False) path: disparity update from the full solution x[nf + real index]
__global__ void k_dense_dxd(const double* __restrict__ x, int nf, const int64_t* __restrict__ doff,
                            const int64_t* __restrict__ roff, const int32_t* __restrict__ npix, int K,
                            const double* __restrict__ dcur, float* __restrict__ dnxt, double* __restrict__ dnxt64,
                            double* __restrict__ dxd, unsigned long long* __restrict__ step_bits) {
  const int k = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K || n >= npix[k]) return;
  const double dx = x[nf + roff[k] + n];
  const int64_t p = doff[k] + n;
  const double v = fmax(dcur[p] + dx, kDispFloor64);   // solver.py:336-338, fp64 master
  dnxt64[p] = v;
  dnxt[p] = (float)v;
  dxd[p] = dx;
  const double m = fabs(dx);
  if (m > 0.0) atomicMax(step_bits, (unsigned long long)__double_as_longlong(m));
}

void launch_dense_dxd(const double* x, int nf, const int64_t* doff, const int64_t* roff, const int32_t* npix,
                      int maxpix, int K, const DevState& cur, const DevState& nxt, double* dxd,
                      unsigned long long* step_bits, cudaStream_t st) {
  if (K <= 0 || maxpix <= 0) return;
  dim3 g((maxpix + 255) / 256, K);
  k_dense_dxd<<<g, 256, 0, st>>>(x, nf, doff, roff, npix, K, cur.disp64, nxt.disp, nxt.disp64, dxd, step_bits);
  launch_count();
}

__global__ void k_widen(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (double)a[i];
}
__global__ void k_narrow(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}
void launch_widen(const float* src, double* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_widen<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, n);
  launch_count();
}
void launch_narrow(const double* src, float* dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_narrow<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, n);
  launch_count();
}

// full symmetric row-major copy of the lower triangle (column-major, leading dim ld) of
// the n x n reduced system, and g = scale * rhs (export of H_red / g_red for parity tests)
__global__ void k_export_sym(const double* __restrict__ H, int64_t ld, int n, double* __restrict__ out,
                             const double* __restrict__ rhs, double scale, double* __restrict__ g) {
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const int lo = r > c ? c : r, hi = r > c ? r : c;
    out[(int64_t)r * n + c] = H[(int64_t)lo * ld + hi];
  }
  if (threadIdx.x == 0 && g) g[r] = scale * rhs[r];
}
void launch_export_sym(const double* H, int64_t ld, int n, double* out, const double* rhs, double scale, double* g,
                       cudaStream_t st) {
  if (n <= 0) return;
  k_export_sym<<<n, 256, 0, st>>>(H, ld, n, out, rhs, scale, g);
  launch_count();
}

// identity padding of the tile-padded matrix (rows/cols n..npad) and zero rhs padding
__global__ void k_pad_identity(double* H, int64_t ld, int n, int npad, double* rhs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)npad * (npad - n);
  if (i >= tot) return;
  const int c = n + (int)(i / npad), r = (int)(i % npad);
  const double v = (r == c) ? 1.0 : 0.0;
  H[(int64_t)c * ld + r] = v;   // padded columns
  H[(int64_t)r * ld + c] = v;   // padded rows
  if (r == c && rhs) rhs[c] = 0.0;
}
void launch_pad_identity(double* H, int64_t ld, int n, int npad, double* rhs, cudaStream_t st) {
  if (npad <= n) return;
  const int64_t tot = (int64_t)npad * (npad - n);
  k_pad_identity<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(H, ld, n, npad, rhs);
  launch_count();
}

// ---------------------------------------------------------------------------
// Cholesky

// dx_full[n*sdof + r] from the free-layout solution (zeros at frozen keyframes)
__global__ void k_scatter_dx(const double* __restrict__ x, const int32_t* __restrict__ fmap, int npv,
                             double* __restrict__ dx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npv) dx[i] = fmap[i] >= 0 ? x[fmap[i]] : 0.0;
}
void launch_scatter_dx(const double* x, const int32_t* fmap, int npv, double* dx, cudaStream_t st) {
  if (npv <= 0) return;
  k_scatter_dx<<<(npv + 255) / 256, 256, 0, st>>>(x, fmap, npv, dx);
  launch_count();
}

// Batched segment copy (vba_copy_segments): one CTA per segment, 16-byte vectors when
// source, destination and length allow, else 4-byte words, else bytes.
__global__ void k_copy_segments(const vba_copy_seg* __restrict__ segs) {
  const vba_copy_seg g = segs[blockIdx.x];
  const uintptr_t a = (uintptr_t)g.src | (uintptr_t)g.dst | (uintptr_t)g.bytes;
  if ((a & 15) == 0) {
    const int4* s = reinterpret_cast<const int4*>(g.src);
    int4* d = reinterpret_cast<int4*>(g.dst);
    for (int64_t i = threadIdx.x; i < g.bytes / 16; i += blockDim.x) d[i] = s[i];
  } else if ((a & 3) == 0) {
    const int* s = reinterpret_cast<const int*>(g.src);
    int* d = reinterpret_cast<int*>(g.dst);
    for (int64_t i = threadIdx.x; i < g.bytes / 4; i += blockDim.x) d[i] = s[i];
  } else {
    const char* s = reinterpret_cast<const char*>(g.src);
    char* d = reinterpret_cast<char*>(g.dst);
    for (int64_t i = threadIdx.x; i < g.bytes; i += blockDim.x) d[i] = s[i];
  }
}
void launch_copy_segments(const vba_copy_seg* segs, int n, cudaStream_t st) {
  k_copy_segments<<<n, 256, 0, st>>>(segs);
  launch_count();
}

}  // namespace vba
