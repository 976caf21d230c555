// vba_chol.cu — dense fp64 Cholesky solve of the reduced system as ONE persistent
// kernel executing a tile-task DAG (sm_100a).
//
// Replaces np.linalg.solve(Hred, -gred) of solver.py:287 (/root/reference/pkg/src/vislam/)
// for the symmetric positive-definite damped Schur complement.  The matrix is
// column-major with 128x128 tiles; tasks (built once per solve on the host):
//
//   POTRF(k)      factor the diagonal tile, write L_kk^-1 to a side buffer,
//                 forward-substitute y_k = L_kk^-1 rhs_k
//   TRSM(i,k)     L_ik = A_ik L_kk^-T  (a GEMM with the inverse), rhs_i -= L_ik y_k
//   GEMM(i,j,k)   A_ij -= L_ik L_jk^T  (SYRK when i == j)
//   BUPD(j,k)     p_jk = L_kj^T x_k                (backward substitution, j < k)
//   BSOL(k)       x_k = L_kk^-T (y_k - sum_k' p_kk')
//
// GEMM-shaped tasks run on the fp64 tensor cores (mma.sync m8n8k4 f64, DMMA)
// with cp.async double-buffered operand chunks.  Persistent CTAs (one per SM,
// all co-resident) take tasks in a topological order with lookahead (the next
// panel column is updated and factored before the rest of the trailing
// update) and wait on per-tile counters: upd[i][j] = updates applied,
// done[i][j] = tile final.  Matrix data written inside the kernel is only read
// through L2 (.cg), so no stale L1 lines are observed.  A non-positive pivot
// sets *status (mapped to the reference's "singular reduced pose system").
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <tuple>

#include "vba_internal.cuh"
#include "vba_tc.cuh"

namespace vba {

constexpr int CT = 128;          // tile size
constexpr int KC = 32;           // K chunk per pipeline stage
constexpr int SP = CT + 4;       // smem column stride (doubles): conflict-free fragment loads
constexpr int CHOL_THREADS = 256;
constexpr int SB = 36;           // 32x32 block stride in POTRF (doubles, = 4 mod 16)
constexpr size_t CHOL_SMEM = (size_t)2 * 2 * KC * SP * sizeof(double);   // 2 stages x (A, B)

enum TaskType { T_POTRF = 0, T_TRSM = 1, T_GEMM = 2, T_BUPD = 3, T_BSOL = 4, T_DIAG = 5, T_CHAIN = 6, T_TILE = 7, T_CONV = 8, T_PREP = 9 };
// TILE task modes (CholTask::expect): the chain's SYRK target (W written, upd = columns),
// the chain's TRSM operand (W and its hi/lo images written, upd = columns + 1), or an
// off-chain tile whose TRSM follows in the same task (done = 1)
enum TileMode { TILE_SYRK_TARGET = 0, TILE_TRSM = 1, TILE_OPERAND = 2 };

struct CholTask {
  int32_t type, i, j, k;
  int32_t expect;   // updates expected on the target tile before this task (envelope-ready)
  int32_t k2;       // GEMM: second update column applied in the same task (-1: none)
  int32_t pad[2];
};

// ---------------------------------------------------------------------------
// low-level helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void stcg(double* p, double v) { __stcg(p, v); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// wait until *flag >= want (one thread), then CTA barrier
__device__ __forceinline__ void wait_geq(const int* flag, int want) {
  if (threadIdx.x == 0) {
    int ns = 32;
    while (ld_acquire(flag) < want) {
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
    }
  }
}

// ---------------------------------------------------------------------------
// GEMM core: acc(c, r) = sum_m opA(c, m) * opB(r, m) over m in [0, CT)
//   opA / opB: 128x128 column-major tiles (element (row, m) at base[m*lda + row])
// Warp w owns rows c in [64*(w%2), +64) and r in [32*(w/2), +32): 8 x 4 DMMA tiles.
// acc[mt][nt][0/1] = (c = 64wm + 8mt + lane/4, r = 32wn + 8nt + 2*(lane%4) + {0,1})
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_chunk(double* sA, double* sB, const double* A, int64_t lda, const double* B,
                                           int64_t ldb, int m0) {
  // each operand chunk: 128 rows x KC cols -> smem [KC][SP]; 16-byte cp.async of 2 rows
  for (int t = threadIdx.x; t < KC * (CT / 2); t += CHOL_THREADS) {
    const int m = t / (CT / 2), r2 = (t % (CT / 2)) * 2;
    cp_async16(sA + m * SP + r2, A + (int64_t)(m0 + m) * lda + r2);
    cp_async16(sB + m * SP + r2, B + (int64_t)(m0 + m) * ldb + r2);
  }
  cp_async_commit();
}

__device__ __forceinline__ void gemm_tile(double* smem, const double* A, int64_t lda, const double* B, int64_t ldb,
                                          double (&acc)[8][4][2], bool zero = true) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wm = w & 1, wn = w >> 1;
  // stage s: A at smem + s*2*KC*SP, B right after it (arithmetic, no pointer arrays)
  if (zero) {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  }
  load_chunk(smem, smem + KC * SP, A, lda, B, ldb, 0);
  const int ar = 64 * wm + (lane >> 2), br = 32 * wn + (lane >> 2), kq = lane & 3;
#pragma unroll 1
  for (int kc = 0; kc < CT / KC; ++kc) {
    const int s = kc & 1;
    if (kc + 1 < CT / KC) {
      double* nxt = smem + (s ^ 1) * 2 * KC * SP;
      load_chunk(nxt, nxt + KC * SP, A, lda, B, ldb, (kc + 1) * KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* pa = smem + s * 2 * KC * SP;
    const double* pb = pa + KC * SP;
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const int m = ks * 4 + kq;
      double af[8], bf[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = pa[m * SP + ar + 8 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = pb[m * SP + br + 8 * b];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// tasks
// ---------------------------------------------------------------------------
struct CholArgs {
  double* A;
  int64_t ld;
  int nt;
  double* rhs;       // [nt*CT]   in: -g_red, out: y (forward-substituted)
  double* x;         // [nt*CT]   solution
  double* Linv;      // [nt][CT*CT] column-major inverses of the diagonal factors
  double* part;      // [nt][nt][CT] backward-substitution partials
  int* upd;          // [nt*nt]
  int* done;         // [nt*nt]
  int* bcnt;         // [nt]  BUPD tasks completed for row block j
  int* counter;      // task dispenser
  const CholTask* tasks;
  int ntasks;
  int* status;
  unsigned long long* trace;   // optional [ntasks][4]: t_grab, t_ready, t_done, smid
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double* tile(const CholArgs& a, int i, int j) {
  return a.A + (int64_t)j * CT * a.ld + (int64_t)i * CT;
}

// Warp-synchronous Cholesky + inverse of a 32x32 SPD block: lane r holds row r
// of the block (a[]) and of the identity (m[]); 32 right-looking steps with
// shuffles.  On return the block (column-major, stride sw) holds L and Ib
// (column-major 32x32) holds L^-1.  Non-positive pivot -> *bad.
// CTA-wide Cholesky + inverse of a 32x32 SPD block held in shared memory
// (column-major, stride sw): right-looking elimination of [W | I] with all 256
// threads (thread = (row r, column group cg), 4 columns each), two barriers per
// step.  On return W holds L (lower) and Ib (column-major, stride SB) L^-1.
__device__ __forceinline__ void cta_potrf32(double* W, int sw, double* Ib, int* bad) {
  const int tid = threadIdx.x, r = tid & 31, cg = tid >> 5;   // 4 columns per thread: c = cg + 8q
#pragma unroll
  for (int q = 0; q < 4; ++q) Ib[(cg + 8 * q) * SB + r] = (cg + 8 * q == r) ? 1.0 : 0.0;
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    __syncthreads();                                   // updates of step j-1 complete
    double piv = W[j * sw + j];
    if (!(piv > 0.0)) {
      if (tid == 0) *bad = 1;
      piv = 1.0;
    }
    const double inv = rsqrt(piv);
    __syncthreads();                                   // every thread has read the pivot
    if (cg == 0) {                                     // column j of L
      if (r > j) W[j * sw + r] *= inv;
      else if (r == j) W[j * sw + j] = piv * inv;
    } else if (cg == 1 && r <= j) {                    // row j of L^-1
      Ib[r * SB + j] *= inv;
    }
    __syncthreads();
    if (r > j) {
      // all loads first (independent), then the updates: no aliasing-serialised RMW chains
      const double lr = W[j * sw + r];
      double cur[4], piv4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = cg + 8 * q;
        double* dst = (c > j) ? &W[c * sw + r] : &Ib[c * SB + r];
        cur[q] = *dst;
        piv4[q] = (c > j) ? W[j * sw + c] : Ib[c * SB + j];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = cg + 8 * q;
        if (c <= r) {
          double* dst = (c > j) ? &W[c * sw + r] : &Ib[c * SB + r];
          *dst = cur[q] - lr * piv4[q];
        }
      }
    }
  }
  __syncthreads();
}

// Shared-memory DMMA GEMM for the in-tile block work of POTRF:
//   C(M x N) = beta*C + alpha * A(M x K) * op(B)
//   A(m, k) at A[k*lda + m];  BT: op(B)(k, n) = B(n, k) at B[k*ldb + n];  !BT: (k, n) at B[n*ldb + k]
//   C(m, n) at C[n*ldc + m].  M, N multiples of 8, K of 4; strides = 4 mod 16 (conflict-free).
//   lower: skip 8x8 output tiles strictly above the diagonal.
// Warps take 8x8 output tiles two at a time (two independent DMMA chains).
template <bool BT>
__device__ __forceinline__ void sgemm8(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int M,
                                       int N, int K, double alpha, bool beta, bool lower) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tm = M >> 3, nt = tm * (N >> 3);
  const int am = lane >> 2, ak = lane & 3;
  for (int t = warp; t < nt; t += 16) {
    const int t2 = t + 8;
    const int bi0 = t % tm, bj0 = t / tm;
    const bool v1 = t2 < nt;
    const int bi1 = v1 ? t2 % tm : bi0, bj1 = v1 ? t2 / tm : bj0;
    const bool on0 = !(lower && bj0 > bi0), on1 = v1 && !(lower && bj1 > bi1);
    double c00 = 0, c01 = 0, c10 = 0, c11 = 0;
    for (int k = 0; k < K; k += 4) {
      const double a0 = A[(k + ak) * lda + bi0 * 8 + am];
      const double a1 = A[(k + ak) * lda + bi1 * 8 + am];
      const double b0 = BT ? B[(k + ak) * ldb + bj0 * 8 + am] : B[(bj0 * 8 + am) * ldb + k + ak];
      const double b1 = BT ? B[(k + ak) * ldb + bj1 * 8 + am] : B[(bj1 * 8 + am) * ldb + k + ak];
      dmma(c00, c01, a0, b0);
      dmma(c10, c11, a1, b1);
    }
    const int r = am, cc = 2 * ak;
    if (on0) {
      double* p = C + (bj0 * 8 + cc) * ldc + bi0 * 8 + r;
      p[0] = (beta ? p[0] : 0.0) + alpha * c00;
      p[ldc] = (beta ? p[ldc] : 0.0) + alpha * c01;
    }
    if (on1) {
      double* p = C + (bj1 * 8 + cc) * ldc + bi1 * 8 + r;
      p[0] = (beta ? p[0] : 0.0) + alpha * c10;
      p[ldc] = (beta ? p[ldc] : 0.0) + alpha * c11;
    }
  }
}

constexpr int SW = CT + 4;        // POTRF tile stride (doubles, = 4 mod 16)
constexpr int TB = 100;           // TRSM temporary stride (96 rows)
constexpr size_t POTRF_SMEM = (size_t)(CT * SW + 8 * 32 * SB) * sizeof(double);
constexpr size_t DAG_SMEM = POTRF_SMEM > CHOL_SMEM ? POTRF_SMEM : CHOL_SMEM;

// POTRF(k): blocked (4 panels of 32) factorisation of the diagonal tile in shared
// memory.  Per panel: warp-synchronous factor + inverse of the 32x32 diagonal
// block, in-tile TRSM of the rows below, SYRK of the trailing lower triangle.
// Then M = L^-1 by block forward substitution, written to the side buffer, and
// the forward substitution y_k = M rhs_k.
__device__ void task_potrf(const CholArgs& a, int k, double* smem) {
  double* W = smem;                      // 128 x 128 column-major (stride SW), lower part used
  double* I = smem + CT * SW;            // 4 blocks: L_pp^-1 (stride SB)
  double* Mc = I + 4 * 32 * SB;          // 4 blocks: column p of M (rows i >= p), or the TRSM temp (stride TB)
  __shared__ double ys[CT];
  __shared__ int bad;
  const int tid = threadIdx.x;
  const double* Ak = tile(a, k, k);
  if (tid == 0) bad = 0;
  // async tile load (all loads in flight at once; no register staging)
  for (int t = tid; t < CT * (CT / 2); t += CHOL_THREADS) {
    const int r2 = (t % (CT / 2)) * 2, c = t / (CT / 2);
    cp_async16(W + c * SW + r2, Ak + (int64_t)c * a.ld + r2);
  }
  cp_async_commit();
  if (tid < CT) ys[tid] = ldcg(a.rhs + (int64_t)k * CT + tid);
  cp_async_wait<0>();
  __syncthreads();
  unsigned long long* ph = a.trace ? a.trace + 4 * (size_t)a.ntasks + 16 * (size_t)k : nullptr;   // phase stamps
  if (ph && tid == 0) ph[0] = gtimer();
  for (int p = 0; p < 4; ++p) {
    const int c0 = 32 * p, r0 = c0 + 32, nr = CT - r0;
    cta_potrf32(W + c0 * SW + c0, SW, I + p * 32 * SB, &bad);
    if (ph && tid == 0) ph[1 + 2 * p] = gtimer();
    if (nr > 0) {
      // TRSM: X = W[r0:, c0:c0+32] * Ip^T   (Ip(c, m) at I[m*SB + c])
      sgemm8<true>(W + c0 * SW + r0, SW, I + p * 32 * SB, SB, Mc, TB, nr, 32, 32, 1.0, false, false);
      __syncthreads();
      for (int t = tid; t < nr * 32; t += CHOL_THREADS) {
        const int r = t % nr, c = t / nr;
        W[(c0 + c) * SW + r0 + r] = Mc[c * TB + r];
      }
      __syncthreads();
      // SYRK: W[r0:, r0:] -= X X^T   (lower 8x8 tiles)
      sgemm8<true>(W + c0 * SW + r0, SW, W + c0 * SW + r0, SW, W + r0 * SW + r0, SW, nr, nr, 32, -1.0, true, true);
      __syncthreads();
    }
    if (ph && tid == 0) ph[2 + 2 * p] = gtimer();
  }
  if (tid == 0 && bad) atomicExch(a.status, 1);
  // M = L^-1 by column blocks:  M_pp = I_p,  M_ip = -I_i sum_{m=p}^{i-1} L_im M_mp;
  // each finished column block goes to the side buffer and into y = M rhs.
  double* Li = a.Linv + (int64_t)k * CT * CT;
  double yacc = 0.0;   // thread r < CT accumulates y_r
  for (int p = 0; p < 4; ++p) {
    for (int i = p + 1; i < 4; ++i) {
      double* T = Mc + i * 32 * SB;
      for (int m = p; m < i; ++m) {
        const double* Mmp = (m == p) ? I + p * 32 * SB : Mc + m * 32 * SB;
        sgemm8<false>(W + (32 * m) * SW + 32 * i, SW, Mmp, SB, T, SB, 32, 32, 32, 1.0, m != p, false);
        __syncthreads();
      }
      // M_ip = -I_i T on the tensor cores into the free slot Mc[p], then copied over T
      double* tmp = Mc + p * 32 * SB;
      sgemm8<false>(I + i * 32 * SB, SB, T, SB, tmp, SB, 32, 32, 32, -1.0, false, false);
      __syncthreads();
      {
        const int r = tid & 31, cq = tid >> 5;
#pragma unroll
        for (int q = 0; q < 4; ++q) T[(cq + 8 * q) * SB + r] = tmp[(cq + 8 * q) * SB + r];
      }
      __syncthreads();
    }
    // write column block p and accumulate y
    for (int t = tid; t < CT * 32; t += CHOL_THREADS) {
      const int r = t % CT, c = t / CT, i = r >> 5;
      double v = 0.0;
      if (i == p) v = I[p * 32 * SB + c * SB + (r & 31)];
      else if (i > p) v = Mc[i * 32 * SB + c * SB + (r & 31)];
      stcg(Li + (int64_t)(32 * p + c) * CT + r, v);
    }
    if (tid < CT) {
      const int r = tid, i = r >> 5;
      if (i >= p) {
        const double* blk = (i == p) ? I + p * 32 * SB : Mc + i * 32 * SB;
        for (int c = 0; c < 32; ++c) yacc += blk[c * SB + (r & 31)] * ys[32 * p + c];
      }
    }
    __syncthreads();
  }
  if (tid < CT) stcg(a.rhs + (int64_t)k * CT + tid, yacc);
  if (ph && tid == 0) ph[9] = gtimer();
}

// TRSM(i,k): L_ik = A_ik Linv^T ; rhs_i -= L_ik y_k
__device__ void task_trsm(const CholArgs& a, int i, int k, double* smem) {
  double acc[8][4][2];
  double* Aik = tile(a, i, k);
  const double* Li = a.Linv + (int64_t)k * CT * CT;
  // acc(c, r) = sum_m Linv(c, m) * A_ik(r, m)  ==  L_ik(r, c)
  gemm_tile(smem, Li, CT, Aik, a.ld, acc);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wm = w & 1, wn = w >> 1;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int c = 64 * wm + 8 * mt + (lane >> 2);
      const int r = 32 * wn + 8 * nt + 2 * (lane & 3);
      double* p = Aik + (int64_t)c * a.ld + r;
      __stcg(reinterpret_cast<double2*>(p), make_double2(acc[mt][nt][0], acc[mt][nt][1]));
    }
  __threadfence();
  __syncthreads();
  // rhs_i -= L_ik y_k   (two threads per row, loads batched 16 at a time)
  __shared__ double yk[CT];
  if (threadIdx.x < CT) yk[threadIdx.x] = ldcg(a.rhs + (int64_t)k * CT + threadIdx.x);
  __syncthreads();
  {
    const int r = threadIdx.x >> 1, h = threadIdx.x & 1;
    double s = 0.0;
#pragma unroll 16
    for (int c = h; c < CT; c += 2) s += ldcg(Aik + (int64_t)c * a.ld + r) * yk[c];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (h == 0) {
      double* ri = a.rhs + (int64_t)i * CT + r;
      stcg(ri, ldcg(ri) - s);
    }
  }
}

// GEMM(i,j,k[,k2]): A_ij -= L_ik L_jk^T (+ L_ik2 L_jk2^T), one read-modify-write of A_ij
__device__ void task_gemm(const CholArgs& a, int i, int j, int k, int k2, double* smem) {
  double acc[8][4][2];
  // acc(c, r) = sum_m L_jk(c, m) L_ik(r, m) = (L_ik L_jk^T)(r, c)
  gemm_tile(smem, tile(a, j, k), a.ld, tile(a, i, k), a.ld, acc);
  if (k2 >= 0) gemm_tile(smem, tile(a, j, k2), a.ld, tile(a, i, k2), a.ld, acc, false);
  double* C = tile(a, i, j);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wm = w & 1, wn = w >> 1;
  // read-modify-write in two batches of 16 independent loads (L2 latency overlapped)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double2 v[4][4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 64 * wm + 8 * (4 * h + mt) + (lane >> 2);
        const int r = 32 * wn + 8 * nt + 2 * (lane & 3);
        v[mt][nt] = __ldcg(reinterpret_cast<const double2*>(C + (int64_t)c * a.ld + r));
      }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 64 * wm + 8 * (4 * h + mt) + (lane >> 2);
        const int r = 32 * wn + 8 * nt + 2 * (lane & 3);
        double2 o = v[mt][nt];
        o.x -= acc[4 * h + mt][nt][0];
        o.y -= acc[4 * h + mt][nt][1];
        __stcg(reinterpret_cast<double2*>(C + (int64_t)c * a.ld + r), o);
      }
  }
}

// BUPD(j,k): part[j][k] = L_kj^T x_k
__device__ void task_bupd(const CholArgs& a, int j, int k) {
  __shared__ double xs[CT];
  const double* Lkj = tile(a, k, j);
  if (threadIdx.x < CT) xs[threadIdx.x] = ldcg(a.x + (int64_t)k * CT + threadIdx.x);
  __syncthreads();
  // warp per column: lanes read 4 x 32 consecutive rows (coalesced), then warp-reduce
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 2
  for (int c = warp; c < CT; c += CHOL_THREADS / 32) {
    const double* col = Lkj + (int64_t)c * a.ld;
    double s = ldcg(col + lane) * xs[lane] + ldcg(col + 32 + lane) * xs[32 + lane] +
               ldcg(col + 64 + lane) * xs[64 + lane] + ldcg(col + 96 + lane) * xs[96 + lane];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) stcg(a.part + ((int64_t)j * a.nt + k) * CT + c, s);
  }
}

// BSOL(k): x_k = Linv_k^T (y_k - sum_{k'>k} part[k][k'])
__device__ void task_bsol(const CholArgs& a, int k) {
  __shared__ double ys[CT];
  const int tid = threadIdx.x;
  if (tid < CT) {
    double v = ldcg(a.rhs + (int64_t)k * CT + tid);
#pragma unroll 8
    for (int kk = k + 1; kk < a.nt; ++kk) v -= ldcg(a.part + ((int64_t)k * a.nt + kk) * CT + tid);
    ys[tid] = v;
  }
  __syncthreads();
  {   // x_k(c) = sum_{r >= c} Linv(r, c) y'(r): warp per column, coalesced
    const int lane = tid & 31, warp = tid >> 5;
    for (int c = warp; c < CT; c += CHOL_THREADS / 32) {
      const double* Li = a.Linv + (int64_t)k * CT * CT + (int64_t)c * CT;   // Linv zero above the diagonal
      double s = ldcg(Li + lane) * ys[lane] + ldcg(Li + 32 + lane) * ys[32 + lane] +
                 ldcg(Li + 64 + lane) * ys[64 + lane] + ldcg(Li + 96 + lane) * ys[96 + lane];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) stcg(a.x + (int64_t)k * CT + c, s);
    }
  }
}

__global__ void __launch_bounds__(CHOL_THREADS, 1) k_chol_dag(CholArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int tsk;
  const int nt = a.nt;
  while (true) {
    if (threadIdx.x == 0) tsk = atomicAdd(a.counter, 1);
    __syncthreads();
    const int t = tsk;
    __syncthreads();
    if (t >= a.ntasks) break;
    const CholTask T = a.tasks[t];
    unsigned long long t0 = 0;
    if (a.trace && threadIdx.x == 0) t0 = gtimer();
    switch (T.type) {
      case T_POTRF:
        wait_geq(&a.upd[T.k * nt + T.k], T.expect);
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[4 * t + 1] = gtimer();
        task_potrf(a, T.k, smem);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release(&a.done[T.k * nt + T.k], 1);
        break;
      case T_TRSM:
        wait_geq(&a.done[T.k * nt + T.k], 1);
        wait_geq(&a.upd[T.i * nt + T.k], T.expect);
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[4 * t + 1] = gtimer();
        task_trsm(a, T.i, T.k, smem);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release(&a.done[T.i * nt + T.k], 1);
        break;
      case T_GEMM:
        wait_geq(&a.done[T.i * nt + T.k], 1);
        wait_geq(&a.done[T.j * nt + T.k], 1);
        if (T.k2 >= 0) {
          wait_geq(&a.done[T.i * nt + T.k2], 1);
          wait_geq(&a.done[T.j * nt + T.k2], 1);
        }
        wait_geq(&a.upd[T.i * nt + T.j], T.expect);
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[4 * t + 1] = gtimer();
        task_gemm(a, T.i, T.j, T.k, T.k2, smem);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release(&a.upd[T.i * nt + T.j], T.expect + (T.k2 >= 0 ? 2 : 1));
        break;
      case T_BUPD:
        wait_geq(&a.done[T.k * nt + T.k], 2);        // x_k solved (BSOL sets done[k][k] = 2)
        wait_geq(&a.done[T.k * nt + T.j], 1);
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[4 * t + 1] = gtimer();
        task_bupd(a, T.j, T.k);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(&a.bcnt[T.j], 1);
        break;
      case T_BSOL:
        wait_geq(&a.done[T.k * nt + T.k], 1);
        wait_geq(&a.bcnt[T.k], T.expect);
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[4 * t + 1] = gtimer();
        task_bsol(a, T.k);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release(&a.done[T.k * nt + T.k], 2);
        break;
    }
    if (a.trace && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      a.trace[4 * t + 0] = t0;
      a.trace[4 * t + 2] = gtimer();
      a.trace[4 * t + 3] = smid;
    }
  }
}

// ---------------------------------------------------------------------------
// host side: task list (dense, lookahead 1) and launch
// ---------------------------------------------------------------------------
size_t chol_task_bytes() { return sizeof(CholTask); }

int chol_plan_tasks(int nt, void* outv, int cap) {
  CholTask* out = reinterpret_cast<CholTask*>(outv);
  int n = 0;
  auto push = [&](int type, int i, int j, int k, int expect, int k2 = -1) {
    if (n < cap) out[n] = CholTask{type, i, j, k, expect, k2, {0, 0}};
    ++n;
  };
  if (nt <= 0) return 0;
  // Lookahead-1 order.  Tile (i,j) receives updates k = 0..j-1: the last one
  // (k = j-1, the next panel column) is a single high-priority task; the earlier
  // ones are merged statically in pairs (0,1), (2,3), ... (a lone last one when
  // j-2 is even), placed at the step of their second column.  Static pairing keeps
  // the summation order — and the result — bitwise reproducible.
  push(T_POTRF, 0, 0, 0, 0);
  for (int i = 1; i < nt; ++i) push(T_TRSM, i, 0, 0, 0);
  for (int s = 0; s + 1 < nt; ++s) {
    for (int i = s + 1; i < nt; ++i) push(T_GEMM, i, s + 1, s, s);      // next panel column first
    push(T_POTRF, s + 1, s + 1, s + 1, s + 1);
    for (int i = s + 2; i < nt; ++i) push(T_TRSM, i, s + 1, s + 1, s + 1);
    for (int j = s + 2; j < nt; ++j)
      for (int i = j; i < nt; ++i) {
        if (s & 1) push(T_GEMM, i, j, s - 1, s - 1, s);                  // pair (s-1, s)
        else if (s == j - 2) push(T_GEMM, i, j, s, s);                   // lone last non-critical update
      }
  }
  for (int k = nt - 1; k >= 0; --k) {
    push(T_BSOL, k, k, k, nt - 1 - k);
    for (int j = 0; j < k; ++j) push(T_BUPD, j, j, k, 0);
  }
  return n;
}

// Task list of the tensor-core DAG: as chol_plan_tasks, but the critical chain of
// each step -- POTRF(k), TRSM(k+1,k), GEMM(k+1,k+1,k) -- is one DIAG(k) task run
// back to back by one CTA (no flag hand-offs or task grabs between them), and
// there is no substitution (the triangular solves are separate kernels).
int chol_plan_tasks_tc(int nt, void* outv, int cap) {
  CholTask* out = reinterpret_cast<CholTask*>(outv);
  int n = 0;
  auto push = [&](int type, int i, int j, int k, int expect) {
    if (n < cap) out[n] = CholTask{type, i, j, k, expect, -1, {0, 0}};
    ++n;
  };
  if (nt <= 0) return 0;
  // Left-looking: the chain task, then one TILE task per off-chain lower tile in the order
  // the chain needs them.  At "step" s: the chain's TRSM operand (s+2, s+1) and SYRK target
  // (s+2, s+2) of step s+1, then the tiles of column s+1 (each accumulating columns 0..s and
  // applying its TRSM once the chain publishes Linv_{s+1}), the one feeding step s+2's
  // operand first.  TILE fields: k = number of columns accumulated, expect = TILE_* mode.
  // (Right-looking orders with per-update GEMM tasks left the chain waiting 6-41 us per step
  // in the first third -- each update re-read and re-wrote its fp32 tile through L2.)
  push(T_CHAIN, 0, 0, 0, 0);
  if (nt > 1) push(T_TILE, 1, 0, 0, TILE_OPERAND);
  for (int i = 2; i < nt; ++i) push(T_TRSM, i, 0, 0, 0);
  for (int s = 0; s + 2 < nt; ++s) {
    push(T_TILE, s + 2, s + 1, s + 1, TILE_OPERAND);
    push(T_TILE, s + 2, s + 2, s + 1, TILE_SYRK_TARGET);
    for (int i = s + 3; i < nt; ++i) push(T_TILE, i, s + 1, s + 1, TILE_TRSM);
  }
  for (int k = 0; k < nt; ++k) push(T_CONV, k, k, k, 0);   // fp32 Linv_kk, L_{k+1,k} for the solves
  // the triangular solves' folded matrices (kinds 0-4 of tc_task_prep), each as soon as its
  // tiles are final: overlapped with the end of the chain instead of a kernel after it
  for (int k = 0; k < nt; ++k)
    for (int kind = 0; kind < 5; ++kind)
      if (!((kind == 1 && k < 1) || (kind == 2 && k < 2) || (kind == 3 && k + 1 >= nt) || (kind == 4 && k + 2 >= nt)))
        push(T_PREP, k, kind, k, 0);
  return n;
}

// Launch with every CTA guaranteed co-resident (cooperative launch).  The DAG Cholesky
// kernels and the triangular-solve chains hand work between CTAs through flags in global
// memory, so a CTA that never got an SM would leave the others spinning (e.g. next to other
// work on the GPU); a grid that cannot be co-resident fails the launch (reported as
// VBA_E_CUDA by the caller's error check) instead of hanging.
template <class... KArgs, class... Args>
static void launch_coresident(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3((unsigned)block);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaLaunchKernelEx(&lc, k, args...);
}

size_t chol_smem_bytes() { return CHOL_SMEM; }

int chol_dag_launch(double* A, int64_t ld, int nt, double* rhs, double* x, double* Linv, double* part, int* flags,
                    const void* tasks, int ntasks, int* status, cudaStream_t st, unsigned long long* trace) {
  if (nt <= 0) return 0;
  static int grid = 0;
  if (grid == 0) {
    cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DAG_SMEM);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_dag, CHOL_THREADS, DAG_SMEM);
    grid = sms * (per > 0 ? per : 1);
  }
  // flags: upd[nt*nt] done[nt*nt] bcnt[nt] counter[1]
  cudaMemsetAsync(flags, 0, sizeof(int) * ((size_t)2 * nt * nt + nt + 1), st);
  CholArgs a;
  a.A = A;
  a.ld = ld;
  a.nt = nt;
  a.rhs = rhs;
  a.x = x;
  a.Linv = Linv;
  a.part = part;
  a.upd = flags;
  a.done = flags + (size_t)nt * nt;
  a.bcnt = flags + (size_t)2 * nt * nt;
  a.counter = flags + (size_t)2 * nt * nt + nt;
  a.tasks = reinterpret_cast<const CholTask*>(tasks);
  a.ntasks = ntasks;
  a.status = status;
  a.trace = trace;
  const int g = ntasks < grid ? ntasks : grid;
  launch_coresident(k_chol_dag, g, CHOL_THREADS, DAG_SMEM, st, a);
  launch_count();
  return 0;
}

}  // namespace vba

namespace vba {
void chol_task_fields5(const void* tasks, int n, int* out5) {
  const CholTask* t = reinterpret_cast<const CholTask*>(tasks);
  for (int q = 0; q < n; ++q) {
    out5[5 * q + 0] = t[q].type;
    out5[5 * q + 1] = t[q].i;
    out5[5 * q + 2] = t[q].j;
    out5[5 * q + 3] = t[q].k;
    out5[5 * q + 4] = t[q].expect;
  }
}
void chol_task_fields(const void* tasks, int n, int* out4) {
  const CholTask* t = reinterpret_cast<const CholTask*>(tasks);
  for (int q = 0; q < n; ++q) {
    out4[4 * q + 0] = t[q].type;
    out4[4 * q + 1] = t[q].i;
    out4[4 * q + 2] = t[q].j;
    out4[4 * q + 3] = t[q].k;
  }
}
}  // namespace vba

namespace vba {

// ===========================================================================
// Mixed-precision SPD solve on the 5th-gen tensor cores (tcgen05, kind::f16).
//
// A tile DAG on a Jacobi-scaled fp32 copy of the lower triangle:
//   As = D H D,  D = diag(H)^-1/2      (the scaling makes cond(As) ~1e4 here)
// one chain task (POTRF -> TRSM -> SYRK of every step, one CTA) and left-looking tile
// tasks (each off-chain tile accumulates all its updates in TMEM and is written once,
// then its TRSM follows), claimed in list order by persistent co-resident CTAs.  Tile
// products split every fp32 operand into fp16 hi + lo (A B^T ~ Ah Bh^T + Ah Bl^T + Al Bh^T,
// fp32 accumulation in TMEM), so the factor has ~fp32 accuracy at tensor-core speed.  The
// fp64 answer of np.linalg.solve (solver.py:287) is then recovered by iterative refinement
// against the fp64 H:  x += D (L L^T)^-1 D (b - H x)   (fp64 residuals).
//
// Tile storage (nt x nt lower tiles, linear index i(i+1)/2 + j):
//   W    fp32 row-major 128x128: working tile; after the factorisation
//        L_ij (i > j) and L_kk^-1 (diagonal) for the triangular solves
//   IMG  per tile two operand images (fp16 hi, lo) in the UMMA canonical K-major
//        SWIZZLE_128B layout: 2 K-chunks of 64 fp16 x 128 rows (16 KB each),
//        8-row atoms of 1 KB, 16-byte units XOR-swizzled by (row mod 8); a
//        chunk is one contiguous cp.async.bulk into shared memory.
// ===========================================================================

constexpr int TKC = 32;                       // 4-byte words per chunk row (one 128-B swizzle row = 64 fp16)
constexpr int TNCH = CT / (2 * TKC);          // 2 K-chunks of 64 per tile
constexpr uint32_t TCHUNK = CT * TKC * 4;     // 16 KB
constexpr int TC_STAGES = 3;
constexpr uint32_t TSTAGE = 4 * TCHUNK;       // A_hi A_lo B_hi B_lo
constexpr size_t TC_RING = (size_t)TC_STAGES * TSTAGE;
// epilogue staging (fp32 128 x 132, padded rows) after the 4 hi/lo chunk images of a TRSM result
constexpr size_t TC_EPI_OFF = (size_t)8 * TCHUNK;
constexpr size_t TC_EPI_END = TC_EPI_OFF + (size_t)CT * (CT + 4) * 4;
constexpr size_t TC_SMEM_0 = TC_RING > POTRF_SMEM ? TC_RING : POTRF_SMEM;
// the chain's TRSM A operand (W_{k+1,k} hi/lo images, 64 KB), prefetched while POTRF(k) runs:
// above POTRF's two 128 x 132 fp32 tiles (Ws, Xf: 135 KB)
constexpr size_t TC_ABUF_OFF = (size_t)136 * 1024;
constexpr size_t TC_ABUF_END = TC_ABUF_OFF + (size_t)4 * TCHUNK;
constexpr size_t TC_SMEM_1 = TC_SMEM_0 > TC_EPI_END ? TC_SMEM_0 : TC_EPI_END;
constexpr size_t TC_SMEM = (TC_SMEM_1 > TC_ABUF_END ? TC_SMEM_1 : TC_ABUF_END) + 1024;
constexpr int64_t TILE_F = (int64_t)CT * CT;  // floats per tile (= the two fp16 image parts of a tile)
constexpr int64_t IMGP_F = TILE_F / 2;        // one fp16 image part, in 4-byte words
// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t tc_idesc(int n) {   // D f32, A/B f16 (format 0), both K-major, M = 128
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(CT >> 4) << 24);
}
constexpr uint32_t TC_IDESC = tc_idesc(CT);        // M = N = 128
constexpr uint32_t TC_IDESC2 = tc_idesc(2 * CT);   // M = 128, N = 256
// The accumulator spans 256 TMEM columns: 3xTF32 is issued as
//   D[:, 0:256] (+)= A_hi [B_hi; B_lo]^T   (one N = 256 MMA: B_lo is stored right after B_hi)
//   D[:, 0:128]  += A_lo B_hi^T
// and the epilogue adds the two 128-column halves (an N = 256 MMA costs one N = 128
// MMA's issue slot twice over, measured: 130 vs 3 x 97-130 cycles per K-step).
constexpr int TC_TMEM_COLS = 2 * CT;

struct TcArgs {
  float* W;           // [ntl][CT*CT]
  float* img;         // [ntl][2][CT*CT]
  int nt;
  int* upd;
  int* done;
  int* counter;
  const CholTask* tasks;
  int ntasks;
  int* status;
  unsigned long long* trace;   // optional [ntasks][4]: t_grab, t_ready, t_done, smid
  float* Fm;                   // folded solve matrices (PREP tasks)
  int* convd;                  // [nt]: CONV(k) has written its fp32 tiles
};
__device__ void tc_task_prep(const TcArgs& a, int k, int kind, float* A, float* B);

__device__ __forceinline__ int64_t tlin(int i, int j) { return (int64_t)i * (i + 1) / 2 + j; }
// fp16 offset of element (row r, col c) inside one image part (see layout above):
// 64-column K-chunks, 8-row atoms of 1 KB, 16-byte units (8 fp16) XOR-swizzled by row
__device__ __forceinline__ int img_off(int r, int c) {
  const int q = c >> 6, e = c & 63, u = e >> 3;
  return q * (CT * 64) + (r >> 3) * 512 + (r & 7) * 64 + ((u ^ (r & 7)) << 3) + (e & 7);
}
// x = hi + lo with hi, lo fp16 (2 x 11 significant bits; the Jacobi-scaled factors are
// O(1), well inside the fp16 range): 4 values -> 4 hi + 4 lo halves (8 B each)
__device__ __forceinline__ void split4_h(const float4 x, uint2& hi, uint2& lo) {
  const __half h0 = __float2half_rn(x.x), h1 = __float2half_rn(x.y), h2 = __float2half_rn(x.z),
               h3 = __float2half_rn(x.w);
  const __half l0 = __float2half_rn(x.x - __half2float(h0)), l1 = __float2half_rn(x.y - __half2float(h1)),
               l2 = __float2half_rn(x.z - __half2float(h2)), l3 = __float2half_rn(x.w - __half2float(h3));
  hi.x = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
  hi.y = (uint32_t)__half_as_ushort(h2) | ((uint32_t)__half_as_ushort(h3) << 16);
  lo.x = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
  lo.y = (uint32_t)__half_as_ushort(l2) | ((uint32_t)__half_as_ushort(l3) << 16);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc,
                                       uint32_t idesc = TC_IDESC) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(acc), "r"(idesc));
}
// one K-step (8 tf32) of 3xTF32 into the 256-column accumulator; b_hi is followed by b_lo
__device__ __forceinline__ void tc_mma3(uint32_t tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi, bool first) {
  tc_mma(tmem, tc_sdesc(a_hi), tc_sdesc(b_hi), first ? 0u : 1u, TC_IDESC2);
  tc_mma(tmem, tc_sdesc(a_lo), tc_sdesc(b_hi), 1u, TC_IDESC);
}
// columns c .. c+31 of the 3xTF32 result: accumulator columns c and c + 128 summed
__device__ __forceinline__ void tmem_ld_sum(uint32_t taddr, float* v) {
  float u[32];
  tmem_ld32(taddr, v);
  tmem_ld32(taddr + CT, u);
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] += u[k];
}

// Coalesced epilogue.  The accumulator comes out of TMEM as rows per lane
// (32x32b shape: lane = tile row), which would make every lane touch its own
// 512-B row in global memory; it is staged through a padded shared-memory tile
// (row stride CT + 4 floats: conflict-free both ways) and global memory is read
// and written a full 512-B row per warp instruction.  Thread (w, lane) owns rows
// 16 w .. 16 w + 15, float4 column `lane`.
constexpr int EPS = CT + 4;
__device__ __forceinline__ void tc_epi_prefetch(const float* Cg, float4 (&o)[16]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 16; ++q) o[q] = __ldcg(reinterpret_cast<const float4*>(Cg) + (16 * w + q) * (CT / 4) + lane);
}
// TMEM accumulator -> S (fp32, row stride EPS); caller syncs before reading S
__device__ __forceinline__ void tc_epi_stage(uint32_t tmem, float* S) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = 32 * (w & 3) + lane, c0 = 64 * (w >> 2);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float v[32];
    tmem_ld_sum(tmem + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(c0 + 32 * h), v);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(S + row * EPS + c0 + 32 * h + 4 * q) =
          make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}
// Cg -= S (o = the prefetched Cg), coalesced
__device__ __forceinline__ void tc_epi_sub_store(float* Cg, const float4 (&o)[16], const float* S) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 d = *reinterpret_cast<const float4*>(S + (16 * w + q) * EPS + 4 * lane);
    float4 t = o[q];
    t.x -= d.x; t.y -= d.y; t.z -= d.z; t.w -= d.w;
    __stcg(reinterpret_cast<float4*>(Cg) + (16 * w + q) * (CT / 4) + lane, t);
  }
}
__device__ __forceinline__ void tc_bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(su32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tc_bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tc_bulk_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;\n cp.async.bulk.wait_group 0;" ::: "memory");
}

// Pipeline bookkeeping shared by all threads (identical updates everywhere; only
// thread 0 issues copies / MMAs).  Stage s = n % TC_STAGES of the n-th fill.
struct TcRing {
  uint64_t* full;
  uint64_t* empty;
  unsigned char* base;
  uint32_t nfill, ncons;
};

// one K-chunk of 3xTF32 MMAs from stage s into the accumulator
__device__ __forceinline__ void tc_chunk_mma(const TcRing& R, int s, uint32_t tmem, bool first) {
  const uint32_t a_hi = su32(R.base + (size_t)s * TSTAGE), a_lo = a_hi + TCHUNK;
  const uint32_t b_hi = a_hi + 2 * TCHUNK;   // B_lo follows at + TCHUNK (the N = 256 descriptor spans both)
#pragma unroll
  for (int kk = 0; kk < TKC / 8; ++kk) {   // 16 fp16 (32 B) of K per MMA
    const uint32_t o = 32u * kk;
    tc_mma3(tmem, a_hi + o, a_lo + o, b_hi + o, first && kk == 0);
  }
}

// TRSM(i,k):  L_ik = W_ik Linv_kk^T   (A = W_ik split by the threads, B = Linv images)
__device__ void tc_task_trsm(const TcArgs& a, TcRing& R, uint64_t* accf, uint32_t& nacc, uint32_t tmem, int i,
                             int k, bool keep_smem = false) {
  const int tid = threadIdx.x;
  const float* Wik = a.W + tlin(i, k) * TILE_F;
  const float* ib = a.img + tlin(k, k) * TILE_F;
  if (tid == 0) proxy_fence_global();
  // the thread's share of A: 16-B unit u = tid % 8 of rows tid / 8 + 32 q of each chunk
  // (a warp reads four full 128-B chunk rows per instruction); all loads first
  const int u0 = tid & 7, m0 = tid >> 3;
  float4 areg[TNCH][4][2];   // unit u0 (8 columns) of rows m0 + 32 q of each 64-column chunk
#pragma unroll
  for (int ch = 0; ch < TNCH; ++ch)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        areg[ch][q][v] =
            __ldcg(reinterpret_cast<const float4*>(Wik + (int64_t)(m0 + 32 * q) * CT + 64 * ch + 8 * u0 + 4 * v));
#pragma unroll
  for (int ch = 0; ch < TNCH; ++ch) {
    const uint32_t n = R.nfill++;
    R.ncons++;
    const int s = n % TC_STAGES;
    if (n >= TC_STAGES) tc_mbar_wait(&R.empty[s], ((n / TC_STAGES) - 1) & 1);
    unsigned char* st = R.base + (size_t)s * TSTAGE;
    if (tid == 0) {
      tc_expect_tx(&R.full[s], 2 * TCHUNK);
      tc_bulk(st + 2 * TCHUNK, ib + ch * (CT * TKC), TCHUNK, &R.full[s]);
      tc_bulk(st + 3 * TCHUNK, ib + IMGP_F + ch * (CT * TKC), TCHUNK, &R.full[s]);
    }
    {
      unsigned char* hi = st;
      unsigned char* lo = st + TCHUNK;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint2 h0, l0, h1, l1;
        split4_h(areg[ch][q][0], h0, l0);
        split4_h(areg[ch][q][1], h1, l1);
        const int m = m0 + 32 * q;
        const int off = (m >> 3) * 1024 + (m & 7) * 128 + ((u0 ^ (m & 7)) << 4);   // bytes
        *reinterpret_cast<uint4*>(hi + off) = make_uint4(h0.x, h0.y, h1.x, h1.y);
        *reinterpret_cast<uint4*>(lo + off) = make_uint4(l0.x, l0.y, l1.x, l1.y);
      }
    }
    proxy_fence_shared();
    __syncthreads();
    if (tid == 0) {
      tc_mbar_wait(&R.full[s], (n / TC_STAGES) & 1);
      tc_fence_after();
      tc_chunk_mma(R, s, tmem, ch == 0);
      tc_commit(&R.empty[s]);
    }
  }
  if (tid == 0) tc_commit(accf);
  tc_mbar_wait(accf, nacc & 1);
  ++nacc;
  tc_fence_after();
  // epilogue: L_ik (fp32) staged row-padded at TC_EPI_OFF and its hi/lo chunk images
  // (the global image layout) at 2 ch TCHUNK (hi), + TCHUNK (lo) of the idle ring;
  // then the images leave by bulk copies and the fp32 rows by coalesced stores.
  // keep_smem: the images stay for the following SYRK of the DIAG task.
  {
    const int w = tid >> 5, lane = tid & 31;
    const int row = 32 * (w & 3) + lane, c0 = 64 * (w >> 2);
    float* S = reinterpret_cast<float*>(R.base + TC_EPI_OFF);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v[32];
      tmem_ld_sum(tmem + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(c0 + 32 * h), v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int cc = c0 + 32 * h + 4 * q, ch = cc >> 6;
        const float4 x = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        *reinterpret_cast<float4*>(S + row * EPS + cc) = x;
        uint2 hh, ll;
        split4_h(x, hh, ll);
        const int o2 = img_off(row, cc) - ch * (CT * 64);   // fp16 units within the chunk
        unsigned char* sh = R.base + (size_t)2 * ch * TCHUNK;
        *reinterpret_cast<uint2*>(sh + 2 * o2) = hh;
        *reinterpret_cast<uint2*>(sh + TCHUNK + 2 * o2) = ll;
      }
    }
    tc_fence_before();
    proxy_fence_shared();   // generic writes -> bulk-copy / tcgen05 reads of the images
    __syncthreads();
    float* ihi = a.img + tlin(i, k) * TILE_F;
    if (tid == 0) {
#pragma unroll
      for (int ch = 0; ch < TNCH; ++ch) {
        tc_bulk_store(ihi + ch * (CT * TKC), R.base + (size_t)2 * ch * TCHUNK, TCHUNK);
        tc_bulk_store(ihi + IMGP_F + ch * (CT * TKC), R.base + (size_t)(2 * ch + 1) * TCHUNK, TCHUNK);
      }
    }
    float* Lg = a.W + tlin(i, k) * TILE_F;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      __stcg(reinterpret_cast<float4*>(Lg) + (16 * w + q) * (CT / 4) + lane,
             *reinterpret_cast<const float4*>(S + (16 * w + q) * EPS + 4 * lane));
    if (tid == 0) tc_bulk_commit_wait();   // image writes complete before the caller's fences
  }
}

// TILE(i,j) (left-looking): W_ij = A_ij - sum_{m < mend} L_im L_jm^T with the sum formed
// on the tensor cores and kept on chip -- column pairs accumulate in TMEM, each pair is
// drained (fp32, round-to-nearest) into a register tile, and W_ij is written once -- then,
// for trsm, L_ij = W_ij Linv_jj^T as tc_task_trsm.  The operand chunks of all columns are
// one stream through the ring (the next pair's loads are in flight while a pair drains);
// column m's images are waited for (done flags) when its first chunk is loaded.
__device__ void tc_task_tile(const TcArgs& a, TcRing& R, uint64_t* accf, uint32_t& nacc, uint32_t tmem, int i,
                             int j, int mend, int mode) {
  const int tid = threadIdx.x, nt = a.nt;
  const int w = tid >> 5, lane = tid & 31;
  const int c0 = 64 * (w >> 2);
  const uint32_t trow = (uint32_t)(32 * (w & 3)) << 16;
  float acc[64];
#pragma unroll
  for (int q = 0; q < 64; ++q) acc[q] = 0.f;
  constexpr int GCH = 2 * TNCH;   // chunks per column pair
  const int nchunks = mend * TNCH;
  constexpr int PRE = TC_STAGES - 1;
  for (int q = 0; q < nchunks + PRE; ++q) {
    const int qc = q - PRE;
    if (tid == 0) {
      if (q < nchunks) {
        const int m = q / TNCH, ch = q % TNCH;
        if (ch == 0) {
          int ns = 32;
          while (ld_acquire(&a.done[i * nt + m]) < 1 || ld_acquire(&a.done[j * nt + m]) < 1) {
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
          }
          proxy_fence_global();   // images written by other CTAs (generic) -> our bulk reads (async)
        }
        const uint32_t n = R.nfill++;
        const int s = n % TC_STAGES;
        if (n >= TC_STAGES) tc_mbar_wait(&R.empty[s], ((n / TC_STAGES) - 1) & 1);
        const float* ia = a.img + tlin(i, m) * TILE_F + ch * (CT * TKC);
        const float* ib = a.img + tlin(j, m) * TILE_F + ch * (CT * TKC);
        unsigned char* st = R.base + (size_t)s * TSTAGE;
        tc_expect_tx(&R.full[s], TSTAGE);
        tc_bulk(st, ia, TCHUNK, &R.full[s]);
        tc_bulk(st + TCHUNK, ia + IMGP_F, TCHUNK, &R.full[s]);
        tc_bulk(st + 2 * TCHUNK, ib, TCHUNK, &R.full[s]);
        tc_bulk(st + 3 * TCHUNK, ib + IMGP_F, TCHUNK, &R.full[s]);
      }
      if (qc >= 0) {
        const uint32_t n = R.ncons++;
        const int s = n % TC_STAGES;
        tc_mbar_wait(&R.full[s], (n / TC_STAGES) & 1);
        tc_fence_after();
        tc_chunk_mma(R, s, tmem, qc % GCH == 0);
        tc_commit(&R.empty[s]);
        if (qc % GCH == GCH - 1 || qc == nchunks - 1) tc_commit(accf);
      }
    }
    if (qc >= 0 && (qc % GCH == GCH - 1 || qc == nchunks - 1)) {   // a pair is complete: drain it
      tc_mbar_wait(accf, nacc & 1);
      ++nacc;
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
        tmem_ld_sum(tmem + trow + (uint32_t)(c0 + 32 * h), v);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc[32 * h + k] += v[k];
      }
      tc_fence_before();
      __syncthreads();   // every lane has read the pair before the next pair's first MMA overwrites it
    }
  }
  if (tid != 0) {
    R.nfill += nchunks;
    R.ncons += nchunks;
  }
  // W_ij = A_ij - acc, staged through shared memory (the ring is idle) and written coalesced
  float* Cg = a.W + tlin(i, j) * TILE_F;
  float4 o[16];
  tc_epi_prefetch(Cg, o);
  float* S = reinterpret_cast<float*>(R.base + TC_EPI_OFF);
  {
    const int row = 32 * (w & 3) + lane;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      *reinterpret_cast<float4*>(S + row * EPS + c0 + 4 * q) =
          make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
  __syncthreads();
  if (mode == TILE_OPERAND) {
    // W_ij (fp32) and its hi/lo chunk images (the chain's TRSM A operand), the images
    // built in the idle ring (global layout) and copied out by bulk stores
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int r = 16 * w + q, c = 4 * lane, ch = c >> 6;
      const float4 d = *reinterpret_cast<const float4*>(S + r * EPS + c);
      float4 t = o[q];
      t.x -= d.x; t.y -= d.y; t.z -= d.z; t.w -= d.w;
      __stcg(reinterpret_cast<float4*>(Cg) + r * (CT / 4) + lane, t);
      uint2 hh, ll;
      split4_h(t, hh, ll);
      const int o2 = img_off(r, c) - ch * (CT * 64);   // fp16 units within the chunk
      unsigned char* sh = R.base + (size_t)2 * ch * TCHUNK;
      *reinterpret_cast<uint2*>(sh + 2 * o2) = hh;
      *reinterpret_cast<uint2*>(sh + TCHUNK + 2 * o2) = ll;
    }
    proxy_fence_shared();   // generic image writes -> bulk-copy reads
    __syncthreads();
    if (tid == 0) {
      float* ihi = a.img + tlin(i, j) * TILE_F;
#pragma unroll
      for (int ch = 0; ch < TNCH; ++ch) {
        tc_bulk_store(ihi + ch * (CT * TKC), R.base + (size_t)2 * ch * TCHUNK, TCHUNK);
        tc_bulk_store(ihi + IMGP_F + ch * (CT * TKC), R.base + (size_t)(2 * ch + 1) * TCHUNK, TCHUNK);
      }
      tc_bulk_commit_wait();   // the images are complete before the caller's fences and release
    }
    __syncthreads();
    return;
  }
  tc_epi_sub_store(Cg, o, S);
  proxy_fence_shared();   // generic staging writes before later bulk copies into the ring
  __syncthreads();        // W_ij complete (the TRSM below reads it back)
  if (mode == TILE_TRSM) {
    wait_geq(&a.done[j * nt + j], 1);
    __syncthreads();
    tc_task_trsm(a, R, accf, nacc, tmem, i, j);
  }
}

// TRSM(k+1,k) of the chain: B = Linv_kk images already in shared memory at 2 ch TCHUNK
// (POTRF's output), A = W_{k+1,k}'s hi/lo images, written by its TILE_OPERAND task, bulk
// copied to TC_ABUF_OFF -- while POTRF(k) runs when the operand is ready by then.
// The epilogue leaves L_ik's hi/lo images in shared memory (the SYRK's operands) and starts
// (does not wait for) their bulk stores.  done[k][k] is published with done[k+1][k] (the
// TILE tasks waiting for Linv_kk are ~20 us off the chain's critical path).  The chain
// stores only images: one SM's store bandwidth (~0.1 TB/s) made the fp32 copies of Linv_kk
// and L_{k+1,k} cost ~2 us per step; CONV tasks rebuild them (hi + lo) off the chain.
// A operand of the chain's TRSM(i,k): W_ik's hi/lo images -> TC_ABUF_OFF (thread 0)
__device__ __forceinline__ void tc_chain_operand_load(const TcArgs& a, unsigned char* base, int i, int k,
                                                      uint64_t* lbar) {
  proxy_fence_global();   // the images were written by another CTA
  const float* ia = a.img + tlin(i, k) * TILE_F;
  unsigned char* abuf = base + TC_ABUF_OFF;
  tc_expect_tx(lbar, 2 * TNCH * TCHUNK);
#pragma unroll
  for (int ch = 0; ch < TNCH; ++ch) {
    tc_bulk(abuf + (size_t)2 * ch * TCHUNK, ia + ch * (CT * TKC), TCHUNK, lbar);
    tc_bulk(abuf + (size_t)(2 * ch + 1) * TCHUNK, ia + IMGP_F + ch * (CT * TKC), TCHUNK, lbar);
  }
}
__device__ int tc_diag_trsm(const TcArgs& a, TcRing& R, uint64_t* accf, uint32_t& nacc, uint32_t tmem, int i,
                            int k, uint64_t* lbar, uint32_t& lcnt, bool prefetched, const int* sflag) {
  int sv = 0;   // (thread 0) *sflag, loaded once the MMAs are issued
  const int tid = threadIdx.x;
  unsigned long long* ph = a.trace ? a.trace + 4 * (size_t)a.ntasks + 16 * (size_t)k : nullptr;
  unsigned char* abuf = R.base + TC_ABUF_OFF;
  if (tid == 0) {
    if (!prefetched) tc_chain_operand_load(a, R.base, i, k, lbar);
    tc_mbar_wait(lbar, lcnt & 1);
    tc_fence_after();
#pragma unroll
    for (int ch = 0; ch < TNCH; ++ch) {
      const uint32_t ah = su32(abuf + (size_t)2 * ch * TCHUNK), al = ah + TCHUNK,
                     bh = su32(R.base + (size_t)2 * ch * TCHUNK);
#pragma unroll
      for (int kk = 0; kk < TKC / 8; ++kk) tc_mma3(tmem, ah + 32u * kk, al + 32u * kk, bh + 32u * kk, ch == 0 && kk == 0);
    }
    tc_commit(accf);
    sv = ld_acquire(sflag);
  }
  ++lcnt;
  if (ph && tid == 0) ph[2] = gtimer();
  tc_mbar_wait(accf, nacc & 1);
  ++nacc;
  tc_fence_after();
  if (ph && tid == 0) ph[8] = gtimer();
  {
    const int w = tid >> 5, lane = tid & 31;
    const int row = 32 * (w & 3) + lane, c0 = 64 * (w >> 2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v[32];
      tmem_ld_sum(tmem + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(c0 + 32 * h), v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int cc = c0 + 32 * h + 4 * q, ch = cc >> 6;
        const float4 x = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        uint2 hh, ll;
        split4_h(x, hh, ll);
        const int o2 = img_off(row, cc) - ch * (CT * 64);   // fp16 units within the chunk
        unsigned char* sh = R.base + (size_t)2 * ch * TCHUNK;
        *reinterpret_cast<uint2*>(sh + 2 * o2) = hh;
        *reinterpret_cast<uint2*>(sh + TCHUNK + 2 * o2) = ll;
      }
    }
    tc_fence_before();
    proxy_fence_shared();
    __syncthreads();
    if (tid == CHOL_THREADS - 1) {   // the chain's publishing thread
      float* ihi = a.img + tlin(i, k) * TILE_F;
#pragma unroll
      for (int ch = 0; ch < TNCH; ++ch) {
        tc_bulk_store(ihi + ch * (CT * TKC), R.base + (size_t)2 * ch * TCHUNK, TCHUNK);
        tc_bulk_store(ihi + IMGP_F + ch * (CT * TKC), R.base + (size_t)(2 * ch + 1) * TCHUNK, TCHUNK);
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  return sv;
}

// ---------------------------------------------------------------------------
// POTRF(k) of the tensor-core DAG, fp32 (the factor is fp32-accurate anyway;
// iterative refinement restores fp64).  Shared-memory layout (floats):
//   Ws  128 x 128 column-major, stride SWF: the tile, then L (lower)
//   Xf  128 x 128 row-major, stride SWF: Y = L^-1
// ---------------------------------------------------------------------------
constexpr int SWF = CT + 4;      // 132: float4-aligned columns
static_assert(TC_ABUF_OFF >= (size_t)2 * CT * SWF * sizeof(float), "chain A-operand buffer overlaps POTRF's tiles");

// 8x8 Cholesky + inverse of the diagonal block at (c0, c0) by ONE thread in
// registers (no barriers): L overwrites the block of Ws (column-major, upper part
// zeroed), the inverse goes to the same block of Xf (row-major).  Stride SWF.
__device__ __forceinline__ void diag8(float* Ws, float* Xf, int c0, int* bad) {
  float l[8][8], x[8][8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) l[r][c] = (r >= c) ? Ws[(c0 + c) * SWF + c0 + r] : 0.f;
  float rinv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float d = l[j][j];
    if (!(d > 0.f)) { *bad = 1; d = 1.f; }
    const float rs = rsqrtf(d);
    rinv[j] = rs;                                 // 1 / L[j][j]
    l[j][j] = d * rs;
#pragma unroll
    for (int r = j + 1; r < 8; ++r) l[r][j] *= rs;
#pragma unroll
    for (int c = j + 1; c < 8; ++c)
#pragma unroll
      for (int r = c; r < 8; ++r) l[r][c] = fmaf(-l[r][j], l[c][j], l[r][c]);
  }
  // X = L^-1, column by column of X (forward substitution of L x = e_c)
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < c) { x[r][c] = 0.f; continue; }
      float s = (r == c) ? 1.f : 0.f;
#pragma unroll
      for (int m = c; m < r; ++m) s = fmaf(-l[r][m], x[m][c], s);
      x[r][c] = s * rinv[r];
    }
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      Ws[(c0 + c) * SWF + c0 + r] = l[r][c];
      Xf[(c0 + r) * SWF + c0 + c] = x[r][c];
    }
}

// POTRF(k) of the tensor-core DAG, fp32 (the factor is fp32-accurate anyway;
// iterative refinement restores fp64): right-looking over 16 panels of 8
// columns.  Per panel, three barrier-separated phases:
//   1. one thread factors and inverts the 8x8 diagonal block in registers;
//   2. panel TRSM (a row per thread) and, on other threads, Y_s <- X_ss Y_s for
//      the panel's block row of Y (a column per thread);
//   3. rank-8 trailing update of A and the matching update of Y's rows below,
//      Y_t -= L_ts Y_s (4x4 register blocks),
// where Y starts as I and ends as L^-1 (forward substitution L Y = I fused into
// the factorisation).  Linv goes to W_kk (fp32 row-major, zeros above the
// diagonal, for the triangular solves) and to its hi/lo images (TRSM operand).
// from_smem: the updated diagonal tile is already in Ws (handed over by the chain's SYRK)
// pf: (chain) the flag of the next TRSM operand W_{k+1,k}; the last thread polls it between
// panels and starts the operand's bulk load (tc_chain_operand_load) once it is set (*pre = 1)
__device__ void tc_task_potrf(const TcArgs& a, int k, double* smem_d, bool defer = false, bool from_smem = false,
                              const int* pf = nullptr, uint64_t* lbar = nullptr, int* pre = nullptr) {
  float* Ws = reinterpret_cast<float*>(smem_d);   // tile, then L (column-major, SWF)
  float* Xf = Ws + CT * SWF;                      // Y -> Linv (row-major, SWF)
  __shared__ int bad;
  __shared__ unsigned short tri_tab[(CT / 4) * (CT / 4 + 1) / 2];   // triangle index -> (row << 5) | col
  const int tid = threadIdx.x;
  for (int rb = 0; rb < CT / 4; ++rb)
    for (int cw = tid; cw <= rb; cw += CHOL_THREADS) tri_tab[rb * (rb + 1) / 2 + cw] = (unsigned short)((rb << 5) | cw);
  float* Wk = a.W + tlin(k, k) * TILE_F;
  if (tid == 0) bad = 0;
  unsigned long long* ph = a.trace ? a.trace + 4 * (size_t)a.ntasks + 16 * (size_t)k : nullptr;   // phase stamps
  if (ph && tid == 0) { ph[0] = gtimer(); ph[11] = clock64(); }
  {   // The diagonal tile is symmetric (up to the rounding of its updates), so its
      // row-major image is read as column-major without a transpose.  Loads first.
    float4 q[16];
    if (!from_smem) {
#pragma unroll
      for (int u = 0; u < 16; ++u) q[u] = __ldcg(reinterpret_cast<const float4*>(Wk) + tid + u * CHOL_THREADS);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int t4 = 4 * (tid + u * CHOL_THREADS), c = t4 / CT, r = t4 % CT;
      if (!from_smem) *reinterpret_cast<float4*>(Ws + c * SWF + r) = q[u];
      const float4 id = make_float4(r == c ? 1.f : 0.f, r + 1 == c ? 1.f : 0.f, r + 2 == c ? 1.f : 0.f,
                                    r + 3 == c ? 1.f : 0.f);
      *reinterpret_cast<float4*>(Xf + c * SWF + r) = id;
    }
  }
  __syncthreads();
  if (ph && tid == 0) ph[1] = gtimer();
  // 4x4 register-blocked rank-8 updates of panel c0 (L columns c0..c0+7 of Ws):
  //   A block (rows r.., cols c.., r0 <= c <= r):  A[r][c] -= sum_m L[r][c0+m] L[c][c0+m]
  //   Y block (rows r >= r0, cols c < r0):          Y[r][c] -= sum_m L[r][c0+m] Y[c0+m][c]
  auto ablock = [&](int c0, int r, int c) {   // packed FFMA2 over row pairs (u, u+1)
    float2 acc[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float4 lr = *reinterpret_cast<const float4*>(Ws + (c0 + m) * SWF + r);
      const float4 lc = *reinterpret_cast<const float4*>(Ws + (c0 + m) * SWF + c);
      const float2 ra[2] = {make_float2(lr.x, lr.y), make_float2(lr.z, lr.w)};
      const float ca[4] = {lc.x, lc.y, lc.z, lc.w};
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = __ffma2_rn(ra[u], make_float2(ca[v], ca[v]), acc[u][v]);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      float4* d = reinterpret_cast<float4*>(Ws + (c + v) * SWF + r);
      float4 o = *d;
      o.x -= acc[0][v].x; o.y -= acc[0][v].y; o.z -= acc[1][v].x; o.w -= acc[1][v].y;
      *d = o;
    }
  };
  auto yblock = [&](int c0, int r, int c) {   // packed FFMA2 over column pairs (v, v+1)
    float2 acc[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) acc[u][v] = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float4 lr = *reinterpret_cast<const float4*>(Ws + (c0 + m) * SWF + r);
      const float4 yc = *reinterpret_cast<const float4*>(Xf + (c0 + m) * SWF + c);
      const float ra[4] = {lr.x, lr.y, lr.z, lr.w};
      const float2 ya[2] = {make_float2(yc.x, yc.y), make_float2(yc.z, yc.w)};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) acc[u][v] = __ffma2_rn(make_float2(ra[u], ra[u]), ya[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float4* d = reinterpret_cast<float4*>(Xf + (r + u) * SWF + c);
      float4 o = *d;
      o.x -= acc[u][0].x; o.y -= acc[u][0].y; o.z -= acc[u][1].x; o.w -= acc[u][1].y;
      *d = o;
    }
  };
  if (tid == 0) diag8(Ws, Xf, 0, &bad);
  __syncthreads();
  for (int sp = 0; sp < CT / 8; ++sp) {
    const int c0 = 8 * sp, r0 = c0 + 8, nr = CT - r0;
    if (tid < nr) {   // panel TRSM: L[r][c0+c] = sum_{m<=c} A[r][c0+m] X[c][m]
      const int r = r0 + tid;
      float av[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) av[m] = Ws[(c0 + m) * SWF + r];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float sum = 0.f;
#pragma unroll
        for (int m = 0; m <= c; ++m) sum = fmaf(av[m], Xf[(c0 + c) * SWF + c0 + m], sum);
        Ws[(c0 + c) * SWF + r] = sum;
      }
    } else if (tid >= 128 && tid - 128 < c0) {   // Y_s[:, c] <- X_ss Y_s[:, c] for columns c < c0
      const int c = tid - 128;
      float yv[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) yv[m] = Xf[(c0 + m) * SWF + c];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float sum = 0.f;
#pragma unroll
        for (int m = 0; m <= r; ++m) sum = fmaf(Xf[(c0 + r) * SWF + c0 + m], yv[m], sum);
        Xf[(c0 + r) * SWF + c] = sum;
      }
    }
    __syncthreads();
    if (nr == 0) break;
    // Look-ahead: warp 0 updates the next panel's 8x8 diagonal block (three 4x4
    // blocks) and one of its threads factors it (diag8) while warps 1..7 do the rest
    // of this panel's updates; the diagonal block is disjoint from everything they
    // read or write.
    if (tid < 32) {
      if (tid < 3) ablock(c0, r0 + (tid ? 4 : 0), r0 + (tid == 2 ? 4 : 0));
      __syncwarp();
      if (tid == 0) diag8(Ws, Xf, r0, &bad);
    } else {
      // operand poll: a relaxed load issued here, looked at after this panel's updates
      int fv = 0;
      const bool poll = pf && tid == CHOL_THREADS - 1 && !*pre;
      if (poll) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(fv) : "l"(pf) : "memory");
      const int nb4 = nr / 4, nsy = nb4 * (nb4 + 1) / 2, nyc = r0 / 4, nblk = nsy + nb4 * nyc;
      for (int b = tid - 32; b < nblk; b += CHOL_THREADS - 32) {
        if (b < nsy) {
          // mirrored so that consecutive b (lanes) walk down a block column: contiguous
          // float4 rows of the column-major tile, conflict-free; (rb, b - rb (rb+1)/2) of
          // the triangle index from the table
          const int tb = tri_tab[b], rb = tb >> 5, cw = tb & 31;
          const int cbk = nb4 - 1 - rb, rbk = nb4 - 1 - cw;
          if (rbk >= 2) ablock(c0, r0 + 4 * rbk, r0 + 4 * cbk);   // rbk < 2: warp 0's diagonal block
        } else {
          const int bb = b - nsy, rb = bb / nyc, cbk = bb - rb * nyc;
          yblock(c0, r0 + 4 * rb, 4 * cbk);
        }
      }
      if (poll && fv >= k + 1) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");   // acquire the release that set the flag
        tc_chain_operand_load(a, reinterpret_cast<unsigned char*>(smem_d), k + 1, k, lbar);
        *pre = 1;
      }
    }
    __syncthreads();
  }
  if (tid == 0 && bad) atomicExch(a.status, 1);
  if (ph && tid == 0) ph[9] = gtimer();
  // outputs: Linv row-major fp32 to W_kk (coalesced stores) and its hi/lo chunk images,
  // built in shared memory at 2 ch TCHUNK (hi) / + TCHUNK (lo) -- the B operand of the
  // DIAG task's TRSM -- and copied out by bulk stores.  With `defer` the caller waits
  // for the bulk stores (tc_bulk_commit_wait) and fences before publishing done[k][k].
  float4 xo[CT * CT / 4 / CHOL_THREADS];
#pragma unroll
  for (int u = 0; u < CT * CT / 4 / CHOL_THREADS; ++u) {
    const int t4 = tid + u * CHOL_THREADS, r = t4 / (CT / 4), c = 4 * (t4 % (CT / 4));
    const float4 y = *reinterpret_cast<const float4*>(Xf + r * SWF + c);
    xo[u] = make_float4(c <= r ? y.x : 0.f, c + 1 <= r ? y.y : 0.f, c + 2 <= r ? y.z : 0.f, c + 3 <= r ? y.w : 0.f);
  }
  __syncthreads();   // Ws / Xf are dead: the images overwrite them
  unsigned char* sbase = reinterpret_cast<unsigned char*>(smem_d);
#pragma unroll
  for (int u = 0; u < CT * CT / 4 / CHOL_THREADS; ++u) {
    const int t4 = tid + u * CHOL_THREADS, r = t4 / (CT / 4), c = 4 * (t4 % (CT / 4)), ch = c >> 6;
    const float4 x = xo[u];
    uint2 hh, ll;
    split4_h(x, hh, ll);
    const int o2 = img_off(r, c) - ch * (CT * 64);   // fp16 units within the chunk
    unsigned char* sh = sbase + (size_t)2 * ch * TCHUNK;
    *reinterpret_cast<uint2*>(sh + 2 * o2) = hh;
    *reinterpret_cast<uint2*>(sh + TCHUNK + 2 * o2) = ll;
  }
  proxy_fence_shared();   // generic image writes -> bulk-copy / tcgen05 reads
  __syncthreads();
  if (tid == (defer ? CHOL_THREADS - 1 : 0)) {   // deferred: the chain's publishing thread
    float* ihi = a.img + tlin(k, k) * TILE_F;
#pragma unroll
    for (int ch = 0; ch < TNCH; ++ch) {
      tc_bulk_store(ihi + ch * (CT * TKC), sbase + (size_t)2 * ch * TCHUNK, TCHUNK);
      tc_bulk_store(ihi + IMGP_F + ch * (CT * TKC), sbase + (size_t)(2 * ch + 1) * TCHUNK, TCHUNK);
    }
    if (!defer) tc_bulk_commit_wait();
    else asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (ph && tid == 0) { ph[10] = gtimer(); ph[12] = clock64(); }
  if (!defer) __syncthreads();
}

// CONV(k): the fp32 tiles of the chain's outputs for the triangular solves, rebuilt from
// their hi/lo images (hi + lo: 22 significant bits, the precision the factor's products
// carry): W_kk = Linv_kk (zeros above the diagonal) and W_{k+1,k} = L_{k+1,k}
__device__ void tc_task_conv(const TcArgs& a, int k) {
  const int tid = threadIdx.x, nt = a.nt;
  for (int t = 0; t < 2 && k + t < nt; ++t) {
    const int i = k + t;
    wait_geq(&a.done[i * nt + k], 1);
    __syncthreads();
    const __half* ih = reinterpret_cast<const __half*>(a.img + tlin(i, k) * TILE_F);
    const __half* il = ih + 2 * IMGP_F;
    float* Wg = a.W + tlin(i, k) * TILE_F;
#pragma unroll 4
    for (int u = 0; u < CT * CT / 4 / CHOL_THREADS; ++u) {
      const int t4 = tid + u * CHOL_THREADS, r = t4 / (CT / 4), c = 4 * (t4 % (CT / 4));
      const int o = img_off(r, c);
      const uint2 h = __ldcg(reinterpret_cast<const uint2*>(ih + o));
      const uint2 l = __ldcg(reinterpret_cast<const uint2*>(il + o));
      const float2 h0 = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
      const float2 h1 = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
      const float2 l0 = __half22float2(*reinterpret_cast<const __half2*>(&l.x));
      const float2 l1 = __half22float2(*reinterpret_cast<const __half2*>(&l.y));
      __stcg(reinterpret_cast<float4*>(Wg + r * CT + c),
             make_float4(h0.x + l0.x, h0.y + l0.y, h1.x + l1.x, h1.y + l1.y));
    }
  }
}

__global__ void __launch_bounds__(CHOL_THREADS, 1) k_chol_tc(TcArgs a) {
  extern __shared__ __align__(16) unsigned char tc_raw[];
  // 1024-B aligned (SW128 operand images) by pointer arithmetic on the __shared__
  // array itself, so the compiler keeps the shared state space (LDS/STS, not generic)
  unsigned char* sm = tc_raw + ((1024u - (su32(tc_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[TC_STAGES], empty[TC_STAGES], accf, lbar;
  __shared__ uint32_t tmem_sh;
  __shared__ int tsk, pre_sh;
  const int tid = threadIdx.x, nt = a.nt;
  uint32_t lcnt = 0;   // phases of lbar completed (identical in every thread)
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_sh)),
                 "n"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      tc_mbar_init(&full[s], 1);
      tc_mbar_init(&empty[s], 1);
    }
    tc_mbar_init(&accf, 1);
    tc_mbar_init(&lbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  TcRing R{full, empty, sm, 0u, 0u};
  uint32_t nacc = 0;
  while (true) {
    if (tid == 0) tsk = atomicAdd(a.counter, 1);
    __syncthreads();
    const int t = tsk;
    __syncthreads();
    if (t >= a.ntasks) break;
    const CholTask T = a.tasks[t];
    unsigned long long t0 = 0;
    if (a.trace && tid == 0) t0 = gtimer();
    switch (T.type) {
      case T_TRSM:
        wait_geq(&a.done[T.k * nt + T.k], 1);
        wait_geq(&a.upd[T.i * nt + T.k], T.expect);
        __syncthreads();
        if (a.trace && tid == 0) a.trace[4 * t + 1] = gtimer();
        tc_task_trsm(a, R, &accf, nacc, tmem, T.i, T.k);
        proxy_fence_global();
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release(&a.done[T.i * nt + T.k], 1);
        break;
      case T_CHAIN:   // POTRF(k) -> TRSM(k+1,k) -> SYRK(k+1) for every k, in one CTA
        if (a.trace && tid == 0) a.trace[4 * t + 1] = gtimer();
        for (int k = 0; k < nt; ++k) {
          const bool cont = k > 0;   // the tile is in Ws: the previous step's SYRK put it there
          if (k + 1 >= nt) {
            tc_task_potrf(a, k, reinterpret_cast<double*>(sm), false, cont);
            proxy_fence_global();
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release(&a.done[k * nt + k], 1);
            break;
          }
          // POTRF's outputs stay in shared memory as the TRSM's B operand; done[k][k] is
          // published inside tc_diag_trsm once POTRF's stores have drained
          if (tid == 0) pre_sh = 0;   // set once the TRSM operand's load is under way
          tc_task_potrf(a, k, reinterpret_cast<double*>(sm), true, cont, &a.upd[(k + 1) * nt + k], &lbar, &pre_sh);
          unsigned long long* ph = a.trace ? a.trace + 4 * (size_t)a.ntasks + 16 * (size_t)k : nullptr;
          wait_geq(&a.upd[(k + 1) * nt + k], k + 1);   // W_{k+1,k} and its images (TILE_OPERAND)
          __syncthreads();
          if (ph && tid == 0) ph[4] = gtimer();
          // the SYRK target's flag is read (acquire) by thread 0 while the TRSM's MMAs run
          const int sv = tc_diag_trsm(a, R, &accf, nacc, tmem, k + 1, k, &lbar, lcnt, pre_sh != 0,
                                      &a.upd[(k + 1) * nt + k + 1]);
          if (ph && tid == 0) ph[5] = gtimer();
          if (tid == 0 && sv < k) wait_geq(&a.upd[(k + 1) * nt + k + 1], k);
          __syncthreads();
          if (ph && tid == 0) ph[6] = gtimer();
          {   // SYRK(k+1) from the images in shared memory; L_{k+1,k} is published while it runs
            float* Cg = a.W + tlin(k + 1, k + 1) * TILE_F;
            if (tid == 0) {
              tc_fence_after();
              for (int ch = 0; ch < TNCH; ++ch) {
                const uint32_t hi = su32(R.base + (size_t)2 * ch * TCHUNK), lo = hi + TCHUNK;
#pragma unroll
                for (int kk = 0; kk < TKC / 8; ++kk)
                  tc_mma3(tmem, hi + 32u * kk, lo + 32u * kk, hi + 32u * kk, ch == 0 && kk == 0);
              }
              tc_commit(&accf);
            }
            const int w = tid >> 5, lane = tid & 31;
            float* S = reinterpret_cast<float*>(R.base + TC_EPI_OFF);
            float4 o[16];
            tc_epi_prefetch(Cg, o);
            if (tid == CHOL_THREADS - 1) {   // publish Linv_kk and L_{k+1,k} (the images are all the
              tc_bulk_wait_all();            // chain CTA writes: no CTA-wide fence needed)
              proxy_fence_global();
              __threadfence();
              st_release(&a.done[k * nt + k], 1);
              st_release(&a.done[(k + 1) * nt + k], 1);
            }
            __syncthreads();
            tc_mbar_wait(&accf, nacc & 1);
            ++nacc;
            tc_fence_after();
            tc_epi_stage(tmem, S);
            tc_fence_before();
            __syncthreads();
            // next POTRF's input straight into Ws (symmetric tile: row-major = column-major)
            float* Wn = reinterpret_cast<float*>(sm);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float4 d = *reinterpret_cast<const float4*>(S + (16 * w + q) * EPS + 4 * lane);
              float4 v = o[q];
              v.x -= d.x; v.y -= d.y; v.z -= d.z; v.w -= d.w;
              *reinterpret_cast<float4*>(Wn + (16 * w + q) * SWF + 4 * lane) = v;
            }
            proxy_fence_shared();   // S (generic writes) is where the next operand prefetch lands
            __syncthreads();
          }
          if (ph && tid == 0) ph[7] = gtimer();
        }
        break;
      case T_CONV:
        if (a.trace && tid == 0) a.trace[4 * t + 1] = gtimer();
        tc_task_conv(a, T.k);
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release(&a.convd[T.k], 1);
        break;
      case T_PREP: {   // inputs: the fp32 tiles CONV wrote (Linv_kk, L_{k+1,k}, L_{k,k-1}) or a TILE's TRSM
        const int k = T.i, kind = T.j;
        wait_geq(&a.convd[k], 1);
        if (kind == 1) wait_geq(&a.convd[k - 1], 1);
        if (kind == 2) wait_geq(&a.done[k * nt + k - 2], 1);
        if (kind == 4) wait_geq(&a.done[(k + 2) * nt + k], 1);
        __syncthreads();
        if (a.trace && tid == 0) a.trace[4 * t + 1] = gtimer();
        float* A = reinterpret_cast<float*>(sm);
        tc_task_prep(a, k, kind, A, A + TILE_F);
        break;
      }
      case T_TILE:
        if (a.trace && tid == 0) a.trace[4 * t + 1] = gtimer();
        tc_task_tile(a, R, &accf, nacc, tmem, T.i, T.j, T.k, T.expect);
        proxy_fence_global();
        __threadfence();
        __syncthreads();
        if (tid == 0) {
          if (T.expect == TILE_TRSM) st_release(&a.done[T.i * nt + T.j], 1);
          else st_release(&a.upd[T.i * nt + T.j], T.k + (T.expect == TILE_OPERAND ? 1 : 0));
        }
        break;
      default:
        break;
    }
    if (a.trace && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      a.trace[4 * t + 0] = t0;
      a.trace[4 * t + 2] = gtimer();
      a.trace[4 * t + 3] = smid;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS));
}

// ---------------------------------------------------------------------------
// scaling / conversion, triangular solves, fp64 residual
// ---------------------------------------------------------------------------
// D = diag(H)^-1/2 (padding rows: 1)
__global__ void k_tc_diag(const double* __restrict__ H, int64_t ld, int n, int npad, double* __restrict__ D) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= npad) return;
  double d = 1.0;
  if (r < n) {
    const double h = H[(int64_t)r * ld + r];
    d = h > 0.0 ? rsqrt(h) : 1.0;   // non-positive diagonal: the factorisation reports it
  }
  D[r] = d;
}

// W_ij = fp32(D_i H_ij D_j) from the lower triangle (identity padding); one CTA per lower tile
constexpr int kCvS = CT / 2 + 1;   // staging row stride (one 64-column half of a tile)
__global__ void __launch_bounds__(256) k_tc_convert(const double* __restrict__ H, int64_t ld, int n, int nt,
                                                    const double* __restrict__ D, float* __restrict__ W) {
  // one 128x128 tile per CTA, in two 64-column halves: H read column-major (a warp reads
  // contiguous rows of a column), transposed through a padded 128 x 64 shared buffer (33 KB:
  // 6 CTAs per SM) and written row-major, 256 B of a row per warp instruction
  extern __shared__ float ttile[];   // [CT][kCvS]
  const int64_t id = blockIdx.x;
  int i = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= id) ++i;
  while ((int64_t)i * (i + 1) / 2 > id) --i;
  const int j = (int)(id - (int64_t)i * (i + 1) / 2);
  float* Wt = W + id * TILE_F;
  const int tid = threadIdx.x;
  // interior off-diagonal tile (all of it in the stored lower triangle): 16-B loads of row pairs
  const bool fast = i != j && CT * (i + 1) <= n;
  const double dr0 = D[CT * i + 2 * (tid & 63)], dr1 = D[CT * i + 2 * (tid & 63) + 1];
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    if (fast) {
      double2 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int idx = tid + 256 * q, c = idx >> 6, rp = idx & 63;
        v[q] = __ldcs(reinterpret_cast<const double2*>(H + (int64_t)(CT * j + 64 * half + c) * ld + CT * i + 2 * rp));
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int idx = tid + 256 * q, c = idx >> 6, rp = idx & 63;
        const double dc = D[CT * j + 64 * half + c];
        ttile[(2 * rp) * kCvS + c] = (float)(dr0 * v[q].x * dc);
        ttile[(2 * rp + 1) * kCvS + c] = (float)(dr1 * v[q].y * dc);
      }
    } else {
      float v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int idx = tid + 256 * q, c = idx >> 7, r = idx & 127;
        const int R = CT * i + r, C = CT * j + 64 * half + c;
        if (R < n && C < n) {
          const int64_t a = (R >= C) ? (int64_t)C * ld + R : (int64_t)R * ld + C;   // lower triangle
          v[q] = (float)(D[R] * __ldcs(H + a) * D[C]);
        } else {
          v[q] = (R == C) ? 1.0f : 0.0f;
        }
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int idx = tid + 256 * q, c = idx >> 7, r = idx & 127;
        ttile[r * kCvS + c] = v[q];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < 8; ++q) {   // 16-B stores, a warp writes two 256-B half rows
      const int idx = tid + 256 * q, r = idx >> 4, c = 4 * (idx & 15);
      const float* t = ttile + r * kCvS + c;
      *reinterpret_cast<float4*>(Wt + r * CT + 64 * half + c) = make_float4(t[0], t[1], t[2], t[3]);
    }
    __syncthreads();
  }
}

// Triangular solves with the fp32 factor.  The solves only need the factor's
// (fp32) accuracy -- the fp64 residual of the refinement does the rest -- so the
// vectors are fp32.  One CTA per row tile (grid = nt <= #SMs, all resident).
// Hand-offs carry their own flag: every element of a published block is a
// 64-bit word (value, generation), written with one single-copy-atomic store,
// and the consumer polls the words of the block it needs (no memory fence on the
// critical chain).  Off the chain, each CTA folds its neighbour tile into the
// inverse of its diagonal tile (M = Linv_kk L_{k,k-1}, resp. T = L_{k+1,k} Linv_kk),
// so that one 128x128 matvec per step remains on the chain.
constexpr size_t TRI_SMEM = 3 * (size_t)TILE_F * sizeof(float) + 64;
#define TRI_STAMP(dir, what, k)

__device__ __forceinline__ void put_tagged(unsigned long long* p, float v, int gen) {
  const unsigned long long w = ((unsigned long long)(unsigned)gen << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ float get_tagged(const unsigned long long* p, int gen) {
  unsigned long long w;
  do {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  } while ((int)(w >> 32) < gen);
  return __uint_as_float((unsigned)w);
}
// block of 128 tagged values -> shared memory (threads < CT poll one word each)
__device__ __forceinline__ void fetch_block(const unsigned long long* src, float* dst, int gen) {
  if (threadIdx.x < CT) dst[threadIdx.x] = get_tagged(src + threadIdx.x, gen);
  __syncthreads();
}
// out[r] = sum_c A[r][c] v[c] for a row-major 128x128 smem tile (2 threads per row)
__device__ __forceinline__ float rowdot(const float* A, const float* v) {
  const int row = threadIdx.x >> 1, h = threadIdx.x & 1;
  const float4* p = reinterpret_cast<const float4*>(A + row * CT + 64 * h);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 a = p[q];
    const int c = 64 * h + 4 * q;
    s0 = fmaf(a.x, v[c], s0);
    s1 = fmaf(a.y, v[c + 1], s1);
    s2 = fmaf(a.z, v[c + 2], s2);
    s3 = fmaf(a.w, v[c + 3], s3);
  }
  float s = (s0 + s1) + (s2 + s3);
  return s + __shfl_xor_sync(0xffffffffu, s, 1);
}
// out[c] = sum_r A[r][c] v[r] (column sums; threads c and c + 128 take row halves)
__device__ __forceinline__ float coldot(const float* A, const float* v, float* part, bool glob) {
  const int col = threadIdx.x & (CT - 1), h = threadIdx.x >> 7;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 4
  for (int rr = 0; rr < 64; rr += 4) {
    const int r = 64 * h + rr;
    const float a0 = glob ? __ldcg(A + r * CT + col) : A[r * CT + col];
    const float a1 = glob ? __ldcg(A + (r + 1) * CT + col) : A[(r + 1) * CT + col];
    const float a2 = glob ? __ldcg(A + (r + 2) * CT + col) : A[(r + 2) * CT + col];
    const float a3 = glob ? __ldcg(A + (r + 3) * CT + col) : A[(r + 3) * CT + col];
    s0 = fmaf(a0, v[r], s0);
    s1 = fmaf(a1, v[r + 1], s1);
    s2 = fmaf(a2, v[r + 2], s2);
    s3 = fmaf(a3, v[r + 3], s3);
  }
  const float s = (s0 + s1) + (s2 + s3);
  if (h == 1) part[col] = s;
  __syncthreads();
  const float t = (h == 0) ? s + part[col] : 0.f;
  __syncthreads();
  return t;   // valid on threads < 128
}
// C = A B for row-major 128x128 smem tiles (C stored transposed if transC); A lower
// triangular if lowA, B lower if lowB.  C may alias A or B (all reads precede the writes).
__device__ __forceinline__ void smem_gemm128(float* C, const float* A, const float* B, bool lowA, bool lowB,
                                             bool transC = false) {
  const int t = threadIdx.x, r0 = 8 * (t >> 4), c0 = 8 * (t & 15);
  float acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.f;
  const int qlo = lowB ? c0 : 0, qhi = lowA ? r0 + 8 : CT;
  for (int q = qlo; q < qhi; ++q) {
    float av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = A[(r0 + u) * CT + q];
    const float4 b0 = *reinterpret_cast<const float4*>(B + q * CT + c0);
    const float4 b1 = *reinterpret_cast<const float4*>(B + q * CT + c0 + 4);
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
  }
  __syncthreads();   // all reads of A / B done (C may alias B)
  if (transC) {
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      *reinterpret_cast<float4*>(C + (c0 + v) * CT + r0) = make_float4(acc[0][v], acc[1][v], acc[2][v], acc[3][v]);
      *reinterpret_cast<float4*>(C + (c0 + v) * CT + r0 + 4) =
          make_float4(acc[4][v], acc[5][v], acc[6][v], acc[7][v]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      *reinterpret_cast<float4*>(C + (r0 + u) * CT + c0) = make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
      *reinterpret_cast<float4*>(C + (r0 + u) * CT + c0 + 4) =
          make_float4(acc[u][4], acc[u][5], acc[u][6], acc[u][7]);
    }
  }
  __syncthreads();
}

// in-place transpose of a row-major 128x128 smem tile
__device__ __forceinline__ void smem_transpose128(float* A) {
  float tmp[64];
  const int t = threadIdx.x;
#pragma unroll
  for (int q = 0; q < 64; ++q) {
    const int e = t + 256 * q, r = e >> 7, c = e & (CT - 1);
    tmp[q] = A[c * CT + r];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 64; ++q) A[t + 256 * q] = tmp[q];
  __syncthreads();
}

__device__ __forceinline__ void tri_prefetch(float* d0, const float* s0, float* d1, const float* s1, float* d2,
                                             const float* s2, uint64_t* bar) {
  if (threadIdx.x == 0) {
    tc_mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t tb = (uint32_t)(TILE_F * sizeof(float));
    tc_expect_tx(bar, tb * (1u + (s1 ? 1u : 0u) + (s2 ? 1u : 0u)));
    tc_bulk(d0, s0, tb, bar);
    if (s1) tc_bulk(d1, s1, tb, bar);
    if (s2) tc_bulk(d2, s2, tb, bar);
  }
}

// Per factorisation (not per pass): the folded neighbour matrices of the solves,
// one CTA per (k, kind), written to global memory in the layout their matvec
// reads conflict-free (out[r] = sum_c X[c][r] v[c], i.e. transposed for the
// forward solve):
//   kind 0: LinvT_k                     (forward base, Linv_kk acc)
//   kind 1: (Linv_kk L_{k,k-1})^T       (forward chain)
//   kind 2: (Linv_kk L_{k,k-2})^T
//   kind 3: L_{k+1,k} Linv_kk           (backward chain, read as column sums)
//   kind 4: L_{k+2,k} Linv_kk
__device__ void tc_task_prep(const TcArgs& a, int k, int kind, float* A, float* B) {
  const int nt = a.nt;
  float* out = a.Fm + ((int64_t)kind * nt + k) * TILE_F;
  const float* Lin = a.W + tlin(k, k) * TILE_F;
  const float* other = Lin;
  if (kind == 1) other = a.W + tlin(k, k - 1) * TILE_F;
  if (kind == 2) other = a.W + tlin(k, k - 2) * TILE_F;
  if (kind == 3) other = a.W + tlin(k + 1, k) * TILE_F;
  if (kind == 4) other = a.W + tlin(k + 2, k) * TILE_F;
  // kinds 1, 2: C = Lin X (A = Lin, B = X);  kinds 3, 4: C = X Lin (A = X, B = Lin)
  const float4* sa = reinterpret_cast<const float4*>(kind >= 3 ? other : Lin);
  const float4* sb = reinterpret_cast<const float4*>(kind >= 3 ? Lin : other);
  for (int e = threadIdx.x; e < TILE_F / 4; e += blockDim.x) {
    reinterpret_cast<float4*>(A)[e] = __ldcg(sa + e);
    if (kind != 0) reinterpret_cast<float4*>(B)[e] = __ldcg(sb + e);
  }
  __syncthreads();
  if (kind == 0) {
    smem_transpose128(A);
  } else {
    smem_gemm128(A, A, B, kind <= 2, kind >= 3, kind <= 2);   // in place; transposed output for kinds 1, 2
  }
  for (int e = threadIdx.x; e < TILE_F / 4; e += blockDim.x)
    __stcg(reinterpret_cast<float4*>(out) + e, reinterpret_cast<const float4*>(A)[e]);
  __syncthreads();   // shared memory is reused by the next task
}

// forward: L y = v, v = D r.  With M1 = Linv_kk L_{k,k-1}, M2 = Linv_kk L_{k,k-2}:
//   y_k = Linv_kk (v_k - sum_{j<k-2} L_kj y_j) - M2 y_{k-2} - M1 y_{k-1}
// LinvT, M1^T, M2^T come precomputed (PREP tasks of the DAG, tc_task_prep); the chain sees one 128x128
// shared-memory matvec per step.  Off-chain tiles are register-prefetched two deep.
// one butterfly stage of a warp transpose-reduction: lanes with bit LB set keep the
// upper ST values (adding their partner's), the others the lower ST
template <int ST, int LB>
__device__ __forceinline__ void bfly_stage(float* pr, int ln) {
  const bool up = ln & LB;
#pragma unroll
  for (int m = 0; m < ST; ++m) {
    const float give = up ? pr[m] : pr[m + ST];
    const float keep = up ? pr[m + ST] : pr[m];
    pr[m] = keep + __shfl_xor_sync(0xffffffffu, give, LB);
  }
}

// forward: L y = D r (row tile k; one CTA per row tile, all co-resident).
//   acc_k = D r_k - sum_{j <= k-3} V[k][j],   V[k][j] = L_kj y_j
//   y_k = Linv_kk acc_k - M2 y_{k-2} - M1 y_{k-1}     (M1, M2 folded by tc_task_prep)
// The off-chain products V[i][k] (i >= k+3) are computed by CTA k right after it
// publishes y_k (a column sweep over tiles L_ik, prefetched before y_k is known) and
// handed over as tagged words, so every row tile's off-chain sum is ready long
// before the chain reaches it; the chain step is fetch y_{k-1}, one 128x128
// shared-memory matvec, publish.  Sums run in fixed order (deterministic).
__global__ void __launch_bounds__(256, 1) k_tc_fwd(const float* __restrict__ W, const float* __restrict__ F,
                                                   int nt, const double* __restrict__ r,
                                                   const double* __restrict__ D, unsigned long long* __restrict__ y,
                                                   unsigned long long* __restrict__ V, int gen,
                                                   const int* __restrict__ stop, int helpers) {
  extern __shared__ __align__(16) unsigned char tri_raw[];
  float* Lin = reinterpret_cast<float*>(tri_raw);     // Linv_kk^T
  float* M1 = Lin + TILE_F;                           // M1^T
  float* M2 = M1 + TILE_F;                            // M2^T
  uint64_t* bar = reinterpret_cast<uint64_t*>(M2 + TILE_F);
  __shared__ float vs[CT], acc[CT], base[CT], part[CT];
  if (*stop) return;   // refinement converged in an earlier pass
  // CTAs nt .. 2 nt - 1 (when helpers): sweep-only helpers taking every other tile of column k
  const int tid = threadIdx.x;
  const bool helper = (int)blockIdx.x >= nt;
  const int k = helper ? (int)blockIdx.x - nt : (int)blockIdx.x;
  if (k >= nt) return;
  const int sstep = helpers ? 2 : 1, i0 = k + 3 + (helper ? 1 : 0);
  TRI_STAMP(0, 0, k)
  if (!helper)
    tri_prefetch(Lin, F + (int64_t)k * TILE_F, M1, k > 0 ? F + ((int64_t)nt + k) * TILE_F : nullptr, M2,
                 k > 1 ? F + ((int64_t)2 * nt + k) * TILE_F : nullptr, bar);
  // the first two tiles of this CTA's column sweep (independent of y); coalesced:
  // warp w reads rows 16 w .. 16 w + 15, lane l the float4 column l of each
  const int wq = tid >> 5, ln = tid & 31;
  auto ld_tile = [&](int i, float4* dst) {
    const float4* p = reinterpret_cast<const float4*>(W + tlin(i, k) * TILE_F) + 16 * wq * (CT / 4) + ln;
#pragma unroll
    for (int q = 0; q < 16; ++q) dst[q] = __ldcg(p + q * (CT / 4));
  };
  float4 bx[16], by[16];
  if (i0 < nt) ld_tile(i0, bx);
  if (i0 + sstep < nt) ld_tile(i0 + sstep, by);
  if (helper) {
    fetch_block(y + CT * k, vs, gen);
  } else {
  // off-chain sum, slots in order j = 0 .. k-3 (four polls in flight)
  if (tid < CT) {
    float a = (float)(D[CT * k + tid] * r[CT * k + tid]);
    const unsigned long long* src = V + (int64_t)k * nt * CT + tid;
    int j = 0;
    for (; j + 3 + 2 < k; j += 4) {
      const float v0 = get_tagged(src + (int64_t)j * CT, gen), v1 = get_tagged(src + (int64_t)(j + 1) * CT, gen);
      const float v2 = get_tagged(src + (int64_t)(j + 2) * CT, gen), v3 = get_tagged(src + (int64_t)(j + 3) * CT, gen);
      a -= v0; a -= v1; a -= v2; a -= v3;
    }
    for (; j + 2 < k; ++j) a -= get_tagged(src + (int64_t)j * CT, gen);
    acc[tid] = a;
  }
  __syncthreads();
  TRI_STAMP(0, 1, k)
  tc_mbar_wait(bar, 0);
  TRI_STAMP(0, 2, k)
  {
    const float b = coldot(Lin, acc, part, false);   // (Linv acc)[r] = sum_c LinvT[c][r] acc[c]
    if (tid < CT) base[tid] = b;
  }
  __syncthreads();
  if (k > 1) {
    fetch_block(y + CT * (k - 2), vs, gen);
    const float s = coldot(M2, vs, part, false);
    if (tid < CT) base[tid] -= s;
    __syncthreads();
  }
  if (k > 0) {   // the chain: y_k = base - M1 y_{k-1}
    fetch_block(y + CT * (k - 1), vs, gen);
    const float s = coldot(M1, vs, part, false);
    __syncthreads();   // vs is reused for y_k below
    if (tid < CT) {
      const float yk = base[tid] - s;
      put_tagged(y + CT * k + tid, yk, gen);
      vs[tid] = yk;
    }
  } else if (tid < CT) {
    put_tagged(y + CT * k + tid, base[tid], gen);
    vs[tid] = base[tid];
  }
  TRI_STAMP(0, 3, k)
  __syncthreads();
  }   // chain CTA
  // column sweep: V[i][k] = L_ik y_k for i >= k+3.  Each lane dots its float4 of 16
  // rows with y, then a 5-stage butterfly (16 shuffles) leaves row
  // 16 w + (l4 l3 l2 l1) summed over the warp in lanes with l0 = 0 (fixed order).
  const float4 yv = reinterpret_cast<const float4*>(vs)[ln];
  auto sweep = [&](int i, float4* buf) {
    float pr[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
      pr[q] = fmaf(buf[q].w, yv.w, fmaf(buf[q].z, yv.z, fmaf(buf[q].y, yv.y, buf[q].x * yv.x)));
    bfly_stage<8, 16>(pr, ln);
    bfly_stage<4, 8>(pr, ln);
    bfly_stage<2, 4>(pr, ln);
    bfly_stage<1, 2>(pr, ln);
    const float sp = pr[0] + __shfl_xor_sync(0xffffffffu, pr[0], 1);
    const int r = 16 * wq + (((ln >> 4) & 1) << 3 | ((ln >> 3) & 1) << 2 | ((ln >> 2) & 1) << 1 | ((ln >> 1) & 1));
    if ((ln & 1) == 0) put_tagged(V + ((int64_t)i * nt + k) * CT + r, sp, gen);
    if (i + 2 * sstep < nt) ld_tile(i + 2 * sstep, buf);
  };
  for (int i = i0; i < nt; i += 2 * sstep) {
    sweep(i, bx);
    if (i + sstep < nt) sweep(i + sstep, by);
  }
}

// backward: L^T z = y.  With T1 = L_{k+1,k} Linv_kk, T2 = L_{k+2,k} Linv_kk:
//   z_k = Linv^T (y_k - sum_{i>k+2} L_ik^T z_i) - T2^T z_{k+2} - T1^T z_{k+1};
// then x += D z (fp64) with max |dx|, max |x|.  T1, T2 precomputed (tc_task_prep).
__global__ void __launch_bounds__(256, 1) k_tc_bwd(const float* __restrict__ W, const float* __restrict__ F,
                                                   int nt, const unsigned long long* __restrict__ y,
                                                   unsigned long long* __restrict__ z,
                                                   unsigned long long* __restrict__ U, const double* __restrict__ D,
                                                   double* __restrict__ x, double* __restrict__ dxmax,
                                                   double* __restrict__ xmax, int gen, const int* __restrict__ stop,
                                                   int helpers) {
  extern __shared__ __align__(16) unsigned char tri_raw[];
  float* Lin = reinterpret_cast<float*>(tri_raw);     // Linv_kk
  float* T1 = Lin + TILE_F;
  float* T2 = T1 + TILE_F;
  uint64_t* bar = reinterpret_cast<uint64_t*>(T2 + TILE_F);
  __shared__ float vs[CT], acc[CT], base[CT], part[CT];
  if (*stop) return;
  const int tid = threadIdx.x;
  // CTAs nt .. 2 nt - 1 (when helpers): sweep-only helpers taking every other tile of row k
  const bool helper = (int)blockIdx.x >= nt;
  const int bk = helper ? (int)blockIdx.x - nt : (int)blockIdx.x;
  if (bk >= nt) return;
  const int k = nt - 1 - bk;
  const int sstep = helpers ? 2 : 1, k0 = k - 3 - (helper ? 1 : 0);
  if (!helper)
    tri_prefetch(Lin, W + tlin(k, k) * TILE_F, T1, k + 1 < nt ? F + ((int64_t)3 * nt + k) * TILE_F : nullptr, T2,
                 k + 2 < nt ? F + ((int64_t)4 * nt + k) * TILE_F : nullptr, bar);
  // the first two tiles of this CTA's row sweep L_{k,kk}, kk = k-3, k-4, ... (contiguous);
  // coalesced: warp w reads rows 16 w .. 16 w + 15, lane l the float4 column l of each
  const int wq = tid >> 5, ln = tid & 31;
  float4 cx[16], cy[16];
  auto ld_col = [&](int kk, float4* dst) {
    const float4* p = reinterpret_cast<const float4*>(W + tlin(k, kk) * TILE_F) + 16 * wq * (CT / 4) + ln;
#pragma unroll
    for (int q = 0; q < 16; ++q) dst[q] = __ldcg(p + q * (CT / 4));
  };
  if (k0 >= 0) ld_col(k0, cx);
  if (k0 - sstep >= 0) ld_col(k0 - sstep, cy);
  if (helper) {
    fetch_block(z + CT * k, vs, gen);
  } else {
  // off-chain sum: acc = y_k - sum_{i = nt-1 down to k+3} U[k][i],  U[k][i] = L_ik^T z_i
  if (tid < CT) {
    float a = get_tagged(y + CT * k + tid, gen);   // y_k (the forward pass is complete)
    const unsigned long long* src = U + (int64_t)k * nt * CT + tid;
    int i = nt - 1;
    for (; i - 3 > k + 2; i -= 4) {
      const float v0 = get_tagged(src + (int64_t)i * CT, gen), v1 = get_tagged(src + (int64_t)(i - 1) * CT, gen);
      const float v2 = get_tagged(src + (int64_t)(i - 2) * CT, gen), v3 = get_tagged(src + (int64_t)(i - 3) * CT, gen);
      a -= v0; a -= v1; a -= v2; a -= v3;
    }
    for (; i > k + 2; --i) a -= get_tagged(src + (int64_t)i * CT, gen);
    acc[tid] = a;
  }
  __syncthreads();
  tc_mbar_wait(bar, 0);
  {
    const float b = coldot(Lin, acc, part, false);
    if (tid < CT) base[tid] = b;
  }
  __syncthreads();
  if (k + 2 < nt) {
    fetch_block(z + CT * (k + 2), vs, gen);
    const float s = coldot(T2, vs, part, false);
    if (tid < CT) base[tid] -= s;
    __syncthreads();
  }
  float zk = 0.f;
  if (k + 1 < nt) {   // the chain: z_k = base - T1^T z_{k+1}
    fetch_block(z + CT * (k + 1), vs, gen);
    const float s = coldot(T1, vs, part, false);
    zk = (tid < CT) ? base[tid] - s : 0.f;
  } else {
    zk = (tid < CT) ? base[tid] : 0.f;
  }
  __syncthreads();   // vs is reused for z_k below
  if (tid < CT) {
    put_tagged(z + CT * k + tid, zk, gen);
    vs[tid] = zk;
    const double dxv = D[CT * k + tid] * (double)zk;
    const double xn = x[CT * k + tid] + dxv;
    x[CT * k + tid] = xn;
    // max |dx|, max |x| (non-negative doubles order like their bit patterns): warp max, one atomic per warp
    double m1 = fabs(dxv), m2 = fabs(xn);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
      m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    }
    if ((tid & 31) == 0) {
      if (dxmax) atomicMax(reinterpret_cast<unsigned long long*>(dxmax), (unsigned long long)__double_as_longlong(m1));
      if (xmax) atomicMax(reinterpret_cast<unsigned long long*>(xmax), (unsigned long long)__double_as_longlong(m2));
    }
  }
  __syncthreads();
  }   // chain CTA
  // row sweep: U[kk][k] = L_{k,kk}^T z_k for kk <= k-3 (column sums): per-warp float4
  // partials over 16 rows, then the 8 warps' partials summed in order through smem
  __shared__ float4 red[8][CT / 4];
  auto sweep = [&](int kk, float4* buf) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float zr = vs[16 * wq + q];
      a.x = fmaf(buf[q].x, zr, a.x);
      a.y = fmaf(buf[q].y, zr, a.y);
      a.z = fmaf(buf[q].z, zr, a.z);
      a.w = fmaf(buf[q].w, zr, a.w);
    }
    red[wq][ln] = a;
    __syncthreads();
    if (tid < CT) {
      const float* rf = reinterpret_cast<const float*>(red);
      float sp = rf[tid];
#pragma unroll
      for (int w2 = 1; w2 < 8; ++w2) sp += rf[w2 * CT + tid];
      put_tagged(U + ((int64_t)kk * nt + k) * CT + tid, sp, gen);
    }
    __syncthreads();
    if (kk - 2 * sstep >= 0) ld_col(kk - 2 * sstep, buf);
  };
  for (int kk = k0; kk >= 0; kk -= 2 * sstep) {
    sweep(kk, cx);
    if (kk - sstep >= 0) sweep(kk - sstep, cy);
  }
}

// symmetric H x from the lower triangle, 64x64 fp64 blocks: P[a][b][0..64) = contribution
// of block (max(a,b), min(a,b)) to rows of block a
constexpr int SYB = 64;
__global__ void __launch_bounds__(256) k_tc_symv(const double* __restrict__ H, int64_t ld, int n, int nb,
                                                 const double* __restrict__ x, double* __restrict__ P,
                                                 const int* __restrict__ stop) {
  // Warp w holds columns w, w+8, .., w+56 of the block, lane l rows 2l, 2l+1 (16-B loads, a
  // warp reads one 512-B column).  Column sums (H^T x_i) are warp reductions; row sums
  // (H x_j) are per-lane partials over the warp's 8 columns, summed over the 8 warps through
  // shared memory -- no transpose of the block.  Diagonal blocks (lower half stored): rows
  // use c <= r, columns r > c, so the two sums together are the symmetric product.
  __shared__ double xi[SYB], xj[SYB];
  __shared__ double rowp[8][SYB], colv[SYB];
  if (*stop) return;
  const int64_t id = blockIdx.x;
  int i = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= id) ++i;
  while ((int64_t)i * (i + 1) / 2 > id) --i;
  const int j = (int)(id - (int64_t)i * (i + 1) / 2);
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  double2 v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = w + 8 * q;
    v[q] = __ldcg(reinterpret_cast<const double2*>(H + (int64_t)(SYB * j + c) * ld + SYB * i) + l);
  }
  if (tid < SYB) {
    const int R = SYB * i + tid, C = SYB * j + tid;
    xi[tid] = R < n ? x[R] : 0.0;
    xj[tid] = C < n ? x[C] : 0.0;
  }
  __syncthreads();
  const int r0 = 2 * l, r1 = 2 * l + 1;
  const bool rin0 = SYB * i + r0 < n, rin1 = SYB * i + r1 < n;
  const bool diag = i == j;
  double rs0 = 0.0, rs1 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = w + 8 * q;
    const bool cin = SYB * j + c < n;
    const double h0 = (cin && rin0) ? v[q].x : 0.0, h1 = (cin && rin1) ? v[q].y : 0.0;
    // rows of block i: H(r, c) x_j[c] (diagonal block: c <= r)
    rs0 = fma((!diag || c <= r0) ? h0 : 0.0, xj[c], rs0);
    rs1 = fma((!diag || c <= r1) ? h1 : 0.0, xj[c], rs1);
    // rows of block j (column c): sum_r H(r, c) x_i[r] (diagonal block: r > c)
    double cs = fma((!diag || r0 > c) ? h0 : 0.0, xi[r0], ((!diag || r1 > c) ? h1 : 0.0) * xi[r1]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
    if (l == 0) colv[c] = cs;
  }
  rowp[w][r0] = rs0;
  rowp[w][r1] = rs1;
  __syncthreads();
  if (tid < SYB) {
    double s = rowp[0][tid];
#pragma unroll
    for (int u = 1; u < 8; ++u) s += rowp[u][tid];
    if (diag) s += colv[tid];
    P[((int64_t)i * nb + j) * SYB + tid] = s;
  } else if (tid < 2 * SYB && !diag) {
    P[((int64_t)j * nb + i) * SYB + (tid - SYB)] = colv[tid - SYB];
  }
}

// r = b - H x  (fixed-order sum of the block partials); padding rows 0
__global__ void k_tc_resid(const double* __restrict__ b, const double* __restrict__ P, int n, int npad, int nb,
                           double* __restrict__ r, const int* __restrict__ stop) {
  if (*stop) return;
  const int R = blockIdx.x * blockDim.x + threadIdx.x;
  if (R >= npad) return;
  if (R >= n) { r[R] = 0.0; return; }
  const int a = R / SYB, rr = R % SYB;
  double s = 0.0;
  for (int c = 0; c < nb; ++c) s += P[((int64_t)a * nb + c) * SYB + rr];
  r[R] = b[R] - s;
}

// after a refinement pass: stop when the correction is below tol max|x|, else
// Refinement stopping rule.  out[0] = max |correction| of this pass, out[1] = max |x|,
// out[2] = passes run, out[3] = the previous pass's relative correction, out[4] = 1 once
// accepted.  With the measured per-pass contraction rho = rel_k / rel_{k-1}, the error left
// after pass k is bounded by rel_k * rho / (1 - rho) (geometric tail); the solve is accepted
// when rel_k <= tol AND that bound is <= tol_err (both relative to max |x|).  A solve that
// never meets both within `iters` passes is redone on the fp64 path by the caller.
// The maxima are cleared for the next pass (the last pass's values stay in out).
__global__ void k_tc_check(double* out, int* stop, double tol, double tol_err, int last) {
  if (*stop) return;
  out[2] += 1.0;   // passes run
  const double rel = out[1] > 0.0 ? out[0] / out[1] : 0.0;
  bool ok = false;
  if (rel == 0.0) ok = true;
  else if (rel <= tol && out[3] > 0.0) {
    const double rho = rel / out[3];
    ok = rho < 0.5 && rel * rho / (1.0 - rho) <= tol_err;
  }
  if (ok) {
    out[4] = 1.0;
    *stop = 1;
  } else if (!last) {
    out[3] = rel;
    out[0] = out[1] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// host: workspace and driver
// ---------------------------------------------------------------------------
size_t chol_tc_smem_bytes() { return TC_SMEM; }

// bytes of the mixed-precision workspace for an npad x npad system
size_t chol_tc_ws_bytes(int npad) {
  const int nt = npad / CT;
  const int64_t ntl = (int64_t)nt * (nt + 1) / 2;
  const int nb = (npad + SYB - 1) / SYB;
  return sizeof(float) * (size_t)ntl * TILE_F * 3                  // W + two image parts
         + sizeof(float) * (size_t)5 * nt * TILE_F                  // folded solve matrices
         + sizeof(double) * ((size_t)npad * 4)                      // D, r, y, z
         + sizeof(unsigned long long) * (size_t)2 * nt * npad       // off-chain slots of the solves
         + sizeof(double) * (size_t)nb * nb * SYB                   // symv partials
         + sizeof(int) * ((size_t)2 * nt * nt + 2 + 3 * (size_t)nt) + 256 * 12;
}

// Solve H x = b (H: fp64 column-major, lower triangle read, npad = nt * 128,
// rows >= n are padding) with the tcgen05 factorisation + `iters` fp64
// refinement passes.  *status: 1 = non-positive pivot in the fp32 factor.
// Writes x[npad].  `ws` holds chol_tc_ws_bytes(npad) bytes; `tasks` the DAG
// from chol_plan_tasks(nt) (substitution tasks are skipped); `gen` must grow
// by at least 2 * iters between calls sharing `ws` (flag generations).
int chol_tc_solve(const double* H, int64_t ld, int n, int npad, const double* b, double* x, void* ws,
                  const void* tasks, int ntasks, int iters, int* status, int gen, cudaStream_t st, double* out2,
                  unsigned long long* trace, cudaEvent_t* ev3) {
  const int nt = npad / CT;
  if (nt <= 0) return 0;
  const int64_t ntl = (int64_t)nt * (nt + 1) / 2;
  const int nb = (npad + SYB - 1) / SYB;
  char* p = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* q = p; p += (bytes + 255) / 256 * 256; return q; };
  float* W = reinterpret_cast<float*>(take(sizeof(float) * ntl * TILE_F));
  float* img = reinterpret_cast<float*>(take(sizeof(float) * ntl * TILE_F * 2));
  float* Fm = reinterpret_cast<float*>(take(sizeof(float) * (size_t)5 * nt * TILE_F));
  double* D = reinterpret_cast<double*>(take(sizeof(double) * npad));
  double* r = reinterpret_cast<double*>(take(sizeof(double) * npad));
  unsigned long long* y = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * npad));
  unsigned long long* z = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * npad));
  unsigned long long* Vs = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * (size_t)nt * npad));
  unsigned long long* Us = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * (size_t)nt * npad));
  double* P = reinterpret_cast<double*>(take(sizeof(double) * (size_t)nb * nb * SYB));
  int* flags = reinterpret_cast<int*>(take(sizeof(int) * ((size_t)2 * nt * nt + 1 + nt)));
  int* sfl = reinterpret_cast<int*>(take(sizeof(int) * 2 * (size_t)nt));
  int* stop = reinterpret_cast<int*>(take(sizeof(int)));
  static int grid = 0, sms = 0;
  if (grid == 0) {
    cudaFuncSetAttribute(k_chol_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM);
    cudaFuncSetAttribute(k_tc_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRI_SMEM);
    cudaFuncSetAttribute(k_tc_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRI_SMEM);
    cudaFuncSetAttribute(k_tc_convert, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)CT * kCvS * sizeof(float)));
    int dev = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chol_tc, CHOL_THREADS, TC_SMEM);
    grid = sms * (per > 0 ? per : 1);
  }
  k_tc_diag<<<(npad + 255) / 256, 256, 0, st>>>(H, ld, n, npad, D);
  k_tc_convert<<<(unsigned)ntl, 256, (size_t)CT * kCvS * sizeof(float), st>>>(H, ld, n, nt, D, W);
  cudaMemsetAsync(flags, 0, sizeof(int) * ((size_t)2 * nt * nt + 1 + nt), st);
  TcArgs a;
  a.W = W;
  a.img = img;
  a.nt = nt;
  a.upd = flags;
  a.done = flags + (size_t)nt * nt;
  a.counter = flags + (size_t)2 * nt * nt;
  a.tasks = reinterpret_cast<const CholTask*>(tasks);
  a.ntasks = ntasks;
  a.status = status;
  a.trace = trace;
  a.Fm = Fm;
  a.convd = flags + (size_t)2 * nt * nt + 1;
  if (ev3) cudaEventRecord(ev3[0], st);
  launch_coresident(k_chol_tc, ntasks < grid ? ntasks : grid, CHOL_THREADS, TC_SMEM, st, a);
  launch_count();
  launch_count();
  launch_count();
  if (ev3) cudaEventRecord(ev3[1], st);
  cudaMemsetAsync(x, 0, sizeof(double) * npad, st);
  cudaMemsetAsync(stop, 0, sizeof(int), st);
  cudaMemsetAsync(out2, 0, sizeof(double) * 5, st);
  if (nt > sms) return 1;   // caller must solve on the fp64 path (out2[4] stays 0: not accepted)   // one resident CTA per row tile (n <= 148 * 128 here)
  // passes until the correction is <= kTcRefineTol max|x| (early-exit kernels after that), at most `iters`
  for (int it = 0; it < iters; ++it) {
    const double* rhs = b;
    if (it > 0) {
      k_tc_symv<<<(unsigned)((int64_t)nb * (nb + 1) / 2), 256, 0, st>>>(H, ld, n, nb, x, P, stop);
      k_tc_resid<<<(npad + 255) / 256, 256, 0, st>>>(b, P, n, npad, nb, r, stop);
      launch_count();
      launch_count();
      rhs = r;
    }
    // one chain CTA per block row, plus a sweep helper per block row when 2 nt CTAs
    // fit on the GPU at once (all CTAs of these kernels must be co-resident)
    const int hlp = 2 * nt <= sms ? 1 : 0;
    launch_coresident(k_tc_fwd, nt * (1 + hlp), 256, TRI_SMEM, st, (const float*)W, (const float*)Fm, nt, rhs,
                      (const double*)D, y, Vs, gen + 2 * it, (const int*)stop, hlp);
    launch_coresident(k_tc_bwd, nt * (1 + hlp), 256, TRI_SMEM, st, (const float*)W, (const float*)Fm, nt,
                      (const unsigned long long*)y, z, Us, (const double*)D, x, out2, out2 + 1, gen + 2 * it,
                      (const int*)stop, hlp);
    // stop once a pass corrects x by <= kTcRefineTol max|x| (vba_internal.cuh)
    k_tc_check<<<1, 1, 0, st>>>(out2, stop, kTcRefineTol, kTcErrTol, it == iters - 1);
    launch_count();
    launch_count();
    launch_count();
  }
  if (ev3) cudaEventRecord(ev3[2], st);
  return 0;
}

// Summary of a task trace ([ntasks][4] globaltimer stamps) on stderr (diagnostics).
void chol_trace_print(const char* tag, const unsigned long long* d_trace, const void* d_tasks, int ntasks, int nt) {
  {
    std::vector<unsigned long long> ph((size_t)16 * nt);
    cudaMemcpy(ph.data(), d_trace + 4 * (size_t)ntasks, ph.size() * 8, cudaMemcpyDeviceToHost);
    double ld = 0, u = 0, inv = 0, clk = 0, ns = 0, d[4] = {0, 0, 0, 0};
    int nd = 0;
    for (int k = 0; k < nt; ++k) {
      const unsigned long long* q = &ph[16 * (size_t)k];
      if (!q[0] || !q[10]) continue;
      ld += (double)(q[1] - q[0]) * 1e-3;
      u += (double)(q[9] - q[1]) * 1e-3;
      inv += (double)(q[10] - q[9]) * 1e-3;
      if (q[12] > q[11]) { clk += (double)(q[12] - q[11]); ns += (double)(q[10] - q[0]); }
      if (q[4] && q[7]) {   // DIAG task: wait for TRSM(k+1,k) operand, TRSM, wait for SYRK target, SYRK
        d[0] += (double)(q[4] - q[10]) * 1e-3;
        d[1] += (double)(q[5] - q[4]) * 1e-3;
        d[2] += (double)(q[6] - q[5]) * 1e-3;
        d[3] += (double)(q[7] - q[6]) * 1e-3;
        ++nd;
      }
    }
    if (ns > 0) fprintf(stderr, "  POTRF SM clock %.0f MHz\n", 1e3 * clk / ns);
    if (getenv("VBA_CHOL_TRACE_STEPS"))   // per chain step: POTRF, operand wait, TRSM, SYRK wait, SYRK (us)
      for (int k = 0; k < nt; ++k) {
        const unsigned long long* q = &ph[16 * (size_t)k];
        if (!q[0] || !q[10] || !q[4] || !q[7]) continue;
        fprintf(stderr, "   step %2d at %7.1f: potrf %5.1f wait %5.1f trsm %5.1f [mma-issued %4.1f acc %4.1f] wait %4.1f syrk %4.1f\n", k,
                (double)(q[0] - ph[0]) * 1e-3, (double)(q[10] - q[0]) * 1e-3, (double)(q[4] - q[10]) * 1e-3,
                (double)(q[5] - q[4]) * 1e-3, (double)(q[2] - q[4]) * 1e-3,
                (double)(q[8] - q[4]) * 1e-3, (double)(q[6] - q[5]) * 1e-3, (double)(q[7] - q[6]) * 1e-3);
      }
    fprintf(stderr, "  POTRF phases (avg us): load %.2f | panels %.2f | inverse+store %.2f\n", ld / nt, u / nt,
            inv / nt);
    if (nd)
      fprintf(stderr, "  DIAG after POTRF (avg us): wait %.2f | TRSM %.2f | wait %.2f | SYRK %.2f\n", d[0] / nd,
              d[1] / nd, d[2] / nd, d[3] / nd);
  }
  std::vector<unsigned long long> tr((size_t)4 * ntasks);
  std::vector<CholTask> tk(ntasks);
  cudaMemcpy(tr.data(), d_trace, tr.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(tk.data(), d_tasks, tk.size() * sizeof(CholTask), cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, t1 = 0;
  double busy[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, wait[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int cnt[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int q = 0; q < ntasks; ++q) {
    if (tr[4 * q] == 0) continue;
    t0 = std::min(t0, tr[4 * q]);
    t1 = std::max(t1, tr[4 * q + 2]);
    const int ty = tk[q].type;
    busy[ty] += (double)(tr[4 * q + 2] - tr[4 * q + 1]) * 1e-3;
    wait[ty] += (double)(tr[4 * q + 1] - tr[4 * q]) * 1e-3;
    cnt[ty] += 1;
  }
  {   // the DIAG chain: idle gaps between DIAG(k) done and DIAG(k+1) ready
    std::vector<std::pair<int, int>> dg;
    for (int q = 0; q < ntasks; ++q)
      if (tk[q].type == T_DIAG && tr[4 * q]) dg.push_back({tk[q].k, q});
    std::sort(dg.begin(), dg.end());
    double gap = 0.0, gmax = 0.0;
    int kmax = -1;
    for (size_t u = 1; u < dg.size(); ++u) {
      const double g = ((double)tr[4 * dg[u].second + 1] - (double)tr[4 * dg[u - 1].second + 2]) * 1e-3;
      gap += g;
      if (g > gmax) { gmax = g; kmax = dg[u].first; }
    }
    if (getenv("VBA_CHOL_TRACE_TILE")) {   // all tasks on the tiles (k,k), (k+1,k) of one DIAG(k)
      const int kk = atoi(getenv("VBA_CHOL_TRACE_TILE"));
      for (int q = 0; q < ntasks; ++q) {
        const CholTask& T = tk[q];
        const bool hit = (T.type == T_GEMM && T.j == kk && (T.i == kk || T.i == kk + 1)) ||
                         (T.type == T_GEMM && T.j == kk - 1 && T.i == kk + 1) ||
                         (T.type == T_TRSM && (T.i == kk || T.i == kk + 1)) || (T.type == T_DIAG && T.k >= kk - 2 && T.k <= kk);
        if (hit && tr[4 * q])
          fprintf(stderr, "   task %6d type %d (i %d j %d k %d k2 %d exp %d): grab %8.1f ready %8.1f done %8.1f sm %llu\n", q,
                  T.type, T.i, T.j, T.k, T.k2, T.expect, ((double)tr[4 * q] - (double)t0) * 1e-3,
                  ((double)tr[4 * q + 1] - (double)t0) * 1e-3, ((double)tr[4 * q + 2] - (double)t0) * 1e-3, tr[4 * q + 3]);
      }
    }
    if (getenv("VBA_CHOL_TRACE_GAPS")) {
      fprintf(stderr, "  gaps:");
      for (size_t u = 1; u < dg.size(); ++u)
        fprintf(stderr, " %.0f", ((double)tr[4 * dg[u].second + 1] - (double)tr[4 * dg[u - 1].second + 2]) * 1e-3);
      fprintf(stderr, "\n");
    }
    if (!dg.empty())
      fprintf(stderr, "  DIAG chain: first ready at %.1f us, gaps %.1f us total (max %.1f us before k=%d), last done %.1f us\n",
              ((double)tr[4 * dg[0].second + 1] - (double)t0) * 1e-3, gap, gmax, kmax,
              ((double)tr[4 * dg.back().second + 2] - (double)t0) * 1e-3);
  }
  const char* nm[10] = {"POTRF", "TRSM", "GEMM", "BUPD", "BSOL", "DIAG", "CHAIN", "TILE", "CONV", "PREP"};
  fprintf(stderr, "[%s trace] nt=%d tasks=%d span %.1f us\n", tag, nt, ntasks, (double)(t1 - t0) * 1e-3);
  for (int ty = 0; ty < 10; ++ty)
    if (cnt[ty])
      fprintf(stderr, "  %-5s n=%6d  avg busy %8.2f us  avg wait %8.2f us  total busy %.1f us\n", nm[ty], cnt[ty],
              busy[ty] / cnt[ty], wait[ty] / cnt[ty], busy[ty]);
}

}  // namespace vba
