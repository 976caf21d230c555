// vba_plan.h — host-side contribution-list planner for block-symmetric systems
// (shared by the VI-BA context, vba_host.cu, and the pose-graph context, vba_pgba.cu).
//
// A system is assembled on the device by k_assemble (vba_dense.cu): one CTA per lower
// block (a >= b) sums, in a fixed order, the contributions listed for it -- plain
// blocks first, then the diagonal damping, then the Schur fill-in ("fill") blocks --
// so the result is deterministic and independent of how the blocks were produced.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "vba_internal.cuh"

namespace vba {

// contribution-list planner for the block matrix (reduced or export layout)
// ---------------------------------------------------------------------------
struct BlkBuilder {
  int nbr;
  std::vector<std::vector<Contrib>> ff, fl;   // per lower block: H_ff-type, fill-type
  std::vector<std::vector<Vec>> seg;
  explicit BlkBuilder(int n) : nbr(n), ff((size_t)n * (n + 1) / 2), fl((size_t)n * (n + 1) / 2), seg(n) {}
  static size_t id(int a, int b) { return (size_t)a * (a + 1) / 2 + b; }
  // add matrix M (rows x cols, row-major ld) as block (a,b) of the symmetric matrix
  void add(int a, int b, int64_t off, int ld, int rows, int cols, int sign, bool fill) {
    if (a < 0 || b < 0) return;
    auto& L = [&]() -> std::vector<std::vector<Contrib>>& { return fill ? fl : ff; }();
    Contrib c{};
    c.ld = ld;
    c.sign = (int8_t)sign;
    if (a > b) {
      c.off = off; c.rows = (int16_t)rows; c.cols = (int16_t)cols; c.trans = 0;
      L[id(a, b)].push_back(c);
    } else if (a < b) {
      c.off = off; c.rows = (int16_t)cols; c.cols = (int16_t)rows; c.trans = 1;
      L[id(b, a)].push_back(c);
    } else {
      c.off = off; c.rows = (int16_t)rows; c.cols = (int16_t)cols; c.trans = 0;
      L[id(a, a)].push_back(c);
    }
  }
  // off-diagonal pair block that maps onto a diagonal block: add M and M^T
  void add_both(int a, int b, int64_t off, int ld, int rows, int cols, int sign, bool fill) {
    add(a, b, off, ld, rows, cols, sign, fill);
    if (a == b && a >= 0) {
      auto& L = fill ? fl : ff;
      Contrib c{};
      c.off = off; c.ld = ld; c.rows = (int16_t)cols; c.cols = (int16_t)rows; c.trans = 1; c.sign = (int8_t)sign;
      L[id(a, a)].push_back(c);
    }
  }
  void addv(int a, int64_t off, int len, int sign) {
    if (a < 0) return;
    seg[a].push_back(Vec{off, len, sign});
  }
};


struct BlkPlan {
  int nbr = 0, nseg = 0;
  int32_t *bptr = nullptr, *bnff = nullptr, *roff = nullptr, *rdim = nullptr;
  Contrib* cs = nullptr;
  int32_t *sptr = nullptr, *soff = nullptr;   // soff: [nseg offsets][nseg dims]
  Vec* vs = nullptr;
  int32_t* blist = nullptr;                    // lower blocks with contributions (+ diagonal)
  int nblist = 0;
};

// device upload of a vector into a fresh allocation recorded in `allocs`
template <class T>
inline cudaError_t plan_upload(std::vector<void*>& allocs, T** p, const std::vector<T>& h, cudaStream_t st) {
  *p = nullptr;
  const size_t n = h.empty() ? 1 : h.size();
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) return e;
  allocs.push_back((void*)*p);
  if (!h.empty()) e = cudaMemcpyAsync(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st);
  return e;
}

inline cudaError_t upload_blk_plan(std::vector<void*>& allocs, BlkBuilder& B, const std::vector<int32_t>& roff,
                                   const std::vector<int32_t>& rdim, BlkPlan& pl, cudaStream_t st) {
  pl.nbr = B.nbr;
  pl.nseg = B.nbr;
  std::vector<int32_t> bptr(1, 0), bnff;
  std::vector<Contrib> cs;
  for (size_t i = 0; i < B.ff.size(); ++i) {
    for (auto& x : B.ff[i]) cs.push_back(x);
    bnff.push_back((int32_t)B.ff[i].size());
    for (auto& x : B.fl[i]) cs.push_back(x);
    bptr.push_back((int32_t)cs.size());
  }
  std::vector<int32_t> sptr(1, 0), soff;
  std::vector<Vec> vs;
  for (int a = 0; a < B.nbr; ++a) {
    for (auto& v : B.seg[a]) vs.push_back(v);
    sptr.push_back((int32_t)vs.size());
  }
  soff = roff;
  soff.insert(soff.end(), rdim.begin(), rdim.end());
  std::vector<int32_t> blist;
  {
    int64_t id = 0;
    for (int a = 0; a < B.nbr; ++a)
      for (int b = 0; b <= a; ++b, ++id)
        if (a == b || bptr[id + 1] > bptr[id]) blist.push_back((int32_t)id);
  }
  pl.nblist = (int)blist.size();
  cudaError_t e;
  if ((e = plan_upload(allocs, &pl.blist, blist, st)) || (e = plan_upload(allocs, &pl.bptr, bptr, st)) ||
      (e = plan_upload(allocs, &pl.bnff, bnff, st)) || (e = plan_upload(allocs, &pl.cs, cs, st)) ||
      (e = plan_upload(allocs, &pl.roff, roff, st)) || (e = plan_upload(allocs, &pl.rdim, rdim, st)) ||
      (e = plan_upload(allocs, &pl.sptr, sptr, st)) || (e = plan_upload(allocs, &pl.vs, vs, st)) ||
      (e = plan_upload(allocs, &pl.soff, soff, st)))
    return e;
  return cudaSuccess;
}

}  // namespace vba
