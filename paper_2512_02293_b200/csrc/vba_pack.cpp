// _vbapack: native host-side packing of a reference-style FrameGraph's vision edges
// into the padded, source-sorted fp32 layout the kernels stream.
//
// The drop-in entry point (paper_2512_02293_b200.solver.solve_vi_ba) receives the
// reference's Python objects: one VisionEdge per edge holding three fp64 (N, 2)
// numpy arrays (pixels, targets, weights; residuals.py:97-113).  Converting those
// with numpy costs ~25 us of interpreter + casting-loop time per edge; this module
// reads the arrays through the buffer protocol, releases the GIL and converts every
// edge on a pool of threads:
//
//   flow[r]    = (float)(targets[r] - pixels[r])   (u* - u: fp64 difference, one rounding)
//   weights[r] = (float)weights[r]
//   padding rows (up to the 4-pixel multiple) = 0
//
// and reports whether any edge's pixels differ from its source keyframe's pixels
// (pixel-mode detection; an edge sharing its keyframe's buffer is equal without a
// read) and whether any weight is negative (the reference's ValueError,
// residuals.py:112-113).  Host-only; no CUDA.  The result is bitwise identical to
// the numpy fill in device.HostLayout (test_host.py checks it).
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct View {
  const char* p = nullptr;
  Py_ssize_t rows = 0, s0 = 0, s1 = 0;
  double at(Py_ssize_t r, int c) const { return *reinterpret_cast<const double*>(p + r * s0 + c * s1); }
  bool contiguous() const { return s1 == (Py_ssize_t)sizeof(double) && s0 == 2 * (Py_ssize_t)sizeof(double); }
};

// an (n, 2) fp64 buffer view of `obj`; false (with a Python error set) otherwise
bool get_view(PyObject* obj, Py_buffer* b, View* v, Py_ssize_t rows, const char* what) {
  if (PyObject_GetBuffer(obj, b, PyBUF_STRIDES | PyBUF_FORMAT) != 0) return false;
  const bool fmt_ok = b->format && (std::strcmp(b->format, "d") == 0 || std::strcmp(b->format, "<d") == 0 ||
                                     std::strcmp(b->format, "=d") == 0);
  if (!fmt_ok || b->ndim != 2 || b->shape[1] != 2 || b->shape[0] != rows || b->itemsize != 8) {
    PyErr_Format(PyExc_TypeError, "%s: expected a float64 array of shape (%zd, 2)", what, rows);
    PyBuffer_Release(b);
    return false;
  }
  v->p = static_cast<const char*>(b->buf);
  v->rows = rows;
  v->s0 = b->strides[0];
  v->s1 = b->strides[1];
  return true;
}

bool equal_views(const View& a, const View& b) {
  if (a.p == b.p && a.s0 == b.s0 && a.s1 == b.s1) return true;   // same buffer, same layout
  if (a.contiguous() && b.contiguous()) return std::memcmp(a.p, b.p, (size_t)a.rows * 16) == 0;
  for (Py_ssize_t r = 0; r < a.rows; ++r)
    for (int c = 0; c < 2; ++c)
      if (a.at(r, c) != b.at(r, c)) return false;
  return true;
}

template <class T>
bool int64_buffer(PyObject* o, Py_buffer* b, const T** out, Py_ssize_t* n) {
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) != 0) return false;
  if (b->itemsize != 8) {
    PyErr_SetString(PyExc_TypeError, "expected an int64 array");
    PyBuffer_Release(b);
    return false;
  }
  *out = static_cast<const T*>(b->buf);
  *n = b->len / 8;
  return true;
}

// pack_edges(edges, order, ei_sorted, rows, eoff_pad, rows_pad, kpix, flow, wts, nthreads, check_neg)
//   edges: sequence of VisionEdge-like objects; order[k]: edge index at sorted position k;
//   ei_sorted[k]: its source keyframe index; rows/eoff_pad/rows_pad[k]: real rows, padded
//   row offset, padded row count; kpix: per-keyframe pixel arrays; flow/wts: writable
//   float32 buffers of n_rows_pad * 2.  Returns (pixels_mismatch, negative_weight).
PyObject* pack_edges(PyObject*, PyObject* args) {
  PyObject *edges, *order_o, *ei_o, *rows_o, *eoff_o, *rpad_o, *kpix, *flow_o, *wts_o;
  int nthreads = 1, check_neg = 1;
  if (!PyArg_ParseTuple(args, "OOOOOOOOOii", &edges, &order_o, &ei_o, &rows_o, &eoff_o, &rpad_o, &kpix, &flow_o,
                        &wts_o, &nthreads, &check_neg))
    return nullptr;
  Py_buffer bo{}, bi{}, br{}, be{}, bp{}, bf{}, bw{};
  const int64_t *order, *ei, *rows, *eoff, *rpad;
  Py_ssize_t E, n1, n2, n3, n4;
  std::vector<Py_buffer*> held;
  auto release_all = [&]() {
    for (Py_buffer* b : held) PyBuffer_Release(b);
    held.clear();
  };
  if (!int64_buffer(order_o, &bo, &order, &E)) return nullptr;
  held.push_back(&bo);
  if (!int64_buffer(ei_o, &bi, &ei, &n1)) { release_all(); return nullptr; }
  held.push_back(&bi);
  if (!int64_buffer(rows_o, &br, &rows, &n2)) { release_all(); return nullptr; }
  held.push_back(&br);
  if (!int64_buffer(eoff_o, &be, &eoff, &n3)) { release_all(); return nullptr; }
  held.push_back(&be);
  if (!int64_buffer(rpad_o, &bp, &rpad, &n4)) { release_all(); return nullptr; }
  held.push_back(&bp);
  if (n1 != E || n2 != E || n3 != E || n4 != E) {
    release_all();
    PyErr_SetString(PyExc_ValueError, "pack_edges: index arrays of different lengths");
    return nullptr;
  }
  if (PyObject_GetBuffer(flow_o, &bf, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) != 0) { release_all(); return nullptr; }
  held.push_back(&bf);
  if (PyObject_GetBuffer(wts_o, &bw, PyBUF_WRITABLE | PyBUF_C_CONTIGUOUS) != 0) { release_all(); return nullptr; }
  held.push_back(&bw);
  float* flow = static_cast<float*>(bf.buf);
  float* wts = static_cast<float*>(bw.buf);
  const Py_ssize_t cap = bf.len / 4;
  if (bw.len / 4 != cap) {
    release_all();
    PyErr_SetString(PyExc_ValueError, "pack_edges: flow and weight buffers differ in size");
    return nullptr;
  }
  // keyframe pixel views, fetched lazily per source keyframe
  PyObject* kseq = PySequence_Fast(kpix, "kpix must be a sequence");
  if (!kseq) { release_all(); return nullptr; }
  const Py_ssize_t K = PySequence_Fast_GET_SIZE(kseq);
  std::vector<Py_buffer> kbuf((size_t)K);
  std::vector<View> kview((size_t)K);
  std::vector<char> khave((size_t)K, 0);
  PyObject* eseq = PySequence_Fast(edges, "edges must be a sequence");
  if (!eseq) { Py_DECREF(kseq); release_all(); return nullptr; }
  const Py_ssize_t nE = PySequence_Fast_GET_SIZE(eseq);
  std::vector<Py_buffer> ebuf((size_t)E * 3);
  std::vector<View> eview((size_t)E * 3);
  Py_ssize_t got = 0;
  bool ok = true;
  static const char* names[3] = {"pixels", "targets", "weights"};
  for (Py_ssize_t k = 0; k < E && ok; ++k) {
    const int64_t e = order[k], i = ei[k];
    if (e < 0 || e >= nE || i < 0 || i >= K || eoff[k] < 0 || eoff[k] + rpad[k] > cap / 2 || rows[k] > rpad[k]) {
      PyErr_SetString(PyExc_ValueError, "pack_edges: index out of range");
      ok = false;
      break;
    }
    PyObject* eo = PySequence_Fast_GET_ITEM(eseq, e);
    for (int a = 0; a < 3 && ok; ++a) {
      PyObject* arr = PyObject_GetAttrString(eo, names[a]);
      if (!arr) { ok = false; break; }
      ok = get_view(arr, &ebuf[3 * k + a], &eview[3 * k + a], rows[k], names[a]);
      Py_DECREF(arr);   // the Py_buffer keeps the exporter alive
      if (ok) ++got;
    }
    if (ok && !khave[i]) {
      ok = get_view(PySequence_Fast_GET_ITEM(kseq, i), &kbuf[i], &kview[i], rows[k], "keyframe pixels");
      if (ok) khave[i] = 1;
    }
  }
  bool mismatch = false, neg = false;
  if (ok) {
    std::vector<char> mm((size_t)std::max(1, nthreads), 0), ng((size_t)std::max(1, nthreads), 0);
    Py_BEGIN_ALLOW_THREADS
    auto work = [&](int t, Py_ssize_t k0, Py_ssize_t k1) {
      bool m = false, n = false;
      for (Py_ssize_t k = k0; k < k1; ++k) {
        const View& px = eview[3 * k];
        const View& tg = eview[3 * k + 1];
        const View& wt = eview[3 * k + 2];
        float* fo = flow + 2 * eoff[k];
        float* wo = wts + 2 * eoff[k];
        const Py_ssize_t R = rows[k];
        if (px.contiguous() && tg.contiguous() && wt.contiguous()) {
          const double* P = reinterpret_cast<const double*>(px.p);
          const double* T = reinterpret_cast<const double*>(tg.p);
          const double* W = reinterpret_cast<const double*>(wt.p);
          for (Py_ssize_t x = 0; x < 2 * R; ++x) {
            fo[x] = (float)(T[x] - P[x]);
            wo[x] = (float)W[x];
            n |= W[x] < 0.0;
          }
        } else {
          for (Py_ssize_t r = 0; r < R; ++r)
            for (int c = 0; c < 2; ++c) {
              fo[2 * r + c] = (float)(tg.at(r, c) - px.at(r, c));
              const double w = wt.at(r, c);
              wo[2 * r + c] = (float)w;
              n |= w < 0.0;
            }
        }
        for (Py_ssize_t x = 2 * R; x < 2 * rpad[k]; ++x) fo[x] = wo[x] = 0.0f;
        if (!m) m = !equal_views(px, kview[ei[k]]);
      }
      mm[t] = m;
      ng[t] = n;
    };
    const int T = (int)std::max<Py_ssize_t>(1, std::min<Py_ssize_t>(nthreads, E));
    if (T <= 1) {
      work(0, 0, E);
    } else {
      // balanced by rows: contiguous ranges of sorted positions
      std::vector<Py_ssize_t> cut((size_t)T + 1, E);
      int64_t total = 0;
      for (Py_ssize_t k = 0; k < E; ++k) total += rows[k];
      int64_t acc = 0;
      int t = 1;
      cut[0] = 0;
      for (Py_ssize_t k = 0; k < E && t < T; ++k) {
        acc += rows[k];
        while (t < T && acc * T >= total * t) cut[t++] = k + 1;
      }
      std::vector<std::thread> th;
      for (int q = 0; q < T; ++q) th.emplace_back(work, q, cut[q], cut[q + 1]);
      for (auto& x : th) x.join();
    }
    Py_END_ALLOW_THREADS
    for (size_t q = 0; q < mm.size(); ++q) {
      mismatch |= mm[q] != 0;
      neg |= (ng[q] != 0) && check_neg;
    }
  }
  for (Py_ssize_t q = 0; q < got; ++q) PyBuffer_Release(&ebuf[q]);
  for (Py_ssize_t i = 0; i < K; ++i)
    if (khave[i]) PyBuffer_Release(&kbuf[i]);
  Py_DECREF(eseq);
  Py_DECREF(kseq);
  release_all();
  if (!ok) return nullptr;
  return Py_BuildValue("(OO)", mismatch ? Py_True : Py_False, neg ? Py_True : Py_False);
}

PyMethodDef methods[] = {
    {"pack_edges", pack_edges, METH_VARARGS, "Threaded fp32 flow/weight packing of vision edges (see module doc)."},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_vbapack",
                      "Native host packing of VI-BA vision edges (paper_2512_02293_b200).", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__vbapack(void) { return PyModule_Create(&moddef); }
