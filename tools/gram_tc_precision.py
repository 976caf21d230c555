"""Emulate the tensor-core Schur Gram's arithmetic on the CPU (oracle, fp64 numpy).

The fill-in C = W^T W (W = per-pixel coupling / sqrt(h), plus the g_d column; solver.py:282-285)
is formed as in csrc/vba_vision.cu:k_gram_tc: w = hi + lo with hi = w rounded to 11 significant
bits, lo = w - hi (read by the tensor core at tf32 precision), three products
hi.hi^T + hi.lo^T + lo.hi^T accumulated in fp32 over a pixel range, ranges summed in fp64.
Prints the resulting relative change of the reduced system and of the Schur step against the
exact fp64 fill-in -- on BASELINE configs (`python tools/gram_tc_precision.py cfg 3`) or on the
reference's golden windows (`python tools/gram_tc_precision.py golden`).
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from oracle import vi_ba as O  # noqa: E402


def split_hi(x):
    u = x.astype(np.float32).view(np.uint32)
    return ((u + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def tf32_trunc(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


RANGE = int(os.environ.get("RANGE", "1536"))
TRUNC = os.environ.get("TRUNC", "0") == "1"   # model: each MMA's fp32 accumulation truncates


def trunc32(x):
    """fp64 -> fp32 rounding toward zero."""
    f = x.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(x)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f


def fill(Wc, exact, R=None):
    R = R or RANGE
    if exact:
        return Wc @ Wc.T
    W32 = Wc.astype(np.float32)
    hi = split_hi(W32)
    lo = tf32_trunc(W32 - hi)
    out = np.zeros((Wc.shape[0],) * 2)
    for a in range(0, Wc.shape[1], R):
        h, l = hi[:, a:a + R], lo[:, a:a + R]
        if not TRUNC:
            out += (h @ h.T + h @ l.T + l @ h.T).astype(np.float64)
            continue
        acc = np.zeros((Wc.shape[0],) * 2, np.float32)
        for s in range(0, h.shape[1], 8):   # one K = 8 MMA step, three products
            for A, B in ((h, h), (h, l), (l, h)):
                acc = trunc32(acc.astype(np.float64) + A[:, s:s + 8].astype(np.float64) @ B[:, s:s + 8].T.astype(np.float64))
        out += acc.astype(np.float64)
    return out


def step(P, opts, exact):
    o = dict(O.DEFAULT_OPTS)
    o.update(opts)
    L = O.Layout(P, o)
    H_pp, Hpd, H_dd, g_p, g_d = O.linearize_sparse(P, L)
    lam, ridge = o["damping"], o.get("ridge", 1e-10)
    inv = 1.0 / O._damp(H_dd, lam, ridge)
    H = H_pp.copy()
    idx = np.arange(L.npv)
    H[idx, idx] = O._damp(np.diag(H_pp), lam, ridge)
    g = g_p.copy()
    for n in range(L.K):
        if not Hpd[n]:
            continue
        sl = slice(L.doff[n], L.doff[n + 1])
        kfs = sorted(Hpd[n])
        cols = np.concatenate([L.cols(k, 0, 6) for k in kfs])
        B = np.concatenate([Hpd[n][k] for k in kfs], axis=0)
        s = np.sqrt(inv[sl])
        F = fill(np.vstack([B * s, (g_d[sl] * s)[None]]), exact)
        H[np.ix_(cols, cols)] -= F[:-1, :-1]
        g[cols] -= F[:-1, -1]
    free = L.free_mask()
    Hf = H[np.ix_(free, free)]
    dxf = np.linalg.solve(Hf, -g[free])
    dx = np.zeros(L.npv)
    dx[free] = dxf
    dxd = inv * (-g_d)
    for n in range(L.K):
        if not Hpd[n]:
            continue
        sl = slice(L.doff[n], L.doff[n + 1])
        acc = -g_d[sl].copy()
        for k in sorted(Hpd[n]):
            acc -= Hpd[n][k].T @ dx[L.cols(k, 0, 6)]
        dxd[sl] = inv[sl] * acc
    return Hf, dx, dxd


def rel(a, b):
    s = np.abs(b).max()
    return float(np.abs(a - b).max() / s) if s > 0 else 0.0


def report(name, P, opts):
    H0, x0, d0 = step(P, opts, True)
    H1, x1, d1 = step(P, opts, False)
    print(f"{name}: H_red {rel(H1, H0):.2e}  dx {rel(x1, x0):.2e}  dx_d {rel(d1, d0):.2e}", flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["cfg"]:
        from paper_2512_02293_b200.problem import pack_graph
        from paper_2512_02293_b200.workloads import CONFIGS, make_workload
        for c in sys.argv[2:]:
            report(f"cfg{c}", pack_graph(make_workload(int(c))), {"max_iterations": CONFIGS[int(c)].iterations})
    else:
        import conftest
        for name in conftest.golden_names():
            P, _, opts = conftest.load_golden(name)
            report(name, P, opts)
