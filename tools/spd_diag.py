"""Diagnostics: tensor-core SPD solve error vs refinement passes (mode 2, no fallback)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02293_b200 import _lib  # noqa: E402

for n, cond in [(100, 1e3), (200, 1e2), (256, 1e2), (300, 1e3), (300, 1e6), (1000, 1e5)]:
    g = torch.Generator().manual_seed(n)
    Q, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64))
    ev = torch.logspace(0, float(np.log10(cond)), n, dtype=torch.float64)
    H = (Q * ev) @ Q.T
    H = 0.5 * (H + H.T)
    b = torch.randn(n, generator=g, dtype=torch.float64)
    ref = torch.linalg.solve(H, b)
    errs = []
    for it in (1, 2, 3, 4, 8):
        x, _ = _lib.spd_solve(H.cuda(), b.cuda(), mode=2, iters=it)
        errs.append(((x.cpu() - ref).abs().max() / ref.abs().max()).item())
    print(f"n={n} cond={cond:.0e}: " + " ".join(f"{e:.1e}" for e in errs), flush=True)

# timing: tensor-core (8 passes max) vs fp64 DAG
for n in (1905, 7665):
    g = torch.Generator().manual_seed(n)
    A = torch.randn(n, n, generator=g, dtype=torch.float64) / n ** 0.5
    H = (A @ A.T + torch.eye(n, dtype=torch.float64)).cuda()
    b = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    for mode in (2, 1):
        for it in range(3):
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            x, _ = _lib.spd_solve(H, b, mode=mode)
            t1.record()
            torch.cuda.synchronize()
        ref = torch.linalg.solve(H, b)
        err = ((x - ref).abs().max() / ref.abs().max()).item()
        print(f"n={n} mode={mode}: {t0.elapsed_time(t1):.2f} ms (incl. alloc/copies) err {err:.1e}", flush=True)
