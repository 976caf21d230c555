"""One tensor-core SPD solve (mode 2) of a synthetic n x n system, for kernel-level timing."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_02293_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 7665
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = torch.Generator().manual_seed(n)
A = torch.randn(n, n, generator=g, dtype=torch.float64) / n ** 0.5
H = (A @ A.T + torch.eye(n, dtype=torch.float64)).cuda()
b = torch.randn(n, generator=g, dtype=torch.float64).cuda()
x, _ = _lib.spd_solve(H, b, mode=mode)
torch.cuda.synchronize()
print("ok", n, mode)
