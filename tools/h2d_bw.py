"""Pinned host->device copy bandwidth for one e2e window of config 4 (611 MB), DESIGN.md §6."""
import torch, time
n = 611072648 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 611 MB pinned: {ms:.2f} ms = {611.07/ms:.1f} GB/s")
