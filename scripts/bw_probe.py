"""Bandwidth probes on the GPU (tuning only): torch copy of a table-sized buffer,
and the corner sweep with/without its top-row re-read."""
import os
import sys

import torch

n = int(os.environ.get("N", str(11 * 2**30 // 8)))
a = torch.empty(n, dtype=torch.int64, device="cuda")
b = torch.empty_like(a)
a.fill_(1)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"torch copy {2 * n * 8 / 1e9:.1f} GB: {ms:.3f} ms  {2 * n * 8 / ms / 1e6:.0f} GB/s", flush=True)
del a, b
