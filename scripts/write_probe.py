"""Write-only vs copy HBM bandwidth (tuning only)."""
import torch

n = 8 * 2**30 // 8
a = torch.empty(n, dtype=torch.int64, device="cuda")
b = torch.empty_like(a)


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = t(lambda: a.fill_(7))
print(f"fill  {n * 8 / 1e9:.1f} GB: {ms:.3f} ms {n * 8 / ms / 1e6:.0f} GB/s")
ms = t(lambda: a.zero_())
print(f"zero  {n * 8 / 1e9:.1f} GB: {ms:.3f} ms {n * 8 / ms / 1e6:.0f} GB/s")
ms = t(lambda: b.copy_(a))
print(f"copy  {2 * n * 8 / 1e9:.1f} GB: {ms:.3f} ms {2 * n * 8 / ms / 1e6:.0f} GB/s")
ms = t(lambda: a.sum())
print(f"read  {n * 8 / 1e9:.1f} GB: {ms:.3f} ms {n * 8 / ms / 1e6:.0f} GB/s")
