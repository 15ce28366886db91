"""End-to-end (pinned host in/out) C5 through ssb_swa_host: PCIe ceilings and band sizes (tuning only)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2410_16291_b200 import _lib, synthetic

rows, cols, w = 70000, 85000, 256
lib = _lib.load()
dev = torch.device("cuda", 0)
oc, orr = cols - w + 1, rows - w + 1
hin = torch.empty((rows, cols), dtype=torch.uint8, pin_memory=True)
hin.numpy()[:] = synthetic.c5()
hout = torch.empty((orr, oc), dtype=torch.int64, pin_memory=True)

g = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
hb = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
for name, fn in (("D2H", lambda: hb.copy_(g, non_blocking=True)), ("H2D", lambda: g.copy_(hb, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{name} pinned 4 GiB: {3 * (4 << 30) / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
del g, hb
torch.cuda.empty_cache()

for band in (0, 1024, 2048, 8192):
    def call():
        _lib.check(lib.ssb_swa_host(hin.data_ptr(), 0, rows, cols, cols, w, 1, 1, hout.data_ptr(), None, None, oc,
                                    0, 0, band))
    call()
    t = time.perf_counter()
    for _ in range(2):
        call()
    dt = (time.perf_counter() - t) / 2
    print(f"ssb_swa_host band_rows={band}: {dt:.3f} s  {rows * cols / dt / 1e9:.2f} Gpx/s  "
          f"(D2H-equivalent {orr * oc * 8 / dt / 1e9:.1f} GB/s)", flush=True)
