"""Device time of the fused (no-table) pipeline at C5 (tuning only)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import _device, _lib, synthetic  # noqa: E402

rows, cols, w = int(os.environ.get("ROWS", 70000)), 85000, int(os.environ.get("W", 256))
lib = _lib.load()
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, rows, cols, 0.01, 0, rows), dev)
oc = cols - w + 1
out = _device.empty((rows - w + 1, oc), np.uint64, dev, "o")
st = torch.cuda.current_stream().cuda_stream


def f():
    _lib.check(lib.ssb_window_fused(x.data_ptr(), 0, rows, cols, cols, w, _lib.SUM, out.data_ptr(), None, None, oc,
                                    None, int(os.environ.get("SEG", 0)), st))


for _ in range(3):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(8):
    f()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 8
print(json.dumps({"seg": os.environ.get("SEG", "0"), "w": w, "fused_ms": ms, "gpx_s": rows * cols / ms / 1e6}))
