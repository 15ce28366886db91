"""One ssb_window_fused call at C5 (u8 sums, w=256) for ncu (tuning only)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import _device, _lib, synthetic  # noqa: E402

R, C, W = int(os.environ.get("ROWS", 70000)), 85000, 256
lib = _lib.load()
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, R, C, 0.01, 0, R), dev)
out = _device.empty((R - W + 1, C - W + 1), np.uint64, dev, "o")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.check(lib.ssb_window_fused(x.data_ptr(), 0, R, C, C, W, _lib.SUM, out.data_ptr(), None, None, C - W + 1, None, 0, st))
torch.cuda.synchronize()
print("ok")
