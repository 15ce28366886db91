"""Sweep the corner-sweep kernel's L2 knobs on a resident C5 slice (tuning only)."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import _device, _engine, _lib, synthetic  # noqa: E402

rows = int(os.environ.get("ROWS", "16384"))
C, W = 85000, 256
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, rows, C, 0.01), dev)
lib = _lib.load()
ld = _engine.sat_ld_for(C)
sat = _device.empty((rows + 1, ld), np.uint64, dev, "t")
ws_b = int(lib.ssb_sat_workspace_bytes(0, rows, C, 0))
ws = _device.empty((ws_b,), np.uint8, dev, "w")
st = torch.cuda.current_stream().cuda_stream
_lib.check(lib.ssb_sat_build(x.data_ptr(), 0, rows, C, C, sat.data_ptr(), None, ld, None, None, ws.data_ptr(), ws_b, None, st))
out_c = C - W + 1
out = _device.empty((rows - W + 1, out_c), np.uint64, dev, "o")
byts = (rows + 1) * (C + 1) * 8 + (rows - W + 1) * out_c * 8
grid = [tuple(c.split(",")) for c in os.environ["CONFIGS"].split(";")] if "CONFIGS" in os.environ else itertools.product(["12", "24", "48", "96"], ["0", "1", "2"], ["0", "32"])
for mb, h, k in grid:
    os.environ["SSB_EVAL_L2_MB"], os.environ["SSB_EVAL_HINTS"], os.environ["SSB_EVAL_ROWS_IN_FLIGHT"] = mb, h, k
    f = lambda: _lib.check(lib.ssb_window_eval(sat.data_ptr(), None, 0, rows, C, ld, W, 1, 1, out.data_ptr(), None, None, out_c, st))  # noqa
    f(); f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"L2_MB={mb:>3s} hints={h} k={k:>2s}: {ms:7.3f} ms  {byts / ms / 1e6:7.0f} GB/s", flush=True)
