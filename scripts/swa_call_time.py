"""Device time of the headline call (ssb_sat_build_swa) at C5, 3 x 20 calls (tuning only; pair with ab_run.sh)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2410_16291_b200 import _device, _engine, _lib, synthetic
rows, cols, w = 70000, 85000, 256
dev = torch.device("cuda", 0); lib = _lib.load()
x = _device.to_device(synthetic.c5(0, rows), dev)
ld = _engine.sat_ld_for(cols)
sat = _device.empty((rows + 1, ld), np.uint64, dev, "t"); out = _device.empty((rows - w + 1, cols - w + 1), np.uint64, dev, "o")
wsb = int(lib.ssb_sat_swa_workspace_bytes(0, rows, cols)); ws = _device.empty((wsb,), np.uint8, dev, "ws")
st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.check(lib.ssb_sat_build_swa(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), ld, w, 1, out.data_ptr(), None, cols - w + 1, ws.data_ptr(), wsb, st))
for _ in range(3): f()
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    print(f"ssb_sat_build_swa {a.elapsed_time(b) / 20:.3f} ms")
