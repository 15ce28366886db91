"""Phase breakdown of the single-pass table build (tuning only).

Builds a variant library with -DSSB_ONEPASS_PROF (globaltimer marks per tile
phase, thread 0 of each CTA) into /tmp, runs the C5 build a few times, and
prints the mean time per tile spent in each phase."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib_path = Path("/tmp/libssb_prof.so")
os.environ["SSB_LIB"] = str(lib_path)  # before the package binds its library path
from paper_2410_16291_b200 import build_ext  # noqa: E402

WORKERS = int(os.environ.get("WORKERS", 4))
build_ext.build(defines=("SSB_ONEPASS_PROF", f"SSB_ONE_WORKERS={WORKERS}"), lib=lib_path)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_16291_b200 import _device, _engine, _lib, synthetic  # noqa: E402
from paper_2410_16291_b200.grid import ElemKind  # noqa: E402

rows = int(os.environ.get("ROWS", 70000))
cols = 85000
lib = _lib.load()
lib.ssb_debug_onepass_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, rows, cols, 0.01, 0, rows), dev)
ld = _engine.sat_ld_for(cols)
sat = _device.empty((rows + 1, ld), np.uint64, dev, "t")
wsb = int(lib.ssb_sat_lookback_workspace_bytes(0, rows, cols, 0))
ws = _device.empty((wsb,), np.uint8, dev, "ws")
st = torch.cuda.current_stream().cuda_stream
buf = (ctypes.c_ulonglong * 8)()


def run():
    _lib.check(lib.ssb_sat_build_lookback(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), None, ld, None, None,
                                          ws.data_ptr(), wsb, st))


for _ in range(2):
    run()
torch.cuda.synchronize()
lib.ssb_debug_onepass_prof(buf, 1)
n = 3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    run()
e1.record()
torch.cuda.synchronize()
lib.ssb_debug_onepass_prof(buf, 0)
info = (ctypes.c_int64 * 4)()
SR = 16 * WORKERS
tiles = ((cols + 1 + 511) // 512) * ((rows + 1 + SR - 1) // SR)
names = ["ticket", "staged", "pass1", "hlookback", "ctl_publish_fence", "vlookback", "pass2", "ctl_hloop"]
per = {nm: buf[i] / (n * tiles) / 1000.0 for i, nm in enumerate(names)}
print(json.dumps({"workers": WORKERS, "ms_per_build": e0.elapsed_time(e1) / n, "tiles": tiles, "us_per_tile_by_phase": per,
                  "us_per_tile_total": sum(v for k, v in per.items() if not k.startswith("ctl"))}))
