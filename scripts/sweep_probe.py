"""Time the one-pass table + window sweep (ssb_sat_build_swa) against the two-kernel
table pipeline at BASELINE C5 (70,000 x 85,000 u8, w=256), device-resident.
Usage: python scripts/sweep_probe.py [rows]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2410_16291_b200 import _device, _engine, _lib, synthetic
from paper_2410_16291_b200.grid import ElemKind, StatKind

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 70000
cols, w = 85000, 256
dev = torch.device("cuda", 0)
lib = _lib.load()
x = _device.to_device(synthetic.c5(0, rows) if rows == 70000 else synthetic.bernoulli_rows(5, rows, cols, 0.01, 0, rows), dev)
ld = _engine.sat_ld_for(cols)
sat = _device.empty((rows + 1, ld), np.uint64, dev, "t")
out = _device.empty((rows - w + 1, cols - w + 1), np.uint64, dev, "o")
wsb = int(lib.ssb_sat_swa_workspace_bytes(0, rows, cols))
ws = _device.empty((max(wsb, int(lib.ssb_sat_workspace_bytes(0, rows, cols, 0))),), np.uint8, dev, "ws")
st = torch.cuda.current_stream(dev).cuda_stream


def sweep(fn=None):
    _lib.check((fn or lib.ssb_sat_build_swa)(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), ld, w, 1, out.data_ptr(),
                                     None, cols - w + 1, ws.data_ptr(), ws.numel(), st))


def two():
    _lib.check(lib.ssb_sat_build(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), None, ld, None, None,
                                 ws.data_ptr(), ws.numel(), None, st))
    _lib.check(lib.ssb_window_eval(sat.data_ptr(), None, 0, rows, cols, ld, w, 1, 1, out.data_ptr(), None, None,
                                   cols - w + 1, st))


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def prep():
    _lib.check(lib.ssb_sat_prepare(x.data_ptr(), 0, rows, cols, cols, 0, ws.data_ptr(), ws.numel(), None, None, None,
                                   st))


import os

def onepass():
    sweep(lib.ssb_sat_build_swa_onepass)


if os.environ.get("PROBE_FAST"):  # tuning: one-pass and its reduce phase only
    a, b = timeit(onepass), timeit(prep)
    print(f"one-pass {a:.3f} ms  reduce+carries {b:.3f} ms  sweep kernel {a - b:.3f} ms  {rows * cols / a / 1e6:.1f} Gpx/s")
    sys.exit(0)
two()
ref = out.clone()
reft = sat.view(torch.int64).sum(dim=1)  # per-row checksums (the table itself is 44 GiB)
sat.zero_()
onepass()
torch.cuda.synchronize()
print("equal outputs:", bool(torch.equal(out, ref)), "equal table row checksums:",
      bool(torch.equal(sat.view(torch.int64).sum(dim=1), reft)))
del ref, reft
for name, fn in (("build+sweep", two), ("one-pass", onepass), ("build+fused (ssb_sat_build_swa)", sweep)):
    ms = timeit(fn)
    px = rows * cols
    b = px + (rows + 1) * (cols + 1) * 8 + (rows - w + 1) * (cols - w + 1) * 8
    print(f"{name}: {ms:.3f} ms  {px / ms / 1e6:.1f} Gpx/s  one-pass bytes {b / 1e9:.1f} GB -> {b / ms / 1e6:.0f} GB/s")
