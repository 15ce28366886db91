"""Does running the table build and the fused window kernel concurrently (two
streams) beat running them back to back?  C5, device-resident."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2410_16291_b200 import _device, _engine, _lib, synthetic

rows, cols, w = 70000, 85000, 256
dev = torch.device("cuda", 0)
lib = _lib.load()
x = _device.to_device(synthetic.c5(0, rows), dev)
ld = _engine.sat_ld_for(cols)
sat = _device.empty((rows + 1, ld), np.uint64, dev, "t")
out = _device.empty((rows - w + 1, cols - w + 1), np.uint64, dev, "o")
ws = _device.empty((int(lib.ssb_sat_workspace_bytes(0, rows, cols, 0)),), np.uint8, dev, "ws")
sa = torch.cuda.current_stream(dev)
sb_ = torch.cuda.Stream(dev, priority=int(os.environ.get("SIDE_PRIO", 0)))  # -1 = high priority
if os.environ.get("MAIN_PRIO"):
    sa = torch.cuda.Stream(dev, priority=int(os.environ["MAIN_PRIO"]))
    torch.cuda.set_stream(sa)


def build(st):
    _lib.check(lib.ssb_sat_build(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), None, ld, None, None,
                                 ws.data_ptr(), ws.numel(), None, st.cuda_stream))


def finish(st):  # phase 3 only, on carries left in the workspace by an earlier build (probe: a free reduce)
    _lib.check(lib.ssb_sat_finish(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), None, ld, None, None,
                                  ws.data_ptr(), ws.numel(), st.cuda_stream))


def fused(st):
    _lib.check(lib.ssb_window_fused(x.data_ptr(), 0, rows, cols, cols, w, 1, out.data_ptr(), None, None,
                                    cols - w + 1, None, int(os.environ.get("FSEG", 0)), st.cuda_stream))


def seq():
    build(sa)
    fused(sa)


def conc(order=0):
    e = torch.cuda.Event()
    e.record(sa)
    sb_.wait_event(e)
    if order == 0:
        build(sa)
        fused(sb_)
    else:
        fused(sb_)
        build(sa)
    e2 = torch.cuda.Event()
    e2.record(sb_)
    sa.wait_event(e2)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(sa)
    for _ in range(n):
        fn()
    b.record(sa)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print(f"sequential {timeit(seq):.3f} ms")
print(f"concurrent build-first {timeit(lambda: conc(0)):.3f} ms")
print(f"concurrent fused-first {timeit(lambda: conc(1)):.3f} ms")
def conc_finish():
    e = torch.cuda.Event()
    e.record(sa)
    sb_.wait_event(e)
    finish(sa)
    fused(sb_)
    e2 = torch.cuda.Event()
    e2.record(sb_)
    sa.wait_event(e2)


print(f"concurrent scan-only (probe: reduce + carries free) {timeit(conc_finish):.3f} ms")
print(f"build alone {timeit(lambda: build(sa)):.3f} ms  fused alone {timeit(lambda: fused(sa)):.3f} ms")
