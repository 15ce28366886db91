"""C5 device times (tuning only): table prepare (reduce + carries), scan
(ssb_sat_finish), the whole build, the fused windows alone, and the headline
step ssb_sat_build_swa (build || windows).  One JSON line; SSB_LIB picks a
library variant."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import _device, _engine, _lib, synthetic  # noqa: E402

R, C, W = int(os.environ.get("ROWS", 70000)), 85000, 256
OR, OC = R - W + 1, C - W + 1
lib = _lib.load()
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, R, C, 0.01, 0, R), dev)
ld = _engine.sat_ld_for(C)
sat = _device.empty((R + 1, ld), np.uint64, dev, "t")
out = _device.empty((OR, OC), np.uint64, dev, "o")
wsb = max(int(lib.ssb_sat_workspace_bytes(0, R, C, 0)), int(lib.ssb_sat_swa_workspace_bytes(0, R, C)))
ws = _device.empty((wsb,), np.uint8, dev, "ws")
st = torch.cuda.current_stream().cuda_stream


def prep():
    _lib.check(lib.ssb_sat_prepare(x.data_ptr(), 0, R, C, C, 0, ws.data_ptr(), wsb, None, None, None, st))


def fin():
    _lib.check(lib.ssb_sat_finish(x.data_ptr(), 0, R, C, C, sat.data_ptr(), None, ld, None, None, ws.data_ptr(), wsb, st))


def build():
    _lib.check(lib.ssb_sat_build(x.data_ptr(), 0, R, C, C, sat.data_ptr(), None, ld, None, None, ws.data_ptr(), wsb,
                                 None, st))


def windows():
    _lib.check(lib.ssb_window_fused(x.data_ptr(), 0, R, C, C, W, _lib.SUM, out.data_ptr(), None, None, OC, None, 0, st))


def step():
    _lib.check(lib.ssb_sat_build_swa(x.data_ptr(), 0, R, C, C, sat.data_ptr(), ld, W, _lib.SUM, out.data_ptr(), None,
                                     OC, ws.data_ptr(), wsb, st))


def t(fn, n=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n, 3)


def concurrent(n=8):
    """build on this stream, windows on a side stream, both forked from one event:
    (build end, windows end) relative to the fork, ms"""
    side = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    b_end, w_end = [], []
    for i in range(3 + n):
        e0, e1, f1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(cur)
        side.wait_event(e0)
        build()
        e1.record(cur)
        _lib.check(lib.ssb_window_fused(x.data_ptr(), 0, R, C, C, W, _lib.SUM, out.data_ptr(), None, None, OC, None, 0,
                                        side.cuda_stream))
        f1.record(side)
        cur.wait_event(f1)
        torch.cuda.synchronize()
        if i >= 3:
            b_end.append(e0.elapsed_time(e1))
            w_end.append(e0.elapsed_time(f1))
    return round(sum(b_end) / n, 3), round(sum(w_end) / n, 3)


prep()
res = {"lib": os.environ.get("SSB_LIB", "product"), "prepare": t(prep), "scan": t(fin), "build": t(build),
       "windows": t(windows), "step": t(step, 10), "concurrent_build_windows_end": concurrent()}
print(json.dumps(res), flush=True)
