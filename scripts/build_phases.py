"""Device time of the table-build phases at C5 (tuning only): ssb_sat_prepare
(reduce + carries), ssb_sat_finish (scan), and the single-pass look-back build."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import _device, _engine, _lib, synthetic  # noqa: E402

rows, cols = int(os.environ.get("ROWS", 70000)), 85000
lib = _lib.load()
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, rows, cols, 0.01, 0, rows), dev)
ld = _engine.sat_ld_for(cols)
sat = _device.empty((rows + 1, ld), np.uint64, dev, "t")
wsb = max(int(lib.ssb_sat_workspace_bytes(0, rows, cols, 0)), int(lib.ssb_sat_lookback_workspace_bytes(0, rows, cols, 0)))
ws = _device.empty((wsb,), np.uint8, dev, "ws")
st = torch.cuda.current_stream().cuda_stream


def prep():
    _lib.check(lib.ssb_sat_prepare(x.data_ptr(), 0, rows, cols, cols, 0, ws.data_ptr(), wsb, None, None, None, st))


def fin():
    _lib.check(lib.ssb_sat_finish(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), None, ld, None, None,
                                  ws.data_ptr(), wsb, st))


def one():
    _lib.check(lib.ssb_sat_build_lookback(x.data_ptr(), 0, rows, cols, cols, sat.data_ptr(), None, ld, None, None,
                                          ws.data_ptr(), wsb, st))


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
    return a.elapsed_time(b) / n


def pf():
    prep()
    fin()


print(json.dumps({"prepare_ms": t(prep), "prepare+finish_ms": t(pf), "lookback_ms": t(one)}))
