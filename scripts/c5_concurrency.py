"""C5 concurrency probe (tuning only): the table build (ssb_sat_prepare +
ssb_sat_finish) and the fused windows (ssb_window_fused) on two streams with
different priorities / launch orders / window segment counts; prints the
step time (fork to both done) for each variant.  SSB_LIB picks the library."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import _device, _engine, _lib, synthetic  # noqa: E402

R, C, W = 70000, 85000, 256
OR, OC = R - W + 1, C - W + 1
lib = _lib.load()
dev = torch.device("cuda", 0)
x = _device.to_device(synthetic.bernoulli_rows(5, R, C, 0.01, 0, R), dev)
ld = _engine.sat_ld_for(C)
sat = _device.empty((R + 1, ld), np.uint64, dev, "t")
out = _device.empty((OR, OC), np.uint64, dev, "o")
wsb = int(lib.ssb_sat_workspace_bytes(0, R, C, 0))
ws = _device.empty((wsb,), np.uint8, dev, "ws")


def prep(s):
    _lib.check(lib.ssb_sat_prepare(x.data_ptr(), 0, R, C, C, 0, ws.data_ptr(), wsb, None, None, None, s.cuda_stream))


def fin(s):
    _lib.check(lib.ssb_sat_finish(x.data_ptr(), 0, R, C, C, sat.data_ptr(), None, ld, None, None, ws.data_ptr(), wsb,
                                  s.cuda_stream))


def win(s, seg):
    _lib.check(lib.ssb_window_fused(x.data_ptr(), 0, R, C, C, W, _lib.SUM, out.data_ptr(), None, None, OC, None, seg,
                                    s.cuda_stream))


def run(name, pb, pw, order, seg=0, n=8):
    sb_ = torch.cuda.Stream(priority=pb)
    sw = torch.cuda.Stream(priority=pw)
    main = torch.cuda.current_stream()
    ts = []
    for i in range(3 + n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        mid = torch.cuda.Event()
        e0.record(main)
        sb_.wait_event(e0)
        sw.wait_event(e0)
        if order == "build_first":
            prep(sb_); fin(sb_); win(sw, seg)
        elif order == "win_first":
            win(sw, seg); prep(sb_); fin(sb_)
        elif order == "win_after_prep":
            prep(sb_); mid.record(sb_); sw.wait_event(mid); fin(sb_); win(sw, seg)
        main.wait_stream(sb_)
        main.wait_stream(sw)
        e1.record(main)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(json.dumps({"variant": name, "ms": round(sum(ts) / n, 3), "lib": os.environ.get("SSB_LIB", "product")}),
          flush=True)


for order in ("build_first", "win_first", "win_after_prep"):
    run(f"{order} equal", 0, 0, order)
    run(f"{order} build_hi", -1, 0, order)
    run(f"{order} win_hi", 0, -1, order)
for seg in (42, 60):
    run(f"build_first build_hi seg{seg}", -1, 0, "build_first", seg)
    run(f"build_first equal seg{seg}", 0, 0, "build_first", seg)
