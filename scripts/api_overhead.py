"""Where does the public-API time go? (diagnostics)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_16291_b200 as sb  # noqa: E402
from paper_2410_16291_b200 import _device, _engine, synthetic  # noqa: E402

rows = int(os.environ.get("ROWS", "70000"))
x = _device.to_device(synthetic.bernoulli_rows(5, rows, 85000, 0.01), torch.device("cuda", 0))
def api():
    for pipe in ("table", "fused"):
        for i in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = sb.swa_stats(x, 256, ("sum",), pipeline=pipe)
            t1 = time.perf_counter()
            e1.record()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            print(f"{pipe} call {i}: host {1e3 * (t1 - t0):8.2f} ms, device {e0.elapsed_time(e1):8.2f} ms, wall {1e3 * (t2 - t0):8.2f} ms", flush=True)
            del r


def raw():
    # raw C-ABI sequence (as bench.py) in the same process
    from paper_2410_16291_b200 import _lib  # noqa: E402
    lib = _lib.load()
    R, C, W = rows, 85000, 256
    ld = _engine.sat_ld_for(C)
    sat = _device.empty((R + 1, ld), np.uint64, x.device, "t")
    out = _device.empty((R - W + 1, C - W + 1), np.uint64, x.device, "o")
    wsb = int(lib.ssb_sat_workspace_bytes(0, R, C, 0))
    ws = _device.empty((wsb,), np.uint8, x.device, "w")
    st = torch.cuda.current_stream().cuda_stream
    for i in range(4):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        _lib.check(lib.ssb_sat_prepare(x.data_ptr(), 0, R, C, C, 0, ws.data_ptr(), wsb, None, None, None, st))
        e[1].record()
        _lib.check(lib.ssb_sat_finish(x.data_ptr(), 0, R, C, C, sat.data_ptr(), None, ld, None, None, ws.data_ptr(), wsb, st))
        e[2].record()
        _lib.check(lib.ssb_window_eval(sat.data_ptr(), None, 0, R, C, ld, W, 1, 1, out.data_ptr(), None, None, C - W + 1, st))
        e[3].record()
        torch.cuda.synchronize()
        print(f"raw {i}: prep {e[0].elapsed_time(e[1]):.2f} fin {e[1].elapsed_time(e[2]):.2f} eval {e[2].elapsed_time(e[3]):.2f} total {e[0].elapsed_time(e[3]):.2f}", flush=True)
    del sat, out, ws
    for i in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        img = sb.ImageGrid(x)
        s, q, ldd = _engine.build_tables(x, img.elem_kind, R, C, x.device, squared=False)
        e[1].record()
        o = _engine.eval_tables(s, q, ldd, img.elem_kind, R, C, W, 1, [sb.StatKind.SUM], x.device)
        e[2].record()
        torch.cuda.synchronize()
        print(f"engine {i}: build {e[0].elapsed_time(e[1]):.2f} eval {e[1].elapsed_time(e[2]):.2f}", flush=True)
        del s, o


if os.environ.get('RAW_FIRST'):
    raw(); api()
else:
    api(); raw()
