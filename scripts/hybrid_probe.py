"""Would mixing the one-pass kernel with the concurrent build || fused pair pay?
C5 split into two 35,000-row halves (independent tables): half 1 through
ssb_sat_build_swa_onepass and half 2 through ssb_sat_build || ssb_window_fused,
all on separate streams at once, vs the pair on both halves (tuning only)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2410_16291_b200 import _device, _engine, _lib, synthetic

rows, cols, w = 70000, 85000, 256
h = rows // 2
dev = torch.device("cuda", 0)
lib = _lib.load()
x = _device.to_device(synthetic.c5(0, rows), dev)
ld = _engine.sat_ld_for(cols)
sat = _device.empty((rows + 2, ld), np.uint64, dev, "t")
oc = cols - w + 1
out = _device.empty((rows - w + 1, oc), np.uint64, dev, "o")
wsb = max(int(lib.ssb_sat_swa_workspace_bytes(0, h, cols)), int(lib.ssb_sat_workspace_bytes(0, h, cols, 0)))
ws = [_device.empty((wsb,), np.uint8, dev, "ws") for _ in range(2)]
xs = [x[:h], x[h:]]
sats = [sat[: h + 1], sat[h + 1: 2 * h + 2]]
outs = [out[: h - w + 1], out[h - w + 1: 2 * (h - w + 1)]]
S = [torch.cuda.Stream(dev) for _ in range(3)]
main = torch.cuda.current_stream(dev)


def onepass(i, st):
    _lib.check(lib.ssb_sat_build_swa_onepass(xs[i].data_ptr(), 0, h, cols, cols, sats[i].data_ptr(), ld, w, 1,
                                             outs[i].data_ptr(), None, oc, ws[i].data_ptr(), wsb, st.cuda_stream))


def build(i, st):
    _lib.check(lib.ssb_sat_build(xs[i].data_ptr(), 0, h, cols, cols, sats[i].data_ptr(), None, ld, None, None,
                                 ws[i].data_ptr(), wsb, None, st.cuda_stream))


def fused(i, st):
    _lib.check(lib.ssb_window_fused(xs[i].data_ptr(), 0, h, cols, cols, w, 1, outs[i].data_ptr(), None, None, oc,
                                    None, 0, st.cuda_stream))


def pair(i, st):
    _lib.check(lib.ssb_sat_build_swa(xs[i].data_ptr(), 0, h, cols, cols, sats[i].data_ptr(), ld, w, 1,
                                     outs[i].data_ptr(), None, oc, ws[i].data_ptr(), wsb, st.cuda_stream))


def run(tasks):
    e = torch.cuda.Event()
    e.record(main)
    for (fn, i), st in zip(tasks, S):
        st.wait_event(e)
        fn(i, st)
    for st in S[: len(tasks)]:
        ev = torch.cuda.Event()
        ev.record(st)
        main.wait_event(ev)


def timeit(fn, n=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(n):
        fn()
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print(f"pair(h1) then pair(h2), one stream: {timeit(lambda: (pair(0, main), pair(1, main))):.3f} ms")
print(f"pair(h1) || pair(h2): {timeit(lambda: run([(pair, 0), (pair, 1)])):.3f} ms")
print(f"onepass(h1) || build(h2) || fused(h2): {timeit(lambda: run([(onepass, 0), (build, 1), (fused, 1)])):.3f} ms")
print(f"onepass(h1) || onepass(h2): {timeit(lambda: run([(onepass, 0), (onepass, 1)])):.3f} ms")
print(f"onepass(h1) then onepass(h2): {timeit(lambda: (onepass(0, main), onepass(1, main))):.3f} ms")
