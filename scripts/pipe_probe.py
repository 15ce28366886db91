import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2410_16291_b200 as sb
from paper_2410_16291_b200 import _device
dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
for dt, w in ((np.uint16, 100), (np.uint16, 256), (np.uint8, 50), (np.int32, 100), (np.uint8, 400)):
    x = (rng.integers(0, 3, size=(10000, 10000))).astype(dt)
    xd = _device.to_device(x, dev)
    for pipe in ("table", "fused"):
        for st in (("sum",), ("sum", "mean"), ("std",)) if dt != np.int32 else (("sum",), ("sum","mean")):
            f = lambda: sb.swa_stats(xd, w, st, pipeline=pipe)
            f(); f(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): f()
            e1.record(); torch.cuda.synchronize()
            print(np.dtype(dt).name, w, pipe, st, round(e0.elapsed_time(e1) / 10, 3), "ms", flush=True)
