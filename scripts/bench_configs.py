"""Device-resident throughput of every BASELINE config (C1-C5) on both pipelines
(reporting only; bench.py is the contract line for C5).

Algorithmic bytes: table pipeline B_mat = in + 2 T n_tables + sum(out)
(in + T + out when the table is never read back: single-window integer sum/mean);
fused pipeline B_fused = in + sum(out).  T = (R+1)(C+1)*8."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_16291_b200 as sb  # noqa: E402
from paper_2410_16291_b200 import _device, synthetic  # noqa: E402
from bench import ClockSampler  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6443.2
dev = torch.device("cuda", 0)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    for name in names:
        cfg = synthetic.CONFIGS[name]
        t0 = time.time()
        x_host = synthetic.generate(name)
        gen = time.time() - t0
        x = _device.to_device(x_host, dev)
        R, C = x_host.shape
        es = x_host.dtype.itemsize
        del x_host
        n_tab = 2 if "std" in cfg.stats else 1
        T = (R + 1) * (C + 1) * 8
        for pipe in ("table", "fused"):
            if len(cfg.windows) > 1:
                fn = lambda: sb.multi_window(x, list(cfg.windows), cfg.stats[0], pipeline=pipe)  # noqa: E731
                outs = sum((R - w + 1) * (C - w + 1) * 8 for w in cfg.windows)
            else:
                w = cfg.windows[0]
                fn = lambda: sb.swa_stats(x, w, cfg.stats, pipeline=pipe)  # noqa: E731
                outs = len(cfg.stats) * (R - w + 1) * (C - w + 1) * 8
            try:
                with ClockSampler(0) as clk:
                    ms = timeit(fn, reps=int(os.environ.get("REPS", 3 if name in ("C3", "C5") else 5)))
            except Exception as exc:  # pragma: no cover
                print(json.dumps({"config": name, "pipeline": pipe, "error": str(exc)}), flush=True)
                continue
            nin = R * C * es * (len(cfg.windows) if (pipe == "fused") else 1)
            # single-window integer sum/mean: the table pipeline writes the table once and
            # never reads it back (ssb_sat_build_swa); otherwise the table is written and read
            from paper_2410_16291_b200 import _engine
            from paper_2410_16291_b200.grid import ElemKind, StatKind
            ek = ElemKind.from_dtype(np.dtype(str(x.dtype).split(".")[-1]))
            one = (len(cfg.windows) == 1 and R * C >= 1 << 24 and _engine.sweep_supported(
                ek, cfg.windows[0], 1, tuple(StatKind.parse(s_) for s_ in cfg.stats))
                and (ek is ElemKind.U8 and cfg.windows[0] <= 256 or ek is ElemKind.U16 and cfg.windows[0] <= 128))
            bytes_ = nin + ((T * n_tab if one else 2 * T * n_tab) if pipe == "table" else 0) + outs
            print(json.dumps({"config": name, "pipeline": pipe, "ms": round(ms, 3),
                              "gpx_s": round(R * C / ms / 1e6, 1), "alg_GB": round(bytes_ / 1e9, 2),
                              "roofline_frac": round(bytes_ / ms / 1e6 / PEAK, 3), "gen_s": round(gen, 1),
                              "alloc_retries": torch.cuda.memory_stats().get("num_alloc_retries", 0),
                              "clocks": clk.summary()}), flush=True)
            torch.cuda.empty_cache()
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
