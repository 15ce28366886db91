"""e2e probe: pinned PCIe ceilings and ssb_swa_host at C5 (band rows / buffer sets from argv/env).

python scripts/e2e_probe.py [band_rows ...]   (SSB_HOST_SETS selects the buffer-set count)"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_16291_b200 as sb  # noqa: E402
from paper_2410_16291_b200 import _engine, synthetic  # noqa: E402
from paper_2410_16291_b200.grid import ImageGrid, StatKind  # noqa: E402


def pcie(nbytes=4 << 30, streams=1, reps=3):
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = nbytes // streams
    res = {}
    for name, fn in (("d2h", lambda s, a, b: h[a:b].copy_(d[a:b], non_blocking=True)),
                     ("h2d", lambda s, a, b: d[a:b].copy_(h[a:b], non_blocking=True))):
        best = 0
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for k, s in enumerate(ss):
                with torch.cuda.stream(s):
                    fn(s, k * chunk, (k + 1) * chunk)
            torch.cuda.synchronize()
            best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
        res[name] = best
    del d, h
    return res


def main():
    bands = [int(a) for a in sys.argv[1:]] or [0]
    if os.environ.get("E2E_SKIP_PCIE"):
        return run_bands(bands)
    # a C5-sized result read-back (47.3 GB) as one stream of 1.4 GB copies: the sustained ceiling
    d = torch.empty(1400 << 20, dtype=torch.uint8, device="cuda")
    big = torch.empty((34, 1400 << 20), dtype=torch.uint8, pin_memory=True)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(34):
            big[k].copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"sustained_d2h_47GB_s": ts, "gbs": [34 * (1400 << 20) / t / 1e9 for t in ts]}), flush=True)
    del big, d
    print(json.dumps({"pcie_1stream": pcie(streams=1), "pcie_2streams": pcie(streams=2),
                      "sets": os.environ.get("SSB_HOST_SETS", "default")}), flush=True)
    run_bands(bands)


def run_bands(bands):
    img = synthetic.c5(threads=os.cpu_count())
    hin = torch.empty(img.shape, dtype=torch.uint8, pin_memory=True)
    hin.numpy()[...] = img
    del img
    out_r, out_c = 70000 - 255, 85000 - 255
    hout = torch.empty((out_r, out_c), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    grid = ImageGrid(hin.numpy(), _check_finite=False)
    for br in bands:
        ts = []
        for _ in range(int(os.environ.get("E2E_REPS", "3"))):
            t0 = time.perf_counter()
            _engine.run_host(grid, 256, 1, [StatKind.SUM], "table", outs={StatKind.SUM: hout}, band_rows=br)
            ts.append(time.perf_counter() - t0)
        print(json.dumps({"band_rows": br, "s": ts, "min": min(ts), "median": sorted(ts)[len(ts) // 2],
                          "gpx_s": 5.95 / min(ts), "d2h_gbs": out_r * out_c * 8 / min(ts) / 1e9}),
              flush=True)


if __name__ == "__main__":
    main()
