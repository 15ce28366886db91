"""Per-config device timing of the fused / table pipelines (C2, C4) for A/B and ncu.

python scripts/configs_probe.py C4 fused [steps]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_16291_b200 as sb  # noqa: E402
from paper_2410_16291_b200 import synthetic  # noqa: E402

CASES = {
    "C2": (synthetic.c2, 100, ("sum", "mean")),
    "C4": (synthetic.c4, 64, ("mean", "std")),
}


def c3(pipe, steps):
    x = torch.from_numpy(synthetic.c3()).to("cuda:0")
    ws = [25, 50, 100, 200, 400]
    for _ in range(2):
        sb.multi_window(x, ws, "sum", pipeline=pipe)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        sb.multi_window(x, ws, "sum", pipeline=pipe)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    floor = 30000 * 30000 + sum((30000 - w + 1) ** 2 * 8 for w in ws)
    print(json.dumps({"config": "C3", "pipeline": pipe, "ms": ms, "floor_GB": floor / 1e9,
                      "floor_frac": floor / (ms * 1e-3) / 6554.6e9}), flush=True)


def main():
    name, pipe = sys.argv[1], sys.argv[2]
    if name == "C3":
        return c3(pipe, int(sys.argv[3]) if len(sys.argv) > 3 else 10)
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    gen, w, stats = CASES[name]
    x = torch.from_numpy(gen()).to("cuda:0")
    for _ in range(2):
        sb.swa_stats(x, w, stats, pipeline=pipe)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        sb.swa_stats(x, w, stats, pipeline=pipe)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    r, c = x.shape
    floor = r * c * x.element_size() + len(stats) * (r - w + 1) * (c - w + 1) * 8
    print(json.dumps({"config": name, "pipeline": pipe, "ms": ms, "floor_GB": floor / 1e9,
                      "floor_frac": floor / (ms * 1e-3) / 6554.6e9}), flush=True)


if __name__ == "__main__":
    main()
