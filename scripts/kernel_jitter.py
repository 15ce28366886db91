"""Per-kernel duration spread over repeated public-API calls (CUPTI via torch.profiler; diagnostic)."""
import collections
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_16291_b200 as sb  # noqa: E402
from paper_2410_16291_b200 import _device, synthetic  # noqa: E402

dev = torch.device("cuda", 0)
for name in sys.argv[1:] or ["C3", "C4"]:
    cfg = synthetic.CONFIGS[name]
    x = _device.to_device(synthetic.generate(name), dev)
    if len(cfg.windows) > 1:
        fn = lambda: sb.multi_window(x, list(cfg.windows), cfg.stats[0])  # noqa: E731
    else:
        fn = lambda: sb.swa_stats(x, cfg.windows[0], cfg.stats)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(int(os.environ.get("REPS", 30))):
            fn()
            torch.cuda.synchronize()
    kev = sorted((ev for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda e: e.time_range.start)
    gaps = collections.defaultdict(list)
    for a, b in zip(kev, kev[1:]):
        g = (b.time_range.start - a.time_range.end) / 1000.0
        gaps[(a.name[:40], b.name[:40])].append(g)
    for k, v in gaps.items():
        v.sort()
        print(json.dumps({"config": name, "gap_after": k[0], "before": k[1], "n": len(v), "med_ms": round(v[len(v) // 2], 3),
                          "max_ms": round(v[-1], 3), "top": [round(t, 2) for t in v[-4:]]}), flush=True)
    cpu = collections.defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CPU:
            cpu[ev.name[:50]].append(ev.cpu_time_total / 1000.0)
    for k, v in sorted(cpu.items(), key=lambda kv: -max(kv[1]))[:6]:
        v.sort()
        print(json.dumps({"config": name, "cpu_op": k, "n": len(v), "med_ms": round(v[len(v) // 2], 3),
                          "max_ms": round(v[-1], 3), "top": [round(t, 2) for t in v[-4:]]}), flush=True)
    per = collections.defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            per[ev.name[:60]].append(ev.device_time / 1000.0)
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        v.sort()
        print(json.dumps({"config": name, "kernel": k, "n": len(v), "min": round(v[0], 3),
                          "med": round(v[len(v) // 2], 3), "max": round(v[-1], 3)}), flush=True)
    del x
    torch.cuda.empty_cache()
