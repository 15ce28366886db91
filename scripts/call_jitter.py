"""Per-call device time distribution through the public API (diagnostic).

Each call is bracketed by events with a synchronize on both sides, so host
gaps between calls are excluded; the spread shows kernel-side variance."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_16291_b200 as sb  # noqa: E402
from paper_2410_16291_b200 import _device, synthetic  # noqa: E402

dev = torch.device("cuda", 0)
for name in sys.argv[1:] or ["C2", "C4"]:
    cfg = synthetic.CONFIGS[name]
    x = _device.to_device(synthetic.generate(name), dev)
    if len(cfg.windows) > 1:
        fn = lambda: sb.multi_window(x, list(cfg.windows), cfg.stats[0])  # noqa: E731
    else:
        fn = lambda: sb.swa_stats(x, cfg.windows[0], cfg.stats)  # noqa: E731
    for _ in range(3):
        fn()
    ts = []
    for _ in range(int(os.environ.get("REPS", 30))):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"config": name, "min": round(ts[0], 3), "med": round(ts[len(ts) // 2], 3),
                      "max": round(ts[-1], 3), "all": [round(t, 2) for t in ts]}), flush=True)
    del x
    torch.cuda.empty_cache()
