"""Front-door throughput (reporting only): PGM/raw file -> device raster.

Compares read_pgm(device="cuda") (ssb_file_to_device: pinned double-buffered
staging, parallel preads) with the reference-style route (whole-file bytes ->
numpy -> torch H2D).  The file is written first, so both read from the page
cache; the GB/s are payload bytes over wall time."""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16291_b200 import imgio  # noqa: E402

rows, cols = int(os.environ.get("ROWS", 20000)), int(os.environ.get("COLS", 85000))
d = Path(tempfile.mkdtemp(dir=os.environ.get("IO_DIR", "/dev/shm")))
for maxval in (255, 65535):
    dt = np.uint8 if maxval <= 255 else np.uint16
    a = np.random.default_rng(1).integers(0, maxval + 1, size=(rows, cols), dtype=dt)
    p = d / "x.pgm"
    body = a.tobytes() if dt == np.uint8 else a.astype(">u2").tobytes()
    p.write_bytes(f"P5\n{cols} {rows}\n{maxval}\n".encode() + body)
    del body
    nbytes = a.nbytes
    g = imgio.read_pgm(p, device="cuda")  # warm
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        del g
        t0 = time.perf_counter()
        g = imgio.read_pgm(p, device="cuda")
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t_native = min(ts)
    assert np.array_equal(g.values.cpu().numpy(), a)
    t0 = time.perf_counter()
    for _ in range(3):
        h = imgio.read_pgm(p)  # host numpy, like the reference
        x = torch.from_numpy(h.values.copy()).to("cuda")
    torch.cuda.synchronize()
    t_host = (time.perf_counter() - t0) / 3
    print(json.dumps({"format": f"pgm maxval {maxval}", "payload_GB": round(nbytes / 1e9, 2),
                      "native_GBps": round(nbytes / t_native / 1e9, 2), "native_s": [round(t, 3) for t in ts],
                      "chunk_mb": os.environ.get("SSB_IO_CHUNK_MB", "32"), "readers": os.environ.get("SSB_IO_READERS", "4"),
                      "host_numpy_then_h2d_GBps": round(nbytes / t_host / 1e9, 2)}), flush=True)
    p.unlink()
os.rmdir(d)
