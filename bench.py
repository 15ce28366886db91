"""Benchmark: integral image + window sum on the BASELINE.json headline config.

Workload (BASELINE.json `metric`, configs[4] = C5): a 70,000 x 85,000 uint8
binary mask (5.95 Gpx; seeded synthetic stand-in, paper_2410_16291_b200/synthetic.py),
its integral image (uint64) AND the window sums w=256 stride 1 (69,745 x 84,745
uint64 outputs).  One step = one pass of the hot path over the whole image:

  N = 1: one ssb_sat_build_swa call -- the table build (ssb_sat_build) on the
  step's stream and, concurrently on a forked stream, the window sums from the
  raster (ssb_window_fused); same table and same outputs as the reference's
  build_sat + sweep_window_sums (pkg/src/satsweep/integral.py:109-116, :141-163).
  N > 1 (one rank per GPU): rank g owns a row band; the (w-1)-row halo arrives
  over NCCL P2P, the band's windows run on a side stream, and the GLOBAL table
  rows of the band are written with the carry row from an NCCL all-gather +
  exclusive scan of the bands' column totals (shard.swa_table_sharded) -- the
  same products as at N = 1, strong scaling of the fixed image.

`value` is device-resident throughput (input already in HBM, outputs
preallocated; inputs 5.95 GB >> 126 MB L2, so no flush is needed); `e2e` runs
the public API with pinned host buffers (host->device input copy and
device->host result copy inside every timed step).  `--impl reference` times
the reference itself (`satsweep` installed under baseline/_ref, its
bench.run_timed("parallel") on all host cores) on a bounded band of the same
workload; `configs` holds C1-C4 through the public API (device-resident).

`python bench.py --gpus N` relaunches itself under torch.distributed.run with N
ranks when WORLD_SIZE is not set.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

ROWS, COLS, W = 70000, 85000, 256
OUT_R, OUT_C = ROWS - W + 1, COLS - W + 1
METRIC = "Gpixels/s (integral image + window sum) at 70k×85k; % HBM roofline; 1/2/4/8 GPU"
UNIT = "Gpixels/s"
WORKLOAD = "C5 70000x85000 u8 mask, integral image (u64) + window sum w=256 stride 1"


def peaks() -> dict:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in rows for n, v in zip(names, r[3]) if v.lower().startswith("active")})
        loaded = [r for r in rows if r[2] > 300.0] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "power_w_max": max(r[2] for r in rows)}




# ----------------------------------------------------------------------------- helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def emit(obj: dict) -> None:
    print(json.dumps(obj), flush=True)


def relaunch(n: int) -> int:
    """Re-run this script as N ranks (one per GPU) under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- CPU reference
class Reference:
    """The reference implementation on the host cores.

    Preferred: the reference package itself, installed unmodified under
    baseline/_ref (`pip install --target baseline/_ref`), called through its
    own benchmark entry point satsweep.bench.run_timed (bench.py:79-105), which
    times the build and query phases of swa_parallel (all os.cpu_count()
    workers, parallel.py:71-72) or the sequential swa_integral.  If it is not
    installed, the numpy restatement oracle/satsweep_oracle.swa_threaded stands
    in (kind "port")."""

    def __init__(self):
        self.kind = "port"
        self.mod = None
        ref = REPO / "baseline" / "_ref"
        if (ref / "satsweep" / "bench.py").exists():
            sys.path.insert(0, str(ref))
            import satsweep
            import satsweep.bench

            if Path(satsweep.__file__).resolve().is_relative_to(ref.resolve()):
                self.mod = satsweep
                self.kind = "reference"
        self._bands: dict = {}

    def band(self, out_rows: int) -> np.ndarray:
        """Input rows of C5 output rows [0, out_rows) (generated once, untimed)."""
        from paper_2410_16291_b200 import synthetic

        if out_rows not in self._bands:
            self._bands[out_rows] = synthetic.c5(0, out_rows + W - 1, threads=os.cpu_count() or 1)
        return self._bands[out_rows]

    def run(self, out_rows: int, method: str = "parallel") -> dict:
        """One timed run on a band; returns seconds (build/query split when the reference runs)."""
        band = self.band(out_rows)
        if self.mod is not None:
            sb = self.mod
            img = sb.ImageGrid(band)
            r = sb.bench.run_timed(method, img, sb.WindowSpec(W), sb.StatKind.SUM, threads=0)
            res = {"s": r.total_s, "build_s": r.build_s, "query_s": r.query_s, "workers": r.workers}
            del r
            return res
        from oracle import satsweep_oracle as oracle

        t0 = time.perf_counter()
        out = oracle.swa_threaded(band, W, "sum", 1, (os.cpu_count() or 1) if method == "parallel" else 1)
        dt = time.perf_counter() - t0
        del out
        return {"s": dt, "workers": (os.cpu_count() or 1) if method == "parallel" else 1}

    @staticmethod
    def pixels(out_rows: int) -> float:
        """Pixel credit of a band: its share of the image's output rows x the image's pixels."""
        return out_rows / OUT_R * ROWS * COLS

    def describe(self) -> str:
        if self.kind == "reference":
            return "satsweep (the reference, baseline/_ref) bench.run_timed"
        return "oracle/satsweep_oracle.swa_threaded (numpy restatement of satsweep.swa_parallel)"


def cores() -> dict:
    try:
        import psutil

        phys = psutil.cpu_count(logical=False)
    except Exception:  # pragma: no cover
        phys = None
    return {"logical": os.cpu_count(), "physical": phys}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    ref = Reference()
    out_rows = args.ref_rows
    ref.band(out_rows)
    times = []
    for i in range(args.warmup + args.steps):
        r = ref.run(out_rows, "parallel")
        if i >= args.warmup:
            times.append(r["s"])
    t = statistics.median(times)
    v = ref.pixels(out_rows) / t / 1e9
    c = cores()
    sample = (f"C5 output rows [0, {out_rows}) ({out_rows + W - 1} input rows x {COLS} cols) per step, credited "
              f"{out_rows}/{OUT_R} of the image's {ROWS * COLS} px; {ref.describe()}('parallel', threads=0 -> "
              f"{c['logical']} workers); value from the median step")
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
          "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
          "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded C5 recipe)",
          "config": {"workload": WORKLOAD, "sample_rows": out_rows},
          "step_s": times,
          "cpu_baseline": {"value": v, "unit": UNIT, "cores": c["logical"], "physical_cores": c["physical"],
                           "kind": ref.kind, "sample": sample},
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


def cpu_baseline(args) -> dict:
    """The reference on a bounded sample (rank 0, N = 1): median of 3 parallel
    runs on all host cores plus one single-thread run ("integral")."""
    ref = Reference()
    par = [ref.run(args.cpu_rows, "parallel") for _ in range(max(1, args.cpu_reps))]
    t = statistics.median(r["s"] for r in par)
    seq = ref.run(args.cpu_rows_seq, "integral")
    c = cores()
    return {"value": ref.pixels(args.cpu_rows) / t / 1e9, "unit": UNIT, "cores": c["logical"],
            "physical_cores": c["physical"], "kind": ref.kind,
            "sample": (f"median of {len(par)} runs of {ref.describe()}('parallel', threads=0) on C5 output rows "
                       f"[0, {args.cpu_rows}) ({args.cpu_rows + W - 1} input rows), credited {args.cpu_rows}/{OUT_R} "
                       f"of the image"),
            "runs_s": [r["s"] for r in par],
            "build_query_s": [[r.get("build_s"), r.get("query_s")] for r in par],
            "single_thread": {"value": ref.pixels(args.cpu_rows_seq) / seq["s"] / 1e9, "unit": UNIT, "cores": 1,
                              "method": "integral", "sample_rows": args.cpu_rows_seq, "s": seq["s"],
                              "build_s": seq.get("build_s"), "query_s": seq.get("query_s")}}


# ----------------------------------------------------------------------------- C1-C4 CPU reference samples
# per config, the reference itself on the host cores -- C1 and C2
# whole (C2 as its uint16 cast, SUM and MEAN as the separate calls the
# reference makes), C3's multi_window (single-threaded in the reference,
# integral.py:209) and C4's MEAN and STD on bounded row bands, credited with
# the band's share of the image's output rows.
CPU_SAMPLES = {
    "C1": (None, 50, ("sum",), "parallel"),
    "C2": (None, 100, ("sum", "mean"), "parallel"),
    "C3": (3000, None, None, "multi_window"),
    "C4": (4000, 64, ("mean", "std"), "parallel"),
}


def cpu_config_sample(ref, name: str, host: np.ndarray) -> dict:
    rows_in, w, stats, method = CPU_SAMPLES[name]
    sb = ref.mod
    x = host if rows_in is None else host[:rows_in]
    if name == "C2":
        x = x.astype(np.uint16)  # the reference has no int32 kind; counts fit uint16
    t0 = time.perf_counter()
    if method == "multi_window":
        ws_ = [25, 50, 100, 200, 400]
        sb.multi_window(x, ws_, "sum")
        out_rows, full_rows = x.shape[0] - 400 + 1, host.shape[0] - 400 + 1
        parts = None
    else:
        img = sb.ImageGrid(x)
        parts = {}
        for st in stats:
            r = sb.bench.run_timed(method, img, sb.WindowSpec(w), sb.StatKind.parse(st), threads=0)
            parts[st] = r.total_s
        out_rows, full_rows = x.shape[0] - w + 1, host.shape[0] - w + 1
    s = time.perf_counter() - t0
    px = out_rows / full_rows * host.shape[0] * host.shape[1]
    return {"s": s, "gpx_s": px / s / 1e9, "sample_rows": int(x.shape[0]), "calls_s": parts,
            "method": method, "kind": ref.kind}


# ----------------------------------------------------------------------------- C1-C4 through the public API
def run_configs(args, dev, pk) -> dict:
    """BASELINE configs C1-C4, device-resident, through the public API (auto
    pipelines), K timed calls each bracketed by CUDA events on the API's stream."""
    import torch

    import paper_2410_16291_b200 as sb
    from paper_2410_16291_b200 import _lib, synthetic

    res = {}
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        l0 = _lib.launch_count()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) / steps, (_lib.launch_count() - l0) / steps

    cases = [
        ("C1", "2048x2048 u8 Bernoulli(0.05), sum w=50", synthetic.c1, lambda x: sb.swa(x, 50, "sum"),
         lambda r, c: r * c + (r - 49) * (c - 49) * 8),
        ("C2", "10000x10000 int32 Thomas counts, sum + mean w=100", synthetic.c2,
         lambda x: sb.swa_stats(x, 100, ("sum", "mean")), lambda r, c: r * c * 4 + 2 * (r - 99) * (c - 99) * 8),
        ("C3", "30000x30000 u8 mask, sums for w in 25/50/100/200/400 from one table", synthetic.c3,
         lambda x: sb.multi_window(x, [25, 50, 100, 200, 400], "sum"),
         lambda r, c: r * c + sum((r - w + 1) * (c - w + 1) * 8 for w in (25, 50, 100, 200, 400))),
        ("C4", "20000x24000 f32 lognormal, mean + std w=64 (fp64)", synthetic.c4,
         lambda x: sb.swa_stats(x, 64, ("mean", "std")), lambda r, c: r * c * 4 + 2 * (r - 63) * (c - 63) * 8),
    ]
    ref = Reference() if not args.no_cpu else None
    for name, desc, gen, call, floor in cases:
        try:
            host = gen()
            x = torch.from_numpy(host).to(dev)
            r, c = host.shape
            cpu = None
            if ref is not None and ref.mod is not None:
                try:
                    cpu = cpu_config_sample(ref, name, host)
                except Exception as exc:  # pragma: no cover - reporting only
                    cpu = {"error": repr(exc)}
            del host
            steps = 20 if name == "C1" else max(3, args.steps // 2)
            ms, launches = timed(lambda: call(x), steps)
            fb = floor(r, c)
            res[name] = {"workload": desc, "ms_per_call": ms, "gpx_s": r * c / (ms * 1e-3) / 1e9, "steps": steps,
                         "floor_bytes": fb, "floor_frac": fb / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                         "launches_per_call": launches,
                         "floor": "input read once + every output written once (the fused-pipeline floor, SURVEY 8d)"}
            if cpu is not None:
                res[name]["cpu_reference"] = cpu
                if "gpx_s" in cpu:
                    res[name]["vs_cpu_reference"] = res[name]["gpx_s"] / cpu["gpx_s"]
            del x
            sb.release_scratch()
        except Exception as exc:  # pragma: no cover - reporting only
            res[name] = {"error": repr(exc)}
    return res


# ----------------------------------------------------------------------------- our arm
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-rows", type=int, default=16384, help="output rows per reference step (bounded sample)")
    ap.add_argument("--cpu-rows", type=int, default=16384, help="output rows of the cpu_baseline sample")
    ap.add_argument("--cpu-rows-seq", type=int, default=4096, help="output rows of the single-thread sample")
    ap.add_argument("--cpu-reps", type=int, default=3, help="parallel runs of the cpu_baseline sample (median)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other pipelines' lines")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))

    import torch

    from paper_2410_16291_b200 import _device, _lib, shard, synthetic
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    kind = ElemKind.U8
    pk = peaks()

    # ---- inputs: this rank's owned rows, generated on the host, copied once (untimed)
    a_own, b_own = shard.window_input_bands(ROWS, W, 1, world)[rank]
    t_gen = time.perf_counter()
    host_band = synthetic.c5(a_own, b_own, threads=os.cpu_count() or 1)
    gen_s = time.perf_counter() - t_gen
    # zero-copy halo layout: the band lives at the head of a buffer with room
    # for its halo, which NCCL receives in place each step (no concatenation)
    storage, x_own = shard.band_storage(ROWS, COLS, W, 1, torch.uint8, dev)
    x_own.copy_(torch.from_numpy(host_band))
    del host_band
    need = shard.window_needed_rows(ROWS, W, 1, world)[rank]
    nr = need[1] - need[0]
    own_r = b_own - a_own
    out_lo, out_hi = shard.output_partition(OUT_R, world)[rank]
    n_out = out_hi - out_lo
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    from paper_2410_16291_b200 import _engine

    ld = _engine.sat_ld_for(COLS)
    if world == 1:
        sat = _device.empty((ROWS + 1, ld), np.uint64, dev, "table")
        out = _device.empty((OUT_R, OUT_C), np.uint64, dev, "result")
        ws_bytes = max(int(lib.ssb_sat_workspace_bytes(kind.abi_code, ROWS, COLS, 0)),
                       int(lib.ssb_sat_swa_workspace_bytes(kind.abi_code, ROWS, COLS)))
        ws = _device.empty((ws_bytes,), np.uint8, dev, "workspace")

        def step():
            # the timed step: one ssb_sat_build_swa call -- the table build on
            # this stream and, concurrently on the library's forked side stream,
            # the window sums from the raster, joined back before it returns
            _lib.check(lib.ssb_sat_build_swa(x_own.data_ptr(), kind.abi_code, ROWS, COLS, COLS, sat.data_ptr(), ld,
                                             W, _lib.SUM, out.data_ptr(), None, OUT_C, ws.data_ptr(), ws_bytes, sptr))
    else:
        backend = shard.CudaBackend(dev)

        def step():
            # the timed step at N > 1: halo (NCCL P2P) -> windows on a side
            # stream || band totals -> NCCL all-gather -> carry -> global table rows
            shard.swa_table_sharded(x_own, ROWS, COLS, kind, W, (StatKind.SUM,), backend, storage=storage)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = _lib.launch_count()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            step()
        stop.record(stream)
        barrier()
    launches = _lib.launch_count() - launches0
    ms_total = start.elapsed_time(stop)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        lt = torch.tensor([launches], device=dev, dtype=torch.int64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    ms_step = ms_total / args.steps

    # ---- algorithmic bytes: the image read once, the table and
    # the window sums written once (17 B/px at C5)
    px = ROWS * COLS
    tab_bytes = (ROWS + 1) * (COLS + 1) * 8
    out_bytes = OUT_R * OUT_C * 8
    b_alg = px + tab_bytes + out_bytes
    b_mat = px + 2 * tab_bytes + out_bytes  # the reference structure (table written, then read back)
    value = px / (ms_step * 1e-3) / 1e9
    achieved = b_alg / (ms_step * 1e-3) / 1e9
    peak_all = pk["hbm_gbs"] * world
    traffic = None
    tfile = REPO / "profiles" / "traffic.json"
    if tfile.exists():
        tr = json.loads(tfile.read_text())
        traffic = tr.get("step_total")
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded C5 recipe, synthetic.py)",
        "config": {"workload": WORKLOAD,
                   "pipeline": ("ssb_sat_build_swa: ssb_sat_build || ssb_window_fused on a forked stream, joined"
                                if world == 1 else
                                "row bands: NCCL halo -> ssb_window_fused (side stream) || ssb_sat_prepare -> NCCL "
                                "all-gather -> ssb_band_carry -> ssb_sat_finish (global table rows)"),
                   "parallelism": f"rowband{world}",
                   "l2": "inputs 5.95 GB >> 126 MB L2; no flush needed", "gen_s": round(gen_s, 1)},
        "roofline": {"bound": "hbm", "achieved": achieved / world, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peak_all, "traffic": traffic,
                     "traffic_over_algorithmic": (traffic / b_alg) if traffic else None,
                     "kernel": "one step: ssb_sat_build (table) || ssb_window_fused (window sums), concurrent",
                     "bytes_per_launch": b_alg, "ms_per_launch": ms_step,
                     "bytes": "image read once + table written once + window sums written once (17 B/px); "
                              "per GPU at N > 1",
                     "peak_source": pk["source"]},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    # rows of the timed step's window sums, kept for a cross-check of the e2e (host path) result below
    check_rows = [0, 1, OUT_R // 3, OUT_R // 2 + 7, OUT_R - 1]
    dev_rows = out[check_rows].cpu().numpy().view(np.uint64) if world == 1 else None

    if world == 1 and not args.no_extra:
        # per-kernel times in context: the same launches issued from here with
        # events around each kernel group (untimed pass)
        side = torch.cuda.Stream(dev)
        ev = {"build": [], "windows": []}
        for i in range(args.warmup + args.steps):
            e0, e1, f0, f1 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            e0.record(stream)
            side.wait_event(e0)
            _lib.check(lib.ssb_sat_build(x_own.data_ptr(), kind.abi_code, ROWS, COLS, COLS, sat.data_ptr(), None,
                                         ld, None, None, ws.data_ptr(), ws_bytes, None, sptr))
            e1.record(stream)
            f0.record(side)
            _lib.check(lib.ssb_window_fused(x_own.data_ptr(), kind.abi_code, ROWS, COLS, COLS, W, _lib.SUM,
                                            out.data_ptr(), None, None, OUT_C, None, 0, side.cuda_stream))
            f1.record(side)
            stream.wait_event(f1)
            if i >= args.warmup:
                ev["build"].append((e0, e1))
                ev["windows"].append((f0, f1))
        barrier()
        result["phases_ms"] = {k: sum(a.elapsed_time(b) for a, b in v) / len(v) for k, v in ev.items()}
        result["phases_ms"]["step"] = ms_step

        def time_steps(fn):
            for _ in range(3):
                fn()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(args.steps):
                fn()
            a1.record(stream)
            barrier()
            return a0.elapsed_time(a1) / args.steps

        def sweep_step():
            _lib.check(lib.ssb_sat_build(x_own.data_ptr(), kind.abi_code, ROWS, COLS, COLS, sat.data_ptr(), None, ld,
                                         None, None, ws.data_ptr(), ws_bytes, None, sptr))
            _lib.check(lib.ssb_window_eval(sat.data_ptr(), None, kind.abi_code, ROWS, COLS, ld, W, 1, _lib.SUM,
                                           out.data_ptr(), None, None, OUT_C, sptr))

        def onepass_step():
            _lib.check(lib.ssb_sat_build_swa_onepass(x_own.data_ptr(), kind.abi_code, ROWS, COLS, COLS,
                                                     sat.data_ptr(), ld, W, _lib.SUM, out.data_ptr(), None, OUT_C,
                                                     ws.data_ptr(), ws_bytes, sptr))

        def fused_step():
            _lib.check(lib.ssb_window_fused(x_own.data_ptr(), kind.abi_code, ROWS, COLS, COLS, W, _lib.SUM,
                                            out.data_ptr(), None, None, OUT_C, None, 0, sptr))

        for name, fn, b, api in (
                ("corner_sweep_pipeline", sweep_step, b_mat, "ssb_sat_build -> ssb_window_eval (table read back)"),
                ("onepass_pipeline", onepass_step, b_alg, "ssb_sat_build_swa_onepass"),
                ("fused_windows_only", fused_step, px + out_bytes, "ssb_window_fused (no table)")):
            try:
                ms = time_steps(fn)
                result[name] = {"value": px / (ms * 1e-3) / 1e9, "ms_per_step": ms, "bytes_per_step": b,
                                "roofline_frac": b / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], "api": api}
            except Exception as exc:  # pragma: no cover - reporting only
                result[name] = {"error": repr(exc)}
        del sat, ws, out
        torch.cuda.empty_cache()

    # ---- e2e through the public API with pinned host buffers: every rank runs
    # swa on its own input rows (band + halo) on its own GPU and reads back its
    # output band; the step time is the max over ranks
    if not args.no_e2e:
        try:
            import paper_2410_16291_b200 as sb

            if world > 1:
                del backend
            torch.cuda.empty_cache()
            x_need = shard.halo_exchange(x_own, ROWS, W, 1, storage=storage)
            host_in = torch.empty((nr, COLS), dtype=torch.uint8, pin_memory=True)
            for a in range(0, nr, 4096):
                host_in[a:a + 4096].copy_(x_need[a:a + 4096].cpu())
            host_out = torch.empty((max(n_out, 1), OUT_C), dtype=torch.int64, pin_memory=True)
            hin = host_in.numpy()
            hout = host_out.numpy().view(np.uint64)[:n_out]

            def e2e_step():
                if n_out > 0:
                    sb.swa(hin, W, "sum", pipeline="table", out=hout, devices=[local])

            e2e_step()  # warm-up
            times = []
            for _ in range(args.e2e_steps):
                barrier()
                t0 = time.perf_counter()
                e2e_step()
                times.append(time.perf_counter() - t0)
            te = statistics.median(times)
            h2d, d2h = nr * COLS, n_out * OUT_C * 8
            wire = {}
            if n_out > 0:
                # what actually crossed PCIe: since w^2 * 255 < 2^32, ssb_swa_host sends the sums as uint32, or
                # uint16 for bands whose largest sum is below 2^16, and widens them into the uint64 result on the host
                c_h2d, c_d2h = ctypes.c_int64(), ctypes.c_int64()
                lib.ssb_host_last_copy_bytes(ctypes.byref(c_h2d), ctypes.byref(c_d2h))
                h2d, d2h = int(c_h2d.value), int(c_d2h.value)
                wire["bits_per_sum"] = 8.0 * d2h / (n_out * OUT_C)  # 16 / 32 per band, 64 = straight copy
                if d2h < n_out * OUT_C * 8 and world == 1:
                    # the same call at the wider wire formats, for the record (best of 2 after a warm-up)
                    for bits in (32, 64):
                        lib.ssb_host_wire(bits)
                        try:
                            e2e_step()
                            tw = []
                            for _ in range(2):
                                t0 = time.perf_counter()
                                e2e_step()
                                tw.append(time.perf_counter() - t0)
                            lib.ssb_host_last_copy_bytes(ctypes.byref(c_h2d), ctypes.byref(c_d2h))
                        finally:
                            lib.ssb_host_wire(0)
                        wire[f"wire{bits}"] = {"value": px / min(tw) / 1e9, "s_per_step": min(tw),
                                               "d2h_bytes_per_step": int(c_d2h.value)}
            if world > 1:
                import torch.distributed as dist

                agg = torch.tensor([te, float(h2d), float(d2h)], dtype=torch.float64, device=dev)
                mx = agg[:1].clone()
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                dist.all_reduce(agg, op=dist.ReduceOp.SUM)
                te, h2d, d2h = float(mx.item()), int(agg[1].item()), int(agg[2].item())
            if dev_rows is not None:  # the host path's uint64 result against the device-resident step's, row for row
                wire["rows_equal_device_step"] = bool(np.array_equal(hout[check_rows], dev_rows))
            result["e2e"] = {"value": px / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
                             "d2h_bytes_per_step": d2h, "s_per_step": te, "steps_s": times,
                             "d2h_gbs": d2h / te / 1e9, "wire": wire,
                             "host_result_bytes_per_step": n_out * OUT_C * 8,
                             "api": "paper_2410_16291_b200.swa(pinned numpy, 256, 'sum', pipeline='table', out=pinned,"
                                    " devices=[this GPU]) -> ssb_swa_host (banded H2D, table + windows, D2H of the sums as "
                                    "uint32 -- uint16 for bands whose largest sum is below 2^16 -- since w^2*255 < 2^32, "
                                    "zero-extended into the pinned uint64 result by the library's host threads); per rank on its band + halo; median step, max over ranks"}
            del host_in, host_out, hin, hout
        except Exception as exc:  # pragma: no cover
            result["e2e"] = {"error": repr(exc)}

    # ---- C1-C4 through the public API (N = 1)
    if world == 1 and not args.no_configs:
        result["configs"] = run_configs(args, dev, pk)

    # ---- CPU baseline: the reference on a bounded band, rank 0 at N = 1
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            result["cpu_baseline"] = cpu_baseline(args)
        except Exception as exc:  # pragma: no cover
            result["cpu_baseline"] = {"error": repr(exc)}

    if rank == 0:
        emit(result)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
