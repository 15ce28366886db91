"""Benchmark: integral image + window sum on the BASELINE.json headline config.

Workload (BASELINE.json `metric`, configs[4] = C5): a 70,000 x 85,000 uint8
binary mask (5.95 Gpx; seeded synthetic stand-in, paper_2410_16291_b200/synthetic.py),
integral image (uint64/int64) + window sum w=256 stride 1 (69,745 x 84,745
uint64 outputs).  One step = one pass of the hot path over the whole image:

  headline `value`: the launches of ssb_sat_build_swa -- ssb_sat_build (the
  integral image written to HBM) then ssb_window_fused (the window sums,
  evaluated from the raster instead of reading the table back).  Same table
  and same outputs as the reference's build_sat + sweep_window_sums
  (pkg/src/satsweep/integral.py:109-116, :141-163).  Also reported: the
  corner-sweep table pipeline (ssb_sat_build -> ssb_window_eval, the
  reference's structure), the one-pass kernel (ssb_sat_build_swa_onepass),
  and the fused window sums alone (no table).

`value` is device-resident throughput (input already in HBM, outputs
preallocated, inputs 5.95 GB >> 126 MB L2, so no flush is needed); `e2e` runs
the public API with pinned host buffers (host->device input copy and
device->host result copy inside every timed step).  `--impl reference` times
the reference algorithm (the numpy port under oracle/, all host threads) on a
bounded band of the same workload.

Multi-GPU: `python -m torch.distributed.run --nproc-per-node N bench.py --gpus N`
shards output rows across ranks (strong scaling of the fixed image); each rank
receives its (w-1)-row halo over NCCL inside the timed step.
"""

from __future__ import annotations

import argparse
import json
import os
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
METRIC = "Gpixels/s (integral image + window sum) at 70k×85k; % HBM roofline; 1/2/4/8 GPU"
UNIT = "Gpixels/s"


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


_BANDS: dict = {}


def cpu_port_band(out_rows: int, threads: int = 0):
    """Reference algorithm (oracle port) on output rows [0, out_rows) of C5; returns (seconds, pixels).

    The band is generated once per size (untimed) and reused across steps."""
    from oracle import satsweep_oracle as oracle
    from paper_2410_16291_b200 import synthetic

    if out_rows not in _BANDS:
        _BANDS[out_rows] = synthetic.c5(0, out_rows + W - 1)
    band = _BANDS[out_rows]
    t0 = time.perf_counter()
    res = oracle.swa_threaded(band, W, "sum", 1, threads or (os.cpu_count() or 1))
    dt = time.perf_counter() - t0
    del res
    # pixel credit: the band's own output rows' share of the image (halo rows are overhead)
    return dt, out_rows * COLS


# ----------------------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    out_rows = args.ref_rows
    times = []
    for i in range(args.warmup + args.steps):
        dt, px = cpu_port_band(out_rows, threads)
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    v = px / t / 1e9
    sample = (f"C5 band of {out_rows} output rows x {COLS} cols ({out_rows + W - 1} input rows) per step; "
              f"oracle/satsweep_oracle.swa_threaded (numpy restatement of satsweep.swa_parallel)")
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
          "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
          "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded C5 recipe)",
          "config": {"workload": "C5 70000x85000 u8, integral image + window sum w=256 stride 1",
                     "sample_rows": out_rows},
          "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ----------------------------------------------------------------------------- our arm
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-rows", type=int, default=16384, help="output rows per reference/CPU step")
    ap.add_argument("--cpu-rows", type=int, default=16384, help="output rows of the cpu_baseline sample")
    ap.add_argument("--cpu-reps", type=int, default=8, help="repetitions of the cpu_baseline sample (~10-30 s of CPU work)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--rows", type=int, default=ROWS, help="(debug) smaller image")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    from paper_2410_16291_b200 import _device, _engine, _lib, shard, synthetic
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    rows = args.rows
    kind = ElemKind.U8

    # ---- inputs: this rank's owned rows, generated on the host, copied once (untimed)
    a_own, b_own = shard.window_input_bands(rows, W, 1, world)[rank]
    t_gen = time.perf_counter()
    host_band = synthetic.c5(a_own, b_own) if rows == ROWS else synthetic.bernoulli_rows(5, rows, COLS, 0.01, a_own, b_own)
    gen_s = time.perf_counter() - t_gen
    # zero-copy halo layout: the band lives at the head of a buffer with room
    # for its halo, which NCCL receives in place each step (no concatenation)
    storage, x_own = shard.band_storage(rows, COLS, W, 1, torch.uint8, dev)
    x_own.copy_(torch.from_numpy(host_band))
    del host_band
    need = shard.window_needed_rows(rows, W, 1, world)[rank]
    nr = need[1] - need[0]
    out_lo, out_hi = shard.output_partition(rows - W + 1, world)[rank]
    n_out = out_hi - out_lo
    out_c = COLS - W + 1
    ld = _engine.sat_ld_for(COLS)
    sat = _device.empty((nr + 1, ld), np.uint64, dev, "table")
    out = _device.empty((n_out, out_c), np.uint64, dev, "result")
    ws_bytes = max(int(lib.ssb_sat_workspace_bytes(kind.abi_code, nr, COLS, 0)),
                   int(lib.ssb_sat_swa_workspace_bytes(kind.abi_code, nr, COLS)))
    ws = _device.empty((ws_bytes,), np.uint8, dev, "workspace")
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def get_x():
        if world == 1:
            return x_own
        return shard.halo_exchange(x_own, rows, W, 1, group, storage=storage)

    ev = {k: [] for k in ("build", "windows", "group", "group_phase")}

    side = torch.cuda.Stream(dev)

    def step(record: bool):
        # the timed step: one ssb_sat_build_swa call -- the table build
        # (reduce-then-scan; SSB_SAT_PATH=one selects the single-pass look-back
        # kernel) on this stream and, concurrently on the library's forked side
        # stream, the window sums from the raster, joined back before it returns
        # (the step's duration is the group's: start/stop events bracket the loop)
        x = get_x()
        _lib.check(lib.ssb_sat_build_swa(x.data_ptr(), kind.abi_code, nr, COLS, COLS, sat.data_ptr(), ld, W, _lib.SUM,
                                         out.data_ptr(), None, out_c, ws.data_ptr(), ws_bytes, sptr))

    def phase_step(record: bool):
        # the same launches issued from here with an event around each kernel
        # group (per-kernel times in context; not the timed step)
        x = get_x()
        e0, e1, f0, f1, ej = (torch.cuda.Event(enable_timing=True) for _ in range(5))
        e0.record(stream)
        side.wait_event(e0)
        _lib.check(lib.ssb_sat_build(x.data_ptr(), kind.abi_code, nr, COLS, COLS, sat.data_ptr(), None, ld, None,
                                     None, ws.data_ptr(), ws_bytes, None, sptr))
        e1.record(stream)
        f0.record(side)
        _lib.check(lib.ssb_window_fused(x.data_ptr(), kind.abi_code, nr, COLS, COLS, W, _lib.SUM, out.data_ptr(),
                                        None, None, out_c, None, 0, side.cuda_stream))
        f1.record(side)
        stream.wait_event(f1)
        ej.record(stream)
        if record:
            ev["build"].append((e0, e1))
            ev["windows"].append((f0, f1))
            ev["group_phase"].append((e0, ej))

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step(False)
    barrier()
    launches0 = _lib.launch_count()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            step(True)
        stop.record(stream)
        barrier()
    launches = _lib.launch_count() - launches0
    ms_total = start.elapsed_time(stop)
    for i in range(args.warmup + args.steps):  # per-kernel phases of the same step (untimed pass)
        phase_step(i >= args.warmup)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    barrier()
    phase_ms = {k: sum(a.elapsed_time(b) for a, b in v) / len(v) for k, v in ev.items() if v}
    phase_ms["group_phase_pass"] = phase_ms.pop("group_phase")
    phase_ms["group"] = ms_step  # the timed step is exactly the group (one ssb_sat_build_swa call)

    # ---- algorithmic bytes: in + table write | table read + out write
    px_in = nr * COLS
    tab_bytes = (nr + 1) * (COLS + 1) * 8
    out_bytes = n_out * out_c * 8
    # the step's two kernel groups run concurrently, so the roofline is taken on
    # the group: each kernel's algorithmic bytes (sat_build: image read + table
    # write; window_fused: image read + window sums write) over the group's
    # duration (fork event -> join event on the step's stream)
    kernels = {
        "sat_build (image read + table write)": (px_in + tab_bytes, phase_ms["build"]),
        "window_fused (image read + window sums write)": (px_in + out_bytes, phase_ms["windows"]),
    }
    pk = peaks()
    dom = "sat_build || window_fused (concurrent kernel group of one step)"
    dom_bytes, dom_ms = sum(b for b, _ in kernels.values()), phase_ms["group"]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tfile = REPO / "profiles" / "traffic.json"
    if tfile.exists():
        tr = json.loads(tfile.read_text())
        if "sat_build" in tr and "window_fused" in tr:
            traffic = tr["sat_build"] + tr["window_fused"]
    b_alg = px_in + tab_bytes + out_bytes  # every distinct array read or written once
    b_mat = px_in + 2 * tab_bytes + out_bytes  # the reference structure (table written, then read back)
    value = rows * COLS / (ms_step * 1e-3) / 1e9

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded C5 recipe, synthetic.py)",
        "config": {"workload": "C5 70000x85000 u8 mask, integral image (u64) + window sum w=256 stride 1",
                   "pipeline": "table + windows: ssb_sat_build_swa (ssb_sat_build || ssb_window_fused on a "
                               "forked stream, joined)",
                   "parallelism": f"rowband{world}",
                   "sat_path": "single-pass decoupled look-back" if os.environ.get("SSB_SAT_PATH", "").startswith("o")
                   else "reduce-then-scan",
                   "l2": "inputs 5.95 GB >> 126 MB L2; no flush needed", "gen_s": round(gen_s, 1)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "kernel": dom,
                     "bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms, "peak_source": pk["source"]},
        "pipeline_roofline": {"bytes_per_step": b_alg, "achieved_gbs": b_alg / (ms_step * 1e-3) / 1e9,
                              "frac": b_alg / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"],
                              "bytes": "image read + table write + window sums write, each once"},
        "phases_ms": phase_ms,
        "phase_gbs": {k: b / (ms * 1e-3) / 1e9 for k, (b, ms) in kernels.items()},  # in context (overlapping)
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    # ---- the other pipelines on the same resident input (reported, not the headline)
    def time_steps(fn):
        for _ in range(3):
            fn()
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            fn()
        a1.record(stream)
        barrier()
        return a0.elapsed_time(a1) / args.steps

    try:
        x = get_x()

        def sweep_step():
            _lib.check(lib.ssb_sat_build(x.data_ptr(), kind.abi_code, nr, COLS, COLS, sat.data_ptr(), None, ld, None,
                                         None, ws.data_ptr(), ws_bytes, None, sptr))
            _lib.check(lib.ssb_window_eval(sat.data_ptr(), None, kind.abi_code, nr, COLS, ld, W, 1, _lib.SUM,
                                           out.data_ptr(), None, None, out_c, sptr))

        def onepass_step():
            _lib.check(lib.ssb_sat_build_swa_onepass(x.data_ptr(), kind.abi_code, nr, COLS, COLS, sat.data_ptr(), ld,
                                                     W, _lib.SUM, out.data_ptr(), None, out_c, ws.data_ptr(),
                                                     ws_bytes, sptr))

        def swa_call_step():
            _lib.check(lib.ssb_sat_build_swa(x.data_ptr(), kind.abi_code, nr, COLS, COLS, sat.data_ptr(), ld, W,
                                             _lib.SUM, out.data_ptr(), None, out_c, ws.data_ptr(), ws_bytes, sptr))

        for name, fn, b in (("corner_sweep_pipeline", sweep_step, b_mat), ("onepass_pipeline", onepass_step, b_alg),
                            ("ssb_sat_build_swa_call", swa_call_step, b_alg)):
            ms = time_steps(fn)
            result[name] = {"value": rows * COLS / (ms * 1e-3) / 1e9, "ms_per_step": ms, "bytes_per_step": b,
                            "roofline_frac": b / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]}
        result["corner_sweep_pipeline"]["api"] = "ssb_sat_build -> ssb_window_eval (table read back)"
        result["onepass_pipeline"]["api"] = "ssb_sat_build_swa_onepass"
        result["ssb_sat_build_swa_call"]["api"] = "ssb_sat_build_swa (the headline step as one C-ABI call)"
    except Exception as exc:  # pragma: no cover - reporting only
        result["corner_sweep_pipeline"] = {"error": str(exc)}

    # ---- fused window sums alone on the same resident input (no table)
    try:
        x = get_x()

        def fused_step():
            _lib.check(lib.ssb_window_fused(x.data_ptr(), kind.abi_code, nr, COLS, COLS, W, _lib.SUM,
                                            out.data_ptr(), None, None, out_c, None, 0, sptr))

        for _ in range(3):
            fused_step()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            fused_step()
        f1.record(stream)
        barrier()
        fms = f0.elapsed_time(f1) / args.steps
        fb = px_in + out_bytes
        result["fused"] = {"value": rows * COLS / (fms * 1e-3) / 1e9, "ms_per_step": fms,
                           "roofline_frac": fb / (fms * 1e-3) / 1e9 / pk["hbm_gbs"], "bytes_per_step": fb}
    except Exception as exc:  # pragma: no cover - reporting only
        result["fused"] = {"error": str(exc)}

    # ---- e2e through the public API with pinned host buffers: every rank runs
    # swa on its own input rows (band + halo) and reads back its output band;
    # the step time is the max over ranks
    if not args.no_e2e:
        try:
            x_need = get_x()
            del sat, ws
            torch.cuda.empty_cache()
            host_in = torch.empty((nr, COLS), dtype=torch.uint8, pin_memory=True)
            _copy_chunks(host_in, x_need)
            host_out = torch.empty((max(n_out, 1), out_c), dtype=torch.int64, pin_memory=True)
            import paper_2410_16291_b200 as sb

            hin = host_in.numpy()
            hout = host_out.numpy().view(np.uint64)[:n_out]

            def e2e_step():
                if n_out > 0:
                    sb.swa(hin, W, "sum", pipeline="table", out=hout)

            e2e_step()  # warm-up
            times = []
            for _ in range(args.e2e_steps):
                barrier()
                t0 = time.perf_counter()
                e2e_step()
                times.append(time.perf_counter() - t0)
            te = sum(times) / len(times)
            h2d, d2h = nr * COLS, n_out * out_c * 8
            if world > 1:
                import torch.distributed as dist

                agg = torch.tensor([te, float(h2d), float(d2h)], dtype=torch.float64, device=dev)
                mx = agg[:1].clone()
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                dist.all_reduce(agg, op=dist.ReduceOp.SUM)
                te, h2d, d2h = float(mx.item()), int(agg[1].item()), int(agg[2].item())
            result["e2e"] = {"value": rows * COLS / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
                             "d2h_bytes_per_step": d2h, "s_per_step": te,
                             "api": "paper_2410_16291_b200.swa(numpy pinned, 256, 'sum', pipeline='table', out=pinned)"
                                    " -> ssb_swa_host, per rank on its band + halo; max over ranks"}
        except Exception as exc:  # pragma: no cover
            result["e2e"] = {"error": str(exc)}

    # ---- CPU baseline: the reference algorithm on a bounded band, rank 0 at N=1
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            tot_t, tot_px = 0.0, 0
            for _ in range(max(1, args.cpu_reps)):
                dt, px = cpu_port_band(args.cpu_rows)
                tot_t += dt
                tot_px += px
            result["cpu_baseline"] = {
                "value": tot_px / tot_t / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                "sample": f"{args.cpu_reps} x C5 output rows [0, {args.cpu_rows}) ({args.cpu_rows + W - 1} input rows x "
                          f"{COLS}); oracle.swa_threaded = numpy restatement of satsweep.swa_parallel; "
                          f"{tot_t:.1f} s of CPU work"}
        except Exception as exc:  # pragma: no cover
            result["cpu_baseline"] = {"error": str(exc)}

    if rank == 0:
        emit(result)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def _copy_chunks(dst_host, src_dev, rows_per=4096):
    for a in range(0, src_dev.shape[0], rows_per):
        dst_host[a:a + rows_per].copy_(src_dev[a:a + rows_per].cpu())


if __name__ == "__main__":
    main()
