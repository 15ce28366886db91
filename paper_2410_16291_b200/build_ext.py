"""Build libsatsweep_b200.so in-tree with nvcc for sm_100a.

Used by ``__graft_entry__.build()`` and importable on its own:
``python -m paper_2410_16291_b200.build_ext``.  The shared library is written
next to this file so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libsatsweep_b200.so"
SOURCES = ["sat_build.cu", "sat_onepass.cu", "sat_sweep.cu", "window_eval.cu", "window_fused.cu", "capi.cu", "io.cu", "shard.cu", "selftest.cu", "host_widen.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "satsweep_b200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple = (), lib: Path | None = None) -> Path:
    """``defines``/``lib``: tuning variants (e.g. SSB_ONEPASS_PROF) built next to, never over, the product library."""
    target = lib or LIB
    if not force and not defines and lib is None and not _stale():
        return LIB
    out_dir = PKG / ("_build" if not defines else "_build_variant")
    out_dir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = out_dir / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = target.with_suffix(".so.tmp")
    subprocess.run([nvcc(), *ARCH, "-shared", *objs, "-o", str(tmp), "-cudart", "static"], check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
