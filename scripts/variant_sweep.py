"""Build library variants with extra -D defines and run a script against each (tuning only).

usage: python scripts/variant_sweep.py "scripts/build_phases.py" "SSB_REDUCE_MINB=3" "SSB_REDUCE_MINB=4,SSB_X=1" ...
Each variant is built into /tmp and selected through SSB_LIB; output lines are prefixed with the variant."""
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    script, variants = sys.argv[1], sys.argv[2:]
    for i, v in enumerate(variants):
        defines = tuple(d for d in v.split(",") if d)
        lib = Path(f"/tmp/libssb_variant_{i}.so")
        code = ("import sys; sys.path.insert(0, %r); from paper_2410_16291_b200 import build_ext; "
                "build_ext.build(defines=%r, lib=__import__('pathlib').Path(%r))" % (str(REPO), defines, str(lib)))
        subprocess.run([sys.executable, "-c", code], check=True)
        env = dict(os.environ, SSB_LIB=str(lib))
        parts = script.split()
        out = subprocess.run([sys.executable, str(REPO / parts[0]), *parts[1:]], env=env, capture_output=True, text=True)
        for line in (out.stdout + out.stderr).strip().splitlines()[-3:]:
            print(f"[{v}] {line}", flush=True)


if __name__ == "__main__":
    main()
