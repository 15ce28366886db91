#!/bin/bash
# Tuning: build a library variant that differs only in one source file and/or -D defines.
# usage: scripts/ab_build.sh NAME SRC_FILE [DEFINES...]   -> _ablibs/NAME.so (git-ignored, travels to the GPU box)
# SRC_FILE replaces the same-named file of csrc/; the other objects come from the product build (_build/).
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
defs=""; for d in "$@"; do defs="$defs -D$d"; done
mkdir -p _ablibs /tmp/ab_$name
base=$(basename "$src" .cu)
cp paper_2410_16291_b200/csrc/*.cuh /tmp/ab_$name/
cp "$src" /tmp/ab_$name/$base.cu
mkdir -p /tmp/ab_$name/../include; cp include/satsweep_b200.h /tmp/include/ 2>/dev/null || true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $defs \
  -I paper_2410_16291_b200/csrc -c /tmp/ab_$name/$base.cu -o /tmp/ab_$name/$base.o
objs=""; for o in paper_2410_16291_b200/_build/*.o; do [ "$(basename $o .o)" = "$base" ] && objs="$objs /tmp/ab_$name/$base.o" || objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o _ablibs/$name.so -cudart static
echo "_ablibs/$name.so"
