#!/bin/bash
# Tuning: run a probe script against every library in _ablibs/ (SSB_LIB), e.g.
#   scripts/ab_run.sh "scripts/sweep_probe.py"
mkdir -p gpurun_out
for lib in _ablibs/*.so; do
  echo "== $lib"
  SSB_LIB=$lib timeout 300 python $1 2>&1 | tail -${2:-3}
done
