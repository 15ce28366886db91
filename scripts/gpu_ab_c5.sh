# A/B of _ablibs/*.so on the C5 phases (scripts/c5_phases.py)
mkdir -p gpurun_out
for i in 1 2; do for lib in _ablibs/*.so; do
  SSB_LIB=$lib timeout 300 python scripts/c5_phases.py 2>&1 | tail -1
done; done > gpurun_out/ab_c5.log 2>&1
