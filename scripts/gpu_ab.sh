# A/B of _ablibs/*.so: C4 / C2 fused timings and the C5 step (bench.py, no e2e/cpu/configs/extra)
mkdir -p gpurun_out
for i in 1 2; do for lib in _ablibs/*.so; do
  echo "== $lib"
  SSB_LIB=$lib timeout 300 python scripts/configs_probe.py C4 fused 20 2>&1 | tail -1
  SSB_LIB=$lib timeout 300 python scripts/configs_probe.py C2 fused 20 2>&1 | tail -1
  SSB_LIB=$lib timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-configs --no-extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['ms_per_step'], d['value'])"
done; done > gpurun_out/ab.log 2>&1
