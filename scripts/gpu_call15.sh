mkdir -p gpurun_out
for i in 1 2; do for lib in _ablibs/head.so _ablibs/work.so; do
  echo "== $lib"
  SSB_LIB=$lib timeout 300 python scripts/configs_probe.py C3 auto 10 2>&1 | tail -1
  SSB_LIB=$lib timeout 300 python scripts/c5_phases.py 2>&1 | tail -1
done; done > gpurun_out/ab15.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sweep.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py tests/test_gpu_shard.py -x -q -m gpu > gpurun_out/t_sub.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub.log
