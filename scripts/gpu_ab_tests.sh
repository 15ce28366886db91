bash scripts/gpu_ab.sh
SSB_LIB=_ablibs/work.so timeout 300 python scripts/configs_probe.py C3 auto 10 >> gpurun_out/ab.log 2>&1
SSB_LIB=_ablibs/head.so timeout 300 python scripts/configs_probe.py C3 auto 10 >> gpurun_out/ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sweep.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/t_sub.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub.log
