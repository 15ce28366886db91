bash scripts/gpu_ab_c5.sh
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sweep.py tests/test_gpu_scale.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/t_sub.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub.log
