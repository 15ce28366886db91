mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sweep.py tests/test_gpu_configs.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/t_sub.log 2>&1; echo "rc=$?" >> gpurun_out/t_sub.log
