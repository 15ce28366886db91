mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/t_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/t_sweep.log
timeout 300 python scripts/sweep_probe.py > gpurun_out/sweep_probe.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_probe.log
