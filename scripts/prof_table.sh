set -x
mkdir -p gpurun_out
B="python bench.py --rows 8192 --steps 2 --no-e2e --no-cpu"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/t2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t2.log
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sat_scan|window_eval|sat_reduce|sat_rowcarry" -s 4 -c 4 -o gpurun_out/prof_table $B > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"window_fused" -c 1 -o gpurun_out/prof_fused $B > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
