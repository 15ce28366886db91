# Round-end evidence on one B200: GPU tests, smoke, the default bench line, the
# reference arm, the C5 launch list and ncu --set full of the step's kernels and C4/C2.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/f_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench_ref.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs --no-extra"
$B > gpurun_out/f_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv $B > /dev/null 2>&1
$B > gpurun_out/f_plain2.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fused_strip|sat_scan|sat_reduce" -s 3 -c 3 -o gpurun_out/f_c5 $B > gpurun_out/f_ncu_c5.log 2>&1
timeout 300 python scripts/configs_probe.py C4 fused 1 > gpurun_out/f_c4_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_strip -c 1 -o gpurun_out/f_c4 python scripts/configs_probe.py C4 fused 1 > gpurun_out/f_ncu_c4.log 2>&1
timeout 300 python scripts/configs_probe.py C2 fused 1 > gpurun_out/f_c2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_strip -c 1 -o gpurun_out/f_c2 python scripts/configs_probe.py C2 fused 1 > gpurun_out/f_ncu_c2.log 2>&1
echo done > gpurun_out/f_done.txt
