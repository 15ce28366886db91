# round profile of the headline step: bench (full JSON), launch list, ncu --set full of the hot kernels
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $B > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused_strip|sat_scan|sat_reduce" -s 3 -c 3 -o gpurun_out/r2_kernels $B > gpurun_out/r2_ncu.log 2>&1
echo done >> gpurun_out/r2_ncu.log
