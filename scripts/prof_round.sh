# round profile: full C5 launch list + ncu --set full captures of the three table kernels
mkdir -p gpurun_out
B="python bench.py --steps 2 --no-e2e --no-cpu"
$B > gpurun_out/r1_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"window_eval_tma|sat_scan|sat_reduce" -s 3 -c 3 -o gpurun_out/r1_table $B > gpurun_out/r1_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"window_fused" -s 1 -c 1 -o gpurun_out/r1_fused $B >> gpurun_out/r1_ncu.log 2>&1
echo done
