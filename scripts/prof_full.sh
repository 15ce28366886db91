# launch list of the full C5 bench + one full ncu capture of the reduce kernel
mkdir -p gpurun_out
B="python bench.py --steps 2 --no-e2e --no-cpu"
$B > gpurun_out/plain_full.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${PROF_K:-sat_reduce}" -s ${PROF_S:-2} -c 1 -o gpurun_out/prof_full_${PROF_TAG:-reduce} $B > gpurun_out/ncu_full.log 2>&1
echo done
