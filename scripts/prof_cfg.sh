# usage: CFG=C3 PROF_K=regex PROF_S=skip PROF_TAG=tag bash scripts/prof_cfg.sh
mkdir -p gpurun_out
B="python scripts/bench_configs.py ${CFG:-C3}"
$B > gpurun_out/plain_${PROF_TAG}.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${PROF_TAG}.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${PROF_K}" -s ${PROF_S:-1} -c 1 -o gpurun_out/prof_${PROF_TAG} $B > gpurun_out/ncu_${PROF_TAG}.log 2>&1
echo done
