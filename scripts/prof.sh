# usage: PROF_TAG=name PROF_K='regex' PROF_S=skip PROF_C=count bash scripts/prof.sh  (bench on an 8192-row slice)
mkdir -p gpurun_out
B="python bench.py --rows ${PROF_ROWS:-8192} --steps 2 --no-e2e --no-cpu"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
$B > gpurun_out/plain_${PROF_TAG}.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${PROF_TAG}.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${PROF_K}" -s ${PROF_S:-4} -c ${PROF_C:-4} -o gpurun_out/prof_${PROF_TAG} $B > gpurun_out/ncu_${PROF_TAG}.log 2>&1
echo done
