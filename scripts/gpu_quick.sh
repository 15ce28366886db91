# quick GPU validation: parity tests, smoke, a short bench on a 8192-row slice, then full C5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py --rows 8192 --steps 5 --no-e2e --no-cpu > gpurun_out/bench_small.log 2>&1; echo "rc=$?" >> gpurun_out/bench_small.log
if [ "$FULL" = "1" ]; then timeout 600 python bench.py --steps 5 --no-cpu --no-e2e > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log; fi
