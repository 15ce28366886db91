mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sat_sweep -s 1 -c 1 -o gpurun_out/sweep_full python scripts/sweep_probe.py 20000 > gpurun_out/sweep_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_ncu.log
