mkdir -p gpurun_out
timeout 300 python scripts/configs_probe.py C4 fused 1 > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_strip -c 1 -o gpurun_out/c4_prof2 python scripts/configs_probe.py C4 fused 1 > gpurun_out/c4_ncu.log 2>&1
