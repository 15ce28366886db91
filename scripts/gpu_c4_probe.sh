mkdir -p gpurun_out
for i in 1 2; do for lib in _ablibs/fin0.so _ablibs/fin1.so; do echo "== $lib"; SSB_LIB=$lib timeout 300 python scripts/configs_probe.py C4 fused 20 2>&1 | tail -1; done; done > gpurun_out/c4ab.log 2>&1
timeout 300 python scripts/configs_probe.py C2 fused 20 >> gpurun_out/c4ab.log 2>&1
./scripts/probes/wr_probe > gpurun_out/wr_probe.log 2>&1
timeout 300 python scripts/configs_probe.py C4 fused 1 > gpurun_out/c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_strip -c 1 -o gpurun_out/c4_prof python scripts/configs_probe.py C4 fused 1 > gpurun_out/c4_ncu.log 2>&1
