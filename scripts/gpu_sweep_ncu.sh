mkdir -p gpurun_out
export SSB_SWEEP_M=5 PROBE_FAST=1
for v in ${VARIANTS:-base}; do
SSB_LIB=_ablibs/$v.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sat_sweep -s 1 -c 1 -o gpurun_out/sweep_$v python scripts/sweep_probe.py 35000 > gpurun_out/sweep_ncu_$v.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_ncu_$v.log
done
