mkdir -p gpurun_out
bash scripts/gpu_ab_c5.sh
for k in 42 170 340; do SSB_FUSED_SEGMENTS=$k SSB_LIB=_ablibs/il0.so timeout 300 python scripts/c5_phases.py 2>&1 | tail -1 | sed "s/^/seg$k /"; done >> gpurun_out/ab_c5.log
