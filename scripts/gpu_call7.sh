bash scripts/gpu_ab.sh
