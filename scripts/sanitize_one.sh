# One compute-sanitizer tool per gpurun call (the profiling guide's rule):
#   TOOL=memcheck bash scripts/sanitize_one.sh  -> gpurun_out/sanitizer_<tool>.txt
# The driver's plain run first (it must exit 0), then the tool.
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
timeout 300 python scripts/sanitize_driver.py > gpurun_out/sanitize_plain.txt 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.txt
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 50 python scripts/sanitize_driver.py > gpurun_out/sanitizer_$TOOL.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer_$TOOL.txt
