#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_driver.py);
# logs to gpurun_out/sanitizer_<tool>.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python scripts/sanitize_driver.py $SAN_ARGS \
    > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
