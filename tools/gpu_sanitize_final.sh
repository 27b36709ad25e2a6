#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py
# (every data-plane kernel at ragged sizes + engine iterations with NVMe and
# both ZeRO-3 exchanges) with the current build.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
done
