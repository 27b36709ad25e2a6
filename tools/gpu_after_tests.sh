#!/bin/bash
# Does the bench right after `pytest -m gpu` (the driver's order) see a slower
# PCIe? Records host dirty/writeback memory and load before each bench.
mkdir -p gpurun_out
o=gpurun_out/after_tests.txt; : > $o
snap() { echo "== $1 $(date +%s) load=$(cut -d' ' -f1-3 /proc/loadavg) $(grep -E '^(Dirty|Writeback|Cached|MemFree):' /proc/meminfo | tr -s ' ' | tr '\n' ' ')" >> $o; }
snap start
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $o
for i in 1 2 3; do
  snap "bench$i"
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'h2d_busy', d['pcie']['h2d_GBps_busy'], 'stall', d['stall_ms_per_step'])" >> $o 2>&1
done
snap end
cat $o
