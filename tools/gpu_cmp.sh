#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|E )" gpurun_out/pytest_gpu.log | head -20
for pol in l2l zero-infinity; do
  timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --policy $pol > gpurun_out/bench_$pol.json 2> gpurun_out/bench_$pol.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$pol.json')); print('$pol', d['ms_per_step'], d['hit_rate'], d['migrated_bytes_per_step'], d['phase_ms_last_step'])" || tail -5 gpurun_out/bench_$pol.err
done
