#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/c4_threads.txt
for t in 4 8 16; do
  TC_NVME_THREADS=$t timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c4t.json 2>>gpurun_out/c4t.err
  python -c "
import json; d=json.load(open('gpurun_out/c4t.json')); print('threads=$t', d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/c4_threads.txt 2>&1
done
cat gpurun_out/c4_threads.txt
