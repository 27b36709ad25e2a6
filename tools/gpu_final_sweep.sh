#!/bin/bash
# Same-box sweep of C2 spares x stages with the end-of-round executor.
mkdir -p gpurun_out
: > gpurun_out/final_sweep.txt
for rep in 1 2; do
for cfg in "16 12" "8 12" "24 12" "16 8" "16 16" "32 12"; do
  set -- $cfg
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gpu-spares $1 --stages $2 > gpurun_out/fs.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/fs.json')); print('spares=$1 stages=$2', d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/final_sweep.txt 2>&1
done
done
cat gpurun_out/final_sweep.txt
