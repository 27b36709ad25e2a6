#!/bin/bash
# C2: forward->backward edge fill of the stage ring, per ring size (A/B on one box).
mkdir -p gpurun_out
: > gpurun_out/edge_sweep.txt
for rep in 1 2; do
for st in 12 16 18 20 24; do
  for ef in 0 1; do
    TC_EDGE_FILL=$ef timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stages $st > gpurun_out/es.json 2>>gpurun_out/es.err
    python -c "
import json; d=json.load(open('gpurun_out/es.json')); print('stages=$st edge=$ef', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['stall_ms_per_step'])" >> gpurun_out/edge_sweep.txt 2>&1
  done
done
done
cat gpurun_out/edge_sweep.txt
