#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ring_sweep2.txt
for cfg in "16 12 1" "16 12 0" "32 12 1" "32 12 0" "48 12 1" "32 8 1" "32 10 1" "32 14 1" "4 12 1" "79 12 1"; do
  set -- $cfg
  TC_EDGE_FILL=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stages $2 --gpu-spares $1 > gpurun_out/rs.json 2>>gpurun_out/rs.err
  python -c "
import json; d=json.load(open('gpurun_out/rs.json')); print('spares=$1 stages=$2 edge=$3', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['stall_ms_per_step'], d['phase_ms_last_step'])" >> gpurun_out/ring_sweep2.txt 2>&1
done
cat gpurun_out/ring_sweep2.txt
