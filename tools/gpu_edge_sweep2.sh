#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/edge_sweep2.txt
for rep in 1 2; do
for cfg in "12 0 -1" "16 1 -1" "18 1 -1" "20 1 -1" "16 0 15" "20 0 19"; do
  set -- $cfg
  TC_EDGE_FILL=$2 TC_PRESTAGE_FWD=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stages $1 > gpurun_out/es.json 2>>gpurun_out/es.err
  python -c "
import json; d=json.load(open('gpurun_out/es.json')); print('stages=$1 edge=$2 fwd=$3', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['stall_ms_per_step'], d['migrated_bytes_per_step']['optimizer_h2d'])" >> gpurun_out/edge_sweep2.txt 2>&1
done
done
cat gpurun_out/edge_sweep2.txt
