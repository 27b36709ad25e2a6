#!/bin/bash
# C2: GPU spare slots x stage ring (edge fill on), one box.
mkdir -p gpurun_out
: > gpurun_out/ring_sweep.txt
for sp in ${SPARES:-4 8 16}; do
  for st in ${STAGES_LIST:-12 20 32}; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stages $st --gpu-spares $sp > gpurun_out/rs.json 2>>gpurun_out/rs.err
    python -c "
import json; d=json.load(open('gpurun_out/rs.json')); print('spares=$sp stages=$st', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['stall_ms_per_step'], d['phase_ms_last_step'])" >> gpurun_out/ring_sweep.txt 2>&1
  done
done
cat gpurun_out/ring_sweep.txt
