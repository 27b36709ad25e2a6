#!/bin/bash
# C2 forward pre-staging sweep: ring size x forward budget x gate.
mkdir -p gpurun_out
: > gpurun_out/prestage_sweep.txt
for st in ${STAGES_LIST:-12 16 20 24}; do
  for fwd in -1 $((st - 1)); do
    for gate in 0 1; do
      TC_PRESTAGE_FWD=$fwd TC_PRESTAGE_GATE=$gate timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stages $st > gpurun_out/ps.json 2>>gpurun_out/ps.err
      python -c "
import json; d=json.load(open('gpurun_out/ps.json')); print('stages=$st fwd=$fwd gate=$gate', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['stall_ms_per_step'])" >> gpurun_out/prestage_sweep.txt 2>&1
    done
  done
done
cat gpurun_out/prestage_sweep.txt
