#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/c4_hs.txt
for hs in 1 4 8 16; do
  timeout 900 python bench.py --config c4 --host-spares $hs --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/hs.json 2>>gpurun_out/hs.err
  python -c "
import json; d=json.load(open('gpurun_out/hs.json')); print('host_spares=$hs', d['ms_per_step'], d['e2e']['ms_per_step'], d['migration_hidden_frac'])" >> gpurun_out/c4_hs.txt 2>&1
done
cat gpurun_out/c4_hs.txt
