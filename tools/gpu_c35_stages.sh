#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/c35_stages.txt
for st in 128 256; do
  timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --stages $st > gpurun_out/s.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s.json')); print('c5 stages=$st', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['migration_hidden_frac'])" >> gpurun_out/c35_stages.txt 2>&1
done
for st in 128 256; do
  timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --stages $st > gpurun_out/s.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/s.json')); print('c3 stages=$st', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['migration_hidden_frac'])" >> gpurun_out/c35_stages.txt 2>&1
  cp gpurun_out/s.json gpurun_out/c3_s$st.json
done
cat gpurun_out/c35_stages.txt
