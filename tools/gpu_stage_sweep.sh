#!/bin/bash
# HBM optimizer-stage ring sweep (C5 and C2): ms/step and PCIe fractions per ring size.
mkdir -p gpurun_out
for st in ${C5_STAGES:-48 128 256}; do
  timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --stages $st > gpurun_out/sweep_c5_s$st.json 2>> gpurun_out/sweep.err
done
for st in ${C2_STAGES:-24 48 96}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --stages $st > gpurun_out/sweep_c2_s$st.json 2>> gpurun_out/sweep.err
done
for f in gpurun_out/sweep_*.json; do python -c "
import json; d=json.load(open('$f')); p=d['pcie']; print('$f', d['ms_per_step'], d['value'], p['duplex_frac'], d['migration_hidden_frac'], d['roofline']['avg_launch_us'], d['e2e']['ms_per_step'])" 2>/dev/null || echo "$f failed"; done
tail -n 5 gpurun_out/sweep.err
