#!/bin/bash
# A/B runs of the C2 bench in one session (variance + options).
mkdir -p gpurun_out
i=0
for args in "$@"; do
  i=$((i+1))
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args > gpurun_out/ab_$i.json 2>> gpurun_out/ab.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab_$i.json')); print('$args', d['ms_per_step'], d['pcie']['h2d_GBps_step'], d['phase_ms_last_step'], d['roofline']['frac'], d['migration_hidden_frac'])"
done
