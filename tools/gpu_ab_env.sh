#!/bin/bash
# A/B of env settings on the C2 bench: each arg is an env assignment list ("" = baseline)
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abe_$i.json 2>> gpurun_out/abe.err
  python -c "
import json; d=json.load(open('gpurun_out/abe_$i.json')); print('[$envs]', d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['pcie']['h2d_GBps_step'])"
done
