#!/bin/bash
# auto stage ring vs the earlier fixed choices, same box
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
: > gpurun_out/autostage.txt
for cfg in "--tokens 16384" "--tokens 16384 --stages 12" "--tokens 32768" "--tokens 32768 --stages 12" "--config c3" "--config c3 --stages 128" "--config c5" "--config c5 --stages 128"; do
  TC_SETUP_TIMING=1 timeout 900 python bench.py $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/as.json 2> gpurun_out/as.err
  ring=$(grep "stage ring" gpurun_out/as.err | head -1 | sed 's/.*ring: //')
  python -c "
import json; d=json.load(open('gpurun_out/as.json')); print('$cfg', '| ring', '$ring', '|', d['ms_per_step'], d['e2e']['ms_per_step'], d['migration_hidden_frac'])" >> gpurun_out/autostage.txt 2>&1
done
cat gpurun_out/autostage.txt
