#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E |Error" gpurun_out/pytest_gpu.log | head -20
: > gpurun_out/lookahead_ab.txt
for rep in 1 2; do for la in 0 1; do
  TC_LOOKAHEAD=$la timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/la.json 2>>gpurun_out/la.err
  python -c "
import json; d=json.load(open('gpurun_out/la.json')); print('lookahead=$la', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['migration_hidden_frac'])" >> gpurun_out/lookahead_ab.txt 2>&1
done; done
cat gpurun_out/lookahead_ab.txt
