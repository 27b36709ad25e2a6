#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "nvme or random or many or comparison" 2>&1 | tail -2
: > gpurun_out/nvme_files.txt
for f in 1 8 16; do
  TC_NVME_FILES=$f timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/nf.json 2>>gpurun_out/nf.err
  python -c "
import json; d=json.load(open('gpurun_out/nf.json')); print('files=$f', d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/nvme_files.txt 2>&1
done
cat gpurun_out/nvme_files.txt
