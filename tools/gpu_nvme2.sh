#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/nvme2.txt
for t in 8 16; do
  TC_NVME_THREADS=$t timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/n2.json 2>>gpurun_out/n2.err
  python -c "
import json; d=json.load(open('gpurun_out/n2.json')); print('c4 threads=$t', d['ms_per_step'], d['e2e']['ms_per_step'], d['migrated_bytes_per_step']['nvme_read'])" >> gpurun_out/nvme2.txt 2>&1
  cp gpurun_out/n2.json gpurun_out/c4_t$t.json
done
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --direct-io > gpurun_out/n2.json 2>>gpurun_out/n2.err
python -c "
import json; d=json.load(open('gpurun_out/n2.json')); print('c4 odirect', d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/nvme2.txt 2>&1
cp gpurun_out/n2.json gpurun_out/c4_odirect.json
for pol in zero-infinity l2l; do
timeout 900 python bench.py --policy $pol --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/n2.json 2>>gpurun_out/n2.err
python -c "
import json; d=json.load(open('gpurun_out/n2.json')); print('c2 $pol', d['ms_per_step'], d['e2e']['ms_per_step'], d['hit_rate'])" >> gpurun_out/nvme2.txt 2>&1
cp gpurun_out/n2.json gpurun_out/c2_$pol.json
done
cat gpurun_out/nvme2.txt
