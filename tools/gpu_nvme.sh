#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^E " gpurun_out/pytest_gpu.log | head -5
timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', d['ms_per_step'], d['migrated_bytes_per_step']['nvme_read'], d['phase_ms_last_step'])" || tail -3 gpurun_out/bench_c4.err
TC_NVME_THREADS=1 timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4_1t.json 2>> gpurun_out/bench_c4.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c4_1t.json')); print('c4 1 thread', d['ms_per_step'])"
timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --direct-io > gpurun_out/bench_c4_odirect.json 2>> gpurun_out/bench_c4.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c4_odirect.json')); print('c4 O_DIRECT', d['ms_per_step'])"
