#!/bin/bash
# tests + C2 x2 + C5 + C5 timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log; grep -E "^E " gpurun_out/pytest_gpu.log | head
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b$i.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b$i.json')); print('c2', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['migration_hidden_frac'])"; done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/c5.json')); print('c5', d['ms_per_step'], d['e2e']['ms_per_step'], d['pcie']['duplex_frac'], d['migration_hidden_frac'])"
if [ -n "$TL" ]; then CFG=c5 STAGES=128 ITERS=4 timeout 900 python tools/timeline.py > gpurun_out/tl_c5.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/timeline_c5.json')); print(json.dumps(d['iters'])); print(d['h2d_gaps_over_1ms_abs'], d['d2h_gaps_over_1ms_abs'])"; fi
