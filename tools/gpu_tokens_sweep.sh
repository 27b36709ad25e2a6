#!/bin/bash
# C2 compute/migration balance: tokens per step vs step time, hidden fraction, PCIe.
mkdir -p gpurun_out
: > gpurun_out/tokens_sweep.txt
for tok in 4096 16384 32768 65536 131072; do
  timeout 600 python bench.py --tokens $tok --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/tk.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tk.json')); print(json.dumps({'tokens': $tok, 'ms_per_step': d['ms_per_step'], 'e2e_ms': d['e2e']['ms_per_step'], 'hidden': d['migration_hidden_frac'], 'duplex_frac': d['pcie']['duplex_frac'], 'ontime': d['ontime_rate'], 'compute_ms': d['phase_ms_last_step']}))" >> gpurun_out/tokens_sweep.txt 2>&1
done
cat gpurun_out/tokens_sweep.txt
