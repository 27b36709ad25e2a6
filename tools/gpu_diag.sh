#!/bin/bash
mkdir -p gpurun_out
{ echo "memory.max: $(cat /sys/fs/cgroup/memory.max 2>/dev/null)"; echo "ulimit -l: $(ulimit -l)"; free -g; nproc; } > gpurun_out/diag.txt
python - >> gpurun_out/diag.txt 2>&1 <<'PY'
import torch, time
for gb in (16, 32, 64, 80):
    t=time.time()
    try:
        x=torch.empty(gb<<30, dtype=torch.uint8, pin_memory=True); print("pinned", gb, "GB in", round(time.time()-t,1), "s"); del x
    except Exception as e:
        print("pin", gb, "failed", e); break
PY
cat gpurun_out/diag.txt
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"; tail -c 1500 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
dmesg 2>/dev/null | tail -5
