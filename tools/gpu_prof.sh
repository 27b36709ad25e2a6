#!/bin/bash
# Profiling session: kernels alone, ncu full set on AdamW (variant $V), launch list of a short bench.
mkdir -p gpurun_out
V=${V:-2}
timeout 300 python tools/prof_adamw.py > gpurun_out/kernels_alone.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adamw -s 2 -c 2 \
   -o gpurun_out/prof_adamw_v$V -f env KALONE_OUT=0 REPS=4 VARIANTS=$V python tools/prof_adamw.py > gpurun_out/ncu_adamw.log 2>&1
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
fi
echo done
