#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "captured or comparison or zero3" > gpurun_out/pytest_sel.log 2>&1; tail -2 gpurun_out/pytest_sel.log
timeout 1200 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json')); [print(k, d[k]) for k in ('ms_per_step','value','value_definition','pcie','phase_ms_last_step','setup_s','roofline','hit_rate')]" || tail -5 gpurun_out/bench_c3.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json | cut -c1-400
