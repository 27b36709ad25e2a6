#!/bin/bash
# One GPU session: tests, smoke, bench(es). Output under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps ${BENCH_STEPS:-5} --warmup ${BENCH_WARMUP:-3} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "$BENCH_EXTRA" ]; then timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline $BENCH_EXTRA > gpurun_out/bench_extra.json 2>> gpurun_out/bench.err; fi
if [ -n "$PROF" ]; then bash tools/gpu_prof.sh; fi
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench.json; cat gpurun_out/bench_extra.json 2>/dev/null; tail -5 gpurun_out/bench.err
