#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --zero3 --gpus 1 --steps 2 --warmup 1 > gpurun_out/bench_zero3_torchrun.json 2> gpurun_out/bench_zero3_torchrun.err; echo "torchrun rc=$?"; tail -c 700 gpurun_out/bench_zero3_torchrun.json; tail -3 gpurun_out/bench_zero3_torchrun.err
