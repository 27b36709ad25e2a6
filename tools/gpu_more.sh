#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --tokens 65536 > gpurun_out/bench_t64k.json 2> gpurun_out/bench_t64k.err
python -c "
import json; d=json.load(open('gpurun_out/bench_t64k.json')); print('t64k', d['ms_per_step'], d['migration_hidden_frac'], d['ontime_rate'], d['stall_ms_per_step'], d['phase_ms_last_step'])"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --zero3 --gpus 1 --steps 3 --warmup 2 > gpurun_out/bench_zero3_p2p.json 2> gpurun_out/bench_zero3_p2p.err; echo "torchrun p2p rc=$?"; tail -1 gpurun_out/bench_zero3_p2p.json | cut -c1-900; tail -3 gpurun_out/bench_zero3_p2p.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29556 bench.py --zero3 --exchange nccl --gpus 1 --steps 3 --warmup 2 > gpurun_out/bench_zero3_nccl.json 2> gpurun_out/bench_zero3_nccl.err; echo "torchrun nccl rc=$?"; tail -1 gpurun_out/bench_zero3_nccl.json | cut -c1-400
