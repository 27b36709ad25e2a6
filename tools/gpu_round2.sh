#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/pcie_sweep.py > gpurun_out/pcie_sweep.log 2>&1; tail -c 600 gpurun_out/pcie_sweep.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['roofline'], d['cpu_baseline'], d['migration_hidden_frac'])"
