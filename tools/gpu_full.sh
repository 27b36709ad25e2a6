#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o faulthandler_timeout=240 > gpurun_out/pytest_gpu_$i.log 2>&1; echo "pytest $i rc=$?"; tail -2 gpurun_out/pytest_gpu_$i.log; grep -E "^E |Timeout|File \"" gpurun_out/pytest_gpu_$i.log | head -20
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
