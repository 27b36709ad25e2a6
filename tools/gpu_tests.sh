#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_zero3_p2p_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "p2p or zero3" > gpurun_out/pytest_p2p.log 2>&1; echo "p2p rc=$?"; tail -3 gpurun_out/pytest_p2p.log; grep -E "^E |Error" gpurun_out/pytest_p2p.log | head -20
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
