cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; lscpu > gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
timeout 900 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/r2_ref_c3.json 2> gpurun_out/r2_ref_c3.err; echo "ref c3 rc $?"
timeout 600 python bench.py --impl reference --config c2 > gpurun_out/r2_ref_c2.json 2> gpurun_out/r2_ref_c2.err; echo "ref c2 rc $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2_pytest_gpu.log
