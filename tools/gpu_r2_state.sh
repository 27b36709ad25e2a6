# Round 2 (session 3): state of HEAD on a fresh box: default bench (C3 headline + C2), reference arm, GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/s3_nvsmi.txt 2>&1; lscpu > gpurun_out/s3_lscpu.txt
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/s3_ref_c3.json 2> gpurun_out/s3_ref_c3.err; echo "ref c3 rc $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/s3_pytest_gpu.log
