# Session 3: closed-loop GEMM stand-in + split master: GPU suite, default bench, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3b_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/s3b_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/s3b_ref_c3.json 2> gpurun_out/s3b_ref_c3.err; echo "ref rc $?"
timeout 600 python bench.py --config c3 --secondary "" --no-cpu-baseline --full-master > gpurun_out/s3b_c3_full.json 2> gpurun_out/s3b_c3_full.err; echo "c3 full rc $?"
