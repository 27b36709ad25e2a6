# Session 3: split-master optimizer states — GPU tests (kernels + engine), then C3/C2 A/B (split vs full master).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_split_master_gpu.py tests/test_engine_gpu.py tests/test_kernels_gpu.py -x -q > gpurun_out/s3_split_tests.log 2>&1; echo "split tests rc $?"
tail -3 gpurun_out/s3_split_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/s3_smoke.log
for M in split full; do
  F=""; [ $M = full ] && F="--full-master"
  timeout 900 python bench.py --config c3 --secondary "" --no-cpu-baseline $F > gpurun_out/s3_c3_$M.json 2> gpurun_out/s3_c3_$M.err; echo "c3 $M rc $?"
done
for M in split full; do
  F=""; [ $M = full ] && F="--full-master"
  timeout 600 python bench.py --config c2 --secondary "" --no-cpu-baseline $F > gpurun_out/s3_c2_$M.json 2> gpurun_out/s3_c2_$M.err; echo "c2 $M rc $?"
done
