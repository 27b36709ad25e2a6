# Session 3: C3 (split master) stage-ring and AdamW-batch sweep; C2 stage sweep.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for S in 0 64 128 200 300; do
  TC_SETUP_TIMING=1 timeout 600 python bench.py --config c3 --secondary "" --no-cpu-baseline --stages $S > gpurun_out/s3_c3_st$S.json 2> gpurun_out/s3_c3_st$S.err; echo "c3 stages $S rc $?"
done
for B in 1 2 8; do
  TC_ADAM_BATCH=$B timeout 600 python bench.py --config c3 --secondary "" --no-cpu-baseline > gpurun_out/s3_c3_b$B.json 2> gpurun_out/s3_c3_b$B.err; echo "c3 batch $B rc $?"
done
for S in 0 24 48; do
  TC_SETUP_TIMING=1 timeout 600 python bench.py --config c2 --secondary "" --no-cpu-baseline --stages $S > gpurun_out/s3_c2_st$S.json 2> gpurun_out/s3_c2_st$S.err; echo "c2 stages $S rc $?"
done
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q > gpurun_out/s3_engine_tests.log 2>&1; echo "engine tests rc $?"; tail -2 gpurun_out/s3_engine_tests.log
