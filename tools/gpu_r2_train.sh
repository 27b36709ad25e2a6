cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_training_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/r2_train.log 2>&1; echo "train rc $?"
tail -30 gpurun_out/r2_train.log
