# Interleaved A/B of the AdamW batch size (TC_ADAM_BATCH) on one box, C2 and C3, 8 timed steps each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_training_gpu.py -x -q -s > gpurun_out/r2_train.log 2>&1; echo "train rc $?"
for R in 1 2; do for B in 1 2 4; do
  TC_ADAM_BATCH=$B timeout 600 python bench.py --config c2 --secondary "" --no-cpu-baseline --steps 8 > gpurun_out/r2_ab_c2_b${B}_r$R.json 2>/dev/null; echo "c2 b$B r$R rc $?"
  TC_ADAM_BATCH=$B timeout 900 python bench.py --config c3 --secondary "" --no-cpu-baseline --steps 8 > gpurun_out/r2_ab_c3_b${B}_r$R.json 2>/dev/null; echo "c3 b$B r$R rc $?"
done; done
