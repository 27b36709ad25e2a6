# Round 2: GPU suite, big-launch kernel roofline (events + ncu DRAM bytes), AdamW batch A/B on C2 and C3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2_pytest_gpu.log
timeout 300 python tools/prof_kernels.py --out gpurun_out/r2_kernels_big.json > gpurun_out/r2_kernels_big.log 2>&1; echo "kernels rc $?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:"adamw|cast|pack|checksum" python tools/prof_kernels.py --reps 2 --out /tmp/x.json > gpurun_out/r2_ncu_kernels_big.csv 2> gpurun_out/r2_ncu_kernels_big.err; echo "ncu rc $?"
for B in 1 4; do
  TC_ADAM_BATCH=$B timeout 600 python bench.py --config c2 --secondary "" --no-cpu-baseline > gpurun_out/r2_bench_c2_batch$B.json 2> gpurun_out/r2_bench_c2_batch$B.err; echo "c2 batch $B rc $?"
  TC_ADAM_BATCH=$B timeout 900 python bench.py --config c3 --secondary "" --no-cpu-baseline > gpurun_out/r2_bench_c3_batch$B.json 2> gpurun_out/r2_bench_c3_batch$B.err; echo "c3 batch $B rc $?"
done
