# Session 3: full prestage of the ring when the forward has no prefetches; timeline + bench C3/C2/C5.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=c3 COMPUTE=2 STAGES=150 ITERS=5 timeout 600 python tools/timeline.py > gpurun_out/s3c_timeline_c3.txt 2>&1; echo "timeline rc $?"
cp gpurun_out/timeline_c3.json gpurun_out/s3c_timeline_c3.json
for S in 0 150; do
  TC_SETUP_TIMING=1 timeout 600 python bench.py --config c3 --secondary "" --no-cpu-baseline --stages $S > gpurun_out/s3c_c3_st$S.json 2> gpurun_out/s3c_c3_st$S.err; echo "c3 stages $S rc $?"
done
TC_SETUP_TIMING=1 timeout 600 python bench.py --config c2 --secondary "" --no-cpu-baseline > gpurun_out/s3c_c2.json 2> gpurun_out/s3c_c2.err; echo "c2 rc $?"
TC_SETUP_TIMING=1 timeout 900 python bench.py --config c5 --secondary "" --no-cpu-baseline > gpurun_out/s3c_c5.json 2> gpurun_out/s3c_c5.err; echo "c5 rc $?"
