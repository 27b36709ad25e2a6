#!/bin/bash
# Flexible GPU session: STEPS env lists what to run.
mkdir -p gpurun_out
for s in $STEPS; do
case $s in
  tests) timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log ;;
  smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log ;;
  bench) timeout 900 python bench.py --steps ${BENCH_STEPS:-5} --warmup ${BENCH_WARMUP:-3} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json ;;
  c4) timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline $C4_ARGS > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 800 gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err ;;
  ref) timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json ;;
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; wc -l gpurun_out/launches.csv ;;
  prof) V=2 bash tools/gpu_prof.sh ;;
  disk) (dd if=/dev/zero of=/tmp/ddtest bs=64M count=32 oflag=direct 2>&1 | tail -1; dd if=/tmp/ddtest of=/dev/null bs=64M iflag=direct 2>&1 | tail -1; rm -f /tmp/ddtest) > gpurun_out/disk.txt; cat gpurun_out/disk.txt ;;
esac
done
