mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for f in gpurun_out/bench_c2.json gpurun_out/bench_c3.json; do python -c "
import json; d=json.load(open('$f')); p=d['pcie']; print('$f', d['ms_per_step'], d['value'], p['duplex_frac'], d['migration_hidden_frac'], d['roofline']['avg_launch_us'], d['e2e'])" 2>/dev/null || (echo "$f failed"; tail -n 5 ${f%.json}.err); done
