mkdir -p gpurun_out
timeout 300 python tools/adamw_contention.py > gpurun_out/contention.log 2>&1
for v in 2 0 4; do
  TC_ADAMW_VARIANT=$v timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v$v.json 2>>gpurun_out/b.err
done
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --compute none > gpurun_out/bench_nocompute.json 2>>gpurun_out/b.err
cat gpurun_out/contention.log
for f in gpurun_out/bench_v*.json gpurun_out/bench_cks16.json gpurun_out/bench_nocompute.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']; print('$f', d['ms_per_step'], r['avg_launch_us'], r['frac'], (r.get('resident_span') or {}).get('avg_us'))"; done
tail -5 gpurun_out/b.err
