#!/bin/bash
# The GPU-side recipes behind profiles/, one entry point (run through gpurun:
#   gpurun --timeout 2400 -- 'bash tools/gpu.sh tests bench'
# ). Outputs land in gpurun_out/ (TAG prefixes the file names); summaries worth
# keeping are copied into profiles/. Every A/B inside one call runs on one box
# (box-to-box spread is up to ~7 %).
#
#   tests      pytest -m gpu + smoke()
#   bench      default bench line (C3 headline, C2 secondary, CPU baselines) + the reference arm
#   ab-master  C3 and C2 with split-master states vs the full fp32 master on the host
#   stages     C3 / C2 / C5 HBM stage-ring sweep (auto, then fixed sizes)
#   batch      C3 AdamW batch size (TC_ADAM_BATCH) sweep
#   timeline   absolute per-copy timeline of C3 (tools/timeline.py, GEMM stand-in)
#   nvme       C4 with the NVMe tier: buffered (page cache) and O_DIRECT
#   launches   ncu launch list (gpu__time_duration) of a short default bench
#   ncu        ncu --set full of the fused AdamW inside a C3 step
#   kernels    every data-plane kernel alone at >= 1 GB per launch (events + ncu DRAM bytes)
#   sanitize   compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py
#   contention the packed AdamW alone / beside PCIe DMA / beside or after the GEMMs (tools/adamw_contention_r2.py)
#   adamstream C3 AdamW placement A/B (compute vs optimizer stream, batch size)
#   packedab   C3 packed-only 4-CTA AdamW launches vs the general 3-CTA kernel (TC_ADAM_GENERAL), ROUNDS rounds
#   ncupacked  ncu --set full of the packed AdamW alone
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}" || exit 1
mkdir -p gpurun_out
T=${TAG:-run}
bench() { timeout ${BT:-900} python bench.py "$@"; }
for what in "$@"; do
  case $what in
  tests)
    timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
    echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest_gpu.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
    echo "smoke rc $?"; tail -1 gpurun_out/${T}_smoke.log ;;
  bench)
    bench > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc $?"
    bench --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "reference arm rc $?" ;;
  ab-master)
    for c in c3 c2; do for m in split full; do
      f=""; [ $m = full ] && f="--full-master"
      bench --config $c --secondary "" --no-cpu-baseline $f > gpurun_out/${T}_${c}_$m.json 2> gpurun_out/${T}_${c}_$m.err
      echo "$c $m rc $?"
    done; done ;;
  stages)
    for c in c3 c2 c5; do for s in 0 ${STAGES:-64 128 200}; do
      TC_SETUP_TIMING=1 bench --config $c --secondary "" --no-cpu-baseline --stages $s \
        > gpurun_out/${T}_${c}_st$s.json 2> gpurun_out/${T}_${c}_st$s.err; echo "$c stages $s rc $?"
    done; done ;;
  batch)
    for b in 1 2 4 8; do
      TC_ADAM_BATCH=$b bench --config c3 --secondary "" --no-cpu-baseline > gpurun_out/${T}_c3_b$b.json 2> gpurun_out/${T}_c3_b$b.err
      echo "c3 batch $b rc $?"
    done ;;
  timeline)
    CFG=c3 COMPUTE=2 STAGES=${STAGES:-150} ITERS=5 timeout 600 python tools/timeline.py > gpurun_out/${T}_timeline.txt 2>&1
    echo "timeline rc $?"; cp gpurun_out/timeline_c3.json gpurun_out/${T}_timeline_c3.json ;;
  nvme)
    bench --config c4 --secondary "" --no-cpu-baseline > gpurun_out/${T}_c4_pagecache.json 2> gpurun_out/${T}_c4_pagecache.err
    echo "c4 page cache rc $?"
    bench --config c4 --secondary "" --no-cpu-baseline --direct-io --nvme-dir /tmp > gpurun_out/${T}_c4_odirect.json 2> gpurun_out/${T}_c4_odirect.err
    echo "c4 O_DIRECT rc $?" ;;
  launches)
    # the timed region only (NVTX range), GEMM stand-in at its alone rate (replays would shrink the closed loop)
    TC_STANDIN_OPEN_LOOP=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx \
      --nvtx-include "bench.timed/" --log-file gpurun_out/${T}_launches.csv \
      python bench.py --steps 1 --warmup 3 --secondary "" --no-cpu-baseline > gpurun_out/${T}_launches_bench.log 2>&1
    echo "launch list rc $?" ;;
  ncu)
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:adamw_tma -s 120 -c 1 \
      -o gpurun_out/${T}_adamw_c3 python bench.py --config c3 --steps 1 --warmup 3 --secondary "" --no-cpu-baseline \
      > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc $?" ;;
  kernels)
    timeout 300 python tools/prof_kernels.py --out gpurun_out/${T}_kernels_big.json > gpurun_out/${T}_kernels_big.log 2>&1
    echo "kernels rc $?"
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      -k regex:"adamw|cast|pack|checksum|state_" python tools/prof_kernels.py --reps 2 --out /tmp/k.json \
      > gpurun_out/${T}_ncu_kernels_big.csv 2> gpurun_out/${T}_ncu_kernels_big.err; echo "ncu kernels rc $?" ;;
  sanitize)
    for tool in memcheck racecheck synccheck; do
      timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize.py \
        > gpurun_out/${T}_sanitize_$tool.log 2>&1
      echo "$tool rc $?"; tail -2 gpurun_out/${T}_sanitize_$tool.log
    done ;;
  contention)
    timeout 600 python tools/adamw_contention_r2.py > gpurun_out/${T}_contention.log 2>&1; echo "contention rc $?"
    cp gpurun_out/adamw_contention_r2.json gpurun_out/${T}_adamw_contention_r2.json ;;
  adamstream)
    # C3 AdamW placement A/B, interleaved: compute stream (world-1 default) vs the opt stream, batch sizes
    for r in 1 2; do for v in "ON=1" "ON=1 B=8" "ON=0"; do
      on=${v#ON=}; on=${on%% *}; b=""; [[ $v == *B=* ]] && b=${v##*B=}
      tag=c3_on${on}_b${b:-d}_r$r
      ( export TC_ADAM_ON_COMPUTE=$on; [ -n "$b" ] && export TC_ADAM_BATCH=$b
        bench --config c3 --secondary "" --no-cpu-baseline > gpurun_out/${T}_$tag.json 2> gpurun_out/${T}_$tag.err )
      echo "$tag rc $?"
    done; done ;;
  packedab)
    # packed-only AdamW launches (4 CTAs/SM) vs the general kernel (3 CTAs/SM), interleaved on C3
    for r in ${ROUNDS:-1 2 3}; do for v in packed general; do
      ( [ $v = general ] && export TC_ADAM_GENERAL=1
        bench --config c3 --secondary "" --no-cpu-baseline > gpurun_out/${T}_c3_${v}_r$r.json 2> gpurun_out/${T}_c3_${v}_r$r.err )
      echo "c3 $v r$r rc $?"
    done; done ;;
  ncupacked)
    # ncu --set full of the packed-only AdamW alone (64 Mi elements, tools/prof_kernels.py's split-master case)
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:adamw_tma_kernelILi256ELi2ELb1 -c 1 \
      -o gpurun_out/${T}_adamw_packed_alone python tools/prof_kernels.py --reps 1 --out /tmp/k.json \
      > gpurun_out/${T}_ncupacked.log 2>&1; echo "ncu packed rc $?" ;;
  *) echo "unknown recipe $what"; exit 2 ;;
  esac
done
