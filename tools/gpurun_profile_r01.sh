#!/bin/bash
# Round-1 profiling pass (run on the GPU box from the repo root, one GPU):
#   1. plain bench lines (no profiler) for cfg2/cfg3/cfg4
#   2. ncu launch lists (gpu__time_duration.sum, clocks uncontrolled) of the
#      steady state: the warm-up launches are skipped
#   3. one `ncu --set full` capture of each dominant kernel
# Summaries are written by tools/ncu_summary.py into profiles/.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
python bench.py --config cfg3 --no-cpu-baseline > $OUT/bench_cfg3.json 2>&1
python bench.py --config cfg4 --no-cpu-baseline > $OUT/bench_cfg4.json 2>&1
export PSB_BENCH_NO_CLOCKS=1
# eager steps, 30 warm-up steps skipped (cfg2: 4 launches/step, cfg3: 1, cfg4: 6)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 125 --launch-count 40 --csv \
  --log-file $OUT/launches_cfg2.csv python bench.py --config cfg2 --steps 10 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_launch_cfg2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 33 --launch-count 10 --csv \
  --log-file $OUT/launches_cfg3.csv python bench.py --config cfg3 --steps 10 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_launch_cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 185 --launch-count 60 --csv \
  --log-file $OUT/launches_cfg4.csv python bench.py --config cfg4 --steps 10 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_launch_cfg4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_scanIfLi0E --launch-skip 30 --launch-count 1 \
  -o $OUT/k_scan_cfg2 python bench.py --steps 3 --warmup 30 --no-cpu-baseline --eager > $OUT/ncu_kscan.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cand --launch-skip 30 --launch-count 1 \
  -o $OUT/k_cand_cfg2 python bench.py --steps 3 --warmup 30 --no-cpu-baseline --eager > $OUT/ncu_kcand.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_q8_step1 --launch-skip 30 --launch-count 1 \
  -o $OUT/k_q8_step1_cfg3 python bench.py --config cfg3 --steps 3 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_kq8.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:k_scanIfLi0E --launch-skip 30 --launch-count 1 \
  -o $OUT/k_scan_cfg4 python bench.py --config cfg4 --steps 3 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_kscan4.log 2>&1
ls -la $OUT
