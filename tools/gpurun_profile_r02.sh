#!/bin/bash
# Round-2 profiling pass (one GPU, from the repo root):
#   1. bench lines (no profiler) for cfg2/cfg3/cfg4/cfg2m at the driver's settings
#   2. ncu launch lists (gpu__time_duration + dram bytes, clocks uncontrolled),
#      steady state (warm-up launches skipped), eager steps
#   3. one `ncu --set full` capture of each dominant kernel, and of the P = 8 apply
# Summaries: python tools/ncu_summary.py gpurun_out/prof2 profiles/r02
set -x
OUT=gpurun_out/prof2
mkdir -p $OUT
python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg3.json 2>&1
python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg4.json 2>&1
python bench.py --config cfg2m --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg2m.json 2>&1
export PSB_BENCH_NO_CLOCKS=1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"^k_" --launch-skip 120 --launch-count 40 --csv \
  --log-file $OUT/launches_cfg2.csv python bench.py --config cfg2 --steps 10 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_launch_cfg2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"^k_" --launch-skip 30 --launch-count 10 --csv \
  --log-file $OUT/launches_cfg3.csv python bench.py --config cfg3 --steps 10 --warmup 30 --no-cpu-baseline --eager \
  > $OUT/ncu_launch_cfg3.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"^k_" --launch-skip 180 --launch-count 60 --csv \
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
PROBE_P=8 PROBE_ITERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sparse_apply_bm --launch-skip 2 --launch-count 1 \
  -o $OUT/k_sparse_apply_bm_p8 python tools/probe_apply.py ring > $OUT/ncu_apply8.log 2>&1
PROBE_P=4 PROBE_ITERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sparse_apply_bm --launch-skip 2 --launch-count 1 \
  -o $OUT/k_sparse_apply_bm_p4 python tools/probe_apply.py ring > $OUT/ncu_apply4.log 2>&1
ls -la $OUT
