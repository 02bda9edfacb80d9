#!/bin/bash
# SURVEY 8d cfg5 sweep on one B200: N x rho, top-k + EF, sync, one rank,
# at the driver's bench settings (--steps 20 --warmup 5).  Run from the repo root.
OUT=${OUT:-gpurun_out/sweep}
mkdir -p $OUT
export PSB_BENCH_NO_CLOCKS=1
for n in 1000000 16000000 125000000 500000000 1000000000; do
  for rho in 0.001 0.01 0.1; do
    timeout 300 python bench.py --n $n --rho $rho --steps 20 --warmup 5 --no-cpu-baseline \
      > $OUT/n${n}_rho${rho}.json 2> $OUT/n${n}_rho${rho}.err || echo "fail n=$n rho=$rho"
  done
done
ls $OUT
