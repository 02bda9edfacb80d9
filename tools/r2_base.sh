set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2_base_bench$i.json; done
PROBE_STEPS=80 python tools/probe_misses.py > gpurun_out/r2_base_misses.txt 2>&1
python tools/probe_cand.py > gpurun_out/r2_base_cand.txt 2>&1
