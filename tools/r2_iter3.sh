for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/it_bench$i.json; done
python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/it_bench_cfg4.json
PSB_BENCH_NO_CLOCKS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(topk_begin|scan|fallback|cand)" --launch-skip 120 --launch-count 40 --csv \
  --log-file gpurun_out/it_launches_cfg2.csv python bench.py --config cfg2 --steps 10 --warmup 30 --no-cpu-baseline --eager > gpurun_out/it_ncu.log 2>&1
