timeout 900 python -m pytest tests/test_apply_gpu.py -q -x -k "async" > gpurun_out/it_tests.txt 2>&1
for i in 1 2; do python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/it_bench_cfg4_$i.json; done
python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline --eager 2>&1 | tail -1 > gpurun_out/it_bench_cfg4_eager.json
