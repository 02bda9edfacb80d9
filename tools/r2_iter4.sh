python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/it_smoke.txt 2>&1
timeout 900 python -m pytest tests/test_topk_gpu.py tests/test_bench_paths_gpu.py tests/test_apply_gpu.py tests/test_facade_gpu.py tests/test_train_gpu.py -x -q > gpurun_out/it_tests.txt 2>&1
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/it_bench$i.json; done
python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/it_bench_cfg4.json
PSB_LIB=libpsb_trace.so python tools/probe_cand_trace.py > gpurun_out/it_cand_trace.txt 2>&1
