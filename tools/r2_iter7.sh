timeout 900 python -m pytest tests/test_apply_gpu.py tests/test_bench_paths_gpu.py -q -x > gpurun_out/it_tests.txt 2>&1
PSB_TILE_DENSITY=0.0001 timeout 900 python -m pytest tests/test_apply_gpu.py -q -x >> gpurun_out/it_tests.txt 2>&1
for D in 0 0.04; do echo "tile_density=$D"; PSB_TILE_DENSITY=$D PROBE_P=4,8 python tools/probe_apply.py ring; PSB_TILE_DENSITY=$D PROBE_P=8 python tools/probe_apply.py naive; done > gpurun_out/it_apply.txt 2>&1
