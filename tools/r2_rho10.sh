mkdir -p gpurun_out/rho10
timeout 900 python -m pytest tests/test_bench_paths_gpu.py -q -x -k "merge or unstaged" 2>&1 | tail -2
for rho in 0.1 0.05 0.03; do for v in 5 0; do
PSB_DENSE_MERGE_PCT=$v python bench.py --rho $rho --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rho $rho merge_pct $v ms', round(d['ms_per_step'],4), 'step_frac', round(d['roofline']['step_frac'],3))"
done; done
