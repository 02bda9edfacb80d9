timeout 600 python -m pytest tests/test_apply_gpu.py -q -x 2>&1 | tail -2
for r in 0.01 0.03 0.1; do for v in 20 0; do echo "== rho $r dense_pct $v"; PSB_DENSE_FOLD_PCT=$v PROBE_RHO=$r PROBE_P=2,4,8 PROBE_ITERS=5 python tools/probe_apply.py ring; done; done
