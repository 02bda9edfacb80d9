timeout 600 python -m pytest tests/test_apply_gpu.py -q -x 2>&1 | tail -2
echo "== light 32 (default)"; python tools/probe_apply.py ring; PROBE_P=8 python tools/probe_apply.py naive
echo "== light off"; PSB_APPLY_LIGHT=0 python tools/probe_apply.py ring
