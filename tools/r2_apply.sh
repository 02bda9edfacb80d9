timeout 600 python -m pytest tests/test_apply_gpu.py -x -q 2>&1 | tail -2
python tools/probe_apply.py ring; PROBE_P=8 python tools/probe_apply.py naive; PSB_APPLY_NO_TMA=1 PROBE_P=8 python tools/probe_apply.py ring
