set -x
python -m pytest tests/test_apply_gpu.py -x -q 2>&1 | tail -3
for o in ring naive; do PSB_LIB=libpsb_base.so python tools/probe_apply.py $o; python tools/probe_apply.py $o; done
PROBE_P=3,16 python tools/probe_apply.py ring
