for D in 0 4 8 16; do echo "dense=$D"; PSB_APPLY_DENSE=$D python tools/probe_apply.py ring; done > gpurun_out/it_apply.txt 2>&1
