# per-phase CTA time and one ncu --set full capture of the P = 8 apply
PSB_LIB=libpsb_atrace.so PROBE_P=2,4,8 python tools/probe_apply_trace.py > gpurun_out/r2_apply_trace.txt 2>&1
PROBE_P=8 PROBE_ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sparse_apply_bm -s 3 -c 1 \
  -o gpurun_out/r2_apply_p8 python tools/probe_apply.py ring > gpurun_out/r2_apply_ncu.log 2>&1
