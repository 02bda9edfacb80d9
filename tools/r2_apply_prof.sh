# ncu --set full of the final TMA-staged apply at P = 4 and 8 (cfg2 payloads)
for P in 4 8; do
PROBE_P=$P PROBE_ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sparse_apply_bm -s 3 -c 1 \
  -o gpurun_out/r2_apply_final_p$P python tools/probe_apply.py ring > gpurun_out/r2_apply_ncu_p$P.log 2>&1
done
