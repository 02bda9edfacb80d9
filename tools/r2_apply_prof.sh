# launch list of the P-payload apply at P = 4 / 8 (light + TMA kernels), cfg2 payloads
for P in 4 8; do
PROBE_P=$P PROBE_ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_sparse_apply|k_seg_offsets" --csv --log-file gpurun_out/apply_launches_p$P.csv python tools/probe_apply.py ring > /dev/null 2>&1
done
