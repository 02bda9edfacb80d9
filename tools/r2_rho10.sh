mkdir -p gpurun_out/rho10
PSB_LIB=libpsb_trace.so PROBE_RHO=0.1 PROBE_NAMES=sb_scan,refine,win_copy,copy_wait,resolve,early_scatter,count,slots,end python tools/probe_cand_trace.py > gpurun_out/rho10/cand_trace2.txt 2>&1
PSB_LIB=libpsb_trace.so PROBE_RHO=0.01 PROBE_NAMES=sb_scan,refine,win_copy,copy_wait,resolve,early_scatter,count,slots,end python tools/probe_cand_trace.py > gpurun_out/rho10/cand_trace2_rho1.txt 2>&1
