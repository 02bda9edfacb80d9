mkdir -p gpurun_out/rho10
python tools/probe_phases.py > gpurun_out/rho10/phases.txt 2>&1
PSB_LIB=libpsb_trace.so PROBE_RHO=0.1 python tools/probe_cand_trace.py > gpurun_out/rho10/cand_trace.txt 2>&1
