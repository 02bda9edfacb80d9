PROBE_NB=3 PROBE_OUT=gpurun_out/tdrift_nb3.json python tools/probe_tdrift.py > gpurun_out/tdrift_nb3.txt 2>&1
PROBE_NB=8 PROBE_OUT=gpurun_out/tdrift_nb8.json python tools/probe_tdrift.py > gpurun_out/tdrift_nb8.txt 2>&1
PSB_LIB=libpsb_trace.so python tools/probe_scan_trace.py > gpurun_out/scan_trace.txt 2>&1
