python tools/probe_cand.py > gpurun_out/it2_cand.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/it2_launches.csv python tools/probe_cand.py > gpurun_out/it2_ncu.log 2>&1
