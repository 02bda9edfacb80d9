#!/bin/bash
# One 4-GPU gpurun call: NCCL calibration at N=2 and N=4, the cfg2 bench at N=1/2/4, the model report.
set -u
mkdir -p gpurun_out/topo
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python bench.py --steps 50 --warmup 5 > gpurun_out/topo/b1.json 2> gpurun_out/topo/b1.err || exit 1
for N in 2 4; do
  timeout 300 $TR --nproc-per-node $N --master-port $((29600+N)) tools/topology_probe.py calibrate \
      --out gpurun_out/topo/cal$N.json > gpurun_out/topo/cal$N.log 2>&1 || { tail gpurun_out/topo/cal$N.log; exit 1; }
  timeout 300 $TR --nproc-per-node $N --master-port $((29700+N)) bench.py --gpus $N --steps 50 --warmup 5 \
      > gpurun_out/topo/b$N.json 2> gpurun_out/topo/b$N.err || { tail gpurun_out/topo/b$N.err; exit 1; }
done
python tools/topology_probe.py report --bench1 gpurun_out/topo/b1.json \
    --bench gpurun_out/topo/b2.json gpurun_out/topo/cal2.json --bench gpurun_out/topo/b4.json gpurun_out/topo/cal4.json \
    | tee gpurun_out/topo/report.json
