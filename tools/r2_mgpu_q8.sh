N=${N:-2}
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q -x -k "q8" > gpurun_out/mg${N}_q8tests.txt 2>&1
for mode in 1 0; do
  PSB_PEER_MODE=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config cfg3 --steps 20 --warmup 5 > gpurun_out/mg${N}_bench_cfg3_m$mode.json 2> gpurun_out/mg${N}_bench_cfg3_m$mode.err
done
