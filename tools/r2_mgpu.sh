N=${N:-2}
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/mg${N}_tests.txt 2>&1
for cfg in cfg2 cfg3 cfg4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg --steps 20 --warmup 5 > gpurun_out/mg${N}_bench_$cfg.json 2> gpurun_out/mg${N}_bench_$cfg.err
done
