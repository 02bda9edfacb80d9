# final multi-GPU check: GPU tests on 4 GPUs, bench lines at N=2 and N=4 (N=2 through bench.py's own launcher)
mkdir -p gpurun_out/final7
timeout 1800 python -m pytest tests/test_multigpu_gpu.py -q > gpurun_out/final7/mg4_tests.txt 2>&1
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 2>/dev/null | grep "^{" > gpurun_out/final7/bench_cfg2_n2_selflaunch.json
for N in 2 4; do
  for cfg in cfg2 cfg3 cfg4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N * 10 + RANDOM % 9)) bench.py --gpus $N --config $cfg --steps 20 --warmup 5 2>/dev/null | grep "^{" > gpurun_out/final7/bench_${cfg}_n$N.json
  done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29690 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 2>/dev/null | grep "^{" > gpurun_out/final7/bench_reference_n4.json
