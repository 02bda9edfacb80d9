run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline $2 2>/dev/null | grep "^{" ; }
echo "graph nb8 nccl"; PSB_PEER_MODE=0 run 29531 ""
echo "graph nb8 nowire16"; PSB_NO_WIRE16=1 run 29532 ""
echo "graph nb5"; PSB_BENCH_NB=5 run 29533 ""
echo "eager nb3"; PSB_BENCH_NB=3 run 29534 "--eager"
echo "graph nb8 steps40"; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4 --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{"
