run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline $2 2>/dev/null | grep "^{" ; }
echo "graph nb8"; run 29521 ""
echo "eager nb8"; run 29522 "--eager"
echo "graph nb3"; PSB_BENCH_NB=3 run 29523 ""
echo "graph nb8 w30"; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --steps 20 --warmup 30 --no-cpu-baseline 2>/dev/null | grep "^{"
