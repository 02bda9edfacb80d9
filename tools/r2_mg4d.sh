run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline $2 2>/dev/null | grep "^{" ; }
for i in 1 2 3; do echo "graph nb8 #$i"; run 2954$i ""; done
echo "graph nb3"; PSB_BENCH_NB=3 run 29545 ""
