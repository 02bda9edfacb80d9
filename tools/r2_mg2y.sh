run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" ; }
for i in 1 2; do echo "clocks 40 #$i"; run 2959$i 40; done
for i in 3 4; do echo "noclocks 40 #$i"; PSB_BENCH_NO_CLOCKS=1 run 2959$i 40; done
echo "clocks 20"; run 29595 20
echo "noclocks 20"; PSB_BENCH_NO_CLOCKS=1 run 29596 20
