run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 --steps $3 --warmup 5 --no-cpu-baseline $2 2>/dev/null | grep "^{" ; }
for i in 1 2 3; do echo "graph #$i"; run 2957$i "" 20; done
echo "eager"; run 29575 "--eager" 20
echo "graph 40"; run 29576 "" 40
