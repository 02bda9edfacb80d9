run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" ; }
for N in 2 4; do
  for i in 1 2; do echo "N=$N pipe #$i"; run $N 296$N$i; echo "N=$N serial #$i"; PSB_BENCH_NO_PIPE=1 run $N 297$N$i; done
done
