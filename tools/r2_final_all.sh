# final: 4-GPU multi-rank suite + the full -m gpu suite + smoke + bench lines (one 4-GPU box)
mkdir -p gpurun_out/final10
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/final10/gputest_4gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final10/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final10/smoke.txt
python bench.py > gpurun_out/final10/bench_default.json 2> gpurun_out/final10/bench_default.err
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N * 10 + RANDOM % 9)) bench.py --gpus $N --steps 20 --warmup 5 2>/dev/null | grep "^{" > gpurun_out/final10/bench_cfg2_n$N.json
done
