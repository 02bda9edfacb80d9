# P-payload apply (tools/probe_apply.py, us per apply), then the 4-GPU suite and cfg2 bench lines
python tools/probe_apply.py ring; PROBE_P=8 python tools/probe_apply.py naive
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q -x 2>&1 | tail -3
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" ; }
for i in 1 2; do run 2 2957$i; run 4 2958$i; done
