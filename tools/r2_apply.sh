# TMA-staged apply at 4 CTAs/SM: parity (1 and 4 GPUs), us per apply, cfg2 bench lines at N = 2, 4
timeout 600 python -m pytest tests/test_apply_gpu.py -x -q 2>&1 | tail -2
python tools/probe_apply.py ring; PROBE_P=8 python tools/probe_apply.py naive; PROBE_P=3,16 python tools/probe_apply.py ring
timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q -x 2>&1 | tail -3
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],4), 'exchange', d.get('exchange'))"; }
for i in 1 2; do run 2 2957$i; run 4 2958$i; done
