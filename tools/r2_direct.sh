run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],4), 'by_rank', d['ms_per_step_by_rank'], 'ap', d.get('apply_ms_per_step'))"; }
for i in 1 2; do run 4 2958$i; done
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x -k "direct or exchange_paths" 2>&1 | tail -2
