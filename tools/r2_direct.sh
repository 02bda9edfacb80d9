timeout 1500 python -m pytest tests/test_multigpu_gpu.py -q -x 2>&1 | tail -2
timeout 600 python -m pytest tests/test_apply_gpu.py -q -x -k "pipeline" 2>&1 | tail -1
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],4), 'ap', d.get('apply_ms_per_step'))"; }
for i in 1 2; do run 2 2957$i; run 4 2958$i; done
