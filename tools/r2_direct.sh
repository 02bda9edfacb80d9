# direct mode with wire16 arenas (TMA-staged apply reads the peers in place) vs pull, cfg2
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x -k "direct" 2>&1 | tail -2
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],4), 'by_rank', d['ms_per_step_by_rank'], 'ex', d.get('exchange',{}).get('ms_per_step'), 'ap', d.get('apply_ms_per_step'))"; }
for N in 2 4; do echo "== direct wire16 N=$N"; PSB_PEER_MODE=4 run $N 2958$N; echo "== direct u32 N=$N"; PSB_NO_WIRE16=1 PSB_PEER_MODE=4 run $N 2959$N; done
