# run-to-run variance of the multi-GPU cfg2 step: per-rank step times, exchange, apply, misses
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],4), 'by_rank', d['ms_per_step_by_rank'], 'ex', round(d['exchange']['ms_per_step'],4), 'ap', round(d['apply_ms_per_step'],4), 'k1', round(d['roofline']['avg_launch_ms'],4), 'miss', d['config']['k1_misses_in_timed_window_max_over_ranks'], 'clk', d['clocks']['sm_mhz'])"; }
nvidia-smi topo -m
for i in 1 2 3 4 5; do run 4 2958$i; done
for i in 1 2; do run 2 2957$i; done
