mkdir -p gpurun_out/q8
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x -k "q8" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_apply_gpu.py -q -x -k "q8" 2>&1 | tail -1
PROBE_COMP=q8 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29610 + RANDOM % 50)) tools/probe_step_marks.py full 2>&1 | grep "us per"
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29660 + RANDOM % 50)) bench.py --gpus $N --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 N=$N ms', d['ms_per_step'])"
done
