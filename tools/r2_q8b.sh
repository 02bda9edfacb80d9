for v in 0 1; do
echo "== scales in place $v"
PSB_Q8_SCALES_INPLACE=$v PROBE_COMP=q8 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29610 + RANDOM % 50)) tools/probe_step_marks.py full 2>&1 | grep "us per"
PSB_Q8_SCALES_INPLACE=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29660 + RANDOM % 50)) bench.py --gpus 2 --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 N=2 ms', d['ms_per_step'])"
done
PSB_Q8_SCALES_INPLACE=1 timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x -k "q8" 2>&1 | tail -2
