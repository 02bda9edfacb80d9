# the driver's round-end GPU checks on one GPU: full -m gpu suite, smoke, default bench line
mkdir -p gpurun_out/final8
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/final8/gputest_1gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final8/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final8/smoke.txt
python bench.py > gpurun_out/final8/bench_default.json 2> gpurun_out/final8/bench_default.err
python bench.py --impl reference > gpurun_out/final8/bench_reference.json 2> gpurun_out/final8/bench_reference.err
