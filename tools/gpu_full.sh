# full round check: all GPU tests, smoke, full bench line (with cpu baseline), reference arm
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 900 2>&1 | tail -4
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err; tail -c 4000 gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.err
