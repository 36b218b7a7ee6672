mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_v10.json 2> gpurun_out/bench_v10.err; tail -2 gpurun_out/bench_v10.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -c 200
