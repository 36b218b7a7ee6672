# usage: bash tools/gpu_quick.sh "<pytest -k expr>"   (runs selected gpu tests + kernel probe + bench)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x -k "$1" 2>&1 | tail -4
timeout 300 python tools/probe_perf.py 2>&1 | tail -14
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'gemm', round(d['roofline']['achieved'],1)); print(json.dumps(d['kernels'])); print(d['e2e'])" || tail -5 gpurun_out/bench_q.err
