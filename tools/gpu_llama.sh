mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_llama.py -q -rf -s --timeout 1200 2>&1 | grep -E "tiny llama|125M|passed|failed|Error|assert" | head -20
timeout 900 python bench.py --workload llama7b --layers 32 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_7b.json 2>gpurun_out/bench_7b.err; python -c "import json; d=json.load(open('gpurun_out/bench_7b.json')); print('7B tok/s', round(d['value']), 'ms', round(d['ms_per_step'],1), 'gemm TF', round(d['roofline']['achieved']), 'share', round(d['roofline']['share_of_step'],3)); print(json.dumps(d['kernels'])); print(d['e2e'])" || tail -5 gpurun_out/bench_7b.err
nvidia-smi --query-gpu=memory.used --format=csv
