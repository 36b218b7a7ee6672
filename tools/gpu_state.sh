set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 900 -x 2>&1 | tail -25
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err; tail -c 3000 gpurun_out/bench_layer.json; tail -5 gpurun_out/bench_layer.err
timeout 900 python bench.py --workload llama7b --layers 32 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_7b.json 2>gpurun_out/bench_7b.err; cat gpurun_out/bench_7b.json; tail -20 gpurun_out/bench_7b.err
timeout 600 python tools/prof_7b.py 4 > gpurun_out/prof_7b.txt 2>&1; head -60 gpurun_out/prof_7b.txt
