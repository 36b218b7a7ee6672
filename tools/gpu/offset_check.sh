#!/bin/bash
# LayerStack loss offset: producer tests, and long bench runs that crashed with mean(y^2)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_producers.py tests/test_gpu_nn.py tests/test_gpu_graph_dp.py -k "glue or mean_square or offset or layer_stack or graph" > gpurun_out/offset_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/offset_tests.log)"
python bench.py --steps 1000 --warmup 300 --no-cpu-baseline --no-e2e --no-llama --no-fp8-roof 2>gpurun_out/bench_long.err | tail -1 > gpurun_out/bench_long.json
tail -2 gpurun_out/bench_long.err
python -c "
import json; d=json.load(open('gpurun_out/bench_long.json')); k=d['kernels']; print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'], 'K1 cupti', round(k['quantize']['cupti_frac_of_hbm'],3), 'replay', round(k['quantize']['replay_frac_of_hbm'],3))"
