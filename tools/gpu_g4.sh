timeout 300 python tools/gemm_ksweep.py 2>&1 | grep -E "^K=|ours:|cublas:"
timeout 600 python tools/cublas_cmp.py 2>&1 | tail -13
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nn.py -x -q --timeout 600 2>&1 | tail -2
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err; python -c "import json; d=json.load(open('gpurun_out/bench_layer.json')); print(d['value'], d['ms_per_step'], d['clocks'], json.dumps(d['roofline']))"
