mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "two_level or fast_division" 2>&1 | tail -3
timeout 300 python tools/probe_perf.py 2>&1 | grep quant
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench2.json 2>gpurun_out/bench2.err; cat gpurun_out/bench2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['kernels']), d['e2e'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"quant_mx2|amax" -s 6 -c 4 -o gpurun_out/prof_quant2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out
