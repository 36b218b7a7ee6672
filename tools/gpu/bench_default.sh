#!/bin/bash
# one default bench line (the driver's N=1 command) + the reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi.txt
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_d.log 2> gpurun_out/bench_d.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s" >> gpurun_out/bench_d.err
tail -2 gpurun_out/bench_d.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_d.log').read().strip().splitlines()[-1])
k=d['kernels']
print('value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
for n in ('quantize','adamw_fp8','producers'):
    q=k[n]; print(n, {x: round(q[x],3) for x in q if 'frac' in x})
l=d['llama7b']; print('7B tok/s', round(l['tokens_per_s']), 'ms', round(l['ms_per_step'],1), 'peak GB', round(l['peak_allocated_gb'],1), 'clk', l['clocks']['sm_mhz'])
PY
