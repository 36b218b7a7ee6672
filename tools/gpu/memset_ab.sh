#!/bin/bash
# memset graph nodes (MOSS_MEMSET_NODE=1) vs one-thread zeroing kernels (default): layer step + 7B step
mkdir -p gpurun_out
for rep in 1 2; do for v in 0 1; do
MOSS_MEMSET_NODE=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-fp8-roof --steps 60 > gpurun_out/msab_${v}_$rep.json 2>/dev/null
python - gpurun_out/msab_${v}_$rep.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['kernels']['replay_kernel_ms_per_step']
print("MEMSET_NODE", sys.argv[2], "layer", round(d['value']), "TF/s", round(d['ms_per_step'],3), "ms clk", d['clocks']['sm_mhz'],
      "| memset/memcpy", r.get('memset/memcpy'), "| 7B", round(d['llama7b']['tokens_per_s']), "tok/s clk", d['llama7b']['clocks']['sm_mhz'])
PY
done; done
