#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --workload llama7b --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-fp8-roof > gpurun_out/b7_gaps.json 2>gpurun_out/b7_gaps.err
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-llama --no-e2e --no-fp8-roof > gpurun_out/bl_gaps.json 2>gpurun_out/bl_gaps.err
for f in b7_gaps bl_gaps; do python - gpurun_out/$f.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=d["kernels"]
print(sys.argv[1], round(d["value"]), "ms", round(d["ms_per_step"],3), "sm", d["clocks"]["sm_mhz"], "gaps", k.get("replay_gaps"))
print("  ", {a: {x: round(y,3) for x,y in b.items()} for a,b in k["replay_kernel_ms_per_step"].items()})
PY
done
