#!/bin/bash
mkdir -p gpurun_out
for b in 3 2 1; do
timeout 900 python bench.py --workload llama7b --llama-batch $b --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-fp8-roof > gpurun_out/b7_b$b.json 2>gpurun_out/b7_b$b.err
python - gpurun_out/b7_b$b.json $b <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("batch", sys.argv[2], "7B tok/s", round(d["value"]), "ms", round(d["ms_per_step"],2), "sm", d["clocks"]["sm_mhz"], "peak GB", d["memory"]["peak_allocated_gb"], "replay", d["kernels"].get("replay_kernel_ms_per_step"))
except Exception as e:
    print("batch", sys.argv[2], "failed", e)
PY
tail -3 gpurun_out/b7_b$b.err
done
