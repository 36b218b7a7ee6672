#!/bin/bash
# tail split: tests, then bench (layer + 7B) with and without the split, CUPTI in-graph kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm_split.py tests/test_gpu_gemm_vs_cublas.py tests/test_gpu_gemm_amax.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider > gpurun_out/t_split.log 2>&1; echo "rc=$?" >> gpurun_out/t_split.log
tail -5 gpurun_out/t_split.log
for sp in 1 0; do
  MOSS_GEMM2_SPLIT=$sp timeout 600 python bench.py --workload llama7b --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-fp8-roof > gpurun_out/b7_split$sp.json 2>gpurun_out/b7_split$sp.err
  python - gpurun_out/b7_split$sp.json $sp <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
rk=d["kernels"].get("replay_kernel_ms_per_step")
print("split", sys.argv[2], "7B tok/s", round(d["value"]), "ms", round(d["ms_per_step"],2), "sm", d["clocks"]["sm_mhz"], "gemm_replay", d["roofline"].get("achieved_replay_cupti"), rk)
PY
done
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-llama > gpurun_out/b_layer.json 2>gpurun_out/b_layer.err
python - gpurun_out/b_layer.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=d["kernels"]
print("layer", round(d["value"]), "e2e", round(d["e2e"]["value"]), "gemm", round(d["roofline"]["achieved"]), "gemm_replay", d["roofline"].get("achieved_replay_cupti"), "frac", d["roofline"]["frac"], "sm", d["clocks"]["sm_mhz"])
for n in ("quantize","adamw_fp8","producers"):
    print(n, {a: (round(b,4) if isinstance(b,float) else b) for a,b in k[n].items()})
PY
