#!/bin/bash
# bench's graph-replay quantizer times in launch order + how the captured step's quantizers got their amax
mkdir -p gpurun_out
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-llama --no-e2e --no-fp8-roof > gpurun_out/bk_1.json 2>gpurun_out/bk_1.err
python - gpurun_out/bk_1.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=d["kernels"]; rk=k["replay_kernel_ms_per_step"]
print(round(d["value"]), "timed clocks", d["clocks"]["sm_mhz"], "replay clocks", rk.get("clocks"))
print("captured modes", k.get("captured_quant_amax_modes"))
print("quant replay ms", rk["quant"], "gemm", rk["gemm"])
print(rk["last_replay_quant_gemm_us"])
PY
python tools/replay_vs_eager.py 2>&1 | grep -v Warn | head -4
