#!/bin/bash
# final round-2 evidence: ncu launch list of the default bench command, ncu --set full of K1 (producer
# mode, 8192x4096 and 8192x22016 with the dynamic tail), K3, and the layer GEMM qkv fwd
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-llama --no-fp8-roof"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv $B > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/r02f_launches.csv > gpurun_out/r02f_launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_mx2_v4 -s 2 -c 1 -o gpurun_out/r02f_full_quant python tools/quant_one.py > /dev/null 2>&1
cat > /tmp/quant_big.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2511_05811_b200 import _lib
from paper_2511_05811_b200.quantize import sf_buffer
rows, cols = 8192, 22016
x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
am = x.abs().max().float().reshape(1)
fl = _lib.FlagWord()
codes = torch.empty(rows, cols, dtype=torch.uint8, device="cuda"); sf = sf_buffer(rows, cols, "cuda")
ct = torch.empty(cols, rows, dtype=torch.uint8, device="cuda"); sft = sf_buffer(cols, rows, "cuda")
g = torch.empty(1, device="cuda")
for _ in range(3):
    _lib.quant_mx2_fused(x, am, fl, amax_given=True, codes=codes, sf=sf, codes_t=ct, sf_t=sft, g_out=g)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_mx2_v4 -s 2 -c 1 -o gpurun_out/r02f_full_quant_big python /tmp/quant_big.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adamw_fp8 -s 3 -c 1 -o gpurun_out/r02f_full_adamw python tools/adamw_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_mxf8_2cta -s 2 -c 1 -o gpurun_out/r02f_full_gemm python tools/gemm_one.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02f_full_*.ncu-rep > gpurun_out/r02f_ncu_full.json 2>&1
head -25 gpurun_out/r02f_launches.txt
python -c "
import json; d=json.load(open('gpurun_out/r02f_ncu_full.json'))
for k,v in d.items():
    for r in v: print(k.split('/')[-1], r['kernel'][:40], r.get('gpu__time_duration.sum'), r.get('dram__bytes_read.sum'), r.get('dram__bytes_write.sum'), r.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'), r.get('sm__cycles_elapsed.avg.per_second'))
"
