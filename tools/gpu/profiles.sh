#!/bin/bash
# round 2 evidence: launch list + GEMM traffic of the bench layer step, ncu --set full of K1/K2/K3/RMSNorm v3
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-llama --no-fp8-roof"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_mxf8 -s 36 -c 12 --csv --log-file gpurun_out/r02_gemm_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-llama --no-fp8-roof > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_mx2_v4 -s 2 -c 1 -o gpurun_out/r02_full_quant python tools/quant_one.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rmsnorm_fwd_v3 -s 3 -c 1 -o gpurun_out/r02_full_rms_fwd python tools/rmsnorm_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rmsnorm_bwd_v3 -s 3 -c 1 -o gpurun_out/r02_full_rms_bwd python tools/rmsnorm_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adamw_fp8 -s 3 -c 1 -o gpurun_out/r02_full_adamw python tools/adamw_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_mxf8_2cta -s 2 -c 1 -o gpurun_out/r02_full_gemm python tools/gemm_one.py > /dev/null 2>&1
ls -la gpurun_out/r02_*
python tools/ncu_summary.py gpurun_out/r02_full_*.ncu-rep > gpurun_out/r02_ncu_full.json 2>&1; head -c 600 gpurun_out/r02_ncu_full.json
