mkdir -p gpurun_out
timeout 300 python tools/quant_probe.py 2>&1 | tail -8
timeout 600 python tools/cublas_cmp.py 2>&1 | tail -16
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"quant_mx2_v3|amax" -s 10 -c 4 -o gpurun_out/prof_quant3 python tools/quant_probe.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_quant3.ncu-rep > gpurun_out/prof_quant3.json; head -c 4000 gpurun_out/prof_quant3.json
