mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant_fused.py -x -q --timeout 600 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "two_level or division" 2>&1 | tail -2
timeout 300 python tools/quant_probe.py 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"quant_mx2_v4" -s 2 -c 2 -o gpurun_out/prof_q4b python tools/ncu_targets.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_q4b.ncu-rep > gpurun_out/prof_q4b.json; grep -E '"kernel"|duration|dram_th|bytes_' gpurun_out/prof_q4b.json
