timeout 600 python -m pytest tests/test_gpu_quant_fused.py -q -x 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_mx2_v4 -s 2 -c 1 -o gpurun_out/prof_q4 python tools/quant_one.py > /dev/null 2>&1
ls -la gpurun_out/prof_q4.ncu-rep
