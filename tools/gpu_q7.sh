timeout 600 ncu --set full --clock-control none --import-source on -k regex:"quant_mx2_v4" -s 2 -c 1 -o gpurun_out/prof_q7 python tools/ncu_targets.py > /dev/null 2>&1
ls -la gpurun_out/prof_q7.ncu-rep
