mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quant_mx2_v3|gemm_mxf8_2cta|nvjet|cutlass|sm100" -s 1 -c 3 -o gpurun_out/prof_tgt python tools/ncu_targets.py > gpurun_out/ncu_tgt.log 2>&1
tail -5 gpurun_out/ncu_tgt.log
python tools/ncu_summary.py gpurun_out/prof_tgt.ncu-rep > gpurun_out/prof_tgt.json; grep -E '"kernel"|duration|pipe_tensor|dram_th' gpurun_out/prof_tgt.json
