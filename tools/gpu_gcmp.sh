mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"gemm_mxf8|nvjet|cutlass|gemm|sm100" -o gpurun_out/prof_gcmp python tools/ncu_gemm_cmp.py 8192,12288,4096 12288,4096,8192 8192,11008,4096 > gpurun_out/ncu_gcmp.log 2>&1
tail -3 gpurun_out/ncu_gcmp.log
python tools/ncu_summary.py gpurun_out/prof_gcmp.ncu-rep > gpurun_out/prof_gcmp.json; grep -E '"kernel"|duration|pipe_tensor_cycles|dram_th|elapsed.avg.per' gpurun_out/prof_gcmp.json
