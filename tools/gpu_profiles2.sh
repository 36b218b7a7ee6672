# final round-1 ncu set: hot kernels of the layer step + the 7B producers (one launch each)
mkdir -p gpurun_out
for k in gemm_mxf8_2cta quant_mx2_v4 adamw_fp8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/v3_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-llama > /dev/null 2>&1
done
for k in rmsnorm_fwd_warp rmsnorm_bwd swiglu_bwd rope_fwd; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/v3_$k python tools/prof_7b.py 2 > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/v3_*.ncu-rep > gpurun_out/ncu_full_v3.json
grep -E '"kernel"|duration|dram_th|bytes_read|bytes_write|pipe_tensor_cycles' gpurun_out/ncu_full_v3.json
