# round-1 profile set: launch list of one bench step + ncu --set full of each hot kernel
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_layer.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; wc -l gpurun_out/launches_layer.csv
for k in gemm_mxf8_2cta quant_mx2_v4 adamw_fp8 swiglu_fwd rmsnorm_fwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o gpurun_out/full_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
done
for k in rmsnorm_bwd rope_bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/full_$k python tools/prof_7b.py 2 > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/full_*.ncu-rep > gpurun_out/ncu_full_r01.json; grep -E '"kernel"|duration|dram_th|bytes_read|bytes_write|pipe_tensor_cycles' gpurun_out/ncu_full_r01.json
timeout 300 python bench.py --zero1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -c 600
