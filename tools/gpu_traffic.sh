mkdir -p gpurun_out
# every GEMM launch of one eager layer step: DRAM bytes + duration (bench --steps 1 --warmup 3: skip warm-up launches)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_mxf8 -s 36 -c 12 --csv --log-file gpurun_out/gemm_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
wc -l gpurun_out/gemm_traffic.csv
for k in swiglu_fwd rmsnorm_fwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/full_$k python tools/prof_7b.py 2 > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/full_swiglu_fwd.ncu-rep gpurun_out/full_rmsnorm_fwd.ncu-rep > gpurun_out/ncu_prod.json; grep -E '"kernel"|duration|dram_th|bytes_' gpurun_out/ncu_prod.json
