mkdir -p gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_mxf8 -s 36 -c 12 --csv --log-file gpurun_out/gemm_traffic_v5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-llama > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-llama > /dev/null 2>&1
wc -l gpurun_out/gemm_traffic_v5.csv gpurun_out/launches_v5.csv
