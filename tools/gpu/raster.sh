mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm_vs_cublas.py tests/test_gpu_shape_sweep.py -q -x 2>&1 | tail -2
for mb in ${MBS:-0 40 80}; do
  MOSS_GEMM2_L2MB=$mb timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_mxf8 -s 36 -c 12 --csv --log-file gpurun_out/gemm_traffic_$mb.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-llama > /dev/null 2>&1
  MOSS_GEMM2_L2MB=$mb timeout 300 python bench.py --no-llama --no-cpu-baseline --no-e2e > gpurun_out/bench_raster_$mb.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_raster_$mb.json').read().strip().splitlines()[-1])
print('L2MB=$mb', round(d['value'],1), round(d['ms_per_step'],3), d['kernels']['gemm_ms_per_step'])"
done
