timeout 300 python -m pytest tests/test_gpu_producers.py -q -x -k "glue or fused_block" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glue_kernel -s 8 -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-llama --no-graph 2>/dev/null | grep -v "^==" | cut -d, -f5,13- | tail -12
timeout 300 python bench.py --no-llama --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), d['kernels']['producers'])"
