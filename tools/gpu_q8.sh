timeout 900 python -m pytest tests/test_gpu_quant_fused.py -q -x 2>&1 | tail -1
for i in 1 2; do
timeout 300 python bench.py --no-llama --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; q=k['quantize_standalone']
print(round(d['value'],1), 'instep', round(k['quantize']['frac_of_hbm'],3), round(k['quantize']['ms_per_step'],3), 'single', round(q['single_launch_amax']['frac_of_hbm'],3), 'producer', round(q['producer_amax']['frac_of_hbm'],3))"
done
