#!/bin/bash
# K1 producer mode: dynamic tile counter (MOSS_Q4_DYN=1, default) vs static round-robin (=0)
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity_full.py -k "quantizer" tests/test_gpu_quant_fused.py \
  tests/test_gpu_kernels.py tests/test_gpu_nn.py tests/test_gpu_producers.py -k "two_level or bf16 or quant or fused or producer or amax or graph" > gpurun_out/k1dyn_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/k1dyn_tests.log)"
for rep in 1 2; do for v in 1 0; do
echo "== DYN=$v"; MOSS_Q4_DYN=$v timeout 300 python tools/quant_probe.py 2>&1 | sed 's/.*| row+col/row+col/' | grep -v -i warn
done; done
cd paper_2511_05811_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -ftz=false -prec-div=true -prec-sqrt=true -fmad=true -DQ4_TIMELINE -o ../_build/libmoss_q4tl.so *.cu && cd ../..
for v in 1 0; do echo "== timeline DYN=$v"; MOSS_Q4_DYN=$v MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_q4tl.so python tools/k1_timeline.py 100 2>&1 | grep "==\|exit\|tiles"; done
for v in 1 0; do MOSS_Q4_DYN=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-fp8-roof --no-llama > gpurun_out/k1dyn_b$v.json 2>/dev/null
python - gpurun_out/k1dyn_b$v.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); q=d['kernels']['quantize']
print("DYN", sys.argv[2], "layer", round(d['value']), "clk", d['clocks']['sm_mhz'], "K1 cupti", round(q['cupti_frac_of_hbm'],3), "replay", round(q['replay_frac_of_hbm'],3), q['replay_ms_per_step'])
PY
done
