#!/bin/bash
# K1 general (scaled) path: parity tests, tiny-gradient rate, layer-step K1 after 400 steps
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity_full.py -k "quantizer" tests/test_gpu_quant_fused.py \
  tests/test_gpu_kernels.py -k "two_level or bf16 or quant or fused" > gpurun_out/k1gp_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/k1gp_tests.log)"
python tools/quant_tiny_probe.py 2>&1 | grep -v -i warn
cd paper_2511_05811_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -ftz=false -prec-div=true -prec-sqrt=true -fmad=true -DQ4_TIMELINE -o ../_build/libmoss_q4tl.so *.cu && cd ../..
MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_q4tl.so python tools/k1_timeline.py 400 2>&1 | grep "==\|exit\|MHz"
