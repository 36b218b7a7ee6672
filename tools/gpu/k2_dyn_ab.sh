#!/bin/bash
# K2 dynamic tile order (MOSS_GEMM2_DYN=1, default) vs static (=0): parity, GEMM rates, layer-step graph A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_kernels.py tests/test_gpu_gemm_bkn.py tests/test_gpu_gemm_amax.py \
  tests/test_gpu_gemm_split.py tests/test_gpu_gemm_vs_cublas.py tests/test_gpu_parity_full.py tests/test_gpu_nn.py -k "gemm or layer or linear or moss" > gpurun_out/k2dyn_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/k2dyn_tests.log)"
for v in 1 0 1 0; do echo "== DYN=$v"; MOSS_GEMM2_DYN=$v python tools/cublas_cmp.py 2>&1 | grep -v -i warn | awk '{print $1, $5, $6}' | tr '\n' ' '; echo; done
python tools/k1_dyn_graph_ab.py 8 MOSS_GEMM2_DYN=1,0 2>&1 | grep MOSS
python tools/k1_dyn_graph_ab.py 8 MOSS_GEMM2_DYN=0,1 2>&1 | grep MOSS
