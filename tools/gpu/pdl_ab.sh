#!/bin/bash
# PDL (MOSS_PDL=1) vs plain launches: parity under PDL, then step time / idle in the layer step graph
mkdir -p gpurun_out
MOSS_PDL=1 timeout 1500 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_nn.py tests/test_gpu_producers.py tests/test_gpu_quant_fused.py \
  tests/test_gpu_graph_dp.py tests/test_gpu_error_contract.py tests/test_gpu_gemm_split.py tests/test_gpu_gemm_amax.py tests/test_gpu_config1.py \
  -k "not two_ranks" > gpurun_out/pdl_tests.log 2>&1; echo "PDL tests: $(tail -1 gpurun_out/pdl_tests.log)"
python tools/k1_dyn_graph_ab.py 10 MOSS_PDL=0,1 2>&1 | grep MOSS_PDL
python tools/k1_dyn_graph_ab.py 10 MOSS_PDL=1,0 2>&1 | grep MOSS_PDL
