#!/bin/bash
# K1 producer mode: staggered initial loads (MOSS_Q4_STAGGER=1) vs all three at once (=0)
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_quant_fused.py tests/test_gpu_parity_full.py tests/test_gpu_nn.py -k "quant or fused or producer or dynamic or moss or linear" > gpurun_out/stagger_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/stagger_tests.log)"
for v in 1 0 1 0; do echo "== STAGGER=$v"; MOSS_Q4_STAGGER=$v python tools/quant_probe.py 2>&1 | sed 's/.*producer-amax/producer-amax/' | grep -v -i warn; done
python tools/k1_dyn_graph_ab.py 8 MOSS_Q4_STAGGER=1,0 2>&1 | grep MOSS
python tools/k1_dyn_graph_ab.py 8 MOSS_Q4_STAGGER=0,1 2>&1 | grep MOSS
