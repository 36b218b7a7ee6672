#!/bin/bash
# K1 column pass: ldmatrix.trans loads (MOSS_Q4_LDSM=1, default) vs LDS.32 + PRMT (=0):
# quantizer parity tests under both, then alternated rate probes.
mkdir -p gpurun_out
for v in 1 0; do
MOSS_Q4_LDSM=$v timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_quant_fused.py tests/test_gpu_shape_sweep.py \
  tests/test_gpu_kernels.py tests/test_gpu_parity_full.py -k "quant or shape or bf16 or fused" > gpurun_out/qab_test_$v.log 2>&1
echo "LDSM=$v tests: $(tail -1 gpurun_out/qab_test_$v.log)"
done
for rep in 1 2; do for v in 1 0; do
MOSS_Q4_LDSM=$v timeout 300 python tools/quant_probe.py > gpurun_out/qab_probe_${v}_$rep.log 2>&1
echo "== LDSM=$v rep $rep"; cat gpurun_out/qab_probe_${v}_$rep.log | sed 's/amax .* | row+col/row+col/'
done; done
