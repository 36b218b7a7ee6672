mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "gemm or nn" 2>&1 | tail -2
for shape in "8192 4096 12288" "8192 11008 4096" "4096 8192 11008" "8192 4096 4096"; do
  for m in 2 1; do MOSS_GEMM2_MODE=$m python tools/gemm_one.py $shape; done; MOSS_GEMM_VARIANT=1 python tools/gemm_one.py $shape
done
