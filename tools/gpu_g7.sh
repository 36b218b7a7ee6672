timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm 2>&1 | tail -1
MOSS_GEMM2_MODE=3 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_gemm_vs_cublas.py tests/test_gpu_shape_sweep.py -x -q -k "gemm" 2>&1 | tail -1
for m in 2 3; do echo "MODE $m"; MOSS_GEMM2_MODE=$m timeout 600 python tools/cublas_cmp.py 2>&1 | tail -12; MOSS_GEMM2_MODE=$m timeout 300 python tools/gemm_ksweep.py 2>&1 | grep -E "^K=|ours:"; done
