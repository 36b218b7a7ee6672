timeout 600 python tools/gemm_ksweep.py 2>&1 | tail -8
timeout 600 python tools/cublas_cmp.py 2>&1 | tail -14
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "gemm" 2>&1 | tail -2
