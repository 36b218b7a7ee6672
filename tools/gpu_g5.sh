MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_tl.so timeout 300 python tools/gemm_timeline.py 8192 9472 4096 2>&1 | head -8
timeout 300 python tools/gemm_ksweep.py 2>&1 | grep -E "^K=|ours:|cublas:"
timeout 600 python tools/cublas_cmp.py 2>&1 | tail -13
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k gemm 2>&1 | tail -2
