timeout 900 python -m pytest tests/test_gpu_producers.py tests/test_gpu_gemm_vs_cublas.py -x -q --timeout 600 2>&1 | tail -3
timeout 600 python tools/prof_7b.py 4 > gpurun_out/prof_7b.txt 2>&1; grep -E "rmsnorm|swiglu|rope" gpurun_out/prof_7b.txt | cut -c1-90,160-240
