timeout 900 python -m pytest tests/test_gpu_zero.py tests/test_gpu_llama.py -x -q --timeout 600 -k "zero or transpose or graph" 2>&1 | tail -15
