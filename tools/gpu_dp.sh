timeout 900 python -m pytest tests/test_gpu_dp_gloo.py -x -q --timeout 800 2>&1 | tail -15
