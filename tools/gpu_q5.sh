timeout 900 python -m pytest tests/test_gpu_quant_fused.py -x -q --timeout 600 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 600 -k "two_level or division" 2>&1 | tail -2
timeout 300 python tools/quant_probe.py 2>&1 | tail -6
