mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_producers.py -x -q --timeout 600 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_llama.py -x -q --timeout 900 -k "tiny or graph" -s 2>&1 | grep -E "tiny llama|passed|failed|Error|assert" | head
