python -m pytest tests/test_gpu_config1.py tests/test_gpu_graph_dp.py -q -p no:cacheprovider -x 2>&1 | grep -E "^(E  |FAILED|tests/|paper_)|Error|passed|failed" | head -40
python -m pytest tests/test_gpu_config1.py "tests/test_gpu_graph_dp.py::test_graphed_exchange_matches_eager[allreduce]" -q -p no:cacheprovider 2>&1 | tail -1
python -m pytest tests/test_gpu_config1.py tests/test_gpu_llama.py::test_cuda_graph_training_matches_eager -q -p no:cacheprovider 2>&1 | tail -1
