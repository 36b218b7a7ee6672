#!/bin/bash
# round 2: new parity / error-contract tests, then the whole GPU suite, then the default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_error_contract.py tests/test_gpu_parity_full.py tests/test_gpu_graph_dp.py -q -p no:cacheprovider > gpurun_out/new_tests.log 2>&1; echo "new rc=$?" >> gpurun_out/new_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -n 30 gpurun_out/new_tests.log
tail -n 15 gpurun_out/gputest.log
tail -c 600 gpurun_out/bench.log; tail -n 5 gpurun_out/bench.err
