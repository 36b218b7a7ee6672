#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm_split.py -x -q -p no:cacheprovider 2>&1 | tail -3
for sp in 0 1 0 1; do MOSS_GEMM2_SPLIT=$sp timeout 300 python tools/gemm_split_probe.py; done > gpurun_out/split_probe2.txt 2>&1
grep total gpurun_out/split_probe2.txt
bash tools/gpu/split_timeline.sh 2>&1 | grep -E "split=|round 3|done|entry"
