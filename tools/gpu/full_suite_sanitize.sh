#!/bin/bash
# full GPU test suite + compute-sanitizer on K1/K2/K3 (incl. K1's dynamic tail and general path)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest_full.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -3 gpurun_out/gputest_full.log
for tool in memcheck racecheck synccheck; do echo "== $tool"; grep -E "ERROR SUMMARY|Race|rc=" gpurun_out/sanitize_$tool.log | tail -4; done
