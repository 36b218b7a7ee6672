#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) on K1, K2, K3 and one LayerStack step
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
for tool in memcheck racecheck synccheck; do echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$|rc=" gpurun_out/sanitize_$tool.log | tail -6; done
