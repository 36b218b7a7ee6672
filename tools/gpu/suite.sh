#!/bin/bash
# full GPU suite + smoke + default bench + reference arm (the round-end sequence)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest3.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest3.log
timeout 900 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench3.log 2> gpurun_out/bench3.err; echo "bench rc=$?" >> gpurun_out/bench3.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench3_ref.log 2> gpurun_out/bench3_ref.err
tail -c 1500 gpurun_out/gputest3.log; cat gpurun_out/smoke.log | tail -2; tail -c 300 gpurun_out/bench3.err; tail -c 600 gpurun_out/bench3.log; tail -c 300 gpurun_out/bench3_ref.log
