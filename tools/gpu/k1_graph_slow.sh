#!/bin/bash
# why are the backward K1 launches 2-2.5x slower inside the graph replays than in eager steps?
# (eager 8 launches, then graph-replay 8 launches, us)
mkdir -p gpurun_out
run() { echo "=== $*"; env "$@" python tools/quant_clock_probe.py 2>&1 | grep "post K1" | awk '{print $(NF-1)}' | head -16 | tr '\n' ' '; echo; }
run MOSS_CARVEOUT=-1
run X=1
run MOSS_CARVEOUT=-1
run X=1
