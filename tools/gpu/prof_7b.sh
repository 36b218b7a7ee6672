#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/prof_7b.py 32 > gpurun_out/prof7b_32.txt 2>&1
grep -v "moss::" gpurun_out/prof7b_32.txt | head -45
