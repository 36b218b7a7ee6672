for m in 2 1 0; do echo "MODE $m"; MOSS_GEMM2_MODE=$m timeout 300 python tools/gemm_ksweep.py 2>&1 | grep -E "^K=|ours:"; done
