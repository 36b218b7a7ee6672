mkdir -p gpurun_out
python tools/gemm_one.py; MOSS_GEMM_VARIANT=1 python tools/gemm_one.py
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -s 3 -c 1 -o gpurun_out/prof_g2 python tools/gemm_one.py > /dev/null 2>&1
MOSS_GEMM_VARIANT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -s 3 -c 1 -o gpurun_out/prof_g1 python tools/gemm_one.py > /dev/null 2>&1
ls gpurun_out
