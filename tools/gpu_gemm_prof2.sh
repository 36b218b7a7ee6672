mkdir -p gpurun_out
python tools/gemm_one.py
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -s 3 -c 1 -o gpurun_out/prof_g2b python tools/gemm_one.py > /dev/null 2>&1
ls gpurun_out
