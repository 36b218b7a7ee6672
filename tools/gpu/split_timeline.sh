#!/bin/bash
mkdir -p gpurun_out
cd paper_2511_05811_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -ftz=false -prec-div=true -prec-sqrt=true -DG2_TIMELINE -o ../_build/libmoss_tl.so *.cu && cd ../..
for sp in 0 1; do for shp in "4096 4096 4096" "4096 4096 22016"; do
MOSS_GEMM2_SPLIT=$sp MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_tl.so timeout 300 python tools/gemm_split_timeline.py $shp
done; done
