for v in tl tl31 tlrel; do echo "== $v"; MOSS_B200_LIB=paper_2511_05811_b200/_build/libmoss_$v.so timeout 300 python tools/gemm_timeline.py 8192 9472 4096 | head -4; done
