timeout 900 python -m pytest tests/test_gpu_quant_fused.py -q -x 2>&1 | tail -1
for v in old new old new; do echo "== $v"; MOSS_B200_LIB=paper_2511_05811_b200/_build/ab/$v.so timeout 300 python tools/quant_probe.py 2>&1 | grep -o "^[0-9x]*:\|fused .*" | paste - - | cut -c1-200; done
