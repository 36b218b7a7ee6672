#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_producers.py tests/test_gpu_llama.py -q -p no:cacheprovider -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for m in 0 1 2 3; do MOSS_RMS_V2=$m python tools/rmsnorm_probe.py; done > gpurun_out/rms.txt 2>&1; cat gpurun_out/rms.txt
python tools/graph_timeline.py > gpurun_out/timeline3.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/timeline3.json')); print({k:v for k,v in d.items() if k!='kernels'}); print([round(k['ms']*1e3,1) for k in d['kernels'] if k['kind']=='quant'])"
