#!/bin/bash
# A/B on the box: K1 producer-mode tile order (MOSS_Q4_REV) x K2 L2 eviction hints (MOSS_GEMM2_L2HINT)
# (in-step kernel figures from bench's instrumented pass) + per-kernel DRAM bytes of one eager step
# with --cache-control none (the producer -> consumer L2 reuse is what is being measured)
mkdir -p gpurun_out
Q="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-llama --no-fp8-roof"
for rep in 1 2; do
for cfg in "0 0" "1 0" "1 1" "1 2" "1 3"; do
  set -- $cfg
  MOSS_Q4_REV=$1 MOSS_GEMM2_L2HINT=$2 timeout 300 $Q > gpurun_out/ab_$1_$2_$rep.json 2>/dev/null
  python - "$1" "$2" gpurun_out/ab_$1_$2_$rep.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
k=d["kernels"]; r=d["roofline"]
print(f"rev={sys.argv[1]} hint={sys.argv[2]}: step {d['ms_per_step']:.3f} ms {d['value']:.0f} TF/s | gemm {r['achieved']:.0f} TF/s gemm_ms {k['gemm_ms_per_step']:.3f} | quant {k['quantize']['ms_per_step']*1e3:.1f} us frac {k['quantize']['frac_of_hbm']:.3f} | prod {k['producers']['frac_of_hbm']:.3f} | sm {d['clocks']['sm_mhz']}")
PY
done
done
for cfg in "0 0" "1 3" "1 1"; do
  set -- $cfg
  MOSS_Q4_REV=$1 MOSS_GEMM2_L2HINT=$2 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/step_traffic_$1_$2.csv python tools/layer_step_ncu.py > /dev/null 2>&1
  python tools/step_traffic.py gpurun_out/step_traffic_$1_$2.csv
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_llama.py::test_llama_125m_gpu_vs_cpu_reference_converged_loss > gpurun_out/gputest2.log 2>&1; echo "gputest rc=$?" >> gpurun_out/gputest2.log
tail -c 1500 gpurun_out/gputest2.log
