set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 2>&1 | tail -25
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -c 3000 gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_mxf8 -s 8 -c 2 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls -la gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_mx2 -s 4 -c 2 -o gpurun_out/prof_quant python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adamw -s 4 -c 1 -o gpurun_out/prof_adamw python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
