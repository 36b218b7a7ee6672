mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; tail -2 gpurun_out/bench_v9.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-llama > /dev/null 2>&1; wc -l gpurun_out/launches_v3.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glue_kernel -s 8 -c 4 -o gpurun_out/prof_glue2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-llama --no-graph > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_glue2.ncu-rep > gpurun_out/ncu_glue.json 2>&1; head -c 300 gpurun_out/ncu_glue.json
