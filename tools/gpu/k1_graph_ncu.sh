#!/bin/bash
# ncu of the K1 launches of one layer step: eager vs one CUDA-graph replay (graph-profiling node)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active
for mode in eager graph; do
  arg=""; [ $mode = graph ] && arg="--graph"
  timeout 600 ncu --profile-from-start off --graph-profiling node --cache-control none --clock-control none \
    --kernel-name regex:quant_mx2 --metrics $M --csv --log-file gpurun_out/k1ncu_$mode.csv python tools/layer_step_ncu.py $arg > gpurun_out/k1ncu_$mode.log 2>&1
  echo "== $mode rc=$?"
  python - gpurun_out/k1ncu_$mode.csv <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; rows=rows[1:]
iid=h.index("ID"); im=h.index("Metric Name"); iv=h.index("Metric Value")
d=collections.OrderedDict()
for r in rows: d.setdefault(r[iid],{})[r[im]]=r[iv]
for k,v in d.items(): print(k, {m.split('__')[-1][:28]: v[m] for m in v})
PY
done
