#!/bin/bash
# K2 vs cuBLASLt MXFP8: L2 -> SM bytes, L2 output throughput, tensor pipe activity (ncu, one launch each)
mkdir -p gpurun_out
MET=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size,launch__cluster_dim_x,lts__throughput.avg.pct_of_peak_sustained_elapsed
for shp in "8192 12288 4096" "8192 4096 4096" "8192 4096 22016"; do
timeout 600 ncu --metrics $MET --clock-control none --csv -k "regex:gemm|nvjet|cutlass|xmma|sm10" -c 4 python tools/gemm_l2_ncu.py $shp 2>/dev/null | grep -v "^==" > gpurun_out/gemm_l2_${shp// /x}.csv
echo "== $shp"
python - gpurun_out/gemm_l2_${shp// /x}.csv <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; rows=rows[1:]
iid=h.index("ID"); ik=h.index("Kernel Name"); im=h.index("Metric Name"); iv=h.index("Metric Value")
d=collections.OrderedDict()
for r in rows: d.setdefault((r[iid], r[ik][:40]),{})[r[im]]=r[iv]
for k,v in d.items(): print(k[1], {m.split('__')[-1][:40]: v[m] for m in v})
PY
done
