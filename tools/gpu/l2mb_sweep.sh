#!/bin/bash
# K2 raster L2 budget sweep on the long-K N=4096 shapes: DRAM bytes + duration (ncu, our kernel only)
mkdir -p gpurun_out
for mb in 32 48 64 80; do for shp in "8192 4096 22016" "8192 4096 12288" "8192 4096 11008"; do
MOSS_GEMM2_L2MB=$mb timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:gemm_mxf8 -c 2 python tools/gemm_l2_ncu.py $shp 2>/dev/null | grep -v "^==" > /tmp/l2.csv
python - /tmp/l2.csv "$mb" "$shp" <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; rows=rows[1:]
iid=h.index("ID"); im=h.index("Metric Name"); iv=h.index("Metric Value")
d=collections.OrderedDict()
for r in rows: d.setdefault(r[iid],{})[r[im]]=float(r[iv])
v=list(d.values())[-1]
print(f"L2MB {sys.argv[2]:>3s} {sys.argv[3]:18s} dur {v['gpu__time_duration.sum']/1e3:7.1f} us  DRAM read {v['dram__bytes_read.sum']/1e6:7.1f} MB")
PY
done; done
