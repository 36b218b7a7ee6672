#!/bin/bash
# K2 raster budget on the K = 4096 shapes: L2 read sectors (dedup) + duration, our kernel only
mkdir -p gpurun_out
for mb in 0 8 16 32 48 80 128; do for shp in "8192 12288 4096" "8192 22016 4096"; do
MOSS_GEMM2_L2MB=$mb timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k regex:gemm_mxf8 -c 2 python tools/gemm_l2_ncu.py $shp 2>/dev/null | grep -v "^==" > /tmp/l2.csv
python - /tmp/l2.csv "$mb" "$shp" <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; rows=rows[1:]
iid=h.index("ID"); im=h.index("Metric Name"); iv=h.index("Metric Value")
d=collections.OrderedDict()
for r in rows: d.setdefault(r[iid],{})[r[im]]=float(r[iv])
v=list(d.values())[-1]
print(f"L2MB {sys.argv[2]:>3s} {sys.argv[3]:16s} dur {v['gpu__time_duration.sum']/1e3:7.1f} us  L2 rd {v['lts__t_sectors_srcunit_tex_op_read.sum']*32/1e9:5.2f} GB  DRAM rd {v['dram__bytes_read.sum']/1e6:6.1f} MB  tensor {v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:5.1f}")
PY
done; done
