"""profiles/ncu_gemm_traffic.json from an ncu --csv launch list of the 12 GEMM
launches of one eager LayerStack step (tools/gpu_traffic.sh / gpu_raster.sh)."""
import collections
import csv
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.DictReader(l for l in open(src) if not l.startswith("==")))
per = collections.OrderedDict()
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
for r in rows:
    per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale.get(
        r["Metric Unit"], 1.0)
launches = [{"us": round(d["gpu__time_duration.sum"], 1),
             "dram_read_MB": round(d["dram__bytes_read.sum"], 1),
             "dram_write_MB": round(d["dram__bytes_write.sum"], 1)} for d in per.values()]
flops = 828928688128.0           # LayerStack: 3 GEMMs x 4 linears per step / 12 launches (workloads.py)
tot_us = sum(l["us"] for l in launches)
doc = {"kernel": "moss::gemm_mxf8_2cta_kernel",
       "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over the "
                 f"{len(launches)} GEMM launches of one eager layer step ({src}), round 2 (after the amax epilogue), L2-budget raster "
                 f"(csrc/gemm2.cu g2_raster, MOSS_GEMM2_L2MB=80); all 12 layer GEMMs incl. the MN-major dgrads",
       "dram_bytes_per_launch": sum(l["dram_read_MB"] + l["dram_write_MB"] for l in launches) / len(launches) * 1e6,
       "launches": len(launches), "algorithmic_flops_per_launch": flops,
       "serialized_tflops": flops * len(launches) / (tot_us * 1e-6) / 1e12, "ms_total": tot_us / 1e3,
       "previous_raster_fixed_8_m_pairs_bytes_per_launch": 436.7e6,
       "per_launch": launches}
json.dump(doc, open(dst, "w"), indent=1)
print(doc["dram_bytes_per_launch"] / 1e6, doc["serialized_tflops"])
