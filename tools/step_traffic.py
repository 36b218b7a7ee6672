"""Summarise an ncu CSV of dram__bytes_read/write + gpu__time_duration per launch:
one line per kernel launch (name, MB read, MB written, us) and totals per kernel family."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = {}
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        if key not in per:
            per[key] = {"name": d["Kernel Name"].split("(")[0].replace("void ", "")[:48]}
            order.append(key)
        v = float(d["Metric Value"].replace(",", ""))
        per[key][d["Metric Name"]] = v
    fam = defaultdict(lambda: [0.0, 0.0, 0.0, 0])
    print(f"# {path}")
    for k in order:
        p = per[k]
        rd, wr, t = p.get("dram__bytes_read.sum", 0) / 1e6, p.get("dram__bytes_write.sum", 0) / 1e6, p.get("gpu__time_duration.sum", 0) / 1e3
        print(f"{p['name']:48s} R {rd:8.1f} MB  W {wr:8.1f} MB  {t:8.1f} us")
        f = fam[p["name"].split("<")[0]]
        f[0] += rd; f[1] += wr; f[2] += t; f[3] += 1
    for name, (rd, wr, t, n) in sorted(fam.items(), key=lambda x: -x[1][2]):
        print(f"TOTAL {name:42s} x{n:3d} R {rd:8.1f} W {wr:8.1f} MB {t:9.1f} us")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
