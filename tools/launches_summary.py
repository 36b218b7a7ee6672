"""profiles/r01_launches_*.txt from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

src = sys.argv[1]
EXCLUDE = ("spin_kernel", "cutlass3x_sm100", "distribution_elementwise")   # device sleep, cuBLASLt reference, init
rows = [r for r in csv.DictReader(l for l in open(src) if not l.startswith("==")) if r["Metric Name"] == "gpu__time_duration.sum"
        and not any(e in r["Kernel Name"] for e in EXCLUDE)]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows:
    t = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    a = agg.setdefault(r["Kernel Name"], [0.0, 0])
    a[0] += t
    a[1] += 1
tot = sum(a[0] for a in agg.values())
print(f"# total {tot / 1e3:.3f} ms over {len(rows)} launches")
for name, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100 * t / tot:6.2f}% {t:11.1f} us {n:5d} launches  {name[:100]}")
