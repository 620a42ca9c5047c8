"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches and time per profiled step.
    python scripts/launch_summary.py gpurun_out/x.csv [steps]"""
import collections
import csv
import io
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = open(path).read().splitlines()
i = next(j for j, line in enumerate(rows) if line.startswith('"ID"'))
r = [x for x in csv.DictReader(io.StringIO("\n".join(rows[i:]))) if x["Metric Name"] == "gpu__time_duration.sum"]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for x in r:
    n = x["Kernel Name"]
    n = n[:44] if "gemm" in n else n.split("(")[0]
    agg[n][0] += 1
    agg[n][1] += float(x["Metric Value"].replace(",", "")) * scale[x["Metric Unit"]]
tot = sum(a[1] for a in agg.values())
print(f"total {tot / steps:.1f} us per step ({len(r) / steps:.0f} launches)")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:64s} {c / steps:6.1f} {t / steps:10.1f} us {t / tot:6.1%}")
