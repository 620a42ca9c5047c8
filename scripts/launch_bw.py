"""Per-launch duration, DRAM bytes and bandwidth from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv) for the kernels whose name contains a pattern, last profiled step.
    python scripts/launch_bw.py gpurun_out/x.csv PATTERN [steps]"""
import collections
import csv
import io
import sys

path, pat = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rows = open(path).read().splitlines()
i = next(j for j, line in enumerate(rows) if line.startswith('"ID"'))
d = collections.defaultdict(dict)
tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for x in csv.DictReader(io.StringIO("\n".join(rows[i:]))):
    e = d[x["ID"]]
    e["name"] = x["Kernel Name"].split("(")[0]
    v = float(x["Metric Value"].replace(",", ""))
    u = x["Metric Unit"]
    e[x["Metric Name"]] = v * (tscale[u] if x["Metric Name"] == "gpu__time_duration.sum" else bscale[u])
ids = sorted(d, key=int)
tot_t = tot_b = 0.0
for k in ids[-len(ids) // steps:]:
    e = d[k]
    if pat not in e["name"]:
        continue
    b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    t = e["gpu__time_duration.sum"]
    tot_t += t
    tot_b += b
    print(f"{e['name'][-44:]:44s} {t:8.1f} us {b / 1e6:8.1f} MB {b / t / 1e3:6.0f} GB/s")
print(f"total {tot_t:.1f} us {tot_b / 1e6:.1f} MB {tot_b / max(tot_t, 1e-9) / 1e3:.0f} GB/s")
