"""Per-kernel time / DRAM bytes / GB/s of an ncu launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.

usage: python scripts/ncu_split.py LAUNCHES.csv [first_id]
Per-launch times under ncu are serialised and cold-cache: compare shares.
"""
import csv
import re
import sys
from collections import defaultdict

rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d, order = defaultdict(dict), []
scale_t = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in csv.DictReader(rows):
    k = int(r["ID"])
    if k < first:
        continue
    if k not in d:
        order.append(k)
    d[k]["name"] = re.sub(r"\(.*$", "", r["Kernel Name"]).replace("void ", "").replace("pd::<unnamed>::", "")
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        d[k]["us"] = v * scale_t.get(r["Metric Unit"], 1)
    else:
        d[k][r["Metric Name"]] = v * scale_b.get(r["Metric Unit"], 1)
agg = defaultdict(lambda: [0.0, 0.0, 0])
for k in order:
    e = d[k]
    agg[e["name"]][0] += e["us"]
    agg[e["name"]][1] += e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    agg[e["name"]][2] += 1
tot = sum(a[0] for a in agg.values())
print(f"{len(order)} launches, {tot / 1e3:.2f} ms")
for n, (us, b, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:44s} {us / 1e3:8.2f} ms {100 * us / tot:5.1f}% {b / 1e9:8.2f} GB {b / us / 1e3:6.0f} GB/s n={c}")
