"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python scripts/launch_share.py LAUNCHES.csv [TITLE]
Per-launch times under ncu are serialised and cold-cache: compare SHARES.
"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
rows = [ln for ln in open(path) if ln.startswith('"')]
tot, cnt = defaultdict(float), defaultdict(int)
for r in csv.DictReader(rows):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    name = re.sub(r"\(.*$", "", name)           # drop the argument list
    name = re.sub(r"^.*::", "", name) if "<" not in name else re.sub(r"^[^<]*::", "", name)
    ns = float(r["Metric Value"].replace(",", ""))
    if r["Metric Unit"] == "us":
        ns *= 1e3
    elif r["Metric Unit"] == "ms":
        ns *= 1e6
    tot[name] += ns
    cnt[name] += 1
total = sum(tot.values())
print(title)
print("per-launch device time, serialised and cold-cache under ncu: compare SHARES, not absolutes")
print(f"total {total / 1e6:.1f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v / total < 0.001:
        continue
    print(f"{k[:44]:44s} {v / 1e6:9.2f} ms {100 * v / total:5.1f}%  n={cnt[k]}")
