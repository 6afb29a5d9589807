"""Per-kernel stall-reason totals and top SASS lines from an ncu report.
usage: python scripts/ncu_stalls.py REPORT.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append((r[1], cur))
    elif cur is not None:
        cur.append(r)
for name, b in blocks:
    h = b[0]
    ix = {k: i for i, k in enumerate(h)}
    reasons = [k for k in h if k.startswith("stall_") and "Not" not in k]
    tot = {k: 0.0 for k in reasons}
    top, ninst = [], 0
    for r in b[1:]:
        if len(r) != len(h):
            continue
        for k in reasons:
            try:
                tot[k] += float(r[ix[k]])
            except ValueError:
                pass
        try:
            ninst += int(r[ix["Instructions Executed"]])
            top.append((float(r[ix["Warp Stall Sampling (All Samples)"]]), r[ix["Address"]][-5:],
                        r[ix["Source"]].strip(),
                        {k[6:]: r[ix[k]] for k in reasons if r[ix[k]] not in ("0", "")}))
        except ValueError:
            pass
    s = sum(tot.values()) or 1.0
    print(name[:90])
    print("  warp instructions:", ninst)
    print("  ", {k[6:]: round(100 * v / s, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])
                 if v / s > 0.01})
    for t in sorted(top, key=lambda x: -x[0])[:top_n]:
        print("   ", int(t[0]), t[1], t[2][:56], t[3])
