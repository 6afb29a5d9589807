"""Aggregate ncu warp-stall samples of one kernel per CUDA source line.

usage: python scripts/ncu_lines.py REPORT.ncu-rep OBJECT.o KERNEL_SUBSTRING [N]
Maps SASS offsets (ncu source page) to source lines with nvdisasm -g line info.
"""
import csv
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
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
name, b = next((n, b) for n, b in blocks if kname in n)
h = b[0]
ix = {k: i for i, k in enumerate(h)}
samples = []
for r in b[1:]:
    if len(r) != len(h):
        continue
    try:
        samples.append((int(r[ix["Address"]], 16), float(r[ix["Warp Stall Sampling (All Samples)"]]),
                        int(r[ix["Instructions Executed"]]), r[ix["Source"]]))
    except ValueError:
        pass
base = min(a for a, *_ in samples)
tmp = Path(tempfile.mkdtemp())
subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=tmp, capture_output=True)
cubin = next(tmp.glob("*.cubin"))
dis = subprocess.run(["nvdisasm", "-g", str(cubin)], capture_output=True, text=True).stdout
# find the function section whose SASS matches the profiled kernel (by instruction text)
funcs = re.split(r"\n\s*\.text\.", dis)
want = [s for _, _, _, s in sorted(samples)[:40]]
best = None
for f in funcs:
    lines = {}
    cur_line = None
    for ln in f.splitlines():
        m = re.search(r'line (\d+)', ln) if "//##" in ln else None
        if m:
            cur_line = int(m.group(1))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", ln)
        if m:
            lines[int(m.group(1), 16)] = (cur_line, m.group(2).strip())
    if not lines:
        continue
    hits = sum(1 for (a, _, _, s) in sorted(samples)[:40]
               if lines.get(a - base, (None, ""))[1].split()[:1] == s.split()[:1])
    if best is None or hits > best[0]:
        best = (hits, lines)
lines = best[1]
agg = defaultdict(lambda: [0.0, 0])
for a, st, n, s in samples:
    ln = lines.get(a - base, (None, ""))[0]
    agg[ln][0] += st
    agg[ln][1] += n
tot = sum(v[0] for v in agg.values())
ninstr = sum(v[1] for v in agg.values())
print(f"{name[:80]}\n samples {tot:.0f}, warp instructions {ninstr}")
for ln, (st, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  line {ln}: {100 * st / tot:5.1f}% stalls, {n} instr")
