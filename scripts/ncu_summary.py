"""Summarise an `ncu --set full` report into a JSON list (one entry per captured kernel):
time, DRAM bytes, SM / memory throughput, registers, occupancy, L1 hit rate.

usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.json
"""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
ix = {k: i for i, k in enumerate(hdr)}


def val(r, key, default=None):
    i = ix.get(key)
    if i is None or r[i] in ("", "n/a"):
        return default
    return float(r[i].replace(",", ""))


def to_bytes(r, key):
    v = val(r, key, 0.0)
    u = units[ix[key]] if key in ix else "byte"
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def to_ms(r, key):
    v = val(r, key, 0.0)
    u = units[ix[key]]
    return v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1,
                "s": 1e3, "second": 1e3}.get(u, 1)


peak = 6553.0
res = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    ms = to_ms(r, "gpu__time_duration.sum")
    rd, wr = to_bytes(r, "dram__bytes_read.sum"), to_bytes(r, "dram__bytes_write.sum")
    res.append({
        "kernel": r[ix["Kernel Name"]].split("(")[0].replace("void pd::", "").replace(
            "<unnamed>::", ""),
        "grid": r[ix["Grid Size"]], "block": r[ix["Block Size"]], "ms": ms,
        "dram_read_B": rd, "dram_write_B": wr,
        "sm_throughput_pct": val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "mem_throughput_pct": val(
            r, "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
        "regs": val(r, "launch__registers_per_thread"),
        "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "l1_hit_pct": val(r, "l1tex__t_sector_hit_rate.pct"),
        "dram_GBps": (rd + wr) / ms / 1e6 if ms else None,
        "dram_frac_of_6553": (rd + wr) / ms / 1e6 / peak if ms else None,
    })
json.dump(res, open(out, "w"), indent=1)
for e in res:
    print(f"{e['kernel'][:44]:44s} {e['ms']:.3f} ms  {e['dram_GBps']:.0f} GB/s "
          f"({100 * e['dram_frac_of_6553']:.1f}%)  sm {e['sm_throughput_pct']}  regs {e['regs']}")
