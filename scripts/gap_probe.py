"""Kernel timeline of one C2 SMG solve (torch.profiler / CUPTI): busy time vs
span, and the idle gaps between consecutive kernels.  usage: python scripts/gap_probe.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

cfg = pd.baseline_config("C2")
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
b = N.to_device(s.rhs())
x = N.zeros(b.numel())
for _ in range(2):
    x.zero_()
    h.solve_dev(b, x, 1e-10, 1e-10)
torch.cuda.synchronize()
x.zero_()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    h.solve_dev(b, x, 1e-10, 1e-10)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
ks = [k for k in ks if k[1] > k[0]]
span = ks[-1][1] - ks[0][0]
busy = sum(e - s_ for s_, e, _ in ks)
gaps = [ks[i + 1][0] - ks[i][1] for i in range(len(ks) - 1)]
gaps_pos = [g for g in gaps if g > 0]
print(f"kernels={len(ks)} span={span/1e3:.2f} ms busy={busy/1e3:.2f} ms "
      f"idle={(span-busy)/1e3:.2f} ms ({(span-busy)/span*100:.1f}%)")
print(f"gap median={np.median(gaps):.2f} us mean={np.mean(gaps):.2f} us max={max(gaps):.1f} us")
big = sorted(((g, ks[i][2][:40], ks[i + 1][2][:40]) for i, g in enumerate(gaps)), reverse=True)[:8]
for g, a, c in big:
    print(f"  gap {g:8.1f} us after {a} before {c}")
