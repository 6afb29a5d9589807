"""Time the K1 operator on the C2 system (sliding-window 2D kernel vs the r1 tile kernel).

    python scripts/k1_probe.py            # both variants, L2-cold and L2-warm timings
    python scripts/k1_probe.py run C3     # periodic 512^2 x 32 (PD_NO_GRID_K1=1: general kernel)
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if len(sys.argv) < 2:
    for label, env in (("window", {}), ("tile (r1)", {"PD_K1_NO_WINDOW": "1"})):
        out = subprocess.run([sys.executable, __file__, "run"], env={**os.environ, **env},
                             capture_output=True, text=True)
        print(label, out.stdout.strip(), out.stderr.strip()[-300:])
    sys.exit(0)

import numpy as np
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

name = sys.argv[2] if len(sys.argv) > 2 else "C2"  # C3: the periodic structured kernel
cfg = pd.baseline_config(name) if name == "C2" else pd.baseline_config("C3", Nt=32)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T), 0.0,
                       cfg.u0())
x = N.to_device(s.rhs() + 1.0)
y = N.empty(s.size)
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")  # 256 MB > L2
for _ in range(3):
    s.apply_dev(x, y)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
cold = []
for _ in range(10):
    flush.zero_()
    ev[0].record()
    s.apply_dev(x, y)
    ev[1].record()
    torch.cuda.synchronize()
    cold.append(ev[0].elapsed_time(ev[1]))
torch.cuda.synchronize()
ev[0].record()
for _ in range(20):
    s.apply_dev(x, y)
ev[1].record()
torch.cuda.synchronize()
warm = ev[0].elapsed_time(ev[1]) / 20
alg = (16.0 + 8.0 / 3) * s.size
cold_ms = float(np.median(cold))
print(f"K1 apply {name} ({cfg.spec.n}^2 x {cfg.Nt}): L2-flushed {cold_ms:.4f} ms = {alg / cold_ms / 1e6:.0f} GB/s; back-to-back "
      f"{warm:.4f} ms = {alg / warm / 1e6:.0f} GB/s (algorithmic 16 + 8/M B/dof)")
