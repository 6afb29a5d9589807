"""P-fast smoother at BASELINE config 5 size (255^3-class periodic grid, M=3,
32 steps, dt=1e-3, coef 0.1): per-sweep device time and per-kernel split.

usage: python scripts/pfast_probe.py [n] [Nt] [sweeps]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2006_12883_b200 import _native as N
from paper_2006_12883_b200.pfast import PfastSolver
from paper_2006_12883_b200.problems import StencilSpec

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
Nt = int(sys.argv[2]) if len(sys.argv) > 2 else 32
K = int(sys.argv[3]) if len(sys.argv) > 3 else 5
spec = StencilSpec(3, n, "periodic", 0.1)
t0 = time.time()
s = PfastSolver(spec, 3, Nt, 1e-3)
print("levels", s.levels, "dofs", s.n, "setup", round(time.time() - t0, 2), "s")
g = torch.Generator(device="cuda").manual_seed(0)
b = torch.rand(s.n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
x = torch.zeros(s.n, dtype=torch.float64, device="cuda")
for _ in range(2):
    s.sweep(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    s.sweep(b, x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
_, r = s.residual(x, b)
print(f"sweep {ms:.2f} ms  {s.n / ms / 1e6:.2f} GDOF/s per sweep  |r|={r:.3e}")
