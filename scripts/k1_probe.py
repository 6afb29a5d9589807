"""Time the K1 operator on the C2 system vs the CSR SpMV of the same matrix."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N
cfg = pd.baseline_config("C2")
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
x = N.to_device(s.rhs() + 1.0)
y = N.empty(s.size)
for _ in range(3): s.apply_dev(x, y)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize(); ev[0].record()
for _ in range(20): s.apply_dev(x, y)
ev[1].record(); torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 20
print(f"K1 apply C2: {ms:.4f} ms  {16.0*s.size/ms/1e6 + 8*s.size/3/ms/1e6:.0f} GB/s algorithmic (16+8/M B/dof)")
