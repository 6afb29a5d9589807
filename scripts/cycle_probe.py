"""One C2 SMG solve inside cudaProfilerStart/Stop (for ncu launch lists)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

Nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = pd.baseline_config("C2", Nt=Nt)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
b = N.to_device(s.rhs())
x = N.zeros(s.size)
h.solve_dev(b, x, 1e-10, 1e-10, 100)
x.zero_()
torch.cuda.synchronize()
torch.cuda.profiler.start()
_, rep = h.solve_dev(b, x, 1e-10, 1e-10, 100)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("cycles", rep.iterations)
