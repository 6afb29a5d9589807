"""ncu target: two PFASST iterations of the C4 first window (P=32) in a profiler range."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import pfasst as PF

cfg = pd.baseline_config("C4")
ops = pd.fd_space(cfg.spec)
P = 32
hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, pd.TimeGrid(P, cfg.dt * P), 0.0, L=2, nu=1,
                                 space=ops, M_coarse=cfg.M_coarse)
PF.pfasst_run(hier, cfg.u0(), P, P, 1e-10, 1e-10, max_iters=2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
PF.pfasst_run(hier, cfg.u0(), P, P, 1e-10, 1e-10, max_iters=2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
