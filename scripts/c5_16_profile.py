"""Timing of the C5 16^3 x 8 Newton + STMG parity case (setup / solve split)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2006_12883_b200 as pd

t0 = time.perf_counter()
cfg = pd.baseline_config("C5", n=16, Nt=8)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       cfg.gamma, cfg.u0())
h = pd.build_hierarchy(s, "STMG", 3, 3)
torch.cuda.synchronize()
t1 = time.perf_counter()
x, rep = pd.newton_solve(s, pd.mg_linear_solver(h, tol_rel=1e-8, tol_abs=1e-8), tol=1e-8)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"build {t1 - t0:.1f} s, newton {t2 - t1:.1f} s ({rep.iterations} steps, inner {rep.inner_iterations})")
