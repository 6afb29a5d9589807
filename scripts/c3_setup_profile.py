"""cProfile of build_hierarchy + one Newton refresh on a reduced C3 system."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2006_12883_b200 as pd

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Nt = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = pd.baseline_config("C3", n=n, Nt=Nt)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       cfg.gamma, cfg.u0(), reaction_kind="fisher")
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
h = pd.build_hierarchy(s, "SMG", 5, 3)
torch.cuda.synchronize()
t1 = time.perf_counter()
solver = pd.mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9)
x, rep = pd.newton_solve(s, solver, tol=1e-9)
torch.cuda.synchronize()
t2 = time.perf_counter()
pr.disable()
print(f"build {t1 - t0:.1f} s, newton {t2 - t1:.1f} s ({rep.iterations} steps, inner {rep.inner_iterations})")
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
