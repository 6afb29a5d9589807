"""Where the C3 128^2 x 32 parity test spends its time (setup / Newton+SMG / PFASST)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import pfasst as PF


def tick(label, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"{label}: {t - t0:.1f} s", flush=True)
    return t


t = time.perf_counter()
cfg = pd.baseline_config("C3", n=128, Nt=32)
ops = pd.fd_space(cfg.spec)
s = pd.assemble_system(pd.make_tableau(3), ops, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma, cfg.u0(),
                       reaction_kind="fisher")
t = tick("assemble", t)
h = pd.build_hierarchy(s, "SMG", 6, 3)
t = tick("build_hierarchy", t)
print("wavefront", h.wavefront, "grid_spmv", h.grid_spmv, flush=True)
solver = pd.mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9)
import paper_2006_12883_b200.spacetime as ST

orig = solver.__call__ if hasattr(solver, "__call__") else None
x, rep = pd.newton_solve(s, solver, tol=1e-9)
t = tick(f"newton ({rep.iterations} steps, inner {rep.inner_iterations})", t)
hier = PF.build_pfasst_hierarchy(3, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma, L=2, nu=1,
                                 mode="imex", space=ops, M_coarse=2, reaction_kind="fisher")
t = tick("pfasst hierarchy", t)
x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, 8, tol_rel=1e-9, tol_abs=1e-9)
t = tick(f"pfasst (windows {rep.inner_iterations})", t)
