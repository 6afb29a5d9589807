"""PFASST at full BASELINE sizes on one B200 (C1, C4; C3 IMEX optional).

usage: python scripts/pfasst_full.py [C4] [workers] [max_windows]
Prints per-window iterations, device time and GDOF/s per fine SDC sweep
(N_local = P*M*S per window, sweeps = nu * iterations).
"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import pfasst as PF

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 32
max_windows = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = pd.baseline_config(name)
Nt = cfg.Nt if max_windows <= 0 else min(cfg.Nt, P * max_windows)
ops = pd.fd_space(cfg.spec)
t0 = time.perf_counter()
grid = pd.TimeGrid(Nt, cfg.dt * Nt)
hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, grid, cfg.gamma, L=2, nu=1, space=ops,
                                 M_coarse=cfg.M_coarse,
                                 mode="imex" if cfg.gamma != 0.0 else "implicit",
                                 reaction_kind=cfg.reaction)
print(f"{name}: S={cfg.spec.ndof} M={cfg.M}/{cfg.M_coarse} Nt={Nt} P={P} "
      f"setup {time.perf_counter() - t0:.1f}s", flush=True)
u0 = cfg.u0()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, r = PF.pfasst_run(hier, u0, Nt, P, 1e-10, 1e-10)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    sweeps = sum(r.inner_iterations)  # nu=1: one fine sweep per iteration per window
    dofs = P * cfg.M * cfg.spec.ndof
    print(f"  run {rep}: iterations max {r.iterations} per window {list(r.inner_iterations)} "
          f"converged={r.converged} {t:.2f} s, {dofs * sweeps / t / 1e9:.3f} GDOF/s per fine "
          f"sweep, {Nt * cfg.M * cfg.spec.ndof / t / 1e9:.3f} GDOF/s solved", flush=True)
if os.environ.get("PD_PFASST_PROFILE"):
    from paper_2006_12883_b200.timeslab import phase_profile

    print("phase seconds (both runs):", {k: round(v, 3) for k, v in phase_profile().items()})
