"""BASELINE config 3 at full size (512^2 periodic Fisher, Nt=128, M=3) on one B200:
  (a) Newton + P-fast space-time multigrid (matrix-free; the CSR path would need ~20 GB of
      host assembly), tol 1e-8 as config 5;
  (b) PFASST IMEX (M=3/2, L=2, nu=1), windows of P steps, tol 1e-10.

    python scripts/c3_full_probe.py [stmg|pfasst] [P] [max_windows]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

mode = sys.argv[1] if len(sys.argv) > 1 else "stmg"
cfg = pd.baseline_config("C3")
spec = cfg.spec
if mode == "stmg":
    from paper_2006_12883_b200.pfast import PfastStmg, pfast_rhs

    for nu_t in (1, 2):
        s = PfastStmg(spec, cfg.M, cfg.Nt, cfg.dt, nu_t=nu_t)
        print("levels (steps, grid):", [(a, sp.n) for a, sp, _, _ in s.sched], flush=True)
        b = N.to_device(pfast_rhs(spec, cfg.M, cfg.Nt, cfg.u0()))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, rep = s.newton(b, cfg.gamma, cfg.reaction, tol=1e-8)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        _, res = s.nl_residual(u, b, cfg.gamma, cfg.reaction)
        print(f"C3 Newton + P-fast STMG V({nu_t},{nu_t}): newton={rep.newton_iterations} "
              f"inner={rep.inner_iterations} damped={rep.damped_steps} conv={rep.converged} "
              f"hist={[f'{v:.3e}' for v in rep.residual_history]} |F|={res:.3e} {t:.2f} s", flush=True)
        del s
else:
    from paper_2006_12883_b200 import pfasst as PF

    P = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    W = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    Nt = min(cfg.Nt, P * W)
    ops = pd.fd_space(spec)
    hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, pd.TimeGrid(Nt, cfg.dt * Nt), cfg.gamma, L=2,
                                     nu=1, space=ops, M_coarse=cfg.M_coarse, mode="imex",
                                     reaction_kind=cfg.reaction)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, r = PF.pfasst_run(hier, cfg.u0(), Nt, P, 1e-10, 1e-10)
    torch.cuda.synchronize()
    print(f"C3 PFASST IMEX P={P} Nt={Nt}: per window {list(r.inner_iterations)} "
          f"converged={r.converged} diverged={r.diverged} hist={r.residual_history} "
          f"{time.perf_counter() - t0:.1f} s", flush=True)
