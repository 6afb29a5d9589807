"""Wavefront vs level-scheduled ILU(0) apply on a C2 level (timing + bitwise check).

usage: python scripts/wf_probe.py [Nt] [level]   (level 0 = fine 255^2, 1 = 127^2 Galerkin...)
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

Nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ksteps = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1]
cfg = pd.baseline_config("C2", Nt=Nt)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       0.0, cfg.u0())
A = s.global_matrix()
spec = cfg.spec
if level > 0:
    h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
    A = h.matrices[level]
    for _ in range(level):
        spec = spec.coarse()
    del h
A = pd.linalg.as_csr(A)
ilu = pd.BlockJacobiPrecond(A, 8)
b = N.to_device(np.random.default_rng(0).standard_normal(A.shape[0]))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(reps=10):
    out = N.empty(A.shape[0])
    for _ in range(2):
        ilu.solve_dev(b, out)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(reps):
        ilu.solve_dev(b, out)
    ev1.record()
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / reps, out.clone()


t_lvl, x_lvl = timed()
for k in ksteps:
    t0 = time.perf_counter()
    ok = ilu.set_wavefront(3, spec.n, spec.n, 3 * k)
    t_plan = time.perf_counter() - t0
    t_wf, x_wf = timed()
    same = bool(torch.equal(x_lvl, x_wf))
    print(f"level={level} k={k} n={A.shape[0]} nnz={A.nnz} levels={ilu.levels()} plan_ok={ok} "
          f"plan_s={t_plan:.2f} level_ms={t_lvl:.3f} wavefront_ms={t_wf:.3f} bitwise={same}",
          flush=True)
