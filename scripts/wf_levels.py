"""Wavefront vs level-scheduled ILU(0) applies on every C2 SMG level, for
several lower-sweep task sizes (time steps per CTA); bitwise check each.

usage: python scripts/wf_levels.py [Nt] [k,k,...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

Nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ks = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
cfg = pd.baseline_config("C2", Nt=Nt)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
mats = [pd.linalg.as_csr(m) for m in h.matrices[:-1]]
specs = [cfg.spec]
for _ in range(len(mats) - 1):
    specs.append(specs[-1].coarse())
del h
torch.cuda.empty_cache()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
total = {}
for l, (A, spec) in enumerate(zip(mats, specs)):
    ilu = pd.BlockJacobiPrecond(A, 8)
    b = N.to_device(np.random.default_rng(l).standard_normal(A.shape[0]))

    def timed(reps=20):
        out = N.empty(A.shape[0])
        for _ in range(3):
            ilu.solve_dev(b, out)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            ilu.solve_dev(b, out)
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps, out.clone()

    t_lvl, x_lvl = timed()
    line = [f"level={l} n={A.shape[0]} side={spec.n} levels={ilu.levels()} level_sched={t_lvl:.3f}ms"]
    for k in ks:
        if 3 * k * spec.n > 768 and k > 1:
            continue
        ok = ilu.set_wavefront(3, spec.n, spec.n, 3 * k)
        t, x = timed()
        same = bool(torch.equal(x_lvl, x))
        line.append(f"k={k}:{t:.3f}ms{'' if ok else '(no plan)'}{'' if same else ' MISMATCH'}")
        total.setdefault(k, 0.0)
    print("  ".join(line), flush=True)
    del ilu
