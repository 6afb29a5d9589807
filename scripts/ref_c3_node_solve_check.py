"""Build container only (imports the REAL reference from /root/reference, read-only).

Does the reference's own PFASST node solver (pfasst.py:118-132: GMRES(30) + ILU(0),
at most 200 iterations, tol 1e-13) converge on BASELINE config 3 at full size
(512^2 periodic, dt = 0.01, M = 3)?  Measured here: node 0 converges in 186
iterations; nodes 1 and 2 hit the 200-iteration cap (diverged=True), so the
reference's sweep raises SolverError("node solve failed at node 1") in the first
PFASST iteration — the same outcome, at the same node, as the device path
(gpurun: scripts/c3_full_probe.py pfasst).

    python scripts/ref_c3_node_solve_check.py
"""
import os
import sys
import tempfile
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pd_numba_"))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paradiff.collocation import make_tableau
from paradiff.linalg import Ilu0, as_csr, gmres

import paper_2006_12883_b200.problems as PB

cfg = PB.baseline_config("C3")
ops = PB.fd_space(cfg.spec)
tab = make_tableau(3)
dt = cfg.T / cfg.Nt
u0 = cfg.u0()
b = ops.Mh @ u0
for m in range(3):
    q = dt * tab.QDeltaImplicit[m, m]
    A = as_csr(ops.Mh + q * ops.Kh)
    t0 = time.time()
    x, rep = gmres(A, b, precond=Ilu0(A), x0=u0.copy(), tol_rel=1e-13,
                   tol_abs=1e-13 * max(1.0, np.linalg.norm(b)), restart=30, max_it=200)
    print(f"node {m}: {rep.iterations} iterations converged={rep.converged} "
          f"diverged={rep.diverged} residual {rep.residual_history[0]:.3e} -> "
          f"{rep.residual_history[-1]:.3e} ({time.time() - t0:.1f} s)")
