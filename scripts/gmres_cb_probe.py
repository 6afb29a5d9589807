"""Probe: GMRES histories of the native and the callable paths vs the oracle across restarts."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import scipy.sparse as sp

import paper_2006_12883_b200 as pd
from oracle import paradiff_oracle as O

np.set_printoptions(precision=6, linewidth=200)
A = sp.csr_matrix(np.diag([1.0, 2.0, 3.0, 4.0, 5.0, 6.0]))
b = np.ones(6)
for R in (1, 2, 3):
    for mi in (R, 3 * R):
        x, rep = pd.gmres(A, b, tol_rel=1e-30, tol_abs=0.0, restart=R, max_it=mi)
        xo, repo = O.gmres(A, b, None, tol_rel=1e-30, tol_abs=0.0, restart=R, max_it=mi)
        ok = np.allclose(rep.residual_history, repo.residual_history, rtol=1e-9) and np.allclose(x, xo)
        print(f"R={R} max_it={mi} match={ok}")
