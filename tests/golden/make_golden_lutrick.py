"""Golden PFASST/SDC runs of the REAL reference with the "lu-trick" Q_delta
(collocation.py:119-123).  Build container only:

    python tests/golden/make_golden_lutrick.py

Writes tests/golden/lutrick.npz; tests/test_gpu_pfasst.py checks the device sweeps
against it.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pd_numba_"))
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import paradiff  # noqa: E402
from paradiff import (SpaceMesh, TimeGrid, build_pfasst_hierarchy, heat_problem,  # noqa: E402
                      monodomain_problem, pfasst_run)
from paradiff.pfasst import sdc_solve_step, spread_state  # noqa: E402

assert str(Path(paradiff.__file__).resolve()).startswith(REF), paradiff.__file__

out = {}
heat = heat_problem()
mesh = SpaceMesh(32, heat.X)
hier = build_pfasst_hierarchy(3, mesh, TimeGrid(8, heat.T), 0.0, L=2, nu=1, qdelta="lu-trick")
U, rep = pfasst_run(hier, heat.u0(mesh.vertices), 8, 4, tol_rel=1e-10, tol_abs=1e-10)
out.update(heat_U=U, heat_its=np.array(rep.inner_iterations), heat_conv=rep.converged)
# one fine sweep and a single-step SDC solve from the spread state
st = spread_state(heat.u0(mesh.vertices), 3)
out["heat_sweep1"] = hier.fine.sweep(st).U
st2, rep2 = sdc_solve_step(heat.u0(mesh.vertices), hier.fine, tol_rel=1e-11, tol_abs=1e-12)
out.update(heat_step_U=st2.U, heat_step_its=rep2.iterations)
mono = monodomain_problem()
mesh2 = SpaceMesh(64, mono.X)
hier2 = build_pfasst_hierarchy(3, mesh2, TimeGrid(8, 0.5), mono.gamma, L=2, nu=1, mode="imex",
                               qdelta="lu-trick")
U2, r2 = pfasst_run(hier2, mono.u0(mesh2.vertices), 8, 2, tol_rel=1e-9, tol_abs=1e-9)
out.update(mono_U=U2, mono_its=np.array(r2.inner_iterations), mono_conv=r2.converged)
np.savez_compressed(HERE / "lutrick.npz", **out)
print({k: (v.shape if hasattr(v, "shape") and v.ndim else v) for k, v in out.items()})
