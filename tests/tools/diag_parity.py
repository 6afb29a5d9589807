"""Print GPU-vs-reference parity numbers for the golden MG / GMRES cases."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import scipy.sparse as sp

import paper_2006_12883_b200 as pd
from oracle import paradiff_oracle as O
from pd_util import per_node_rel, rel_l2

G = ROOT / "tests" / "golden"
g = dict(np.load(G / "linalg.npz"))
A = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]))
x, rep = pd.gmres(A, g["b"], precond=pd.Ilu0(A), tol_rel=1e-10, tol_abs=1e-12, restart=7, max_it=200)
print("gmres its", rep.iterations, int(g["gm_its"]), "rel", rel_l2(x, g["gm_x"]))
print(" hist gpu", np.array(rep.residual_history)[:5], "\n hist ref", g["gm_hist"][:5])
n = 200
A2 = sp.diags([np.full(n - 1, -1.0), np.full(n, 4.0), np.full(n - 1, -1.0)], [-1, 0, 1], format="csr")
rng = np.random.default_rng(3)
b = rng.standard_normal(n); x0 = rng.standard_normal(n)
for M in (None, "ilu"):
    xg, rg = pd.gmres(A2, b, precond=pd.Ilu0(A2) if M else None, x0=x0, tol_rel=1e-12, tol_abs=0.0, restart=6, max_it=100)
    xo, ro = O.gmres(A2, b, M=O.OIlu0(A2) if M else None, x0=x0, tol_rel=1e-12, tol_abs=0.0, restart=6, max_it=100)
    print("gmres x0", M, rg.iterations, ro.iterations, rel_l2(xg, xo), rg.residual_history[-3:], ro.residual_history[-3:])

g = dict(np.load(G / "mg_fem1d.npz"))
prob = pd.heat_problem(); mesh = pd.SpaceMesh(64, 1.0)
s = pd.assemble_system(pd.make_tableau(3), pd.assemble_space(mesh), pd.TimeGrid(16, 1.0), 0.0, prob.u0(mesh.vertices))
for strat in ("SMG", "STMG", "SMMG"):
    for P in (1, 4):
        h = pd.build_hierarchy(s, strat, 3, 3, partitions=P)
        key = f"{strat}_P{P}"
        v1 = h.vcycle(s.rhs(), np.zeros(s.size))
        xx, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10)
        print(key, rep.iterations, int(g[key + "_its"]), "v1", rel_l2(v1, g[key + "_v1"]), "x glob", rel_l2(xx, g[key + "_x"]),
              "node", per_node_rel(xx, g[key + "_x"], (16, 3, 65)))
        print("   hist", rep.residual_history[-2:], g[key + "_hist"][-2:])
