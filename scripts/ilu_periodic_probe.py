"""Time the ILU(0) setup / refactor / apply on a periodic 2D space-time level (C3 128^2 x 32)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
Nt = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = pd.baseline_config("C3", n=n, Nt=Nt)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       cfg.gamma, cfg.u0(), reaction_kind="fisher")
A = pd.linalg.as_csr(s.global_matrix())
print("rows", A.shape[0], "nnz", A.nnz, flush=True)


def tick(label, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"{label}: {t - t0:.2f} s", flush=True)
    return t


t = time.perf_counter()
ilu = pd.Ilu0(A)
t = tick("Ilu0 create (pattern analysis + factor)", t)
lv = (ctypes.c_int * 2)()
N.call("pd_ilu0_levels", ilu.handle, lv)
print("dependency levels lower/upper:", lv[0], lv[1], flush=True)
N.call("pd_ilu0_refactor", ilu.ctx.handle, ilu.handle)
t = tick("refactor", t)
b = N.to_device(np.random.default_rng(0).standard_normal(A.shape[0]))
y = ilu.solve_dev(b)
t = tick("first apply", t)
for _ in range(5):
    ilu.solve_dev(b, out=y)
t = tick("5 applies", t)
