"""Small ILU(0)/SpMV probe for ncu captures: C2 grid with Nt=8, fine-level kernels."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

cfg = pd.baseline_config("C2", Nt=int(sys.argv[1]) if len(sys.argv) > 1 else 8)
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
ilu = ctypes.c_void_p()
N.call("pd_mg_level_precond", h._mg, 0, ctypes.byref(ilu))
b = N.to_device(s.rhs() + 1.0)
y = N.empty(s.size)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(2):
    N.call("pd_ilu0_solve", h.ctx.handle, ilu, N.ptr(b), N.ptr(y))
    N.call("pd_csr_spmv", h.ctx.handle, h._dev_mats[0].handle, N.ptr(b), N.ptr(y), 0, None)
    s.apply_dev(b, y)  # K1 matrix-free operator
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", float(y.abs().max()))
