"""ncu target: one ILU(0) apply on C2 SMG levels 0 and 1 (wavefront sweeps) in a
profiler range.  usage: python scripts/wf_ncu_probe.py [levels=0,1]"""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

levels = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1]
cfg = pd.baseline_config("C2")
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
print("wavefront levels:", h.wavefront, flush=True)
for l in levels:
    ilu = ctypes.c_void_p()
    N.call("pd_mg_level_precond", h._mg, l, ctypes.byref(ilu))
    n = h.dims[l].size
    b = N.to_device(torch.randn(n, dtype=torch.float64).numpy())
    y = N.empty(n)
    for _ in range(3):
        N.call("pd_ilu0_solve", h.ctx.handle, ilu, N.ptr(b), N.ptr(y))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    N.call("pd_ilu0_solve", h.ctx.handle, ilu, N.ptr(b), N.ptr(y))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("ok")
