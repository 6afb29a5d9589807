"""ncu target for the round's top kernels on C2 (inside one profiler range):
fine-level ILU(0) apply (wavefront lower+upper), 127^2-level ILU apply,
127^2 Galerkin structured SpMV, K1 structured operator."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

cfg = pd.baseline_config("C2")
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                       0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
print("wavefront", h.wavefront, "grid spmv", h.grid_spmv, flush=True)
vecs = {l: N.to_device(torch.randn(h.dims[l].size, dtype=torch.float64).numpy()) for l in (0, 1)}
outs = {l: N.empty(h.dims[l].size) for l in (0, 1)}
ilus = {}
for l in (0, 1):
    ilus[l] = ctypes.c_void_p()
    N.call("pd_mg_level_precond", h._mg, l, ctypes.byref(ilus[l]))


def run():
    for l in (0, 1):
        N.call("pd_ilu0_solve", h.ctx.handle, ilus[l], N.ptr(vecs[l]), N.ptr(outs[l]))
    h._dev_mats[1].matvec_dev(vecs[1], out=outs[1])
    s.apply_dev(vecs[0], outs[0])


for _ in range(3):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
