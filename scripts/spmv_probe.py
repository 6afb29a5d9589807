"""Time the CSR SpMV on every C2 SMG Galerkin level (and the fine CSR)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

cfg = pd.baseline_config("C2")
s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for l, dm in enumerate(h._dev_mats):
    A = h.matrices[l]
    n = A.shape[0]
    x = N.to_device(np.random.default_rng(l).standard_normal(A.shape[1]))
    y = N.empty(n)
    f = lambda: N.call("pd_csr_spmv", h.ctx.handle, dm.handle, N.ptr(x), N.ptr(y), 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize(); ev[0].record()
    for _ in range(20): f()
    ev[1].record(); torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 20
    byt = 12 * A.nnz + 20 * n
    ref = A @ x.cpu().numpy()
    same = np.array_equal(ref, y.cpu().numpy())
    print(f"level {l}: n={n} nnz={A.nnz} {ms:.4f} ms {byt/ms/1e6:.0f} GB/s alg bitwise={same}", flush=True)
