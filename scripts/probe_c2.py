"""Probe BASELINE C2 on the GPU: setup phases, STMG/SMG solves, kernel timings."""
import ctypes
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import _native as N

strategies = sys.argv[1].split(",") if len(sys.argv) > 1 else ["STMG", "SMG"]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
Nt = int(sys.argv[3]) if len(sys.argv) > 3 else 64
cfg = pd.baseline_config("C2", Nt=Nt)
t0 = time.time()
ops = pd.fd_space(cfg.spec)
s = pd.assemble_system(pd.make_tableau(3), ops, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
A = s.global_matrix()
print(f"assembly {time.time()-t0:.1f}s N={s.size} nnz={A.nnz}", flush=True)
for strat in strategies:
    t0 = time.time()
    h = pd.build_hierarchy(s, strat, 7, 3, partitions=P)
    torch.cuda.synchronize()
    print(f"{strat} hierarchy {time.time()-t0:.1f}s dims={[d.size for d in h.dims]} nnz={[m.nnz for m in h.matrices]}", flush=True)
    b = N.to_device(s.rhs())
    for rep_i in range(2):
        x = N.zeros(s.size)
        torch.cuda.synchronize(); t0 = time.time()
        x, rep = h.solve_dev(b, x, 1e-10, 1e-10, 300)
        torch.cuda.synchronize(); dt = time.time() - t0
        gdofs = s.size * 2 * 3 * rep.iterations / dt / 1e9
        print(f"  solve {strat} P={P}: {rep.iterations} cycles conv={rep.converged} {dt:.3f}s "
              f"({dt/max(rep.iterations,1)*1e3:.1f} ms/cycle, {gdofs:.3f} GDOF/s per sweep) hist={rep.residual_history[:3]}...{rep.residual_history[-1]:.3e}", flush=True)
    ilu = ctypes.c_void_p()
    N.call("pd_mg_level_precond", h._mg, 0, ctypes.byref(ilu))
    lo, up = ctypes.c_int32(), ctypes.c_int32()
    N.call("pd_ilu0_levels", ilu, ctypes.byref(lo), ctypes.byref(up))
    print(f"  fine ILU levels lo={lo.value} up={up.value}")
    ctx = N.context()
    y = N.empty(s.size)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for name, fn in (("ilu_solve", lambda: N.call("pd_ilu0_solve", ctx.handle, ilu, N.ptr(b), N.ptr(y))),
                     ("spmv", lambda: N.call("pd_csr_spmv", ctx.handle, h._dev_mats[0].handle, N.ptr(b), N.ptr(y), 0, None))):
        for _ in range(3): fn()
        ev[0].record()
        for _ in range(10): fn()
        ev[1].record(); torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 10
        nnz_row = h.matrices[0].nnz / s.size
        alg = (12 * nnz_row + (24 if name == "ilu_solve" else 20)) * s.size
        print(f"  {name}: {ms:.3f} ms  alg {alg/ms/1e6:.0f} GB/s")
    del h
    torch.cuda.empty_cache()
print("launches", N.load_library().pd_launch_count())
