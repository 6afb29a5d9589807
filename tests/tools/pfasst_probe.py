"""PFASST timing on the GPU vs the CPU oracle for a few sizes."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import pfasst as PF
from oracle import paradiff_oracle as O

def oracle_levels(spec, M, Mc, dt):
    spc = spec.coarse(); f, c = pd.fd_space(spec), pd.fd_space(spc)
    tf, tc = O.tableau(M), O.tableau(Mc)
    lv = [O.OSdcLevel(tf, f.Kh, f.lumped_diagonal, dt, 0.0), O.OSdcLevel(tc, c.Kh, c.lumped_diagonal, dt, 0.0)]
    Rs, Ps = pd.fd_transfers(spec)
    return lv, [O.OTransfer(Rs, Ps, O.node_eval(tf.nodes, tc.nodes), O.node_eval(tc.nodes, tf.nodes))]

for name, n, Nt, P in (("C1", 127, 16, 16), ("C1-1023", 1023, 64, 64), ("C2-2D63", 63, 16, 16)):
    base = "C2" if "2D" in name else "C1"
    cfg = pd.baseline_config(base, n=n, Nt=Nt)
    ops = pd.fd_space(cfg.spec)
    hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, L=2, nu=1, space=ops, M_coarse=cfg.M_coarse)
    PF.pfasst_run(hier, cfg.u0(), cfg.Nt, P, 1e-10, 1e-10)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, P, 1e-10, 1e-10)
    torch.cuda.synchronize(); tg = time.perf_counter() - t0
    sweeps = sum(rep.inner_iterations) * P
    dofs = cfg.M * cfg.spec.ndof
    lv, trs = oracle_levels(cfg.spec, cfg.M, cfg.M_coarse, cfg.dt)
    t0 = time.perf_counter(); xo, ro = O.pfasst(lv, trs, 1, cfg.u0(), cfg.Nt, P, 1e-10, 1e-10); tc = time.perf_counter() - t0
    print(f"{name}: S={cfg.spec.ndof} Nt={Nt} P={P} its={rep.iterations}/{ro.iterations} GPU {tg:.3f}s ({dofs*sweeps/tg/1e9:.4f} GDOF/s per sweep)  CPU-oracle {tc:.2f}s  speedup {tc/tg:.1f}x", flush=True)
