"""P-fast STMG probes on the device: cycle counts vs Nt, and config 5 (cubic Newton) at size.

    python scripts/pfast_stmg_probe.py flat  [n] [nu_t] # linear solves, Nt = 32..256 on n^3
    python scripts/pfast_stmg_probe.py c5    [n] [Nt]   # Newton + STMG on the C5 problem
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2006_12883_b200.pfast import PfastSolver, PfastStmg
from paper_2006_12883_b200.problems import StencilSpec

mode = sys.argv[1] if len(sys.argv) > 1 else "flat"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda")


def rhs_for(spec, M, Nt, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    u0 = torch.rand(spec.ndof, dtype=torch.float64, device=dev, generator=g) * 2 - 1
    from paper_2006_12883_b200.collocation import make_tableau
    l0 = torch.tensor(make_tableau(M).left_values, dtype=torch.float64, device=dev)
    b = torch.zeros(Nt, M, spec.ndof, dtype=torch.float64, device=dev)
    b[0] = l0[:, None] * (spec.mass * u0)[None, :]
    return b.reshape(-1)


if mode == "flat":
    # keep mu = kappa dt / h^2 of config 5 (6.55) on the n^3 grid
    spec = StencilSpec(3, n, "periodic", 0.1)
    dt = 6.5536 * spec.h ** 2 / 0.1
    nu_t = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    for Nt in (32, 64, 128, 256):
        s = PfastStmg(spec, 3, Nt, dt, nu_t=nu_t)
        b = rhs_for(spec, 3, Nt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = s.solve(b, tol_rel=1e-8)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        line = f"Nt={Nt} levels={[(a, sp.n) for a, sp, _, _ in s.sched]} cycles={rep.iterations} conv={rep.converged} {t:.2f}s"
        del s
        if Nt <= 64 and nu_t == 1:
            bj = PfastSolver(spec, 3, Nt, dt)
            _, r2 = bj.solve(b, tol_rel=1e-8, max_sweeps=400)
            line += f" | block-Jacobi alone: {r2.iterations} sweeps"
            del bj
        print(line, flush=True)
else:
    Nt = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    spec = StencilSpec(3, n, "periodic", 0.1)
    s = PfastStmg(spec, 3, Nt, 1e-3)
    print("levels", [(a, sp.n, d, f) for a, sp, d, f in s.sched], flush=True)
    b = rhs_for(spec, 3, Nt)
    print("mem after setup GB", torch.cuda.mem_get_info()[0] / 1e9, flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = s.newton(b, 1.0, "cubic", tol=1e-8)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"C5 {n}^3 x {Nt}: newton={rep.newton_iterations} inner={rep.inner_iterations} "
          f"damped={rep.damped_steps} conv={rep.converged} hist={rep.residual_history} {t:.2f}s",
          flush=True)
    print("mem free GB", torch.cuda.mem_get_info()[0] / 1e9)
    # one linear cycle timing
    x = torch.zeros_like(b)
    s.cycle(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        s.cycle(b, x)
    e1.record()
    torch.cuda.synchronize()
    print(f"linear cycle {e0.elapsed_time(e1) / 3:.1f} ms")
