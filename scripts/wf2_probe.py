"""A/B of the ILU(0) sweep executors on every SMG level of BASELINE C2 (GPU).

    python scripts/wf2_probe.py [--n 255] [--levels 7]

For each level: the template-structured skewed wavefront (pd_wf2.cu, kind 2) and
the pattern-table wavefront (pd_wavefront.cu, kind 1) on the same block-Jacobi
factor; prints ms per ILU apply (CUDA events, 20 applies after warm-up) and checks
the two outputs are bitwise equal.
"""

import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_12883_b200 as pd  # noqa: E402
from paper_2006_12883_b200 import _native as N  # noqa: E402


def time_apply(pre, b, reps=20):
    y = N.empty(b.numel())
    for _ in range(3):
        pre.solve_dev(b, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pre.solve_dev(b, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, y.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=255)
    ap.add_argument("--levels", type=int, default=7, help="hierarchy depth (coarsest dense)")
    ap.add_argument("--time-levels", type=int, default=6, help="levels timed")
    ap.add_argument("--nt", type=int, default=64)
    a = ap.parse_args()
    cfg = pd.baseline_config("C2", n=a.n, Nt=a.nt)
    t0 = time.perf_counter()
    s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                           0.0, cfg.u0())
    h = pd.build_hierarchy(s, "SMG", a.levels, 3, partitions=8)
    print(f"setup {time.perf_counter() - t0:.1f}s", flush=True)
    spec = cfg.spec
    rng = np.random.default_rng(0)
    total = {1: 0.0, 2: 0.0, 3: 0.0}
    for l, A in enumerate(h.matrices[:-1]):
        if l >= a.time_levels:
            break
        A = pd.linalg.as_csr(A)
        b = N.to_device(rng.standard_normal(A.shape[0]))
        res = {}
        for flag in ("1", "0"):
            os.environ["PD_WF2"] = flag
            pre = pd.BlockJacobiPrecond(A, 8)
            t1 = time.perf_counter()
            ok = pre.set_wavefront(3, spec.n, spec.n)
            tp = time.perf_counter() - t1
            kind = pre.sweep_kind()
            ms, y = time_apply(pre, b)
            res[1 if kind == 1 else 2] = (ms, y)
            nnz_row = A.nnz / A.shape[0]
            gbs = (12 * nnz_row + 24) * A.shape[0] / ms / 1e6
            print(f"level {l} n={spec.n}^2 rows={A.shape[0]} nnz/row={nnz_row:.1f} kind={kind} "
                  f"ok={ok} plan {tp:.1f}s: {ms:.3f} ms/apply ({gbs:.0f} GB/s alg)", flush=True)
            del pre
        if 1 in res and 2 in res:
            same = np.array_equal(res[1][1], res[2][1])
            print(f"   bitwise equal: {same}; speed-up {res[1][0] / res[2][0]:.2f}x", flush=True)
            total[1] += res[1][0]
            total[2] += res[2][0]  # template (kinds 2/3)
        spec = spec.coarse()
    os.environ.pop("PD_WF2", None)
    print(f"sum over levels: pattern-table {total[1]:.3f} ms, template {total[2]:.3f} ms")


if __name__ == "__main__":
    main()
