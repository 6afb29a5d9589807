"""CPU restatement of the P-fast smoother — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this
module, as the checker.  P-fast has no reference counterpart (SURVEY §7.1,
§8(c)): it restates the same algorithm as csrc/pd_pfast.cu in plain numpy so
the device path can be checked against it (tolerance 1e-12 relative L2 and
equal sweep counts; summation orders differ).  The pieces it follows from the
reference: the space-time operator L = I⊗Aqh + S₋₁⊗Bqh (spacetime.py:77-80,
117-124), the right-hand side (spacetime.py:110-114), the outer stopping and
divergence rules (multigrid.py:275-305) and one time block per step
(linalg.py:152-189).  Parity is therefore "P-fast CPU restatement vs P-fast
GPU", never vs the reference.

Arrays are (Nt, M, n, ..., n) views of the flat (Nt, M, n^d) C-order vectors.
"""

from __future__ import annotations

import numpy as np


class PfastLevel:
    def __init__(self, dim, n, periodic, kappa, M, dt, Kq, Mq, omega_s):
        self.dim, self.n, self.periodic = dim, n, periodic
        h = 1.0 / n if periodic else 1.0 / (n + 1)
        mh = h ** dim
        ks = kappa * h ** (dim - 2)
        self.mh = mh
        self.Ac = Kq * mh + dt * Mq * (ks * 2.0 * dim)
        self.Ao = -dt * Mq * ks
        self.Dinv = omega_s * np.linalg.inv(self.Ac)

    def nbsum(self, x):
        """Σ of the 2·dim grid neighbours (zero outside a Dirichlet grid)."""
        s = np.zeros_like(x)
        for ax in range(2, 2 + self.dim):
            if self.periodic:
                s += np.roll(x, 1, axis=ax) + np.roll(x, -1, axis=ax)
            else:
                lo = [slice(None)] * x.ndim
                hi = [slice(None)] * x.ndim
                lo[ax], hi[ax] = slice(1, None), slice(None, -1)
                s[tuple(lo)] += x[tuple(hi)]
                s[tuple(hi)] += x[tuple(lo)]
        return s

    def apply(self, x):
        return (np.einsum("mk,tk...->tm...", self.Ac, x)
                + np.einsum("mk,tk...->tm...", self.Ao, self.nbsum(x)))

    def jacobi(self, x, b):
        if x is None:
            return np.einsum("mk,tk...->tm...", self.Dinv, b)
        return x + np.einsum("mk,tk...->tm...", self.Dinv, b - self.apply(x))


def _restrict_axis(f, ax, periodic):
    nf = f.shape[ax]
    take = lambda i: np.take(f, i, axis=ax)
    if periodic:
        c = np.arange(nf // 2)
        return 0.5 * take((2 * c - 1) % nf) + take(2 * c) + 0.5 * take((2 * c + 1) % nf)
    c = np.arange((nf - 1) // 2)
    return 0.5 * take(2 * c) + take(2 * c + 1) + 0.5 * take(2 * c + 2)


def _prolong_axis(cg, ax, periodic):
    nc = cg.shape[ax]
    nf = 2 * nc if periodic else 2 * nc + 1
    shape = list(cg.shape)
    shape[ax] = nf
    out = np.zeros(shape)
    sl = lambda i: tuple(slice(None) if a != ax else i for a in range(cg.ndim))
    if periodic:
        out[sl(slice(0, nf, 2))] = cg
        out[sl(slice(1, nf, 2))] = 0.5 * (cg + np.roll(cg, -1, axis=ax))
    else:
        out[sl(slice(1, nf, 2))] = cg
        out[sl(slice(0, nf, 2))] = 0.0
        out[sl(slice(2, nf - 1, 2))] += 0.5 * (np.take(cg, np.arange(nc - 1), axis=ax)
                                            + np.take(cg, np.arange(1, nc), axis=ax))
        out[sl(slice(0, 1))] = 0.5 * np.take(cg, [0], axis=ax)
        out[sl(slice(nf - 1, nf))] = 0.5 * np.take(cg, [nc - 1], axis=ax)
    return out


class PfastOracle:
    def __init__(self, dim, n, periodic, kappa, M, Nt, dt, Kq, Mq, l0, levels, nu=2,
                 coarse_sweeps=10, omega_s=0.8, omega_t=1.0):
        self.dim, self.M, self.Nt, self.periodic = dim, M, Nt, periodic
        self.nu, self.coarse_sweeps, self.omega_t = nu, coarse_sweeps, omega_t
        self.levels = []
        nl = n
        for l in range(levels):
            if l > 0:
                nl = nl // 2 if periodic else (nl - 1) // 2
            self.levels.append(PfastLevel(dim, nl, periodic, kappa, M, dt, np.asarray(Kq),
                                          np.asarray(Mq), omega_s))
        self.n0 = n
        self.cprev = -np.asarray(l0) * self.levels[0].mh

    def shape(self):
        return (self.Nt, self.M) + (self.n0,) * self.dim

    def residual(self, x, b, halo=None):
        """b − L x (spacetime.py:117-124 structure); `halo` = the previous time
        slab's last node when the steps are one rank's slab."""
        L0 = self.levels[0]
        r = b - L0.apply(x)
        cp = self.cprev.reshape((1, self.M) + (1,) * self.dim)
        r[1:] -= cp * x[:-1, -1:]
        if halo is not None:
            r[:1] -= cp * np.asarray(halo).reshape((1, 1) + (self.n0,) * self.dim)
        return r

    def vcycle(self, l, b):
        Lv = self.levels[l]
        last = l == len(self.levels) - 1
        e = None
        for _ in range(self.coarse_sweeps if last else self.nu):
            e = Lv.jacobi(e, b)
        if last:
            return e
        r = b - Lv.apply(e)
        bc = r
        for ax in range(2, 2 + self.dim):
            bc = _restrict_axis(bc, ax, self.periodic)
        ec = self.vcycle(l + 1, bc)
        for ax in range(2, 2 + self.dim):
            ec = _prolong_axis(ec, ax, self.periodic)
        e = e + ec
        for _ in range(self.nu):
            e = Lv.jacobi(e, b)
        return e

    def sweep(self, x, b, halo=None):
        return x + self.omega_t * self.vcycle(0, self.residual(x, b, halo))

    def solve(self, b, x0=None, tol_rel=1e-10, tol_abs=0.0, max_sweeps=1000):
        """Returns (x flat, sweeps, converged, diverged, history) (multigrid.py:275-305)."""
        b = np.asarray(b, dtype=np.float64).reshape(self.shape())
        x = np.zeros(self.shape()) if x0 is None else np.array(x0, dtype=np.float64).reshape(self.shape())
        r = np.linalg.norm(self.residual(x, b))
        thr = max(tol_abs, tol_rel * r)
        lowest, hist, it = r, [r], 0
        conv = div = False
        while True:
            if r <= thr:
                conv = True
                break
            if it >= max_sweeps:
                div = True
                break
            x = self.sweep(x, b)
            it += 1
            r = np.linalg.norm(self.residual(x, b))
            hist.append(r)
            lowest = min(lowest, r)
            if r > 10.0 * lowest:
                div = True
                break
        return x.ravel(), it, conv, div, hist


class OracleSlab:
    """One rank's time slab for pfast.solve_time_slabs (CPU, numpy)."""

    def __init__(self, orc: PfastOracle, b):
        self.o = orc
        self.b = np.asarray(b, dtype=np.float64).reshape(orc.shape())
        self.x = np.zeros(orc.shape())
        self.halo = None

    def last_node(self):
        return self.x[-1, -1].ravel().copy()

    def set_halo(self, h):
        self.halo = None if h is None else np.asarray(h, dtype=np.float64)

    def residual_norm2(self):
        r = self.o.residual(self.x, self.b, self.halo)
        return float(np.sum(r * r))

    def sweep(self):
        self.x = self.o.sweep(self.x, self.b, self.halo)

    def solution(self):
        return self.x.ravel()
