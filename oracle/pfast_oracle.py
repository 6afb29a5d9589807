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

Round 2 adds, for the same algorithm family (csrc/pd_pfast.cu, pd_pfast_st.cu):
* the Newton linearisation J = L + γ(I⊗Mqh)diag(r'(u)) (spacetime.py:126-129,
  144-151) folded into the point blocks as a per-point weight array W, and the
  nonlinear residual (spacetime.py:131-142) for the cubic / Fisher reactions;
* `PfastStmgOracle`: the space-time V-cycle around the block-Jacobi-in-time
  smoother (level schedule of multigrid.py:148-157's STMG rule, coarsening space
  only while μ = κ·dt/h² stays above `mu_crit`), rediscretised coarse operators,
  time transfers = the coarse element's collocation polynomial evaluated at the
  two fine elements' nodes (restriction = its transpose);
* `newton_oracle`: newton_solve's loop (spacetime.py:212-258) around it.

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
        self.M, self.Mq, self.omega_s = M, np.asarray(Mq, dtype=np.float64), omega_s
        self.Ainv = np.linalg.inv(self.Ac)
        self.G = self.Ainv @ self.Mq  # point block = Ac (I + G diag(w))
        self.W = None  # (Nt, M, grid) linearisation weights γ·dt·h^d·r'(u), or None

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
        y = (np.einsum("mk,tk...->tm...", self.Ac, x)
             + np.einsum("mk,tk...->tm...", self.Ao, self.nbsum(x)))
        if self.W is not None:  # + Mq·diag(w)·x  (spacetime.py:126-129,144-151)
            y += np.einsum("mk,tk...->tm...", self.Mq, self.W * x)
        return y

    def block_solve(self, r):
        """ω_s · (point block)⁻¹ r; with weights the block is Ac(I + G·diag(w)):
        d0 = Ac⁻¹ r, then (I + G diag(w)) d = d0 per grid point."""
        if self.W is None:
            return np.einsum("mk,tk...->tm...", self.Dinv, r)
        d0 = np.einsum("mk,tk...->tm...", self.Ainv, r)
        Wm = np.moveaxis(self.W, 1, -1)  # (Nt, grid, M)
        blocks = np.eye(self.M) + self.G * Wm[..., None, :]  # G[m,k]·w_k
        d = np.linalg.solve(blocks, np.moveaxis(d0, 1, -1)[..., None])[..., 0]
        return self.omega_s * np.moveaxis(d, -1, 1)

    def jacobi(self, x, b):
        if x is None:
            return self.block_solve(b)
        return x + self.block_solve(b - self.apply(x))


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

    def set_weights(self, W0):
        """Linearisation weights of the finest spatial level (None = linear operator);
        coarser spatial levels take Pᵀ W (the full-weighting sum, so the mass factor
        h^d grows by 2^d with the rediscretised operator)."""
        W = None if W0 is None else np.asarray(W0, dtype=np.float64).reshape(self.shape())
        for lv in self.levels:
            lv.W = W
            if W is not None and lv is not self.levels[-1]:
                for ax in range(2, 2 + self.dim):
                    W = _restrict_axis(W, ax, self.periodic)

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


def reaction(kind, u):
    """r(u): spacetime.py:44-46 (cubic u³−u); the BASELINE Fisher form u²−u."""
    return u * u * u - u if kind == "cubic" else u * u - u


def reaction_deriv(kind, u):
    """r'(u): spacetime.py:48-50 (3u²−1); Fisher 2u−1."""
    return 3.0 * u * u - 1.0 if kind == "cubic" else 2.0 * u - 1.0


def lagrange_eval(nodes, t):
    """Cardinal polynomials of `nodes` at t."""
    nodes = np.asarray(nodes, dtype=np.float64)
    out = np.ones(nodes.size)
    for j in range(nodes.size):
        for k in range(nodes.size):
            if k != j:
                out[j] *= (t - nodes[k]) / (nodes[j] - nodes[k])
    return out


def time_transfer_matrices(nodes):
    """(P1, P2, E, half): the coarse element's polynomial (through its M nodes on
    (0, 1]) at the nodes of its first / second fine element (rows = fine node);
    E[m] = fine-element cardinal values at coarse node m, which lies in fine
    element half[m] (0/1) of the pair."""
    nodes = np.asarray(nodes, dtype=np.float64)
    P1 = np.array([lagrange_eval(nodes, 0.5 * t) for t in nodes])
    P2 = np.array([lagrange_eval(nodes, 0.5 + 0.5 * t) for t in nodes])
    half = np.array([0 if 2.0 * t <= 1.0 else 1 for t in nodes])
    E = np.array([lagrange_eval(nodes, 2.0 * t - h) for t, h in zip(nodes, half)])
    return P1, P2, E, half


def spatial_levels_for(n, periodic, coarsest=3):
    """Spatial V-cycle depth of a smoother on an n^d grid (pfast.max_levels)."""
    L = 1
    while True:
        if periodic:
            if n % 2 or n < 4 or n // 2 < coarsest:
                return L
            n //= 2
        else:
            if n % 2 == 0 or n < 3 or (n - 1) // 2 < coarsest:
                return L
            n = (n - 1) // 2
        L += 1


def st_schedule(dim, n, periodic, kappa, Nt, dt, mu_crit=0.3, min_nt=2, max_levels=64,
                coarsest=3):
    """Space-time level schedule: (nt, n, dt, space_coarsened_to_next) per level.
    Time is halved on every level (multigrid.py:148-157, STMG); space is halved too
    while the coarse level keeps μ = κ·dt/h² >= mu_crit (block-Jacobi in time
    smooths in space only for μ above a critical value) and the grid allows it."""
    out = []
    nl, ntl, dtl = int(n), int(Nt), float(dt)
    while True:
        h = 1.0 / nl if periodic else 1.0 / (nl + 1)
        mu = kappa * dtl / (h * h)
        last = ntl <= min_nt or ntl % 2 == 1 or len(out) + 1 >= max_levels
        if last:
            out.append((ntl, nl, dtl, False))
            return out
        if periodic:
            can = nl % 2 == 0 and nl >= 4 and nl // 2 >= coarsest
        else:
            can = nl % 2 == 1 and nl >= 3 and (nl - 1) // 2 >= coarsest
        space = bool(can and mu / 2.0 >= mu_crit)
        out.append((ntl, nl, dtl, space))
        if space:
            nl = nl // 2 if periodic else (nl - 1) // 2
        ntl //= 2
        dtl *= 2.0


class PfastStmgOracle:
    """Space-time multigrid V(ν_t, ν_t) cycle whose smoother on every level is the
    P-fast block-Jacobi-in-time sweep (ω_t damped; one spatial V-cycle per step)."""

    def __init__(self, dim, n, periodic, kappa, M, Nt, dt, Kq, Mq, l0, nodes, nu_t=1,
                 omega_t=0.5, mu_crit=0.3, min_nt=2, coarse_t_sweeps=None, nu=2,
                 coarse_sweeps=10, omega_s=0.8, max_levels=64, schedule=None):
        self.dim, self.M, self.periodic = dim, M, periodic
        self.nu_t = nu_t
        self.sched = schedule or st_schedule(dim, n, periodic, kappa, Nt, dt, mu_crit, min_nt,
                                             max_levels)
        self.P1, self.P2, self.E, self.half = time_transfer_matrices(nodes)
        self.sm = []
        for i, (ntl, nl, dtl, _) in enumerate(self.sched):
            last = i == len(self.sched) - 1
            self.sm.append(PfastOracle(dim, nl, periodic, kappa, M, ntl, dtl, Kq, Mq, l0,
                                       spatial_levels_for(nl, periodic), nu, coarse_sweeps,
                                       omega_s, 1.0 if last else omega_t))
        # the coarsest level: undamped block Jacobi, exact after nt sweeps when the
        # block solves are exact
        self.coarse_t_sweeps = coarse_t_sweeps or self.sched[-1][0] + 1

    def shape(self):
        return self.sm[0].shape()

    # -- transfers between space-time levels l and l+1
    def restrict(self, l, r):
        if self.sched[l][3]:
            for ax in range(2, 2 + self.dim):
                r = _restrict_axis(r, ax, self.periodic)
        return (np.einsum("km,tk...->tm...", self.P1, r[0::2])
                + np.einsum("km,tk...->tm...", self.P2, r[1::2]))

    def prolong(self, l, ec):
        e = np.zeros((2 * ec.shape[0],) + ec.shape[1:])
        e[0::2] = np.einsum("mk,tk...->tm...", self.P1, ec)
        e[1::2] = np.einsum("mk,tk...->tm...", self.P2, ec)
        if self.sched[l][3]:
            for ax in range(2, 2 + self.dim):
                e = _prolong_axis(e, ax, self.periodic)
        return e

    def restrict_weights(self, l, W):
        """Weights of level l+1: Pᵀ in space, then the fine elements' polynomial of
        the weights evaluated at the coarse nodes, × 2 for dt_{l+1} = 2 dt_l."""
        if self.sched[l][3]:
            for ax in range(2, 2 + self.dim):
                W = _restrict_axis(W, ax, self.periodic)
        Wc = np.zeros((W.shape[0] // 2,) + W.shape[1:])
        for m in range(self.M):
            src = W[self.half[m]::2]
            Wc[:, m] = 2.0 * np.einsum("k,tk...->t...", self.E[m], src)
        return Wc

    def set_weights(self, W0):
        W = None if W0 is None else np.asarray(W0, dtype=np.float64).reshape(self.shape())
        for l, sm in enumerate(self.sm):
            sm.set_weights(W)
            if W is not None and l + 1 < len(self.sm):
                W = self.restrict_weights(l, W)

    def cycle(self, l, b, x=None, halo_fn=None):
        """One V-cycle on level l.  halo_fn(l, x) -> the previous slab's last node at
        level l (time-slab sharding), None for the serial solve."""
        sm = self.sm[l]
        hf = (lambda xx: halo_fn(l, xx)) if halo_fn else (lambda xx: None)
        if x is None:
            x = np.zeros_like(b)
        if l == len(self.sm) - 1:
            for _ in range(self.coarse_t_sweeps):
                x = sm.sweep(x, b, hf(x))
            return x
        for _ in range(self.nu_t):
            x = sm.sweep(x, b, hf(x))
        r = sm.residual(x, b, hf(x))
        ec = self.cycle(l + 1, self.restrict(l, r), None, halo_fn)
        x = x + self.prolong(l, ec)
        for _ in range(self.nu_t):
            x = sm.sweep(x, b, hf(x))
        return x

    def solve(self, b, x0=None, tol_rel=1e-8, tol_abs=0.0, max_cycles=1000):
        """Cycles to |b − Jx| <= max(tol_abs, tol_rel·|b − Jx0|) (multigrid.py:275-305).
        Returns (x flat, cycles, converged, diverged, history)."""
        sm = self.sm[0]
        b = np.asarray(b, dtype=np.float64).reshape(self.shape())
        x = (np.zeros(self.shape()) if x0 is None
             else np.array(x0, dtype=np.float64).reshape(self.shape()))
        r = np.linalg.norm(sm.residual(x, b))
        thr = max(tol_abs, tol_rel * r)
        lowest, hist, it = r, [r], 0
        conv = div = False
        while True:
            if r <= thr:
                conv = True
                break
            if it >= max_cycles:
                div = True
                break
            x = self.cycle(0, b, x)
            it += 1
            r = np.linalg.norm(sm.residual(x, b))
            hist.append(r)
            if not np.isfinite(r):
                div = True
                break
            lowest = min(lowest, r)
            if r > 10.0 * lowest:
                div = True
                break
        return x.ravel(), it, conv, div, hist


def newton_oracle(stmg, rhs, gamma, kind, u_init=None, tol=1e-8, max_newton=50,
                  inner_tol_rel=1e-9, inner_tol_abs=1e-9, max_cycles=1000):
    """newton_solve (spacetime.py:212-258) with the P-fast STMG as the inner solver
    (mg_linear_solver semantics, multigrid.py:339-364): F(u) = L u + γ(I⊗Mqh) r(u) −
    rhs, J = L + γ(I⊗Mqh) diag(r'(u)); full steps, halved up to 8 times on residual
    growth.  Returns (u flat, dict(newton, inner, damped, converged, diverged, hist))."""
    sm = stmg.sm[0]
    shp = stmg.shape()
    dt = stmg.sched[0][2]
    mh = sm.levels[0].mh
    Mq = sm.levels[0].Mq
    rhs = np.asarray(rhs, dtype=np.float64).reshape(shp)
    u = np.zeros(shp) if u_init is None else np.array(u_init, dtype=np.float64).reshape(shp)

    def neg_F(v):  # rhs − L v − γ·dt·h^d·Mq r(v)
        stmg.sm[0].levels[0].W, keep = None, stmg.sm[0].levels[0].W
        out = sm.residual(v, rhs) - gamma * dt * mh * np.einsum(
            "mk,tk...->tm...", Mq, reaction(kind, v))
        stmg.sm[0].levels[0].W = keep
        return out

    mF = neg_F(u)
    res = float(np.linalg.norm(mF))
    thr = max(tol, tol * res)
    info = dict(newton=0, inner=[], damped=0, converged=False, diverged=False, hist=[res])
    for _ in range(max_newton):
        if res <= thr:
            info["converged"] = True
            break
        stmg.set_weights(gamma * dt * mh * reaction_deriv(kind, u))
        delta, its, conv, div, _ = stmg.solve(mF, tol_rel=inner_tol_rel, tol_abs=inner_tol_abs,
                                              max_cycles=max_cycles)
        delta = delta.reshape(shp)
        info["inner"].append(its)
        if div:
            info["diverged"] = True
            break
        step = 1.0
        for _h in range(8):
            cand = neg_F(u + step * delta)
            new = float(np.linalg.norm(cand))
            if new < res or new <= thr:
                break
            step *= 0.5
            info["damped"] += 1
        u = u + step * delta
        mF = neg_F(u)
        res = new
        info["newton"] += 1
        info["hist"].append(res)
    else:
        info["diverged"] = res > thr
    if res <= thr:
        info["converged"] = True
    return u.ravel(), info


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


class OracleStmgSlab:
    """One time slab of the sharded space-time cycle (pfast.stmg_cycle_slabs), CPU."""

    def __init__(self, stmg: PfastStmgOracle, b):
        self.o = stmg
        self.levels, self.nu_t = len(stmg.sm), stmg.nu_t
        self.coarse_t_sweeps = stmg.coarse_t_sweeps
        self.b = [np.asarray(b, dtype=np.float64).reshape(stmg.shape())] + [None] * (self.levels - 1)
        self.x = [np.zeros(stmg.shape())] + [None] * (self.levels - 1)
        self.halo = [None] * self.levels

    def last_node(self, l):
        return self.x[l][-1, -1].ravel().copy()

    def set_halo(self, l, h):
        self.halo[l] = None if h is None else np.asarray(h, dtype=np.float64)

    def sweep(self, l):
        self.x[l] = self.o.sm[l].sweep(self.x[l], self.b[l], self.halo[l])

    def restrict(self, l):
        r = self.o.sm[l].residual(self.x[l], self.b[l], self.halo[l])
        self.b[l + 1] = self.o.restrict(l, r)
        self.x[l + 1] = np.zeros_like(self.b[l + 1])

    def prolong(self, l):
        self.x[l] = self.x[l] + self.o.prolong(l, self.x[l + 1])

    def residual_norm2(self):
        r = self.o.sm[0].residual(self.x[0], self.b[0], self.halo[0])
        return float(np.sum(r * r))

    def solution(self):
        return self.x[0].ravel()
