"""P-fast profile: matrix-free block-Jacobi-in-time smoother with inner spatial
V-cycles for structured-grid space-time systems.

The reference has no matrix-free solver; this is the north_star's subsystem (2)
for the sizes the reference's CSR path cannot hold (config 5: ~420 GB of CSR per
GPU).  The operator is the reference's space-time matrix
``L = I⊗Aqh + S₋₁⊗Bqh`` (spacetime.py:77-80,117-124) for
``Kh = coef·h^d·(−Δ_h)``, ``Mh = h^d·I`` (``problems.StencilSpec``); the outer
loop keeps the reference's stopping and divergence rules
(multigrid.py:275-305) and its time blocks are linalg.py:152-189's block-Jacobi
ranges with one block per step.  Each block solve is one spatial V-cycle
(point-block damped Jacobi, full weighting, bilinear/trilinear prolongation,
rediscretised coarse operators) batched over all steps in
``csrc/pd_pfast.cu``.  Parity is against the CPU restatement
``oracle/pfast_oracle.py`` — never against the reference.
There is no CPU fallback: without the native library or a GPU every call
raises.

Round 2: `PfastStmg` wraps that smoother in the space-time V-cycle the
north_star's subsystem (2) names (time halved per level as multigrid.py:148-157's
STMG rule, space while μ = κ·dt/h² allows, rediscretised operators, polynomial
time transfers), carries the Newton linearisation of the cubic / Fisher reaction
in the point blocks (spacetime.py:126-151) and runs newton_solve's loop
(spacetime.py:212-258) around it; `solve_time_slabs_stmg` is its time-slab sharded
form (per level and sweep one send/recv of the slab-end state).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as N
from .collocation import make_tableau
from .errors import ConfigurationError, SolverError
from .problems import StencilSpec
from .report import SolveReport


def max_levels(spec: StencilSpec, coarsest: int = 3) -> int:
    """Levels until the grid cannot be halved or reaches `coarsest` points per axis."""
    L, s = 1, spec
    while True:
        try:
            c = s.coarse()
        except ConfigurationError:
            return L
        if c.n < coarsest:
            return L
        L, s = L + 1, c


def pfast_rhs(spec: StencilSpec, M: int, Nt: int, u0: np.ndarray, tableau=None) -> np.ndarray:
    """``SpaceTimeSystem.rhs`` (spacetime.py:110-114): first block l(0)⊗Mh·u0."""
    tab = tableau or make_tableau(M)
    b = np.zeros((Nt, M, spec.ndof))
    b[0] = np.outer(tab.left_values, spec.mass * np.asarray(u0, dtype=np.float64))
    return b.ravel()


REACTIONS = {"cubic": 0, "fisher": 1}


def _reaction_kind(name: str) -> int:
    try:
        return REACTIONS[name]
    except KeyError:
        raise ConfigurationError(f"unknown reaction {name!r}; expected one of {sorted(REACTIONS)}")


def _hptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _opt(t):
    return N.ptr(t) if t is not None else ctypes.c_void_p()


class PfastSolver:
    """Device P-fast solver for one structured space-time system (Nt, M, n^d):
    block-Jacobi in time, one spatial V-cycle per step and sweep."""

    def __init__(self, spec: StencilSpec, M: int, Nt: int, dt: float, levels: int | None = None,
                 nu: int = 2, coarse_sweeps: int = 10, omega_s: float = 0.8,
                 omega_t: float = 1.0, tableau=None):
        if spec.dim not in (2, 3):
            raise ConfigurationError("P-fast needs a 2D or 3D structured grid")
        self.spec, self.M, self.Nt, self.dt = spec, int(M), int(Nt), float(dt)
        self.levels = max_levels(spec) if levels is None else int(levels)
        self.nu, self.coarse_sweeps = int(nu), int(coarse_sweeps)
        self.omega_s, self.omega_t = float(omega_s), float(omega_t)
        tab = tableau or make_tableau(self.M)
        self.tableau = tab
        self.n = self.Nt * self.M * spec.ndof
        self.ctx = N.context()
        Kq = np.ascontiguousarray(tab.Kq, dtype=np.float64)
        Mq = np.ascontiguousarray(tab.Mq, dtype=np.float64)
        l0 = np.ascontiguousarray(tab.left_values, dtype=np.float64)
        h = ctypes.c_void_p()
        N.call("pd_pfast_create", self.ctx.handle, spec.dim, spec.n,
               1 if spec.bc == "periodic" else 0, spec.coef, self.M, self.Nt, self.dt,
               _hptr(Kq), _hptr(Mq), _hptr(l0), self.levels, self.nu, self.coarse_sweeps,
               self.omega_s, self.omega_t, ctypes.byref(h))
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.load_library().pd_pfast_destroy(self.handle)
        except Exception:
            pass

    def _dev(self, v, n=None):
        n = self.n if n is None else n
        t = v if N.is_tensor(v) else N.to_device(np.asarray(v, dtype=np.float64).ravel(), self.ctx)
        if t.numel() != n:
            raise ConfigurationError(f"vector has {t.numel()} entries, expected {n}")
        return t

    def _halo(self, halo):
        return None if halo is None else self._dev(halo, self.spec.ndof)

    def set_state(self, u, gamma: float = 1.0, reaction: str = "cubic") -> None:
        """Linearise around u: later residuals / sweeps / solves act on
        J = L + γ(I⊗Mqh)diag(r'(u)) (spacetime.py:144-151); u=None restores L."""
        self.ctx.sync_stream()
        if u is None:
            N.call("pd_pfast_set_state", self.handle, ctypes.c_void_p(), 0.0, 0)
            return
        N.call("pd_pfast_set_state", self.handle, N.ptr(self._dev(u)), float(gamma),
               _reaction_kind(reaction))

    def nl_residual(self, u, rhs, gamma: float = 1.0, reaction: str = "cubic", halo=None):
        """rhs − L u − γ(I⊗Mqh) r(u) = −F(u) (spacetime.py:131-142) and its 2-norm."""
        self.ctx.sync_stream()
        ud, bd, hd = self._dev(u), self._dev(rhs), self._halo(halo)
        r = N.empty(self.n, self.ctx)
        nrm = N.empty(1, self.ctx)
        N.call("pd_pfast_nl_residual", self.handle, N.ptr(ud), N.ptr(bd), N.ptr(r), _opt(hd),
               float(gamma), _reaction_kind(reaction), N.ptr(nrm))
        return r, float(np.sqrt(nrm.item()))

    def residual(self, x, b, halo=None):
        """b − L x and its 2-norm (device tensor, float)."""
        self.ctx.sync_stream()
        xd, bd, hd = self._dev(x), self._dev(b), self._halo(halo)
        r = N.empty(self.n, self.ctx)
        nrm = N.empty(1, self.ctx)
        N.call("pd_pfast_residual", self.handle, N.ptr(xd), N.ptr(bd), N.ptr(r), _opt(hd),
               N.ptr(nrm))
        return r, float(np.sqrt(nrm.item()))

    def sweep(self, b, x, halo=None) -> None:
        """One outer smoother sweep in place on the device tensor x."""
        self.ctx.sync_stream()
        bd, hd = self._dev(b), self._halo(halo)
        N.call("pd_pfast_sweep", self.handle, N.ptr(bd), N.ptr(x), _opt(hd))

    def solve(self, b, x0=None, tol_rel: float = 1e-10, tol_abs: float = 0.0,
              max_sweeps: int = 1000, halo=None):
        """Sweeps to ``|b − Lx| <= max(tol_abs, tol_rel·|b − Lx0|)``; returns (x, SolveReport).
        A non-finite residual reports ``diverged`` (multigrid.py:296-300), it does not raise.

        numpy in → numpy out, device tensors in → device tensor out."""
        self.ctx.sync_stream()
        bd, hd = self._dev(b), self._halo(halo)
        x = N.zeros(self.n, self.ctx) if x0 is None else self._dev(x0).clone()
        rep = N.SolveReportC()
        hist = np.zeros(max_sweeps + 1)
        N.call("pd_pfast_solve", self.handle, N.ptr(bd), N.ptr(x), _opt(hd), float(tol_rel),
               float(tol_abs), int(max_sweeps), ctypes.byref(rep), _hptr(hist))
        report = SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                             diverged=bool(rep.diverged),
                             residual_history=hist[:rep.hist_len].tolist())
        out = x if N.is_tensor(b) else N.to_host(x)
        return out, report


class DeviceSlab:
    """One time slab on the device for `solve_time_slabs`: the solver's Nt steps
    are this slab's steps; the previous slab's last node arrives as the halo,
    which this slab owns (a copy) and hands to the library with every call."""

    def __init__(self, solver: PfastSolver, b):
        self.s = solver
        self.b = solver._dev(b)
        self.x = N.zeros(solver.n, solver.ctx)
        S = solver.spec.ndof
        self.halo_buf = N.zeros(S, solver.ctx)
        self.halo = None
        self.norm = N.empty(1, solver.ctx)
        self.r = N.empty(solver.n, solver.ctx)
        self._last = slice(solver.n - S, solver.n)

    def last_node(self):
        return self.x[self._last]

    def set_halo(self, h):
        if h is None:
            self.halo = None
        else:
            self.halo_buf.copy_(h if N.is_tensor(h) else N.to_device(np.asarray(h)))
            self.halo = self.halo_buf

    def residual_norm2(self):
        N.call("pd_pfast_residual", self.s.handle, N.ptr(self.x), N.ptr(self.b), N.ptr(self.r),
               _opt(self.halo), N.ptr(self.norm))
        return float(self.norm.item())

    def sweep(self):
        N.call("pd_pfast_sweep", self.s.handle, N.ptr(self.b), N.ptr(self.x), _opt(self.halo))

    def solution(self):
        return self.x


def _comm(group=None, device=None):
    from .mg_sharded import Comm

    return Comm(group, device)


def _exchange(slabs, comm, last_of, set_halo_of):
    """halo of slab i = last node of slab i-1 (within the process) / of the previous
    rank's last slab (Comm.shift_next: global-rank mapping, gloo host staging)."""
    prev = None
    if comm.size > 1:
        torch = N.torch_mod()
        last = last_of(slabs[-1])
        send = last if N.is_tensor(last) else torch.from_numpy(np.ascontiguousarray(last))
        send = send.contiguous()
        recv = torch.empty_like(send) if comm.rank > 0 else None
        comm.shift_next(send if comm.rank + 1 < comm.size else None, recv)
        prev = recv
    halos = [prev] + [last_of(s) for s in slabs[:-1]]
    for s, h in zip(slabs, halos):
        set_halo_of(s, h)


def _stopping_loop(resid, step, tol_rel, tol_abs, max_it):
    """multigrid.py:275-305: stop at max(tol_abs, tol_rel·r0); diverged on a non-finite
    residual, > 10× the lowest seen, or the iteration cap."""
    r = resid()
    hist, it = [r], 0
    conv = div = False
    if not math.isfinite(r):
        return 0, False, True, hist
    thr = max(tol_abs, tol_rel * r)
    lowest = r
    while True:
        if r <= thr:
            conv = True
            break
        if it >= max_it:
            div = True
            break
        step()
        it += 1
        r = resid()
        hist.append(r)
        if not math.isfinite(r):
            div = True
            break
        lowest = min(lowest, r)
        if r > 10.0 * lowest:
            div = True
            break
    return it, conv, div, hist


def solve_time_slabs(slabs, tol_rel: float = 1e-10, tol_abs: float = 0.0,
                     max_sweeps: int = 1000, group=None):
    """P-fast over time slabs (north_star subsystem 4): `slabs` are this
    process's consecutive slabs in time order; with a torch.distributed group,
    ranks hold consecutive groups of slabs.  Per sweep the only exchange is
    each slab's last node to its successor (send/recv between ranks) plus one
    sum-allreduce of |r|^2 — block-Jacobi in time has no other coupling.
    Same stopping/divergence rules and iterates as the serial solve
    (multigrid.py:275-305).  Returns (sweeps, converged, diverged, history)."""
    last = slabs[0].last_node()
    comm = _comm(group, last.device if N.is_tensor(last) else None)

    def resid():
        _exchange(slabs, comm, lambda s: s.last_node(), lambda s, h: s.set_halo(h))
        return math.sqrt(comm.allreduce_sum(sum(s.residual_norm2() for s in slabs)))

    def step():
        for s in slabs:
            s.sweep()  # the halos set by resid() still describe the current x

    return _stopping_loop(resid, step, tol_rel, tol_abs, max_sweeps)


# ---------------------------------------------------------------- space-time multigrid
def _cardinal(nodes: np.ndarray, t: float) -> np.ndarray:
    """Lagrange cardinal values of `nodes` at t (barycentric form)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    diff = t - nodes
    hit = np.flatnonzero(diff == 0.0)
    if hit.size:
        out = np.zeros(nodes.size)
        out[hit[0]] = 1.0
        return out
    w = np.array([1.0 / np.prod(nodes[j] - np.delete(nodes, j)) for j in range(nodes.size)])
    q = w / diff
    return q / q.sum()


def time_transfer_matrices(nodes):
    """(P1, P2, E, half) for a 2:1 coarsening of the time elements: the coarse
    element's collocation polynomial (through its M nodes on (0, 1]) evaluated at the
    nodes of its first (P1) and second (P2) fine element — prolongation rows per fine
    node, restriction = transpose; E[m] = the cardinal values of the fine element
    holding coarse node m (element `half[m]` of the pair) at that node (used to
    carry the Newton weights to the coarse level)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    P1 = np.array([_cardinal(nodes, 0.5 * t) for t in nodes])
    P2 = np.array([_cardinal(nodes, 0.5 + 0.5 * t) for t in nodes])
    half = np.array([0 if 2.0 * t <= 1.0 else 1 for t in nodes], dtype=np.int32)
    E = np.array([_cardinal(nodes, 2.0 * t - h) for t, h in zip(nodes, half)])
    return P1, P2, E, half


def st_schedule(spec: StencilSpec, Nt: int, dt: float, mu_crit: float = 0.3, min_nt: int = 2,
                max_st_levels: int = 64, coarsest: int = 3):
    """Space-time levels [(nt, StencilSpec, dt, space_coarsened_to_next)]: the steps are
    halved on every level (multigrid.py:148-157, STMG); the grid is halved with them
    while the coarse level keeps μ = κ·dt/h² >= mu_crit — block-Jacobi in time damps
    the spatially oscillatory error only above a critical μ (time-only coarsening
    raises μ by 2, space-time coarsening lowers it by 2)."""
    out = []
    sp, nt, d = spec, int(Nt), float(dt)
    while True:
        mu = sp.coef * d / (sp.h * sp.h)
        if nt <= min_nt or nt % 2 or len(out) + 1 >= max_st_levels:
            out.append((nt, sp, d, False))
            return out
        try:
            c = sp.coarse()
            can = c.n >= coarsest
        except ConfigurationError:
            c, can = None, False
        space = bool(can and mu / 2.0 >= mu_crit)
        out.append((nt, sp, d, space))
        if space:
            sp = c
        nt //= 2
        d *= 2.0


class PfastStmg:
    """Space-time multigrid V(ν_t, ν_t) around the P-fast smoother, on the device.

    Level l smooths with ω_t-damped block-Jacobi in time (one spatial V-cycle per
    step); the coarsest level runs `coarse_t_sweeps` undamped sweeps (default
    nt_coarsest + 1: exact for exact block solves).  `min_nt` bounds the coarsest
    level's steps — a time-slab sharded run over G ranks equals the serial solver with
    min_nt = G·(the per-rank min_nt)."""

    def __init__(self, spec: StencilSpec, M: int, Nt: int, dt: float, nu_t: int = 1,
                 omega_t: float = 0.5, mu_crit: float = 0.3, min_nt: int = 2,
                 coarse_t_sweeps: int | None = None, nu: int = 2, coarse_sweeps: int = 10,
                 omega_s: float = 0.8, max_st_levels: int = 64, tableau=None):
        if spec.dim not in (2, 3):
            raise ConfigurationError("P-fast needs a 2D or 3D structured grid")
        self.spec, self.M, self.Nt, self.dt = spec, int(M), int(Nt), float(dt)
        tab = tableau or make_tableau(self.M)
        self.tableau = tab
        self.sched = st_schedule(spec, Nt, dt, mu_crit, min_nt, max_st_levels)
        self.nu_t = int(nu_t)
        self.coarse_t_sweeps = int(coarse_t_sweeps or self.sched[-1][0] + 1)
        self.n = self.Nt * self.M * spec.ndof
        self.ctx = N.context()
        P1, P2, E, half = time_transfer_matrices(tab.nodes)
        c = lambda a, t=np.float64: np.ascontiguousarray(a, dtype=t)
        Kq, Mq, l0 = c(tab.Kq), c(tab.Mq), c(tab.left_values)
        P1, P2, E, half = c(P1), c(P2), c(E), c(half, np.int32)
        nts = c([lv[0] for lv in self.sched], np.int64)
        ns = c([lv[1].n for lv in self.sched], np.int64)
        dts = c([lv[2] for lv in self.sched])
        sl = c([max_levels(lv[1]) for lv in self.sched], np.int32)
        h = ctypes.c_void_p()
        N.call("pd_pfast_st_create", self.ctx.handle, spec.dim, 1 if spec.bc == "periodic" else 0,
               spec.coef, self.M, _hptr(Kq), _hptr(Mq), _hptr(l0), len(self.sched), _hptr(nts),
               _hptr(ns), _hptr(dts), _hptr(sl), _hptr(P1), _hptr(P2), _hptr(E), _hptr(half),
               self.nu_t, self.coarse_t_sweeps, int(nu), int(coarse_sweeps), float(omega_s),
               float(omega_t), ctypes.byref(h))
        self.handle = h
        p0 = ctypes.c_void_p()
        N.call("pd_pfast_st_level_plan", self.handle, 0, ctypes.byref(p0))
        self._plan0 = p0  # borrowed: the level-0 smoother (residuals)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.load_library().pd_pfast_st_destroy(self.handle)
        except Exception:
            pass

    @property
    def levels(self):
        return len(self.sched)

    def level_ndof(self, l: int) -> int:
        return self.sched[l][1].ndof

    def _dev(self, v, n=None):
        n = self.n if n is None else n
        t = v if N.is_tensor(v) else N.to_device(np.asarray(v, dtype=np.float64).ravel(), self.ctx)
        if t.numel() != n:
            raise ConfigurationError(f"vector has {t.numel()} entries, expected {n}")
        return t

    def set_state(self, u, gamma: float = 1.0, reaction: str = "cubic") -> None:
        """Linearise every level around u (None: the linear operator)."""
        self.ctx.sync_stream()
        if u is None:
            N.call("pd_pfast_st_set_state", self.handle, ctypes.c_void_p(), 0.0, 0)
            return
        N.call("pd_pfast_st_set_state", self.handle, N.ptr(self._dev(u)), float(gamma),
               _reaction_kind(reaction))

    def residual(self, x, b, halo=None, out=None):
        """b − J x on level 0 and its 2-norm."""
        self.ctx.sync_stream()
        xd, bd = self._dev(x), self._dev(b)
        hd = None if halo is None else self._dev(halo, self.spec.ndof)
        r = N.empty(self.n, self.ctx) if out is None else out
        nrm = N.empty(1, self.ctx)
        N.call("pd_pfast_residual", self._plan0, N.ptr(xd), N.ptr(bd), N.ptr(r), _opt(hd),
               N.ptr(nrm))
        return r, float(np.sqrt(nrm.item()))

    def nl_residual(self, u, rhs, gamma: float = 1.0, reaction: str = "cubic", halo=None,
                    out=None):
        """rhs − L u − γ(I⊗Mqh) r(u) = −F(u) and its 2-norm."""
        self.ctx.sync_stream()
        ud, bd = self._dev(u), self._dev(rhs)
        hd = None if halo is None else self._dev(halo, self.spec.ndof)
        r = N.empty(self.n, self.ctx) if out is None else out
        nrm = N.empty(1, self.ctx)
        N.call("pd_pfast_nl_residual", self._plan0, N.ptr(ud), N.ptr(bd), N.ptr(r), _opt(hd),
               float(gamma), _reaction_kind(reaction), N.ptr(nrm))
        return r, float(np.sqrt(nrm.item()))

    def cycle(self, b, x) -> None:
        """One space-time V-cycle in place on the device tensor x."""
        self.ctx.sync_stream()
        N.call("pd_pfast_st_cycle", self.handle, N.ptr(self._dev(b)), N.ptr(x))

    def solve(self, b, x0=None, tol_rel: float = 1e-8, tol_abs: float = 0.0,
              max_cycles: int = 1000):
        """Cycles to ``|b − Jx| <= max(tol_abs, tol_rel·|b − Jx0|)`` (multigrid.py:275-305);
        returns (x, SolveReport); numpy in → numpy out, device in → device out."""
        self.ctx.sync_stream()
        bd = self._dev(b)
        x = N.zeros(self.n, self.ctx) if x0 is None else self._dev(x0).clone()
        rep = N.SolveReportC()
        hist = np.zeros(max_cycles + 1)
        N.call("pd_pfast_st_solve", self.handle, N.ptr(bd), N.ptr(x), float(tol_rel),
               float(tol_abs), int(max_cycles), ctypes.byref(rep), _hptr(hist))
        report = SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                             diverged=bool(rep.diverged),
                             residual_history=hist[:rep.hist_len].tolist())
        return (x if N.is_tensor(b) else N.to_host(x)), report

    def newton(self, rhs, gamma: float = 1.0, reaction: str = "cubic", u_init=None,
               tol: float = 1e-8, max_newton: int = 50, inner_tol_rel: float = 1e-9,
               inner_tol_abs: float = 1e-9, max_cycles: int = 1000):
        """newton_solve (spacetime.py:212-258) with this solver as the inner linear
        solver (mg_linear_solver, multigrid.py:339-364): full steps, halved up to 8
        times on residual growth, stop at ‖F‖ <= max(tol, tol·‖F(u_init)‖).
        Returns (u, SolveReport) — numpy in → numpy out, device in → device out."""
        import time as _time

        t0 = _time.perf_counter()
        self.ctx.sync_stream()
        bd = self._dev(rhs)
        u = N.zeros(self.n, self.ctx) if u_init is None else self._dev(u_init).clone()
        mF = N.empty(self.n, self.ctx)
        cand = N.empty(self.n, self.ctx)
        cres = N.empty(self.n, self.ctx)
        report = SolveReport()
        _, res = self.nl_residual(u, bd, gamma, reaction, out=mF)
        thr = max(tol, tol * res)
        report.residual_history.append(res)
        try:
            for _ in range(max_newton):
                if res <= thr:
                    report.converged = True
                    break
                self.set_state(u, gamma, reaction)
                delta, inner = self.solve(mF, tol_rel=inner_tol_rel, tol_abs=inner_tol_abs,
                                          max_cycles=max_cycles)
                report.inner_iterations.append(inner.iterations)
                if inner.diverged:
                    report.diverged = True
                    break
                step = 1.0
                for _h in range(8):
                    N.call("pd_axpy_to", self.ctx.handle, N.ptr(cand), N.ptr(u), N.ptr(delta),
                           float(step), self.n)  # cand = u + step·delta
                    _, new = self.nl_residual(cand, bd, gamma, reaction, out=cres)
                    if new < res or new <= thr:
                        break
                    step *= 0.5
                    report.damped_steps += 1
                u, cand = cand, u
                mF, cres = cres, mF
                res = new
                report.newton_iterations += 1
                report.residual_history.append(res)
            else:
                report.diverged = res > thr
        finally:
            self.set_state(None)
        if res <= thr:
            report.converged = True
        report.iterations = report.newton_iterations
        N.torch_mod().cuda.synchronize(self.ctx.torch_device)
        report.wall_time = _time.perf_counter() - t0
        return (u if N.is_tensor(rhs) else N.to_host(u)), report


class DeviceStmgSlab:
    """One time slab of the sharded space-time cycle on the device (level primitives of
    `PfastStmg`; the slab owns its per-level halo copies)."""

    def __init__(self, solver: PfastStmg, b):
        self.s = solver
        self.b = solver._dev(b)
        self.x = N.zeros(solver.n, solver.ctx)
        self.levels, self.nu_t = solver.levels, solver.nu_t
        self.coarse_t_sweeps = solver.coarse_t_sweeps
        self._hbuf = [N.zeros(solver.level_ndof(l), solver.ctx) for l in range(self.levels)]
        self._last = [N.zeros(solver.level_ndof(l), solver.ctx) for l in range(self.levels)]
        self._halo = [None] * self.levels
        self.norm = N.empty(1, solver.ctx)
        self.r = N.empty(solver.n, solver.ctx)

    def _vec(self, l):
        return (N.ptr(self.b), N.ptr(self.x)) if l == 0 else (ctypes.c_void_p(), ctypes.c_void_p())

    def last_node(self, l):
        _, x = self._vec(l)
        N.call("pd_pfast_st_level_last", self.s.handle, l, x, N.ptr(self._last[l]))
        return self._last[l]

    def set_halo(self, l, h):
        if h is None:
            self._halo[l] = None
        else:
            self._hbuf[l].copy_(h if N.is_tensor(h) else N.to_device(np.asarray(h)))
            self._halo[l] = self._hbuf[l]

    def sweep(self, l):
        b, x = self._vec(l)
        N.call("pd_pfast_st_level_sweep", self.s.handle, l, b, x, _opt(self._halo[l]))

    def restrict(self, l):
        b, x = self._vec(l)
        N.call("pd_pfast_st_level_restrict", self.s.handle, l, b, x, _opt(self._halo[l]))

    def prolong(self, l):
        _, x = self._vec(l)
        N.call("pd_pfast_st_level_prolong", self.s.handle, l, x)

    def residual_norm2(self):
        N.call("pd_pfast_residual", self.s._plan0, N.ptr(self.x), N.ptr(self.b), N.ptr(self.r),
               _opt(self._halo[0]), N.ptr(self.norm))
        return float(self.norm.item())

    def solution(self):
        return self.x


def stmg_cycle_slabs(slabs, comm) -> None:
    """One space-time V-cycle over time slabs: every sweep / residual of a level is
    preceded by one exchange of that level's slab-end states (block-Jacobi in time
    reads the predecessor's old iterate, so all slabs sweep concurrently)."""
    L = slabs[0].levels

    def exch(l):
        _exchange(slabs, comm, lambda s: s.last_node(l), lambda s, h: s.set_halo(l, h))

    def sweeps(l, count):
        for _ in range(count):
            exch(l)
            for s in slabs:
                s.sweep(l)

    def cyc(l):
        if l == L - 1:
            sweeps(l, slabs[0].coarse_t_sweeps)
            return
        sweeps(l, slabs[0].nu_t)
        exch(l)
        for s in slabs:
            s.restrict(l)
        cyc(l + 1)
        for s in slabs:
            s.prolong(l)
        sweeps(l, slabs[0].nu_t)

    cyc(0)


def solve_time_slabs_stmg(slabs, tol_rel: float = 1e-8, tol_abs: float = 0.0,
                          max_cycles: int = 1000, group=None):
    """The P-fast STMG solve over time slabs (this process's consecutive slabs; ranks
    hold consecutive groups).  Every level of every slab halves its own steps, so
    the transfers are slab-local; the only exchanges are the per-level slab-end
    states (send/recv to the successor) and one sum-allreduce of |r|² per cycle.
    Equal to the serial `PfastStmg` whose coarsest level holds the slabs'
    coarsest steps together (min_nt = n_slabs · per-slab min_nt, same
    coarse_t_sweeps).  Returns (cycles, converged, diverged, history)."""
    last = slabs[0].last_node(0)
    comm = _comm(group, last.device if N.is_tensor(last) else None)

    def resid():
        _exchange(slabs, comm, lambda s: s.last_node(0), lambda s, h: s.set_halo(0, h))
        return math.sqrt(comm.allreduce_sum(sum(s.residual_norm2() for s in slabs)))

    return _stopping_loop(resid, lambda: stmg_cycle_slabs(slabs, comm), tol_rel, tol_abs,
                          max_cycles)
