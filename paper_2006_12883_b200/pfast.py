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
"""

from __future__ import annotations

import ctypes

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


class PfastSolver:
    """Device P-fast solver for one structured space-time system (Nt, M, n^d)."""

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
               Kq.ctypes.data_as(ctypes.c_void_p), Mq.ctypes.data_as(ctypes.c_void_p),
               l0.ctypes.data_as(ctypes.c_void_p), self.levels, self.nu, self.coarse_sweeps,
               self.omega_s, self.omega_t, ctypes.byref(h))
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.load_library().pd_pfast_destroy(self.handle)
        except Exception:
            pass

    def _dev(self, v):
        t = v if N.is_tensor(v) else N.to_device(np.asarray(v, dtype=np.float64).ravel(), self.ctx)
        if t.numel() != self.n:
            raise ConfigurationError(f"vector has {t.numel()} entries, expected {self.n}")
        return t

    def residual(self, x, b):
        """b − L x and its 2-norm (device tensor, float)."""
        self.ctx.sync_stream()
        xd, bd = self._dev(x), self._dev(b)
        r = N.empty(self.n, self.ctx)
        nrm = N.empty(1, self.ctx)
        N.call("pd_pfast_residual", self.handle, N.ptr(xd), N.ptr(bd), N.ptr(r), N.ptr(nrm))
        return r, float(np.sqrt(nrm.item()))

    def sweep(self, b, x) -> None:
        """One outer smoother sweep in place on the device tensor x."""
        self.ctx.sync_stream()
        bd = self._dev(b)
        N.call("pd_pfast_sweep", self.handle, N.ptr(bd), N.ptr(x))

    def solve(self, b, x0=None, tol_rel: float = 1e-10, tol_abs: float = 0.0,
              max_sweeps: int = 1000):
        """Sweeps to ``|b − Lx| <= max(tol_abs, tol_rel·|b − Lx0|)``; returns (x, SolveReport).

        numpy in → numpy out, device tensors in → device tensor out."""
        self.ctx.sync_stream()
        bd = self._dev(b)
        x = N.zeros(self.n, self.ctx) if x0 is None else self._dev(x0).clone()
        rep = N.SolveReportC()
        hist = np.zeros(max_sweeps + 1)
        N.call("pd_pfast_solve", self.handle, N.ptr(bd), N.ptr(x), float(tol_rel), float(tol_abs),
               int(max_sweeps), ctypes.byref(rep), hist.ctypes.data_as(ctypes.c_void_p))
        report = SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                             diverged=bool(rep.diverged),
                             residual_history=hist[:rep.hist_len].tolist())
        out = x if N.is_tensor(b) else N.to_host(x)
        return out, report


class DeviceSlab:
    """One time slab on the device for `solve_time_slabs`: the solver's Nt steps
    are this slab's steps; the previous slab's last node arrives as the halo."""

    def __init__(self, solver: PfastSolver, b):
        self.s = solver
        self.b = solver._dev(b)
        self.x = N.zeros(solver.n, solver.ctx)
        S = solver.spec.ndof
        self.halo_buf = N.zeros(S, solver.ctx)
        self.norm = N.empty(1, solver.ctx)
        self.r = N.empty(solver.n, solver.ctx)
        self._last = slice(solver.n - S, solver.n)

    def last_node(self):
        return self.x[self._last]

    def set_halo(self, h):
        if h is None:
            N.call("pd_pfast_set_halo", self.s.handle, ctypes.c_void_p())
        else:
            self.halo_buf.copy_(h if N.is_tensor(h) else N.to_device(np.asarray(h)))
            N.call("pd_pfast_set_halo", self.s.handle, N.ptr(self.halo_buf))

    def residual_norm2(self):
        N.call("pd_pfast_residual", self.s.handle, N.ptr(self.x), N.ptr(self.b), N.ptr(self.r),
               N.ptr(self.norm))
        return float(self.norm.item())

    def sweep(self):
        N.call("pd_pfast_sweep", self.s.handle, N.ptr(self.b), N.ptr(self.x))

    def solution(self):
        return self.x


def solve_time_slabs(slabs, tol_rel: float = 1e-10, tol_abs: float = 0.0,
                     max_sweeps: int = 1000, group=None):
    """P-fast over time slabs (north_star subsystem 4): `slabs` are this
    process's consecutive slabs in time order; with a torch.distributed group,
    ranks hold consecutive groups of slabs.  Per sweep the only exchange is
    each slab's last node to its successor (send/recv between ranks) plus one
    sum-allreduce of |r|^2 — block-Jacobi in time has no other coupling.
    Same stopping/divergence rules and iterates as the serial solve
    (multigrid.py:275-305).  Returns (sweeps, converged, diverged, history)."""
    import math

    torch = N.torch_mod()
    dist = None
    if group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
        dist = torch.distributed
    rank = dist.get_rank(group) if dist else 0
    world = dist.get_world_size(group) if dist else 1

    def exchange():
        # halo of slab i = last node of slab i-1 (within the process) / of the
        # previous rank's last slab
        prev = None
        if dist and world > 1:
            last = slabs[-1].last_node()
            send = last if N.is_tensor(last) else torch.from_numpy(np.ascontiguousarray(last))
            recv = torch.empty_like(send)
            reqs = []
            if rank + 1 < world:
                reqs.append(dist.isend(send.contiguous(), rank + 1, group=group))
            if rank > 0:
                reqs.append(dist.irecv(recv, rank - 1, group=group))
            for q in reqs:
                q.wait()
            prev = recv if rank > 0 else None
        halos = [prev] + [s.last_node() for s in slabs[:-1]]
        for s, h in zip(slabs, halos):
            s.set_halo(h)

    def resid():
        exchange()
        n2 = sum(s.residual_norm2() for s in slabs)
        if dist and world > 1:
            t = torch.tensor([n2], dtype=torch.float64,
                             device=slabs[0].last_node().device if N.is_tensor(slabs[0].last_node())
                             else "cpu")
            dist.all_reduce(t, group=group)
            n2 = float(t.item())
        return math.sqrt(n2)

    r = resid()
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
        for s in slabs:
            s.sweep()  # the halos set by resid() still describe the current x
        it += 1
        r = resid()
        hist.append(r)
        if not math.isfinite(r):
            raise SolverError("non-finite residual in P-fast sweep")
        lowest = min(lowest, r)
        if r > 10.0 * lowest:
            div = True
            break
    return it, conv, div, hist
