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
from .errors import ConfigurationError
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
