"""SDC sweeps, FAS corrections and the windowed PFASST driver on the GPU
(drop-in for paradiff/pfasst.py).

The reference runs one Python thread per time step of a window (pfasst.py:
369-587).  Here the P steps of a window are P "workers" whose states live in
one device array per level, U[P][M][S]; fine sweeps, FAS corrections,
transfers and residuals are single batched kernels over all workers, and the
coarsest level's serial forward chain (pfasst.py:441-455) runs worker by
worker on the device.  The message schedule is the reference's exactly: the
fine initial value of worker w is worker w-1's fine terminal from the
PREVIOUS iteration; the coarsest initial value is worker w-1's coarse
terminal from the CURRENT iteration; no fine post-sweep after interpolation;
residuals use the U0 received at the start of the iteration.  One host sync
per iteration reads the P residual norms (the convergence/divergence test).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .collocation import CollocationTableau, LagrangeBasis, make_tableau
from .errors import ConfigurationError, SolverError
from .fem1d import SpaceMesh, SpaceOperators, assemble_space
from .linalg import DeviceCsr, as_csr
from .multigrid import spatial_prolongation, spatial_restriction
from .report import SolveReport
from .spacetime import TimeGrid, reaction

MODES = ("implicit", "imex")
_REACTION = {"cubic": 1, "fisher": 2}
_ERR_TEXT = {1: "non-finite values entered an SDC sweep", 2: "zero pivot in a node operator",
             4: "node solve failed", 8: "node solve did not converge within the refinement budget"}


def _vp(t, offset_elems: int = 0):
    return ctypes.c_void_p(t.data_ptr() + 8 * offset_elems) if t is not None else ctypes.c_void_p()


def _host(mat) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(mat, dtype=np.float64))


@dataclass
class SweeperState:
    """Node values (M, ndof), step initial value (ndof,) and FAS term (M, ndof)."""

    U: object
    U0: object
    tau: object = None

    def copy(self) -> "SweeperState":
        return SweeperState(self.U.copy(), self.U0.copy(),
                            None if self.tau is None else self.tau.copy())

    @property
    def terminal(self):
        return self.U[-1]


def spread_state(u0, M: int) -> SweeperState:
    u0 = np.asarray(u0, dtype=np.float64)
    return SweeperState(np.tile(u0, (M, 1)), u0.copy())


class SdcLevel:
    """Operators and device node solvers for SDC sweeps on one level (pfasst.py:60-200)."""

    def __init__(self, tableau: CollocationTableau, space: SpaceOperators, dt: float,
                 gamma: float, mode: str = "implicit", reaction_kind: str = "cubic"):
        if mode not in MODES:
            raise ConfigurationError(f"unknown sweep mode {mode!r}; expected {MODES}")
        self.tableau = tableau
        self.space = space
        self.dt = float(dt)
        self.gamma = float(gamma)
        self.mode = mode
        self.reaction_kind = reaction_kind
        self.mh = space.lumped_diagonal
        self.Kh = as_csr(space.Kh)
        self._dev = None
        self._cap = 0
        self.ctx = None

    @property
    def M(self) -> int:
        return self.tableau.M

    @property
    def ndof(self) -> int:
        return self.mh.size

    # ---- device level -------------------------------------------------------
    def device(self, workers: int):
        if self._dev is not None and workers <= self._cap:
            return self._dev
        self._release()
        self.ctx = N.context()
        Kd = DeviceCsr(self.Kh, self.ctx)
        mh = _host(self.mh)
        T = self.tableau
        phi, mu, sdim, sn, ss = self._spectral()
        h = ctypes.c_void_p()
        N.call("pd_sdc_level_create", self.ctx.handle, Kd.handle,
               mh.ctypes.data_as(ctypes.c_void_p), self.M,
               _host(T.Q).ctypes.data_as(ctypes.c_void_p),
               _host(T.QDeltaImplicit).ctypes.data_as(ctypes.c_void_p),
               _host(T.QDeltaExplicit).ctypes.data_as(ctypes.c_void_p), self.dt, self.gamma,
               _REACTION[self.reaction_kind], 1 if self.mode == "imex" else 0, int(workers),
               phi.ctypes.data_as(ctypes.c_void_p) if phi is not None else None,
               mu.ctypes.data_as(ctypes.c_void_p) if mu is not None else None, sdim, sn, ss,
               ctypes.byref(h))
        self._dev, self._cap = h, workers
        return h

    def _spectral(self):
        """Eigen-description of a structured FD Kh (enables the spectral node solver).

        Kh = s * sum_axes T (problems.stencil_matrix) with the 1D second
        difference T = Phi diag(mu) Phi^T (orthonormal, numpy eigh — host M x M
        scale setup).  The device applies (mh + q Kh)^{-1} exactly up to
        rounding and keeps the reference's refinement/residual test on the CSR.
        """
        spec = getattr(self.space, "stencil", None)
        if spec is None or spec.dim < 2:
            return None, None, 0, 0, 0.0
        from .problems import _second_difference

        Tm = _second_difference(spec.n, spec.bc).toarray()
        mu, phi = np.linalg.eigh(Tm)
        s = spec.coef * spec.h ** spec.dim / spec.h ** 2
        return (np.ascontiguousarray(phi, dtype=np.float64),
                np.ascontiguousarray(mu, dtype=np.float64), spec.dim, spec.n, float(s))

    def _release(self):
        if self._dev is not None:
            N.load_library().pd_sdc_level_destroy(self._dev)
            self._dev = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass

    def check_errors(self):
        """Raise the device-side failure of this level, if any; the exception's `worker`
        is the lowest failing worker of the batch (the window driver counts an
        iteration only for the workers before it, pfasst.py:471-507)."""
        e = (ctypes.c_int * 2)()
        N.call("pd_sdc_errors", self._dev, e)
        if e[0]:
            bit = next(b for b in (1, 2, 4, 8) if e[0] & b)
            err = SolverError(_ERR_TEXT[bit])
            err.worker = int(e[1])
            raise err

    # ---- batched device primitives (W workers) --------------------------------
    def sweep_dev(self, U, U0, tau, W: int, w_off: int = 0):
        """In-place sweep of workers [w_off, w_off+W) of the device arrays."""
        M, S = self.M, self.ndof
        dev = self._dev if (self._dev is not None and self._cap >= W) else self.device(W)
        N.call("pd_sdc_sweep", dev, _vp(U, w_off * M * S), _vp(U0, w_off * S),
               _vp(tau, w_off * M * S) if tau is not None else ctypes.c_void_p(), W)

    def residual_dev(self, U, U0, tau, W: int, out):
        N.call("pd_sdc_residual", self.device(W), _vp(U), _vp(U0),
               _vp(tau) if tau is not None else ctypes.c_void_p(), W, _vp(out))
        return out

    def coll_op_dev(self, U, out, W: int):
        N.call("pd_sdc_coll_op", self.device(W), _vp(U), _vp(out), W)
        return out

    # ---- reference-shaped API (numpy in/out; device inside) ---------------------
    def _state_dev(self, state: SweeperState):
        ctx = N.context()
        U = N.to_device(np.asarray(state.U, dtype=np.float64).ravel(), ctx).clone()
        U0 = N.to_device(np.asarray(state.U0, dtype=np.float64).ravel(), ctx)
        tau = (N.to_device(np.asarray(state.tau, dtype=np.float64).ravel(), ctx)
               if state.tau is not None else None)
        return U, U0, tau

    def sweep(self, state: SweeperState) -> SweeperState:
        U, U0, tau = self._state_dev(state)
        self.sweep_dev(U, U0, tau, 1)
        self.check_errors()
        return SweeperState(U.cpu().numpy().reshape(self.M, self.ndof), state.U0, state.tau)

    def residual_norm(self, state: SweeperState) -> float:
        U, U0, tau = self._state_dev(state)
        out = N.empty(1)
        self.residual_dev(U, U0, tau, 1, out)
        return float(out.cpu().item())

    def collocation_residual(self, state: SweeperState) -> np.ndarray:
        """U - U0 - dt*Q F(U) - tau (pfasst.py:107-112); C(U) on device, U0/tau removed after."""
        U, U0, tau = self._state_dev(state)
        out = N.empty(self.M * self.ndof)
        self.coll_op_dev(U, out, 1)
        res = out.cpu().numpy().reshape(self.M, self.ndof) - np.asarray(state.U0)
        return res - state.tau if state.tau is not None else res

    # host helpers kept for API parity (inspection only; not on the solver path)
    def f_diffusion(self, U):
        return -(self.Kh @ np.asarray(U).T).T / self.mh

    def f_reaction(self, U):
        if self.gamma == 0.0:
            return np.zeros_like(U)
        return -self.gamma * reaction(np.asarray(U), self.reaction_kind)

    def f_total(self, U):
        return self.f_diffusion(U) + self.f_reaction(U)


def sdc_sweep_implicit(state, tableau, dt, space, gamma=0.0) -> SweeperState:
    return SdcLevel(tableau, space, dt, gamma, "implicit").sweep(state)


def sdc_sweep_imex(state, tableau, dt, space, gamma=0.0) -> SweeperState:
    return SdcLevel(tableau, space, dt, gamma, "imex").sweep(state)


def sdc_solve_step(u0, level: SdcLevel, tol_rel: float = 1e-9, tol_abs: float = 1e-9,
                   max_sweeps: int = 1000):
    """Sweep one step until the collocation residual meets the tolerance (pfasst.py:223-249)."""
    M, S = level.M, level.ndof
    u0 = np.asarray(u0, dtype=np.float64)
    ctx = N.context()
    u0d = N.to_device(u0, ctx)
    U = N.empty(M * S, ctx)
    U0 = N.empty(S, ctx)
    N.call("pd_spread", ctx.handle, _vp(u0d), _vp(U), _vp(U0), 1, M, S)
    res_d = N.empty(1, ctx)
    res = float(level.residual_dev(U, U0, None, 1, res_d).cpu().item())
    report = SolveReport(residual_history=[res])
    threshold = max(tol_abs, tol_rel * res)
    lowest = res
    while res > threshold:
        if report.iterations >= max_sweeps:
            report.diverged = True
            break
        level.sweep_dev(U, U0, None, 1)
        res = float(level.residual_dev(U, U0, None, 1, res_d).cpu().item())
        level.check_errors()
        report.iterations += 1
        report.residual_history.append(res)
        if not np.isfinite(res) or res > 10.0 * lowest:
            report.diverged = True
            break
        lowest = min(lowest, res)
    report.converged = res <= threshold
    return SweeperState(U.cpu().numpy().reshape(M, S), u0.copy()), report


# ---------------------------------------------------------------- transfers
class LevelTransfer:
    """Space (CSR) and node (M_c x M_f / M_f x M_c) transfers (pfasst.py:253-270)."""

    def __init__(self, space_restrict, space_prolong, node_restrict, node_prolong):
        self.space_restrict = as_csr(space_restrict)
        self.space_prolong = as_csr(space_prolong)
        self.node_restrict = _host(node_restrict)
        self.node_prolong = _host(node_prolong)
        self._dev = None

    def _devs(self):
        if self._dev is None:
            ctx = N.context()
            self._dev = (DeviceCsr(self.space_restrict, ctx), DeviceCsr(self.space_prolong, ctx))
        return self._dev

    @property
    def Sf(self):
        return self.space_restrict.shape[1]

    @property
    def Sc(self):
        return self.space_restrict.shape[0]

    def restrict_dev(self, Uf, out, tmp, W: int, Mf: int, Mc: int):
        """out[W][Mc][Sc] = Rn (Rs Uf) ; tmp holds W*Mf*Sc doubles."""
        ctx = N.context()
        Rs, _ = self._devs()
        N.call("pd_csr_spmm", ctx.handle, Rs.handle, _vp(Uf), self.Sf, _vp(tmp), self.Sc,
               W * Mf, 0)
        N.call("pd_node_mix", ctx.handle, _vp(tmp), _vp(out), W, Mf, Mc, self.Sc,
               self.node_restrict.ctypes.data_as(ctypes.c_void_p), 0)
        return out

    def prolong_add_dev(self, Vc, Uf, tmp, W: int, Mc: int, Mf: int):
        """Uf[W][Mf][Sf] += Pn (Ps Vc) ; tmp holds W*Mc*Sf doubles."""
        ctx = N.context()
        _, Ps = self._devs()
        N.call("pd_csr_spmm", ctx.handle, Ps.handle, _vp(Vc), self.Sc, _vp(tmp), self.Sf,
               W * Mc, 0)
        N.call("pd_node_mix", ctx.handle, _vp(tmp), _vp(Uf), W, Mc, Mf, self.Sf,
               self.node_prolong.ctypes.data_as(ctypes.c_void_p), 1)
        return Uf

    def restrict_u0_dev(self, u0, out):
        ctx = N.context()
        Rs, _ = self._devs()
        N.call("pd_csr_spmm", ctx.handle, Rs.handle, _vp(u0), self.Sf, _vp(out), self.Sc, 1, 0)
        return out

    # numpy API of the reference
    def restrict_nodes(self, U):
        U = np.asarray(U, dtype=np.float64)
        Mf, Mc = U.shape[0], self.node_restrict.shape[0]
        ctx = N.context()
        Ud = N.to_device(U.ravel(), ctx)
        out, tmp = N.empty(Mc * self.Sc, ctx), N.empty(Mf * self.Sc, ctx)
        return self.restrict_dev(Ud, out, tmp, 1, Mf, Mc).cpu().numpy().reshape(Mc, self.Sc)

    def prolong_nodes(self, U):
        U = np.asarray(U, dtype=np.float64)
        Mc, Mf = U.shape[0], self.node_prolong.shape[0]
        ctx = N.context()
        Ud = N.to_device(U.ravel(), ctx)
        out, tmp = N.zeros(Mf * self.Sf, ctx), N.empty(Mc * self.Sf, ctx)
        return self.prolong_add_dev(Ud, out, tmp, 1, Mc, Mf).cpu().numpy().reshape(Mf, self.Sf)

    def restrict_u0(self, u0):
        ctx = N.context()
        out = N.empty(self.Sc, ctx)
        return self.restrict_u0_dev(N.to_device(u0, ctx), out).cpu().numpy()


def _node_eval_restriction(fine_nodes, coarse_nodes) -> np.ndarray:
    """Fine nodal polynomial evaluated at the coarse nodes (pfasst.py:272-280)."""
    return LagrangeBasis(fine_nodes).matrix(coarse_nodes)


def fas_correction_dev(fine: SdcLevel, coarse: SdcLevel, tr: LevelTransfer, Uf, tau_f, W: int,
                       tau_out, RU_out, scratch):
    """tau = C_c(R U) - R C_f(U) (+ R tau_f) for W workers (pfasst.py:283-303)."""
    ctx = N.context()
    Mf, Mc, Sf, Sc = fine.M, coarse.M, fine.ndof, coarse.ndof
    tmp_fc = scratch["tmp_fc"]    # W*Mf*Sc
    cf = scratch["cf"]            # W*Mf*Sf
    rcf = scratch["rcf"]          # W*Mc*Sc
    tr.restrict_dev(Uf, RU_out, tmp_fc, W, Mf, Mc)
    coarse.coll_op_dev(RU_out, tau_out, W)                 # C_c(RU)
    fine.coll_op_dev(Uf, cf, W)                            # C_f(U)
    tr.restrict_dev(cf, rcf, tmp_fc, W, Mf, Mc)            # R C_f(U)
    n = W * Mc * Sc
    N.call("pd_sub", ctx.handle, _vp(tau_out), _vp(tau_out), _vp(rcf), n)
    if tau_f is not None:
        tr.restrict_dev(tau_f, rcf, tmp_fc, W, Mf, Mc)
        N.call("pd_axpy_to", ctx.handle, _vp(tau_out), _vp(tau_out), _vp(rcf), 1.0, n)
    return tau_out


def fas_correction(fine_level: SdcLevel, coarse_level: SdcLevel, transfer: LevelTransfer,
                   fine_state: SweeperState) -> np.ndarray:
    ctx = N.context()
    Mf, Mc, Sf, Sc = fine_level.M, coarse_level.M, fine_level.ndof, coarse_level.ndof
    Uf = N.to_device(np.asarray(fine_state.U).ravel(), ctx)
    tau_f = (N.to_device(np.asarray(fine_state.tau).ravel(), ctx)
             if fine_state.tau is not None else None)
    scratch = {"tmp_fc": N.empty(Mf * Sc, ctx), "cf": N.empty(Mf * Sf, ctx),
               "rcf": N.empty(Mc * Sc, ctx)}
    tau, RU = N.empty(Mc * Sc, ctx), N.empty(Mc * Sc, ctx)
    fas_correction_dev(fine_level, coarse_level, transfer, Uf, tau_f, 1, tau, RU, scratch)
    return tau.cpu().numpy().reshape(Mc, Sc)


class PfasstHierarchy:
    def __init__(self, levels: list[SdcLevel], transfers: list[LevelTransfer], nu: int):
        self.levels = levels
        self.transfers = transfers
        self.nu = nu

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    @property
    def fine(self) -> SdcLevel:
        return self.levels[0]


def build_pfasst_hierarchy(M: int, mesh: SpaceMesh, grid: TimeGrid, gamma: float, L: int,
                           nu: int = 1, mode: str = "implicit", qdelta: str = "implicit-euler",
                           space: SpaceOperators | None = None, M_coarse: int = 1,
                           reaction_kind: str = "cubic") -> PfasstHierarchy:
    """pfasst.py:323-365 (fine M; coarser levels M_coarse nodes, bisected meshes).

    With ``space`` carrying an FD stencil (problems.fd_space) the levels are
    rediscretised FD grids with full-weighting / bilinear transfers — the
    BASELINE configs (coarse M=2 or 3).
    """
    if L < 1:
        raise ConfigurationError("need at least one level")
    spec = getattr(space, "stencil", None) if space is not None else None
    tab_fine = make_tableau(M, qdelta)
    tab_coarse = make_tableau(M_coarse, qdelta)
    levels, transfers = [], []
    if spec is None:
        if mesh.Nx % 2 ** (L - 1) != 0:
            raise ConfigurationError(f"Nx={mesh.Nx} not divisible by 2^{L - 1} for {L} levels")
        for l in range(L):
            sp_l = assemble_space(SpaceMesh(mesh.Nx // 2**l, mesh.X))
            levels.append(SdcLevel(tab_fine if l == 0 else tab_coarse, sp_l, grid.dt, gamma, mode,
                                   reaction_kind))
        pairs = [(spatial_restriction(levels[l].ndof), spatial_prolongation(levels[l].ndof))
                 for l in range(L - 1)]
    else:
        from .problems import fd_space, fd_transfers

        specs = [spec]
        for _ in range(L - 1):
            specs.append(specs[-1].coarse())
        for l, s in enumerate(specs):
            levels.append(SdcLevel(tab_fine if l == 0 else tab_coarse, fd_space(s), grid.dt,
                                   gamma, mode, reaction_kind))
        pairs = [fd_transfers(specs[l]) for l in range(L - 1)]
    for l in range(L - 1):
        mf, mc = levels[l].M, levels[l + 1].M
        if mf != mc:
            nr = _node_eval_restriction(levels[l].tableau.nodes, levels[l + 1].tableau.nodes)
            npr = _node_eval_restriction(levels[l + 1].tableau.nodes, levels[l].tableau.nodes)
        else:
            nr = npr = np.eye(mf)
        transfers.append(LevelTransfer(pairs[l][0], pairs[l][1], nr, npr))
    return PfasstHierarchy(levels, transfers, nu)


# ---------------------------------------------------------------- the windowed driver
class GpuPfasstEngine:
    """Device state of this rank's workers of a window + the PFASST steps on them.

    Implements the engine interface of timeslab.run_windows; all arithmetic is
    native (csrc/pd_sdc.cu), the host only sequences launches.
    """

    def __init__(self, hier: PfasstHierarchy, u_init_dev, Nt: int, P: int, rank: int = 0,
                 size: int = 1, out=None):
        from .timeslab import worker_range

        self.ctx = ctx = N.context()
        self.h = hier
        self.P = P
        self.w0, self.w1 = worker_range(P, rank, size)
        self.W = W = self.w1 - self.w0
        self.rank, self.size = rank, size
        lv = hier.levels
        self.L = L = len(lv)
        for l in lv:
            l.device(W)
        self.U = [N.empty(W * l.M * l.ndof, ctx) for l in lv]
        self.U0 = [N.empty(W * l.ndof, ctx) for l in lv]
        self.tau = [None] + [N.empty(W * l.M * l.ndof, ctx) for l in lv[1:]]
        self.chain = [N.empty(l.ndof, ctx) for l in lv]
        self.nrecv = max(L - 1, 1)
        self.msgs = [N.empty(W * lv[l].ndof, ctx) for l in range(self.nrecv)]
        self.halo_in = [N.empty(lv[l].ndof, ctx) for l in range(self.nrecv)]
        self.halo_out = [N.empty(lv[l].ndof, ctx) for l in range(self.nrecv)]
        self.c_in = N.empty(lv[-1].ndof, ctx)
        self.c_out = N.empty(lv[-1].ndof, ctx)
        self.res = N.empty(W, ctx)
        self.u_start = u_init_dev.clone()
        self.fine_term = N.empty(lv[0].ndof, ctx)
        self.scratch = []
        for l in range(L - 1):
            f, c = lv[l], lv[l + 1]
            self.scratch.append({
                "tmp_fc": N.empty(W * f.M * c.ndof, ctx), "cf": N.empty(W * f.M * f.ndof, ctx),
                "rcf": N.empty(W * c.M * c.ndof, ctx), "RU": N.empty(W * c.M * c.ndof, ctx),
                "diff": N.empty(W * c.M * c.ndof, ctx),
                "tmp_cf": N.empty(W * c.M * f.ndof, ctx)})
        S, M = lv[0].ndof, lv[0].M
        self.out = out if out is not None else N.empty(Nt * M * S, ctx)
        self._r0 = 0.0

    num_levels = property(lambda self: self.L)
    local_workers = property(lambda self: self.W)

    def _c(self, name, *args):
        N.call(name, self.ctx.handle, *args)

    def setup_window(self, start):
        lv, trs = self.h.levels, self.h.transfers
        self._c("pd_scale", _vp(self.chain[0]), _vp(self.u_start), 1.0, lv[0].ndof)
        for l in range(self.L - 1):
            trs[l].restrict_u0_dev(self.chain[l], self.chain[l + 1])
        for l, lev in enumerate(lv):
            self._c("pd_spread", _vp(self.chain[l]), _vp(self.U[l]), _vp(self.U0[l]), self.W,
                    lev.M, lev.ndof)
        lv[0].residual_dev(self.U[0], self.U0[0], None, self.W, self.res)
        r = self.res.cpu().numpy()
        self._r0 = float(r[0])  # every worker starts from the same spread state
        return r

    def window_r0(self):
        return self._r0

    def halo_buffers(self):
        return self.halo_in

    def halo_out_buffers(self):
        return self.halo_out

    def receive(self, halo):
        """U0 of levels < L-1 from the predecessor's previous-iteration terminal."""
        lv = self.h.levels
        for l in range(self.nrecv):
            n = lv[l].ndof
            if self.W > 1:
                self._c("pd_scale", _vp(self.U0[l], n), _vp(self.msgs[l]), 1.0, (self.W - 1) * n)
            if halo is not None:
                self._c("pd_scale", _vp(self.U0[l]), _vp(halo[l]), 1.0, n)

    def fine_sweeps(self):
        for _ in range(self.h.nu):
            self.h.fine.sweep_dev(self.U[0], self.U0[0], None, self.W)

    def coarse_down(self):
        lv, trs, nu = self.h.levels, self.h.transfers, self.h.nu
        for l in range(1, self.L):
            fas_correction_dev(lv[l - 1], lv[l], trs[l - 1], self.U[l - 1], self.tau[l - 1],
                               self.W, self.tau[l], self.U[l], self.scratch[l - 1])
            if l < self.L - 1:
                for _ in range(nu):
                    lv[l].sweep_dev(self.U[l], self.U0[l], self.tau[l], self.W)

    def coarse_start_buffer(self):
        return self.c_in

    def load_coarse_start(self, buf):
        self._c("pd_scale", _vp(buf), _vp(self.chain[-1]), 1.0, self.h.levels[-1].ndof)

    def coarse_chain(self, u0c):
        c = self.h.levels[-1]
        Mc, Sc = c.M, c.ndof
        U, U0, tau = self.U[-1], self.U0[-1], self.tau[-1]
        N.call("pd_sdc_chain", c.device(self.W), _vp(U), _vp(U0), _vp(tau), self.W, _vp(u0c),
               int(self.h.nu))
        self._c("pd_terminal", _vp(U, (self.W - 1) * Mc * Sc), _vp(self.c_out), 1, Mc, Sc)
        return self.c_out

    def coarse_last_buffer(self):
        return self.c_out

    def coarse_up(self):
        lv, trs, nu = self.h.levels, self.h.transfers, self.h.nu
        for l in range(self.L - 2, -1, -1):
            sc = self.scratch[l]
            f, cl = lv[l], lv[l + 1]
            trs[l].restrict_dev(self.U[l], sc["RU"], sc["tmp_fc"], self.W, f.M, cl.M)
            self._c("pd_sub", _vp(sc["diff"]), _vp(self.U[l + 1]), _vp(sc["RU"]),
                    self.W * cl.M * cl.ndof)
            trs[l].prolong_add_dev(sc["diff"], self.U[l], sc["tmp_cf"], self.W, cl.M, f.M)
            if 0 < l < self.L - 1:
                for _ in range(nu):
                    lv[l].sweep_dev(self.U[l], self.U0[l], self.tau[l], self.W)

    def publish(self):
        lv = self.h.levels
        for l in range(self.nrecv):
            M, S = lv[l].M, lv[l].ndof
            self._c("pd_terminal", _vp(self.U[l]), _vp(self.msgs[l]), self.W, M, S)
            self._c("pd_scale", _vp(self.halo_out[l]), _vp(self.msgs[l], (self.W - 1) * S), 1.0, S)
        lv[0].residual_dev(self.U[0], self.U0[0], None, self.W, self.res)
        r = self.res.cpu().numpy()
        first = None
        for lev in lv:  # read (and clear) every level's flags; report the lowest worker
            try:
                lev.check_errors()
            except SolverError as e:
                if first is None or getattr(e, "worker", 0) < getattr(first, "worker", 0):
                    first = e
        if first is not None:
            first.worker = self.w0 + max(getattr(first, "worker", 0), 0)
            raise first
        return r

    def store_window(self, start):
        M, S = self.h.fine.M, self.h.fine.ndof
        self._c("pd_scale", _vp(self.out, (start + self.w0) * M * S), _vp(self.U[0]), 1.0,
                self.W * M * S)

    def last_fine_terminal(self):
        M, S = self.h.fine.M, self.h.fine.ndof
        self._c("pd_terminal", _vp(self.U[0], (self.W - 1) * M * S), _vp(self.fine_term), 1, M, S)
        return self.fine_term

    def set_window_start(self, t):
        self._c("pd_scale", _vp(self.u_start), _vp(t), 1.0, self.h.fine.ndof)


def pfasst_run_dev(hierarchy: PfasstHierarchy, u_init_dev, Nt: int, P: int, tol_rel=1e-9,
                   tol_abs=1e-9, max_iters=1000, comm=None):
    """Device-resident driver: returns (flat CUDA tensor (Nt, M, S), SolveReport).

    With ``comm`` (timeslab.TorchComm over NCCL) the window's workers are
    sharded over the ranks; each rank's tensor then holds its own steps only.
    """
    from .timeslab import LocalComm, run_windows

    comm = comm or LocalComm()
    eng = GpuPfasstEngine(hierarchy, u_init_dev, Nt, P, comm.rank, comm.size)
    report = run_windows(eng, comm, Nt, P, tol_rel, tol_abs, max_iters)
    return eng.out, report


def pfasst_run_distributed(hierarchy: PfasstHierarchy, u_init, Nt: int, workers: int,
                           tol_rel: float = 1e-9, tol_abs: float = 1e-9, max_iters: int = 1000,
                           group=None, gather: bool = True):
    """pfasst_run with each window's workers sharded over the ranks of ``group``.

    One process per GPU (torch.distributed, NCCL).  Returns the full flat
    solution on every rank when ``gather`` (an all_gather of the slabs).
    """
    import torch
    import torch.distributed as dist

    from .timeslab import TorchComm

    comm = TorchComm(group)
    ctx = N.context()
    out, report = pfasst_run_dev(hierarchy, N.to_device(u_init, ctx), Nt, workers, tol_rel,
                                 tol_abs, max_iters, comm)
    if not gather:
        return out, report
    M, S = hierarchy.fine.M, hierarchy.fine.ndof
    W = workers // comm.size
    parts = [torch.empty_like(out) for _ in range(comm.size)]
    dist.all_gather(parts, out, group=group)
    full = out.clone().view(Nt // workers, workers, M * S)
    for r, part in enumerate(parts):
        pv = part.view(Nt // workers, workers, M * S)
        full[:, r * W:(r + 1) * W] = pv[:, r * W:(r + 1) * W]
    return full.reshape(-1).cpu().numpy(), report


def pfasst_run(hierarchy: PfasstHierarchy, u_init, Nt: int, workers: int, tol_rel: float = 1e-9,
               tol_abs: float = 1e-9, max_iters: int = 1000):
    """Pipelined PFASST over all steps in windows of ``workers`` (pfasst.py:509-587)."""
    if workers < 1 or workers > Nt:
        raise ConfigurationError(f"worker count must be in [1, Nt={Nt}], got {workers}")
    if Nt % workers != 0:
        raise ConfigurationError(f"worker count {workers} must divide Nt={Nt}")
    S = hierarchy.fine.ndof
    u_init = np.asarray(u_init, dtype=np.float64)
    if u_init.size != S:
        raise ConfigurationError("initial state does not match the fine mesh")
    ctx = N.context()
    out, report = pfasst_run_dev(hierarchy, N.to_device(u_init, ctx), Nt, workers, tol_rel,
                                 tol_abs, max_iters)
    return out.cpu().numpy(), report
