"""Space-time multigrid on the GPU (drop-in for paradiff/multigrid.py).

Host side (setup, mirroring the reference): transfer operators
(multigrid.py:37-126), level dimensions (:148-169), composite Kronecker
transfers (:172-191) and Galerkin products R A P (:224-233, scipy — the same
canonical CSR the reference builds, so coarse operators agree bitwise).
Device side (the hot path, csrc/pd_krylov.cu): per-level ILU(0) or
block-Jacobi ILU(0) factors, GMRES(nu) smoothing with device-resident control,
V(nu,nu) cycles, the coarsest dense LU and the residual-stopped solve loop.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .collocation import LagrangeBasis, radau_nodes
from .errors import ConfigurationError
from .linalg import DeviceCsr, as_csr, kron
from .report import SolveReport

STRATEGIES = ("SMG", "STMG", "SMMG")


# ---------------------------------------------------------------- transfers
def _full_weighting(n_fine: int, n_coarse: int) -> sp.csr_matrix:
    rows, cols, vals = [], [], []
    for i in range(n_coarse):
        for off, w in ((-1, 0.25), (0, 0.5), (1, 0.25)):
            f = 2 * i + off
            if 0 <= f < n_fine:
                rows.append(i)
                cols.append(f)
                vals.append(w)
    R = sp.csr_matrix((vals, (rows, cols)), shape=(n_coarse, n_fine))
    scale = np.asarray(R.sum(axis=1)).ravel()
    return as_csr(sp.diags(1.0 / scale) @ R)


def spatial_restriction(n_fine: int) -> sp.csr_matrix:
    """[1,2,1]/4 over vertex dofs, boundary rows renormalised (multigrid.py:37-56)."""
    if (n_fine - 1) % 2 != 0 or n_fine < 3:
        raise ConfigurationError(f"cannot bisect {n_fine} vertex dofs")
    return _full_weighting(n_fine, (n_fine - 1) // 2 + 1)


def spatial_prolongation(n_fine: int) -> sp.csr_matrix:
    """Linear interpolation coarse -> fine vertices (multigrid.py:59-72)."""
    if (n_fine - 1) % 2 != 0 or n_fine < 3:
        raise ConfigurationError(f"cannot bisect {n_fine} vertex dofs")
    n_coarse = (n_fine - 1) // 2 + 1
    rows, cols, vals = [], [], []
    for f in range(n_fine):
        c, odd = divmod(f, 2)
        if not odd:
            rows.append(f); cols.append(c); vals.append(1.0)
        else:
            rows += [f, f]; cols += [c, c + 1]; vals += [0.5, 0.5]
    return as_csr(sp.csr_matrix((vals, (rows, cols)), shape=(n_fine, n_coarse)))


def time_restriction(nt_fine: int) -> sp.csr_matrix:
    """[1,2,1]/4 over the element index (multigrid.py:75-90)."""
    if nt_fine % 2 != 0 or nt_fine < 2:
        raise ConfigurationError(f"cannot bisect {nt_fine} time elements")
    return _full_weighting(nt_fine, nt_fine // 2)


def time_prolongation(nt_fine: int) -> sp.csr_matrix:
    """Linear over elements, constant past the last coarse node (multigrid.py:93-108)."""
    if nt_fine % 2 != 0 or nt_fine < 2:
        raise ConfigurationError(f"cannot bisect {nt_fine} time elements")
    nt_coarse = nt_fine // 2
    rows, cols, vals = [], [], []
    for f in range(nt_fine):
        c, odd = divmod(f, 2)
        if not odd or c + 1 >= nt_coarse:
            rows.append(f); cols.append(c); vals.append(1.0)
        else:
            rows += [f, f]; cols += [c, c + 1]; vals += [0.5, 0.5]
    return as_csr(sp.csr_matrix((vals, (rows, cols)), shape=(nt_fine, nt_coarse)))


def node_prolongation(m_coarse: int, m_fine: int) -> sp.csr_matrix:
    if m_coarse > m_fine:
        raise ConfigurationError("node prolongation must not reduce the node count")
    basis = LagrangeBasis(radau_nodes(m_coarse))
    return as_csr(sp.csr_matrix(basis.matrix(radau_nodes(m_fine))))


def node_restriction(m_coarse: int, m_fine: int) -> sp.csr_matrix:
    R = sp.csr_matrix(node_prolongation(m_coarse, m_fine).T)
    scale = np.asarray(R.sum(axis=1)).ravel()
    return as_csr(sp.diags(1.0 / scale) @ R)


@dataclass(frozen=True)
class LevelDims:
    nt: int
    m: int
    nx_dofs: int

    @property
    def size(self) -> int:
        return self.nt * self.m * self.nx_dofs


@dataclass(frozen=True)
class TransferSet:
    restriction: sp.csr_matrix
    prolongation: sp.csr_matrix


def _level_dims(strategy: str, L: int, nt: int, m: int, space_sizes: list[int]) -> list[LevelDims]:
    dims = []
    for l in range(L):
        if strategy == "SMG":
            dims.append(LevelDims(nt, m, space_sizes[l]))
        elif strategy == "STMG":
            dims.append(LevelDims(nt // 2**l, m, space_sizes[l]))
        else:
            dims.append(LevelDims(nt, max(m - l, 1), space_sizes[l]))
    return dims


def _check_divisibility(strategy: str, L: int, nt: int, nx: int) -> None:
    for l in range(1, L):
        if nx % 2**l != 0:
            raise ConfigurationError(
                f"{strategy}: Nx={nx} not divisible by 2^{l} needed for level {l + 1}")
        if strategy == "STMG" and nt % 2**l != 0:
            raise ConfigurationError(
                f"STMG: Nt={nt} not divisible by 2^{l} needed for level {l + 1}")


def _build_transfers(dims: list[LevelDims], space_pairs) -> list[TransferSet]:
    out = []
    for l, (fine, coarse) in enumerate(zip(dims[:-1], dims[1:])):
        if fine.nt != coarse.nt:
            Rt, Pt = time_restriction(fine.nt), time_prolongation(fine.nt)
        else:
            Rt = Pt = sp.eye(fine.nt, format="csr")
        if fine.m != coarse.m:
            Rm, Pm = node_restriction(coarse.m, fine.m), node_prolongation(coarse.m, fine.m)
        else:
            Rm = Pm = sp.eye(fine.m, format="csr")
        Rs, Ps = space_pairs[l]
        out.append(TransferSet(kron(Rt, kron(Rm, Rs)), kron(Pt, kron(Pm, Ps))))
    return out


def lower_task_steps(nt: int, m: int, nline: int, partitions: int, whole_max: int = 384,
                     part_max: int = 192):
    """Time steps per lower-sweep wavefront task, best first.  A task spanning a
    whole block-Jacobi partition has no cross-CTA coupling at all (measured best
    on C2's 15^2/7^2 levels); otherwise tasks of k steps pay off only while the
    CTA stays small (31^2: k=2 at 186 threads; 63^2: k=2 at 378 is slower than
    k=1).  Env PD_WF_LOWER_STEPS pins it (experiments)."""
    env = os.environ.get("PD_WF_LOWER_STEPS")
    if env:
        return [int(env), 1]
    per = nt // partitions if partitions > 0 and nt % partitions == 0 else 1
    ks = [per] if per > 1 and m * per * nline <= whole_max else []
    ks += [k for k in range(per - 1, 1, -1) if per % k == 0 and m * k * nline <= part_max]
    return ks + [1]


# ---------------------------------------------------------------- hierarchy
class MultigridHierarchy:
    """Galerkin hierarchy whose smoothing, cycling and solving run on the GPU."""

    def __init__(self, fine_matrix, strategy: str, dims: list[LevelDims],
                 transfers: list[TransferSet], nu: int, partitions: int, restart: int = 30,
                 smooth_solves: int = 1, grids: list | None = None):
        if nu < 1:
            raise ConfigurationError("need at least one smoothing iteration")
        if len(transfers) != len(dims) - 1:
            raise ConfigurationError("need one transfer set per level transition")
        self.strategy = strategy
        self.dims = dims
        self.transfers = transfers
        self.nu = nu
        self.partitions = partitions
        self.restart = restart
        self.smooth_solves = smooth_solves
        self.matrices: list[sp.csr_matrix] = []
        self.ctx = N.context()
        self._mg = None
        self._dev_mats: list[DeviceCsr] = []
        self.setup_time = 0.0
        # per-level (nline, npoint) of the spatial grid planes (FD, dim >= 2):
        # enables the structured wavefront ILU sweeps on those levels
        self.grids = grids or [None] * len(dims)
        self.wavefront: list[bool] = []
        self.set_fine_matrix(fine_matrix)

    @property
    def num_levels(self) -> int:
        return len(self.dims)

    def _galerkin(self, A) -> list[sp.csr_matrix]:
        """R A P per level exactly as multigrid.py:232-233 evaluates it: (R @ A) @ P.

        The unsorted intermediates R @ A are kept: the device Galerkin refresh
        replays their stored order so later levels stay bitwise scipy's.
        """
        mats = [A]
        self._Ts = []
        for t in self.transfers:
            T = t.restriction @ mats[-1]
            self._Ts.append(T)
            mats.append(as_csr(T @ t.prolongation))
        return mats

    def set_fine_matrix(self, A) -> None:
        """Install a new fine matrix; rebuild Galerkin products and device factors."""
        t0 = time.perf_counter()
        A = as_csr(A)
        if A.shape[0] != self.dims[0].size:
            raise ConfigurationError(
                f"matrix size {A.shape[0]} does not match level 1 size {self.dims[0].size}")
        mats = self._galerkin(A)
        if getattr(self, "_system", None) is not None and hasattr(self, "_fine_installed"):
            self._system = None  # a later fine matrix is not the attached system's operator
        self._fine_installed = True
        if self._mg is not None and getattr(self, "_has_fine_op", False):
            # a new fine matrix (e.g. a Newton Jacobian) no longer matches the
            # matrix-free operator attached by build_hierarchy
            N.call("pd_mg_set_fine_operator", self._mg, None)
            self._has_fine_op = False
        if self._mg is not None and all(d.same_pattern(m) for d, m in zip(self._dev_mats, mats)):
            for d, m in zip(self._dev_mats, mats):
                d.set_values(m.data)
            N.call("pd_mg_refactor", self.ctx.handle, self._mg)
        else:
            self._destroy()
            ctx = self.ctx
            dev = [DeviceCsr(m, ctx) for m in mats]
            Rs = [DeviceCsr(t.restriction, ctx) for t in self.transfers]
            Ps = [DeviceCsr(t.prolongation, ctx) for t in self.transfers]
            L = len(mats)
            arr = (ctypes.c_void_p * L)(*[d.handle for d in dev])
            arr_r = (ctypes.c_void_p * max(L - 1, 1))(*[d.handle for d in Rs])
            arr_p = (ctypes.c_void_p * max(L - 1, 1))(*[d.handle for d in Ps])
            h = ctypes.c_void_p()
            try:
                N.call("pd_mg_create", ctx.handle, L, arr, arr_r, arr_p, int(self.nu),
                       int(self.partitions), int(self.restart), int(self.smooth_solves),
                       ctypes.byref(h))
            finally:
                for d in dev + Rs + Ps:
                    d.release()  # pd_mg_create takes ownership (frees them on failure)
            self._mg = h
            self._dev_mats = dev  # borrowed views for pattern checks/value updates
            self._enable_wavefront()
        self.matrices = mats
        self.setup_time = time.perf_counter() - t0

    def _enable_wavefront(self) -> None:
        from .linalg import set_wavefront

        # structured SpMV for the Galerkin levels of 2D grids (level 0 runs K1)
        self.grid_spmv = [False] * len(self.dims)
        for l in range(1, len(self.dims)):
            g = self.grids[l] if l < len(self.grids) else None
            if g is None or g[0] != g[1]:
                continue
            A = ctypes.c_void_p()
            N.call("pd_mg_level_matrix", self._mg, l, ctypes.byref(A))
            applied = ctypes.c_int()
            d = self.dims[l]
            N.call("pd_csr_set_grid", self.ctx.handle, A, d.nt, d.m, g[0], ctypes.byref(applied))
            self.grid_spmv[l] = bool(applied.value)
        self.wavefront = []
        for l in range(len(self.dims) - 1):
            g = self.grids[l] if l < len(self.grids) else None
            ok = False
            if g is not None:
                ilu = ctypes.c_void_p()
                N.call("pd_mg_level_precond", self._mg, l, ctypes.byref(ilu))
                d = self.dims[l]
                for k in lower_task_steps(d.nt, d.m, g[0], self.partitions):
                    ok = set_wavefront(self.ctx, ilu, d.m, g[0], g[1], d.m * k)
                    if ok:
                        break
            self.wavefront.append(ok)

    # ---- device Newton refresh (§8(f)1) --------------------------------------
    def enable_device_refresh(self) -> None:
        """Upload the R@A intermediates; later fine values are refreshed on device."""
        if self._mg is None or getattr(self, "_device_refresh", False):
            return
        Ts = [DeviceCsr(T, self.ctx, canonical=False) for T in self._Ts]
        arr = (ctypes.c_void_p * max(len(Ts), 1))(*[d.handle for d in Ts])
        N.call("pd_mg_set_galerkin_intermediates", self._mg, len(Ts), arr)
        for d in Ts:
            d.release()
        self._device_refresh = True

    def set_fine_values_dev(self, vals) -> None:
        """New fine-level values on the existing pattern (CUDA tensor, nnz doubles):
        Galerkin products and all factorizations are recomputed on device."""
        self._system = None
        if getattr(self, "_has_fine_op", False):
            N.call("pd_mg_set_fine_operator", self._mg, None)
            self._has_fine_op = False
        N.call("pd_mg_set_fine_values", self._mg, N.ptr(vals))

    def fine_pattern_matches(self, A) -> bool:
        return bool(self._dev_mats) and self._dev_mats[0].same_pattern(A)

    def attach_fine_operator(self, system) -> None:
        """Apply level 1 matrix-free (K1, bitwise the system's global CSR product).

        The CSR stays the input of the level-1 ILU(0) factorization; every
        other use of A_1 (smoother GMRES, residuals, restriction input, the
        solve's stopping test) streams only vectors.
        """
        self._system = system  # the sharded hierarchy builds its slab operators from it
        if self._mg is None:
            return
        op = system.stencil_operator_handle(self.ctx)
        N.call("pd_mg_set_fine_operator", self._mg, op)  # ownership moves to the hierarchy
        self._has_fine_op = True

    def _destroy(self):
        if self._mg is not None:
            N.load_library().pd_mg_destroy(self._mg)
            self._mg = None

    def __del__(self):
        try:
            self._destroy()
        except Exception:
            pass

    # ---- cycling --------------------------------------------------------------
    def vcycle_dev(self, b, x):
        """In-place V(nu, nu) cycle on CUDA tensors (x <- cycle(b, x))."""
        self.ctx.sync_stream()
        N.call("pd_mg_vcycle", self.ctx.handle, self._mg, N.ptr(b), N.ptr(x))
        return x

    def vcycle(self, b, x):
        """One V(nu, nu) cycle for A_1 x = b starting from x (multigrid.py:268-273)."""
        bd = N.to_device(b, self.ctx)
        xd = N.to_device(x, self.ctx).clone()
        return N.like_input(self.vcycle_dev(bd, xd), x)

    def solve_dev(self, b, x, tol_rel=1e-9, tol_abs=1e-9, max_cycles=1000):
        """Device-resident solve: b, x CUDA tensors, x updated in place."""
        self.ctx.sync_stream()
        rep = N.SolveReportC()
        hist = np.zeros(max_cycles + 2)
        t0 = time.perf_counter()
        N.call("pd_mg_solve", self.ctx.handle, self._mg, N.ptr(b), N.ptr(x), float(tol_rel),
               float(tol_abs), int(max_cycles), ctypes.byref(rep),
               hist.ctypes.data_as(ctypes.c_void_p), hist.size)
        wall = time.perf_counter() - t0
        report = SolveReport(iterations=int(rep.iterations), converged=bool(rep.converged),
                             diverged=bool(rep.diverged),
                             residual_history=[float(v) for v in hist[: rep.hist_len]],
                             wall_time=wall)
        return x, report

    def solve(self, b, x0=None, tol_rel: float = 1e-9, tol_abs: float = 1e-9,
              max_cycles: int = 1000, out=None):
        """V-cycle until ||b - Ax|| <= max(tol_abs, tol_rel*||b - Ax0||) (multigrid.py:275-305).

        numpy in -> numpy out (the reference's contract); torch tensors come back
        on their own device; `out` (e.g. a pinned host tensor) receives x in place.
        """
        bd = N.to_device(b, self.ctx)
        xd = N.zeros(bd.numel(), self.ctx) if x0 is None else N.to_device(x0, self.ctx).clone()
        x, rep = self.solve_dev(bd, xd, tol_rel, tol_abs, max_cycles)
        return N.like_input(x, b, out), rep


# ---------------------------------------------------------------- builders
def _space_levels(system, L: int):
    """Per-level spatial sizes and (Rs, Ps) pairs for the system's operator."""
    spec = getattr(system.space, "stencil", None)
    if spec is None:  # the reference's 1D FEM vertex hierarchy
        nx = system.space.mesh.Nx
        sizes = [nx // 2**l + 1 for l in range(L)]
        pairs = [(spatial_restriction(sizes[l]), spatial_prolongation(sizes[l]))
                 for l in range(L - 1)]
        return sizes, pairs, nx
    from .problems import fd_transfers

    specs = [spec]
    for _ in range(L - 1):
        specs.append(specs[-1].coarse())
    sizes = [s.ndof for s in specs]
    pairs = [fd_transfers(specs[l]) for l in range(L - 1)]
    return sizes, pairs, specs


def build_hierarchy(system, strategy: str, L: int, nu: int, partitions: int = 1,
                    restart: int = 30, smooth_solves: int = 1, matrix=None) -> MultigridHierarchy:
    """multigrid.py:308-336; FD stencil systems get full-weighting/bi-linear transfers."""
    strategy = strategy.upper()
    if strategy not in STRATEGIES:
        raise ConfigurationError(f"unknown strategy {strategy!r}; expected {STRATEGIES}")
    if L < 1:
        raise ConfigurationError("need at least one level")
    if nu < 1:
        raise ConfigurationError("need at least one smoothing iteration")
    nt, m = system.grid.Nt, system.tableau.M
    spec = getattr(system.space, "stencil", None)
    if spec is None:
        _check_divisibility(strategy, L, nt, system.space.mesh.Nx)
    elif strategy == "STMG":
        for l in range(1, L):
            if nt % 2**l:
                raise ConfigurationError(
                    f"STMG: Nt={nt} not divisible by 2^{l} needed for level {l + 1}")
    sizes, pairs, specs = _space_levels(system, L)
    dims = _level_dims(strategy, L, nt, m, sizes)
    # 2D FD grids: a time step is [node][line][point] with n points per axis
    grids = ([(sp_.n, sp_.n) if sp_.dim == 2 else None for sp_ in specs]
             if isinstance(specs, list) else None)
    if dims[-1].nx_dofs < 2 and spec is None:
        raise ConfigurationError("coarsest spatial level has fewer than 2 dofs")
    transfers = _build_transfers(dims, pairs)
    A = matrix if matrix is not None else system.global_matrix()
    h = MultigridHierarchy(A, strategy, dims, transfers, nu=nu, partitions=partitions,
                           restart=restart, smooth_solves=smooth_solves, grids=grids)
    if matrix is None:
        h.attach_fine_operator(system)
    return h


def mg_linear_solver(hierarchy: MultigridHierarchy, tol_rel=1e-9, tol_abs=1e-9, max_cycles=1000,
                     fixed_cycles: int | None = None):
    """Newton inner solver refreshing the hierarchy per Jacobian (multigrid.py:339-364)."""

    def solver(J, rhs):
        from .spacetime import DeviceJacobian

        if isinstance(J, DeviceJacobian):
            if getattr(hierarchy, "_device_refresh", False):
                hierarchy.set_fine_values_dev(J.values)  # all on device
            else:
                hierarchy.set_fine_matrix(J.host())  # first step: patterns from scipy
                hierarchy.enable_device_refresh()
        else:
            hierarchy.set_fine_matrix(J)
        if fixed_cycles is not None:
            bd = N.to_device(rhs, hierarchy.ctx)
            x = N.zeros(bd.numel(), hierarchy.ctx)
            for _ in range(fixed_cycles):
                hierarchy.vcycle_dev(bd, x)
            r = hierarchy._dev_mats[0].matvec_dev(x, mode=1, b=bd)
            res = N.norm(r, hierarchy.ctx)
            rep = SolveReport(iterations=fixed_cycles, converged=True, residual_history=[res])
            return N.like_input(x, rhs), rep
        return hierarchy.solve(rhs, tol_rel=tol_rel, tol_abs=tol_abs, max_cycles=max_cycles)

    solver.device_jacobian = True  # newton_solve may hand over device-side Jacobians
    return solver
