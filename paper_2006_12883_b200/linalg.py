"""Device-backed sparse kernels (drop-in for paradiff/linalg.py).

Same names and arguments as the reference module; numpy in -> numpy out (and
CUDA tensors in -> CUDA tensors out).  The work runs in the native library:
CSR SpMV, level-scheduled ILU(0) factor/solve, block-Jacobi masking, dense
LU and a device-resident GMRES (see csrc/).  `kron`/`as_csr` stay host-side
setup helpers exactly as in the reference (linalg.py:47-60).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .errors import ConfigurationError
from .report import SolveReport

THREAD_CAP_ENV = "PARADIFF_MAX_THREADS"
GROWTH_FACTOR = 10.0
_SIZE_LIMIT = 2**31 - 1


def thread_cap(default: int = 16) -> int:
    """Kept for API compatibility (linalg.py:27-34); the GPU path ignores it."""
    raw = os.environ.get(THREAD_CAP_ENV, "")
    try:
        cap = int(raw) if raw else default
    except ValueError:
        cap = default
    return max(1, min(cap, os.cpu_count() or 1))


def as_csr(A) -> sp.csr_matrix:
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    return A


def kron(A, B) -> sp.csr_matrix:
    A, B = sp.coo_matrix(A), sp.coo_matrix(B)
    if A.shape[0] * B.shape[0] > _SIZE_LIMIT or A.shape[1] * B.shape[1] > _SIZE_LIMIT:
        raise ConfigurationError("Kronecker product dimensions overflow index range")
    return as_csr(sp.kron(A, B, format="csr"))


class DeviceCsr:
    """A CSR matrix resident in HBM (int64 row pointers, int32 columns, fp64)."""

    def __init__(self, A, ctx: N.Context | None = None, canonical: bool = True):
        self.ctx = ctx or N.context()
        # canonical=False keeps the stored entry order (e.g. scipy's unsorted
        # R @ A intermediate, whose order the device Galerkin replays)
        A = as_csr(A) if canonical else sp.csr_matrix(A)
        self.shape = A.shape
        self.nnz = int(A.nnz)
        rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.indices, dtype=np.int32)
        va = np.ascontiguousarray(A.data, dtype=np.float64)
        h = ctypes.c_void_p()
        N.call("pd_csr_create", self.ctx.handle, A.shape[0], A.shape[1], self.nnz,
               rp.ctypes.data_as(ctypes.c_void_p), ci.ctypes.data_as(ctypes.c_void_p),
               va.ctypes.data_as(ctypes.c_void_p), 0, ctypes.byref(h))
        self.handle = h
        self._owned = True
        self._indptr, self._indices = rp, ci

    @classmethod
    def borrowed(cls, handle, shape, nnz, ctx):
        self = cls.__new__(cls)
        self.ctx, self.handle, self.shape, self.nnz, self._owned = ctx, handle, shape, nnz, False
        self._indptr = self._indices = None
        return self

    def same_pattern(self, A: sp.csr_matrix) -> bool:
        return (self._indptr is not None and A.nnz == self.nnz and A.shape == self.shape
                and np.array_equal(A.indptr, self._indptr) and np.array_equal(A.indices,
                                                                             self._indices))

    def set_values(self, data) -> None:
        d = np.ascontiguousarray(data, dtype=np.float64)
        N.call("pd_csr_set_values", self.ctx.handle, self.handle,
               d.ctypes.data_as(ctypes.c_void_p), 0)

    def release(self):
        """Transfer ownership to a native object (e.g. the multigrid hierarchy)."""
        self._owned = False
        return self.handle

    def matvec_dev(self, x, out=None, mode=0, b=None):
        ctx = self.ctx
        ctx.sync_stream()
        out = N.empty(self.shape[0], ctx) if out is None else out
        N.call("pd_csr_spmv", ctx.handle, self.handle, N.ptr(x), N.ptr(out), mode,
               N.ptr(b) if b is not None else ctypes.c_void_p())
        return out

    def dot(self, x):
        xd = N.to_device(x, self.ctx)
        return N.like_input(self.matvec_dev(xd), x)

    __matmul__ = dot

    def __del__(self):
        try:
            if getattr(self, "_owned", False) and self.handle:
                N.load_library().pd_csr_destroy(self.handle)
        except Exception:
            pass


def device_csr(A, ctx=None) -> DeviceCsr:
    return A if isinstance(A, DeviceCsr) else DeviceCsr(A, ctx)


class Ilu0:
    """ILU(0) factors on the GPU (linalg.py:116-145): level-scheduled factor and solves."""

    def __init__(self, A, _nblocks: int = 1):
        self.ctx = N.context()
        if isinstance(A, DeviceCsr):
            self._A = A
        else:
            A = as_csr(A)
            if A.shape[0] != A.shape[1]:
                raise ConfigurationError("ILU(0) needs a square matrix")
            self._A = DeviceCsr(A, self.ctx)
        self.n = self._A.shape[0]
        h = ctypes.c_void_p()
        N.call("pd_ilu0_create", self.ctx.handle, self._A.handle, int(_nblocks), ctypes.byref(h))
        self.handle = h

    def levels(self) -> tuple[int, int]:
        lo, up = ctypes.c_int32(), ctypes.c_int32()
        N.call("pd_ilu0_levels", self.handle, ctypes.byref(lo), ctypes.byref(up))
        return lo.value, up.value

    def set_wavefront(self, ngroup: int, nline: int, npoint: int, ngroup_lower: int = 0) -> bool:
        """Structured wavefront sweeps for rows laid out [task][ngroup][nline][npoint]
        (the lower sweep's tasks span `ngroup_lower` grids when > 0)."""
        return set_wavefront(self.ctx, self.handle, ngroup, nline, npoint, ngroup_lower)

    def factors(self) -> tuple[sp.csr_matrix, sp.csr_matrix]:
        """(L, U) as explicit CSR matrices, unit diagonal on L (linalg.py:138-145):
        the device factor values copied back onto the factor's pattern."""
        if type(self) is not Ilu0 or self._A._indptr is None:
            raise ConfigurationError("factors() is defined for a single ILU(0) of a host matrix")
        rp, ci = self._A._indptr, self._A._indices
        vals = np.empty(int(rp[-1]), dtype=np.float64)
        N.call("pd_ilu0_factor_values", self.ctx.handle, self.handle,
               vals.ctypes.data_as(ctypes.c_void_p), int(vals.size))
        full = sp.csr_matrix((vals, ci, rp), shape=(self.n, self.n))
        L = sp.tril(full, k=-1) + sp.eye(self.n, format="csr")
        U = sp.triu(full, k=0)
        return as_csr(L), as_csr(U)

    def update_values(self, A) -> None:
        """New values on the same pattern (e.g. a Newton Jacobian): device refactor."""
        self._A.set_values(as_csr(A).data)
        N.call("pd_ilu0_refactor", self.ctx.handle, self.handle)

    def sweep_kind(self) -> int:
        """2: template-structured wavefront (pd_wf2.cu), 1: pattern-table wavefront,
        0: level-scheduled sweeps."""
        return sweep_kind(self.handle)

    def solve_dev(self, b, out=None):
        self.ctx.sync_stream()
        out = N.empty(self.n, self.ctx) if out is None else out
        N.call("pd_ilu0_solve", self.ctx.handle, self.handle, N.ptr(b), N.ptr(out))
        return out

    def solve(self, b):
        return N.like_input(self.solve_dev(N.to_device(b, self.ctx)), b)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.load_library().pd_ilu0_destroy(self.handle)
        except Exception:
            pass


def set_wavefront(ctx, ilu_handle, ngroup: int, nline: int, npoint: int,
                  ngroup_lower: int = 0) -> bool:
    applied = ctypes.c_int()
    N.call("pd_ilu0_set_wavefront", ctx.handle, ilu_handle, int(ngroup), int(nline), int(npoint),
           int(ngroup_lower), ctypes.byref(applied))
    return bool(applied.value)


def sweep_kind(ilu_handle) -> int:
    k = ctypes.c_int()
    N.call("pd_ilu0_sweep_kind", ilu_handle, ctypes.byref(k))
    return k.value


def ilu0(A) -> Ilu0:
    return Ilu0(A)


class BlockJacobiPrecond(Ilu0):
    """Block-Jacobi ILU(0) over contiguous ranges (linalg.py:152-189).

    The ranges follow the reference rule (size n//P, the last absorbs the
    remainder).  On the GPU all blocks are one masked factorization, so the
    result is independent of any worker count by construction; ``parallel``
    is accepted for API compatibility.
    """

    def __init__(self, A, num_blocks: int, parallel: bool | None = None):
        n = A.shape[0]
        if num_blocks < 1 or num_blocks > n:
            raise ConfigurationError(f"num_blocks must be in [1, {n}], got {num_blocks}")
        size = n // num_blocks
        self.ranges = [(b * size, (b + 1) * size if b < num_blocks - 1 else n)
                       for b in range(num_blocks)]
        self.parallel = parallel
        super().__init__(A, num_blocks)


def block_jacobi(A, num_blocks: int, parallel: bool | None = None) -> BlockJacobiPrecond:
    return BlockJacobiPrecond(A, num_blocks, parallel)


class DenseLU:
    """Coarsest-level dense LU with partial pivoting, factored and solved on device."""

    def __init__(self, A):
        self.ctx = N.context()
        self._A = device_csr(A if not isinstance(A, np.ndarray) else sp.csr_matrix(A), self.ctx)
        if self._A.shape[0] != self._A.shape[1]:
            raise ConfigurationError("dense LU needs a square matrix")
        self.n = self._A.shape[0]
        h = ctypes.c_void_p()
        N.call("pd_dense_lu_create", self.ctx.handle, self._A.handle, ctypes.byref(h))
        self.handle = h

    def solve(self, b):
        bd = N.to_device(b, self.ctx)
        out = N.empty(self.n, self.ctx)
        N.call("pd_dense_lu_solve", self.ctx.handle, self.handle, N.ptr(bd), N.ptr(out))
        return N.like_input(out, b)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.load_library().pd_dense_lu_destroy(self.handle)
        except Exception:
            pass


class BandedLU:
    """Banded LU with partial pivoting, factored and solved on the device
    (pd_band.cu) — the drop-in for the SuperLU solves of spacetime.py:154-195.

    ``order`` (optional permutation, band row i = unknown order[i]) reorders the
    unknowns so that the matrix is banded; vectors passed to ``solve`` stay in the
    caller's order.  A singular matrix raises SolverError.
    """

    def __init__(self, A, order=None):
        self.ctx = N.context()
        A = as_csr(A)
        if A.shape[0] != A.shape[1]:
            raise ConfigurationError("banded LU needs a square matrix")
        self.n = A.shape[0]
        perm = None
        if order is not None:
            perm = np.ascontiguousarray(order, dtype=np.int32)
            if perm.shape != (self.n,) or not np.array_equal(np.sort(perm), np.arange(self.n)):
                raise ConfigurationError("order must be a permutation of the unknowns")
            A = as_csr(A[perm][:, perm])
        coo = A.tocoo()
        off = coo.row.astype(np.int64) - coo.col.astype(np.int64)
        self.kl = int(max(off.max(), 0)) if off.size else 0
        self.ku = int(max(-off.min(), 0)) if off.size else 0
        self._A = DeviceCsr(A, self.ctx)
        h = ctypes.c_void_p()
        N.call("pd_band_lu_create", self.ctx.handle, self._A.handle, self.kl, self.ku,
               perm.ctypes.data_as(ctypes.c_void_p) if perm is not None else None,
               ctypes.byref(h))
        self.handle = h
        self._A = None  # the band copy is all the solve needs

    def solve(self, b):
        self.ctx.sync_stream()
        bd = N.to_device(b, self.ctx)
        if bd.numel() != self.n:
            raise ConfigurationError(f"right-hand side has {bd.numel()} entries, expected {self.n}")
        out = N.empty(self.n, self.ctx)
        N.call("pd_band_lu_solve", self.ctx.handle, self.handle, N.ptr(bd.contiguous()),
               N.ptr(out))
        return N.like_input(out, b)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.load_library().pd_band_lu_destroy(self.handle)
        except Exception:
            pass


def _report_from(rep: N.SolveReportC, hist: np.ndarray) -> SolveReport:
    return SolveReport(iterations=int(rep.iterations), converged=bool(rep.converged),
                       diverged=bool(rep.diverged),
                       residual_history=[float(v) for v in hist[: rep.hist_len]])


def _is_device_operator(A) -> bool:
    return isinstance(A, DeviceCsr) or sp.issparse(A) or isinstance(A, np.ndarray)


def gmres(A, b, precond=None, x0=None, tol_rel: float = 1e-9, tol_abs: float = 1e-9,
          restart: int = 30, max_it: int = 1000):
    """Restarted right-preconditioned GMRES on the GPU (linalg.py:215-311).

    ``A``: scipy sparse matrix / DeviceCsr, or — as in the reference
    (linalg.py:233-237) — any object with ``.dot`` or a callable matvec;
    ``precond``: Ilu0 / BlockJacobiPrecond / None, or any object with
    ``.solve`` or a callable.  Matrices and device factorizations are applied
    by the device kernels; other callables are invoked from the device GMRES
    engine through a host callback (numpy in, numpy out — or CUDA tensors when
    ``b`` is one), with the Krylov vectors and orthogonalisation kept in HBM.
    """
    native_A = _is_device_operator(A)
    native_M = precond is None or isinstance(precond, Ilu0)
    if native_A and native_M:
        Ad = device_csr(A if not isinstance(A, np.ndarray) else sp.csr_matrix(A))
        ctx = Ad.ctx
        ctx.sync_stream()
        bd = N.to_device(b, ctx)
        n = bd.numel()
        x0d = N.to_device(x0, ctx) if x0 is not None else None
        out = N.empty(n, ctx)
        rep = N.SolveReportC()
        hist = np.zeros(int(max(max_it, 1)) + 2)
        N.call("pd_gmres", ctx.handle, Ad.handle, precond.handle if precond is not None else None,
               N.ptr(bd), N.ptr(x0d), N.ptr(out), float(tol_rel), float(tol_abs), int(restart),
               int(max_it), ctypes.byref(rep), hist.ctypes.data_as(ctypes.c_void_p), hist.size)
        return N.like_input(out, b), _report_from(rep, hist)
    return _gmres_callables(A, b, precond, x0, tol_rel, tol_abs, restart, max_it, native_A,
                            native_M)


def _gmres_callables(A, b, precond, x0, tol_rel, tol_abs, restart, max_it, native_A, native_M):
    """GMRES whose operator and/or preconditioner is a host callable
    (pd_gmres_callable): each application hands the callable the engine's
    current vector and takes its result back through two exchange vectors."""
    Ad = None
    if native_A:
        Ad = device_csr(A if not isinstance(A, np.ndarray) else sp.csr_matrix(A))
        ctx = Ad.ctx
    else:
        ctx = precond.ctx if isinstance(precond, Ilu0) else N.context()
    ctx.sync_stream()
    bd = N.to_device(b, ctx)
    n = bd.numel()
    x0d = N.to_device(x0, ctx) if x0 is not None else None
    out = N.empty(n, ctx)
    cb_in, cb_out = N.empty(max(n, 1), ctx), N.empty(max(n, 1), ctx)
    on_device = N.is_tensor(b) and b.is_cuda
    failure: list[BaseException] = []

    def through(fn):
        def run(_user):
            try:
                arg = cb_in[:n].clone() if on_device else N.to_host(cb_in[:n])
                res = fn(arg)
                rd = N.to_device(res if N.is_tensor(res) else np.asarray(res, dtype=np.float64),
                                 ctx)
                if rd.numel() != n:
                    raise ConfigurationError(
                        f"callable returned {rd.numel()} values for a vector of {n}")
                cb_out[:n].copy_(rd.reshape(-1))
                ctx.sync_stream()
                N.torch_mod().cuda.current_stream().synchronize()
                return 0
            except BaseException as exc:  # noqa: BLE001 - re-raised after the C call returns
                failure.append(exc)
                return 1
        return N.APPLY_CB(run)

    matvec_cb = psolve_cb = None
    if not native_A:
        matvec_cb = through(A.dot if hasattr(A, "dot") else A)
    if not native_M:
        psolve_cb = through(precond.solve if hasattr(precond, "solve") else precond)
    rep = N.SolveReportC()
    hist = np.zeros(int(max(max_it, 1)) + 2)
    try:
        N.call("pd_gmres_callable", ctx.handle, int(n), Ad.handle if Ad is not None else None,
               matvec_cb, precond.handle if (native_M and precond is not None) else None,
               psolve_cb, None, N.ptr(cb_in), N.ptr(cb_out), N.ptr(bd), N.ptr(x0d), N.ptr(out),
               float(tol_rel), float(tol_abs), int(restart), int(max_it), ctypes.byref(rep),
               hist.ctypes.data_as(ctypes.c_void_p), hist.size)
    except Exception:
        if failure:
            raise failure[0]
        raise
    return N.like_input(out, b), _report_from(rep, hist)
