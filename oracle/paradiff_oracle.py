"""CPU restatement of the reference solvers — TEST INFRASTRUCTURE ONLY.

Every function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/paradiff/`).  The numerics follow the reference's
operation order where it matters (ILU(0) in C, `oracle/ilu0.c`; GMRES/MGS,
V-cycles, SDC sweeps, FAS and the PFASST window schedule in numpy).  The
threaded PFASST driver is simulated sequentially: the reference's barriers
make it deterministic (worker w reads its predecessor's fine terminal from
the previous iteration and its coarse terminal from the current one).

Pinned against golden vectors from the real reference: tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from numpy.polynomial import legendre
from scipy.sparse.linalg import splu

from .build import build as _build_c


# Reduction hook: the reference uses numpy/BLAS dot products; tests swap in a
# different (equally valid) summation order to measure the rounding floor of
# the reference's own output.
_DOT = np.dot


def set_dot(fn=None):
    """Install a dot-product implementation (None restores numpy.dot)."""
    global _DOT
    _DOT = np.dot if fn is None else fn


def _norm(v):
    return float(np.sqrt(_DOT(v, v))) if _DOT is not np.dot else float(np.linalg.norm(v))


class OracleConfigError(ValueError):
    pass


class OracleSolverError(RuntimeError):
    pass


@dataclass
class Report:
    """Mirror of report.py:8-36 (SolveReport)."""

    iterations: int = 0
    converged: bool = False
    diverged: bool = False
    residual_history: list = field(default_factory=list)
    inner_iterations: list = field(default_factory=list)
    newton_iterations: int = 0
    damped_steps: int = 0
    wall_time: float = 0.0


# --------------------------------------------------------------- reactions
# spacetime.py:44-50 hard-wires r(u) = u^3 - u; the Fisher form r = u^2 - u
# is the BASELINE config-3 variant (SURVEY Appendix A monkeypatch).
def reaction_value(u, kind="cubic"):
    if kind == "cubic":
        return u ** 3 - u
    if kind == "fisher":
        return u ** 2 - u
    raise OracleConfigError(kind)


def reaction_slope(u, kind="cubic"):
    if kind == "cubic":
        return 3.0 * u ** 2 - 1.0
    if kind == "fisher":
        return 2.0 * u - 1.0
    raise OracleConfigError(kind)


# --------------------------------------------------------------- tableau
def radau_right(M):
    """collocation.py:23-42."""
    if M == 1:
        return np.array([1.0])
    c = np.zeros(M + 1)
    c[M - 1], c[M] = 1.0, -1.0
    r = np.real(legendre.legroots(c))
    r = np.sort(r[np.abs(r - 1.0) > 1e-8])
    r = r - legendre.legval(r, c) / legendre.legval(r, legendre.legder(c))
    return np.append((r + 1.0) / 2.0, 1.0)


def lagrange_values(x, t):
    """collocation.py:55-64."""
    out = np.empty(x.size)
    for j in range(x.size):
        v = 1.0
        for k in range(x.size):
            if k != j:
                v *= (t - x[k]) / (x[j] - x[k])
        out[j] = v
    return out


def lagrange_slopes(x, t):
    """collocation.py:66-80."""
    out = np.zeros(x.size)
    for j in range(x.size):
        acc = 0.0
        for i in range(x.size):
            if i == j:
                continue
            term = 1.0 / (x[j] - x[i])
            for k in range(x.size):
                if k != j and k != i:
                    term *= (t - x[k]) / (x[j] - x[k])
            acc += term
        out[j] = acc
    return out


def _gauss(npts, a, b):
    """collocation.py:83-86."""
    x, w = legendre.leggauss(npts)
    return 0.5 * (b - a) * x + 0.5 * (a + b), 0.5 * (b - a) * w


def q_matrix(x):
    """collocation.py:89-102."""
    M = x.size
    Q = np.empty((M, M))
    for m in range(M):
        pts, wts = _gauss(M + 1, 0.0, x[m])
        Q[m] = wts @ np.array([lagrange_values(x, t) for t in pts])
    return Q


def qdelta_matrix(x, kind="implicit-euler"):
    """collocation.py:105-126."""
    M = x.size
    d = np.diff(x, prepend=0.0)
    if kind == "implicit-euler":
        return np.tril(np.tile(d, (M, 1)))
    if kind == "explicit-euler":
        return np.tril(np.tile(d, (M, 1)), k=-1)
    if kind == "lu-trick":
        _, _, U = scipy.linalg.lu(q_matrix(x).T)
        return U.T
    raise OracleConfigError(kind)


def dg_matrices(x):
    """collocation.py:129-149 -> (Kq, Mq, Jq)."""
    M = x.size
    pts, wts = _gauss(M + 1, 0.0, 1.0)
    V = np.array([lagrange_values(x, t) for t in pts])
    D = np.array([lagrange_slopes(x, t) for t in pts])
    Mq = V.T @ (wts[:, None] * V)
    l1, l0 = lagrange_values(x, 1.0), lagrange_values(x, 0.0)
    Kq = -(D.T @ (wts[:, None] * V)) + np.outer(l1, l1)
    return Kq, Mq, np.outer(l0, l1)


@dataclass(frozen=True)
class Tableau:
    """collocation.py:152-188."""

    M: int
    nodes: np.ndarray
    Q: np.ndarray
    QDI: np.ndarray
    QDE: np.ndarray
    Kq: np.ndarray
    Mq: np.ndarray
    Jq: np.ndarray

    @property
    def l0(self):
        return self.Jq[:, -1].copy()


def tableau(M, qdelta="implicit-euler"):
    x = radau_right(M)
    Kq, Mq, Jq = dg_matrices(x)
    return Tableau(M, x, q_matrix(x), qdelta_matrix(x, qdelta),
                   qdelta_matrix(x, "explicit-euler"), Kq, Mq, Jq)


# --------------------------------------------------------------- space (1D FEM)
def fem1d_operators(Nx, X=1.0):
    """fem1d.py:58-74 -> (Kh csr, mh lumped diagonal)."""
    n, h = Nx + 1, X / Nx
    main = np.full(n, 2.0 / h)
    main[0] = main[-1] = 1.0 / h
    off = np.full(n - 1, -1.0 / h)
    Kh = sp.diags([off, main, off], [-1, 0, 1], format="csr")
    mm = np.full(n, 4.0 * h / 6.0)
    mm[0] = mm[-1] = 2.0 * h / 6.0
    mo = np.full(n - 1, h / 6.0)
    Mc = sp.diags([mo, mm, mo], [-1, 0, 1], format="csr")
    return Kh, np.asarray(Mc.sum(axis=1)).ravel()


# --------------------------------------------------------------- sparse helpers
def canon(A):
    """linalg.py:47-52."""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    return A


def skron(A, B):
    """linalg.py:55-60."""
    return canon(sp.kron(sp.coo_matrix(A), sp.coo_matrix(B), format="csr"))


_CLIB = None


def _clib():
    global _CLIB
    if _CLIB is None:
        lib = ctypes.CDLL(str(_build_c()))
        P = ctypes.c_void_p
        lib.oracle_ilu0_factor.restype = ctypes.c_int64
        lib.oracle_ilu0_factor.argtypes = [ctypes.c_int64, P, P, P, P]
        lib.oracle_ilu0_solve.restype = None
        lib.oracle_ilu0_solve.argtypes = [ctypes.c_int64, P, P, P, P, P, P]
        _CLIB = lib
    return _CLIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OIlu0:
    """linalg.py:116-136 (ILU(0) on the CSR pattern; C kernels in ilu0.c)."""

    def __init__(self, A):
        A = canon(A)
        self.n = A.shape[0]
        self.rowptr = A.indptr.astype(np.int64)
        self.col = A.indices.astype(np.int64)
        self.val = A.data.astype(np.float64).copy()
        self.diag = np.empty(self.n, dtype=np.int64)
        bad = _clib().oracle_ilu0_factor(self.n, _ptr(self.rowptr), _ptr(self.col),
                                         _ptr(self.val), _ptr(self.diag))
        if bad >= 0:
            raise OracleSolverError(f"zero pivot in ILU(0) at row {bad}")

    def solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        _clib().oracle_ilu0_solve(self.n, _ptr(self.rowptr), _ptr(self.col), _ptr(self.val),
                                  _ptr(self.diag), _ptr(b), _ptr(x))
        return x


_POOL = None


def _pool(threads):
    global _POOL
    if _POOL is None or _POOL._max_workers != threads:
        _POOL = ThreadPoolExecutor(max_workers=threads)
    return _POOL


def block_ranges(n, nblocks):
    """linalg.py:166-170: size n//P, the last block absorbs the remainder."""
    s = n // nblocks
    return [(b * s, (b + 1) * s if b < nblocks - 1 else n) for b in range(nblocks)]


class OBlockJacobi:
    """linalg.py:152-189; block solves run on a thread pool (C releases the GIL)."""

    def __init__(self, A, nblocks, threads=1):
        A = canon(A)
        n = A.shape[0]
        if nblocks < 1 or nblocks > n:
            raise OracleConfigError("bad block count")
        self.ranges = block_ranges(n, nblocks)
        self.blocks = [OIlu0(A[a:b, a:b]) for a, b in self.ranges]
        self.threads = threads

    def solve(self, v):
        out = np.empty_like(v, dtype=np.float64)
        if self.threads > 1 and len(self.blocks) > 1:
            pool = _pool(self.threads)
            futs = [pool.submit(blk.solve, v[a:b]) for blk, (a, b) in zip(self.blocks, self.ranges)]
            for (a, b), f in zip(self.ranges, futs):
                out[a:b] = f.result()
        else:
            for blk, (a, b) in zip(self.blocks, self.ranges):
                out[a:b] = blk.solve(v[a:b])
        return out


class ODenseLU:
    """linalg.py:196-209."""

    def __init__(self, A):
        A = np.asarray(A.toarray() if sp.issparse(A) else A, dtype=np.float64)
        try:
            self.f = scipy.linalg.lu_factor(A)
        except (ValueError, scipy.linalg.LinAlgError) as exc:
            raise OracleSolverError(str(exc)) from exc

    def solve(self, b):
        return scipy.linalg.lu_solve(self.f, b)


def gmres(A, b, M=None, x0=None, tol_rel=1e-9, tol_abs=1e-9, restart=30, max_it=1000):
    """linalg.py:215-311: restarted, right-preconditioned GMRES with MGS + Givens."""
    mv = A.dot if hasattr(A, "dot") else A
    ps = (lambda v: v) if M is None else (M.solve if hasattr(M, "solve") else M)
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    restart = max(1, min(restart, n))
    r = b - mv(x)
    beta = _norm(r)
    if not np.isfinite(beta):
        raise OracleSolverError("non-finite initial residual")
    thr = max(tol_abs, tol_rel * beta)
    rep = Report(residual_history=[beta])
    if beta <= thr:
        rep.converged = True
        return x, rep
    lowest, total = beta, 0
    while True:
        V = np.empty((restart + 1, n))
        H = np.zeros((restart + 1, restart))
        c = np.empty(restart)
        s = np.empty(restart)
        g = np.zeros(restart + 1)
        V[0] = r / beta
        g[0] = beta
        j = -1
        for j in range(restart):
            w = mv(ps(V[j]))
            for i in range(j + 1):
                H[i, j] = _DOT(w, V[i])
                w -= H[i, j] * V[i]
            hn = _norm(w)
            H[j + 1, j] = hn
            happy = hn <= 1e-14 * max(1.0, beta)
            if not happy:
                V[j + 1] = w / hn
            for i in range(j):
                t = c[i] * H[i, j] + s[i] * H[i + 1, j]
                H[i + 1, j] = -s[i] * H[i, j] + c[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            if d == 0.0:
                c[j], s[j] = 1.0, 0.0
            else:
                c[j], s[j] = H[j, j] / d, H[j + 1, j] / d
            H[j, j] = d
            H[j + 1, j] = 0.0
            g[j + 1] = -s[j] * g[j]
            g[j] = c[j] * g[j]
            res = abs(g[j + 1])
            if not np.isfinite(res):
                raise OracleSolverError("non-finite residual in GMRES iteration")
            total += 1
            rep.residual_history.append(res)
            if res <= thr or happy or total >= max_it:
                break
        k = j + 1
        y = scipy.linalg.solve_triangular(H[:k, :k], g[:k], lower=False)
        x = x + ps(V[:k].T @ y)
        r = b - mv(x)
        beta = _norm(r)
        if not np.isfinite(beta):
            raise OracleSolverError("non-finite residual in GMRES restart")
        rep.residual_history[-1] = beta
        lowest = min(lowest, beta)
        if beta <= thr:
            rep.converged = True
            break
        if total >= max_it or beta > 10.0 * lowest:
            rep.diverged = True
            break
    rep.iterations = total
    return x, rep


# --------------------------------------------------------------- space-time system
class OSystem:
    """spacetime.py:53-199 with injectable (Kh, mh) and reaction kind."""

    def __init__(self, tab, Kh, mh, Nt, T, gamma, u0, reaction="cubic"):
        self.tab, self.Nt, self.T, self.gamma = tab, Nt, T, float(gamma)
        self.Kh = canon(Kh)
        self.mh = np.asarray(mh, dtype=np.float64)
        self.S = self.mh.size
        self.u0 = np.asarray(u0, dtype=np.float64)
        self.kind = reaction
        self.dt = T / Nt
        Mh = sp.diags(self.mh, format="dia")
        self.Mh = Mh
        # spacetime.py:77-80
        self.A = skron(tab.Kq, Mh) + self.dt * skron(tab.Mq, self.Kh)
        self.B = -skron(tab.Jq, Mh)
        self.Mq_h = self.dt * skron(tab.Mq, Mh)
        self._L = None

    @property
    def block(self):
        return self.tab.M * self.S

    @property
    def size(self):
        return self.Nt * self.block

    def padded_u0(self):
        out = np.zeros(self.block)
        out[-self.S:] = self.u0
        return out

    def rhs(self):
        """spacetime.py:110-114."""
        out = np.zeros(self.size)
        out[: self.block] = -self.B @ self.padded_u0()
        return out

    def global_matrix(self):
        """spacetime.py:117-124."""
        if self._L is None:
            Nt = self.Nt
            sub = sp.diags([np.ones(Nt - 1)], [-1], format="csr") if Nt > 1 else sp.csr_matrix((Nt, Nt))
            self._L = skron(sp.eye(Nt, format="csr"), self.A) + skron(sub, self.B)
        return self._L

    def residual(self, u):
        """spacetime.py:131-142."""
        U = u.reshape(self.Nt, self.block)
        res = (self.A @ U.T).T
        if self.gamma != 0.0:
            res += self.gamma * (self.Mq_h @ reaction_value(U, self.kind).T).T
        if self.Nt > 1:
            res[1:] += (self.B @ U[:-1].T).T
        res[0] -= -self.B @ self.padded_u0()
        return res.ravel()

    def jacobian(self, u):
        """spacetime.py:144-151."""
        J = self.global_matrix()
        if self.gamma != 0.0:
            R = skron(sp.eye(self.Nt, format="csr"), self.Mq_h)
            J = J + self.gamma * (R @ sp.diags(reaction_slope(u, self.kind)))
        return sp.csr_matrix(J)

    def solve_sequential(self):
        """spacetime.py:169-183 (linear case)."""
        U = np.zeros((self.Nt, self.tab.M, self.S))
        lu = splu(self.A.tocsc()) if self.gamma == 0.0 else None
        uin, guess = self.u0, np.tile(self.u0, self.tab.M)
        for n in range(self.Nt):
            rb = np.kron(self.tab.l0, self.Mh @ uin)
            if lu is not None:
                sol = lu.solve(rb)
            else:
                sol = self._element_newton(rb, guess)
            U[n] = sol.reshape(self.tab.M, self.S)
            uin, guess = U[n, -1], sol
        return U.ravel()

    def _element_newton(self, rb, guess, tol=1e-13):
        """spacetime.py:154-167."""
        u = guess.copy()
        thr = max(tol, tol * np.linalg.norm(rb))
        for _ in range(50):
            F = self.A @ u + self.gamma * (self.Mq_h @ reaction_value(u, self.kind)) - rb
            if np.linalg.norm(F) <= thr:
                return u
            J = self.A + self.gamma * (self.Mq_h @ sp.diags(reaction_slope(u, self.kind)))
            u -= splu(sp.csc_matrix(J)).solve(F)
        raise OracleSolverError("element Newton did not converge")


def newton(system, linear_solver, u_init=None, tol=1e-9, max_newton=50):
    """spacetime.py:212-258."""
    rep = Report()
    t0 = time.perf_counter()
    u = np.zeros(system.size) if u_init is None else np.array(u_init, dtype=float)
    rn = float(np.linalg.norm(system.residual(u)))
    thr = max(tol, tol * rn)
    rep.residual_history.append(rn)
    for _ in range(max_newton):
        if rn <= thr:
            rep.converged = True
            break
        J = system.jacobian(u)
        delta, inner = linear_solver(J, -system.residual(u))
        rep.inner_iterations.append(inner.iterations)
        if inner.diverged:
            rep.diverged = True
            break
        step = 1.0
        for _ in range(8):
            nn = float(np.linalg.norm(system.residual(u + step * delta)))
            if nn < rn or nn <= thr:
                break
            step *= 0.5
            rep.damped_steps += 1
        u = u + step * delta
        rn = nn
        rep.newton_iterations += 1
        rep.residual_history.append(rn)
    else:
        rep.diverged = rn > thr
    if rn <= thr:
        rep.converged = True
    rep.iterations = rep.newton_iterations
    rep.wall_time = time.perf_counter() - t0
    return u, rep


# --------------------------------------------------------------- MG transfers
def _fw(nf, nc, renorm):
    R = sp.lil_matrix((nc, nf))
    for i in range(nc):
        f = 2 * i
        if f - 1 >= 0:
            R[i, f - 1] = 0.25
        R[i, f] = 0.5
        if f + 1 < nf:
            R[i, f + 1] = 0.25
    R = R.tocsr()
    w = np.asarray(R.sum(axis=1)).ravel()
    return canon(sp.diags(1.0 / w) @ R)


def vertex_restriction(nf):
    """multigrid.py:37-56."""
    if (nf - 1) % 2 or nf < 3:
        raise OracleConfigError("cannot bisect")
    return _fw(nf, (nf - 1) // 2 + 1, True)


def vertex_prolongation(nf):
    """multigrid.py:59-72."""
    nc = (nf - 1) // 2 + 1
    P = sp.lil_matrix((nf, nc))
    for f in range(nf):
        c, r = divmod(f, 2)
        if r == 0:
            P[f, c] = 1.0
        else:
            P[f, c] = 0.5
            P[f, c + 1] = 0.5
    return canon(P)


def time_restriction(ntf):
    """multigrid.py:75-90."""
    if ntf % 2 or ntf < 2:
        raise OracleConfigError("cannot bisect time")
    return _fw(ntf, ntf // 2, True)


def time_prolongation(ntf):
    """multigrid.py:93-108."""
    ntc = ntf // 2
    P = sp.lil_matrix((ntf, ntc))
    for f in range(ntf):
        c, r = divmod(f, 2)
        if r == 0:
            P[f, c] = 1.0
        elif c + 1 < ntc:
            P[f, c] = 0.5
            P[f, c + 1] = 0.5
        else:
            P[f, c] = 1.0
    return canon(P)


def node_prolongation(mc, mf):
    """multigrid.py:111-118."""
    xc, xf = radau_right(mc), radau_right(mf)
    return canon(sp.csr_matrix(np.array([lagrange_values(xc, t) for t in xf])))


def node_restriction(mc, mf):
    """multigrid.py:121-126."""
    R = sp.csr_matrix(node_prolongation(mc, mf).T)
    w = np.asarray(R.sum(axis=1)).ravel()
    return canon(sp.diags(1.0 / w) @ R)


@dataclass(frozen=True)
class Dims:
    nt: int
    m: int
    s: int

    @property
    def size(self):
        return self.nt * self.m * self.s


def level_dims(strategy, L, nt, m, nx):
    """multigrid.py:148-157."""
    out = []
    for l in range(1, L + 1):
        if strategy == "SMG":
            out.append(Dims(nt, m, nx // 2 ** (l - 1) + 1))
        elif strategy == "STMG":
            out.append(Dims(nt // 2 ** (l - 1), m, nx // 2 ** (l - 1) + 1))
        else:
            out.append(Dims(nt, max(m - l + 1, 1), nx // 2 ** (l - 1) + 1))
    return out


def composite_transfers(dims, space_pairs):
    """multigrid.py:172-191 with the spatial factor pairs injectable
    (space_pairs[l] = (Rs, Ps) between level l and l+1)."""
    out = []
    for l, (f, c) in enumerate(zip(dims[:-1], dims[1:])):
        if f.nt != c.nt:
            Rt, Pt = time_restriction(f.nt), time_prolongation(f.nt)
        else:
            Rt = Pt = sp.eye(f.nt, format="csr")
        if f.m != c.m:
            Rm, Pm = node_restriction(c.m, f.m), node_prolongation(c.m, f.m)
        else:
            Rm = Pm = sp.eye(f.m, format="csr")
        Rs, Ps = space_pairs[l]
        out.append((skron(Rt, skron(Rm, Rs)), skron(Pt, skron(Pm, Ps))))
    return out


class OMultigrid:
    """multigrid.py:197-305 (Galerkin hierarchy, GMRES(nu)+ILU smoother, dense-LU coarsest)."""

    def __init__(self, A, dims, transfers, nu, partitions=1, restart=30, smooth_solves=1, threads=1,
                 mats=None):
        self.dims, self.transfers, self.nu = dims, transfers, nu
        self.partitions, self.restart, self.smooth_solves = partitions, restart, smooth_solves
        self.threads = threads
        self.set_fine_matrix(A, mats)

    def set_fine_matrix(self, A, mats=None):
        """multigrid.py:224-241.  `mats`: the level matrices R A P already formed
        (bench.py's CPU leg hands over the GPU arm's host copies of the same scipy
        products to skip the host Galerkin setup)."""
        A = canon(A)
        if A.shape[0] != self.dims[0].size:
            raise OracleConfigError("fine matrix size mismatch")
        self.mats = [A]
        if mats is not None:
            if len(mats) != len(self.dims):
                raise OracleConfigError("level matrix count mismatch")
            self.mats += [canon(m) for m in mats[1:]]
        for R, P in self.transfers[len(self.mats) - 1:]:
            self.mats.append(canon(R @ self.mats[-1] @ P))
        self.pre = []
        for Al in self.mats[:-1]:
            nb = min(self.partitions, Al.shape[0])
            self.pre.append(OBlockJacobi(Al, nb, self.threads) if nb > 1 else OIlu0(Al))
        self.coarse = ODenseLU(self.mats[-1])

    def smooth(self, l, b, x):
        """multigrid.py:243-256."""
        for _ in range(self.smooth_solves):
            r = b - self.mats[l] @ x
            dx, _ = gmres(self.mats[l], r, M=self.pre[l], tol_rel=1e-13, tol_abs=0.0,
                          restart=min(self.nu, self.restart), max_it=self.nu)
            x = x + dx
        return x

    def cycle(self, l, b, x):
        """multigrid.py:258-266."""
        if l == len(self.dims) - 1:
            return self.coarse.solve(b)
        x = self.smooth(l, b, x)
        r = b - self.mats[l] @ x
        R, P = self.transfers[l]
        rc = R @ r
        x = x + P @ self.cycle(l + 1, rc, np.zeros_like(rc))
        return self.smooth(l, b, x)

    def vcycle(self, b, x):
        out = self.cycle(0, b, x.copy())
        if not np.all(np.isfinite(out)):
            raise OracleSolverError("V-cycle produced non-finite values")
        return out

    def solve(self, b, x0=None, tol_rel=1e-9, tol_abs=1e-9, max_cycles=1000):
        """multigrid.py:275-305."""
        t0 = time.perf_counter()
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=float)
        res = float(np.linalg.norm(b - self.mats[0] @ x))
        rep = Report(residual_history=[res])
        thr = max(tol_abs, tol_rel * res)
        lowest = res
        while res > thr:
            if rep.iterations >= max_cycles:
                rep.diverged = True
                break
            x = self.vcycle(b, x)
            res = float(np.linalg.norm(b - self.mats[0] @ x))
            rep.iterations += 1
            rep.residual_history.append(res)
            if not np.isfinite(res) or res > 10.0 * lowest:
                rep.diverged = True
                break
            lowest = min(lowest, res)
        rep.converged = res <= thr
        rep.wall_time = time.perf_counter() - t0
        return x, rep


def mg_newton_solver(mg, tol_rel=1e-9, tol_abs=1e-9, max_cycles=1000):
    """multigrid.py:339-364 (default branch: iterate to tolerance)."""
    def solver(J, rhs):
        mg.set_fine_matrix(J)
        return mg.solve(rhs, tol_rel=tol_rel, tol_abs=tol_abs, max_cycles=max_cycles)
    return solver


def fem_hierarchy(system, strategy, L, nu, partitions=1, threads=1):
    """multigrid.py:308-336 for the reference's own 1D FEM system (Nx = S-1)."""
    nt, m, nx = system.Nt, system.tab.M, system.S - 1
    for l in range(1, L):
        if nx % 2 ** l or (strategy == "STMG" and nt % 2 ** l):
            raise OracleConfigError("divisibility")
    dims = level_dims(strategy, L, nt, m, nx)
    pairs = [(vertex_restriction(d.s), vertex_prolongation(d.s)) for d in dims[:-1]]
    return OMultigrid(system.global_matrix(), dims, composite_transfers(dims, pairs), nu,
                      partitions, threads=threads)


# --------------------------------------------------------------- SDC / PFASST
NODE_TOL = 1e-13  # pfasst.py:33


class OSdcLevel:
    """pfasst.py:60-200 with injectable (Kh, mh) and reaction kind."""

    def __init__(self, tab, Kh, mh, dt, gamma, mode="implicit", reaction="cubic"):
        if mode not in ("implicit", "imex"):
            raise OracleConfigError(mode)
        self.tab, self.dt, self.gamma, self.mode, self.kind = tab, float(dt), float(gamma), mode, reaction
        self.mh = np.asarray(mh, dtype=np.float64)
        self.Kh = canon(Kh)
        self.Mh = sp.diags(self.mh, format="csr")
        qd = tab.QDI
        self.node_ops = [self.Mh + self.dt * qd[m, m] * self.Kh for m in range(tab.M)]
        self.node_pre = [OIlu0(A) for A in self.node_ops]

    @property
    def M(self):
        return self.tab.M

    def f_diff(self, U):
        return -(self.Kh @ U.T).T / self.mh

    def f_react(self, U):
        if self.gamma == 0.0:
            return np.zeros_like(U)
        return -self.gamma * reaction_value(U, self.kind)

    def f_all(self, U):
        return self.f_diff(U) + self.f_react(U)

    def coll_residual(self, U, U0, tau):
        """pfasst.py:107-112."""
        r = U - U0 - self.dt * self.tab.Q @ self.f_all(U)
        return r if tau is None else r - tau

    def res_norm(self, U, U0, tau):
        return float(np.linalg.norm(self.coll_residual(U, U0, tau)))

    def node_linear(self, m, rhs, guess):
        """pfasst.py:118-132."""
        b = self.mh * rhs
        x, rep = gmres(self.node_ops[m], b, M=self.node_pre[m], x0=guess, tol_rel=NODE_TOL,
                       tol_abs=NODE_TOL * max(1.0, float(np.linalg.norm(b))), restart=30, max_it=200)
        if rep.diverged:
            raise OracleSolverError(f"node solve failed at node {m}")
        return x

    def node_newton(self, m, rhs, guess):
        """pfasst.py:134-152."""
        q = self.dt * self.tab.QDI[m, m]
        u = guess.copy()
        b = self.mh * rhs
        scale = max(1.0, float(np.linalg.norm(b)))
        for _ in range(50):
            g = self.mh * u + q * (self.Kh @ u + self.gamma * self.mh * reaction_value(u, self.kind)) - b
            if np.linalg.norm(g) <= 1e-12 * scale:
                return u
            J = self.Mh + q * (self.Kh + self.gamma * sp.diags(self.mh * reaction_slope(u, self.kind)))
            d, rep = gmres(J, -g, M=OIlu0(J), tol_rel=NODE_TOL, tol_abs=NODE_TOL * scale,
                           restart=30, max_it=200)
            if rep.diverged:
                raise OracleSolverError(f"node Newton failed at node {m}")
            u = u + d
        raise OracleSolverError(f"node Newton stalled at node {m}")

    def sweep(self, U, U0, tau):
        """pfasst.py:155-200; returns the new node values."""
        M, dt, Q = self.M, self.dt, self.tab.Q
        qdi, qde = self.tab.QDI, self.tab.QDE
        imex = self.mode == "imex" and self.gamma != 0.0
        with np.errstate(over="ignore", invalid="ignore"):
            if imex:
                base = U0 + dt * ((Q - qdi) @ self.f_diff(U) + (Q - qde) @ self.f_react(U))
            else:
                base = U0 + dt * ((Q - qdi) @ self.f_all(U))
            if tau is not None:
                base = base + tau
            if not np.all(np.isfinite(base)):
                raise OracleSolverError("non-finite values entered an SDC sweep")
            Un = np.empty_like(U)
            fi = np.empty_like(U)
            fe = np.empty_like(U) if imex else None
            for m in range(M):
                rhs = base[m].copy()
                for j in range(m):
                    rhs += dt * qdi[m, j] * fi[j]
                    if imex:
                        rhs += dt * qde[m, j] * fe[j]
                if imex or self.gamma == 0.0:
                    Un[m] = self.node_linear(m, rhs, U[m])
                else:
                    Un[m] = self.node_newton(m, rhs, U[m])
                if imex:
                    fi[m] = self.f_diff(Un[m][None, :])[0]
                    fe[m] = self.f_react(Un[m][None, :])[0]
                else:
                    fi[m] = self.f_all(Un[m][None, :])[0]
        return Un


def sdc_step(u0, lev, tol_rel=1e-9, tol_abs=1e-9, max_sweeps=1000):
    """pfasst.py:223-249."""
    U = np.tile(u0, (lev.M, 1))
    res = lev.res_norm(U, u0, None)
    rep = Report(residual_history=[res])
    thr = max(tol_abs, tol_rel * res)
    lowest = res
    while res > thr:
        if rep.iterations >= max_sweeps:
            rep.diverged = True
            break
        U = lev.sweep(U, u0, None)
        res = lev.res_norm(U, u0, None)
        rep.iterations += 1
        rep.residual_history.append(res)
        if not np.isfinite(res) or res > 10.0 * lowest:
            rep.diverged = True
            break
        lowest = min(lowest, res)
    rep.converged = res <= thr
    return U, rep


@dataclass(frozen=True)
class OTransfer:
    """pfasst.py:253-270."""

    Rs: object
    Ps: object
    Rn: np.ndarray
    Pn: np.ndarray

    def down(self, U):
        return self.Rn @ (self.Rs @ U.T).T

    def up(self, U):
        return self.Pn @ (self.Ps @ U.T).T

    def down_u0(self, u0):
        return self.Rs @ u0


def node_eval(xf, xc):
    """pfasst.py:272-280: fine nodal polynomial evaluated at the coarse nodes."""
    return np.array([lagrange_values(np.asarray(xf, float), t) for t in xc])


def fas_tau(fine, coarse, tr, U, tau_f):
    """pfasst.py:283-303."""
    RU = tr.down(U)
    cc = RU - coarse.dt * coarse.tab.Q @ coarse.f_all(RU)
    cf = U - fine.dt * fine.tab.Q @ fine.f_all(U)
    tau = cc - tr.down(cf)
    if tau_f is not None:
        tau = tau + tr.down(tau_f)
    return tau


def fem_pfasst_levels(M, Nx, X, dt, gamma, L, mode="implicit", qdelta="implicit-euler"):
    """pfasst.py:323-365 (fine M, coarser levels M=1 with bisected 1D FEM meshes)."""
    tf, tc = tableau(M, qdelta), tableau(1, qdelta)
    levels = []
    for l in range(L):
        Kh, mh = fem1d_operators(Nx // 2 ** l, X)
        levels.append(OSdcLevel(tf if l == 0 else tc, Kh, mh, dt, gamma, mode))
    trs = []
    for l in range(L - 1):
        nf = levels[l].mh.size
        if levels[l].M != levels[l + 1].M:
            Rn = node_eval(levels[l].tab.nodes, levels[l + 1].tab.nodes)
            Pn = node_eval(levels[l + 1].tab.nodes, levels[l].tab.nodes)
        else:
            Rn = Pn = np.eye(levels[l].M)
        trs.append(OTransfer(vertex_restriction(nf), vertex_prolongation(nf), Rn, Pn))
    return levels, trs


def pfasst(levels, trs, nu, u_init, Nt, workers, tol_rel=1e-9, tol_abs=1e-9, max_iters=1000):
    """pfasst.py:369-587: windowed pipelined PFASST, sequential simulation."""
    if workers < 1 or workers > Nt or Nt % workers:
        raise OracleConfigError("bad worker count")
    L = len(levels)
    fine = levels[0]
    S, M = fine.mh.size, fine.M
    t0 = time.perf_counter()
    out = np.zeros((Nt, M, S))
    rep = Report()
    u_start = np.asarray(u_init, dtype=np.float64)
    ok = True
    nrecv = max(L - 1, 1)
    for start in range(0, Nt, workers):
        P = workers
        chain = [u_start]
        for tr in trs:
            chain.append(tr.down_u0(chain[-1]))
        # states[w][l] = [U, U0, tau]
        st = [[[np.tile(chain[l], (levels[l].M, 1)), chain[l].copy(), None] for l in range(L)]
              for _ in range(P)]
        r0 = fine.res_norm(st[0][0][0], st[0][0][1], None)
        thr = max(tol_abs, tol_rel * r0)
        resid = np.full(P, r0)
        lowest = np.full(P, max(r0, 1e-300))
        iters = np.zeros(P, dtype=int)
        msgs = [[None] * P for _ in range(nrecv)]
        diverged = False
        if not np.all(resid <= thr):
            for k in range(1, max_iters + 1):
                for w in range(1, P):  # _receive_nonblocking (previous iteration's messages)
                    for l in range(nrecv):
                        if msgs[l][w - 1] is not None:
                            st[w][l][1] = msgs[l][w - 1].copy()
                new_msgs = [[None] * P for _ in range(nrecv)]
                coarse_term = None
                try:
                    for w in range(P):
                        s = st[w]
                        with np.errstate(over="ignore", invalid="ignore"):
                            for _ in range(nu):
                                s[0][0] = fine.sweep(*s[0])
                            if L > 1:
                                for l in range(1, L):
                                    tr = trs[l - 1]
                                    RU = tr.down(s[l - 1][0])
                                    tau = fas_tau(levels[l - 1], levels[l], tr, s[l - 1][0], s[l - 1][2])
                                    s[l] = [RU, s[l][1], tau]
                                    if l < L - 1:
                                        for _ in range(nu):
                                            s[l][0] = levels[l].sweep(*s[l])
                                s[L - 1][1] = chain[L - 1].copy() if w == 0 else coarse_term
                                for _ in range(nu):
                                    s[L - 1][0] = levels[L - 1].sweep(*s[L - 1])
                                coarse_term = s[L - 1][0][-1].copy()
                                for l in range(L - 2, -1, -1):
                                    tr = trs[l]
                                    RU = tr.down(s[l][0])
                                    s[l][0] = s[l][0] + tr.up(s[l + 1][0] - RU)
                                    if 0 < l < L - 1:
                                        for _ in range(nu):
                                            s[l][0] = levels[l].sweep(*s[l])
                        for l in range(nrecv):  # _publish
                            new_msgs[l][w] = s[l][0][-1].copy()
                        res = fine.res_norm(*s[0])
                        resid[w] = res
                        if not np.isfinite(res) or res > 10.0 * lowest[w]:
                            diverged = True
                        lowest[w] = min(lowest[w], max(res, 1e-300))
                        iters[w] = k
                except OracleSolverError:
                    diverged = True
                msgs = new_msgs
                if diverged:
                    break
                if np.all(resid <= thr):
                    break
            else:
                diverged = True
        rep.inner_iterations.append(int(iters.max()))
        rep.residual_history.append(float(np.max(resid)))
        for w in range(P):
            out[start + w] = st[w][0][0]
        if diverged:
            ok = False
            rep.diverged = True
            break
        u_start = st[P - 1][0][0][-1].copy()
    rep.converged = ok and not rep.diverged
    rep.iterations = max(rep.inner_iterations) if rep.inner_iterations else 0
    rep.wall_time = time.perf_counter() - t0
    return out.ravel(), rep
