"""Time-slab sharded space-time multigrid over G ranks (MG half).

The reference runs one process (multigrid.py:197-305); its block-Jacobi
smoother already cuts every level into P contiguous time-slab partitions
(linalg.py:152-189).  Here rank g of G owns partitions [g*P/G, (g+1)*P/G) on
every level: its rows of each Galerkin operator, of the transfers and of the
ILU(0) factors.  What crosses ranks is exactly what the operator couples:

* every operator application needs the predecessor rank's last rows of the
  vector (SMG/SMMG levels couple a time step only to the previous step's last
  node: S_l values, a one-way halo) — one send to g+1 / recv from g-1;
* GMRES dot products and norms — one sum-allreduce each (MGS order kept);
* the coarsest level is solved redundantly after an allgather of its rhs;
* the outer residual norm — one sum-allreduce per cycle.

The smoother's block-Jacobi preconditioner needs nothing: partitions never
straddle ranks.  Transfers of SMG/SMMG are block diagonal in time (checked at
setup).  STMG couples coarse steps to step +1 and is not sharded (rejected).

Compute is delegated to an engine: `DeviceEngine` (native kernels on the
rank's GPU: CSR SpMV, wavefront/level ILU(0), dense LU) or, in the tests, a
CPU engine on the oracle — the same schedule is checked with gloo at world
size 2 (tests/test_mg_sharded_gloo.py).  The GMRES below restates
linalg.py:215-311 (MGS, Givens, happy breakdown 1e-14*max(1,beta), true
residual per restart, divergence at 10x the lowest restart residual) with
host-side Hessenberg arithmetic; with G = 1 it reproduces the serial
solver's iteration counts (tests).
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
import scipy.sparse as sp

from .errors import ConfigurationError, SolverError
from .report import SolveReport


# ---------------------------------------------------------------- layout
def rank_rows(n: int, partitions: int, rank: int, size: int) -> tuple[int, int]:
    """Rows of `rank`: block-Jacobi partitions [rank*P/G, (rank+1)*P/G) of size n//P
    (linalg.py:166-170); requires P % G == 0 and n % P == 0 (equal partitions)."""
    if partitions % size != 0:
        raise ConfigurationError(f"partitions ({partitions}) must be a multiple of ranks ({size})")
    if n % partitions != 0:
        raise ConfigurationError(f"level size {n} must be divisible by partitions ({partitions})")
    per = partitions // size
    blk = n // partitions
    return rank * per * blk, (rank + 1) * per * blk


class LevelShard:
    """Rank-local pieces of one level: operator rows with their halo columns."""

    def __init__(self, A: sp.csr_matrix, r0: int, r1: int, prev_r0: int | None):
        A = sp.csr_matrix(A)
        rows = A[r0:r1]
        if rows.nnz and rows.indices.max() >= r1:
            raise ConfigurationError("operator couples a rank to later time slabs (not sharded)")
        cmin = int(rows.indices.min()) if rows.nnz else r0
        cmin = min(cmin, r0)
        if prev_r0 is not None and cmin < prev_r0:
            raise ConfigurationError("operator halo spans more than one rank")
        if prev_r0 is None and cmin < r0:
            raise ConfigurationError("first rank's rows reference earlier columns")
        self.r0, self.r1, self.halo = r0, r1, r0 - cmin
        self.A_ext = sp.csr_matrix(rows[:, cmin:r1])  # columns: [halo | own]
        self.A_own = sp.csr_matrix(rows[:, r0:r1])    # for the block-Jacobi factors


# ---------------------------------------------------------------- communication
class Comm:
    """torch.distributed collectives for the sharded cycle (any backend); G=1: local."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.size = self.dist.get_world_size(group) if self.dist else 1
        self.device = device

    def _g(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def allreduce_sum(self, value: float) -> float:
        if self.size == 1:
            return float(value)
        import torch

        dev = "cpu" if self._host_staged() else self.device
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    def allreduce_tensor_(self, t) -> None:
        """In-place sum of a (device) tensor over the ranks: asynchronous on the stream
        with NCCL; staged through the host with gloo (CPU tests only)."""
        if self.size == 1:
            return
        if self._host_staged() and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)

    def _host_staged(self) -> bool:
        """gloo moves host tensors only: CUDA vectors are staged through the host."""
        return self.dist.get_backend(self.group) == "gloo"

    def shift_next(self, send_t, recv_t):
        """send_t to rank+1, recv_t from rank-1 (either may be None)."""
        if self.size == 1:
            return
        dist = self.dist
        stage = self._host_staged()
        s_t = send_t.cpu() if (stage and send_t is not None and send_t.is_cuda) else send_t
        r_t = recv_t.cpu() if (stage and recv_t is not None and recv_t.is_cuda) else recv_t
        ops = []
        if s_t is not None and self.rank + 1 < self.size:
            ops.append(dist.P2POp(dist.isend, s_t, self._g(self.rank + 1), self.group))
        if r_t is not None and self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, r_t, self._g(self.rank - 1), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if r_t is not recv_t and recv_t is not None and self.rank > 0:
            recv_t.copy_(r_t)

    def allgather(self, t, counts):
        """Concatenate every rank's 1D piece (sizes `counts`, same on all ranks)."""
        if self.size == 1:
            return t
        import torch

        m = max(counts)
        dev = "cpu" if self._host_staged() else t.device
        pad = torch.zeros(m, dtype=t.dtype, device=dev)
        pad[: t.numel()] = t
        parts = [torch.empty_like(pad) for _ in range(self.size)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)]).to(t.device)


# ---------------------------------------------------------------- engines
class DeviceEngine:
    """Native kernels on this rank's GPU (torch CUDA tensors as vectors)."""

    def __init__(self):
        from . import _native as N

        self.N = N
        self.ctx = N.context()

    def operator(self, A):
        from .linalg import DeviceCsr

        return DeviceCsr(A, self.ctx)

    def preconditioner(self, A_own, nblocks: int, grid=None, m: int = 0):
        from .linalg import BlockJacobiPrecond, Ilu0

        pre = BlockJacobiPrecond(A_own, nblocks) if nblocks > 1 else Ilu0(A_own)
        if grid is not None:
            pre.set_wavefront(m, grid[0], grid[1])  # same structured sweeps as the serial path
        return pre

    def coarse_solver(self, A):
        from .linalg import DenseLU

        return DenseLU(A)

    def slab_stencil(self, system, shard):
        """K1 for the rank's rows of the fine operator when they are whole time steps that
        couple to exactly the previous step's last node grid (SMG/SMMG level 0)."""
        import os

        S = system.space.mesh.ndof
        per_step = system.tableau.M * S
        rows = shard.r1 - shard.r0
        if (os.environ.get("PD_SHARDED_NO_K1") == "1" or rows % per_step or shard.r0 % per_step
                or shard.halo not in (0, S) or (shard.halo == 0) != (shard.r0 == 0)
                or system.gamma != 0.0):
            return None
        try:
            return _SlabStencilOp(system, rows // per_step, shard.halo, self.ctx)
        except ConfigurationError:
            return None

    def smoother(self, n: int, nu: int):
        """Device-resident GMRES(nu) steps driven by the sharded cycle (pd_gms_*)."""
        return _DeviceSmoother(self, n, nu)

    def vec(self, a):
        return self.N.to_device(a, self.ctx)

    def zeros(self, n):
        return self.N.zeros(n, self.ctx)

    def apply(self, op, x):
        return op.matvec_dev(x)

    def residual(self, op, b, x):
        return op.matvec_dev(x, mode=1, b=b)  # b - A x

    def precond(self, pre, v):
        return pre.solve_dev(v)

    def coarse(self, lu, b):
        return lu.solve(b)

    def dot(self, a, b) -> float:
        # the library's own deterministic reduction (no torch / cuBLAS ddot on the path)
        return self.N.dot(a.contiguous(), b.contiguous(), self.ctx)

    def size(self, a) -> int:
        return int(a.numel())

    def cat(self, a, b):
        import torch

        return torch.cat([a, b])

    def slice_tail(self, x, k):
        return x[x.numel() - k:].contiguous()

    def empty(self, n):
        return self.N.empty(n, self.ctx)

    def host(self, x):
        return x.cpu().numpy()

    def comm_tensor(self, x):
        return x


class _SlabStencilOp:
    """Level 0 of a rank's time slab applied matrix-free (K1, pd_stop_apply): bitwise the
    slab's CSR rows.  Takes the extended vector [halo | own] the CSR operator takes — the
    halo (the previous slab's last node grid) is passed to the kernel by pointer."""

    def __init__(self, system, steps: int, halo: int, ctx):
        from . import _native as N

        self.N, self.ctx, self.halo = N, ctx, int(halo)
        self.handle = system.stencil_operator_handle(ctx, Nt=steps)
        self.n = steps * system.tableau.M * system.space.mesh.ndof

    def matvec_dev(self, x_ext, out=None, mode=0, b=None):
        import ctypes

        N = self.N
        self.ctx.sync_stream()
        out = N.empty(self.n, self.ctx) if out is None else out
        own = x_ext[self.halo:] if self.halo else x_ext
        N.call("pd_stop_apply", self.handle, N.ptr(own), N.ptr(out), int(mode),
               N.ptr(b) if b is not None else ctypes.c_void_p(),
               N.ptr(x_ext) if self.halo else ctypes.c_void_p())
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.N.load_library().pd_stop_destroy(self.handle)
        except Exception:
            pass


class _DeviceSmoother:
    """One level's externally driven smoother engine: Krylov vectors, Hessenberg/Givens
    recurrence and stopping test on the device; this class only wraps pointers."""

    def __init__(self, eng: "DeviceEngine", n: int, nu: int):
        import ctypes

        self.eng, self.n, self.nu = eng, int(n), int(nu)
        N = eng.N
        h = ctypes.c_void_p()
        N.call("pd_gms_create", eng.ctx.handle, self.n, self.nu, ctypes.byref(h))
        self.handle = h
        d = ctypes.c_void_p()
        N.call("pd_gms_dots", self.handle, ctypes.byref(d))
        self.dots = N.view(d, self.nu + 2, eng.ctx)  # dots[i]: reduced over ranks after pass i
        self.norm2 = N.zeros(1, eng.ctx)
        self._views = {}

    def init(self, r):
        N = self.eng.N
        N.call("pd_dot_dev", self.eng.ctx.handle, N.ptr(r), N.ptr(r), self.n, N.ptr(self.norm2))
        return self.norm2  # the caller sums it over the ranks, then calls start()

    def start(self, r):
        self._r = r  # the engine reads r on its first step: keep it alive
        N = self.eng.N
        N.call("pd_gms_init", self.handle, N.ptr(r), N.ptr(self.norm2))

    def begin(self, j: int):
        import ctypes

        N = self.eng.N
        v, z, w = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        N.call("pd_gms_begin", self.handle, int(j), ctypes.byref(v), ctypes.byref(z),
               ctypes.byref(w))
        views = self._views.get(j)
        if views is None:  # the engine's buffers never move: wrap each pointer once
            n1 = max(self.n, 1)
            views = self._views[j] = tuple(N.view(p, n1, self.eng.ctx)[:self.n] for p in (v, z, w))
        return views

    def mgs_pass(self, i: int):
        self.eng.N.call("pd_gms_mgs_pass", self.handle, int(i))
        return self.dots[i:i + 1]

    def end(self, slot: int):
        self.eng.N.call("pd_gms_end", self.handle, int(slot))

    def apply(self, x):
        self.eng.N.call("pd_gms_apply", self.handle, self.eng.N.ptr(x))

    def error(self) -> int:
        import ctypes

        e = ctypes.c_int()
        self.eng.N.call("pd_gms_error", self.handle, ctypes.byref(e))
        return int(e.value)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.eng.N.load_library().pd_gms_destroy(self.handle)
        except Exception:
            pass


# ---------------------------------------------------------------- the solver
class ShardedMultigrid:
    """SMG/SMMG V-cycles over G ranks; same interface as MultigridHierarchy.solve."""

    def __init__(self, mats, transfers, nu: int, partitions: int, comm: Comm, engine,
                 restart: int = 30, smooth_solves: int = 1, grids=None, node_counts=None,
                 system=None):
        if nu < 1:
            raise ConfigurationError("need at least one smoothing iteration")
        if len(transfers) != len(mats) - 1:
            raise ConfigurationError("need one transfer set per level transition")
        self.comm, self.eng = comm, engine
        self.nu, self.restart, self.smooth_solves = nu, restart, smooth_solves
        self.partitions = partitions
        g, G = comm.rank, comm.size
        L = len(mats)
        self.shards, self.ops, self.pres, self.R, self.P = [], [], [], [], []
        self.halo_send = []  # per level: rows rank g sends to g+1
        for l in range(L - 1):
            n = mats[l].shape[0]
            spans = [rank_rows(n, partitions, r, G) for r in range(G)]
            r0, r1 = spans[g]
            sh = LevelShard(mats[l], r0, r1, spans[g - 1][0] if g > 0 else None)
            nxt = (LevelShard(mats[l], *spans[g + 1], r0).halo if g + 1 < G else 0)
            self.shards.append(sh)
            self.halo_send.append(nxt)
            op = None
            if l == 0 and system is not None and hasattr(engine, "slab_stencil"):
                op = engine.slab_stencil(system, sh)  # matrix-free K1 on the slab, or None
            self.ops.append(op if op is not None else engine.operator(sh.A_ext))
            grid = grids[l] if grids is not None else None
            m = node_counts[l] if node_counts is not None else 0
            self.pres.append(engine.preconditioner(sh.A_own, partitions // G, grid, m))
            # transfers: block diagonal in time across ranks
            nc = mats[l + 1].shape[0]
            c0, c1 = rank_rows(nc, partitions, g, G)
            R, P = (sp.csr_matrix(t) for t in transfers[l])
            Rl, Pl = R[c0:c1], P[r0:r1]
            if (Rl.nnz and (Rl.indices.min() < r0 or Rl.indices.max() >= r1)) or \
                    (Pl.nnz and (Pl.indices.min() < c0 or Pl.indices.max() >= c1)):
                raise ConfigurationError("transfers couple time slabs of different ranks "
                                         "(STMG is not sharded)")
            self.R.append(engine.operator(Rl[:, r0:r1]))
            self.P.append(engine.operator(Pl[:, c0:c1]))
        nL = mats[-1].shape[0]
        self.coarse_counts = [rank_rows(nL, partitions, r, G) for r in range(G)]
        self.coarse_range = self.coarse_counts[g]
        self.coarse_counts = [b - a for a, b in self.coarse_counts]
        self.coarse_lu = engine.coarse_solver(mats[-1])
        self.sizes = [m.shape[0] for m in mats]
        # device engines keep the smoother's GMRES on the device (no host sync per dot);
        # the CPU engine of the gloo tests runs the host restatement below
        self.gms = None
        if hasattr(engine, "smoother") and os.environ.get("PD_SHARDED_HOST_GMRES") != "1":
            self.gms = [engine.smoother(sh.r1 - sh.r0, min(self.nu, self.restart))
                        for sh in self.shards]

    # ---- distributed vector primitives ------------------------------------
    def _dot(self, a, b) -> float:
        return self.comm.allreduce_sum(self.eng.dot(a, b))

    def _norm(self, a) -> float:
        return math.sqrt(max(self._dot(a, a), 0.0))

    def _ext(self, l, x):
        """[halo from rank g-1 | own] for the level-l operator."""
        sh = self.shards[l]
        k = self.halo_send[l]
        send = self.eng.comm_tensor(self.eng.slice_tail(x, k)) if k else None
        recv = self.eng.empty(sh.halo) if sh.halo else None
        self.comm.shift_next(send, self.eng.comm_tensor(recv) if recv is not None else None)
        return self.eng.cat(recv, x) if recv is not None else x

    def _apply(self, l, x):
        return self.eng.apply(self.ops[l], self._ext(l, x))

    def _residual(self, l, b, x):
        return self.eng.residual(self.ops[l], b, self._ext(l, x))

    # ---- GMRES smoother (linalg.py:215-311) --------------------------------
    def _gmres(self, l, b, tol_rel, tol_abs, restart, max_it):
        eng, pre = self.eng, self.pres[l]
        x = eng.zeros(eng.size(b))
        # x0 = 0: the reference's r = b - A@0 equals b exactly (finite b)
        r = b
        beta = self._norm(r)
        if not np.isfinite(beta):
            raise SolverError("non-finite initial residual")
        thr = max(tol_abs, tol_rel * beta)
        if beta <= thr:
            return x
        lowest, total = beta, 0
        restart = max(1, min(restart, self.sizes[l]))
        while True:
            V = [r / beta]
            H = np.zeros((restart + 1, restart))
            cs, sn = np.empty(restart), np.empty(restart)
            gvec = np.zeros(restart + 1)
            gvec[0] = beta
            j = -1
            for j in range(restart):
                w = self._apply(l, eng.precond(pre, V[j]))
                for i in range(j + 1):
                    hij = self._dot(w, V[i])
                    H[i, j] = hij
                    w = w - hij * V[i]  # python floats: no numpy/torch scalar mixing
                hn = self._norm(w)
                H[j + 1, j] = hn
                happy = hn <= 1e-14 * max(1.0, beta)
                if not happy:
                    V.append(w / hn)
                for i in range(j):
                    t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                    H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                    H[i, j] = t
                d = math.hypot(H[j, j], H[j + 1, j])
                if d == 0.0:
                    cs[j], sn[j] = 1.0, 0.0
                else:
                    cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
                H[j, j] = d
                H[j + 1, j] = 0.0
                gvec[j + 1] = -sn[j] * gvec[j]
                gvec[j] = cs[j] * gvec[j]
                res = abs(gvec[j + 1])
                if not np.isfinite(res):
                    raise SolverError("non-finite residual in GMRES iteration")
                total += 1
                if res <= thr or happy or total >= max_it:
                    break
            k = j + 1
            y = _back_substitute(H[:k, :k], gvec[:k])
            u = V[0] * float(y[0])
            for i in range(1, k):
                u = u + V[i] * float(y[i])
            x = x + eng.precond(pre, u)
            r = self._residual(l, b, x)
            beta = self._norm(r)
            if not np.isfinite(beta):
                raise SolverError("non-finite residual in GMRES restart")
            lowest = min(lowest, beta)
            if beta <= thr or total >= max_it or beta > 10.0 * lowest:
                return x

    # ---- V-cycle (multigrid.py:243-273) ------------------------------------
    def _smooth_device(self, l, b, x):
        """multigrid.py:243-256 with the GMRES(nu) of linalg.py:215-311 on the device: per
        Arnoldi step the rank-local preconditioner, the sharded operator (one halo
        send/recv), j + 2 MGS passes with a one-double all-reduce each; nothing is read
        back to the host.  x is updated in place."""
        eng, sm, pre = self.eng, self.gms[l], self.pres[l]
        nu = sm.nu
        for _ in range(self.smooth_solves):
            r = self._residual(l, b, x)
            self.comm.allreduce_tensor_(sm.init(r))
            sm.start(r)
            for j in range(nu):
                v, z, w = sm.begin(j)
                pre.solve_dev(v, out=z)
                self.ops[l].matvec_dev(self._ext(l, z), out=w)
                for i in range(j + 2):
                    self.comm.allreduce_tensor_(sm.mgs_pass(i))
                sm.end(j)
            sm.apply(x)
        return x

    def _smooth(self, l, b, x):
        if self.gms is not None:
            return self._smooth_device(l, b, x)
        for _ in range(self.smooth_solves):
            r = self._residual(l, b, x)
            x = x + self._gmres(l, r, 1e-13, 0.0, min(self.nu, self.restart), self.nu)
        return x

    def _cycle(self, l, b, x):
        L = len(self.sizes)
        if l == L - 1:
            full = self.comm.allgather(self.eng.comm_tensor(b), self.coarse_counts)
            xc = self.eng.coarse(self.coarse_lu, full)
            a, c = self.coarse_range
            return xc[a:c]
        x = self._smooth(l, b, x)
        r = self._residual(l, b, x)
        rc = self.eng.apply(self.R[l], r)
        x = x + self.eng.apply(self.P[l], self._cycle(l + 1, rc, self.eng.zeros(self.eng.size(rc))))
        return self._smooth(l, b, x)

    def vcycle(self, b, x):
        out = self._cycle(0, b, x)
        if not np.isfinite(self._norm(out)):
            raise SolverError("V-cycle produced non-finite values")
        if self.gms is not None:  # the device smoothers' error codes, once per cycle
            texts = {1: "non-finite initial residual", 2: "non-finite residual in GMRES iteration",
                     3: "non-finite residual in GMRES restart"}
            for sm in self.gms:
                code = sm.error()
                if code:
                    raise SolverError(texts.get(code, f"GMRES error {code}"))
        return out

    def solve(self, b, x0=None, tol_rel: float = 1e-9, tol_abs: float = 1e-9,
              max_cycles: int = 1000):
        """multigrid.py:275-305 on this rank's rows of b (x0 likewise)."""
        t0 = time.perf_counter()
        eng = self.eng
        b = eng.vec(b)
        x = eng.zeros(self.shards[0].r1 - self.shards[0].r0) if x0 is None else eng.vec(x0)
        if self.gms is not None and x0 is not None:
            x = x.clone()  # the device smoother updates x in place
        res = self._norm(self._residual(0, b, x))
        rep = SolveReport(residual_history=[res])
        thr = max(tol_abs, tol_rel * res)
        lowest = res
        while res > thr:
            if rep.iterations >= max_cycles:
                rep.diverged = True
                break
            x = self.vcycle(b, x)
            res = self._norm(self._residual(0, b, x))
            rep.iterations += 1
            rep.residual_history.append(res)
            if not np.isfinite(res) or res > 10.0 * lowest:
                rep.diverged = True
                break
            lowest = min(lowest, res)
        rep.converged = res <= thr
        rep.wall_time = time.perf_counter() - t0
        return x, rep


def _back_substitute(U, g):
    """Upper-triangular solve (scipy solve_triangular, linalg.py:296)."""
    import scipy.linalg

    return scipy.linalg.solve_triangular(U, g, lower=False)


def build_sharded_hierarchy(hierarchy, comm: Comm | None = None, engine=None):
    """Shard a built MultigridHierarchy (its Galerkin matrices and transfers) over
    the ranks of `comm`; every rank passes the same global hierarchy."""
    comm = comm or Comm()
    engine = engine or DeviceEngine()
    if hierarchy.strategy == "STMG":
        raise ConfigurationError("STMG couples coarse steps to later steps: not sharded")
    transfers = [(t.restriction, t.prolongation) for t in hierarchy.transfers]
    grids = getattr(hierarchy, "grids", None)
    nodes = [d.m for d in hierarchy.dims]
    return ShardedMultigrid(hierarchy.matrices, transfers, hierarchy.nu, hierarchy.partitions,
                            comm, engine, hierarchy.restart, hierarchy.smooth_solves,
                            grids=grids, node_counts=nodes,
                            system=getattr(hierarchy, "_system", None))
