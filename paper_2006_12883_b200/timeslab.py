"""Time-slab parallel PFASST driver: windows of P time steps sharded over G ranks.

The reference runs the P steps of a window as P threads of one process
(pfasst.py:369-583).  Here rank g of G owns the contiguous workers
[g*P/G, (g+1)*P/G) of every window (one process per GPU).  Per iteration the
only data crossing GPUs is what the reference passes between threads:

* the fine terminal value of each rank's last worker (S doubles per
  receiving level, LAGGED one iteration: pfasst.py:415-423, 465-473) —
  one send to the successor rank;
* the coarsest terminal value, forwarded serially through the ranks WITHIN
  the iteration (pfasst.py:441-455) — recv from g-1, local chain, send to g+1;
* one max-allreduce of [max residual, failure flag] for the all-converged /
  any-diverged decision (pfasst.py:471-493);
* at the window end the last rank's fine terminal is broadcast as the next
  window's start value (pfasst.py:583).

Compute is delegated to an engine (GpuPfasstEngine below runs the native
kernels; tests plug a CPU engine built on the oracle to check this schedule
with torch.distributed/gloo at world size 2).  With G=1 the driver is the
single-GPU PFASST path used by pfasst_run.
"""

from __future__ import annotations

import sys

import os

import time

import numpy as np

from .errors import ConfigurationError, SolverError
from .report import SolveReport


class LocalComm:
    """G = 1: no communication."""

    rank, size = 0, 1

    def send(self, t, dst):  # pragma: no cover - never called with one rank
        raise RuntimeError("no peers")

    recv = send

    def exchange_next(self, send_tensors, recv_tensors):
        return

    def allreduce_max(self, values):
        return np.asarray(values, dtype=np.float64)

    def broadcast(self, t, src):
        return t


class TorchComm:
    """torch.distributed point-to-point + collectives (nccl for CUDA, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def _g(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def send(self, t, dst):
        self.dist.send(t, self._g(dst), group=self.group)

    def recv(self, t, src):
        self.dist.recv(t, self._g(src), group=self.group)

    def exchange_next(self, send_tensors, recv_tensors):
        """send to rank+1 / receive from rank-1 (batched, deadlock-free)."""
        dist = self.dist
        ops = []
        if self.rank + 1 < self.size:
            ops += [dist.P2POp(dist.isend, t, self._g(self.rank + 1), self.group)
                    for t in send_tensors]
        if self.rank > 0:
            ops += [dist.P2POp(dist.irecv, t, self._g(self.rank - 1), self.group)
                    for t in recv_tensors]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce_max(self, values):
        import torch

        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor(np.asarray(values, dtype=np.float64), device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()

    def broadcast(self, t, src):
        self.dist.broadcast(t, self._g(src), group=self.group)
        return t


_PROFILE = {} if os.environ.get("PD_PFASST_PROFILE") else None


def phase_profile() -> dict:
    """Seconds per driver phase accumulated under PD_PFASST_PROFILE (diagnostics)."""
    return dict(_PROFILE or {})


def worker_range(P: int, rank: int, size: int) -> tuple[int, int]:
    if P % size != 0:
        raise ConfigurationError(f"workers per window ({P}) must be a multiple of ranks ({size})")
    n = P // size
    return rank * n, (rank + 1) * n


def run_windows(engine, comm, Nt: int, P: int, tol_rel: float, tol_abs: float,
                max_iters: int) -> SolveReport:
    """Windowed pipelined PFASST (pfasst.py:509-587) over ranks; engine holds local workers."""
    if P < 1 or P > Nt:
        raise ConfigurationError(f"worker count must be in [1, Nt={Nt}], got {P}")
    if Nt % P != 0:
        raise ConfigurationError(f"worker count {P} must divide Nt={Nt}")
    g, G = comm.rank, comm.size
    L = engine.num_levels
    report = SolveReport()
    t0 = time.perf_counter()
    converged = True
    for start in range(0, Nt, P):
        res = engine.setup_window(start)
        r0 = float(comm.allreduce_max([float(np.max(res)) if res.size else 0.0])[0])
        threshold = max(tol_abs, tol_rel * engine.window_r0())
        lowest = np.maximum(res, 1e-300)
        iters = 0
        diverged = False
        if r0 > threshold:
            halo_in = engine.halo_buffers()
            for k in range(1, max_iters + 1):
                # a SolverError on one rank must not strand its peers inside a
                # send/recv: compute steps are skipped after a failure, every
                # communication step still happens, and the failure is agreed
                # on through the allreduce (the reference's stop event).
                state = {"failed": False}

                def step(fn, *a):
                    if state["failed"]:
                        return None
                    try:
                        if _PROFILE is not None:  # PD_PFASST_PROFILE: device time per phase
                            import torch

                            torch.cuda.synchronize()
                            t_0 = time.perf_counter()
                            out = fn(*a)
                            torch.cuda.synchronize()
                            _PROFILE[fn.__name__] = _PROFILE.get(fn.__name__, 0.0) + (
                                time.perf_counter() - t_0)
                            return out
                        return fn(*a)
                    except SolverError as e:
                        state["failed"] = True
                        # global index of the first failing worker (0 when unknown)
                        state["worker"] = min(state.get("worker", 1 << 30),
                                              max(int(getattr(e, "worker", 0)), 0))
                        if os.environ.get("PD_PFASST_VERBOSE"):
                            print(f"[pfasst] window iteration {k}: {fn.__name__}: {e}",
                                  file=sys.stderr, flush=True)
                        return None

                if k > 1:
                    step(engine.receive, halo_in if g > 0 else None)
                step(engine.fine_sweeps)
                if L > 1:
                    step(engine.coarse_down)
                    u0c = engine.coarse_start_buffer()
                    if g == 0:
                        step(engine.load_coarse_start, u0c)
                    else:
                        comm.recv(u0c, g - 1)
                    step(engine.coarse_chain, u0c)
                    if g + 1 < G:
                        comm.send(engine.coarse_last_buffer(), g + 1)
                    step(engine.coarse_up)
                out = step(engine.publish)
                if out is None:
                    res = np.full(engine.local_workers, np.nan)
                else:
                    res = out
                comm.exchange_next(engine.halo_out_buffers(), halo_in)
                bad = (~np.isfinite(res)) | (res > 10.0 * lowest)
                lowest = np.minimum(lowest, np.maximum(res, 1e-300))
                red = comm.allreduce_max([
                    float(np.max(res)) if np.all(np.isfinite(res)) else np.inf,
                    1.0 if (state["failed"] or bad.any()) else 0.0,
                    1.0 if np.any(~(res <= threshold)) else 0.0,
                    -float(state["worker"]) if state["failed"] else -np.inf])
                # pfasst.py:471-507: a worker counts iteration k once it has published;
                # after a SolverError in worker f the workers before f still finish k,
                # f and its successors (stranded in the coarse chain) stay at k - 1
                iters = k if (red[3] == -np.inf or -red[3] > 0) else k - 1
                res_max = float(red[0])
                if red[1] > 0:
                    diverged = True
                    break
                if red[2] == 0.0:
                    break
            else:
                diverged = True
        else:
            res_max = r0
        report.inner_iterations.append(int(iters))
        report.residual_history.append(float(res_max))
        engine.store_window(start)
        if diverged:
            converged = False
            report.diverged = True
            break
        engine.set_window_start(comm.broadcast(engine.last_fine_terminal(), G - 1))
    report.converged = converged and not report.diverged
    report.iterations = max(report.inner_iterations) if report.inner_iterations else 0
    report.wall_time = time.perf_counter() - t0
    return report
