"""World-size-2 gloo tests of the sharded PFASST schedule (timeslab.run_windows).

Each rank owns half of every window's workers; fine terminals cross ranks
lagged one iteration, the coarsest terminal is forwarded serially within the
iteration, convergence is a max-allreduce.  With the oracle's per-worker
numerics the sharded run must equal the serial oracle bitwise, with the same
per-window iteration counts — the schedule the GPU ranks run over NCCL.
"""

import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = Path(__file__).resolve().parent
REPO = HERE.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    from oracle import paradiff_oracle as O

    if name == "heat_L2":
        lv, trs = O.fem_pfasst_levels(3, 32, 1.0, 1.0 / 8, 0.0, 2)
        x = np.linspace(0, 1, 33)
        u0 = sum(a * np.cos(k * np.pi * x) for k, a in ((1, 1.0), (3, 2.0), (4, 3.0)))
        return lv, trs, 1, u0, 8, 4, 1e-10
    if name == "heat_L3":
        lv, trs = O.fem_pfasst_levels(2, 32, 1.0, 1.0 / 8, 0.0, 3)
        x = np.linspace(0, 1, 33)
        u0 = sum(a * np.cos(k * np.pi * x) for k, a in ((1, 1.0), (3, 2.0), (4, 3.0)))
        return lv, trs, 1, u0, 8, 8, 1e-10
    if name == "mono_diverge":
        lv, trs = O.fem_pfasst_levels(4, 128, 10.0, 0.5, 5.0, 2, "imex")
        x = np.linspace(0, 10, 129)
        return lv, trs, 1, 2.0 * np.exp(-(((x - 5.0) / 0.1) ** 2)), 4, 4, 1e-9
    raise KeyError(name)


def _worker(rank, size, port, name, outdir):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from paper_2006_12883_b200.timeslab import TorchComm, run_windows
    from pd_oracle_engine import OracleEngine

    lv, trs, nu, u0, Nt, P, tol = _case(name)
    eng = OracleEngine(lv, trs, nu, u0, Nt, P, rank, size)
    rep = run_windows(eng, TorchComm(), Nt, P, tol, tol, 150)
    local = torch.from_numpy(eng.out.ravel().copy())
    parts = [torch.zeros_like(local) for _ in range(size)]
    dist.all_gather(parts, local)
    if rank == 0:
        full = sum(p.numpy() for p in parts)  # each rank fills only its own steps
        np.save(Path(outdir) / "x.npy", full)
        Path(outdir, "rep.json").write_text(json.dumps(
            {"its": rep.iterations, "inner": rep.inner_iterations, "conv": rep.converged,
             "div": rep.diverged, "hist": rep.residual_history}))
    dist.destroy_process_group()


def _run(name, tmp_path, size=2):
    mp.start_processes(_worker, args=(size, _free_port(), name, str(tmp_path)), nprocs=size,
                       join=True, start_method="spawn")
    return np.load(tmp_path / "x.npy"), json.loads((tmp_path / "rep.json").read_text())


@pytest.mark.parametrize("name", ["heat_L2", "heat_L3"])
def test_sharded_schedule_equals_serial(tmp_path, name):
    from oracle import paradiff_oracle as O

    x, rep = _run(name, tmp_path)
    lv, trs, nu, u0, Nt, P, tol = _case(name)
    xs, reps = O.pfasst(lv, trs, nu, u0, Nt, P, tol_rel=tol, tol_abs=tol)
    assert rep["conv"] and reps.converged
    assert rep["inner"] == reps.inner_iterations
    assert rep["its"] == reps.iterations
    np.testing.assert_array_equal(x, xs)
    np.testing.assert_allclose(rep["hist"], reps.residual_history, rtol=0, atol=0)


def test_sharded_divergence_agreed_by_all_ranks(tmp_path):
    x, rep = _run("mono_diverge", tmp_path)
    assert rep["div"] and not rep["conv"]


def test_worker_partition_rule():
    from paper_2006_12883_b200.timeslab import worker_range
    from paper_2006_12883_b200.errors import ConfigurationError

    assert [worker_range(8, r, 4) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ConfigurationError):
        worker_range(6, 0, 4)
