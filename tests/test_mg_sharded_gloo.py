"""Sharded space-time multigrid (mg_sharded.py): the schedule on CPU ranks.

Rank g owns block-Jacobi partitions [g*P/G, (g+1)*P/G) of every level; operator
applications exchange the predecessor rank's last time-step rows, GMRES dots
are sum-allreduced, the coarsest level is solved redundantly after an
allgather.  With the oracle's per-rank numerics (tests/pd_mg_cpu_engine.py)
the sharded solve must match the serial oracle V-cycles: equal cycle counts
and a relative L2 difference <= 1e-10 (dot products are split across ranks,
so rounding differs from one numpy dot over the whole vector).
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
    """(oracle multigrid, rhs, partitions, tol) of a reduced BASELINE config."""
    from oracle import paradiff_oracle as O
    from paper_2006_12883_b200 import problems as PB

    cfg = PB.baseline_config({"c2": "C2", "c4": "C4", "c1": "C1"}[name],
                             n={"c2": 15, "c4": 7, "c1": None}[name],
                             Nt={"c2": 8, "c4": 4, "c1": 16}[name])
    ops = PB.fd_space(cfg.spec)
    s = O.OSystem(O.tableau(cfg.M), ops.Kh, ops.lumped_diagonal, cfg.Nt, cfg.T, 0.0, cfg.u0())
    L = 3 if cfg.spec.dim > 1 else 4
    specs = [cfg.spec]
    for _ in range(L - 1):
        specs.append(specs[-1].coarse())
    dims = [O.Dims(cfg.Nt, cfg.M, sp_.ndof) for sp_ in specs]
    pairs = [PB.fd_transfers(specs[l]) for l in range(L - 1)]
    parts = 4
    mg = O.OMultigrid(s.global_matrix(), dims, O.composite_transfers(dims, pairs), 2, parts)
    return mg, s.rhs(), parts, 1e-10


def _sharded(mg, parts, comm):
    from paper_2006_12883_b200.mg_sharded import ShardedMultigrid
    from pd_mg_cpu_engine import CpuEngine

    return ShardedMultigrid(mg.mats, mg.transfers, mg.nu, parts, comm, CpuEngine())


def _worker(rank, size, port, name, outdir):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from paper_2006_12883_b200.mg_sharded import Comm

    mg, b, parts, tol = _case(name)
    smg = _sharded(mg, parts, Comm())
    r0, r1 = smg.shards[0].r0, smg.shards[0].r1
    x, rep = smg.solve(b[r0:r1], tol_rel=tol, tol_abs=tol)
    full = torch.zeros(b.size, dtype=torch.float64)
    full[r0:r1] = x
    dist.all_reduce(full)
    if rank == 0:
        np.save(Path(outdir) / "x.npy", full.numpy())
        Path(outdir, "rep.json").write_text(json.dumps(
            {"its": rep.iterations, "conv": rep.converged, "hist": rep.residual_history}))
    dist.destroy_process_group()


def _check(x, rep, name):
    mg, b, parts, tol = _case(name)
    xs, reps = mg.solve(b, tol_rel=tol, tol_abs=tol)
    assert rep["conv"] and reps.converged
    assert rep["its"] == reps.iterations
    assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_sharded_mg_two_ranks_matches_serial(tmp_path, name):
    mp.start_processes(_worker, args=(2, _free_port(), name, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    x = np.load(tmp_path / "x.npy")
    rep = json.loads((tmp_path / "rep.json").read_text())
    _check(x, rep, name)


def test_sharded_mg_one_rank_matches_serial():
    from paper_2006_12883_b200.mg_sharded import Comm

    mg, b, parts, tol = _case("c1")
    smg = _sharded(mg, parts, Comm())
    x, rep = smg.solve(b, tol_rel=tol, tol_abs=tol)
    _check(x.numpy(), {"conv": rep.converged, "its": rep.iterations}, "c1")


def test_layout_rules_and_stmg_rejected():
    from oracle import paradiff_oracle as O
    from paper_2006_12883_b200 import problems as PB
    from paper_2006_12883_b200.errors import ConfigurationError
    from paper_2006_12883_b200.mg_sharded import Comm, ShardedMultigrid, rank_rows
    from pd_mg_cpu_engine import CpuEngine

    assert [rank_rows(64, 8, r, 4) for r in range(4)] == [(0, 16), (16, 32), (32, 48), (48, 64)]
    with pytest.raises(ConfigurationError):
        rank_rows(64, 6, 0, 4)
    with pytest.raises(ConfigurationError):
        rank_rows(66, 8, 0, 2)
    # STMG's time-coarsened transfers couple consecutive slabs: refused when sharded
    cfg = PB.baseline_config("C1", Nt=8)
    ops = PB.fd_space(cfg.spec)
    s = O.OSystem(O.tableau(3), ops.Kh, ops.lumped_diagonal, cfg.Nt, cfg.T, 0.0, cfg.u0())
    specs = [cfg.spec, cfg.spec.coarse()]
    dims = [O.Dims(8, 3, specs[0].ndof), O.Dims(4, 3, specs[1].ndof)]
    mg = O.OMultigrid(s.global_matrix(), dims,
                      O.composite_transfers(dims, [PB.fd_transfers(specs[0])]), 2, 2)

    class TwoRanks(Comm):
        def __init__(self):
            self.dist, self.group, self.rank, self.size, self.device = None, None, 0, 2, None

    with pytest.raises(ConfigurationError):
        ShardedMultigrid(mg.mats, mg.transfers, 2, 2, TwoRanks(), CpuEngine())


# ---------------------------------------------------------------- device engine, two ranks
def _dev_worker(rank, size, port, outdir, host_gmres):
    """Two ranks over gloo sharing one GPU (vectors staged through the host by Comm): the
    DeviceEngine with the device-resident smoother (pd_gms_*) or the host-GMRES mirror."""
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if host_gmres:
        os.environ["PD_SHARDED_HOST_GMRES"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=size)
    torch.cuda.set_device(0)
    import paper_2006_12883_b200 as pd
    from paper_2006_12883_b200.mg_sharded import Comm, build_sharded_hierarchy

    cfg = pd.baseline_config("C2", n=31, Nt=8)
    system = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                                pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    h = pd.build_hierarchy(system, "SMG", 3, 3, partitions=4)
    b = system.rhs()
    smg = build_sharded_hierarchy(h, Comm(device=torch.device("cuda", 0)))
    assert (smg.gms is None) == bool(host_gmres)
    from paper_2006_12883_b200.mg_sharded import _SlabStencilOp

    assert isinstance(smg.ops[0], _SlabStencilOp)  # level 0 matrix-free (K1 with a halo)
    r0, r1 = smg.shards[0].r0, smg.shards[0].r1
    x, rep = smg.solve(b[r0:r1], tol_rel=1e-10, tol_abs=1e-10)
    full = torch.zeros(b.size, dtype=torch.float64)
    full[r0:r1] = x.cpu()
    dist.all_reduce(full)
    if rank == 0:
        xs, reps = h.solve(b, tol_rel=1e-10, tol_abs=1e-10)  # the serial device multigrid
        np.save(Path(outdir) / "x.npy", full.numpy())
        np.save(Path(outdir) / "xs.npy", np.asarray(xs))
        Path(outdir, "rep.json").write_text(json.dumps(
            {"its": rep.iterations, "conv": rep.converged, "its_serial": reps.iterations,
             "hist": rep.residual_history, "hist_serial": reps.residual_history}))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("host_gmres", [False, True])
def test_gpu_sharded_mg_two_ranks_device_engine(tmp_path, host_gmres):
    """time-slab sharded SMG on the device engine over two ranks == the
    serial device multigrid (equal cycles, 1e-10) — with the smoother's GMRES resident on
    the device (no host read-back inside a cycle) and with the host-scalar mirror."""
    mp.start_processes(_dev_worker, args=(2, _free_port(), str(tmp_path), host_gmres), nprocs=2,
                       join=True, start_method="spawn")
    rep = json.loads((tmp_path / "rep.json").read_text())
    x, xs = np.load(tmp_path / "x.npy"), np.load(tmp_path / "xs.npy")
    assert rep["conv"] and rep["its"] == rep["its_serial"]
    np.testing.assert_allclose(rep["hist"], rep["hist_serial"], rtol=1e-6)
    assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)
