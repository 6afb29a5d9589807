"""P-fast profile (matrix-free block-Jacobi-in-time smoother with inner spatial
V-cycles): the CPU restatement against the package's assembled space-time
operator (CPU), and the device path against the restatement (GPU: 1e-12
relative L2 at every time node, equal sweep counts)."""

import numpy as np
import pytest

from oracle.pfast_oracle import PfastOracle
from paper_2006_12883_b200 import collocation as C
from paper_2006_12883_b200 import problems as PB
from paper_2006_12883_b200 import spacetime as ST

CASES = [  # dim, n, bc, coef, M, Nt, dt, levels
    (2, 15, "dirichlet", 1.0, 3, 4, 1 / 64, 3),
    (2, 16, "periodic", 1.0, 3, 3, 0.01, 3),
    (3, 7, "dirichlet", 1.0, 5, 3, 1 / 256, 2),
    (3, 8, "periodic", 0.1, 3, 4, 1e-3, 3),
]


def _case(dim, n, bc, coef, M, Nt, dt, levels, seed=0):
    spec = PB.StencilSpec(dim, n, bc, coef)
    tab = C.make_tableau(M)
    rng = np.random.default_rng(seed)
    u0 = rng.uniform(-1, 1, spec.ndof)
    orc = PfastOracle(dim, n, bc == "periodic", coef, M, Nt, dt, tab.Kq, tab.Mq, tab.left_values,
                      levels)
    return spec, tab, u0, orc


@pytest.mark.parametrize("case", CASES)
def test_oracle_operator_is_the_reference_space_time_matrix(case):
    """The restatement's b − Lx equals the assembled global matrix's
    (spacetime.py:110-124 as rebuilt by the package's host setup)."""
    dim, n, bc, coef, M, Nt, dt, levels = case
    spec, tab, u0, orc = _case(*case)
    system = ST.assemble_system(tab, PB.fd_space(spec), ST.TimeGrid(Nt, Nt * dt), 0.0, u0)
    L = system.global_matrix()
    b = system.rhs()
    x = np.random.default_rng(1).standard_normal(b.size)
    r_ref = b - L @ x
    r = orc.residual(x.reshape(orc.shape()), b.reshape(orc.shape())).ravel()
    assert np.linalg.norm(r - r_ref) <= 1e-13 * np.linalg.norm(r_ref)
    from paper_2006_12883_b200.pfast import pfast_rhs
    np.testing.assert_allclose(pfast_rhs(spec, M, Nt, u0, tab), b, rtol=0, atol=1e-15)


def test_oracle_converges_and_transfers_are_adjoint():
    spec, tab, u0, orc = _case(*CASES[0])
    from paper_2006_12883_b200.pfast import pfast_rhs
    b = pfast_rhs(spec, 3, 4, u0, tab)
    x, its, conv, div, hist = orc.solve(b, tol_rel=1e-10)
    assert conv and not div and its < 60
    # R = P^T on both boundary kinds
    from oracle.pfast_oracle import _prolong_axis, _restrict_axis
    rng = np.random.default_rng(2)
    for periodic, nf, nc in ((False, 15, 7), (True, 16, 8)):
        f = rng.standard_normal((1, 1, nf))
        c = rng.standard_normal((1, 1, nc))
        lhs = np.sum(_restrict_axis(f, 2, periodic) * c)
        rhs = np.sum(f * _prolong_axis(c, 2, periodic))
        assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_pfast_matches_restatement(case):
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import PfastSolver, pfast_rhs

    dim, n, bc, coef, M, Nt, dt, levels = case
    spec, tab, u0, orc = _case(*case)
    b = pfast_rhs(spec, M, Nt, u0, tab)
    solver = PfastSolver(spec, M, Nt, dt, levels=levels, tableau=tab)
    # one sweep from a random iterate: residual and V-cycle pieces together
    x0 = np.random.default_rng(3).standard_normal(b.size)
    xd = N.to_device(x0)
    solver.sweep(b, xd)
    want = orc.sweep(x0.reshape(orc.shape()), b.reshape(orc.shape())).ravel()
    got = N.to_host(xd)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    # full solve: equal sweep counts, 1e-10 relative L2 at every time node
    x_ref, its, conv, div, hist = orc.solve(b, tol_rel=1e-10)
    x, rep = solver.solve(b, tol_rel=1e-10)
    assert rep.converged == conv and rep.iterations == its
    xr = x_ref.reshape(Nt * M, -1)
    xg = np.asarray(x).reshape(Nt * M, -1)
    for k in range(Nt * M):
        assert np.linalg.norm(xg[k] - xr[k]) <= 1e-10 * max(np.linalg.norm(xr[k]), 1e-300)
    h = np.asarray(rep.residual_history)
    assert h.size == len(hist)
    assert np.all(np.abs(h - np.asarray(hist)) <= 1e-10 * hist[0])


@pytest.mark.gpu
def test_gpu_pfast_config_errors():
    from paper_2006_12883_b200.errors import ConfigurationError
    from paper_2006_12883_b200.pfast import PfastSolver

    with pytest.raises(ConfigurationError):
        PfastSolver(PB.StencilSpec(2, 16, "dirichlet"), 3, 2, 0.1, levels=2)  # even Dirichlet
    with pytest.raises(ConfigurationError):
        PfastSolver(PB.StencilSpec(2, 15, "dirichlet"), 7, 2, 0.1, levels=1)  # M > 5


# ---------------------------------------------------------------- time slabs
def _slab_parts(case, nslab):
    dim, n, bc, coef, M, Nt, dt, levels = case
    spec, tab, u0, orc = _case(*case)
    from paper_2006_12883_b200.pfast import pfast_rhs
    b = pfast_rhs(spec, M, Nt, u0, tab).reshape(Nt, -1)
    k = Nt // nslab
    parts = [b[i * k:(i + 1) * k].ravel() for i in range(nslab)]
    orcs = [PfastOracle(dim, n, bc == "periodic", coef, M, k, dt, tab.Kq, tab.Mq,
                        tab.left_values, levels) for _ in range(nslab)]
    return b.ravel(), parts, orcs, orc


def test_time_slabs_in_process_equal_serial():
    """Block-Jacobi in time over 2 slabs (halo = previous slab's last node):
    the same iterates and sweep counts as the serial restatement."""
    from oracle.pfast_oracle import OracleSlab
    from paper_2006_12883_b200.pfast import solve_time_slabs

    b, parts, orcs, orc = _slab_parts(CASES[3], 2)
    slabs = [OracleSlab(o, p) for o, p in zip(orcs, parts)]
    its, conv, div, hist = solve_time_slabs(slabs, tol_rel=1e-10)
    x_ref, its_ref, conv_ref, _, hist_ref = orc.solve(b, tol_rel=1e-10)
    assert conv and conv_ref and its == its_ref
    x = np.concatenate([s.solution() for s in slabs])
    assert np.linalg.norm(x - x_ref) <= 1e-13 * np.linalg.norm(x_ref)
    np.testing.assert_allclose(hist, hist_ref, rtol=1e-12)


SLAB_CASE = (3, 7, "dirichlet", 1.0, 5, 4, 1 / 256, 2)  # C4-type, 4 steps -> 2 slabs


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist

    from oracle.pfast_oracle import OracleSlab
    from paper_2006_12883_b200.pfast import solve_time_slabs

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    b, parts, orcs, orc = _slab_parts(SLAB_CASE, world)
    mine = [OracleSlab(orcs[rank], parts[rank])]
    its, conv, div, hist = solve_time_slabs(mine, tol_rel=1e-10)
    np.save(f"{out}/x{rank}.npy", mine[0].solution())
    np.save(f"{out}/meta{rank}.npy", np.array([its, conv, div]))
    dist.destroy_process_group()


def test_time_slabs_gloo_world2_equal_serial(tmp_path):
    """Two ranks (gloo), one slab each: only the slab-end state crosses ranks
    (send/recv) plus one allreduce per sweep; equal to the serial restatement."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_gloo_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    b, parts, orcs, orc = _slab_parts(SLAB_CASE, 2)
    x_ref, its_ref, conv_ref, _, _ = orc.solve(b, tol_rel=1e-10)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(2)])
    for r in range(2):
        its, conv, div = np.load(tmp_path / f"meta{r}.npy")
        assert its == its_ref and bool(conv) == conv_ref
    assert np.linalg.norm(x - x_ref) <= 1e-13 * np.linalg.norm(x_ref)


@pytest.mark.gpu
def test_gpu_time_slabs_equal_serial_device():
    """Two device slabs in one process (the per-rank schedule without waiting
    kernels): equal sweep counts and 1e-12 vs the serial device solve."""
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import DeviceSlab, PfastSolver, solve_time_slabs

    dim, n, bc, coef, M, Nt, dt, levels = CASES[3]
    spec, tab, _, _ = _case(*CASES[3])
    b, parts, orcs, orc = _slab_parts(CASES[3], 2)
    slabs = [DeviceSlab(PfastSolver(spec, M, Nt // 2, dt, levels=levels, tableau=tab), p)
             for p in parts]
    its, conv, div, hist = solve_time_slabs(slabs, tol_rel=1e-10)
    x_ser, rep = PfastSolver(spec, M, Nt, dt, levels=levels, tableau=tab).solve(b, tol_rel=1e-10)
    assert conv and rep.converged and its == rep.iterations
    x = np.concatenate([N.to_host(s.solution()) for s in slabs])
    assert np.linalg.norm(x - x_ser) <= 1e-12 * np.linalg.norm(x_ser)
