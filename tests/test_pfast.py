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
@pytest.mark.parametrize("case", [(2, 128, "periodic", 1.0, 3, 2, 0.01, 4),
                                  (3, 64, "periodic", 0.1, 3, 2, 1e-3, 3),
                                  (3, 64, "periodic", 0.1, 2, 1, 1e-3, 2)])
def test_gpu_pair_per_lane_transfers_match_restatement(case, monkeypatch):
    """Periodic levels with a multiple of 32 coarse points run the pair-per-lane
    restriction / prolongation kernels: one sweep vs the restatement (1e-12) and vs the
    general transfer kernels (PD_PF_NO_PAIR_TRANSFERS is read once per process, so the
    comparison is against the restatement only when it was not set at start-up)."""
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import PfastSolver, pfast_rhs

    dim, n, bc, coef, M, Nt, dt, levels = case
    spec, tab, u0, orc = _case(*case)
    b = pfast_rhs(spec, M, Nt, u0, tab)
    solver = PfastSolver(spec, M, Nt, dt, levels=levels, tableau=tab)
    x0 = np.random.default_rng(3).standard_normal(b.size)
    xd = N.to_device(x0)
    solver.sweep(b, xd)
    want = orc.sweep(x0.reshape(orc.shape()), b.reshape(orc.shape())).ravel()
    got = N.to_host(xd)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    solver.sweep(b, xd)
    want = orc.sweep(want.reshape(orc.shape()), b.reshape(orc.shape())).ravel()
    assert np.linalg.norm(N.to_host(xd) - want) <= 1e-12 * np.linalg.norm(want)


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


# ---------------------------------------------------------------- Newton weights + STMG
from oracle import pfast_oracle as PO  # noqa: E402

ST_CASES = [  # dim, n, bc, coef, M, Nt, dt, gamma, reaction
    (2, 16, "periodic", 0.1, 3, 16, 0.02, 1.0, "cubic"),
    (2, 15, "dirichlet", 1.0, 3, 8, 1 / 64, 1.0, "fisher"),
    (3, 8, "periodic", 0.1, 3, 8, 1e-3, 1.0, "cubic"),
    (3, 7, "dirichlet", 1.0, 2, 4, 1 / 256, 0.5, "cubic"),
]


def _st_case(dim, n, bc, coef, M, Nt, dt, gamma, kind, seed=0, **kw):
    spec = PB.StencilSpec(dim, n, bc, coef)
    tab = C.make_tableau(M)
    u0 = np.random.default_rng(seed).uniform(-1, 1, spec.ndof)
    orc = PO.PfastStmgOracle(dim, n, bc == "periodic", coef, M, Nt, dt, tab.Kq, tab.Mq,
                             tab.left_values, tab.nodes, **kw)
    return spec, tab, u0, orc


@pytest.mark.parametrize("case", ST_CASES)
def test_oracle_newton_pieces_are_the_reference_system(case):
    """The restatement's J·v (weights in the point blocks) and −F(u) equal the
    assembled Jacobian / nonlinear residual of the reference restatement
    (spacetime.py:126-151 as oracle/paradiff_oracle.OSystem)."""
    from oracle import paradiff_oracle as O

    dim, n, bc, coef, M, Nt, dt, gamma, kind = case
    spec, tab, u0, orc = _st_case(*case)
    ops = PB.fd_space(spec)
    system = O.OSystem(O.tableau(M), ops.Kh, ops.lumped_diagonal, Nt, Nt * dt, gamma, u0,
                       reaction=kind)
    rng = np.random.default_rng(1)
    u = 0.5 * rng.standard_normal(system.size)
    v = rng.standard_normal(system.size)
    shp = orc.shape()
    orc.set_weights(gamma * dt * spec.mass * PO.reaction_deriv(kind, u.reshape(shp)))
    Jv = -orc.sm[0].residual(v.reshape(shp), np.zeros(shp)).ravel()
    want = system.jacobian(u) @ v
    assert np.linalg.norm(Jv - want) <= 1e-13 * np.linalg.norm(want)
    orc.set_weights(None)
    rhs = system.rhs().reshape(shp)
    mF = orc.sm[0].residual(u.reshape(shp), rhs) - gamma * dt * spec.mass * np.einsum(
        "mk,tk...->tm...", tab.Mq, PO.reaction(kind, u.reshape(shp)))
    F = system.residual(u)
    assert np.linalg.norm(mF.ravel() + F) <= 1e-13 * np.linalg.norm(F)


def test_host_schedule_and_time_transfers_equal_restatement():
    from paper_2006_12883_b200 import pfast as PF

    for dim, n, bc, coef, M, Nt, dt, *_ in ST_CASES + [(3, 64, "periodic", 0.1, 3, 32, 1e-3, 1, "")]:
        spec = PB.StencilSpec(dim, n, bc, coef)
        a = PO.st_schedule(dim, n, bc == "periodic", coef, Nt, dt)
        b = [(nt, sp.n, d, s) for nt, sp, d, s in PF.st_schedule(spec, Nt, dt)]
        assert a == b
        nodes = C.make_tableau(M).nodes
        for A, B in zip(PO.time_transfer_matrices(nodes), PF.time_transfer_matrices(nodes)):
            np.testing.assert_allclose(np.asarray(A, float), np.asarray(B, float), rtol=0, atol=1e-14)
    # the prolongation reproduces polynomials of degree < M, restriction is its transpose
    nodes = C.make_tableau(3).nodes
    P1, P2, E, half = PF.time_transfer_matrices(nodes)
    poly = lambda t: 1.0 - 2.0 * t + 0.5 * t * t
    np.testing.assert_allclose(P1 @ poly(nodes), poly(0.5 * nodes), atol=1e-14)
    np.testing.assert_allclose(P2 @ poly(nodes), poly(0.5 + 0.5 * nodes), atol=1e-14)


def test_oracle_stmg_cycle_count_is_flat_in_nt():
    """Block-Jacobi in time alone needs ~Nt sweeps; the space-time cycle's count
    does not grow with the number of steps."""
    from paper_2006_12883_b200.pfast import pfast_rhs

    counts, sweeps = [], []
    for Nt in (8, 16, 32):
        case = (2, 16, "periodic", 0.1, 3, Nt, 0.02, 0.0, "cubic")
        spec, tab, u0, orc = _st_case(*case)
        b = pfast_rhs(spec, 3, Nt, u0, tab)
        x, its, conv, div, hist = orc.solve(b, tol_rel=1e-8)
        assert conv and not div
        counts.append(its)
        bj = PfastOracle(2, 16, True, 0.1, 3, Nt, 0.02, tab.Kq, tab.Mq, tab.left_values, 3)
        sweeps.append(bj.solve(b, tol_rel=1e-8)[1])
    assert max(counts) - min(counts) <= 1 and max(counts) <= 16, counts
    assert sweeps[-1] > sweeps[0] + 8, sweeps  # the smoother alone does grow


def test_oracle_newton_converges_quadratically():
    case = ST_CASES[0]
    dim, n, bc, coef, M, Nt, dt, gamma, kind = case
    spec, tab, u0, orc = _st_case(*case)
    from paper_2006_12883_b200.pfast import pfast_rhs
    rhs = pfast_rhs(spec, M, Nt, u0, tab)
    u, info = PO.newton_oracle(orc, rhs, gamma, kind, tol=1e-9)
    assert info["converged"] and not info["diverged"] and info["newton"] <= 4
    h = info["hist"]
    assert h[2] < 1e-3 * h[1]


def _stmg_slab_parts(case, nslab, coarse_t_sweeps=5):
    dim, n, bc, coef, M, Nt, dt, gamma, kind = case
    spec, tab, u0, _ = _st_case(*case)
    from paper_2006_12883_b200.pfast import pfast_rhs
    b = pfast_rhs(spec, M, Nt, u0, tab).reshape(Nt, -1)
    k = Nt // nslab
    mk = lambda nt, mn: PO.PfastStmgOracle(dim, n, bc == "periodic", coef, M, nt, dt, tab.Kq,
                                           tab.Mq, tab.left_values, tab.nodes, min_nt=mn,
                                           coarse_t_sweeps=coarse_t_sweeps)
    parts = [b[i * k:(i + 1) * k].ravel() for i in range(nslab)]
    return b.ravel(), parts, [mk(k, 2) for _ in range(nslab)], mk(Nt, 2 * nslab)


def test_stmg_time_slabs_in_process_equal_serial():
    """The sharded space-time cycle (slab-local transfers, per-level slab-end halos)
    equals the serial cycle whose coarsest level holds all slabs' coarsest steps."""
    from paper_2006_12883_b200.pfast import solve_time_slabs_stmg

    b, parts, orcs, ser = _stmg_slab_parts(ST_CASES[0], 2)
    slabs = [PO.OracleStmgSlab(o, p) for o, p in zip(orcs, parts)]
    its, conv, div, hist = solve_time_slabs_stmg(slabs, tol_rel=1e-9)
    x_ref, its_ref, conv_ref, _, hist_ref = ser.solve(b, tol_rel=1e-9)
    assert conv and conv_ref and its == its_ref
    x = np.concatenate([s.solution() for s in slabs])
    assert np.linalg.norm(x - x_ref) <= 1e-13 * np.linalg.norm(x_ref)
    np.testing.assert_allclose(hist, hist_ref, rtol=1e-12)


def _gloo_stmg_worker(rank, world, port, out, device):
    import torch.distributed as dist

    from paper_2006_12883_b200 import pfast as PF

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    case = ST_CASES[0]
    b, parts, orcs, ser = _stmg_slab_parts(case, world)
    if device:
        from paper_2006_12883_b200 import _native as N
        dim, n, bc, coef, M, Nt, dt, gamma, kind = case
        spec = PB.StencilSpec(dim, n, bc, coef)
        sol = PF.PfastStmg(spec, M, Nt // world, dt, min_nt=2, coarse_t_sweeps=5)
        mine = [PF.DeviceStmgSlab(sol, parts[rank])]
        bj = PF.DeviceSlab(PF.PfastSolver(spec, M, Nt // world, dt, levels=3), parts[rank])
        its_bj, conv_bj, _, _ = PF.solve_time_slabs([bj], tol_rel=1e-9)
        np.save(f"{out}/bj{rank}.npy", N.to_host(bj.solution()))
        np.save(f"{out}/bjmeta{rank}.npy", np.array([its_bj, conv_bj]))
        get = lambda s: N.to_host(s.solution())
    else:
        mine = [PO.OracleStmgSlab(orcs[rank], parts[rank])]
        get = lambda s: s.solution()
    its, conv, div, hist = PF.solve_time_slabs_stmg(mine, tol_rel=1e-9)
    np.save(f"{out}/x{rank}.npy", get(mine[0]))
    np.save(f"{out}/meta{rank}.npy", np.array([its, conv, div]))
    dist.destroy_process_group()


def _run_gloo_stmg(tmp_path, device):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_gloo_stmg_worker, args=(2, port, str(tmp_path), device), nprocs=2, join=True)
    b, parts, orcs, ser = _stmg_slab_parts(ST_CASES[0], 2)
    x_ref, its_ref, conv_ref, _, _ = ser.solve(b, tol_rel=1e-9)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(2)])
    for r in range(2):
        its, conv, div = np.load(tmp_path / f"meta{r}.npy")
        assert its == its_ref and bool(conv) == conv_ref
    return x, x_ref, b


def test_stmg_time_slabs_gloo_world2_equal_serial(tmp_path):
    x, x_ref, _ = _run_gloo_stmg(tmp_path, False)
    assert np.linalg.norm(x - x_ref) <= 1e-13 * np.linalg.norm(x_ref)


@pytest.mark.gpu
def test_gpu_time_slabs_gloo_world2_device_slabs(tmp_path):
    """Two ranks over gloo sharing the GPU, DeviceStmgSlab / DeviceSlab per rank (halos
    staged through the host by Comm.shift_next): equal to the serial restatement."""
    x, x_ref, b = _run_gloo_stmg(tmp_path, True)
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    dim, n, bc, coef, M, Nt, dt, gamma, kind = ST_CASES[0]
    tab = C.make_tableau(M)
    bj = PfastOracle(dim, n, True, coef, M, Nt, dt, tab.Kq, tab.Mq, tab.left_values, 3)
    xb, its_b, conv_b, _, _ = bj.solve(b, tol_rel=1e-9)
    got = np.concatenate([np.load(tmp_path / f"bj{r}.npy") for r in range(2)])
    for r in range(2):
        its, conv = np.load(tmp_path / f"bjmeta{r}.npy")
        assert its == its_b and bool(conv) == conv_b
    assert np.linalg.norm(got - xb) <= 1e-10 * np.linalg.norm(xb)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ST_CASES)
def test_gpu_pfast_newton_pieces_match_restatement(case):
    """Device J-residual (weights on every spatial level), −F(u), and one sweep with
    weights vs the restatement: 1e-12."""
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import PfastSolver, pfast_rhs

    dim, n, bc, coef, M, Nt, dt, gamma, kind = case
    spec, tab, u0, _ = _st_case(*case)
    levels = PO.spatial_levels_for(n, bc == "periodic")
    orc = PfastOracle(dim, n, bc == "periodic", coef, M, Nt, dt, tab.Kq, tab.Mq, tab.left_values,
                      levels)
    sol = PfastSolver(spec, M, Nt, dt, levels=levels, tableau=tab)
    rng = np.random.default_rng(4)
    shp = orc.shape()
    u = 0.7 * rng.standard_normal(shp)
    x = rng.standard_normal(shp)
    rhs = pfast_rhs(spec, M, Nt, u0, tab).reshape(shp)
    halo = rng.standard_normal(spec.ndof)
    # −F(u)
    want = orc.residual(u, rhs, halo) - gamma * dt * spec.mass * np.einsum(
        "mk,tk...->tm...", tab.Mq, PO.reaction(kind, u))
    got, nrm = sol.nl_residual(u.ravel(), rhs.ravel(), gamma, kind, halo=halo)
    got = N.to_host(got)
    assert np.linalg.norm(got - want.ravel()) <= 1e-13 * np.linalg.norm(want)
    assert abs(nrm - np.linalg.norm(want)) <= 1e-12 * nrm
    # J residual and a sweep with weights
    orc.set_weights(gamma * dt * spec.mass * PO.reaction_deriv(kind, u))
    sol.set_state(u.ravel(), gamma, kind)
    r, _ = sol.residual(x.ravel(), rhs.ravel(), halo=halo)
    want = orc.residual(x, rhs, halo)
    assert np.linalg.norm(N.to_host(r) - want.ravel()) <= 1e-13 * np.linalg.norm(want)
    xd = N.to_device(x.ravel())
    sol.sweep(rhs.ravel(), xd, halo=halo)
    want = orc.sweep(x, rhs, halo)
    assert np.linalg.norm(N.to_host(xd) - want.ravel()) <= 1e-12 * np.linalg.norm(want)
    # back to the linear operator
    sol.set_state(None)
    orc.set_weights(None)
    r, _ = sol.residual(x.ravel(), rhs.ravel())
    want = orc.residual(x, rhs)
    assert np.linalg.norm(N.to_host(r) - want.ravel()) <= 1e-13 * np.linalg.norm(want)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ST_CASES)
def test_gpu_pfast_stmg_matches_restatement(case):
    """One space-time cycle from a random iterate (1e-12), the solve (equal cycle
    counts, 1e-10 relative L2 at every time node) and the Newton solve (equal
    Newton / inner counts, 1e-10 per node) vs the restatement."""
    from pd_util import per_node_rel

    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import PfastStmg, pfast_rhs

    dim, n, bc, coef, M, Nt, dt, gamma, kind = case
    spec, tab, u0, orc = _st_case(*case)
    sol = PfastStmg(spec, M, Nt, dt, tableau=tab)
    assert [(a, s.n, d, f) for a, s, d, f in sol.sched] == orc.sched
    b = pfast_rhs(spec, M, Nt, u0, tab)
    shp = orc.shape()
    x0 = np.random.default_rng(5).standard_normal(b.size)
    xd = N.to_device(x0)
    sol.cycle(b, xd)
    want = orc.cycle(0, b.reshape(shp), x0.reshape(shp)).ravel()
    assert np.linalg.norm(N.to_host(xd) - want) <= 1e-12 * np.linalg.norm(want)
    x, rep = sol.solve(b, tol_rel=1e-9)
    xo, its, conv, div, hist = orc.solve(b, tol_rel=1e-9)
    assert rep.converged and conv and rep.iterations == its
    np.testing.assert_allclose(rep.residual_history, hist, rtol=1e-6)
    assert per_node_rel(x, xo, (Nt * M, -1)) <= 1e-10
    # Newton
    u, nrep = sol.newton(b, gamma, kind, tol=1e-9)
    uo, info = PO.newton_oracle(orc, b, gamma, kind, tol=1e-9)
    assert nrep.converged and info["converged"]
    assert nrep.newton_iterations == info["newton"] and nrep.inner_iterations == info["inner"]
    assert nrep.damped_steps == info["damped"]
    assert per_node_rel(u, uo, (Nt * M, -1)) <= 1e-10


@pytest.mark.gpu
def test_gpu_stmg_slabs_equal_serial_device():
    """Two device slabs in one process through the level primitives == the serial
    device cycle with the merged coarsest level (bitwise: same kernels, same order)."""
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import (DeviceStmgSlab, PfastStmg, solve_time_slabs_stmg)

    case = ST_CASES[0]
    dim, n, bc, coef, M, Nt, dt, gamma, kind = case
    spec = PB.StencilSpec(dim, n, bc, coef)
    b, parts, _, _ = _stmg_slab_parts(case, 2)
    slabs = [DeviceStmgSlab(PfastStmg(spec, M, Nt // 2, dt, min_nt=2, coarse_t_sweeps=5), p)
             for p in parts]
    its, conv, div, hist = solve_time_slabs_stmg(slabs, tol_rel=1e-9)
    ser = PfastStmg(spec, M, Nt, dt, min_nt=4, coarse_t_sweeps=5)
    x_ser, rep = ser.solve(b, tol_rel=1e-9)
    assert conv and rep.converged and its == rep.iterations
    x = np.concatenate([N.to_host(s.solution()) for s in slabs])
    assert np.linalg.norm(x - x_ser) <= 1e-12 * np.linalg.norm(x_ser)


@pytest.mark.gpu
def test_gpu_stmg_cycle_count_flat_in_nt_and_c5_newton():
    """Device STMG at config 5's μ = κ·dt/h²: the cycle count to 1e-8 does not grow from
    32 to 256 steps (block-Jacobi alone grows with Nt), and the cubic Newton solve
    converges."""
    from paper_2006_12883_b200 import _native as N
    from paper_2006_12883_b200.pfast import PfastSolver, PfastStmg, pfast_rhs

    spec = PB.StencilSpec(3, 32, "periodic", 0.1)
    dt = 6.5536 * spec.h ** 2 / 0.1
    u0 = np.random.default_rng(0).uniform(-1, 1, spec.ndof)
    # V(2,2): flat (|Δ| <= 1 cycle over 8x the steps); V(1,1): about the same sweep
    # total at 32 steps and a slow (logarithmic) growth — CPU restatement, 2D 32^2:
    # V(2,2) 8, 9, 9, 9 and V(1,1) 15, 15, 15, 19 cycles at 32, 64, 128, 256 steps
    counts, counts11 = [], []
    for Nt in (32, 256):
        b = N.to_device(pfast_rhs(spec, 3, Nt, u0))
        _, rep = PfastStmg(spec, 3, Nt, dt, nu_t=2).solve(b, tol_rel=1e-8)
        assert rep.converged
        counts.append(rep.iterations)
        _, rep = PfastStmg(spec, 3, Nt, dt, nu_t=1).solve(b, tol_rel=1e-8)
        assert rep.converged
        counts11.append(rep.iterations)
    assert abs(counts[0] - counts[1]) <= 1 and counts[1] <= 14, (counts, counts11)
    assert counts11[1] <= 1.35 * counts11[0] and counts11[1] <= 24, (counts, counts11)
    b = N.to_device(pfast_rhs(spec, 3, 64, u0))
    _, bj = PfastSolver(spec, 3, 64, dt).solve(b, tol_rel=1e-8, max_sweeps=400)
    # block-Jacobi alone needs about one sweep per step: at a quarter of the steps it
    # already takes far more sweeps than the 256-step STMG takes cycles
    assert bj.iterations >= 64 and bj.iterations > 2 * counts11[1]
    s = PfastStmg(spec, 3, 32, 1e-3)
    b = N.to_device(pfast_rhs(spec, 3, 32, u0))
    u, rep = s.newton(b, 1.0, "cubic", tol=1e-8)
    assert rep.converged and rep.newton_iterations >= 1 and not rep.diverged
    _, res = s.nl_residual(u, b, 1.0, "cubic")
    assert res <= 1e-8
