"""GPU parity: sparse kernels, GMRES and multigrid vs golden fixtures + oracle.

Bar: CSR products and ILU(0) solves bitwise equal to the reference (same
per-row order, separately rounded); solves equal iteration counts and
per-time-node relative L2 <= 1e-10 (BASELINE north_star tolerance).
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2006_12883_b200 as pd
from oracle import paradiff_oracle as O
from pd_util import per_node_rel, rel_l2

pytestmark = pytest.mark.gpu


def _A(g):
    return sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]))


def test_spmv_bitwise_scipy(golden):
    g = golden("linalg")
    A = _A(g)
    x = g["b"]
    np.testing.assert_array_equal(pd.DeviceCsr(A).dot(x), A @ x)


def test_ilu0_solve_bitwise(golden):
    g = golden("linalg")
    ilu = pd.Ilu0(_A(g))
    np.testing.assert_array_equal(ilu.solve(g["b"]), g["ilu_solve"])
    bj = pd.block_jacobi(_A(g), 3)
    assert bj.ranges == [(0, 100), (100, 200), (200, 300)]
    np.testing.assert_array_equal(bj.solve(g["b"]), g["bj_solve"])


def test_zero_pivot_row_reported():
    A = sp.csr_matrix(np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0], [0.0, 1.0, 1.0]]))
    with pytest.raises(pd.SolverError, match="row 1"):
        pd.Ilu0(A)


def test_gmres_matches_reference(golden):
    g = golden("linalg")
    A = _A(g)
    x, rep = pd.gmres(A, g["b"], precond=pd.Ilu0(A), tol_rel=1e-10, tol_abs=1e-12, restart=7,
                      max_it=200)
    assert rep.converged and rep.iterations == int(g["gm_its"])
    assert rel_l2(x, g["gm_x"]) < 1e-10
    # the final entry is the true residual of an iterate converged to 1e-10: rounding-level
    np.testing.assert_allclose(rep.residual_history[:-1], g["gm_hist"][:-1], rtol=1e-5)
    assert rep.residual_history[-1] <= 1e-10 * rep.residual_history[0]
    x2, rep2 = pd.gmres(A, g["b"], precond=pd.block_jacobi(A, 3), tol_rel=1e-10, tol_abs=1e-12,
                        restart=5, max_it=200)
    assert rep2.iterations == int(g["gm2_its"])
    assert rel_l2(x2, g["gm2_x"]) < 1e-10
    # restart=5 over 16 iterations: every cycle's estimates match the reference's
    np.testing.assert_allclose(rep2.residual_history[:-1], g["gm2_hist"][:-1], rtol=1e-5)


def test_gmres_x0_and_unpreconditioned():
    rng = np.random.default_rng(3)
    n = 200
    A = sp.diags([np.full(n - 1, -1.0), np.full(n, 4.0), np.full(n - 1, -1.0)], [-1, 0, 1],
                 format="csr")
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    for M in (None, "ilu"):
        pre_d = pd.Ilu0(A) if M else None
        pre_o = O.OIlu0(A) if M else None
        x, rep = pd.gmres(A, b, precond=pre_d, x0=x0, tol_rel=1e-12, tol_abs=0.0, restart=6,
                          max_it=100)
        xo, repo = O.gmres(A, b, M=pre_o, x0=x0, tol_rel=1e-12, tol_abs=0.0, restart=6,
                           max_it=100)
        assert rep.iterations == repo.iterations
        assert rel_l2(x, xo) < 1e-10


def _heat(Nx=64, Nt=16, M=3):
    prob = pd.heat_problem()
    mesh = pd.SpaceMesh(Nx, 1.0)
    return pd.assemble_system(pd.make_tableau(M), pd.assemble_space(mesh), pd.TimeGrid(Nt, 1.0),
                              0.0, prob.u0(mesh.vertices))


@pytest.mark.parametrize("strategy", ["SMG", "STMG", "SMMG"])
@pytest.mark.parametrize("P", [1, 4])
def test_mg_fem1d_matches_reference(golden, strategy, P):
    g = golden("mg_fem1d")
    s = _heat()
    h = pd.build_hierarchy(s, strategy, 3, 3, partitions=P)
    key = f"{strategy}_P{P}"
    v1 = h.vcycle(s.rhs(), np.zeros(s.size))
    assert rel_l2(v1, g[key + "_v1"]) < 1e-12
    x, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    assert rep.converged and rep.iterations == int(g[key + "_its"])
    assert per_node_rel(x, g[key + "_x"], (16, 3, 65)) < 1e-10
    np.testing.assert_allclose(rep.residual_history, g[key + "_hist"], rtol=1e-4, atol=1e-14)


@pytest.mark.parametrize("strategy", ["SMG", "STMG"])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_c1_mg_matches_reference(golden, strategy, P):
    g = golden("c1")
    cfg = pd.baseline_config("C1")
    system = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                                pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    h = pd.build_hierarchy(system, strategy, 4, 3, partitions=P)
    x, rep = h.solve(system.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    assert rep.iterations == int(g[f"{strategy}_P{P}_its"])
    assert per_node_rel(x, g[f"{strategy}_P{P}_x"], (16, 3, 127)) < 1e-10


def test_c2_small_mg_matches_reference(golden):
    g = golden("c2_small")
    spec = pd.StencilSpec(2, 15, "dirichlet", 1.0)
    system = pd.assemble_system(pd.make_tableau(3), pd.fd_space(spec), pd.TimeGrid(8, 8 / 64),
                                0.0, g["u0"])
    for strat in ("SMG", "STMG"):
        for P in (1, 4):
            h = pd.build_hierarchy(system, strat, 3, 3, partitions=P)
            x, rep = h.solve(system.rhs(), tol_rel=1e-10, tol_abs=1e-10)
            assert rep.iterations == int(g[f"{strat}_P{P}_its"]), (strat, P)
            assert per_node_rel(x, g[f"{strat}_P{P}_x"], (8, 3, 225)) < 1e-10


def test_dense_lu_matches_scipy():
    rng = np.random.default_rng(1)
    A = rng.standard_normal((300, 300)) + 30 * np.eye(300)
    b = rng.standard_normal(300)
    x = pd.DenseLU(sp.csr_matrix(A)).solve(b)
    assert rel_l2(x, np.linalg.solve(A, b)) < 1e-13


def test_spacetime_residual_matches_reference(golden):
    g = golden("spacetime")
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(16, prob.X)
    s = pd.assemble_system(pd.make_tableau(3), pd.assemble_space(mesh), pd.TimeGrid(4, prob.T),
                           prob.gamma, prob.u0(mesh.vertices))
    np.testing.assert_allclose(s.residual(g["u"]), g["res"], rtol=1e-12, atol=1e-12)


def test_newton_mg_matches_reference(golden):
    g = golden("newton")
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(32, prob.X)
    s = pd.assemble_system(pd.make_tableau(2), pd.assemble_space(mesh), pd.TimeGrid(8, prob.T),
                           prob.gamma, prob.u0(mesh.vertices))
    h = pd.build_hierarchy(s, "SMG", 3, 3)
    x, rep = pd.newton_solve(s, pd.mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9), tol=1e-9)
    assert rep.iterations == int(g["its"])
    assert rep.inner_iterations == g["inner"].tolist()
    assert rep.damped_steps == int(g["damped"])
    assert per_node_rel(x, g["x"], (8, 2, 33)) < 1e-9


def test_device_jacobian_bitwise_equals_scipy():
    """pd_jacobian_values reproduces spacetime.py:144-151 (scipy J) bitwise on L's pattern."""
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(32, prob.X)
    s = pd.assemble_system(pd.make_tableau(3), pd.assemble_space(mesh), pd.TimeGrid(4, prob.T),
                           prob.gamma, prob.u0(mesh.vertices))
    u = np.random.default_rng(2).standard_normal(s.size)
    Jh = pd.linalg.as_csr(s.jacobian(u))  # the hierarchy canonicalises J (multigrid.py:226)
    Jd = s.jacobian_device(u)
    L = s.global_matrix()
    assert np.array_equal(Jh.indptr, L.indptr) and np.array_equal(Jh.indices, L.indices)
    np.testing.assert_array_equal(Jd.values.cpu().numpy(), Jh.data)


def test_device_galerkin_refresh_bitwise_equals_scipy():
    """Device R A P (scipy csr_matmat order) equals the host Galerkin levels bitwise."""
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(32, prob.X)
    s = pd.assemble_system(pd.make_tableau(2), pd.assemble_space(mesh), pd.TimeGrid(8, prob.T),
                           prob.gamma, prob.u0(mesh.vertices))
    h = pd.build_hierarchy(s, "SMG", 3, 3)
    u1 = np.random.default_rng(3).standard_normal(s.size)
    u2 = np.random.default_rng(4).standard_normal(s.size)
    h.set_fine_matrix(s.jacobian(u1))
    h.enable_device_refresh()
    h.set_fine_values_dev(s.jacobian_device(u2).values)
    host = pd.build_hierarchy(s, "SMG", 3, 3, matrix=s.jacobian(u2)).matrices
    import ctypes
    from paper_2006_12883_b200 import _native as N
    for l in range(1, 3):
        hnd = ctypes.c_void_p()
        N.call("pd_mg_level_matrix", h._mg, l, ctypes.byref(hnd))
        M = host[l]
        dev = pd.DeviceCsr.borrowed(hnd, M.shape, M.nnz, h.ctx)
        x = np.random.default_rng(l).standard_normal(M.shape[1])
        np.testing.assert_array_equal(dev.dot(x), M @ x)


def test_sharded_mg_device_engine_one_rank_matches_serial():
    """mg_sharded on the GPU engine (G=1: no communication) reproduces the serial
    device multigrid: equal cycle counts, rel L2 <= 1e-10 — through the device-resident
    smoother steps (pd_gms_*), and through the host-scalar GMRES mirror."""
    from paper_2006_12883_b200.mg_sharded import build_sharded_hierarchy

    cfg = pd.baseline_config("C2", n=31, Nt=8)
    system = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                                pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    h = pd.build_hierarchy(system, "SMG", 3, 3, partitions=4)
    b = system.rhs()
    x1, r1 = h.solve(b, tol_rel=1e-10, tol_abs=1e-10)
    smg = build_sharded_hierarchy(h)
    assert smg.gms is not None
    x2, r2 = smg.solve(b, tol_rel=1e-10, tol_abs=1e-10)
    x2 = x2.cpu().numpy()
    assert r1.converged and r2.converged and r1.iterations == r2.iterations
    assert np.linalg.norm(x2 - x1) <= 1e-10 * np.linalg.norm(x1)
    np.testing.assert_allclose(r2.residual_history, r1.residual_history, rtol=1e-6)
    import os

    os.environ["PD_SHARDED_HOST_GMRES"] = "1"
    try:
        smg_h = build_sharded_hierarchy(h)
    finally:
        del os.environ["PD_SHARDED_HOST_GMRES"]
    assert smg_h.gms is None
    x3, r3 = smg_h.solve(b, tol_rel=1e-10, tol_abs=1e-10)
    assert r3.iterations == r1.iterations
    assert np.linalg.norm(x3.cpu().numpy() - x1) <= 1e-10 * np.linalg.norm(x1)


def test_repeated_solves_replay_captured_cycle_bitwise(golden, monkeypatch):
    """A second solve of the same state and vectors replays the V-cycle as a
    captured CUDA graph: results must be bitwise the eager ones, for new
    right-hand sides in the same buffers and after the values change."""
    g = golden("c2_small")
    spec = pd.StencilSpec(2, 15, "dirichlet", 1.0)
    system = pd.assemble_system(pd.make_tableau(3), pd.fd_space(spec), pd.TimeGrid(8, 8 / 64),
                                0.0, g["u0"])
    h = pd.build_hierarchy(system, "SMG", 3, 3, partitions=4)
    N = pd._native
    b = N.to_device(system.rhs())
    x = N.zeros(b.numel())

    def run(bv):
        b.copy_(N.to_device(bv))
        x.zero_()
        _, rep = h.solve_dev(b, x, 1e-10, 1e-10)
        return x.cpu().numpy().copy(), rep.iterations

    lib = N.load_library()
    rhs = system.rhs()
    l0 = lib.pd_launch_count()
    ref, its = run(rhs)  # eager (first sighting)
    eager_launches = lib.pd_launch_count() - l0
    for _ in range(3):  # capture, then replays
        l0 = lib.pd_launch_count()
        got, its2 = run(rhs)
        np.testing.assert_array_equal(got, ref)
        assert its2 == its
        # a replay counts the kernels of its graph, not one launch
        assert lib.pd_launch_count() - l0 == eager_launches
    rhs2 = np.sin(np.arange(rhs.size)) * 1e-3 + rhs
    got2, _ = run(rhs2)
    monkeypatch.setenv("PD_MG_NO_GRAPH", "1")
    eager2, _ = run(rhs2)
    np.testing.assert_array_equal(got2, eager2)
    monkeypatch.delenv("PD_MG_NO_GRAPH")
    # new values (Newton refresh): the captured cycle must not be reused stale
    A2 = system.global_matrix() * 1.5
    h.set_fine_matrix(A2)
    new1, _ = run(rhs)
    new2, _ = run(rhs)
    monkeypatch.setenv("PD_MG_NO_GRAPH", "1")
    h_eager = pd.build_hierarchy(system, "SMG", 3, 3, partitions=4)
    h_eager.set_fine_matrix(A2)
    b2 = N.to_device(rhs)
    x2 = N.zeros(b2.numel())
    h_eager.solve_dev(b2, x2, 1e-10, 1e-10)
    np.testing.assert_array_equal(new1, x2.cpu().numpy())
    np.testing.assert_array_equal(new2, new1)
