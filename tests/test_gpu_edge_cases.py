"""Edge cases of the reference's own unit tests, on the device path.

Mirrors the behaviours pinned by the reference's tests/test_linalg.py
(GMRES, ILU(0), block-Jacobi, dense LU) and test_acceptance.py criterion 5
(partition / worker invariance) — the contracts a drop-in must keep:
immediate convergence, zero right-hand sides, iteration caps reported as
divergence, zero pivots and bad sizes as the reference's exceptions, the
block-range rule, and answers independent of the block/worker split.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2006_12883_b200 as pd
from oracle import paradiff_oracle as O

pytestmark = pytest.mark.gpu


def _random_spd(n, density, seed):
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=rng, format="csr")
    A = A + A.T + sp.eye(n) * (n * density * 2 + 1.0)
    return pd.linalg.as_csr(A)


def test_ilu0_nonsquare_and_zero_pivot():
    with pytest.raises(pd.ConfigurationError):
        pd.Ilu0(sp.csr_matrix(np.ones((3, 4))))
    with pytest.raises(pd.SolverError, match="row 0"):
        pd.Ilu0(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]])))


def test_gmres_identity_one_iteration_and_zero_rhs():
    b = np.arange(1.0, 6.0)
    x, rep = pd.gmres(sp.eye(5, format="csr"), b)
    assert rep.converged and rep.iterations == 1
    np.testing.assert_allclose(x, b, atol=1e-12)
    x, rep = pd.gmres(sp.eye(4, format="csr"), np.zeros(4))
    assert rep.converged and rep.iterations == 0
    np.testing.assert_array_equal(x, 0.0)


def test_gmres_ilu_on_tridiagonal_is_one_iteration():
    ops = pd.assemble_space(pd.SpaceMesh(99, 1.0))
    A = pd.linalg.as_csr(ops.Kh + ops.Mh)
    b = np.sin(np.arange(100.0))
    x, rep = pd.gmres(A, b, precond=pd.Ilu0(A))
    assert rep.converged and rep.iterations == 1
    _, rep_raw = pd.gmres(A, b, restart=100, max_it=1000)
    assert rep_raw.iterations > rep.iterations
    np.testing.assert_allclose(A @ x, b, atol=1e-10)


def test_gmres_history_true_residual_and_cap():
    A = _random_spd(60, 0.08, 11)
    _, rep = pd.gmres(A, np.ones(60), restart=60, tol_rel=1e-10, tol_abs=0.0)
    hist = np.array(rep.residual_history)
    assert np.all(np.diff(hist) <= 1e-9 * hist[0])
    A = _random_spd(30, 0.2, 2)
    b = np.linspace(-1, 1, 30)
    x, rep = pd.gmres(A, b, precond=pd.Ilu0(A), tol_rel=1e-11, tol_abs=0.0)
    assert rep.converged
    assert abs(np.linalg.norm(b - A @ x) - rep.residual_history[-1]) <= 1e-8 * np.linalg.norm(b)
    A = _random_spd(50, 0.1, 9)
    _, rep = pd.gmres(A, np.ones(50), tol_rel=1e-15, tol_abs=0.0, max_it=2, restart=2)
    assert not rep.converged and rep.diverged


def test_block_jacobi_rules():
    A = _random_spd(30, 0.15, 4)
    b = np.arange(30.0)
    np.testing.assert_array_equal(pd.BlockJacobiPrecond(A, 1).solve(b), pd.Ilu0(A).solve(b))
    assert pd.BlockJacobiPrecond(sp.eye(10, format="csr"), 3).ranges == [(0, 3), (3, 6), (6, 10)]
    with pytest.raises(pd.ConfigurationError):
        pd.BlockJacobiPrecond(sp.eye(4, format="csr"), 5)
    # ragged split (remainder in the last block) is bitwise the oracle's
    A = _random_spd(83, 0.07, 12)
    bb = np.sin(np.arange(83.0))
    np.testing.assert_array_equal(pd.BlockJacobiPrecond(A, 4).solve(bb),
                                  O.OBlockJacobi(A, 4).solve(bb))
    ops = pd.assemble_space(pd.SpaceMesh(19, 1.0))
    blk = pd.linalg.as_csr(ops.Kh + ops.Mh)
    A2 = pd.linalg.as_csr(sp.block_diag([blk, blk], format="csr"))
    _, rep = pd.gmres(A2, np.ones(40), precond=pd.BlockJacobiPrecond(A2, 2))
    assert rep.converged and rep.iterations == 1


def test_more_blocks_never_reduce_iterations_on_heat():
    prob = pd.heat_problem()
    mesh = pd.SpaceMesh(64, 1.0)
    system = pd.assemble_system(pd.make_tableau(2), pd.assemble_space(mesh),
                                pd.TimeGrid(16, 1.0), 0.0, prob.u0(mesh.vertices))
    A, b = system.global_matrix(), system.rhs()
    counts = []
    for nb in (1, 2, 4, 8):
        _, rep = pd.gmres(A, b, precond=pd.BlockJacobiPrecond(A, nb), restart=100, max_it=900)
        assert rep.converged
        counts.append(rep.iterations)
    assert all(a <= c for a, c in zip(counts, counts[1:]))


def test_partition_and_worker_invariance():
    """test_acceptance.py criterion 5 on the device path."""
    prob = pd.heat_problem()
    mesh = pd.SpaceMesh(32, 1.0)
    system = pd.assemble_system(pd.make_tableau(2), pd.assemble_space(mesh),
                                pd.TimeGrid(64, 1.0), 0.0, prob.u0(mesh.vertices))
    sols = []
    for P in (1, 2, 4, 8):
        h = pd.build_hierarchy(system, "SMG", 3, 3, partitions=P)
        u, rep = h.solve(system.rhs(), tol_rel=1e-11, tol_abs=1e-11)
        assert rep.converged
        sols.append(u)
    assert max(float(np.max(np.abs(u - sols[0]))) for u in sols[1:]) <= 1e-8
    from paper_2006_12883_b200 import pfasst as PF

    mesh2 = pd.SpaceMesh(16, 1.0)
    u0 = prob.u0(mesh2.vertices)
    counts, psols = [], []
    for P in (1, 2, 4, 8):
        hier = PF.build_pfasst_hierarchy(2, mesh2, pd.TimeGrid(64, 1.0), 0.0, L=2, nu=1)
        u, rep = PF.pfasst_run(hier, u0, 16, P, tol_rel=1e-10, tol_abs=1e-10)
        assert rep.converged
        counts.append(rep.iterations)
        psols.append(u)
    assert max(float(np.max(np.abs(u - psols[0]))) for u in psols[1:]) <= 1e-8
    assert all(a <= c for a, c in zip(counts, counts[1:]))


def test_dense_lu_matches_numpy_and_accepts_dense():
    rng = np.random.default_rng(3)
    Ad = rng.standard_normal((12, 12)) + 12 * np.eye(12)
    b = rng.standard_normal(12)
    np.testing.assert_allclose(pd.DenseLU(Ad).solve(b), np.linalg.solve(Ad, b), rtol=1e-12)
    np.testing.assert_allclose(pd.DenseLU(sp.csr_matrix(Ad)).solve(b), np.linalg.solve(Ad, b),
                               rtol=1e-12)


def test_gmres_accepts_callables_like_the_reference():
    """linalg.py:233-237 (test_linalg.py test_matvec_callable_accepted): A may be a
    callable matvec or any object with .dot, precond any callable / .solve object."""
    D = np.diag([2.0, 3.0, 4.0])
    x, rep = pd.gmres(lambda v: D @ v, np.array([2.0, 3.0, 4.0]))
    assert rep.converged
    np.testing.assert_allclose(x, 1.0, atol=1e-10)

    # callable operator + callable preconditioner vs the oracle's GMRES on the same pair:
    # equal iteration counts and histories
    A = _random_spd(80, 0.06, 5)
    b = np.cos(np.arange(80.0))
    dinv = 1.0 / A.diagonal()
    calls = {"A": 0, "M": 0}

    def mv(v):
        calls["A"] += 1
        return A @ v

    def ps(v):
        calls["M"] += 1
        return dinv * v

    x, rep = pd.gmres(mv, b, precond=ps, tol_rel=1e-11, tol_abs=0.0, restart=10)
    xo, repo = O.gmres(A, b, ps, tol_rel=1e-11, tol_abs=0.0, restart=10)
    assert rep.converged and rep.iterations == repo.iterations
    assert calls["A"] > rep.iterations and calls["M"] >= rep.iterations
    np.testing.assert_allclose(rep.residual_history, repo.residual_history, rtol=1e-6, atol=1e-13)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)

    # mixed: device matrix with a callable preconditioner; callable operator with device ILU(0)
    x1, rep1 = pd.gmres(A, b, precond=ps, tol_rel=1e-11, tol_abs=0.0, restart=10)
    assert rep1.iterations == repo.iterations and np.linalg.norm(x1 - xo) <= 1e-10 * np.linalg.norm(xo)
    ilu = pd.Ilu0(A)
    x2, rep2 = pd.gmres(mv, b, precond=ilu, tol_rel=1e-11, tol_abs=0.0)
    x3, rep3 = pd.gmres(A, b, precond=ilu, tol_rel=1e-11, tol_abs=0.0)
    assert rep2.iterations == rep3.iterations
    assert np.linalg.norm(x2 - x3) <= 1e-12 * np.linalg.norm(x3)

    # an object with .dot / .solve (e.g. a LinearOperator-like wrapper)
    class Op:
        def dot(self, v):
            return A @ v

    class Pre:
        def solve(self, v):
            return dinv * v

    x4, rep4 = pd.gmres(Op(), b, precond=Pre(), x0=np.ones(80), tol_rel=1e-11, tol_abs=0.0)
    xo4, repo4 = O.gmres(A, b, ps, x0=np.ones(80), tol_rel=1e-11, tol_abs=0.0)
    assert rep4.iterations == repo4.iterations
    assert np.linalg.norm(x4 - xo4) <= 1e-10 * np.linalg.norm(xo4)

    # an exception inside the callable surfaces unchanged
    def bad(v):
        raise ValueError("user matvec failed")

    with pytest.raises(ValueError, match="user matvec failed"):
        pd.gmres(bad, b)
    # a wrong-sized result is a configuration error
    with pytest.raises(pd.ConfigurationError):
        pd.gmres(lambda v: np.zeros(3), b)
