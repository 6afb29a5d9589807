"""Device direct solves: banded LU (pd_band.cu), blocked dense LU, and the
sequential / direct space-time solves built on them (reference:
spacetime.py:154-195 `_element_solve`, `solve_sequential`, `solve_direct`, which
call SuperLU; linalg.py:196-209 `DenseLU`).

Parity: against scipy's SuperLU / LAPACK on the same matrices, against the golden
`solve_sequential` outputs of the real reference (fixtures `spacetime`, `c1`), and —
nonlinear — against the oracle's restatement of the element Newton.
"""

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse as sp
from scipy.sparse.linalg import splu

import paper_2006_12883_b200 as pd
from oracle import paradiff_oracle as O
from paper_2006_12883_b200 import problems as PB
from pd_util import per_node_rel, rel_l2

pytestmark = pytest.mark.gpu


def _banded(n, kl, ku, seed, dominant=False):
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for d in range(-kl, ku + 1):
        A += np.diag(rng.standard_normal(n - abs(d)), d)
    if dominant:
        A += np.eye(n) * (kl + ku + 2)
    return sp.csr_matrix(A)


@pytest.mark.parametrize("n,kl,ku", [(1, 0, 0), (7, 1, 1), (64, 3, 5), (300, 40, 17), (257, 100, 100),
                                     (1000, 1, 2), (96, 95, 95)])
def test_banded_lu_matches_superlu_with_pivoting(n, kl, ku):
    A = _banded(n, kl, ku, seed=n + kl)  # not dominant: interchanges happen
    b = np.random.default_rng(1).standard_normal(n)
    x = pd.BandedLU(A).solve(b)
    ref = splu(A.tocsc()).solve(b)
    assert rel_l2(x, ref) < 1e-9 * max(1.0, np.linalg.cond(A.toarray()) * 1e-6)
    assert np.linalg.norm(A @ x - b) <= 1e-10 * max(1.0, np.linalg.norm(b)) * np.linalg.cond(
        A.toarray())


def test_banded_lu_with_order_and_errors():
    # a matrix that is banded only after a permutation of its unknowns
    n = 120
    B = _banded(n, 4, 4, seed=3, dominant=True)
    perm = np.random.default_rng(5).permutation(n)
    inv = np.argsort(perm)
    A = sp.csr_matrix(B[inv][:, inv])  # A[perm][:, perm] == B
    b = np.cos(np.arange(n))
    lu = pd.BandedLU(A, order=perm)
    assert (lu.kl, lu.ku) == (4, 4)
    assert rel_l2(lu.solve(b), splu(A.tocsc()).solve(b)) < 1e-12
    with pytest.raises(pd.ConfigurationError):
        pd.BandedLU(sp.csr_matrix(np.ones((3, 4))))
    with pytest.raises(pd.ConfigurationError):
        pd.BandedLU(B, order=np.zeros(n, dtype=int))
    with pytest.raises(pd.SolverError, match="singular"):
        pd.BandedLU(sp.csr_matrix(np.array([[1.0, 2.0, 0.0], [2.0, 4.0, 0.0], [0.0, 1.0, 1.0]])))
    with pytest.raises(pd.ConfigurationError):
        lu.solve(np.ones(n + 1))


@pytest.mark.parametrize("n", [1, 31, 32, 33, 100, 517])
def test_blocked_dense_lu_matches_lapack(n):
    """The panel-blocked device LU (three launches per 32 columns) agrees with LAPACK
    getrf/getrs, also when interchanges are needed in every panel."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    x = pd.DenseLU(sp.csr_matrix(A)).solve(b)
    ref = scipy.linalg.lu_solve(scipy.linalg.lu_factor(A), b)
    assert rel_l2(x, ref) < 1e-9
    assert np.linalg.norm(A @ x - b) <= 1e-9 * np.linalg.norm(b) * max(1.0, np.linalg.cond(A) * 1e-3)


def test_dense_lu_launch_count_is_per_panel():
    from paper_2006_12883_b200 import _native as N

    n = 320
    A = sp.csr_matrix(np.random.default_rng(0).standard_normal((n, n)) + 20 * np.eye(n))
    lib = N.load_library()
    before = lib.pd_launch_count()
    pd.DenseLU(A)
    assert lib.pd_launch_count() - before <= 3 * (n // 32) + 8


def test_solve_sequential_matches_reference_fixtures(golden):
    g = golden("spacetime")
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(16, prob.X)
    lin = pd.assemble_system(pd.make_tableau(3), pd.assemble_space(mesh), pd.TimeGrid(4, 1.0), 0.0,
                             prob.u0(mesh.vertices))
    np.testing.assert_allclose(lin.solve_sequential(), g["seq"], rtol=1e-11, atol=1e-13)
    # one global banded solve gives the same space-time solution
    assert per_node_rel(lin.solve_direct(), g["seq"], (4, 3, 17)) < 1e-10
    # BASELINE config 1 at full size (127 points, 16 steps, M=3)
    c1 = golden("c1")
    cfg = pd.baseline_config("C1")
    s = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                           pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    assert per_node_rel(s.solve_sequential(), c1["seq"], (cfg.Nt, cfg.M, cfg.spec.ndof)) < 1e-10
    assert per_node_rel(s.solve_direct(), c1["seq"], (cfg.Nt, cfg.M, cfg.spec.ndof)) < 1e-10


def test_nonlinear_sequential_and_direct_match_oracle():
    """gamma > 0: element Newton with refactored banded Jacobians (spacetime.py:154-167)
    and the global Newton (:185-195) vs the oracle's restatement."""
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(16, prob.X)
    s = pd.assemble_system(pd.make_tableau(3), pd.assemble_space(mesh), pd.TimeGrid(4, prob.T),
                           prob.gamma, prob.u0(mesh.vertices))
    Kh, mh = O.fem1d_operators(16, prob.X)
    so = O.OSystem(O.tableau(3), Kh, mh, 4, prob.T, prob.gamma, prob.u0(mesh.vertices))
    ref = so.solve_sequential()
    seq = s.solve_sequential()
    assert per_node_rel(seq, ref, (4, 3, 17)) < 1e-10
    direct = s.solve_direct()
    assert per_node_rel(direct, ref, (4, 3, 17)) < 1e-9
    assert np.linalg.norm(s.residual(direct)) <= 1e-11 * max(1.0, np.linalg.norm(s.rhs()))


def test_element_solve_2d_fd_band():
    """A 2D FD element (point-major band of half width M*n + M - 1) vs SuperLU."""
    cfg = pd.baseline_config("C2", n=15, Nt=2)
    s = pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                           pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    ref = O.OSystem(O.tableau(cfg.M), pd.fd_space(cfg.spec).Kh,
                    pd.fd_space(cfg.spec).lumped_diagonal, cfg.Nt, cfg.T, 0.0,
                    cfg.u0()).solve_sequential()
    assert per_node_rel(s.solve_sequential(), ref, (cfg.Nt, cfg.M, cfg.spec.ndof)) < 1e-10


@pytest.mark.parametrize("n,dim,W", [(5, 2, 3), (31, 3, 2), (127, 2, 1), (40, 3, 1), (130, 2, 2),
                                     (65, 3, 5), (100, 3, 2), (63, 3, 8), (33, 3, 40)])
def test_mode_product_matches_einsum(n, dim, W):
    """The hand-written FP64 mode product (pd_modeprod.cu, no library) along every axis
    of W stacked n^dim grids, with Phi and Phi^T, vs numpy (fp64 summation-order
    tolerance).  The last four shapes are wide enough for the DMMA (tensor) kernels."""
    import torch

    from paper_2006_12883_b200 import _native as N

    rng = np.random.default_rng(n)
    phi = rng.standard_normal((n, n))
    X = rng.standard_normal((W,) + (n,) * dim)
    ctx = N.context()
    xd, pd_ = N.to_device(X.ravel(), ctx), N.to_device(phi.ravel(), ctx)
    out = N.empty(X.size, ctx)
    for axis in range(dim):
        stride = n ** (dim - 1 - axis)
        for tr in (0, 1):
            N.call("pd_mode_product", ctx.handle, N.ptr(xd), N.ptr(out), X.size, n, stride,
                   N.ptr(pd_), tr)
            torch.cuda.synchronize()
            mat = phi.T if tr else phi
            ref = np.moveaxis(np.tensordot(mat, X, axes=([1], [axis + 1])), 0, axis + 1)
            got = N.to_host(out).reshape(X.shape)
            assert np.max(np.abs(got - ref)) <= 1e-12 * n * np.max(np.abs(ref))
