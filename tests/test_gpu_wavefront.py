"""GPU parity of the structured wavefront ILU(0) sweeps (csrc/pd_wavefront.cu).

The wavefront executor only reschedules rows; every row still accumulates in
CSR order with separately rounded operations, so solves must be bitwise those
of the numba reference (restated by oracle/ilu0.c, pinned to the golden
vectors in test_oracle_golden.py) — for the fine space-time matrix, for
Galerkin coarse levels (9/27-point couplings), for block-Jacobi masking, for
periodic wrap-around and for 3D planes.
"""

import numpy as np
import pytest

import paper_2006_12883_b200 as pd
from oracle import paradiff_oracle as O

pytestmark = pytest.mark.gpu


def _system(name, n, Nt):
    cfg = pd.baseline_config(name, n=n, Nt=Nt)
    return cfg, pd.assemble_system(pd.make_tableau(cfg.M), pd.fd_space(cfg.spec),
                                   pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())


def _check(A, ngroup, nline, npoint, parts, seed=0, repeats=2, applies=True, ngroup_lower=0,
           kind=None):
    A = pd.linalg.as_csr(A)
    rng = np.random.default_rng(seed)
    dev = pd.BlockJacobiPrecond(A, parts) if parts > 1 else pd.Ilu0(A)
    assert dev.set_wavefront(ngroup, nline, npoint, ngroup_lower) == applies
    if kind is not None:
        assert dev.sweep_kind() in (kind if isinstance(kind, tuple) else (kind,))
    ref = O.OBlockJacobi(A, parts) if parts > 1 else O.OIlu0(A)
    for _ in range(repeats):  # repeated solves exercise the re-arming protocol
        b = rng.standard_normal(A.shape[0])
        np.testing.assert_array_equal(dev.solve(b), ref.solve(b))


@pytest.mark.parametrize("parts", [1, 2, 4])
def test_wavefront_fine_2d_bitwise(parts):
    cfg, s = _system("C2", 15, 8)
    _check(s.global_matrix(), cfg.M, cfg.spec.n, cfg.spec.n, parts)


def test_wavefront_periodic_2d_bitwise():
    """Periodic wrap-around: the far in-line neighbour is read back from global memory."""
    cfg, s = _system("C3", 16, 4)
    assert cfg.spec.bc == "periodic"
    _check(s.global_matrix(), cfg.M, cfg.spec.n, cfg.spec.n, 2)


def test_wavefront_3d_planes_fall_back():
    """3D planes couple to many other planes: not a wavefront task; level sweeps stay."""
    cfg, s = _system("C4", 7, 4)
    assert cfg.spec.dim == 3
    _check(s.global_matrix(), 1, cfg.spec.n, cfg.spec.n, 2, applies=False)


def test_wavefront_single_group_ring_and_globals_bitwise(monkeypatch):
    """One node grid per task (M=1 layout view): node couplings become globals
    (pattern-table executor)."""
    monkeypatch.setenv("PD_WF2", "0")
    cfg, s = _system("C2", 15, 4)
    A = pd.linalg.as_csr(s.global_matrix())
    # a 2-group task view of a 1-node-per-task split still has <= 2 globals per row
    _check(A, cfg.M, cfg.spec.n, cfg.spec.n, 4, seed=3)


@pytest.mark.parametrize("wf2", ["1", "0"])
def test_wavefront_galerkin_levels_bitwise(monkeypatch, wf2):
    monkeypatch.setenv("PD_WF2", wf2)
    cfg, s = _system("C2", 31, 8)
    h = pd.build_hierarchy(s, "SMG", 4, 2, partitions=2)
    assert h.wavefront == [True, True, True]
    spec = cfg.spec
    for l, A in enumerate(h.matrices[:-1]):
        _check(A, cfg.M, spec.n, spec.n, 2, seed=l)
        spec = spec.coarse()


@pytest.mark.parametrize("k", [2, 4])
def test_wavefront_multistep_lower_tasks_bitwise(monkeypatch, k):
    """Lower-sweep tasks spanning k time steps (time coupling through the ring;
    pattern-table executor, the template executor pinned off)."""
    monkeypatch.setenv("PD_WF2", "0")
    cfg, s = _system("C2", 15, 8)
    _check(s.global_matrix(), cfg.M, cfg.spec.n, cfg.spec.n, 2, seed=k, ngroup_lower=cfg.M * k)
    h = pd.build_hierarchy(s, "SMG", 3, 2, partitions=2)
    spec = cfg.spec.coarse()
    _check(h.matrices[1], cfg.M, spec.n, spec.n, 2, seed=k + 1, ngroup_lower=cfg.M * k)


def test_wavefront_rejects_mismatched_layout():
    cfg, s = _system("C2", 15, 4)
    ilu = pd.Ilu0(s.global_matrix())
    assert not ilu.set_wavefront(3, 14, 15)  # task size does not divide the system
    b = np.ones(s.size)
    np.testing.assert_array_equal(ilu.solve(b), O.OIlu0(pd.linalg.as_csr(s.global_matrix())).solve(b))


@pytest.mark.parametrize("strategy", ["SMG", "STMG"])
def test_wavefront_mg_bitwise_vs_level_sweeps(monkeypatch, strategy):
    """Same V-cycles with and without the wavefront executor: bitwise equal.

    SMG levels all take the wavefront path; STMG's time-coarsened level couples
    to every node of the previous coarse step (too many cross-task entries) and
    keeps the level-scheduled sweeps.
    """
    cfg, s = _system("C2", 31, 8)
    b = s.rhs()
    out = {}
    for mode in ("level", "wavefront"):
        if mode == "level":
            monkeypatch.setenv("PD_NO_WAVEFRONT", "1")
        else:
            monkeypatch.delenv("PD_NO_WAVEFRONT", raising=False)
        h = pd.build_hierarchy(s, strategy, 3, 2, partitions=2)
        if mode == "level":
            assert h.wavefront == [False, False]
        else:
            assert h.wavefront == ([True, True] if strategy == "SMG" else [True, False])
        out[mode] = h.solve(b, tol_rel=1e-10, tol_abs=1e-10)
    (x1, r1), (x2, r2) = out["level"], out["wavefront"]
    assert r1.iterations == r2.iterations and r1.converged
    np.testing.assert_array_equal(x1, x2)


def test_grid_spmv_galerkin_levels_bitwise(monkeypatch):
    """Structured SpMV (pd_csr_set_grid) on SMG Galerkin levels: every level's product
    is bitwise scipy's; whole solves match the CSR path with equal cycle counts (the
    fused residual norms reduce over a different block tree, so GMRES scalars may
    differ in the last bit: rel 1e-12)."""
    from paper_2006_12883_b200 import _native as N

    cfg, s = _system("C2", 31, 8)
    h = pd.build_hierarchy(s, "SMG", 4, 2, partitions=2)
    assert h.grid_spmv[1:3] == [True, True]
    rng = np.random.default_rng(5)
    for l in range(1, 4):
        A = h.matrices[l]
        x = rng.standard_normal(A.shape[1])
        got = h._dev_mats[l].matvec_dev(N.to_device(x)).cpu().numpy()
        np.testing.assert_array_equal(got, pd.linalg.as_csr(A) @ x)
    b = s.rhs()
    x1, r1 = h.solve(b, tol_rel=1e-10, tol_abs=1e-10)
    monkeypatch.setenv("PD_NO_GRID_SPMV", "1")
    h2 = pd.build_hierarchy(s, "SMG", 4, 2, partitions=2)
    assert not any(h2.grid_spmv)
    x2, r2 = h2.solve(b, tol_rel=1e-10, tol_abs=1e-10)
    assert r1.iterations == r2.iterations and r1.converged
    assert np.linalg.norm(x1 - x2) <= 1e-12 * np.linalg.norm(x2)


# ---- template-structured skewed wavefront (csrc/pd_wf2.cu) -------------------------
@pytest.mark.parametrize("n,parts", [(15, 1), (31, 2), (63, 4), (127, 8)])
def test_wf2_fine_level_bitwise(n, parts):
    """Fine level (5-point x M x M, point coupling to the previous step), every
    line-block size class (NLP 32/64/128): template upper sweep with the pattern-table
    lower sweep (kind 3, the default on FINE5 levels) and both template sweeps (kind 2,
    PD_WF2_LOWER=all), bitwise the numba reference."""
    cfg, s = _system("C2", n, 8)
    _check(s.global_matrix(), cfg.M, n, n, parts, seed=n, kind=3)


@pytest.mark.parametrize("n,parts", [(15, 1), (63, 4), (127, 8)])
def test_wf2_fine_level_template_lower_bitwise(monkeypatch, n, parts):
    monkeypatch.setenv("PD_WF2_LOWER", "all")
    cfg, s = _system("C2", n, 8)
    _check(s.global_matrix(), cfg.M, n, n, parts, seed=n + 1, kind=2)


@pytest.mark.parametrize("n,parts", [(31, 1), (63, 2), (127, 8)])
def test_wf2_galerkin_levels_bitwise(n, parts):
    """SMG Galerkin levels (9-point x M x M, 3x3 coupling to the previous step)."""
    cfg, s = _system("C2", n, 8)
    h = pd.build_hierarchy(s, "SMG", 3, 2, partitions=parts)
    spec = cfg.spec
    for l, A in enumerate(h.matrices[:-1]):
        _check(A, cfg.M, spec.n, spec.n, parts, seed=l, kind=3 if l == 0 else 2)
        spec = spec.coarse()


def test_wf2_equals_pattern_table_executor(monkeypatch):
    """Both wavefront executors on a 127^2 fine level and its Galerkin level: bitwise."""
    cfg, s = _system("C2", 127, 8)
    h = pd.build_hierarchy(s, "SMG", 3, 2, partitions=8)
    rng = np.random.default_rng(11)
    spec = cfg.spec
    for A in h.matrices[:-1]:
        A = pd.linalg.as_csr(A)
        b = rng.standard_normal(A.shape[0])
        outs = []
        for flag, kinds in (("1", (2, 3)), ("0", (1,))):
            monkeypatch.setenv("PD_WF2", flag)
            dev = pd.BlockJacobiPrecond(A, 8)
            assert dev.set_wavefront(cfg.M, spec.n, spec.n)
            assert dev.sweep_kind() in kinds
            outs.append(dev.solve(b))
        np.testing.assert_array_equal(outs[0], outs[1])
        spec = spec.coarse()


def test_wf2_refactor_refreshes_values():
    """A values-only refactor (Newton) regathers the step blocks."""
    cfg, s = _system("C2", 31, 4)
    A = pd.linalg.as_csr(s.global_matrix())
    dev = pd.BlockJacobiPrecond(A, 2)
    assert dev.set_wavefront(cfg.M, 31, 31) and dev.sweep_kind() in (2, 3)
    A2 = A.copy()
    A2.data = A2.data * (1.0 + 0.01 * np.random.default_rng(2).standard_normal(A2.nnz))
    dev.update_values(A2)
    b = np.random.default_rng(3).standard_normal(A.shape[0])
    np.testing.assert_array_equal(dev.solve(b), O.OBlockJacobi(A2, 2).solve(b))
