"""Parity AT SIZE against the real reference (fixtures: tests/golden/make_golden_sized.py).

The reference was run here on the benchmarked configuration itself (BASELINE C2:
255^2 x 64 steps x M=3, SMG L=7, P=8) and on the survey's reduced sizes of the other
configs (Appendix A): STMG 63^2 x 64 (L=6, P=8) and STMG on C2 itself (40 cycles, stagnating),
C3 128^2 x 32 periodic Fisher
(Newton + SMG and PFASST IMEX over 4 windows), C4 31^3 x 16 (PFASST M=5/3 at P=4/8
and tol 1e-9/1e-10, multi-window; SMG), C5 16^3 x 8 periodic cubic (Newton + STMG).

Checked: equal iteration counts (MG cycles, Newton steps and inner counts, PFASST
per-window counts and converged/diverged flags); the residual history; per-node
relative L2 of the full first and last time steps; every (step, node) slab's norm and
4 seeded Gaussian projections (pd_util.slab_projections).  The parity metric is
printed both ways: strict (each node against its own norm) and floored at 1e-3 x the
largest node norm (pd_util.per_node_rel).
"""

import numpy as np
import pytest

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import pfasst as PF
from pd_util import per_node_rel, per_node_rel_strict, slab_projections

pytestmark = pytest.mark.gpu
TOL = 1e-10


def compare(x, g, prefix, shape, tol=TOL, full=True):
    """Assert parity of solution x with fixture entries `prefix_*`; returns metrics."""
    X = np.asarray(x).reshape(shape)
    norms = np.linalg.norm(X, axis=-1)
    ref_n = g[prefix + "_norms"]
    scale = np.maximum(ref_n, 1e-3 * ref_n.max())
    out = {"norms_floored": float(np.max(np.abs(norms - ref_n) / scale)),
           "norms_strict": float(np.max(np.abs(norms - ref_n) / np.maximum(ref_n, 1e-300)))}
    gk = np.linalg.norm(np.random.default_rng(12345).standard_normal((4, shape[-1])), axis=1)
    dp = np.abs(slab_projections(X) - g[prefix + "_proj"]) / gk
    out["proj_floored"] = float(np.max(dp / scale[..., None]))
    out["proj_strict"] = float(np.max(dp / np.maximum(ref_n, 1e-300)[..., None]))
    if full and prefix + "_first" in g:
        for which, sl in (("first", X[0]), ("last", X[-1])):
            ref = g[f"{prefix}_{which}"]
            out[f"{which}_floored"] = per_node_rel(sl, ref, ref.shape)
            out[f"{which}_strict"] = per_node_rel_strict(sl, ref, ref.shape)
    print(prefix, {k: f"{v:.2e}" for k, v in out.items()})
    for k, v in out.items():
        if k.endswith("floored"):
            assert v < tol, (prefix, k, v)
    return out


def assert_history(rep, g, prefix, rel=1e-6):
    ref = g[prefix + "_hist"]
    got = np.asarray(rep.residual_history)
    assert got.shape == ref.shape, (prefix, got.shape, ref.shape)
    np.testing.assert_allclose(got, ref, rtol=rel, atol=1e-300)


@pytest.fixture(scope="module")
def c2_system():
    cfg = pd.baseline_config("C2")
    return cfg, pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec),
                                   pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())


def test_c2_full_size_smg_matches_reference(golden, c2_system):
    """The benchmarked configuration, solved to 1e-10, against the reference's own run."""
    g = golden("sized_c2_full")
    cfg, s = c2_system
    h = pd.build_hierarchy(s, "SMG", 7, 3, partitions=8)
    x, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    assert rep.converged and rep.iterations == int(g["smg_its"]) == 3
    assert_history(rep, g, "smg")
    compare(x, g, "smg", (cfg.Nt, 3, cfg.spec.ndof))


def test_stmg_on_c2_stagnates_like_the_reference(golden, c2_system):
    """Why the bench solves C2 with SMG: the reference's STMG (L=7, P=8) on the full C2
    system stagnates near 1.4e-4 (40 cycles, flagged diverged at the cap); the device
    path follows the same residual history."""
    g = golden("sized_stmg_c2")
    cfg, s = c2_system
    h = pd.build_hierarchy(s, "STMG", 7, 3, partitions=8)
    cap = int(g["max_cycles"])
    x, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10, max_cycles=cap)
    assert rep.iterations == int(g["stmg_its"]) == cap
    assert rep.converged == bool(g["stmg_conv"]) and rep.diverged == bool(g["stmg_div"])
    assert not rep.converged
    assert_history(rep, g, "stmg", rel=1e-4)
    assert rep.residual_history[-1] > 1e-2 * rep.residual_history[0]


def test_stmg_63_matches_reference(golden):
    """STMG (space + time coarsening) at 63^2 x 64 x 3, L=6, P=8: the reference needs 67
    cycles (the survey's 46 were another configuration); equal count on the device."""
    g = golden("sized_stmg63")
    spec = pd.StencilSpec(2, 63, "dirichlet", 1.0)
    cfg = pd.BaselineConfig("C2", spec, 64, 1.0, 3, 2, 0.0, "cubic", 0, "reduced 63^2")
    s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(spec), pd.TimeGrid(64, 1.0), 0.0,
                           cfg.u0())
    h = pd.build_hierarchy(s, "STMG", 6, 3, partitions=8)
    x, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    assert rep.converged and rep.iterations == int(g["stmg_its"])
    assert_history(rep, g, "stmg", rel=1e-5)
    compare(x, g, "stmg", (64, 3, spec.ndof))


def test_c3_128_newton_and_pfasst_match_reference(golden):
    g = golden("sized_c3_128")
    cfg = pd.baseline_config("C3", n=128, Nt=32)
    ops = pd.fd_space(cfg.spec)
    np.testing.assert_array_equal(cfg.u0(), g["u0"])
    s = pd.assemble_system(pd.make_tableau(3), ops, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma,
                           cfg.u0(), reaction_kind="fisher")
    h = pd.build_hierarchy(s, "SMG", 6, 3)
    x, rep = pd.newton_solve(s, pd.mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9), tol=1e-9)
    assert rep.converged and rep.iterations == int(g["newton_its"])
    assert rep.inner_iterations == g["newton_inner"].tolist()
    assert rep.damped_steps == int(g["newton_damped"])
    compare(x, g, "newton", (cfg.Nt, 3, cfg.spec.ndof))
    # PFASST IMEX, P=8 over 4 windows: the reference converges window 1 in 20
    # iterations and trips its divergence test in window 2 (pfasst.py:471-472, 496-506)
    hier = PF.build_pfasst_hierarchy(3, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma, L=2,
                                     nu=1, mode="imex", space=ops, M_coarse=2,
                                     reaction_kind="fisher")
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, 8, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["pf_inner"].tolist()
    assert rep.iterations == int(g["pf_its"])
    assert bool(rep.converged) == bool(g["pf_conv"]) and bool(rep.diverged) == bool(g["pf_div"])


@pytest.mark.parametrize("P,tol", [(4, 1e-9), (4, 1e-10), (8, 1e-9), (8, 1e-10)])
def test_c4_31_pfasst_windows_match_reference(golden, P, tol):
    """3D PFASST (M=5 / coarse 3) over 2-4 windows.  At tol 1e-10 the reference's second
    window runs to the iteration cap (n.c.): the device path reproduces that per-window
    behaviour, not just the first window."""
    g = golden("sized_c4_31")
    key = f"pf_P{P}_t{int(round(-np.log10(tol)))}"
    cfg = pd.baseline_config("C4", n=31, Nt=16)
    ops = pd.fd_space(cfg.spec)
    hier = PF.build_pfasst_hierarchy(5, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, L=2, nu=1,
                                     space=ops, M_coarse=3)
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, P, tol_rel=tol, tol_abs=tol, max_iters=200)
    ref_inner, ref_hist = g[key + "_inner"].tolist(), g[key + "_hist"]
    print(key, "device inner", rep.inner_iterations, rep.residual_history,
          "reference", ref_inner, ref_hist.tolist())
    w = next((i for i, (a, b) in enumerate(zip(rep.inner_iterations, ref_inner)) if a != b), None)
    if w is None:
        assert rep.inner_iterations == ref_inner
        assert bool(rep.converged) == bool(g[key + "_conv"])
        if rep.converged:
            compare(x, g, key, (cfg.Nt, 5, cfg.spec.ndof))
        return
    # knife edge: a window whose residual floor sits at the
    # threshold stops in one run and stalls to the cap in the other; earlier windows
    # must agree exactly and the two runs' residuals in that window must be equal to
    # rounding of the floor (later windows start from different states)
    assert 200 in (rep.inner_iterations[w], ref_inner[w]), (w, rep.inner_iterations, ref_inner)
    ratio = rep.residual_history[w] / ref_hist[w]
    print(f"  knife edge in window {w}: residual ratio device/reference {ratio:.4f}")
    assert abs(ratio - 1.0) < 0.05


def test_c4_31_smg_matches_reference(golden):
    g = golden("sized_c4_31")
    cfg = pd.baseline_config("C4", n=31, Nt=16)
    s = pd.assemble_system(pd.make_tableau(5), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                           0.0, cfg.u0())
    h = pd.build_hierarchy(s, "SMG", 4, 3, partitions=2)
    x, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    assert rep.converged and rep.iterations == int(g["smg_its"])
    compare(x, g, "smg", (cfg.Nt, 5, cfg.spec.ndof))


def test_c5_16_newton_stmg_matches_reference(golden):
    g = golden("sized_c5_16")
    cfg = pd.baseline_config("C5", n=16, Nt=8)
    s = pd.assemble_system(pd.make_tableau(3), pd.fd_space(cfg.spec), pd.TimeGrid(cfg.Nt, cfg.T),
                           cfg.gamma, cfg.u0())
    h = pd.build_hierarchy(s, "STMG", 3, 3)
    x, rep = pd.newton_solve(s, pd.mg_linear_solver(h, tol_rel=1e-8, tol_abs=1e-8), tol=1e-8)
    assert rep.converged and rep.iterations == int(g["newton_its"])
    assert rep.inner_iterations == g["newton_inner"].tolist()
    compare(x, g, "newton", (cfg.Nt, 3, cfg.spec.ndof))
