"""GPU parity of the SDC/PFASST path vs golden fixtures from the real reference.

Bar (BASELINE north_star): equal PFASST iteration counts (max over windows and
per window) and per-time-node relative L2 <= 1e-10 (pd_util.per_node_rel).
The device node solves are exact factorizations applied as refinement; the
reference's GMRES(ILU) reaches 1e-13, so single-sweep results agree to ~1e-13.
"""

import numpy as np
import pytest

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200 import pfasst as PF
from oracle import paradiff_oracle as O
from pd_util import per_node_rel, rel_l2

pytestmark = pytest.mark.gpu


def _heat_u0(Nx):
    return pd.heat_problem().u0(pd.SpaceMesh(Nx, 1.0).vertices)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_c1_pfasst_matches_reference(golden, P):
    g = golden("c1")
    cfg = pd.baseline_config("C1")
    ops = pd.fd_space(cfg.spec)
    hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, L=2,
                                     nu=1, space=ops, M_coarse=cfg.M_coarse)
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, P, tol_rel=1e-10, tol_abs=1e-10)
    assert rep.converged
    assert rep.inner_iterations == g[f"PF_P{P}_inner"].tolist()
    assert rep.iterations == int(g[f"PF_P{P}_its"])
    assert per_node_rel(x, g[f"PF_P{P}_x"], (16, 3, 127)) < 1e-10


def test_pfasst_fem1d_heat_matches_reference(golden):
    g = golden("pfasst_fem1d")
    mesh = pd.SpaceMesh(32, 1.0)
    for P in (1, 2, 4):
        hier = PF.build_pfasst_hierarchy(3, mesh, pd.TimeGrid(8, 1.0), 0.0, L=2, nu=1)
        x, rep = PF.pfasst_run(hier, _heat_u0(32), 8, P, tol_rel=1e-10, tol_abs=1e-10)
        assert rep.inner_iterations == g[f"heat_P{P}_inner"].tolist(), P
        assert per_node_rel(x, g[f"heat_P{P}_x"], (8, 3, 33)) < 1e-10
    hier = PF.build_pfasst_hierarchy(2, mesh, pd.TimeGrid(8, 1.0), 0.0, L=3, nu=1)
    x, rep = PF.pfasst_run(hier, _heat_u0(32), 8, 4, tol_rel=1e-10, tol_abs=1e-10)
    assert rep.inner_iterations == g["heatL3_P4_inner"].tolist()
    assert per_node_rel(x, g["heatL3_P4_x"], (8, 2, 33)) < 1e-10


def test_pfasst_monodomain_imex_matches_reference(golden):
    g = golden("pfasst_fem1d")
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(64, prob.X)
    hier = PF.build_pfasst_hierarchy(2, mesh, pd.TimeGrid(16, prob.T), prob.gamma, L=2, nu=1,
                                     mode="imex")
    x, rep = PF.pfasst_run(hier, prob.u0(mesh.vertices), 16, 4, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["mono_imex_inner"].tolist()
    assert per_node_rel(x, g["mono_imex_x"], (16, 2, 65)) < 1e-9


def test_sweep_fas_residual_match_reference(golden):
    g = golden("pfasst_fem1d")
    hier = PF.build_pfasst_hierarchy(3, pd.SpaceMesh(32, 1.0), pd.TimeGrid(8, 1.0), 0.0, L=2,
                                     nu=1)
    u0 = _heat_u0(32)
    st = PF.SweeperState(g["sweep_U_in"].copy(), u0.copy())
    np.testing.assert_allclose(hier.fine.sweep(st).U, g["sweep_U_out"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(
        PF.fas_correction(hier.levels[0], hier.levels[1], hier.transfers[0], st), g["fas_tau"],
        rtol=0, atol=1e-12)
    assert abs(hier.fine.residual_norm(st) - float(g["resnorm"])) < 1e-12
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(64, prob.X)
    lv = PF.SdcLevel(pd.make_tableau(3), pd.assemble_space(mesh), 0.05, prob.gamma, "imex")
    u0m = prob.u0(mesh.vertices)
    np.testing.assert_allclose(lv.sweep(PF.spread_state(u0m, 3)).U, g["imex_sweep"], atol=1e-12)
    s, rp = PF.sdc_solve_step(u0m, lv, tol_rel=1e-10, tol_abs=1e-10)
    assert rp.iterations == int(g["sdc_step_its"])
    np.testing.assert_allclose(s.U, g["sdc_step_U"], atol=1e-10)


def test_c2_small_pfasst_dense_node_solves(golden):
    g = golden("c2_small")
    spec = pd.StencilSpec(2, 15, "dirichlet", 1.0)
    ops = pd.fd_space(spec)
    hier = PF.build_pfasst_hierarchy(3, ops.mesh, pd.TimeGrid(8, 8 / 64), 0.0, L=2, nu=1,
                                     space=ops, M_coarse=2)
    x, rep = PF.pfasst_run(hier, g["u0"], 8, 4, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["PF_P4_inner"].tolist()
    assert per_node_rel(x, g["PF_P4_x"], (8, 3, 225)) < 1e-10


def test_worker_count_validation():
    mesh = pd.SpaceMesh(16, 1.0)
    hier = PF.build_pfasst_hierarchy(2, mesh, pd.TimeGrid(6, 1.0), 0.0, L=1, nu=1)
    with pytest.raises(pd.ConfigurationError):
        PF.pfasst_run(hier, np.zeros(17), 6, 4)


def test_divergent_window_reports_nc():
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(128, prob.X)
    hier = PF.build_pfasst_hierarchy(4, mesh, pd.TimeGrid(4, prob.T), prob.gamma, L=2, nu=1,
                                     mode="imex")
    u, rep = PF.pfasst_run(hier, prob.u0(mesh.vertices), 4, 4, max_iters=150)
    assert not rep.converged and rep.diverged


def test_pfasst_monodomain_implicit_newton_node_solves(golden):
    """Implicit mode: nonlinear node solves by on-device Newton (pfasst.py:134-152)."""
    g = golden("pfasst_fem1d")
    prob = pd.monodomain_problem()
    mesh = pd.SpaceMesh(64, prob.X)
    hier = PF.build_pfasst_hierarchy(2, mesh, pd.TimeGrid(16, prob.T), prob.gamma, L=2, nu=1,
                                     mode="implicit")
    x, rep = PF.pfasst_run(hier, prob.u0(mesh.vertices), 16, 4, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["mono_implicit_inner"].tolist()
    assert per_node_rel(x, g["mono_implicit_x"], (16, 2, 65)) < 1e-9


@pytest.mark.parametrize("solver", ["gmres", "spectral", "dense"])
def test_c2_small_pfasst_node_solvers(golden, monkeypatch, solver):
    """Node solves by the reference's own ILU(0)-GMRES(30) on device (pfasst.py:118-132,
    the default), and the exact alternatives (tensor-product eigen-solve, dense LU)."""
    monkeypatch.setenv("PD_NODE_SOLVER", solver)
    g = golden("c2_small")
    spec = pd.StencilSpec(2, 15, "dirichlet", 1.0)
    ops = pd.fd_space(spec)
    hier = PF.build_pfasst_hierarchy(3, ops.mesh, pd.TimeGrid(8, 8 / 64), 0.0, L=2, nu=1,
                                     space=ops, M_coarse=2)
    x, rep = PF.pfasst_run(hier, g["u0"], 8, 4, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["PF_P4_inner"].tolist()
    assert per_node_rel(x, g["PF_P4_x"], (8, 3, 225)) < 1e-10


def test_reduced_baseline_configs_on_device(golden):
    """C3/C4/C5 at reduced size on the GPU path vs the real reference's fixtures."""
    g = golden("configs_reduced")
    # C3: Newton + STMG (Fisher) and PFASST IMEX
    cfg = pd.baseline_config("C3", n=16, Nt=8)
    ops = pd.fd_space(cfg.spec)
    s = pd.assemble_system(pd.make_tableau(3), ops, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma,
                           cfg.u0(), reaction_kind="fisher")
    h = pd.build_hierarchy(s, "STMG", 2, 3)
    x, rep = pd.newton_solve(s, pd.mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9), tol=1e-9)
    assert rep.iterations == int(g["c3_newton_its"])
    assert rep.inner_iterations == g["c3_newton_inner"].tolist()
    assert per_node_rel(x, g["c3_newton_x"], (8, 3, 256)) < 1e-10
    hier = PF.build_pfasst_hierarchy(3, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma, L=2,
                                     nu=1, mode="imex", space=ops, M_coarse=2,
                                     reaction_kind="fisher")
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, 4, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["c3_pf_inner"].tolist()
    assert per_node_rel(x, g["c3_pf_x"], (8, 3, 256)) < 1e-10
    # C4: 3D PFASST M=5 / coarse 3 and SMG
    cfg = pd.baseline_config("C4", n=7, Nt=8)
    ops = pd.fd_space(cfg.spec)
    hier = PF.build_pfasst_hierarchy(5, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, L=2, nu=1,
                                     space=ops, M_coarse=3)
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, 4, tol_rel=1e-9, tol_abs=1e-9)
    assert rep.inner_iterations == g["c4_pf_inner"].tolist()
    assert per_node_rel(x, g["c4_pf_x"], (8, 5, 343)) < 1e-10
    s = pd.assemble_system(pd.make_tableau(5), ops, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, cfg.u0())
    h = pd.build_hierarchy(s, "SMG", 2, 3, partitions=2)
    x, rep = h.solve(s.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    assert rep.iterations == int(g["c4_smg_its"])
    assert per_node_rel(x, g["c4_smg_x"], (8, 5, 343)) < 1e-10
    # C5: 3D periodic cubic Newton + STMG
    cfg = pd.baseline_config("C5", n=8, Nt=4)
    ops = pd.fd_space(cfg.spec)
    s = pd.assemble_system(pd.make_tableau(3), ops, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma,
                           cfg.u0())
    h = pd.build_hierarchy(s, "STMG", 2, 3)
    x, rep = pd.newton_solve(s, pd.mg_linear_solver(h, tol_rel=1e-8, tol_abs=1e-8), tol=1e-8)
    assert rep.iterations == int(g["c5_newton_its"])
    assert rep.inner_iterations == g["c5_newton_inner"].tolist()
    assert per_node_rel(x, g["c5_newton_x"], (4, 3, 512)) < 1e-10


@pytest.mark.parametrize("name,n", [("C2", 15), ("C4", 7)])
def test_structured_stencil_f_evaluations_bitwise(monkeypatch, name, n):
    """Grid-stencil f(U) = -Kh U / mh (k_bstencil) is bitwise the CSR k_bspmv path:
    whole PFASST runs agree to the last bit with the structured kernel disabled."""
    cfg = pd.baseline_config(name, n=n, Nt=4)
    ops = pd.fd_space(cfg.spec)
    out = []
    for disable in (True, False):
        if disable:
            monkeypatch.setenv("PD_NO_GRID_STENCIL", "1")
        else:
            monkeypatch.delenv("PD_NO_GRID_STENCIL", raising=False)
        hier = PF.build_pfasst_hierarchy(cfg.M, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), 0.0, L=2,
                                         nu=1, space=ops, M_coarse=cfg.M_coarse)
        out.append(PF.pfasst_run(hier, cfg.u0(), cfg.Nt, 4, 1e-10, 1e-10))
    (x1, r1), (x2, r2) = out
    assert r1.iterations == r2.iterations and r1.converged
    np.testing.assert_array_equal(x1, x2)


def test_pfasst_implicit_newton_general_kh_matches_oracle():
    """Implicit mode with gamma > 0 on a 2D periodic 5-point Kh (not tridiagonal):
    per-worker Newton node solves with GMRES(30)+ILU(0) of J (pfasst.py:134-152)
    on the device vs the oracle's restatement: equal counts, per-node rel <= 1e-9."""
    cfg = pd.baseline_config("C3", n=8, Nt=4)
    ops = pd.fd_space(cfg.spec)
    hier = PF.build_pfasst_hierarchy(3, ops.mesh, pd.TimeGrid(cfg.Nt, cfg.T), cfg.gamma, L=2,
                                     nu=1, mode="implicit", space=ops, M_coarse=2,
                                     reaction_kind="fisher")
    x, rep = PF.pfasst_run(hier, cfg.u0(), cfg.Nt, 2, tol_rel=1e-9, tol_abs=1e-9)
    spc = cfg.spec.coarse()
    cops = pd.fd_space(spc)
    tf, tc = O.tableau(3), O.tableau(2)
    lv = [O.OSdcLevel(tf, ops.Kh, ops.lumped_diagonal, cfg.dt, cfg.gamma, mode="implicit",
                      reaction="fisher"),
          O.OSdcLevel(tc, cops.Kh, cops.lumped_diagonal, cfg.dt, cfg.gamma, mode="implicit",
                      reaction="fisher")]
    Rs, Ps = pd.fd_transfers(cfg.spec)
    trs = [O.OTransfer(Rs, Ps, O.node_eval(tf.nodes, tc.nodes), O.node_eval(tc.nodes, tf.nodes))]
    xo, ro = O.pfasst(lv, trs, 1, cfg.u0(), cfg.Nt, 2, 1e-9, 1e-9)
    assert rep.converged and ro.converged
    assert rep.iterations == ro.iterations and rep.inner_iterations == ro.inner_iterations
    assert per_node_rel(x, xo, (cfg.Nt, 3, cfg.spec.ndof)) < 1e-9


def test_lu_trick_qdelta_matches_reference(golden):
    """the "lu-trick" Q_delta (collocation.py:119-123) through the device
    sweeps — one sweep, a single-step SDC solve, PFASST on the heat problem and IMEX
    PFASST on the monodomain problem vs runs of the real reference
    (tests/golden/make_golden_lutrick.py)."""
    g = golden("lutrick")
    heat = pd.heat_problem()
    mesh = pd.SpaceMesh(32, heat.X)
    u0 = heat.u0(mesh.vertices)
    hier = PF.build_pfasst_hierarchy(3, mesh, pd.TimeGrid(8, heat.T), 0.0, L=2, nu=1,
                                     qdelta="lu-trick")
    np.testing.assert_allclose(hier.fine.sweep(PF.spread_state(u0, 3)).U, g["heat_sweep1"],
                               rtol=0, atol=1e-12)
    st, rep = PF.sdc_solve_step(u0, hier.fine, tol_rel=1e-11, tol_abs=1e-12)
    assert rep.iterations == int(g["heat_step_its"])
    np.testing.assert_allclose(st.U, g["heat_step_U"], rtol=0, atol=1e-10)
    x, rp = PF.pfasst_run(hier, u0, 8, 4, tol_rel=1e-10, tol_abs=1e-10)
    assert rp.converged == bool(g["heat_conv"])
    assert rp.inner_iterations == g["heat_its"].tolist()
    assert per_node_rel(x, g["heat_U"], (8, 3, 33)) < 1e-10
    mono = pd.monodomain_problem()
    mesh2 = pd.SpaceMesh(64, mono.X)
    hier2 = PF.build_pfasst_hierarchy(3, mesh2, pd.TimeGrid(8, 0.5), mono.gamma, L=2, nu=1,
                                      mode="imex", qdelta="lu-trick")
    x2, r2 = PF.pfasst_run(hier2, mono.u0(mesh2.vertices), 8, 2, tol_rel=1e-9, tol_abs=1e-9)
    assert r2.converged == bool(g["mono_conv"])
    assert r2.inner_iterations == g["mono_its"].tolist()
    assert per_node_rel(x2, g["mono_U"], (8, 3, 65)) < 1e-9
