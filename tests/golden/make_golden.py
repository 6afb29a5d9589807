"""Generate golden fixtures by running the REAL reference (build container only).

    python tests/golden/make_golden.py

Imports `paradiff` from /root/reference/pkg/src (read-only; NUMBA_CACHE_DIR
and sys.dont_write_bytecode are set first so nothing is written into the
reference tree — SURVEY §8(c)).  Inputs for the BASELINE configs come from
`paper_2006_12883_b200.problems` (seeded generators), and the reference is
driven through its public constructors with injected operators exactly as in
SURVEY Appendix A.  Outputs: tests/golden/*.npz (small, committed).  The GPU
box never runs this script.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pd_numba_"))
os.environ.setdefault("PARADIFF_MAX_THREADS", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

import paradiff  # noqa: E402
from paradiff import (  # noqa: E402
    SpaceMesh, SpaceOperators, TimeGrid, assemble_space, assemble_system, build_hierarchy,
    build_pfasst_hierarchy, heat_problem, make_tableau, mg_linear_solver, monodomain_problem,
    newton_solve, pfasst_run,
)
from paradiff.linalg import Ilu0, gmres, block_jacobi, kron  # noqa: E402
from paradiff.multigrid import (  # noqa: E402
    LevelDims, MultigridHierarchy, TransferSet, node_prolongation, node_restriction,
    spatial_prolongation, spatial_restriction, time_prolongation, time_restriction,
)
from paradiff.pfasst import (  # noqa: E402
    LevelTransfer, PfasstHierarchy, SdcLevel, SweeperState, _node_eval_restriction,
    fas_correction, sdc_solve_step, spread_state,
)

from paper_2006_12883_b200 import problems as PB  # noqa: E402

assert str(Path(paradiff.__file__).resolve()).startswith(REF), paradiff.__file__


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print("wrote", name, sorted(arrays))


def injected(spec):
    ops = PB.fd_space(spec)
    return SpaceOperators(mesh=ops.mesh, Kh=ops.Kh, Mh=ops.Mh, MhConsistent=ops.MhConsistent)


def fd_mg(system, spec, strategy, L, nu, P, Nt, M):
    """MultigridHierarchy with FD interior transfers via the public ctor (Appendix A)."""
    specs = [spec]
    for _ in range(L - 1):
        specs.append(specs[-1].coarse())
    dims = []
    for l, s in enumerate(specs):
        nt = Nt // 2 ** l if strategy == "STMG" else Nt
        m = max(M - l, 1) if strategy == "SMMG" else M
        dims.append(LevelDims(nt, m, s.ndof))
    trs = []
    for l in range(L - 1):
        f, c = dims[l], dims[l + 1]
        Rs, Ps = PB.fd_transfers(specs[l])
        if f.nt != c.nt:
            Rt, Pt = time_restriction(f.nt), time_prolongation(f.nt)
        else:
            Rt = Pt = sp.eye(f.nt, format="csr")
        if f.m != c.m:
            Rm, Pm = node_restriction(c.m, f.m), node_prolongation(c.m, f.m)
        else:
            Rm = Pm = sp.eye(f.m, format="csr")
        trs.append(TransferSet(kron(Rt, kron(Rm, Rs)), kron(Pt, kron(Pm, Ps))))
    return MultigridHierarchy(system.global_matrix(), strategy, dims, trs, nu=nu, partitions=P)


def fd_pfasst(spec, M, Mc, dt, gamma, mode, nu):
    spec_c = spec.coarse()
    tf, tc = make_tableau(M), make_tableau(Mc)
    levels = [SdcLevel(tf, injected(spec), dt, gamma, mode),
              SdcLevel(tc, injected(spec_c), dt, gamma, mode)]
    Rs, Ps = PB.fd_transfers(spec)
    tr = LevelTransfer(Rs, Ps, _node_eval_restriction(tf.nodes, tc.nodes),
                       _node_eval_restriction(tc.nodes, tf.nodes))
    return PfasstHierarchy(levels, [tr], nu)


def main():
    # 1. tableau, FEM, transfers -------------------------------------------------
    arrs = {}
    for M in range(1, 6):
        t = make_tableau(M)
        for k in ("nodes", "Q", "QDeltaImplicit", "QDeltaExplicit", "Kq", "Mq", "Jq"):
            arrs[f"M{M}_{k}"] = getattr(t, k)
        arrs[f"M{M}_lutrick"] = make_tableau(M, "lu-trick").QDeltaImplicit
    sp8 = assemble_space(SpaceMesh(8, 1.0))
    arrs["fem8_Kh"] = sp8.Kh.toarray()
    arrs["fem8_mh"] = sp8.lumped_diagonal
    arrs["R9"] = spatial_restriction(9).toarray()
    arrs["P9"] = spatial_prolongation(9).toarray()
    arrs["Rt8"] = time_restriction(8).toarray()
    arrs["Pt8"] = time_prolongation(8).toarray()
    arrs["Rn23"] = node_restriction(2, 3).toarray()
    arrs["Pn23"] = node_prolongation(2, 3).toarray()
    arrs["Ne35"] = _node_eval_restriction(make_tableau(5).nodes, make_tableau(3).nodes)
    save("tableau", **arrs)

    # 2. ILU(0), block-Jacobi, GMRES on a seeded sparse matrix ---------------------
    rng = np.random.default_rng(7)
    n = 300
    A = sp.random(n, n, density=0.03, random_state=11, format="csr")
    A = (A + A.T + sp.diags(np.full(n, 12.0)) + sp.diags(np.full(n - 1, -1.0), 1)).tocsr()
    A.sum_duplicates(); A.sort_indices()
    ilu = Ilu0(A)
    b = rng.standard_normal(n)
    bj = block_jacobi(A, 3, parallel=False)
    x, rep = gmres(A, b, precond=ilu, tol_rel=1e-10, tol_abs=1e-12, restart=7, max_it=200)
    x2, rep2 = gmres(A, b, precond=bj, tol_rel=1e-10, tol_abs=1e-12, restart=5, max_it=200)
    save("linalg", A_data=A.data, A_indices=A.indices, A_indptr=A.indptr, b=b,
         ilu_data=ilu._data, ilu_diag=ilu._diag_pos, ilu_solve=ilu.solve(b),
         bj_solve=bj.solve(b), gm_x=x, gm_hist=np.array(rep.residual_history),
         gm_its=rep.iterations, gm2_x=x2, gm2_hist=np.array(rep2.residual_history),
         gm2_its=rep2.iterations)

    # 3. space-time system, residual, Jacobian ------------------------------------
    prob = monodomain_problem()
    mesh = SpaceMesh(16, prob.X)
    sysm = assemble_system(make_tableau(3), assemble_space(mesh), TimeGrid(4, prob.T),
                           prob.gamma, prob.u0(mesh.vertices))
    u = rng.standard_normal(sysm.size) * 0.5
    v = rng.standard_normal(sysm.size)
    save("spacetime", u=u, v=v, rhs=sysm.rhs(), res=sysm.residual(u),
         Lv=sysm.global_matrix() @ v, Jv=sysm.jacobian(u) @ v,
         seq=assemble_system(make_tableau(3), assemble_space(mesh), TimeGrid(4, 1.0), 0.0,
                             prob.u0(mesh.vertices)).solve_sequential())

    # 4. MG on the reference's own 1D FEM heat problem ---------------------------------
    heat = heat_problem()
    out = {}
    for strat in ("SMG", "STMG", "SMMG"):
        for P in (1, 4):
            mesh = SpaceMesh(64, 1.0)
            sysh = assemble_system(make_tableau(3), assemble_space(mesh), TimeGrid(16, 1.0),
                                   0.0, heat.u0(mesh.vertices))
            h = build_hierarchy(sysh, strat, 3, 3, partitions=P)
            x, rep = h.solve(sysh.rhs(), tol_rel=1e-10, tol_abs=1e-10)
            key = f"{strat}_P{P}"
            out[key + "_x"] = x
            out[key + "_its"] = rep.iterations
            out[key + "_hist"] = np.array(rep.residual_history)
            out[key + "_v1"] = h.vcycle(sysh.rhs(), np.zeros(sysh.size))
    save("mg_fem1d", **out)

    # 5. BASELINE C1 full size via injected operators (SMG/STMG + PFASST) ------------
    cfg = PB.baseline_config("C1")
    u0 = cfg.u0()
    ops = injected(cfg.spec)
    sysc = assemble_system(make_tableau(cfg.M), ops, TimeGrid(cfg.Nt, cfg.T), 0.0, u0)
    out = {"u0": u0, "seq": sysc.solve_sequential()}
    for strat in ("SMG", "STMG"):
        for P in (1, 2, 4, 8):
            h = fd_mg(sysc, cfg.spec, strat, 4, 3, P, cfg.Nt, cfg.M)
            x, rep = h.solve(sysc.rhs(), tol_rel=1e-10, tol_abs=1e-10)
            out[f"{strat}_P{P}_x"] = x
            out[f"{strat}_P{P}_its"] = rep.iterations
            out[f"{strat}_P{P}_hist"] = np.array(rep.residual_history)
    for P in (1, 2, 4, 8):
        hier = fd_pfasst(cfg.spec, cfg.M, cfg.M_coarse, cfg.dt, 0.0, "implicit", 1)
        x, rep = pfasst_run(hier, u0, cfg.Nt, P, tol_rel=1e-10, tol_abs=1e-10)
        out[f"PF_P{P}_x"] = x
        out[f"PF_P{P}_its"] = rep.iterations
        out[f"PF_P{P}_inner"] = np.array(rep.inner_iterations)
        out[f"PF_P{P}_hist"] = np.array(rep.residual_history)
    save("c1", **out)

    # 6. PFASST / SDC on the reference 1D FEM problems ------------------------------
    out = {}
    mesh = SpaceMesh(32, 1.0)
    u0h = heat.u0(mesh.vertices)
    for P in (1, 2, 4):
        hier = build_pfasst_hierarchy(3, mesh, TimeGrid(8, 1.0), 0.0, L=2, nu=1)
        x, rep = pfasst_run(hier, u0h, 8, P, tol_rel=1e-10, tol_abs=1e-10)
        out[f"heat_P{P}_x"], out[f"heat_P{P}_its"] = x, rep.iterations
        out[f"heat_P{P}_inner"] = np.array(rep.inner_iterations)
    hier3 = build_pfasst_hierarchy(2, SpaceMesh(32, 1.0), TimeGrid(8, 1.0), 0.0, L=3, nu=1)
    x, rep = pfasst_run(hier3, u0h, 8, 4, tol_rel=1e-10, tol_abs=1e-10)
    out["heatL3_P4_x"], out["heatL3_P4_its"] = x, rep.iterations
    out["heatL3_P4_inner"] = np.array(rep.inner_iterations)
    mono = monodomain_problem()
    meshm = SpaceMesh(64, mono.X)
    u0m = mono.u0(meshm.vertices)
    for mode in ("imex", "implicit"):
        hier = build_pfasst_hierarchy(2, meshm, TimeGrid(16, mono.T), mono.gamma, L=2, nu=1,
                                      mode=mode)
        x, rep = pfasst_run(hier, u0m, 16, 4, tol_rel=1e-9, tol_abs=1e-9)
        out[f"mono_{mode}_x"], out[f"mono_{mode}_its"] = x, rep.iterations
        out[f"mono_{mode}_inner"] = np.array(rep.inner_iterations)
    # single sweeps and FAS on a random state
    hier = build_pfasst_hierarchy(3, mesh, TimeGrid(8, 1.0), 0.0, L=2, nu=1)
    st = spread_state(u0h, 3)
    st.U = st.U + 0.1 * rng.standard_normal(st.U.shape)
    out["sweep_U_in"] = st.U.copy()
    out["sweep_U_out"] = hier.fine.sweep(st).U
    out["fas_tau"] = fas_correction(hier.levels[0], hier.levels[1], hier.transfers[0], st)
    out["resnorm"] = hier.fine.residual_norm(st)
    lv = SdcLevel(make_tableau(3), assemble_space(meshm), 0.05, mono.gamma, "imex")
    stm = spread_state(u0m, 3)
    out["imex_sweep"] = lv.sweep(stm).U
    s, rp = sdc_solve_step(u0m, lv, tol_rel=1e-10, tol_abs=1e-10)
    out["sdc_step_U"], out["sdc_step_its"] = s.U, rp.iterations
    save("pfasst_fem1d", **out)

    # 7. Newton + MG on monodomain ----------------------------------------------------
    mesh = SpaceMesh(32, mono.X)
    sysn = assemble_system(make_tableau(2), assemble_space(mesh), TimeGrid(8, mono.T),
                           mono.gamma, mono.u0(mesh.vertices))
    h = build_hierarchy(sysn, "SMG", 3, 3)
    x, rep = newton_solve(sysn, mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9), tol=1e-9)
    save("newton", x=x, its=rep.iterations, inner=np.array(rep.inner_iterations),
         damped=rep.damped_steps, hist=np.array(rep.residual_history))

    # 8. 2D Dirichlet, reduced C2-like (15^2 x 8 steps, M=3) ---------------------------
    spec = PB.StencilSpec(2, 15, "dirichlet", 1.0)
    cfg2 = PB.BaselineConfig("C2", spec, 8, 8 / 64, 3, 2, 0.0, "cubic", 0, "reduced")
    u02 = cfg2.u0()
    sys2 = assemble_system(make_tableau(3), injected(spec), TimeGrid(8, cfg2.T), 0.0, u02)
    out = {"u0": u02}
    for strat, L in (("SMG", 3), ("STMG", 3)):
        for P in (1, 4):
            h = fd_mg(sys2, spec, strat, L, 3, P, 8, 3)
            x, rep = h.solve(sys2.rhs(), tol_rel=1e-10, tol_abs=1e-10)
            out[f"{strat}_P{P}_x"], out[f"{strat}_P{P}_its"] = x, rep.iterations
            out[f"{strat}_P{P}_hist"] = np.array(rep.residual_history)
    hier = fd_pfasst(spec, 3, 2, cfg2.dt, 0.0, "implicit", 1)
    x, rep = pfasst_run(hier, u02, 8, 4, tol_rel=1e-9, tol_abs=1e-9)
    out["PF_P4_x"], out["PF_P4_its"] = x, rep.iterations
    out["PF_P4_inner"] = np.array(rep.inner_iterations)
    save("c2_small", **out)


if __name__ == "__main__" and "--configs" not in sys.argv:
    main()


def fisher_patch():
    """Monkeypatch the four reaction globals to Fisher-KPP."""
    import paradiff.pfasst as ppf
    import paradiff.spacetime as pst

    saved = (pst.reaction, pst.reaction_deriv, ppf.reaction, ppf.reaction_deriv)
    fr = lambda u: u**2 - u  # noqa: E731
    fd = lambda u: 2.0 * u - 1.0  # noqa: E731
    pst.reaction, pst.reaction_deriv, ppf.reaction, ppf.reaction_deriv = fr, fd, fr, fd

    def restore():
        pst.reaction, pst.reaction_deriv, ppf.reaction, ppf.reaction_deriv = saved

    return restore


def configs_reduced():
    out = {}
    # C3: 2D periodic Fisher-KPP, gamma = 1, dt = 0.01, M = 3 (reduced 16^2 x 8 steps)
    cfg3 = PB.baseline_config("C3", n=16, Nt=8)
    u03 = cfg3.u0()
    out["c3_u0"] = u03
    restore = fisher_patch()
    try:
        sys3 = assemble_system(make_tableau(3), injected(cfg3.spec), TimeGrid(cfg3.Nt, cfg3.T),
                               cfg3.gamma, u03)
        h = fd_mg(sys3, cfg3.spec, "STMG", 2, 3, 1, cfg3.Nt, 3)
        x, rep = newton_solve(sys3, mg_linear_solver(h, tol_rel=1e-9, tol_abs=1e-9), tol=1e-9)
        out["c3_newton_x"], out["c3_newton_its"] = x, rep.iterations
        out["c3_newton_inner"] = np.array(rep.inner_iterations)
        hier = fd_pfasst(cfg3.spec, 3, 2, cfg3.dt, cfg3.gamma, "imex", 1)
        x, rep = pfasst_run(hier, u03, cfg3.Nt, 4, tol_rel=1e-9, tol_abs=1e-9)
        out["c3_pf_x"], out["c3_pf_its"] = x, rep.iterations
        out["c3_pf_inner"] = np.array(rep.inner_iterations)
    finally:
        restore()
    # C4: 3D Dirichlet heat, M = 5 (coarse 3), dt = 1/256 (reduced 7^3 x 8 steps)
    cfg4 = PB.baseline_config("C4", n=7, Nt=8)
    u04 = cfg4.u0()
    out["c4_u0"] = u04
    hier = fd_pfasst(cfg4.spec, 5, 3, cfg4.dt, 0.0, "implicit", 1)
    x, rep = pfasst_run(hier, u04, cfg4.Nt, 4, tol_rel=1e-9, tol_abs=1e-9)
    out["c4_pf_x"], out["c4_pf_its"] = x, rep.iterations
    out["c4_pf_inner"] = np.array(rep.inner_iterations)
    sys4 = assemble_system(make_tableau(5), injected(cfg4.spec), TimeGrid(cfg4.Nt, cfg4.T), 0.0, u04)
    h = fd_mg(sys4, cfg4.spec, "SMG", 2, 3, 2, cfg4.Nt, 5)
    x, rep = h.solve(sys4.rhs(), tol_rel=1e-10, tol_abs=1e-10)
    out["c4_smg_x"], out["c4_smg_its"] = x, rep.iterations
    # C5: 3D periodic Allen-Cahn-type (cubic), coef 0.1, gamma 1, dt 1e-3 (reduced 8^3 x 4)
    cfg5 = PB.baseline_config("C5", n=8, Nt=4)
    u05 = cfg5.u0()
    out["c5_u0"] = u05
    sys5 = assemble_system(make_tableau(3), injected(cfg5.spec), TimeGrid(cfg5.Nt, cfg5.T),
                           cfg5.gamma, u05)
    h = fd_mg(sys5, cfg5.spec, "STMG", 2, 3, 1, cfg5.Nt, 3)
    x, rep = newton_solve(sys5, mg_linear_solver(h, tol_rel=1e-8, tol_abs=1e-8), tol=1e-8)
    out["c5_newton_x"], out["c5_newton_its"] = x, rep.iterations
    out["c5_newton_inner"] = np.array(rep.inner_iterations)
    save("configs_reduced", **out)


if __name__ == "__main__" and "--configs" in sys.argv:
    configs_reduced()
