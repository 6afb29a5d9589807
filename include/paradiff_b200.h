/*
 * paradiff-b200 C ABI — the drop-in boundary of the B200 hot path.
 *
 * The reference (`paradiff`, /root/reference/pkg/src/paradiff) has no FFI: its
 * seam is Python duck typing.  Each entry point below replaces
 * one reference interface (cited file:line); the Python package
 * `paper_2006_12883_b200` binds them with ctypes and keeps the reference's
 * names, arguments, (Nt, M, S) C-order fp64 layout, SolveReport fields and
 * exceptions.  Plain pointers and sizes only: device pointers are raw CUDA
 * global-memory addresses (e.g. torch.Tensor.data_ptr()), host pointers are
 * marked `host`.  All calls are asynchronous on the context's stream unless
 * documented as synchronising.
 *
 * Status codes: PD_OK, PD_ERR_CONFIG (-> ConfigurationError), PD_ERR_SOLVER
 * (-> SolverError; pd_last_error_index() carries the row/node), PD_ERR_CUDA.
 * pd_last_error() returns the calling thread's last message.
 */
#ifndef PARADIFF_B200_H
#define PARADIFF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PD_OK = 0, PD_ERR_CONFIG = 1, PD_ERR_SOLVER = 2, PD_ERR_CUDA = 3 };

typedef struct pd_solve_report {
    int32_t iterations; /* V-cycles / GMRES iterations / PFASST max window iterations */
    int32_t converged;
    int32_t diverged;
    int32_t hist_len;   /* entries written to the caller's history buffer */
} pd_solve_report;

const char *pd_last_error(void);
int64_t pd_last_error_index(void);
int pd_version(void);
uint64_t pd_launch_count(void); /* kernels launched by this library since load */

/* ---- context (one per GPU / rank; single-threaded) -------------------- */
int pd_ctx_create(int device, void *stream, void **ctx_out);
int pd_ctx_set_stream(void *ctx, void *stream);
int pd_ctx_destroy(void *ctx);

/* ---- CSR matrices (replaces scipy CSR `A @ x`, linalg.py:47-60 as_csr/kron
 *      products, multigrid.py:245,262,286,296; spacetime.py:117-124) -------- */
int pd_csr_create(void *ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                  const int64_t *rowptr, const int32_t *col, const double *val,
                  int device_src, void **csr_out);
int pd_csr_set_values(void *ctx, void *csr, const double *val, int device_src);
/* mode 0: y = A x; 1: y = b - A x; 2: y = b + A x (y may alias b) */
int pd_csr_spmv(void *ctx, void *csr, const double *x, double *y, int mode, const double *b);
int pd_csr_destroy(void *csr);

/* ---- ILU(0) / block-Jacobi ILU(0) (linalg.py:63-189: _ilu0_factor,
 *      _ilu0_solve, Ilu0, BlockJacobiPrecond with contiguous n//P ranges) ---- */
int pd_ilu0_create(void *ctx, void *csr, int nblocks, void **ilu_out); /* synchronising */
int pd_ilu0_refactor(void *ctx, void *ilu);                            /* synchronising */
int pd_ilu0_solve(void *ctx, void *ilu, const double *b, double *x);
int pd_ilu0_levels(void *ilu, int32_t *lower_levels, int32_t *upper_levels); /* host out */
/* Structured wavefront sweeps for rows laid out [task][ngroup][nline][npoint]
 * (2D FD space-time: one time step = M node grids of nline x npoint points):
 * one CTA per task, one thread per (grid, line), in-task dependencies through
 * shared memory, per-step factor values staged by TMA bulk copies.  Same
 * arithmetic as pd_ilu0_solve (bitwise); *applied = 0 when the schedule does
 * not fit (the level-scheduled sweeps stay in use).  ngroup_lower > 0 lets a
 * lower-sweep task span ngroup_lower grids (several time steps: their time
 * coupling then stays inside the CTA); 0 = ngroup.  A faster schedule for
 * linalg.py:104-113; the reference has no counterpart. */
int pd_ilu0_set_wavefront(void *ctx, void *ilu, int64_t ngroup, int64_t nline, int64_t npoint,
                          int64_t ngroup_lower, int *applied);                    /* synchronising */
/* Copy the factor values (L strictly below, U on and above the diagonal, on the
 * factor's CSR pattern; host or device `out`, `cap` >= nnz) — linalg.py:138-145
 * Ilu0.factors(). */
int pd_ilu0_factor_values(void *ctx, void *ilu, double *out, int64_t cap); /* synchronising */
/* Which executor runs this factor's sweeps: 2 = template-structured skewed
 * wavefront for both sweeps (pd_wf2.cu), 3 = pattern-table lower sweep + template
 * upper sweep, 1 = pattern-table wavefront (pd_wavefront.cu), 0 = level-scheduled
 * value-as-flag sweeps. */
int pd_ilu0_sweep_kind(void *ilu, int *kind);
int pd_ilu0_destroy(void *ilu);
/* Structured SpMV for a 2D-grid space-time operator (SMG Galerkin levels: every
 * row couples to the previous step's last node and to each node of its own
 * step through a 3x3 neighbourhood; nt steps, M nodes, n x n points).  When the
 * CSR has exactly that pattern its values are copied as [position][row] and
 * pd_csr_spmv uses them (bitwise the CSR product: same per-row order); value
 * updates of the CSR refresh the copy.  *applied = 0: pattern differs. */
int pd_csr_set_grid(void *ctx, void *csr, int64_t nt, int M, int64_t n, int *applied);

/* ---- dense LU of the coarsest level (linalg.py:196-209 DenseLU) ---------- */
int pd_dense_lu_create(void *ctx, void *csr, void **lu_out); /* synchronising */
int pd_dense_lu_solve(void *ctx, void *lu, const double *b, double *x);
int pd_dense_lu_destroy(void *lu);

/* ---- mode product of the exact structured-grid node solve (pfasst.py:118-132's linear
 *      system solved by its 1D eigen-decomposition): out[o,a,r] = sum_i Mat[a,i]
 *      in[o,i,r] over the C-order array [total/(n*stride)][n][stride], Mat = Phi^T
 *      (transpose=1) or Phi, phi = n x n row-major on the device.  in != out. */
int pd_mode_product(void *ctx, const double *in, double *out, int64_t total, int64_t n,
                    int64_t stride, const double *phi, int transpose);

/* ---- banded LU with partial pivoting: the direct solves of spacetime.py:154-195
 *      (_element_solve, solve_sequential, solve_direct call SuperLU there).  csr is
 *      the matrix with its unknowns already reordered so that it is banded (kl sub-,
 *      ku super-diagonals); perm_host (n int32, may be NULL) maps band row i to the
 *      caller's unknown perm[i] for b and x of pd_band_lu_solve.  A singular matrix
 *      is PD_ERR_SOLVER (SuperLU: "Factor is exactly singular").  Synchronising. */
int pd_band_lu_create(void *ctx, void *csr, int kl, int ku, const int32_t *perm_host,
                      void **lu_out);
int pd_band_lu_solve(void *ctx, void *lu, const double *b, double *x);
int pd_band_lu_destroy(void *lu);

/* ---- GMRES (linalg.py:215-311 gmres); ilu may be NULL (no preconditioner),
 *      x0 may be NULL (zero start).  hist (host, hist_cap doubles) receives
 *      SolveReport.residual_history.  Synchronising. ------------------------ */
int pd_gmres(void *ctx, void *A, void *ilu, const double *b, const double *x0, double *x,
             double tol_rel, double tol_abs, int restart, int max_it,
             pd_solve_report *rep, double *hist, int hist_cap);

/* The same solve when the operator and/or the preconditioner is a host callable
 * (linalg.py:233-237: "A is a matrix or a callable matvec; precond needs a solve
 * method (or is callable)").  Exactly one of A (CSR handle) / matvec, at most one of
 * ilu / psolve.  A callable reads its argument from cb_in and writes its result to
 * cb_out (device vectors of n doubles owned by the caller; the stream is idle while it
 * runs) and returns 0, or nonzero to abort the solve.  The Krylov vectors, the
 * orthogonalisation and the Givens recurrence stay on the device.  Synchronising. */
typedef int (*pd_apply_cb)(void *user);
int pd_gmres_callable(void *ctx, int64_t n, void *A, pd_apply_cb matvec, void *ilu,
                      pd_apply_cb psolve, void *user, double *cb_in, double *cb_out,
                      const double *b, const double *x0, double *x, double tol_rel,
                      double tol_abs, int restart, int max_it, pd_solve_report *rep,
                      double *hist, int hist_cap);

/* ---- the smoother's GMRES(nu) (multigrid.py:243-256 on linalg.py:215-311) driven step by
 *      step from outside, for the time-slab sharded V-cycle: the caller
 *      applies the rank-local block-Jacobi preconditioner to V[j] -> Z[j] and the sharded
 *      operator (halo exchange inside) to Z[j] -> w, sum-reduces dots[i] over the ranks
 *      after every MGS pass (a device scalar: NCCL all-reduce on the stream), and the
 *      Hessenberg / Givens recurrence, the stopping test and the update x += Z y run on the
 *      device.  No call synchronises except pd_gms_error.
 *      per step j = 0..nu-1: begin(j) | M^{-1}, A | for i in 0..j+1: mgs_pass(i), reduce
 *      dots[i] | end(j);   after the last step: apply(x). */
int pd_gms_create(void *ctx, int64_t n_local, int nu, void **out);
int pd_gms_destroy(void *e);
int pd_gms_init(void *e, const double *r0, const double *norm2_dev); /* |r0|^2 over all ranks */
int pd_gms_begin(void *e, int j, const double **vin, double **zout, double **wout);
int pd_gms_dots(void *e, double **dots_dev);
int pd_gms_mgs_pass(void *e, int i);
int pd_gms_end(void *e, int slot);
int pd_gms_apply(void *e, double *x);
int pd_gms_error(void *e, int *err); /* synchronising; 0 or linalg.py's non-finite cases 1..3 */
int pd_dot_dev(void *ctx, const double *x, const double *y, int64_t n, double *out_dev);

/* ---- space-time multigrid (multigrid.py:197-305 MultigridHierarchy).
 *      Takes ownership of the level matrices mats[0..L) (Galerkin products,
 *      multigrid.py:232-233) and of R[0..L-1), P[0..L-1), also when it fails
 *      (they are freed then).  --------------------------------------------- */
int pd_mg_create(void *ctx, int nlevels, void **mats, void **R, void **P, int nu,
                 int partitions, int restart, int smooth_solves, void **mg_out);
int pd_mg_level_matrix(void *mg, int level, void **csr_out); /* borrowed handle */
int pd_mg_level_precond(void *mg, int level, void **ilu_out); /* borrowed ILU/block-Jacobi */
int pd_mg_refactor(void *ctx, void *mg);                     /* after value updates */
int pd_mg_set_fine_operator(void *mg, void *stop); /* takes ownership; NULL detaches */
/* device Newton refresh (multigrid.py:224-241, §8(f)1): T[l] = R_l A_l patterns in
 * scipy's stored (unsorted) order, ownership moves to the hierarchy; then
 * set_fine_values recomputes every Galerkin level on device (bitwise scipy's
 * csr_matmat order) and refactors ILU(0)s and the coarsest LU. */
int pd_mg_set_galerkin_intermediates(void *mg, int n, void **T);
int pd_mg_set_fine_values(void *mg, const double *vals_dev);
/* J = L + gamma (I (x) Mqh) diag(r'(u)) values on L's pattern (spacetime.py:144-151);
 * Mq_dev: M x M, mh_dev: S (device); kind 1 cubic, 2 Fisher */
int pd_jacobian_values(void *ctx, int64_t Nt, int M, int64_t S, double dt, double gamma, int kind,
                       const double *Mq_dev, const double *mh_dev, void *L, const double *u,
                       double *jv);
int pd_mg_vcycle(void *ctx, void *mg, const double *b, double *x); /* multigrid.py:268-273 */
int pd_mg_solve(void *ctx, void *mg, const double *b, double *x, double tol_rel,
                double tol_abs, int max_cycles, pd_solve_report *rep, double *hist,
                int hist_cap); /* multigrid.py:275-305; synchronising */
int pd_mg_destroy(void *mg);

/* ---- space-time residual on CSR operators (spacetime.py:44-50,131-151):
 *      out = L u - rhs + gamma * MR r(u), MR = I (x) Mqh (may be NULL when
 *      gamma == 0); kind 0 none, 1 cubic u^3-u, 2 Fisher u^2-u; tmp: 2n doubles */
int pd_st_residual_csr(void *ctx, void *L, void *MR, double gamma, int kind, const double *u,
                       const double *rhs, double *out, double *tmp);
int pd_reaction(void *ctx, int kind, int deriv, const double *u, double *out, int64_t n);
int pd_axpy_to(void *ctx, double *y, const double *x, const double *d, double s, int64_t n);
int pd_norm(void *ctx, const double *x, int64_t n, double *host_out); /* synchronising */
int pd_dot(void *ctx, const double *x, const double *y, int64_t n, double *host_out); /* x.y, synchronising */
int pd_scale(void *ctx, double *y, const double *x, double s, int64_t n);

/* ---- K1: matrix-free space-time operator (spacetime.py:77-80,117-142).
 *      L = I (x) (Kq (x) Mh + dt Mq (x) Kh) + S_{-1} (x) (-Jq (x) Mh), with
 *      Jq = l0 l1^T (right Radau: only the last column).  `apply` is bitwise
 *      the assembled CSR SpMV; mode 0 y=Lx, 1 y=b-Lx, 2 y=b+Lx; halo = the
 *      previous step's last-node values for a time slab (NULL: none).
 *      `residual` = F(u) in the reference's blockwise order; kind 0 none,
 *      1 cubic, 2 Fisher. */
int pd_stop_create(void *ctx, int64_t Nt, int M, int64_t S, const double *Kq, const double *Mq,
                   const double *l0, double dt, void *Kh_csr, const double *mh_host,
                   void **op_out);
int pd_stop_destroy(void *op);
int pd_stop_apply(void *op, const double *x, double *y, int mode, const double *b,
                  const double *halo);
int pd_stop_residual(void *op, const double *u, const double *rhs, double *out, double gamma,
                     int kind);

/* ---- SDC / PFASST building blocks, batched over W workers of a window
 *      (pfasst.py:60-303).  State layout: U[W][M][S], U0[W][S], tau[W][M][S]. */
/* spec_* (optional, NULL to skip): Kh = spec_s * sum over spec_dim axes of T,
 * T = Phi diag(spec_mu) Phi^T (spec_n x spec_n, Phi row-major, orthonormal);
 * enables the exact spectral node solver for structured FD operators. */
int pd_sdc_level_create(void *ctx, void *Kh, const double *mh_host, int M, const double *Q,
                        const double *QDI, const double *QDE, double dt, double gamma,
                        int reaction, int imex, int max_workers, const double *spec_phi,
                        const double *spec_mu, int spec_dim, int64_t spec_n, double spec_s,
                        void **lvl_out); /* SdcLevel */
int pd_sdc_level_destroy(void *lvl);
int pd_sdc_sweep(void *lvl, double *U, const double *U0, const double *tau, int W); /* :155-200 */
int pd_sdc_chain(void *lvl, double *U, double *U0, const double *tau, int W, const double *u0c,
                 int nu); /* coarsest serial chain, pfasst.py:441-455 */
int pd_sdc_residual(void *lvl, const double *U, const double *U0, const double *tau, int W,
                    double *res_dev);                            /* :107-115, per worker */
int pd_sdc_coll_op(void *lvl, const double *U, double *out, int W); /* C(u) = u - dt Q F(u) */
int pd_sdc_errors(void *lvl, int *host_out); /* synchronising; host_out[0] = failure
 * kinds (0 none), host_out[1] = lowest failing worker of the batch (-1 none); clears */
int pd_node_mix(void *ctx, const double *in, double *out, int W, int Min, int Mout, int64_t S,
                const double *N_host, int accumulate);           /* node transfer :262-266 */
int pd_csr_spmm(void *ctx, void *A, const double *x, int64_t xs, double *y, int64_t ys,
                int nvec, int mode);                             /* space transfer, batched */
int pd_sub(void *ctx, double *out, const double *a, const double *b, int64_t n);
int pd_spread(void *ctx, const double *u0, double *U, double *U0, int W, int M, int64_t S);
int pd_terminal(void *ctx, const double *U, double *out, int W, int M, int64_t S);

/* ---- P-fast: matrix-free block-Jacobi-in-time smoother with inner spatial
 *      V-cycles on structured grids (SURVEY §7.1 P-fast profile; no reference
 *      counterpart — the outer loop follows multigrid.py:243-305, the time
 *      blocks linalg.py:152-189 with one block per step, the operator
 *      spacetime.py:77-80,117-124 with Kh = kappa h^{d-2}(-Lap stencil),
 *      Mh = h^d I).  Parity: oracle/pfast_oracle.py.  Vectors (nt, M, n^d). -- */
int pd_pfast_create(void *ctx, int dim, int64_t n, int bc_periodic, double kappa, int M,
                    int64_t nt, double dt, const double *Kq, const double *Mq, const double *l0,
                    int levels, int nu, int coarse_sweeps, double omega_s, double omega_t,
                    void **plan_out); /* Kq, Mq (M x M row-major), l0 (M): host */
/* halo (device, n^d doubles, or NULL): time-slab sharding — the plan's steps are one
 * rank's slab and `halo` is the previous slab's x[last step, M-1], coupled to the first
 * step by the residual.  Passed per call; the library keeps no pointer to it. */
int pd_pfast_residual(void *plan, const double *x, const double *b, double *r, const double *halo,
                      double *norm2_dev);
int pd_pfast_sweep(void *plan, const double *b, double *x, const double *halo);
int pd_pfast_solve(void *plan, const double *b, double *x, const double *halo, double tol_rel,
                   double tol_abs, int max_sweeps, pd_solve_report *report,
                   double *hist /* host, optional */);
/* Newton pieces (spacetime.py:126-151): out = rhs - L u - gamma (I (x) Mqh) r(u) = -F(u)
 * (kind 0: cubic u^3-u, spacetime.py:44-50; 1: Fisher u^2-u), and the linearisation
 * state W = gamma dt h^d r'(u) that turns L into J = L + gamma (I (x) Mqh) diag(r'(u))
 * in every later residual/sweep/solve (NULL u: back to L).  set_state synchronises. */
int pd_pfast_nl_residual(void *plan, const double *u, const double *rhs, double *out,
                         const double *halo, double gamma, int kind, double *norm2_dev);
int pd_pfast_set_state(void *plan, const double *u, double gamma, int kind);
int pd_pfast_destroy(void *plan);

/* ---- P-fast STMG: the space-time V(nu_t, nu_t) cycle around that smoother (north_star
 *      subsystem 2: "space-time coarsening and interpolation").  Level l: nt[l] =
 *      nt[0]/2^l steps of dt[l] = 2^l dt[0] on an n[l]^d grid (n[l+1] = n[l] or its 2:1
 *      coarsening; schedule = multigrid.py:148-157's STMG rule with space coarsened
 *      only while kappa dt/h^2 allows it, built by pfast.st_schedule); rediscretised
 *      operators; time transfers P1/P2 (M x M, host): the coarse element's collocation
 *      polynomial at the first/second fine element's nodes, restriction = transpose;
 *      E/half: fine cardinal values at the coarse nodes (weights).  The coarsest level
 *      runs coarse_t_sweeps undamped sweeps.  Parity: oracle/pfast_oracle.py. -- */
int pd_pfast_st_create(void *ctx, int dim, int bc_periodic, double kappa, int M, const double *Kq,
                       const double *Mq, const double *l0, int nlevels, const int64_t *nt,
                       const int64_t *n, const double *dt, const int *space_levels,
                       const double *P1, const double *P2, const double *E, const int *half,
                       int nu_t, int coarse_t_sweeps, int nu, int coarse_sweeps, double omega_s,
                       double omega_t, void **st_out);
int pd_pfast_st_destroy(void *st);
int pd_pfast_st_set_state(void *st, const double *u, double gamma, int kind); /* synchronising */
int pd_pfast_st_cycle(void *st, const double *b, double *x);
int pd_pfast_st_solve(void *st, const double *b, double *x, double tol_rel, double tol_abs,
                      int max_cycles, pd_solve_report *report, double *hist /* host, optional */);
/* level primitives for the time-slab sharded cycle (pfast.StmgSlab drives them; b / x
 * NULL select the level's own vectors on levels >= 1; halo as above, per level) */
int pd_pfast_st_level_plan(void *st, int level, void **plan_out); /* borrowed smoother */
int pd_pfast_st_level_sweep(void *st, int level, const double *b, double *x, const double *halo);
int pd_pfast_st_level_restrict(void *st, int level, const double *b, const double *x,
                               const double *halo);
int pd_pfast_st_level_prolong(void *st, int level, double *x);
int pd_pfast_st_level_last(void *st, int level, const double *x, double *out);

#ifdef __cplusplus
}
#endif

#endif /* PARADIFF_B200_H */
