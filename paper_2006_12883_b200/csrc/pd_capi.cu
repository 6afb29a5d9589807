// extern "C" boundary: status codes, thread-local error text, handle casts.
#include "../../include/paradiff_b200.h"
#include "pd_krylov.h"

#include <cstring>
#include <string>

namespace {
thread_local std::string g_err;
thread_local int64_t g_err_index = -1;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return PD_OK;
    } catch (const pd::ConfigError& e) {
        g_err = e.what();
        g_err_index = -1;
        return PD_ERR_CONFIG;
    } catch (const pd::SolverError& e) {
        g_err = e.what();
        g_err_index = e.index;
        return PD_ERR_SOLVER;
    } catch (const pd::CudaError& e) {
        g_err = e.what();
        g_err_index = -1;
        return PD_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_err_index = -1;
        return PD_ERR_CUDA;
    }
}

pd::Ctx* C(void* p) {
    if (!p) throw pd::ConfigError("null context");
    return static_cast<pd::Ctx*>(p);
}
template <class T>
T* H(void* p, const char* what) {
    if (!p) throw pd::ConfigError(std::string("null ") + what + " handle");
    return static_cast<T*>(p);
}

void fill_report(pd_solve_report* rep, int its, bool conv, bool div,
                 const std::vector<double>& hist, double* out, int cap) {
    if (rep) {
        rep->iterations = its;
        rep->converged = conv ? 1 : 0;
        rep->diverged = div ? 1 : 0;
        rep->hist_len = (int)std::min<size_t>(hist.size(), (size_t)std::max(cap, 0));
    }
    if (out && cap > 0)
        std::memcpy(out, hist.data(), std::min<size_t>(hist.size(), (size_t)cap) * sizeof(double));
}
}  // namespace

void pd_set_error_(const char* msg, int64_t index) {
    g_err = msg;
    g_err_index = index;
}

extern "C" {

const char* pd_last_error(void) { return g_err.c_str(); }
int64_t pd_last_error_index(void) { return g_err_index; }
int pd_version(void) { return 1; }
uint64_t pd_launch_count(void) { return pd::g_launches.load(); }

int pd_ctx_create(int device, void* stream, void** out) {
    return guarded([&] { *out = new pd::Ctx(device, static_cast<cudaStream_t>(stream)); });
}
int pd_ctx_set_stream(void* ctx, void* stream) {
    return guarded([&] { C(ctx)->stream = static_cast<cudaStream_t>(stream); });
}
int pd_ctx_destroy(void* ctx) {
    return guarded([&] { delete static_cast<pd::Ctx*>(ctx); });
}

int pd_csr_create(void* ctx, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rowptr,
                  const int32_t* col, const double* val, int device_src, void** out) {
    return guarded([&] {
        if (nrows < 0 || ncols < 0 || nnz < 0) throw pd::ConfigError("negative CSR size");
        if (ncols > INT32_MAX) throw pd::ConfigError("column count exceeds int32 index range");
        *out = pd::csr_upload(*C(ctx), nrows, ncols, nnz, rowptr, col, val, device_src != 0)
                   .release();
    });
}
int pd_csr_set_values(void* ctx, void* csr, const double* val, int device_src) {
    return guarded(
        [&] { pd::csr_update_values(*C(ctx), *H<pd::Csr>(csr, "csr"), val, device_src != 0); });
}
int pd_csr_spmv(void* ctx, void* csr, const double* x, double* y, int mode, const double* b) {
    return guarded([&] {
        if (mode < 0 || mode > 2) throw pd::ConfigError("bad spmv mode");
        if (mode != 0 && !b) throw pd::ConfigError("spmv mode needs b");
        pd::csr_spmv(*C(ctx), *H<pd::Csr>(csr, "csr"), x, y, mode, b);
    });
}
int pd_csr_destroy(void* csr) {
    return guarded([&] { delete static_cast<pd::Csr*>(csr); });
}

int pd_ilu0_create(void* ctx, void* csr, int nblocks, void** out) {
    return guarded(
        [&] { *out = pd::ilu0_create(*C(ctx), *H<pd::Csr>(csr, "csr"), nblocks).release(); });
}
int pd_ilu0_refactor(void* ctx, void* ilu) {
    return guarded([&] { pd::ilu0_refactor(*C(ctx), *H<pd::Ilu0>(ilu, "ilu")); });
}
int pd_ilu0_solve(void* ctx, void* ilu, const double* b, double* x) {
    return guarded([&] { pd::ilu0_solve(*C(ctx), *H<pd::Ilu0>(ilu, "ilu"), b, x); });
}
int pd_ilu0_levels(void* ilu, int32_t* lo, int32_t* up) {
    return guarded([&] {
        auto* f = H<pd::Ilu0>(ilu, "ilu");
        if (lo) *lo = f->nlevels_lo;
        if (up) *up = f->nlevels_up;
    });
}
int pd_ilu0_set_wavefront(void* ctx, void* ilu, int64_t ngroup, int64_t nline, int64_t npoint,
                          int64_t ngroup_lower, int* applied) {
    return guarded([&] {
        auto* c = H<pd::Ctx>(ctx, "ctx");
        auto* f = H<pd::Ilu0>(ilu, "ilu");
        const bool ok = pd::ilu0_set_wavefront(*c, *f, ngroup, nline, npoint, ngroup_lower);
        if (applied) *applied = ok ? 1 : 0;
    });
}
int pd_ilu0_factor_values(void* ctx, void* ilu, double* out, int64_t cap) {
    return guarded([&] {
        auto* c = H<pd::Ctx>(ctx, "ctx");
        auto* f = H<pd::Ilu0>(ilu, "ilu");
        const pd::Csr& P = f->pat();
        if (cap < P.nnz) throw pd::ConfigError("factor value buffer too small");
        PD_CUDA(cudaStreamSynchronize(c->stream));
        PD_CUDA(cudaMemcpy(out, f->fac.p, P.nnz * sizeof(double), cudaMemcpyDefault));
    });
}
int pd_ilu0_sweep_kind(void* ilu, int* kind) {
    return guarded([&] {
        auto* f = H<pd::Ilu0>(ilu, "ilu");
        *kind = f->w2_lo ? 2 : (f->w2_up && f->wf_lo) ? 3 : f->wf_lo ? 1 : 0;
    });
}
int pd_csr_set_grid(void* ctx, void* csr, int64_t nt, int M, int64_t n, int* applied) {
    return guarded([&] {
        const bool ok = pd::csr_attach_grid(*C(ctx), *H<pd::Csr>(csr, "csr"), nt, M, n);
        if (applied) *applied = ok ? 1 : 0;
    });
}
int pd_ilu0_destroy(void* ilu) {
    return guarded([&] { delete static_cast<pd::Ilu0*>(ilu); });
}

int pd_dense_lu_create(void* ctx, void* csr, void** out) {
    return guarded(
        [&] { *out = pd::dense_lu_from_csr(*C(ctx), *H<pd::Csr>(csr, "csr")).release(); });
}
int pd_dense_lu_solve(void* ctx, void* lu, const double* b, double* x) {
    return guarded([&] { pd::dense_lu_solve(*C(ctx), *H<pd::DenseLU>(lu, "lu"), b, x); });
}
int pd_dense_lu_destroy(void* lu) {
    return guarded([&] { delete static_cast<pd::DenseLU*>(lu); });
}

int pd_mode_product(void* ctx, const double* in, double* out, int64_t total, int64_t n,
                    int64_t stride, const double* phi, int transpose) {
    return guarded([&] {
        if (n < 1 || stride < 1 || total < 0) throw pd::ConfigError("bad mode product shape");
        pd::mode_product(*C(ctx), in, out, total, n, stride, phi, transpose);
    });
}

int pd_band_lu_create(void* ctx, void* csr, int kl, int ku, const int32_t* perm_host, void** out) {
    return guarded([&] {
        *out = pd::band_lu_create(*C(ctx), *H<pd::Csr>(csr, "matrix"), kl, ku, perm_host);
    });
}
int pd_band_lu_solve(void* ctx, void* lu, const double* b, double* x) {
    return guarded([&] {
        if (!lu) throw pd::ConfigError("null banded LU handle");
        pd::band_lu_solve(*C(ctx), *static_cast<pd::BandLU*>(lu), b, x);
    });
}
int pd_band_lu_destroy(void* lu) {
    return guarded([&] { pd::band_lu_destroy(static_cast<pd::BandLU*>(lu)); });
}

int pd_gmres(void* ctx, void* A, void* ilu, const double* b, const double* x0, double* x,
             double tol_rel, double tol_abs, int restart, int max_it, pd_solve_report* rep,
             double* hist, int hist_cap) {
    return guarded([&] {
        pd::Ctx& c = *C(ctx);
        pd::Csr& M = *H<pd::Csr>(A, "matrix");
        auto r = pd::gmres_run(c, M, static_cast<pd::Ilu0*>(ilu), b, x0, x, tol_rel, tol_abs,
                               restart, max_it);
        fill_report(rep, r.iterations, r.converged, r.diverged, r.hist, hist, hist_cap);
    });
}

int pd_gmres_callable(void* ctx, int64_t n, void* A, pd_apply_cb matvec, void* ilu,
                      pd_apply_cb psolve, void* user, double* cb_in, double* cb_out,
                      const double* b, const double* x0, double* x, double tol_rel, double tol_abs,
                      int restart, int max_it, pd_solve_report* rep, double* hist, int hist_cap) {
    return guarded([&] {
        pd::Ctx& c = *C(ctx);
        if ((A == nullptr) == (matvec == nullptr))
            throw pd::ConfigError("give the operator either as a matrix or as a callable");
        if (ilu && psolve) throw pd::ConfigError("give one preconditioner, not two");
        if ((matvec || psolve) && (!cb_in || !cb_out))
            throw pd::ConfigError("callables need the two exchange vectors");
        pd::Csr* M = A ? H<pd::Csr>(A, "matrix") : nullptr;
        if (M && (M->nrows != n || M->ncols != n)) throw pd::ConfigError("matrix size differs from n");
        pd::Ilu0* P = static_cast<pd::Ilu0*>(ilu);
        // a host callable reads cb_in and writes cb_out (device vectors the caller owns);
        // a nonzero return aborts the solve (the caller keeps the exception)
        auto through = [&](pd_apply_cb fn, const char* what) {
            return [&c, fn, user, cb_in, cb_out, n, what](const double* xin, double* yout) {
                pd::vec_copy(c, cb_in, xin, n);
                PD_CUDA(cudaStreamSynchronize(c.stream));
                if (fn(user) != 0) throw pd::SolverError(std::string(what) + " callable failed");
                pd::vec_copy(c, yout, cb_out, n);
            };
        };
        pd::Gmres::ApplyFn fa, fm;
        if (matvec) fa = through(matvec, "matvec");
        else fa = [&c, M](const double* xin, double* yout) {
            pd::csr_spmv(c, *M, xin, yout, pd::SPMV_SET, nullptr, nullptr, 0, nullptr, nullptr);
        };
        if (psolve) fm = through(psolve, "preconditioner");
        else if (P) fm = [&c, P](const double* xin, double* yout) {
            pd::ilu0_solve(c, *P, xin, yout, nullptr, 0);
        };
        auto r = pd::gmres_run_callables(c, n, fa, (psolve || P) ? &fm : nullptr, b, x0, x, tol_rel,
                                         tol_abs, restart, max_it);
        fill_report(rep, r.iterations, r.converged, r.diverged, r.hist, hist, hist_cap);
    });
}

// ---- externally driven GMRES(nu) smoother steps (mg_sharded.py)
int pd_gms_create(void* ctx, int64_t n, int nu, void** out) {
    return guarded([&] {
        if (n < 0 || nu < 1) throw pd::ConfigError("bad smoother size");
        *out = new pd::Gmres(*C(ctx), nullptr, nullptr, n, nu, nu, /*store_z=*/true,
                             /*external=*/true);
    });
}
int pd_gms_destroy(void* e) {
    return guarded([&] { delete static_cast<pd::Gmres*>(e); });
}
int pd_gms_init(void* e, const double* r0, const double* norm2_dev) {
    return guarded([&] {
        H<pd::Gmres>(e, "smoother")->enqueue_init(r0, norm2_dev, 1e-13, 0.0);
    });
}
int pd_gms_begin(void* e, int j, const double** vin, double** zout, double** wout) {
    return guarded([&] { H<pd::Gmres>(e, "smoother")->ext_begin(j, vin, zout, wout); });
}
int pd_gms_dots(void* e, double** dots_dev) {
    return guarded([&] { *dots_dev = H<pd::Gmres>(e, "smoother")->ext_dots(); });
}
int pd_gms_mgs_pass(void* e, int i) {
    return guarded([&] { H<pd::Gmres>(e, "smoother")->ext_mgs_pass(i); });
}
int pd_gms_end(void* e, int slot) {
    return guarded([&] { H<pd::Gmres>(e, "smoother")->ext_end(slot); });
}
int pd_gms_apply(void* e, double* x) {
    return guarded([&] { H<pd::Gmres>(e, "smoother")->ext_apply(x); });
}
int pd_gms_error(void* e, int* err) {
    return guarded([&] { *err = H<pd::Gmres>(e, "smoother")->read_state().err; });
}
int pd_dot_dev(void* ctx, const double* x, const double* y, int64_t n, double* out_dev) {
    return guarded([&] { pd::vec_dot(*C(ctx), x, y, n, out_dev); });
}

int pd_mg_create(void* ctx, int nlevels, void** mats, void** R, void** P, int nu, int partitions,
                 int restart, int smooth_solves, void** out) {
    return guarded([&] {
        if (nlevels < 1) throw pd::ConfigError("need at least one level");
        std::vector<std::unique_ptr<pd::Csr>> m, r, p;
        for (int l = 0; l < nlevels; ++l) m.emplace_back(H<pd::Csr>(mats[l], "level matrix"));
        for (int l = 0; l + 1 < nlevels; ++l) {
            r.emplace_back(H<pd::Csr>(R[l], "restriction"));
            p.emplace_back(H<pd::Csr>(P[l], "prolongation"));
        }
        *out = new pd::Multigrid(*C(ctx), std::move(m), std::move(r), std::move(p), nu, partitions,
                                 restart, smooth_solves);
    });
}
int pd_mg_level_matrix(void* mg, int level, void** out) {
    return guarded([&] {
        auto* M = H<pd::Multigrid>(mg, "multigrid");
        if (level < 0 || level >= M->num_levels()) throw pd::ConfigError("bad level index");
        *out = &M->level_matrix(level);
    });
}
int pd_mg_level_precond(void* mg, int level, void** ilu_out) {
    return guarded([&] {
        auto* M = H<pd::Multigrid>(mg, "multigrid");
        if (level < 0 || level + 1 >= M->num_levels())
            throw pd::ConfigError("level has no smoother (coarsest or out of range)");
        *ilu_out = M->level_precond(level);
    });
}
int pd_mg_set_fine_operator(void* mg, void* stop) {
    return guarded([&] {
        auto* M = H<pd::Multigrid>(mg, "multigrid");
        M->set_fine_operator(std::unique_ptr<pd::StOp>(static_cast<pd::StOp*>(stop)));
    });
}
int pd_mg_set_galerkin_intermediates(void* mg, int n, void** T) {
    return guarded([&] {
        std::vector<std::unique_ptr<pd::Csr>> v;
        for (int l = 0; l < n; ++l) v.emplace_back(H<pd::Csr>(T[l], "intermediate"));
        H<pd::Multigrid>(mg, "multigrid")->set_galerkin_intermediates(std::move(v));
    });
}
int pd_mg_set_fine_values(void* mg, const double* vals) {
    return guarded([&] { H<pd::Multigrid>(mg, "multigrid")->set_fine_values(vals); });
}
int pd_jacobian_values(void* ctx, int64_t Nt, int M, int64_t S, double dt, double gamma, int kind,
                       const double* Mq_dev, const double* mh_dev, void* L, const double* u,
                       double* jv) {
    return guarded([&] {
        if (kind != 1 && kind != 2) throw pd::ConfigError("unknown reaction kind");
        pd::jacobian_values(*C(ctx), Nt, M, S, dt, gamma, kind, Mq_dev, mh_dev,
                            *H<pd::Csr>(L, "L"), u, jv);
    });
}
int pd_mg_refactor(void* ctx, void* mg) {
    (void)ctx;
    return guarded([&] { H<pd::Multigrid>(mg, "multigrid")->refactor(); });
}
int pd_mg_vcycle(void* ctx, void* mg, const double* b, double* x) {
    return guarded([&] {
        auto* M = H<pd::Multigrid>(mg, "multigrid");
        M->enqueue_vcycle(b, x);
        M->check_errors();
        if (pd::vec_has_nonfinite(*C(ctx), x, M->fine_size()))
            throw pd::SolverError("V-cycle produced non-finite values");
    });
}
int pd_mg_solve(void* ctx, void* mg, const double* b, double* x, double tol_rel, double tol_abs,
                int max_cycles, pd_solve_report* rep, double* hist, int hist_cap) {
    (void)ctx;
    return guarded([&] {
        auto r = H<pd::Multigrid>(mg, "multigrid")->solve(b, x, tol_rel, tol_abs, max_cycles);
        fill_report(rep, r.iterations, r.converged, r.diverged, r.hist, hist, hist_cap);
    });
}
int pd_mg_destroy(void* mg) {
    return guarded([&] { delete static_cast<pd::Multigrid*>(mg); });
}

}  // extern "C"
