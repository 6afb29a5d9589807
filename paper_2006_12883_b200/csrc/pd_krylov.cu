// Device-resident GMRES engine and V-cycle runtime (see pd_krylov.h).
//
//   Gmres              <- linalg.py:215-311 (restarted, right-preconditioned,
//                         MGS orthogonalisation, Givens, happy breakdown at
//                         1e-14*max(1,beta), true-residual check per restart,
//                         divergence when beta > 10*min)
//   enqueue_gmres_smooth <- multigrid.py:243-256 (_smooth)
//   Multigrid          <- multigrid.py:197-305 (_cycle, vcycle, solve)
//
// Scalar bookkeeping (Hessenberg, rotations, thresholds) runs in one-thread
// kernels on the device; vector kernels read the phase word and exit early
// when their stage is inactive.  The host only enqueues.
#include "pd_device.cuh"
#include <cstddef>

#include "pd_krylov.h"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace pd {

using namespace dev;

constexpr int KB = 256;
constexpr int64_t kCoarseInverseMax = 8192;  // 512 MB of inverse at most

__device__ __forceinline__ int vphase(const GmDev* s) { return *((volatile const int*)&s->phase); }

__global__ void k_gm_init(GmDev* s, const double* norm2, double tol_rel, double tol_abs,
                          int max_it, int restart, double* hist, int has_x0, int skip_final) {
    const double beta = sqrt(*norm2);
    s->has_x0 = has_x0;
    s->skip_final = skip_final;
    s->final_res = -1;
    s->max_it = max_it;
    s->restart = restart;
    s->tol_rel = tol_rel;
    s->tol_abs = tol_abs;
    s->total = 0;
    s->cycles = 0;
    s->j = 0;
    s->k = 0;
    s->err = 0;
    s->converged = 0;
    s->diverged = 0;
    s->vec_idx = -1;
    s->vec_slot = -1;
    s->beta = beta;
    s->beta0 = beta;
    s->last_res = beta;
    if (hist) hist[0] = beta;
    if (!isfinite(beta)) {
        s->err = 1;
        s->phase = GM_DONE;
        return;
    }
    const double thr = fmax(tol_abs, mul(tol_rel, beta));
    s->thr = thr;
    s->lowest = beta;
    if (beta <= thr) {
        s->converged = 1;
        s->phase = GM_DONE;
    } else {
        s->phase = GM_START;
    }
}

// V0 = r / beta (first cycle reads the initial residual r0, restarts read rg)
__global__ void k_gm_start_vec(const GmDev* s, const double* r0, const double* rg, double* V,
                               int64_t n) {
    if (vphase(s) != GM_START) return;
    const double beta = s->beta;
    const double* src = s->cycles == 0 ? r0 : rg;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        V[i] = src[i] / beta;
}

__global__ void k_gm_start(GmDev* s) {
    if (s->phase != GM_START) return;
    const int R = s->restart;
    for (int i = 0; i < (R + 1) * R; ++i) s->H[i] = 0.0;
    for (int i = 0; i <= R; ++i) s->g[i] = 0.0;
    s->g[0] = s->beta;
    s->j = 0;
    s->phase = GM_RUN;
}

// MGS pass i: (w -= h_{i-1} V_{i-1}) then dot(w, V_i) (or |w|^2 on the last pass)
__global__ void k_gm_mgs(GmDev* s, int i, double* w, const double* V, int64_t n,
                         double* partials, unsigned int* counter) {
    if (vphase(s) != GM_RUN) return;
    const int j = s->j;
    if (i > j + 1) return;
    double acc = 0.0;
    if (i == 0) {
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
             t += (int64_t)gridDim.x * blockDim.x)
            acc = fma(w[t], V[t], acc);
    } else {
        const double h = s->dots[i - 1];
        const double* Vp = V + (int64_t)(i - 1) * n;
        const double* Vi = V + (int64_t)i * n;
        const bool last = (i == j + 1);
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
             t += (int64_t)gridDim.x * blockDim.x) {
            const double wv = sub(w[t], mul(h, Vp[t]));
            w[t] = wv;
            acc = fma(wv, last ? wv : Vi[t], acc);
        }
    }
    grid_sum_finish<KB>(acc, partials, counter, &s->dots[i]);
}

// y = H[:k,:k]^{-1} g[:k]  (column-oriented back substitution, dtrsm order); runs at the
// end of the Arnoldi step that ends a cycle
__device__ void gm_finish_y(GmDev* s) {
    const int k = s->k, R = s->restart;
    for (int i = 0; i < k; ++i) s->y[i] = s->g[i];
    for (int c = k - 1; c >= 0; --c) {
        if (s->y[c] != 0.0) {
            s->y[c] = s->y[c] / s->H[c * R + c];
            const double yc = s->y[c];
            for (int i = 0; i < c; ++i) s->y[i] = sub(s->y[i], mul(yc, s->H[i * R + c]));
        }
    }
}

// Hessenberg column, Givens rotations, residual estimate, stop decision.
__global__ void k_gm_arnoldi(GmDev* s, int slot, double* hist) {
    if (s->phase != GM_RUN) return;
    const int j = s->j, R = s->restart;
    double* H = s->H;
#define HH(r, c) H[(r) * R + (c)]
    for (int i = 0; i <= j; ++i) HH(i, j) = s->dots[i];
    const double hn = sqrt(s->dots[j + 1]);
    HH(j + 1, j) = hn;
    const bool happy = hn <= mul(1e-14, fmax(1.0, s->beta));
    s->hn = hn;
    s->vec_idx = happy ? -1 : j + 1;
    s->vec_slot = slot;
    for (int i = 0; i < j; ++i) {
        const double t = add(mul(s->cs[i], HH(i, j)), mul(s->sn[i], HH(i + 1, j)));
        HH(i + 1, j) = add(mul(-s->sn[i], HH(i, j)), mul(s->cs[i], HH(i + 1, j)));
        HH(i, j) = t;
    }
    const double denom = hypot(HH(j, j), HH(j + 1, j));
    if (denom == 0.0) {
        s->cs[j] = 1.0;
        s->sn[j] = 0.0;
    } else {
        s->cs[j] = HH(j, j) / denom;
        s->sn[j] = HH(j + 1, j) / denom;
    }
    HH(j, j) = denom;
    HH(j + 1, j) = 0.0;
    s->g[j + 1] = mul(-s->sn[j], s->g[j]);
    s->g[j] = mul(s->cs[j], s->g[j]);
    const double res = fabs(s->g[j + 1]);
    if (!isfinite(res)) {
        s->err = 2;
        s->phase = GM_DONE;
        return;
    }
    s->total += 1;
    s->last_res = res;
    if (hist) hist[s->total] = res;
    // the cycle ends on convergence, breakdown, the iteration cap — or when the inner
    // loop `for j in range(restart)` (linalg.py:264) runs out
    if (res <= s->thr || happy || s->total >= s->max_it || j + 1 >= R) {
        s->k = j + 1;
        s->phase = GM_FINISH;
        // the closing true residual decides restarts and the report; a smoother
        // at its iteration cap needs neither (multigrid.py:246-255 drops it)
        s->final_res = (s->skip_final && s->total >= s->max_it) ? -1 : GM_FINISH;
        gm_finish_y(s);
    } else {
        s->j = j + 1;
    }
#undef HH
}

// V[j+1] = w / hn (the next step's preconditioner / operator input is read from V[j+1])
__global__ void k_gm_newvec(const GmDev* s, int slot, const double* w, double* V, int64_t n) {
    if (s->vec_slot != slot || s->vec_idx < 0) return;
    const int ph = vphase(s);
    if (ph != GM_RUN && ph != GM_FINISH) return;
    const double hn = s->hn;
    double* dst = V + (int64_t)s->vec_idx * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = w[i] / hn;
}

// u = V[:k]^T y
__global__ void k_gm_combine(const GmDev* s, const double* V, double* u, int64_t n) {
    if (vphase(s) != GM_FINISH) return;
    const int k = s->k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < k; ++l) acc = add(acc, mul(s->y[l], V[(int64_t)l * n + i]));
        u[i] = acc;
    }
}

// xg (+)= V[:k]^T y in one pass (no preconditioner apply between the two: the smoother's
// stored Z_j, or an unpreconditioned solve); the same sums as k_gm_combine + k_gm_update_x
__global__ void k_gm_combine_update(const GmDev* s, const double* V, double* xg, int64_t n) {
    if (vphase(s) != GM_FINISH) return;
    const int k = s->k;
    const bool first = s->cycles == 0 && !s->has_x0;  // x = 0 + du exactly
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < k; ++l) acc = add(acc, mul(s->y[l], V[(int64_t)l * n + i]));
        xg[i] = first ? acc : add(xg[i], acc);
    }
}

__global__ void k_gm_update_x(const GmDev* s, double* xg, const double* du, int64_t n) {
    if (vphase(s) != GM_FINISH) return;
    const bool first = s->cycles == 0 && !s->has_x0;  // x = 0 + du exactly
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        xg[i] = first ? du[i] : add(xg[i], du[i]);
}

__global__ void k_gm_restart(GmDev* s, const double* norm2, double* hist) {
    if (s->phase != GM_FINISH) return;
    s->cycles += 1;
    if (s->final_res != GM_FINISH) {  // smoother at its cap: done, residual not formed
        s->diverged = 1;
        s->phase = GM_DONE;
        return;
    }
    const double beta = sqrt(*norm2);
    if (!isfinite(beta)) {
        s->err = 3;
        s->phase = GM_DONE;
        return;
    }
    s->beta = beta;
    s->last_res = beta;
    if (hist) hist[s->total] = beta;
    s->lowest = fmin(s->lowest, beta);
    if (beta <= s->thr) {
        s->converged = 1;
        s->phase = GM_DONE;
    } else if (s->total >= s->max_it || beta > mul(10.0, s->lowest)) {
        s->diverged = 1;
        s->phase = GM_DONE;
    } else {
        s->phase = GM_START;
    }
}

// x += dx after the smoother's GMRES (x + 0 when no cycle ran)
__global__ void k_gm_apply(const GmDev* s, double* x, const double* xg, int64_t n) {
    if (s->cycles == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = add(x[i], xg[i]);
}

// ------------------------------------------------------------------ Gmres
Gmres::Gmres(Ctx& c_, const Csr* A_, Ilu0* M_, int64_t n_, int restart_, int max_it_,
             bool store_z_, bool external)
    : c(c_), A(A_), M(M_), n(n_), max_it(max_it_),
      store_z(store_z_ && (M_ != nullptr || external)) {
    restart = std::max<int64_t>(1, std::min<int64_t>(restart_, n_));
    if (restart > kGmMaxRestart)
        throw ConfigError("GMRES restart length above " + std::to_string(kGmMaxRestart));
    st.alloc(1);
    PD_CUDA(cudaMemset(st.p, 0, sizeof(GmDev)));
    V.alloc((size_t)(restart + 1) * std::max<int64_t>(n, 1));
    w.alloc(std::max<int64_t>(n, 1));
    z.alloc(std::max<int64_t>(n, 1));
    u.alloc(std::max<int64_t>(n, 1));
    rg.alloc(std::max<int64_t>(n, 1));
    xg.alloc(std::max<int64_t>(n, 1));
    if (store_z) Z.alloc((size_t)restart * std::max<int64_t>(n, 1));
    norm2.alloc(1);
    PD_CUDA(cudaMemset(norm2.p, 0, sizeof(double)));
    hist.alloc(std::max(max_it, 1) + 2);
}

void Gmres::enqueue_init(const double* r0_, const double* norm2_dev, double tol_rel,
                         double tol_abs, const double* x0) {
    r0 = r0_;
    if (x0) vec_copy(c, xg.p, x0, n);
    launch(k_gm_init, 1, 1, 0, c.stream, st.p, norm2_dev, tol_rel, tol_abs, max_it, restart, hist.p,
           x0 ? 1 : 0, store_z ? 1 : 0);
    PD_LAUNCH_CHECK();
}

void Gmres::enqueue_slot(int slot, int mgs_passes, const double* b) {
    const int g = c.grid_for(n, KB, 8);
    const int gr = std::min(c.grid_for(n, KB, 4), kReduceMaxBlocks);
    const int* ph = &st.p->phase;
    // the host knows this slot's Arnoldi index (callers pass j + 2 passes): the basis
    // vector V[j] is the input of the step, and a stored Z_j is written in place
    const int jh = std::max(0, std::min(mgs_passes - 2, restart - 1));
    const double* vin = V.p + (int64_t)jh * n;
    launch(k_gm_start_vec, g, KB, 0, c.stream, st.p, r0, rg.p, V.p, n);
    launch(k_gm_start, 1, 1, 0, c.stream, st.p);
    const double* zin = vin;
    if (M) {
        double* zout = store_z ? Z.p + (int64_t)jh * n : z.p;
        ilu0_solve(c, *M, vin, zout, ph, GM_RUN);
        zin = zout;
    }
    apply_A(c, *A, op, zin, w.p, SPMV_SET, nullptr, ph, GM_RUN);
    const int passes = std::min(mgs_passes, restart + 1);
    for (int i = 0; i < passes; ++i)
        launch(k_gm_mgs, gr, KB, 0, c.stream, st.p, i, w.p, V.p, n, c.red_partials.p,
                                          c.red_counter.p);
    launch(k_gm_arnoldi, 1, 1, 0, c.stream, st.p, slot, hist.p);
    launch(k_gm_newvec, g, KB, 0, c.stream, st.p, slot, w.p, V.p, n);
    // cycle finish (active only when this step ended the cycle; y is formed by k_gm_arnoldi)
    // x += M^{-1}(V y) (linalg.py:297); with stored Z_j = M^{-1} V_j this is
    // sum_j y_j Z_j — the same linear map, one ILU apply fewer per cycle
    if (!M || store_z) {
        launch(k_gm_combine_update, g, KB, 0, c.stream, st.p, store_z ? Z.p : V.p, xg.p, n);
    } else {
        launch(k_gm_combine, g, KB, 0, c.stream, st.p, V.p, u.p, n);
        ilu0_solve(c, *M, u.p, z.p, ph, GM_FINISH);
        launch(k_gm_update_x, g, KB, 0, c.stream, st.p, xg.p, (const double*)z.p, n);
    }
    apply_A(c, *A, op, xg.p, rg.p, SPMV_RESID, b, &st.p->final_res, GM_FINISH, norm2.p, nullptr);
    launch(k_gm_restart, 1, 1, 0, c.stream, st.p, norm2.p, hist.p);
    PD_LAUNCH_CHECK();
}

// ---- externally driven steps (time-slab sharded smoother, mg_sharded.py)
void Gmres::ext_begin(int j, const double** vin, double** zout, double** wout) {
    if (!store_z) throw ConfigError("external GMRES steps need stored Z vectors");
    if (j < 0 || j >= restart) throw ConfigError("Arnoldi index outside the restart length");
    const int g = c.grid_for(n, KB, 8);
    launch(k_gm_start_vec, g, KB, 0, c.stream, st.p, r0, rg.p, V.p, n);
    launch(k_gm_start, 1, 1, 0, c.stream, st.p);
    PD_LAUNCH_CHECK();
    *vin = V.p + (int64_t)j * n;
    *zout = Z.p + (int64_t)j * n;
    *wout = w.p;
}

void Gmres::ext_mgs_pass(int i) {
    const int gr = std::min(c.grid_for(n, KB, 4), kReduceMaxBlocks);
    launch(k_gm_mgs, gr, KB, 0, c.stream, st.p, i, w.p, V.p, n, c.red_partials.p, c.red_counter.p);
    PD_LAUNCH_CHECK();
}

void Gmres::ext_end(int slot) {
    const int g = c.grid_for(n, KB, 8);
    launch(k_gm_arnoldi, 1, 1, 0, c.stream, st.p, slot, hist.p);
    launch(k_gm_newvec, g, KB, 0, c.stream, st.p, slot, w.p, V.p, n);
    launch(k_gm_combine_update, g, KB, 0, c.stream, st.p, Z.p, xg.p, n);
    // a cycle that ends before the cap (residual estimate below 1e-13 |r0| or a happy
    // breakdown) is taken as converged: norm2 stays 0, so k_gm_restart reads a zero true
    // residual (the serial engine forms it; with tol 1e-13 it confirms the estimate)
    launch(k_gm_restart, 1, 1, 0, c.stream, st.p, norm2.p, hist.p);
    PD_LAUNCH_CHECK();
}

void Gmres::ext_apply(double* x) {
    launch(k_gm_apply, c.grid_for(n, KB, 8), KB, 0, c.stream, st.p, x, xg.p, n);
    PD_LAUNCH_CHECK();
}

// r = b - t (one rounding per entry, as numpy's b - matvec(x))
__global__ void k_gm_sub(double* r, const double* b, const double* t, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        r[i] = sub(b[i], t[i]);
}

void Gmres::slot_with_callables(int slot, int mgs_passes, const double* b, const ApplyFn& fa,
                                const ApplyFn* fm) {
    const int g = c.grid_for(n, KB, 8);
    const int gr = std::min(c.grid_for(n, KB, 4), kReduceMaxBlocks);
    launch(k_gm_start_vec, g, KB, 0, c.stream, st.p, r0, rg.p, V.p, n);
    launch(k_gm_start, 1, 1, 0, c.stream, st.p);
    PD_LAUNCH_CHECK();
    const GmDev& s = read_state();  // synchronising: the callables run on the host's clock
    if (s.phase == GM_RUN) {
        const double* vin = V.p + (int64_t)s.j * n;
        const double* zin = vin;
        if (fm) {
            (*fm)(vin, z.p);
            zin = z.p;
        }
        fa(zin, w.p);
    }
    const int passes = std::min(mgs_passes, restart + 1);
    for (int i = 0; i < passes; ++i)
        launch(k_gm_mgs, gr, KB, 0, c.stream, st.p, i, w.p, V.p, n, c.red_partials.p,
               c.red_counter.p);
    launch(k_gm_arnoldi, 1, 1, 0, c.stream, st.p, slot, hist.p);
    launch(k_gm_newvec, g, KB, 0, c.stream, st.p, slot, w.p, V.p, n);
    launch(k_gm_combine, g, KB, 0, c.stream, st.p, V.p, u.p, n);
    PD_LAUNCH_CHECK();
    read_state();
    if (s.phase != GM_FINISH) return;
    const double* du = u.p;
    if (fm) {
        (*fm)(u.p, z.p);
        du = z.p;
    }
    launch(k_gm_update_x, g, KB, 0, c.stream, st.p, xg.p, du, n);
    PD_CUDA(cudaStreamSynchronize(c.stream));
    if (s.final_res == GM_FINISH) {
        fa(xg.p, w.p);
        launch(k_gm_sub, g, KB, 0, c.stream, rg.p, b, (const double*)w.p, n);
        vec_dot(c, rg.p, rg.p, n, norm2.p);
    }
    launch(k_gm_restart, 1, 1, 0, c.stream, st.p, norm2.p, hist.p);
    PD_LAUNCH_CHECK();
}

const GmDev& Gmres::read_state() {
    // the host mirrors only the scalar header (phase, j, counters, flags)
    if (!host_st) host_st = std::make_unique<GmDev>();
    PD_CUDA(cudaMemcpyAsync(host_st.get(), st.p, offsetof(GmDev, H), cudaMemcpyDeviceToHost,
                            c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return *host_st;
}

void Gmres::debug_dump(int slot) {
    PD_CUDA(cudaStreamSynchronize(c.stream));
    auto full = std::make_unique<GmDev>();
    PD_CUDA(cudaMemcpy(full.get(), st.p, sizeof(GmDev), cudaMemcpyDeviceToHost));
    const GmDev& s = *full;
    fprintf(stderr, "[gm] slot %d phase %d j %d k %d total %d cycles %d final_res %d beta %.6g hn %.6g\n",
            slot, s.phase, s.j, s.k, s.total, s.cycles, s.final_res, s.beta, s.hn);
    fprintf(stderr, "     g %.6g %.6g %.6g  y %.6g %.6g  H00 %.6g H10 %.6g dots %.6g %.6g %.6g\n", s.g[0],
            s.g[1], s.g[2], s.y[0], s.y[1], s.H[0], s.H[s.restart], s.dots[0], s.dots[1], s.dots[2]);
    const int m = (int)std::min<int64_t>(n, 6);
    auto show = [&](const char* name, const double* p) {
        double h[6] = {0};
        PD_CUDA(cudaMemcpy(h, p, m * sizeof(double), cudaMemcpyDeviceToHost));
        fprintf(stderr, "     %-5s", name);
        for (int i = 0; i < m; ++i) fprintf(stderr, " %.6g", h[i]);
        fprintf(stderr, "\n");
    };
    show("V0", V.p);
    show("V1", V.p + n);
    show("w", w.p);
    show("u", u.p);
    show("xg", xg.p);
    show("rg", rg.p);
}

std::vector<double> Gmres::history(int total) {
    std::vector<double> h(total + 1);
    PD_CUDA(cudaMemcpyAsync(h.data(), hist.p, (total + 1) * sizeof(double), cudaMemcpyDeviceToHost,
                            c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return h;
}

void enqueue_gmres_smooth(Ctx& c, Gmres& g, const Csr& A, const StOp* op, const double* b,
                          double* x, double* r_work, int nu, const double* r_norm2) {
    const int64_t n = A.nrows;
    // r = b - A x with |r|^2 (the GMRES initial residual; x0 = 0 so r0 = r)
    if (!r_norm2) {
        apply_A(c, A, op, x, r_work, SPMV_RESID, b, nullptr, 0, c.scalars.p + 8, nullptr);
        r_norm2 = c.scalars.p + 8;
    }
    g.enqueue_init(r_work, r_norm2, 1e-13, 0.0);
    for (int s = 0; s < nu; ++s) g.enqueue_slot(s, s + 2, r_work);
    launch(k_gm_apply, c.grid_for(n, KB, 8), KB, 0, c.stream, g.dev(), x, g.x(), n);
    PD_LAUNCH_CHECK();
}

GmresResult gmres_run(Ctx& c, const Csr& A, Ilu0* M, const double* b, const double* x0, double* x,
                      double tol_rel, double tol_abs, int restart, int max_it) {
    if (A.nrows != A.ncols) throw ConfigError("GMRES needs a square matrix");
    if (max_it < 0) throw ConfigError("max_it must be nonnegative");
    const int64_t n = A.nrows;
    Gmres g(c, &A, M, n, restart, std::max(max_it, 1));
    // r0 = b - A x0 (x0 = 0 when absent: r0 = b, exactly as b - A@0)
    DevBuf<double> r0(std::max<int64_t>(n, 1)), zero;
    const double* xs = x0;
    if (!xs) {
        zero.alloc(std::max<int64_t>(n, 1));
        vec_fill(c, zero.p, n, 0.0);
        xs = zero.p;
    }
    csr_spmv(c, A, xs, r0.p, SPMV_RESID, b, nullptr, 0, c.scalars.p + 16, nullptr);
    g.enqueue_init(r0.p, c.scalars.p + 16, tol_rel, tol_abs, x0);
    const GmDev& s = g.read_state();  // refreshed in place by every read_state()
    // the host mirrors (phase, j) after every Arnoldi step; guards cover the rest
    int slot = 0;
    while (s.phase != GM_DONE && s.total < std::max(max_it, 1)) {
        const int j_eff = (s.phase == GM_START) ? 0 : s.j;
        g.enqueue_slot(slot++, j_eff + 2, b);
        g.read_state();
        if (getenv("PD_GM_DEBUG")) g.debug_dump(slot - 1);
    }
    if (s.err == 1) throw SolverError("non-finite initial residual in GMRES");
    if (s.err == 2) throw SolverError("non-finite residual in GMRES iteration");
    if (s.err == 3) throw SolverError("non-finite residual in GMRES restart");
    // the engine accumulates x = x0 + psolve(V y) per cycle, as the reference
    if (s.cycles > 0) {
        if (x != g.x()) vec_copy(c, x, g.x(), n);
    } else {
        if (x0) vec_copy(c, x, x0, n);
        else vec_fill(c, x, n, 0.0);
    }
    GmresResult r;
    r.hist = g.history(s.total);
    r.iterations = s.total;
    r.converged = s.converged != 0;
    r.diverged = s.diverged != 0;
    return r;
}

GmresResult gmres_run_callables(Ctx& c, int64_t n, const Gmres::ApplyFn& fa,
                                const Gmres::ApplyFn* fm, const double* b, const double* x0,
                                double* x, double tol_rel, double tol_abs, int restart,
                                int max_it) {
    if (n < 0) throw ConfigError("GMRES needs a nonnegative size");
    if (max_it < 0) throw ConfigError("max_it must be nonnegative");
    Gmres g(c, nullptr, nullptr, n, restart, std::max(max_it, 1));
    const int64_t n1 = std::max<int64_t>(n, 1);
    DevBuf<double> r0(n1), t(n1), zero;
    const double* xs = x0;
    if (!xs) {
        zero.alloc(n1);
        vec_fill(c, zero.p, n, 0.0);
        xs = zero.p;
    }
    PD_CUDA(cudaStreamSynchronize(c.stream));
    fa(xs, t.p);  // r0 = b - matvec(x0), also for a zero start (linalg.py:243)
    launch(k_gm_sub, c.grid_for(n, KB, 8), KB, 0, c.stream, r0.p, b, (const double*)t.p, n);
    vec_dot(c, r0.p, r0.p, n, c.scalars.p + 16);
    g.enqueue_init(r0.p, c.scalars.p + 16, tol_rel, tol_abs, x0);
    const GmDev& s = g.read_state();
    int slot = 0;
    while (s.phase != GM_DONE && s.total < std::max(max_it, 1)) {
        const int j_eff = (s.phase == GM_START) ? 0 : s.j;
        g.slot_with_callables(slot++, j_eff + 2, b, fa, fm);
        g.read_state();
    }
    if (s.err == 1) throw SolverError("non-finite initial residual in GMRES");
    if (s.err == 2) throw SolverError("non-finite residual in GMRES iteration");
    if (s.err == 3) throw SolverError("non-finite residual in GMRES restart");
    if (s.cycles > 0) {
        vec_copy(c, x, g.x(), n);
    } else {
        if (x0) {
            if (x != x0) vec_copy(c, x, x0, n);
        } else {
            vec_fill(c, x, n, 0.0);
        }
    }
    GmresResult r;
    r.hist = g.history(s.total);
    r.iterations = s.total;
    r.converged = s.converged != 0;
    r.diverged = s.diverged != 0;
    return r;
}

// ------------------------------------------------------------------ Multigrid
Multigrid::Multigrid(Ctx& c_, std::vector<std::unique_ptr<Csr>> mats,
                     std::vector<std::unique_ptr<Csr>> R, std::vector<std::unique_ptr<Csr>> P,
                     int nu_, int partitions_, int restart_, int smooth_solves_)
    : c(c_), nu(nu_), partitions(partitions_), restart(restart_), smooth_solves(smooth_solves_) {
    const int L = (int)mats.size();
    if (L < 1) throw ConfigError("need at least one level");
    if ((int)R.size() != L - 1 || (int)P.size() != L - 1)
        throw ConfigError("need one restriction/prolongation per level transition");
    if (nu < 1) throw ConfigError("need at least one smoothing iteration");
    lv.resize(L);
    for (int l = 0; l < L; ++l) {
        MgLevel& m = lv[l];
        m.A = std::move(mats[l]);
        m.n = m.A->nrows;
        if (m.A->nrows != m.A->ncols) throw ConfigError("level matrices must be square");
        if (l < L - 1) {
            m.R = std::move(R[l]);
            m.P = std::move(P[l]);
            if (m.R->ncols != m.n || m.P->nrows != m.n)
                throw ConfigError("transfer shapes do not match level " + std::to_string(l + 1));
        }
        if (l > 0) {
            m.b.alloc(std::max<int64_t>(m.n, 1));
            m.x.alloc(std::max<int64_t>(m.n, 1));
        }
        m.r.alloc(std::max<int64_t>(m.n, 1));
    }
    for (int l = 0; l + 1 < L; ++l)
        if (lv[l].R->nrows != lv[l + 1].n)
            throw ConfigError("restriction output does not match level " + std::to_string(l + 2));
    res2.alloc(1);
    nonfinite.alloc(1);
    refactor();
}

void Multigrid::set_fine_operator(std::unique_ptr<StOp> op) {
    ++c.epoch;
    if (op && op->size() != lv[0].n) throw ConfigError("fine operator size does not match level 1");
    fine_op = std::move(op);
    if (lv.size() > 1 && lv[0].gm) lv[0].gm->set_operator(fine_op.get());
}

void Multigrid::set_galerkin_intermediates(std::vector<std::unique_ptr<Csr>> T) {
    ++c.epoch;
    if (T.size() + 1 != lv.size()) throw ConfigError("need one R*A intermediate per transfer");
    for (size_t l = 0; l < T.size(); ++l)
        if (T[l]->nrows != lv[l].R->nrows || T[l]->ncols != lv[l].n)
            throw ConfigError("R*A intermediate has the wrong shape");
    galerkin_T = std::move(T);
}

void Multigrid::set_fine_values(const double* vals) {
    ++c.epoch;
    if (galerkin_T.empty() && lv.size() > 1)
        throw ConfigError("device Galerkin refresh needs the R*A intermediate patterns");
    Csr& A0 = *lv[0].A;
    PD_CUDA(cudaMemcpyAsync(A0.val.p, vals, A0.nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                            c.stream));
    A0.values_changed();
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
        spgemm_values(c, *lv[l].R, *lv[l].A, *galerkin_T[l]);
        spgemm_values(c, *galerkin_T[l], *lv[l].P, *lv[l + 1].A);
    }
    refactor();
}

void Multigrid::refactor() {
    ++c.epoch;
    const int L = (int)lv.size();
    for (int l = 0; l + 1 < L; ++l) {
        MgLevel& m = lv[l];
        const int blocks = (int)std::min<int64_t>(partitions, m.n);
        if (!m.pre) {
            m.pre = ilu0_create(c, *m.A, std::max(blocks, 1));
            m.gm = std::make_unique<Gmres>(c, m.A.get(), m.pre.get(), m.n,
                                           std::min(nu, restart), nu, /*store_z=*/true);
        } else {
            ilu0_refactor(c, *m.pre);
        }
    }
    coarse = dense_lu_from_csr(c, *lv[L - 1].A);
    coarse_inv.release();
    if (lv[L - 1].n <= kCoarseInverseMax) coarse_inv = dense_inverse(c, *coarse);
}

void Multigrid::cycle(int l) {
    MgLevel& m = lv[l];
    const int L = (int)lv.size();
    double* b = m.b.p;
    double* x = m.x.p;
    if (l == L - 1) {
        if (coarse_inv.p) dense_inverse_apply(c, coarse_inv.p, m.n, b, x);
        else dense_lu_solve(c, *coarse, b, x);
        return;
    }
    const StOp* op = (l == 0) ? fine_op.get() : nullptr;
    for (int s = 0; s < smooth_solves; ++s) {
        // the solve loop's stopping test already formed r = b - A x at level 1
        const double* ready = (l == 0 && s == 0) ? fine_r_norm2 : nullptr;
        enqueue_gmres_smooth(c, *m.gm, *m.A, op, b, x, m.r.p, nu, ready);
    }
    if (l == 0) fine_r_norm2 = nullptr;
    apply_A(c, *m.A, op, x, m.r.p, SPMV_RESID, b);
    MgLevel& nx = lv[l + 1];
    csr_spmv(c, *m.R, m.r.p, nx.b.p, SPMV_SET, nullptr);
    if (l + 1 < L - 1) vec_fill(c, nx.x.p, nx.n, 0.0);
    cycle(l + 1);
    csr_spmv(c, *m.P, nx.x.p, x, SPMV_ADD, x);
    for (int s = 0; s < smooth_solves; ++s)
        enqueue_gmres_smooth(c, *m.gm, *m.A, op, b, x, m.r.p, nu);
}

Multigrid::~Multigrid() {
    if (vgraph.exec) cudaGraphExecDestroy(vgraph.exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (status_host) cudaFreeHost(status_host);
}

namespace {
struct MgStatusArgs {
    const GmDev* g[30];
    int nl;
    const double* res2;
    const int* nonfinite;
};
__global__ void k_mg_status(MgStatusArgs a, double* out) {
    if (threadIdx.x != 0) return;
    out[0] = *a.res2;
    out[1] = a.nonfinite ? (double)*a.nonfinite : 0.0;
    for (int l = 0; l < a.nl; ++l) out[2 + l] = (double)a.g[l]->err;
}
}  // namespace

const double* Multigrid::read_status(bool with_errors) {
    const int L = (int)lv.size();
    if (!status_host) {
        PD_CUDA(cudaHostAlloc(&status_host, kStatusMax * sizeof(double), cudaHostAllocDefault));
        status_dev.alloc(kStatusMax);
    }
    MgStatusArgs a{};
    a.nl = with_errors ? std::min(L - 1, 30) : 0;
    for (int l = 0; l < a.nl; ++l) a.g[l] = lv[l].gm->dev();
    a.res2 = res2.p;
    a.nonfinite = with_errors ? nonfinite.p : nullptr;
    launch(k_mg_status, 1, 32, 0, c.stream, a, status_dev.p);
    PD_CUDA(cudaMemcpyAsync(status_host, status_dev.p, (2 + a.nl) * sizeof(double),
                            cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    for (int l = 0; l < a.nl; ++l) {
        const int err = (int)status_host[2 + l];
        if (err == 1) throw SolverError("non-finite initial residual in GMRES");
        if (err == 2) throw SolverError("non-finite residual in GMRES iteration");
        if (err == 3) throw SolverError("non-finite residual in GMRES restart");
    }
    return status_host;
}

void Multigrid::run_vcycle(const double* b, double* x, bool use_graph) {
    if (!use_graph || graph_off) {
        enqueue_vcycle(b, x);
        return;
    }
    if (!(vgraph.exec && vgraph.b == b && vgraph.x == x && vgraph.epoch == c.epoch)) {
        // capture on a private stream (the context's may be the legacy default
        // stream, which cannot be captured); the graph replays on the context's
        if (!cap_stream) PD_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
        const cudaStream_t orig = c.stream;
        cudaGraph_t graph = nullptr;
        c.stream = cap_stream;
        PD_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeRelaxed));
        const unsigned long long l0 = g_launches.load();
        try {
            enqueue_vcycle(b, x);
        } catch (...) {
            cudaStreamEndCapture(cap_stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            c.stream = orig;
            uncount_captured(l0);
            throw;
        }
        const cudaError_t ce = cudaStreamEndCapture(cap_stream, &graph);
        const uint64_t nk = uncount_captured(l0);
        c.stream = orig;
        cudaGraphExec_t exec = nullptr;
        if (ce == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
            if (vgraph.exec) cudaGraphExecDestroy(vgraph.exec);
            vgraph = VGraph{b, x, c.epoch, exec, nk};
        } else {  // something in the cycle is not capturable: stay eager
            (void)cudaGetLastError();
            graph_off = true;
        }
        if (graph) cudaGraphDestroy(graph);
        if (graph_off) {
            enqueue_vcycle(b, x);
            return;
        }
    }
    graph_launch(vgraph.exec, vgraph.kernels, c.stream);
}

void Multigrid::enqueue_vcycle(const double* b, double* x) {
    // level 0 works directly on the caller's vectors
    MgLevel& m = lv[0];
    double* sb = m.b.p;
    double* sx = m.x.p;
    m.b.p = const_cast<double*>(b);
    m.x.p = x;
    try {
        cycle(0);
    } catch (...) {
        m.b.p = sb;
        m.x.p = sx;
        fine_r_norm2 = nullptr;
        throw;
    }
    m.b.p = sb;
    m.x.p = sx;
}

void Multigrid::check_errors() {
    const int L = (int)lv.size();
    std::vector<GmDev> h(L > 1 ? L - 1 : 0);
    for (int l = 0; l + 1 < L; ++l)
        PD_CUDA(cudaMemcpyAsync(&h[l], lv[l].gm->dev(), offsetof(GmDev, H),
                                cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    for (int l = 0; l + 1 < L; ++l) {
        if (h[l].err == 1) throw SolverError("non-finite initial residual in GMRES");
        if (h[l].err == 2) throw SolverError("non-finite residual in GMRES iteration");
        if (h[l].err == 3) throw SolverError("non-finite residual in GMRES restart");
    }
}

Multigrid::Report Multigrid::solve(const double* b, double* x, double tol_rel, double tol_abs,
                                   int max_cycles) {
    Report rep;
    MgLevel& f = lv[0];
    const int64_t n = f.n;
    double* r = f.r.p;
    apply_A(c, *f.A, fine_op.get(), x, r, SPMV_RESID, b, nullptr, 0, res2.p, nullptr);
    double res = std::sqrt(read_status(false)[0]);
    rep.hist.push_back(res);
    const double thr = std::max(tol_abs, tol_rel * res);
    double lowest = res;
    // a repeated solve of the same state and vectors replays the captured cycle
    // (the first solve runs eagerly: it also settles lazily refreshed copies)
    const bool use_graph = !getenv("PD_MG_NO_GRAPH") && vseen.b == b && vseen.x == x &&
                           vseen.epoch == c.epoch;
    vseen = VGraph{b, x, c.epoch, nullptr};
    while (res > thr) {
        if (rep.iterations >= max_cycles) {
            rep.diverged = true;
            break;
        }
        fine_r_norm2 = res2.p;  // lv[0].r holds b - A x for the current x
        run_vcycle(b, x, use_graph);
        fine_r_norm2 = nullptr;
        PD_CUDA(cudaMemsetAsync(nonfinite.p, 0, sizeof(int), c.stream));
        apply_A(c, *f.A, fine_op.get(), x, r, SPMV_RESID, b, nullptr, 0, res2.p, nonfinite.p);
        const double* st = read_status(true);  // synchronises; raises GMRES errors
        if (st[1] != 0.0) throw SolverError("V-cycle produced non-finite values");
        res = std::sqrt(st[0]);
        rep.iterations += 1;
        rep.hist.push_back(res);
        if (!std::isfinite(res) || res > 10.0 * lowest) {
            rep.diverged = true;
            break;
        }
        lowest = std::min(lowest, res);
    }
    rep.converged = res <= thr;
    (void)n;
    return rep;
}

}  // namespace pd
