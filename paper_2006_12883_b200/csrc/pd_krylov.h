// Device-resident restarted GMRES (right preconditioning, MGS, Givens) and the
// space-time multigrid V-cycle built on it.  Host C++ only enqueues kernels;
// all control decisions of linalg.py:215-311 live in a device struct, so a
// smoother pass (multigrid.py:243-256) needs no host synchronisation.
#pragma once

#include <functional>

#include "pd_internal.h"
#include "pd_stencil.h"

namespace pd {

constexpr int kGmMaxRestart = 256;  // restart lengths the reference tests use (up to 100)
enum GmPhase { GM_START = 0, GM_RUN = 1, GM_FINISH = 2, GM_DONE = 3 };

struct GmDev {
    int phase, j, k, total, cycles, vec_idx, vec_slot, err, converged, diverged, max_it, restart,
        has_x0, skip_final, final_res;
    double beta, thr, lowest, hn, last_res, tol_rel, tol_abs, beta0;
    double H[(kGmMaxRestart + 1) * kGmMaxRestart];  // row-major (restart+1) x restart
    double cs[kGmMaxRestart], sn[kGmMaxRestart], g[kGmMaxRestart + 1], y[kGmMaxRestart];
    double dots[kGmMaxRestart + 2];
};

class Gmres {
   public:
    // store_z: keep Z_j = M^{-1} V_j and update x with Z y (no extra preconditioner
    // apply per cycle); the smoother uses it, the standalone gmres mirrors linalg.py
    // external: the operator and the preconditioner are applied by the caller between the
    // engine's steps (time-slab sharded multigrid: halo exchanges and allreduced dots in
    // between); Z_j is kept like in the smoother
    Gmres(Ctx& c, const Csr* A, Ilu0* M, int64_t n, int restart, int max_it,
          bool store_z = false, bool external = false);
    // init from r0 = b - A x0 whose squared norm is at *norm2_dev; x0 may be
    // null (zero start, as in the smoother)
    void enqueue_init(const double* r0, const double* norm2_dev, double tol_rel, double tol_abs,
                      const double* x0 = nullptr);
    // one Arnoldi step slot (mgs_passes = max j + 2 this slot can need) plus
    // the guarded cycle-finish block; `b` = the GMRES right-hand side
    void enqueue_slot(int slot, int mgs_passes, const double* b);
    // the same Arnoldi step slot with the operator / preconditioner applications made
    // by host callables on device vectors (linalg.py:233-237 accepts any callable);
    // the vector work stays on the device, the host syncs around each callable
    using ApplyFn = std::function<void(const double* x, double* y)>;
    void slot_with_callables(int slot, int mgs_passes, const double* b, const ApplyFn& fa,
                             const ApplyFn* fm);
    // ---- externally driven smoother steps (mg_sharded): the caller applies M^{-1} to
    // V[j] into Z[j] and A to Z[j] into w, reduces dots[i] over the ranks after every
    // MGS pass, and calls ext_end; no host synchronisation anywhere
    void ext_begin(int j, const double** vin, double** zout, double** wout);
    void ext_mgs_pass(int i);
    double* ext_dots() { return st.p->dots; }
    void ext_end(int slot);
    void ext_apply(double* x);  // x += solution when a cycle ran
    const GmDev& read_state();  // synchronising; scalar header only (host mirror)
    double* x() { return xg.p; }
    int64_t size() const { return n; }
    GmDev* dev() { return st.p; }
    void set_operator(const StOp* o) { op = o; }
    std::vector<double> history(int total);
    void debug_dump(int slot);  // PD_GM_DEBUG: state and leading vector entries to stderr

   private:
    Ctx& c;
    const Csr* A;
    const StOp* op = nullptr;  // matrix-free A (level 0 of a structured hierarchy)
    Ilu0* M;
    int64_t n;
    int restart, max_it;
    DevBuf<GmDev> st;
    std::unique_ptr<GmDev> host_st;  // host mirror (the struct is ~0.5 MB: kept off the stack)
    bool store_z = false;
    DevBuf<double> V, w, z, u, rg, xg, norm2, hist, Z;
    const double* r0 = nullptr;
};

// Full restarted GMRES (linalg.py:215-311) with host-mirrored control
// (one sync per Arnoldi step): x = x0 + ...; x may alias x0.
struct GmresResult {
    int iterations = 0;
    bool converged = false, diverged = false;
    std::vector<double> hist;
};
GmresResult gmres_run(Ctx& c, const Csr& A, Ilu0* M, const double* b, const double* x0, double* x,
                      double tol_rel, double tol_abs, int restart, int max_it);
// The same solve with A and/or the preconditioner given as host callables on device
// vectors of length n (fm == nullptr: no preconditioner).
GmresResult gmres_run_callables(Ctx& c, int64_t n, const Gmres::ApplyFn& fa,
                                const Gmres::ApplyFn* fm, const double* b, const double* x0,
                                double* x, double tol_rel, double tol_abs, int restart,
                                int max_it);

// Enqueue x += GMRES(A, b - A x) with ILU/block-Jacobi right preconditioning,
// restart=min(nu,restart), max_it=nu, tol_rel=1e-13, tol_abs=0: exactly one
// smoothing solve of multigrid.py:243-256.  No host synchronisation.
// r_ready: r_work already holds b - A x and *r_norm2 its squared norm
void enqueue_gmres_smooth(Ctx& c, Gmres& g, const Csr& A, const StOp* op, const double* b,
                          double* x, double* r_work, int nu, const double* r_norm2 = nullptr);

struct MgLevel {
    std::unique_ptr<Csr> A, R, P;  // R/P: transfer to the next coarser level (unused on coarsest)
    std::unique_ptr<Ilu0> pre;
    std::unique_ptr<Gmres> gm;
    DevBuf<double> b, x, r;
    int64_t n = 0;
};

class Multigrid {
   public:
    Multigrid(Ctx& c, std::vector<std::unique_ptr<Csr>> mats, std::vector<std::unique_ptr<Csr>> R,
              std::vector<std::unique_ptr<Csr>> P, int nu, int partitions, int restart,
              int smooth_solves);
    ~Multigrid();
    Multigrid(const Multigrid&) = delete;
    Multigrid& operator=(const Multigrid&) = delete;
    // replace level matrix values (same patterns) and refactor (Newton refresh)
    void refactor();
    // device Galerkin: T_l = R_l A_l (scipy's stored order), A_{l+1} = T_l P_l
    void set_galerkin_intermediates(std::vector<std::unique_ptr<Csr>> T);
    // new fine values (device pointer, fine pattern) -> Galerkin -> refactor
    void set_fine_values(const double* vals);
    Csr& level_matrix(int l) { return *lv[l].A; }
    Ilu0* level_precond(int l) { return lv[l].pre.get(); }
    // level 0 applies A through a matrix-free operator (values must equal the CSR's)
    void set_fine_operator(std::unique_ptr<StOp> op);
    int num_levels() const { return (int)lv.size(); }
    int64_t fine_size() const { return lv[0].n; }
    // x <- V-cycle(b, x)  (device pointers, n = fine size); no host sync
    void enqueue_vcycle(const double* b, double* x);
    // full solve; returns iterations/flags, fills history; x in/out
    struct Report {
        int iterations = 0;
        bool converged = false, diverged = false;
        std::vector<double> hist;
    };
    Report solve(const double* b, double* x, double tol_rel, double tol_abs, int max_cycles);
    void check_errors();  // synchronising: raise SolverError on device-side failures

   private:
    void cycle(int l);
    // one V-cycle: eager launches, or the captured CUDA graph of the same launch
    // sequence when this (b, x, state epoch) was already solved once
    void run_vcycle(const double* b, double* x, bool use_graph);
    struct VGraph {
        const double* b = nullptr;
        double* x = nullptr;
        uint64_t epoch = ~0ull;
        cudaGraphExec_t exec = nullptr;
        uint64_t kernels = 0;  // this library's kernels in one replay
    };
    VGraph vgraph, vseen;
    bool graph_off = false;
    cudaStream_t cap_stream = nullptr;
    // per-cycle status (|r|^2, non-finite flag, every level's GMRES error code)
    // gathered on the device and read back with one copy into pinned memory
    static constexpr int kStatusMax = 2 + 32;
    DevBuf<double> status_dev;
    double* status_host = nullptr;
    const double* read_status(bool with_errors);
    const double* fine_r_norm2 = nullptr;  // set by solve(): lv[0].r already = b - A x
    Ctx& c;
    std::vector<MgLevel> lv;
    std::unique_ptr<DenseLU> coarse;
    std::unique_ptr<StOp> fine_op;
    std::vector<std::unique_ptr<Csr>> galerkin_T;
    DevBuf<double> coarse_inv;  // A_c^{-1} (row-major) when n_c <= kCoarseInverseMax
    int nu, partitions, restart, smooth_solves;
    DevBuf<double> res2;
    DevBuf<int> nonfinite;
};

}  // namespace pd
