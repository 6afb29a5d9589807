// Internal host-side declarations of the paradiff-b200 native library.
// Everything crossing the C ABI lives in include/paradiff_b200.h; this header
// is the C++ runtime's view (contexts, device buffers, solver objects).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

// records the calling thread's last error for pd_last_error() (pd_capi.cu)
void pd_set_error_(const char* msg, int64_t index);

namespace pd {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
    int64_t index;
    explicit SolverError(const std::string& m, int64_t i = -1) : std::runtime_error(m), index(i) {}
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define PD_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t pd_e_ = (call);                                                          \
        if (pd_e_ != cudaSuccess)                                                            \
            throw ::pd::CudaError(std::string(#call) + ": " + cudaGetErrorString(pd_e_));   \
    } while (0)

#define PD_LAUNCH_CHECK() PD_CUDA(cudaGetLastError())

// Every kernel launch of the library goes through launch(): it counts the
// launches (pd_launch_count(), reported by bench.py as gpu_launches).
extern std::atomic<unsigned long long> g_launches;

template <typename... KArgs, typename... Args>
inline void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args&&... args) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
}

// Kernels launched while a stream is being captured do not run then: capture
// takes them back off the counter and every replay of the graph adds them.
inline uint64_t uncount_captured(unsigned long long before) {
    const unsigned long long k = g_launches.load() - before;
    g_launches.fetch_sub(k, std::memory_order_relaxed);
    return k;
}
inline void graph_launch(cudaGraphExec_t exec, uint64_t kernels, cudaStream_t st) {
    g_launches.fetch_add(kernels, std::memory_order_relaxed);
    PD_CUDA(cudaGraphLaunch(exec, st));
}

// Owning device allocation (cudaMalloc/cudaFree; allocation happens at
// plan/setup time only, never inside a solve).
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) PD_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

constexpr int kReduceMaxBlocks = 1024;

// Per-device context: one stream, a reduction workspace and a device
// property cache.  Single-threaded by contract (one context per GPU/rank).
struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sms = 148;
    DevBuf<double> red_partials;      // kReduceMaxBlocks * 4
    DevBuf<unsigned int> red_counter; // 4 counters
    DevBuf<double> scalars;           // small result slots
    DevBuf<int> flags;                // misc device flags
    // bumped by every call that changes device state a captured CUDA graph
    // would bake in (values, factors, plans): captured V-cycles are re-made
    uint64_t epoch = 0;
    explicit Ctx(int dev, cudaStream_t s);
    ~Ctx();
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
    int grid_for(int64_t n, int bs, int per_sm = 8) const;
};

// out = mode-`stride` product of W stacked grids with the n x n matrix phi
// (row-major; transpose=1: Phi^T, 0: Phi): hand-written FP64 GEMM (pd_modeprod.cu)
void mode_product(Ctx& c, const double* in, double* out, int64_t total, int64_t n,
                  int64_t stride, const double* phi, int transpose);

struct GridSpmv;  // structured copy of a 2D space-time grid operator (pd_gspmv.cu)

// CSR on device: int64 row pointers (nnz may exceed 2^31 at C3/C5 sizes),
// int32 column indices, fp64 values.  Column indices sorted per row.
struct Csr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    DevBuf<int64_t> rowptr;
    DevBuf<int32_t> col;
    DevBuf<double> val;
    // optional structured copy used by csr_spmv; writers of `val` set grid_stale
    mutable std::shared_ptr<GridSpmv> grid;
    mutable bool grid_stale = false;
    void values_changed() const { grid_stale = grid != nullptr; }
};

// Structured wavefront schedule of one ILU(0) triangular sweep (pd_wavefront.cu):
// tasks of G node grids x nline lines x npoint points (one CTA each, thread =
// (grid, line)), per-step blocks of pattern ids + factor values in `blob`.
struct WfPlan {
    int64_t n = 0, nslot = 0;
    int ntask = 0, T = 0, nline = 0, npoint = 0, R = 0, pwo = 0, maxS = 0, blocks = 0, npat = 0,
        ng = 0, threads = 0, stages = 3;
    bool pad = false;     // entry lists zero-padded to the kernel's chunk
    bool gfirst = false;  // cross-task entries lead every pattern (no ring slots)
    bool win = false;     // ... and are the previous step's 3x3 neighbourhood (register window)
    size_t smem = 0, stage_bytes = 0;
    DevBuf<int32_t> nsteps;
    DevBuf<int64_t> boff, bofs, q0;
    DevBuf<int32_t> pattern;         // per pattern: len, ng, global offsets
    DevBuf<int16_t> offs;            // per pattern and ring phase: source offsets
    DevBuf<unsigned char> blob;      // step blocks
    DevBuf<int32_t> srow, sstride, scount;  // value gather slots (one per row)
    DevBuf<int64_t> sval, sdiag;
    DevBuf<unsigned long long> trace;  // PD_WF_TRACE diagnostics
};

struct Wf2Plan;  // skewed-wavefront sweeps for structured 2D levels (pd_wf2.cu)

// ILU(0) factors with level schedules (see pd_sparse.cu).
struct Ilu0 {
    int64_t n = 0;
    const Csr* pattern = nullptr;   // pattern source (owned elsewhere) unless masked
    Csr masked;                     // block-Jacobi masked copy (pattern + values)
    bool use_masked = false;
    DevBuf<double> fac;             // factor values on the pattern
    DevBuf<int64_t> diag;           // diagonal positions
    DevBuf<int32_t> order_lo;       // rows in lower-solve level order
    // order_lo / order_up hold nt_lo / nt_up tasks: the rows in level order with every
    // level padded to a multiple of 32 (-1 = idle lane), so a warp never waits on itself
    int64_t nt_lo = 0, nt_up = 0;
    int max_row_nnz = 0;            // longest row of the pattern (warp-per-row factorization)
    DevBuf<int32_t> order_up;       // rows in upper-solve level order
    DevBuf<int> flag;               // per-row completion epochs
    DevBuf<unsigned long long> counter;
    DevBuf<int> ep;                 // device-resident sweep epoch (factorization)
    DevBuf<double> scratch;         // lower-sweep output, kept armed with the pending sentinel
    int nlevels_lo = 0, nlevels_up = 0;
    // level-ordered copies of each sweep's entries (task t = t-th row in level order)
    DevBuf<int64_t> tp_lo, tp_up;
    DevBuf<int32_t> tcol_lo, tcol_up;
    DevBuf<double> tval_lo, tval_up, tdiag;
    std::vector<std::pair<int64_t, int64_t>> ranges;
    std::unique_ptr<WfPlan> wf_lo, wf_up;  // structured sweeps (optional)
    std::shared_ptr<Wf2Plan> w2_lo, w2_up; // template-structured sweeps (preferred when set)
    const Csr& pat() const { return use_masked ? masked : *pattern; }
};

struct DenseLU {
    int64_t n = 0;
    DevBuf<double> lu;   // column-major n x n
    DevBuf<int32_t> piv; // LAPACK-style row interchanges (0-based)
};

// Banded LU with partial pivoting (pd_band.cu): the device counterpart of the SuperLU
// solves in spacetime.py:154-195.  A is the (already permuted) matrix; perm_host (may be
// null) maps band row i to the caller's unknown perm[i] for the solve's vectors.
struct BandLU;
BandLU* band_lu_create(Ctx& c, const Csr& A, int kl, int ku, const int32_t* perm_host);
void band_lu_solve(Ctx& c, BandLU& f, const double* b, double* x);
void band_lu_destroy(BandLU* f);

// ------------------------------------------------------------------ kernels (host wrappers)
// vector ops
void vec_fill(Ctx& c, double* x, int64_t n, double v);
void vec_copy(Ctx& c, double* y, const double* x, int64_t n);
void vec_axpy_inplace(Ctx& c, double* y, const double* x, int64_t n);  // y = y + x
// out = sqrt(sum x^2) written to device slot; returns nothing (async)
void vec_dot(Ctx& c, const double* x, const double* y, int64_t n, double* out_dev);
double vec_norm_host(Ctx& c, const double* x, int64_t n);  // synchronizing helper
bool vec_has_nonfinite(Ctx& c, const double* x, int64_t n);  // synchronizing

// CSR
enum SpmvMode { SPMV_SET = 0, SPMV_RESID = 1, SPMV_ADD = 2 };
void csr_spmv(Ctx& c, const Csr& A, const double* x, double* y, int mode, const double* b,
              const int* guard = nullptr, int want = 0, double* norm2_out = nullptr,
              int* nonfinite_flag = nullptr);
std::unique_ptr<Csr> csr_upload(Ctx& c, int64_t nrows, int64_t ncols, int64_t nnz,
                                const int64_t* rowptr, const int32_t* col, const double* val,
                                bool device_src);
void csr_update_values(Ctx& c, Csr& A, const double* val, bool device_src);

// structured Galerkin SpMV (pd_gspmv.cu): attach when A has the 2D grid
// space-time pattern (nt steps, M nodes, n x n points); grid_spmv = false when
// A has no structured copy
bool csr_attach_grid(Ctx& c, Csr& A, int64_t nt, int M, int64_t n);
bool grid_spmv(Ctx& c, const Csr& A, const double* x, double* y, int mode, const double* b,
               const int* guard, int want, double* norm2, int* nonfinite);

// ILU(0)
std::unique_ptr<Ilu0> ilu0_create(Ctx& c, const Csr& A, int nblocks);
void ilu0_refactor(Ctx& c, Ilu0& f);  // recompute numeric factor from the pattern's values
void ilu0_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard = nullptr,
                int want = 0);
// structured wavefront sweeps (pd_wavefront.cu): false = schedule not applicable
bool ilu0_set_wavefront(Ctx& c, Ilu0& f, int64_t ngroup, int64_t nline, int64_t npoint,
                        int64_t ngroup_lower);
void wf_gather(Ctx& c, Ilu0& f);
// template-structured sweeps (pd_wf2.cu): rows [task][M][nline][npoint]; false = not applicable
bool ilu0_set_wf2(Ctx& c, Ilu0& f, int M, int64_t nline, int64_t npoint);
void wf2_gather(Ctx& c, Ilu0& f);
void wf2_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard, int want);
// mixed executors: pattern-table lower sweep (b -> scratch), template upper (scratch -> x)
bool wf2_lower_preferred(const Ilu0& f);
void wf2_drop_lower(Ilu0& f);
void wf2_solve_upper(Ctx& c, Ilu0& f, double* x, const int* guard, int want);
void wf_solve_lower(Ctx& c, Ilu0& f, const double* b, const int* guard, int want);
// fill a sweep output with the value-as-flag pending sentinel (coalesced)
void arm_pending(Ctx& c, double* y, int64_t n, const int* guard, int want);  // refresh plan values after a (re)factorization
void wf_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard, int want);

// fixed-pattern SpGEMM values (scipy csr_matmat accumulation order)
void spgemm_values(Ctx& c, const Csr& A, const Csr& B, Csr& C);
// J = L + gamma (I (x) Mqh) diag(r'(u)) values on L's pattern
void jacobian_values(Ctx& c, int64_t Nt, int M, int64_t S, double dt, double gamma, int kind,
                     const double* Mq_dev, const double* mh_dev, const Csr& L, const double* u,
                     double* jv);

// dense LU
std::unique_ptr<DenseLU> dense_lu_from_csr(Ctx& c, const Csr& A);
void dense_lu_solve(Ctx& c, const DenseLU& f, const double* b, double* x);
DevBuf<double> dense_inverse(Ctx& c, const DenseLU& f);  // row-major inverse (synchronising)
void dense_inverse_apply(Ctx& c, const double* inv, int64_t n, const double* b, double* x);

}  // namespace pd
