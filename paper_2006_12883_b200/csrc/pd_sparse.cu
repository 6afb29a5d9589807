// Sparse and dense linear-algebra kernels of the P-ref (reference-exact) path.
//
//   csr_spmv      <- scipy csr_matvec used by every `A @ x` in multigrid.py /
//                    linalg.py (row sums in CSR order, separately rounded, so
//                    the products reproduce scipy bitwise)
//   ilu0_*        <- linalg.py:63-145 (_ilu0_factor/_ilu0_solve/Ilu0) and the
//                    block-Jacobi masking of linalg.py:152-189
//   dense_lu_*    <- linalg.py:196-209 (LAPACK getrf/getrs on the coarsest level)
//
// ILU(0) on the GPU: the dependency DAG of the CSR pattern is analysed once
// (sync-free, per-row level = 1 + max level of its lower/upper neighbours),
// rows are radix-sorted by level, and factor/solve kernels process rows in
// that order with per-row completion flags (acquire/release).  Rows are
// fetched dynamically in topological order, so every waited-on row is owned
// by a thread that is already running: no deadlock for any grid size.  Each
// row's arithmetic follows the reference's sequential order exactly.
#include "pd_device.cuh"

#include "pd_internal.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace pd {

using namespace dev;

std::atomic<unsigned long long> g_launches{0};

Ctx::Ctx(int dev_, cudaStream_t s) : device(dev_), stream(s) {
    PD_CUDA(cudaSetDevice(device));
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    red_partials.alloc(kReduceMaxBlocks * 4);
    red_counter.alloc(4);
    PD_CUDA(cudaMemset(red_counter.p, 0, 4 * sizeof(unsigned int)));
    scalars.alloc(64);
    flags.alloc(64);
    PD_CUDA(cudaMemset(flags.p, 0, 64 * sizeof(int)));
}

Ctx::~Ctx() = default;

int Ctx::grid_for(int64_t n, int bs, int per_sm) const {
    int64_t g = (n + bs - 1) / bs;
    int64_t cap = (int64_t)sms * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ------------------------------------------------------------------ vector kernels
constexpr int BS = 256;
// Sync-free sweeps keep only ~2 blocks per SM resident: enough rows in flight
// to cover a few dependency levels, few enough that flag polling does not
// flood L2 (33 ms -> see profiles/ for the measured effect).
static int sweep_blocks_per_sm() {
    static int v = [] {
        const char* e = getenv("PD_SWEEP_BPS");
        int k = e ? atoi(e) : 2;
        return k > 0 ? k : 2;
    }();
    return v;
}

__global__ void k_fill(double* x, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void k_axpy_inplace(double* y, const double* x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = add(y[i], x[i]);
}

__global__ void k_dot(const double* x, const double* y, int64_t n, double* partials,
                      unsigned int* counter, double* out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s = fma(x[i], y[i], s);
    grid_sum_finish<BS>(s, partials, counter, out);
}

__global__ void k_nonfinite(const double* x, int64_t n, int* flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) bad = true;
    if (bad) atomicOr(flag, 1);
}

bool vec_has_nonfinite(Ctx& c, const double* x, int64_t n) {
    PD_CUDA(cudaMemsetAsync(c.flags.p, 0, sizeof(int), c.stream));
    if (n > 0) launch(k_nonfinite, c.grid_for(n, BS), BS, 0, c.stream, x, n, c.flags.p);
    int h = 0;
    PD_CUDA(cudaMemcpyAsync(&h, c.flags.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return h != 0;
}

void vec_fill(Ctx& c, double* x, int64_t n, double v) {
    if (n <= 0) return;
    launch(k_fill, c.grid_for(n, BS), BS, 0, c.stream, x, n, v);
    PD_LAUNCH_CHECK();
}

void vec_copy(Ctx& c, double* y, const double* x, int64_t n) {
    if (n <= 0 || y == x) return;
    PD_CUDA(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
}

void vec_axpy_inplace(Ctx& c, double* y, const double* x, int64_t n) {
    if (n <= 0) return;
    launch(k_axpy_inplace, c.grid_for(n, BS), BS, 0, c.stream, y, x, n);
    PD_LAUNCH_CHECK();
}

void vec_dot(Ctx& c, const double* x, const double* y, int64_t n, double* out_dev) {
    int g = std::min(c.grid_for(n, BS, 4), kReduceMaxBlocks);
    launch(k_dot, g, BS, 0, c.stream, x, y, n, c.red_partials.p, c.red_counter.p, out_dev);
    PD_LAUNCH_CHECK();
}

double vec_norm_host(Ctx& c, const double* x, int64_t n) {
    vec_dot(c, x, x, n, c.scalars.p);
    double h = 0.0;
    PD_CUDA(cudaMemcpyAsync(&h, c.scalars.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return std::sqrt(h);
}

// ------------------------------------------------------------------ CSR SpMV
// One thread per row, CSR order, sum starting at 0.0 like scipy's csr_matvec
// (so results are bitwise scipy's).  Each CTA owns a tile of BS consecutive
// rows; the tile's contiguous (values, columns) range is streamed through
// shared memory with coalesced loads (padded by one slot per 16 entries to
// spread banks), then every thread walks its own row in order.
// mode: 0 y = Ax, 1 y = b - Ax, 2 y = b + Ax.  Optional fused sum of y^2 and a
// non-finite flag on x (the V-cycle's isfinite check, multigrid.py:271).
constexpr int kSpmvCap = 2048;  // staged entries per chunk (24 KB + padding)
__device__ __forceinline__ int spad(int k) { return k + (k >> 4); }

template <bool REDUCE>
__global__ void __launch_bounds__(BS) k_spmv(int64_t n, const int64_t* __restrict__ rp,
                                             const int32_t* __restrict__ ci,
                                             const double* __restrict__ v,
                                             const double* __restrict__ x, double* y, int mode,
                                             const double* b,  // y may alias b (x += P xc)
                                             const int* guard, int want, double* partials,
                                             unsigned int* counter, double* norm2,
                                             int* nonfinite) {
    if (guard_off(guard, want)) return;
    __shared__ double sv[kSpmvCap + kSpmvCap / 16];
    __shared__ int32_t sc[kSpmvCap + kSpmvCap / 16];
    double acc2 = 0.0;
    bool bad = false;
    for (int64_t r0 = (int64_t)blockIdx.x * BS; r0 < n; r0 += (int64_t)gridDim.x * BS) {
        const int64_t i = r0 + threadIdx.x;
        const int64_t rend = min(r0 + (int64_t)BS, n);
        const int64_t e0 = rp[r0], e1 = rp[rend];
        int64_t a = 0, bnd = 0;
        if (i < n) {
            a = rp[i];
            bnd = rp[i + 1];
        }
        double s = 0.0;
        for (int64_t c0 = e0; c0 < e1; c0 += kSpmvCap) {
            const int cnt = (int)min((int64_t)kSpmvCap, e1 - c0);
            __syncthreads();
            for (int k = threadIdx.x; k < cnt; k += BS) {
                sv[spad(k)] = __ldcs(v + c0 + k);
                sc[spad(k)] = __ldcs(ci + c0 + k);
            }
            __syncthreads();
            // four gathers in flight before their multiply/add chain (same order)
            const int klo = (int)(max(a, c0) - c0), khi = (int)(min(bnd, c0 + cnt) - c0);
            for (int k0 = klo; k0 < khi; k0 += 4) {
                double xv[4], fv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = spad(min(k0 + u, khi - 1));
                    fv[u] = sv[k];
                    xv[u] = __ldg(x + sc[k]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (k0 + u < khi) s = add(s, mul(fv[u], xv[u]));
            }
        }
        if (i < n) {
            double out = s;
            if (mode == 1) out = sub(b[i], s);
            else if (mode == 2) out = add(b[i], s);
            y[i] = out;
            if (REDUCE) {
                acc2 = fma(out, out, acc2);
                if (nonfinite && !isfinite(x[i])) bad = true;
            }
        }
    }
    if (REDUCE) {
        if (bad) atomicOr(nonfinite, 1);
        grid_sum_finish<BS>(acc2, partials, counter, norm2);
    }
}

void csr_spmv(Ctx& c, const Csr& A, const double* x, double* y, int mode, const double* b,
              const int* guard, int want, double* norm2_out, int* nonfinite_flag) {
    if (A.nrows <= 0) return;
    if (A.grid && grid_spmv(c, A, x, y, mode, b, guard, want, norm2_out, nonfinite_flag)) return;
    if (norm2_out) {
        int g = std::min(c.grid_for(A.nrows, BS, 8), kReduceMaxBlocks);
        launch(k_spmv<true>, g, BS, 0, c.stream, A.nrows, A.rowptr.p, A.col.p, A.val.p, x, y,
               mode, b, guard, want, c.red_partials.p, c.red_counter.p, norm2_out,
               nonfinite_flag);
    } else {
        int g = c.grid_for(A.nrows, BS, 8);
        launch(k_spmv<false>, g, BS, 0, c.stream, A.nrows, A.rowptr.p, A.col.p, A.val.p, x, y,
               mode, b, guard, want, (double*)nullptr, (unsigned int*)nullptr, (double*)nullptr,
               (int*)nullptr);
    }
    PD_LAUNCH_CHECK();
}

std::unique_ptr<Csr> csr_upload(Ctx& c, int64_t nrows, int64_t ncols, int64_t nnz,
                                const int64_t* rowptr, const int32_t* col, const double* val,
                                bool device_src) {
    auto A = std::make_unique<Csr>();
    A->nrows = nrows;
    A->ncols = ncols;
    A->nnz = nnz;
    A->rowptr.alloc(nrows + 1);
    A->col.alloc(std::max<int64_t>(nnz, 1));
    A->val.alloc(std::max<int64_t>(nnz, 1));
    auto kind = device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    PD_CUDA(cudaMemcpyAsync(A->rowptr.p, rowptr, (nrows + 1) * sizeof(int64_t), kind, c.stream));
    if (nnz) {
        PD_CUDA(cudaMemcpyAsync(A->col.p, col, nnz * sizeof(int32_t), kind, c.stream));
        PD_CUDA(cudaMemcpyAsync(A->val.p, val, nnz * sizeof(double), kind, c.stream));
    }
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return A;
}

void csr_update_values(Ctx& c, Csr& A, const double* val, bool device_src) {
    ++c.epoch;
    if (!A.nnz) return;
    PD_CUDA(cudaMemcpyAsync(A.val.p, val, A.nnz * sizeof(double),
                            device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            c.stream));
    A.values_changed();
}

// ------------------------------------------------------------------ block-Jacobi masking
// Keep only entries whose column lies in the row's block (linalg.py:166-171:
// A[r0:r1, r0:r1] per block).  ILU(0) of the block-diagonal matrix equals the
// per-block ILU(0)s exactly, so one factorization serves all blocks.
__device__ __forceinline__ int64_t block_of(int64_t i, int64_t size, int64_t nblocks) {
    int64_t b = i / size;
    return b < nblocks - 1 ? b : nblocks - 1;
}

__global__ void k_mask_count(int64_t n, const int64_t* rp, const int32_t* ci, int64_t size,
                             int64_t nblocks, int64_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t bi = block_of(i, size, nblocks), k = 0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
            if (block_of(ci[p], size, nblocks) == bi) ++k;
        cnt[i + 1] = k;
    }
}

__global__ void k_mask_copy(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                            int64_t size, int64_t nblocks, const int64_t* orp, int32_t* oci,
                            double* ov) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t bi = block_of(i, size, nblocks), q = orp[i];
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
            if (block_of(ci[p], size, nblocks) == bi) {
                oci[q] = ci[p];
                ov[q] = v[p];
                ++q;
            }
    }
}

// ------------------------------------------------------------------ level analysis
__device__ __forceinline__ int64_t fetch_batch(unsigned long long* counter) {
    __shared__ long long base;
    if (threadIdx.x == 0) base = (long long)atomicAdd(counter, (unsigned long long)blockDim.x);
    __syncthreads();
    long long b = base;
    __syncthreads();
    return b;
}

// level[i] = 1 + max(level of lower neighbours); natural order fetch.
__global__ void k_levels_lower(int64_t n, const int64_t* rp, const int32_t* ci, int* level,
                               unsigned long long* counter) {
    for (;;) {
        int64_t base = fetch_batch(counter);
        if (base >= n) return;
        int64_t i = base + threadIdx.x;
        if (i < n) {
            int lev = 0;
            for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
                int64_t cc = ci[p];
                if (cc >= i) break;
                int lc;
                while ((lc = ld_acquire(level + cc)) < 0) __nanosleep(32);
                lev = max(lev, lc + 1);
            }
            st_release(level + i, lev);
        }
    }
}

// upper DAG: row i depends on its columns > i; processed from the last row.
__global__ void k_levels_upper(int64_t n, const int64_t* rp, const int32_t* ci, int* level,
                               unsigned long long* counter) {
    for (;;) {
        int64_t base = fetch_batch(counter);
        if (base >= n) return;
        int64_t t = base + threadIdx.x;
        if (t < n) {
            int64_t i = n - 1 - t;
            int lev = 0;
            for (int64_t p = rp[i + 1] - 1; p >= rp[i]; --p) {
                int64_t cc = ci[p];
                if (cc <= i) break;
                int lc;
                while ((lc = ld_acquire(level + cc)) < 0) __nanosleep(32);
                lev = max(lev, lc + 1);
            }
            st_release(level + i, lev);
        }
    }
}

__global__ void k_iota(int32_t* x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (int32_t)i;
}

__global__ void k_fill_int(int* x, int64_t n, int v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void k_max_rowlen(int64_t n, const int64_t* rp, int* out) {
    int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (int)min((int64_t)INT_MAX, rp[i + 1] - rp[i]));
    if (m > 0) atomicMax(out, m);
}

__global__ void k_max_int(const int* x, int64_t n, int* out) {
    int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, x[i]);
    atomicMax(out, m);
}

// ------------------------------------------------------------------ ILU(0) factorization
// Per row, exactly linalg.py:73-96: for each lower entry k (ascending):
// l_ik = a_ik / u_kk; a_ij -= l_ik * u_kj over the intersection of row k's
// upper pattern with row i (two-pointer merge instead of the position map).
// Warp-per-row ILU(0) factorization (IKJ order, linalg.py:78-98): the row lives in shared
// memory; for each lower neighbour k in column order the multiplier l_ik = a_ik / u_kk is
// formed and the lanes sweep row k's upper entries, each finding its column in row i by
// binary search and applying a_ij -= l_ik * u_kj (separately rounded).  The updates of one
// k are independent, so the factors are bitwise those of the row-serial loop; a row costs
// ~nnz_lower dependent L2 round trips instead of ~nnz^2 (the thread-per-row kernel below
// took 0.6 ms per 35-entry row: with the ~2,300 small levels of a periodic 64^2 x 16
// Galerkin level that is 1.4 s per factorization).  Rows are taken in level order, eight
// per 256-thread batch; kFacMaxRow bounds the shared-memory row.
constexpr int kFacMaxRow = 256;

__global__ void __launch_bounds__(BS) k_ilu0_factor_warp(
    int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, double* fac,
    int64_t* diag, const int32_t* __restrict__ order, int* flag, const int* ep,
    unsigned long long* counter, unsigned long long* bad) {
    __shared__ int32_t scol[BS / 32][kFacMaxRow];
    __shared__ double sval[BS / 32][kFacMaxRow];
    __shared__ long long sbase;
    const int epoch = *((volatile const int*)ep);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t* col = scol[wid];
    double* val = sval[wid];
    for (;;) {
        if (threadIdx.x == 0) sbase = (long long)atomicAdd(counter, (unsigned long long)(BS / 32));
        __syncthreads();
        const int64_t t = sbase + wid;
        __syncthreads();
        if (sbase >= n) return;
        if (t >= n || order[t] < 0) continue;
        const int64_t i = order[t];
        const int64_t a = rp[i];
        const int len = (int)(rp[i + 1] - a);
        for (int l = lane; l < len; l += 32) {
            col[l] = ci[a + l];
            val[l] = fac[a + l];
        }
        __syncwarp();
        // diagonal position and number of lower entries (columns sorted)
        int d = -1, pl = 0;
        for (int l = lane; l < len; l += 32) {
            if (col[l] == i) d = l;
            if (col[l] < i) ++pl;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
            pl += __shfl_xor_sync(0xffffffffu, pl, o);
        }
        // every lower neighbour must be fully factored first
        for (int l = lane; l < pl; l += 32) wait_flag(flag + col[l], epoch);
        __syncwarp();
        unsigned long long mybad = ~0ull;
        for (int pk = 0; pk < pl; ++pk) {
            const int64_t k = col[pk];
            const int64_t dk = ldcg(diag + k);
            const double ukk = ldcg(fac + dk);
            if (ukk == 0.0 && mybad == ~0ull) mybad = (unsigned long long)k;
            const double lik = val[pk] / ukk;
            const int64_t ke = rp[k + 1];
            __syncwarp();
            if (lane == 0) val[pk] = lik;
            for (int64_t p = dk + 1 + lane; p < ke; p += 32) {
                const int32_t cp = ci[p];
                int lo = pk + 1, hi = len;  // first q in (pk, len) with col[q] >= cp
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (col[mid] < cp) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < len && col[lo] == cp) val[lo] = sub(val[lo], mul(lik, ldcg(fac + p)));
            }
            __syncwarp();
        }
        if (mybad == ~0ull && (d < 0 || val[d] == 0.0)) mybad = (unsigned long long)i;
        for (int l = lane; l < len; l += 32) fac[a + l] = val[l];
        if (lane == 0) {
            if (mybad != ~0ull) atomicMin(bad, mybad);
            diag[i] = d < 0 ? a : a + d;  // keep a valid index; error is reported
        }
        __threadfence();
        __syncwarp();
        // st.release orders the row's stores (fenced above) before the flag
        if (lane == 0) st_release(flag + i, epoch);
    }
}

__global__ void k_ilu0_factor(int64_t n, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ ci, double* fac, int64_t* diag,
                              const int32_t* __restrict__ order, int* flag, const int* ep,
                              unsigned long long* counter, unsigned long long* bad) {
    const int epoch = *((volatile const int*)ep);
    for (;;) {
        int64_t base = fetch_batch(counter);
        if (base >= n) return;
        int64_t t = base + threadIdx.x;
        if (t < n && order[t] >= 0) {
            const int64_t i = order[t];
            const int64_t a = rp[i], e = rp[i + 1];
            int64_t d = -1;
            for (int64_t p = a; p < e; ++p)
                if (ci[p] == i) { d = p; break; }
            unsigned long long mybad = ~0ull;
            {  // all lower neighbours must be fully factored first
                int64_t pl = a;
                while (pl < e && ci[pl] < i) ++pl;
                wait_all(flag, ci, a, pl, epoch);
            }
            for (int64_t pk = a; pk < e; ++pk) {
                const int64_t k = ci[pk];
                if (k >= i) break;
                const int64_t dk = ldcg(diag + k);
                const double ukk = ldcg(fac + dk);
                if (ukk == 0.0 && mybad == ~0ull) mybad = (unsigned long long)k;
                const double lik = fac[pk] / ukk;
                fac[pk] = lik;
                const int64_t ke = rp[k + 1];
                int64_t q = pk + 1;
                for (int64_t p = dk + 1; p < ke; ++p) {
                    const int32_t cp = ci[p];
                    while (q < e && ci[q] < cp) ++q;
                    if (q >= e) break;
                    if (ci[q] == cp) fac[q] = sub(fac[q], mul(lik, ldcg(fac + p)));
                }
            }
            if (mybad == ~0ull && (d < 0 || fac[d] == 0.0)) mybad = (unsigned long long)i;
            if (mybad != ~0ull) atomicMin(bad, mybad);
            diag[i] = d < 0 ? a : d;  // keep a valid index; error is reported
            // st.release orders the row's stores before the flag
            st_release(flag + i, epoch);
        }
    }
}

// ------------------------------------------------------------------ ILU(0) triangular solves
// Value-as-flag sync-free sweeps.  Every output word starts as a sentinel NaN
// payload; a row publishes its result with one 64-bit strong store (single-copy
// atomic), and dependants poll the value itself, so readiness and data arrive
// in the same L2 round trip — no per-row flag, no fences.  Each row prefetches
// its factor entries before polling, then accumulates strictly in CSR order
// (linalg.py:104-113), separately rounded.  Each sweep's output is armed with
// the sentinel by one coalesced pass (arm_pending) right before it runs.
__constant__ unsigned int poll_ns_max = 256;  // poll backoff cap (PD_POLL_NS_MAX)

// s -= sum_{p in [p0,p1)} fac[p] * src[col[p]]  (in order), polling unpublished entries
template <int kChunk = 16>
__device__ __forceinline__ double accumulate_polling(double s, const int32_t* __restrict__ ci,
                                                     const double* __restrict__ fac,
                                                     const double* src, int64_t p0, int64_t p1) {
    for (int64_t c0 = p0; c0 < p1; c0 += kChunk) {
        const int cnt = (int)min((int64_t)kChunk, p1 - c0);
        double f[kChunk];
        unsigned long long v[kChunk];
        int32_t col[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (k < cnt) {
                col[k] = ci[c0 + k];
                f[k] = fac[c0 + k];
            }
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (k < cnt) v[k] = ld_strong_u64(src + col[k]);
        unsigned int ns = 32;
        const unsigned int ns_max = poll_ns_max;
        for (;;) {
            bool missing = false;
#pragma unroll
            for (int k = 0; k < kChunk; ++k)
                if (k < cnt && v[k] == kPending) {
                    v[k] = ld_strong_u64(src + col[k]);
                    missing |= (v[k] == kPending);
                }
            if (!missing) break;
            __nanosleep(ns);
            if (ns < ns_max) ns <<= 1;
        }
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (k < cnt) s = sub(s, mul(f[k], __longlong_as_double((long long)v[k])));
    }
    return s;
}

// lower: y_i = b_i - sum_{p < diag} L_p y_col (unit diagonal), linalg.py:104-108
__global__ void k_trsv_lower(int64_t n, const int64_t* __restrict__ lp,
                             const int32_t* __restrict__ lcol, const double* __restrict__ lval,
                             const int32_t* __restrict__ order, const double* __restrict__ b,
                             double* y, unsigned long long* counter, const int* guard,
                             int want) {
    if (guard_off(guard, want)) return;
    for (;;) {
        int64_t base = fetch_batch(counter);
        if (base >= n) return;
        int64_t t = base + threadIdx.x;
        if (t < n && order[t] >= 0) {
            const int64_t i = order[t];
            const double s = accumulate_polling(b[i], lcol, lval, y, lp[t], lp[t + 1]);
            st_strong(y + i, s);
        }
    }
}

// upper: x_i = (y_i - sum_{p > diag} U_p x_col) / U_diag, linalg.py:109-113
__global__ void k_trsv_upper(int64_t n, const int64_t* __restrict__ up,
                             const int32_t* __restrict__ ucol, const double* __restrict__ uval,
                             const double* __restrict__ udiag, const int32_t* __restrict__ order,
                             double* y, double* x, unsigned long long* counter, const int* guard,
                             int want) {
    if (guard_off(guard, want)) return;
    for (;;) {
        int64_t base = fetch_batch(counter);
        if (base >= n) return;
        int64_t t = base + threadIdx.x;
        if (t < n && order[t] >= 0) {
            const int64_t i = order[t];
            const double yi = y[i];
            const double s = accumulate_polling(yi, ucol, uval, x, up[t], up[t + 1]);
            st_strong(x + i, s / udiag[t]);
        }
    }
}

// Level-ordered factor layout: the entries each sweep needs, stored task by
// task in the sweep's level order, so consecutive threads stream consecutive
// memory instead of gathering scattered natural-order CSR rows.
__global__ void k_task_counts(int64_t n, const int64_t* rp, const int64_t* diag,
                              const int32_t* order, int upper, int64_t* cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = order[t];
        if (i < 0) {  // padding task
            cnt[t + 1] = 0;
            continue;
        }
        cnt[t + 1] = upper ? rp[i + 1] - diag[i] - 1 : diag[i] - rp[i];
    }
}

__global__ void k_task_gather(int64_t n, const int64_t* rp, const int32_t* ci, const double* fac,
                              const int64_t* diag, const int32_t* order, int upper,
                              const int64_t* tp, int32_t* tcol, double* tval, double* tdiag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = order[t];
        if (i < 0) {
            if (upper) tdiag[t] = 1.0;
            continue;
        }
        const int64_t d = diag[i];
        const int64_t src = upper ? d + 1 : rp[i];
        const int64_t cnt = tp[t + 1] - tp[t];
        for (int64_t k = 0; k < cnt; ++k) {
            tcol[tp[t] + k] = ci[src + k];
            tval[tp[t] + k] = fac[src + k];
        }
        if (upper) tdiag[t] = fac[d];
    }
}

// Arms a sweep's output words with the pending sentinel: one coalesced pass
// (per-row re-arming stores inside the sweeps cost one scattered L2
// transaction each; this costs ~n*8 bytes of streaming writes).
__global__ void k_arm(double* y, int64_t n, const int* guard, int want) {
    if (guard_off(guard, want)) return;
    unsigned long long* u = reinterpret_cast<unsigned long long*>(y);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if ((reinterpret_cast<uintptr_t>(y) & 15) == 0) {
        ulonglong2* u2 = reinterpret_cast<ulonglong2*>(y);
        for (int64_t k = i; k < n / 2; k += stride) u2[k] = make_ulonglong2(kPending, kPending);
        if (i == 0 && (n & 1)) u[n - 1] = kPending;
    } else {
        for (int64_t k = i; k < n; k += stride) u[k] = kPending;
    }
}

void arm_pending(Ctx& c, double* y, int64_t n, const int* guard, int want) {
    if (n > 0) launch(k_arm, c.grid_for(n / 2 + 1, BS, 4), BS, 0, c.stream, y, n, guard, want);
}

__global__ void k_fill_pending(double* y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<unsigned long long*>(y)[i] = kPending;
}

// Starts one sync-free sweep: bumps the device-resident epoch (so CUDA-graph
// replays never see stale completion flags) and rewinds the task counter.
__global__ void k_begin_sweep(int* ep, unsigned long long* c, const int* guard, int want) {
    if (guard_off(guard, want)) return;
    *c = 0ull;
    *ep = *ep + 1;
}

__global__ void k_level_hist(int64_t n, const int* level, int* hist) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(hist + level[i], 1);
}
__global__ void k_pad_order(int64_t n, const int* level, const int32_t* order, const int64_t* start,
                            const int64_t* pstart, int32_t* padded) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = order[t];
        const int lev = level[i];
        padded[pstart[lev] + (t - start[lev])] = i;
    }
}

// Level order with every level padded to whole warps (-1 = idle lane): the tasks of one
// warp then belong to one level, so no thread waits on a row of its own warp.  With small
// levels (periodic grids: a few dozen rows per level) the unpadded order put several
// levels into one warp and the per-row waits of the factorization and of the
// level-scheduled sweeps ran as chains of divergent spin loops.
static int64_t pad_levels(Ctx& c, const int* level, int64_t n, int nlev, DevBuf<int32_t>& order) {
    DevBuf<int> hist((size_t)nlev);
    PD_CUDA(cudaMemsetAsync(hist.p, 0, (size_t)nlev * sizeof(int), c.stream));
    launch(k_level_hist, c.grid_for(n, BS), BS, 0, c.stream, n, level, hist.p);
    std::vector<int> h((size_t)nlev);
    PD_CUDA(cudaMemcpyAsync(h.data(), hist.p, (size_t)nlev * sizeof(int), cudaMemcpyDeviceToHost,
                            c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int64_t> start((size_t)nlev), pstart((size_t)nlev);
    int64_t a = 0, b = 0;
    for (int l = 0; l < nlev; ++l) {
        start[l] = a;
        pstart[l] = b;
        a += h[l];
        b += ((int64_t)h[l] + 31) & ~(int64_t)31;
    }
    if (b >= INT32_MAX) throw ConfigError("level order too long");
    DevBuf<int64_t> ds((size_t)nlev), dp((size_t)nlev);
    PD_CUDA(cudaMemcpyAsync(ds.p, start.data(), (size_t)nlev * 8, cudaMemcpyHostToDevice, c.stream));
    PD_CUDA(cudaMemcpyAsync(dp.p, pstart.data(), (size_t)nlev * 8, cudaMemcpyHostToDevice, c.stream));
    DevBuf<int32_t> padded((size_t)std::max<int64_t>(b, 1));
    PD_CUDA(cudaMemsetAsync(padded.p, 0xff, (size_t)b * sizeof(int32_t), c.stream));  // -1
    launch(k_pad_order, c.grid_for(n, BS), BS, 0, c.stream, n, level, (const int32_t*)order.p,
           (const int64_t*)ds.p, (const int64_t*)dp.p, padded.p);
    PD_LAUNCH_CHECK();
    PD_CUDA(cudaStreamSynchronize(c.stream));
    order = std::move(padded);
    return b;
}

static void sort_by_level(Ctx& c, int* level, int64_t n, DevBuf<int32_t>& order, int& nlev) {
    DevBuf<int> level_sorted(n);
    DevBuf<int32_t> idx(n);
    order.alloc(n);
    launch(k_iota, c.grid_for(n, BS), BS, 0, c.stream, idx.p, n);
    // number of key bits from the max level
    DevBuf<int> mx(1);
    PD_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), c.stream));
    launch(k_max_int, c.grid_for(n, BS), BS, 0, c.stream, level, n, mx.p);
    int hmax = 0;
    PD_CUDA(cudaMemcpyAsync(&hmax, mx.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    nlev = hmax + 1;
    int bits = 1;
    while ((1 << bits) <= hmax) ++bits;
    size_t tmp_bytes = 0;
    PD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, level, level_sorted.p, idx.p,
                                            order.p, (int64_t)n, 0, bits, c.stream));
    DevBuf<unsigned char> tmp(tmp_bytes);
    PD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, level, level_sorted.p, idx.p,
                                            order.p, (int64_t)n, 0, bits, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
}

std::unique_ptr<Ilu0> ilu0_create(Ctx& c, const Csr& A, int nblocks) {
    if (A.nrows != A.ncols) throw ConfigError("ILU(0) needs a square matrix");
    const int64_t n = A.nrows;
    if (nblocks < 1 || nblocks > std::max<int64_t>(n, 1))
        throw ConfigError("num_blocks must be in [1, " + std::to_string(n) + "], got " +
                          std::to_string(nblocks));
    auto f = std::make_unique<Ilu0>();
    f->n = n;
    f->pattern = &A;
    const int64_t size = n / nblocks;
    for (int b = 0; b < nblocks; ++b)
        f->ranges.emplace_back(b * size, b < nblocks - 1 ? (b + 1) * size : n);
    if (nblocks > 1) {
        f->use_masked = true;
        Csr& M = f->masked;
        M.nrows = M.ncols = n;
        M.rowptr.alloc(n + 1);
        PD_CUDA(cudaMemsetAsync(M.rowptr.p, 0, sizeof(int64_t), c.stream));
        launch(k_mask_count, c.grid_for(n, BS), BS, 0, c.stream, n, A.rowptr.p, A.col.p, size,
                                                             nblocks, M.rowptr.p);
        size_t tb = 0;
        PD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, M.rowptr.p, M.rowptr.p, n + 1,
                                              c.stream));
        DevBuf<unsigned char> tmp(tb);
        PD_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, M.rowptr.p, M.rowptr.p, n + 1,
                                              c.stream));
        PD_CUDA(cudaMemcpyAsync(&M.nnz, M.rowptr.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                c.stream));
        PD_CUDA(cudaStreamSynchronize(c.stream));
        M.col.alloc(std::max<int64_t>(M.nnz, 1));
        M.val.alloc(std::max<int64_t>(M.nnz, 1));
        launch(k_mask_copy, c.grid_for(n, BS), BS, 0, c.stream, n, A.rowptr.p, A.col.p, A.val.p,
                                                            size, nblocks, M.rowptr.p, M.col.p,
                                                            M.val.p);
        PD_LAUNCH_CHECK();
    }
    const Csr& P = f->pat();
    f->fac.alloc(std::max<int64_t>(P.nnz, 1));
    f->diag.alloc(std::max<int64_t>(n, 1));
    f->flag.alloc(std::max<int64_t>(n, 1));
    f->counter.alloc(1);
    f->ep.alloc(1);
    f->scratch.alloc(std::max<int64_t>(n, 1));
    if (n > 0) launch(k_fill_pending, c.grid_for(n, BS), BS, 0, c.stream, f->scratch.p, n);
    PD_CUDA(cudaMemsetAsync(f->flag.p, 0, std::max<int64_t>(n, 1) * sizeof(int), c.stream));
    PD_CUDA(cudaMemsetAsync(f->ep.p, 0, sizeof(int), c.stream));
    if (n > 0) {  // longest row: the warp-per-row factorization keeps a row in shared memory
        DevBuf<int> mx(1);
        PD_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), c.stream));
        launch(k_max_rowlen, c.grid_for(n, BS), BS, 0, c.stream, n, P.rowptr.p, mx.p);
        PD_CUDA(cudaMemcpyAsync(&f->max_row_nnz, mx.p, sizeof(int), cudaMemcpyDeviceToHost,
                                c.stream));
        PD_CUDA(cudaStreamSynchronize(c.stream));
    }
    if (n > 0) {
        DevBuf<int> level(n);
        int g = c.grid_for(n, BS, 8);
        // lower levels
        launch(k_fill_int, c.grid_for(n, BS), BS, 0, c.stream, level.p, n, -1);
        PD_CUDA(cudaMemsetAsync(f->counter.p, 0, sizeof(unsigned long long), c.stream));
        launch(k_levels_lower, g, BS, 0, c.stream, n, P.rowptr.p, P.col.p, level.p, f->counter.p);
        PD_LAUNCH_CHECK();
        sort_by_level(c, level.p, n, f->order_lo, f->nlevels_lo);
        f->nt_lo = pad_levels(c, level.p, n, f->nlevels_lo, f->order_lo);

        launch(k_fill_int, c.grid_for(n, BS), BS, 0, c.stream, level.p, n, -1);
        PD_CUDA(cudaMemsetAsync(f->counter.p, 0, sizeof(unsigned long long), c.stream));
        launch(k_levels_upper, g, BS, 0, c.stream, n, P.rowptr.p, P.col.p, level.p, f->counter.p);
        PD_LAUNCH_CHECK();
        sort_by_level(c, level.p, n, f->order_up, f->nlevels_up);
        f->nt_up = pad_levels(c, level.p, n, f->nlevels_up, f->order_up);

    }
    ilu0_refactor(c, *f);
    return f;
}

static void build_task_layout(Ctx& c, Ilu0& f) {
    const Csr& P = f.pat();
    const int64_t n = f.n;
    for (int upper = 0; upper < 2; ++upper) {
        const int64_t n = upper ? f.nt_up : f.nt_lo;  // tasks (rows + level padding)
        DevBuf<int64_t>& tp = upper ? f.tp_up : f.tp_lo;
        DevBuf<int32_t>& tcol = upper ? f.tcol_up : f.tcol_lo;
        DevBuf<double>& tval = upper ? f.tval_up : f.tval_lo;
        const int32_t* order = upper ? f.order_up.p : f.order_lo.p;
        if (!tp.p) {  // pattern-only part, once per hierarchy
            tp.alloc(n + 1);
            PD_CUDA(cudaMemsetAsync(tp.p, 0, sizeof(int64_t), c.stream));
            launch(k_task_counts, c.grid_for(n, BS), BS, 0, c.stream, n, P.rowptr.p, f.diag.p,
                   order, upper, tp.p);
            size_t tb = 0;
            PD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, tp.p, tp.p, n + 1, c.stream));
            DevBuf<unsigned char> tmp(tb);
            PD_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, tp.p, tp.p, n + 1, c.stream));
            int64_t total = 0;
            PD_CUDA(cudaMemcpyAsync(&total, tp.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                    c.stream));
            PD_CUDA(cudaStreamSynchronize(c.stream));
            tcol.alloc(std::max<int64_t>(total, 1));
            tval.alloc(std::max<int64_t>(total, 1));
            if (upper) f.tdiag.alloc(n);
        }
        launch(k_task_gather, c.grid_for(n, BS), BS, 0, c.stream, n, P.rowptr.p, P.col.p, f.fac.p,
               f.diag.p, order, upper, tp.p, tcol.p, tval.p, upper ? f.tdiag.p : (double*)nullptr);
        PD_LAUNCH_CHECK();
    }
    PD_CUDA(cudaStreamSynchronize(c.stream));
}

void ilu0_refactor(Ctx& c, Ilu0& f) {
    ++c.epoch;
    const Csr& P = f.pat();
    const int64_t n = f.n;
    if (n == 0) return;
    if (f.use_masked) {
        // refresh masked values from the source matrix (pattern unchanged)
        const Csr& A = *f.pattern;
        const int64_t size = n / (int64_t)f.ranges.size();
        launch(k_mask_copy, c.grid_for(n, BS), BS, 0, c.stream, 
            n, A.rowptr.p, A.col.p, A.val.p, size, (int64_t)f.ranges.size(), P.rowptr.p,
            f.masked.col.p, f.masked.val.p);
        PD_LAUNCH_CHECK();
    }
    PD_CUDA(cudaMemcpyAsync(f.fac.p, P.val.p, P.nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                            c.stream));
    DevBuf<unsigned long long> bad(1);
    PD_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), c.stream));
    launch(k_begin_sweep, 1, 1, 0, c.stream, f.ep.p, f.counter.p, nullptr, 0);
    static const bool thread_rows = getenv("PD_ILU_FACTOR_THREAD_ROWS") != nullptr;
    const int64_t ntask = f.nt_lo;  // level order, levels padded to whole warps
    if (f.max_row_nnz > 0 && f.max_row_nnz <= kFacMaxRow && !thread_rows) {
        // a warp per row: eight tasks per batch, resident CTAs stride over the level order
        const int g = (int)std::min<int64_t>((ntask + BS / 32 - 1) / (BS / 32),
                                             (int64_t)c.sms * sweep_blocks_per_sm());
        launch(k_ilu0_factor_warp, g, BS, 0, c.stream, ntask, P.rowptr.p, P.col.p, f.fac.p,
               f.diag.p, (const int32_t*)f.order_lo.p, f.flag.p, f.ep.p, f.counter.p, bad.p);
    } else {
        launch(k_ilu0_factor, c.grid_for(ntask, BS, sweep_blocks_per_sm()), BS, 0, c.stream, ntask,
               P.rowptr.p, P.col.p, f.fac.p, f.diag.p, (const int32_t*)f.order_lo.p, f.flag.p,
               f.ep.p, f.counter.p, bad.p);
    }
    PD_LAUNCH_CHECK();
    unsigned long long hbad = 0;
    PD_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(hbad), cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    if (hbad != ~0ull) {
        int64_t row = (int64_t)hbad;
        if (f.use_masked) {  // report the row relative to its block (per-block Ilu0)
            for (auto& r : f.ranges)
                if (row >= r.first && row < r.second) { row -= r.first; break; }
        }
        throw SolverError("zero pivot in ILU(0) at row " + std::to_string(row), row);
    }
    build_task_layout(c, f);
    wf_gather(c, f);
    wf2_gather(c, f);
}

static void configure_polling_once() {
    static bool done = false;
    if (done) return;
    done = true;
    if (const char* e = getenv("PD_POLL_NS_MAX")) {
        unsigned int v = (unsigned int)atoi(e);
        if (v >= 32) PD_CUDA(cudaMemcpyToSymbol(poll_ns_max, &v, sizeof(v)));
    }
}

void ilu0_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard, int want) {
    configure_polling_once();
    const int64_t n = f.n;
    if (n == 0) return;
    if (b == x) throw ConfigError("ILU(0) solve needs distinct input and output buffers");
    if (f.w2_lo) {
        wf2_solve(c, f, b, x, guard, want);
        return;
    }
    if (f.w2_up && f.wf_lo) {  // pattern-table lower sweep + template upper sweep
        wf_solve_lower(c, f, b, guard, want);
        wf2_solve_upper(c, f, x, guard, want);
        return;
    }
    if (f.wf_lo) {
        wf_solve(c, f, b, x, guard, want);
        return;
    }
    // tasks = rows in level order, levels padded to whole warps (nt_lo / nt_up)
    arm_pending(c, f.scratch.p, n, guard, want);
    launch(k_begin_sweep, 1, 1, 0, c.stream, f.ep.p, f.counter.p, guard, want);
    launch(k_trsv_lower, c.grid_for(f.nt_lo, BS, sweep_blocks_per_sm()), BS, 0, c.stream, f.nt_lo,
           f.tp_lo.p, f.tcol_lo.p, f.tval_lo.p, f.order_lo.p, b, f.scratch.p, f.counter.p, guard,
           want);
    arm_pending(c, x, n, guard, want);
    launch(k_begin_sweep, 1, 1, 0, c.stream, f.ep.p, f.counter.p, guard, want);
    launch(k_trsv_upper, c.grid_for(f.nt_up, BS, sweep_blocks_per_sm()), BS, 0, c.stream, f.nt_up,
           f.tp_up.p, f.tcol_up.p, f.tval_up.p, f.tdiag.p, f.order_up.p, f.scratch.p, x,
           f.counter.p, guard, want);
    PD_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ dense LU (coarsest level)
__global__ void k_csr_to_dense_colmajor(int64_t n, const int64_t* rp, const int32_t* ci,
                                        const double* v, double* A) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) A[i + (int64_t)ci[p] * n] += v[p];
}

// Blocked right-looking LU with partial pivoting (dgetrf structure, panels of kLuNB
// columns): three launches per panel instead of two per column.  Every entry still
// receives its rank-1 updates one pivot column at a time, in pivot order, as
// a = fma(-l_ik, u_kj, a) — the operation sequence of the unblocked dgetf2 loop — so
// the factors are bitwise those of the column-by-column elimination.
constexpr int kLuNB = 32;

// Panel [k0, k0+nb): per column the pivot search (first max |a_ik|, like idamax), the
// interchange inside the panel, the column scaling by the reciprocal pivot and the
// rank-1 update of the panel's remaining columns.  One CTA.
__global__ void __launch_bounds__(1024) k_lu_panel(double* A, int64_t n, int64_t k0, int nb,
                                                   int32_t* piv, int* info) {
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    __shared__ double urow[kLuNB];
    __shared__ int64_t sp;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int c = 0; c < nb; ++c) {
        const int64_t k = k0 + c;
        double best = -1.0;
        int64_t bi = k;
        for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
            const double a = fabs(A[i + k * n]);
            if (a > best) { best = a; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_down_sync(0xffffffffu, best, o);
            const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) { sv[wid] = best; si[wid] = bi; }
        __syncthreads();
        if (wid == 0) {
            best = sv[lane];
            bi = si[lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, best, o);
                const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (lane == 0) { sp = bi; piv[k] = (int32_t)bi; }
        }
        __syncthreads();
        const int64_t p = sp;
        // interchange rows k and p inside the panel; keep the pivot row's tail
        if (threadIdx.x < nb) {
            const int64_t j = k0 + threadIdx.x;
            const double t = A[p + j * n];
            if (p != k) {
                A[p + j * n] = A[k + j * n];
                A[k + j * n] = t;
            }
            urow[threadIdx.x] = t;
        }
        __syncthreads();
        const double akk = urow[c];
        if (akk == 0.0) {
            if (threadIdx.x == 0 && *info == 0) *info = (int)(k + 1);
            continue;  // dgetf2 skips the elimination of a zero pivot column
        }
        const double r = 1.0 / akk;
        for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
            const double l = A[i + k * n] * r;
            A[i + k * n] = l;
            for (int cc = c + 1; cc < nb; ++cc) {
                double* a = A + i + (k0 + cc) * n;
                *a = fma(-l, urow[cc], *a);
            }
        }
        __syncthreads();
    }
}

// Columns outside the panel, one thread each: the panel's row interchanges, and for
// columns to its right the unit-lower solve U12 = L11^{-1} A12 (row k of the block
// after rows k' < k, i.e. the rank-1 order).
__global__ void k_lu_cols(double* A, int64_t n, int64_t k0, int nb, const int32_t* piv) {
    __shared__ double L11[kLuNB * kLuNB];
    __shared__ int32_t sp[kLuNB];
    for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
        const int i = t % nb, k = t / nb;
        L11[i * kLuNB + k] = A[(k0 + i) + (k0 + k) * n];
    }
    if (threadIdx.x < nb) sp[threadIdx.x] = piv[k0 + threadIdx.x];
    __syncthreads();
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n - nb) return;
    if (j >= k0) j += nb;
    double* col = A + j * n;
    for (int c = 0; c < nb; ++c) {
        const int64_t p = sp[c];
        if (p != k0 + c) {
            const double t = col[k0 + c];
            col[k0 + c] = col[p];
            col[p] = t;
        }
    }
    if (j < k0) return;
    double u[kLuNB];
#pragma unroll
    for (int i = 0; i < kLuNB; ++i) u[i] = i < nb ? col[k0 + i] : 0.0;
#pragma unroll
    for (int k = 0; k < kLuNB; ++k)
#pragma unroll
        for (int i = k + 1; i < kLuNB; ++i)
            if (i < nb) u[i] = fma(-L11[i * kLuNB + k], u[k], u[i]);
#pragma unroll
    for (int i = 0; i < kLuNB; ++i)
        if (i < nb) col[k0 + i] = u[i];
}

// Trailing update A22 -= L21 U12: 64 x 64 tiles, 4 x 4 per thread, k in pivot order.
__global__ void __launch_bounds__(256) k_lu_trailing(double* A, int64_t n, int64_t k0, int nb) {
    __shared__ double Ls[kLuNB][64];
    __shared__ double Us[kLuNB][65];
    const int64_t r0 = k0 + nb + (int64_t)blockIdx.x * 64, c0 = k0 + nb + (int64_t)blockIdx.y * 64;
    for (int t = threadIdx.x; t < nb * 64; t += 256) {
        const int i = t & 63, k = t >> 6;
        Ls[k][i] = r0 + i < n ? A[(r0 + i) + (k0 + k) * n] : 0.0;
    }
    for (int t = threadIdx.x; t < nb * 64; t += 256) {
        const int k = t % nb, j = t / nb;
        Us[k][j] = c0 + j < n ? A[(k0 + k) + (c0 + j) * n] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i = r0 + tx + 16 * r, j = c0 + ty + 16 * s;
            acc[s][r] = (i < n && j < n) ? A[i + j * n] : 0.0;
        }
    for (int k = 0; k < nb; ++k) {
        double l[4], u[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) l[r] = Ls[k][tx + 16 * r];
#pragma unroll
        for (int s = 0; s < 4; ++s) u[s] = Us[k][ty + 16 * s];
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[s][r] = fma(-l[r], u[s], acc[s][r]);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i = r0 + tx + 16 * r, j = c0 + ty + 16 * s;
            if (i < n && j < n) A[i + j * n] = acc[s][r];
        }
}

std::unique_ptr<DenseLU> dense_lu_from_csr(Ctx& c, const Csr& A) {
    if (A.nrows != A.ncols) throw ConfigError("dense LU needs a square matrix");
    const int64_t n = A.nrows;
    if (n > 29000) throw ConfigError("coarsest level too large for dense LU: n=" + std::to_string(n));
    auto f = std::make_unique<DenseLU>();
    f->n = n;
    f->lu.alloc(std::max<int64_t>(n * n, 1));
    f->piv.alloc(std::max<int64_t>(n, 1));
    PD_CUDA(cudaMemsetAsync(f->lu.p, 0, n * n * sizeof(double), c.stream));
    launch(k_csr_to_dense_colmajor, c.grid_for(n, BS), BS, 0, c.stream, n, A.rowptr.p, A.col.p,
                                                                    A.val.p, f->lu.p);
    DevBuf<int> info(1);
    PD_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), c.stream));
    for (int64_t k0 = 0; k0 < n; k0 += kLuNB) {
        const int nb = (int)std::min<int64_t>(kLuNB, n - k0);
        launch(k_lu_panel, 1, 1024, 0, c.stream, f->lu.p, n, k0, nb, f->piv.p, info.p);
        if (n > nb)
            launch(k_lu_cols, (int)((n - nb + 127) / 128), 128, 0, c.stream, f->lu.p, n, k0, nb,
                   (const int32_t*)f->piv.p);
        const int64_t m = n - k0 - nb;
        if (m > 0) {
            const unsigned t = (unsigned)((m + 63) / 64);
            launch(k_lu_trailing, dim3(t, t), 256, 0, c.stream, f->lu.p, n, k0, nb);
        }
    }
    PD_LAUNCH_CHECK();
    PD_CUDA(cudaStreamSynchronize(c.stream));
    // A singular coarse matrix is not an exception in the reference either
    // (LAPACK getrf info>0 only warns); the solve then yields non-finite values
    // and the V-cycle raises SolverError (multigrid.py:270-271).
    return f;
}

// Single-CTA substitution: LAPACK getrs order (row interchanges, unit-lower
// column sweep, upper column sweep).  The vector lives in shared memory.
__global__ void k_lu_solve(const double* __restrict__ LU, const int32_t* __restrict__ piv,
                           int64_t n, const double* __restrict__ b, double* __restrict__ xout) {
    extern __shared__ double xs[];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) xs[i] = b[i];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = piv[i];
            if (p != i) { double t = xs[i]; xs[i] = xs[p]; xs[p] = t; }
        }
    __syncthreads();
    for (int64_t k = 0; k < n; ++k) {
        const double xk = xs[k];
        for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x)
            xs[i] -= LU[i + k * n] * xk;
        __syncthreads();
    }
    for (int64_t k = n - 1; k >= 0; --k) {
        if (threadIdx.x == 0) xs[k] = xs[k] / LU[k + k * n];
        __syncthreads();
        const double xk = xs[k];
        for (int64_t i = threadIdx.x; i < k; i += blockDim.x) xs[i] -= LU[i + k * n] * xk;
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) xout[i] = xs[i];
}

void dense_lu_solve(Ctx& c, const DenseLU& f, const double* b, double* x) {
    const int64_t n = f.n;
    if (n == 0) return;
    size_t sm = n * sizeof(double);
    // per-device attribute (and cheap): set before every launch that needs it
    if (sm > 48 * 1024)
        PD_CUDA(cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024));
    if (sm > 227 * 1024) throw ConfigError("coarsest level too large for the dense solve");
    launch(k_lu_solve, 1, 1024, sm, c.stream, f.lu.p, f.piv.p, n, b, x);
    PD_LAUNCH_CHECK();
}

}  // namespace pd

namespace pd {
// ------------------------------------------------------------------ coarsest-level inverse
// The V-cycle's coarsest solve (multigrid.py:259-260) runs once per cycle on
// the same matrix, so the hierarchy forms A_c^{-1} from the device LU factors
// at setup (n_c RHS solves, one CTA each) and applies it as one GEMV per
// cycle: n_c^2 * 8 bytes streamed at HBM/L2 rate instead of 2*n_c dependent
// substitution steps on one SM.
__global__ void k_lu_inverse_cols(const double* __restrict__ LU, const int32_t* __restrict__ piv,
                                  int64_t n, double* inv_rowmajor) {
    extern __shared__ double xs[];
    const int64_t j = blockIdx.x;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) xs[i] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = piv[i];
            if (p != i) { double t = xs[i]; xs[i] = xs[p]; xs[p] = t; }
        }
    __syncthreads();
    for (int64_t k = 0; k < n; ++k) {
        const double xk = xs[k];
        for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x) xs[i] -= LU[i + k * n] * xk;
        __syncthreads();
    }
    for (int64_t k = n - 1; k >= 0; --k) {
        if (threadIdx.x == 0) xs[k] = xs[k] / LU[k + k * n];
        __syncthreads();
        const double xk = xs[k];
        for (int64_t i = threadIdx.x; i < k; i += blockDim.x) xs[i] -= LU[i + k * n] * xk;
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) inv_rowmajor[i * n + j] = xs[i];
}

// x = Ainv b, one warp per row, fixed lane-strided order + shuffle tree (deterministic)
__global__ void k_gemv_rows(const double* __restrict__ A, const double* __restrict__ b,
                            double* __restrict__ x, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nw) {
        const double* row = A + i * n;
        double s = 0.0;
        for (int64_t k = lane; k < n; k += 32) s = fma(row[k], __ldg(b + k), s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) x[i] = s;
    }
}

DevBuf<double> dense_inverse(Ctx& c, const DenseLU& f) {
    const int64_t n = f.n;
    DevBuf<double> inv(std::max<int64_t>(n * n, 1));
    if (n == 0) return inv;
    if (n * sizeof(double) > 48 * 1024)  // per-device attribute: set whenever it is needed
        PD_CUDA(cudaFuncSetAttribute(k_lu_inverse_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024));
    launch(k_lu_inverse_cols, (unsigned)n, 256, n * sizeof(double), c.stream, f.lu.p, f.piv.p, n,
           inv.p);
    PD_LAUNCH_CHECK();
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return inv;
}

void dense_inverse_apply(Ctx& c, const double* inv, int64_t n, const double* b, double* x) {
    if (n == 0) return;
    launch(k_gemv_rows, c.grid_for(n * 32, 256, 8), 256, 0, c.stream, inv, b, x, n);
}
}  // namespace pd

namespace pd {
// ------------------------------------------------------------------ fixed-pattern SpGEMM
// C = A B (values only) on a pattern fixed at setup, accumulating every entry
// in scipy csr_matmat's order: rows of A in stored order, rows of B in stored
// order, sums[k] += a*b separately rounded (sparsetools csr.h).  With A = R
// and B = A_l, then A = (R A_l) in its stored (scipy first-touch) order and
// B = P, the coarse operator equals the reference's `R @ A @ P` bitwise
// (multigrid.py:232-233).  One thread per row of C; C rows hold <= a few
// hundred entries, located by linear scan of the row's stored columns.
__global__ void k_spgemm_values(int64_t nrows, const int64_t* __restrict__ arp,
                                const int32_t* __restrict__ aci, const double* __restrict__ av,
                                const int64_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                const double* __restrict__ bv, const int64_t* __restrict__ crp,
                                const int32_t* __restrict__ cci, double* __restrict__ cv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c0 = crp[i], c1 = crp[i + 1];
        for (int64_t q = c0; q < c1; ++q) cv[q] = 0.0;
        for (int64_t jj = arp[i]; jj < arp[i + 1]; ++jj) {
            const int64_t j = aci[jj];
            const double v = av[jj];
            for (int64_t kk = brp[j]; kk < brp[j + 1]; ++kk) {
                const int32_t k = bci[kk];
                int64_t q = c0;
                while (q < c1 && cci[q] != k) ++q;
                if (q < c1) cv[q] = add(cv[q], mul(v, bv[kk]));
            }
        }
    }
}

void spgemm_values(Ctx& c, const Csr& A, const Csr& B, Csr& C) {
    ++c.epoch;
    if (A.nrows != C.nrows || A.ncols != B.nrows || B.ncols != C.ncols)
        throw ConfigError("fixed-pattern SpGEMM shape mismatch");
    if (C.nrows == 0) return;
    launch(k_spgemm_values, c.grid_for(C.nrows, BS, 8), BS, 0, c.stream, C.nrows, A.rowptr.p,
           A.col.p, A.val.p, B.rowptr.p, B.col.p, B.val.p, C.rowptr.p, C.col.p, C.val.p);
    PD_LAUNCH_CHECK();
    C.values_changed();
}

// ------------------------------------------------------------------ Newton Jacobian values
// J = L + gamma (I (x) Mqh) diag(r'(u)) on L's pattern (spacetime.py:144-151):
// for an entry of row (n,m,j) at column (n,m',j): Jv = fl(Lv + fl(gamma*fl(Mqh*r'(u_col))))
// with Mqh = fl(dt*fl(Mq[m][m']*mh_j)); every other entry is L's value.
__global__ void k_jacobian_values(int64_t N, int M, int64_t S, double dt, double gamma, int kind,
                                  const double* __restrict__ Mq, const double* __restrict__ mh,
                                  const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ lv, const double* __restrict__ u,
                                  double* __restrict__ jv) {
    const int64_t MS = (int64_t)M * S;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = r / MS, rem = r - n * MS;
        const int m = (int)(rem / S);
        const int64_t j = rem - (int64_t)m * S;
        for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
            const int64_t col = ci[p];
            double val = lv[p];
            const int64_t nc = col / MS, remc = col - nc * MS;
            const int mc = (int)(remc / S);
            if (nc == n && remc - (int64_t)mc * S == j) {
                const double u0 = u[col];
                const double g = kind == 1 ? sub(mul(3.0, mul(u0, u0)), 1.0) : sub(mul(2.0, u0), 1.0);
                const double mqh = mul(dt, mul(Mq[m * M + mc], mh[j]));
                val = add(val, mul(gamma, mul(mqh, g)));
            }
            jv[p] = val;
        }
    }
}

void jacobian_values(Ctx& c, int64_t Nt, int M, int64_t S, double dt, double gamma, int kind,
                     const double* Mq_dev, const double* mh_dev, const Csr& L, const double* u,
                     double* jv) {
    const int64_t N = Nt * M * S;
    if (L.nrows != N) throw ConfigError("Jacobian pattern does not match the space-time grid");
    launch(k_jacobian_values, c.grid_for(N, BS, 8), BS, 0, c.stream, N, M, S, dt, gamma, kind,
           Mq_dev, mh_dev, L.rowptr.p, L.col.p, L.val.p, u, jv);
    PD_LAUNCH_CHECK();
}
}  // namespace pd
