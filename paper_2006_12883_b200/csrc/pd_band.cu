// Banded LU with partial pivoting on the device: the direct solves of
// paradiff/spacetime.py:154-195 (`_element_solve`, `solve_sequential`, `solve_direct`
// call SuperLU there).  The element system Aqh and the global system are banded once
// their unknowns are ordered point-major (host permutation, passed in): half
// bandwidth M * bw(Kh) + M - 1 for an element, M * S + M for the global matrix.
//
// Storage: LAPACK general-band layout with room for the pivoting fill,
//   a(i, j) = ab[(kl + ku + i - j) + j * ld],  ld = 2 kl + ku + 1,
// so a column is contiguous.  Factorization (dgbtf2 semantics: the multipliers of a
// column stay where they were computed; later interchanges are not applied to them,
// the solve interleaves interchanges and eliminations) in panels of kBandNB columns:
//   k_band_panel  one CTA: per column pivot search, interchange, scaling, rank-1
//                 update of the panel's remaining columns;
//   k_band_cols   one warp per column right of the panel (up to kl + ku of them):
//                 replays the panel's interchanges and eliminations on its column held
//                 in shared memory (multiplier columns read coalesced);
// i.e. two launches per 32 columns.  Solve: one CTA per right-hand side, the active
// window of the vector in a shared-memory ring, one barrier per column.
#include <cuda_runtime.h>

#include <algorithm>

#include "pd_internal.h"

namespace pd {

namespace {

constexpr int kBandNB = 32;

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__global__ void k_csr_to_band(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                              double* ab, int kl, int ku, int64_t ld) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int64_t j = ci[p];
            ab[(kl + ku + i - j) + j * ld] += v[p];
        }
}

__global__ void __launch_bounds__(1024) k_band_panel(double* ab, int64_t n, int kl, int ku,
                                                     int64_t ld, int64_t k0, int nb, int32_t* piv,
                                                     int* info) {
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    __shared__ double urow[kBandNB];
    __shared__ int64_t sp;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int kd = kl + ku;  // row offset of the diagonal inside a stored column
    for (int c = 0; c < nb; ++c) {
        const int64_t k = k0 + c;
        const int64_t km = imin64(kl, n - 1 - k);
        double* colk = ab + k * ld + kd;  // colk[i - k] = a(i, k)
        double best = -1.0;
        int64_t bi = k;
        for (int64_t i = k + threadIdx.x; i <= k + km; i += blockDim.x) {
            const double a = fabs(colk[i - k]);
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
        // columns of the panel still inside row k's band: k .. jmax
        const int64_t jmax = imin64(imin64(k0 + nb - 1, k + kd), n - 1);
        if (threadIdx.x < nb) {
            const int64_t j = k0 + threadIdx.x;
            double t = 0.0;
            if (j >= k && j <= jmax) {
                double* cj = ab + j * ld + kd;  // cj[i - j] = a(i, j)
                t = cj[p - j];
                if (p != k) {
                    cj[p - j] = cj[k - j];
                    cj[k - j] = t;
                }
            }
            urow[threadIdx.x] = t;
        }
        __syncthreads();
        const double akk = urow[c];
        if (akk == 0.0) {
            if (threadIdx.x == 0 && *info == 0) *info = (int)imin64(k + 1, 2147483647);
            continue;
        }
        const double r = 1.0 / akk;
        const int ncol = (int)(jmax - k);  // panel columns right of k
        for (int64_t i = k + 1 + threadIdx.x; i <= k + km; i += blockDim.x) {
            const double l = colk[i - k] * r;
            colk[i - k] = l;
            for (int cc = 1; cc <= ncol; ++cc) {
                double* a = ab + (k + cc) * ld + kd + (i - (k + cc));
                *a = fma(-l, urow[c + cc], *a);
            }
        }
        __syncthreads();
    }
}

// One warp per column j right of the panel; w = rows k0 .. k0 + nb - 1 + kl of column j.
__global__ void k_band_cols(double* ab, int64_t n, int kl, int ku, int64_t ld, int64_t k0, int nb,
                            const int32_t* piv, int64_t ncols) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t jc = blockIdx.x * (int64_t)nw + wid;
    if (jc >= ncols) return;
    const int64_t j = k0 + nb + jc;
    const int kd = kl + ku;
    const int wlen = nb + kl;
    double* w = smem + (size_t)wid * wlen;
    double* cj = ab + j * ld + kd;  // cj[i - j] = a(i, j), valid for j - kd <= i <= j + kl
    const int64_t ilo = j - kd, ihi = imin64(n - 1, k0 + nb - 1 + kl);
    for (int t = lane; t < wlen; t += 32) {
        const int64_t i = k0 + t;
        w[t] = (i >= ilo && i <= ihi) ? cj[i - j] : 0.0;
    }
    __syncwarp();
    for (int c = 0; c < nb; ++c) {
        const int64_t k = k0 + c;
        if (j > k + kd) continue;  // column j lies outside pivot row k's band
        const int64_t km = imin64(kl, n - 1 - k);
        const int p = (int)(piv[k] - k0);
        double uk = w[p];
        __syncwarp();
        if (lane == 0 && p != c) {
            w[p] = w[c];
            w[c] = uk;
        }
        __syncwarp();
        if (uk != 0.0) {
            const double* lk = ab + k * ld + kd;  // lk[i - k] = l(i, k)
            for (int64_t d = 1 + lane; d <= km; d += 32) w[c + d] = fma(-lk[d], uk, w[c + d]);
        }
        __syncwarp();
    }
    for (int t = lane; t < wlen; t += 32) {
        const int64_t i = k0 + t;
        if (i >= ilo && i <= ihi) cj[i - j] = w[t];
    }
}

// x = A^{-1} b for one right-hand side per CTA.  perm (may be null): band row i is the
// caller's unknown perm[i].  Ring of R (power of two > max(kl, kl + ku)) doubles.
__global__ void __launch_bounds__(1024) k_band_solve(const double* __restrict__ ab,
                                                     const int32_t* __restrict__ piv, int64_t n,
                                                     int kl, int ku, int64_t ld, int R,
                                                     const int32_t* __restrict__ perm,
                                                     const double* b, double* x, int64_t stride) {
    extern __shared__ double ring[];
    b += blockIdx.x * stride;
    x += blockIdx.x * stride;
    const int kd = kl + ku, mask = R - 1;
    // forward: L (interchanges interleaved).  The ring holds rows j .. j + kl.
    for (int64_t i = threadIdx.x; i <= imin64(kl, n - 1); i += blockDim.x)
        ring[i & mask] = b[perm ? perm[i] : i];
    __syncthreads();
    for (int64_t j = 0; j < n; ++j) {
        const int64_t km = imin64(kl, n - 1 - j);
        const int64_t p = piv[j];
        const double xp = ring[p & mask], xj = ring[j & mask];
        const double* lj = ab + j * ld + kd;
        double upd[2];  // up to 2 rows per thread per column (kl <= 2 * blockDim)
        int cnt = 0;
        for (int64_t d = 1 + threadIdx.x; d <= km; d += blockDim.x) {
            const int64_t i = j + d;
            const double v = (i == p) ? xj : ring[i & mask];
            const double r = fma(-lj[d], xp, v);
            if (cnt < 2) upd[cnt] = r;
            ++cnt;
        }
        __syncthreads();  // every read of the ring's old values is done
        cnt = 0;
        for (int64_t d = 1 + threadIdx.x; d <= km; d += blockDim.x) {
            if (cnt < 2) ring[(j + d) & mask] = upd[cnt];
            ++cnt;
        }
        if (threadIdx.x == 0) {
            x[j] = xp;  // y_j (band order, scratch use of x)
            const int64_t in = j + kl + 1;
            if (in < n) ring[in & mask] = b[perm ? perm[in] : in];
        }
        __syncthreads();
    }
    // backward: U has kd super-diagonals.  The ring holds rows j - kd .. j.
    for (int64_t i = threadIdx.x; i <= imin64(kd, n - 1); i += blockDim.x)
        ring[(n - 1 - i) & mask] = x[n - 1 - i];
    __syncthreads();
    for (int64_t j = n - 1; j >= 0; --j) {
        const double* uj = ab + j * ld + kd;  // uj[i - j], i <= j
        const double xj = ring[j & mask] / uj[0];
        const int64_t km = imin64(kd, j);
        double upd[4];
        int cnt = 0;
        for (int64_t d = 1 + threadIdx.x; d <= km; d += blockDim.x) {
            const double r = fma(-uj[-d], xj, ring[(j - d) & mask]);
            if (cnt < 4) upd[cnt] = r;
            ++cnt;
        }
        __syncthreads();
        cnt = 0;
        for (int64_t d = 1 + threadIdx.x; d <= km; d += blockDim.x) {
            if (cnt < 4) ring[(j - d) & mask] = upd[cnt];
            ++cnt;
        }
        if (threadIdx.x == 0) {
            ring[j & mask] = xj;
            const int64_t in = j - kd - 1;
            if (in >= 0) ring[in & mask] = x[in];
        }
        __syncthreads();
        // x_j is final; it leaves through the ring slot read below (kept until reused)
        if (threadIdx.x == 0) x[j] = xj;
    }
}

// out[perm[i]] = y[i] (the solve works in band order in a scratch vector)
__global__ void k_band_unpermute(const double* y, const int32_t* perm, double* out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[perm[i]] = y[i];
}

}  // namespace

struct BandLU {
    int64_t n = 0, ld = 0;
    int kl = 0, ku = 0, R = 0;
    DevBuf<double> ab, work;
    DevBuf<int32_t> piv, perm;
    bool has_perm = false;
};

BandLU* band_lu_create(Ctx& c, const Csr& A, int kl, int ku, const int32_t* perm_host) {
    if (A.nrows != A.ncols) throw ConfigError("banded LU needs a square matrix");
    if (kl < 0 || ku < 0) throw ConfigError("bandwidths must be nonnegative");
    const int64_t n = A.nrows;
    auto f = std::make_unique<BandLU>();
    f->n = n;
    f->kl = kl;
    f->ku = ku;
    f->ld = 2 * (int64_t)kl + ku + 1;
    const int kd = kl + ku;
    if (kl > 2 * 1024 || kd > 4 * 1024)
        throw ConfigError("band too wide for the device solve: kl=" + std::to_string(kl) +
                          " ku=" + std::to_string(ku));
    int R = 1;
    while (R <= std::max(kl, kd) + 1) R <<= 1;
    f->R = R;
    const double gb = (double)f->ld * (double)n * 8.0 / 1e9;
    if (gb > 64.0) throw ConfigError("band storage would need " + std::to_string(gb) + " GB");
    f->ab.alloc(std::max<int64_t>(f->ld * n, 1));
    f->piv.alloc(std::max<int64_t>(n, 1));
    f->work.alloc(std::max<int64_t>(n, 1));
    if (perm_host) {
        f->perm.alloc(std::max<int64_t>(n, 1));
        PD_CUDA(cudaMemcpyAsync(f->perm.p, perm_host, n * sizeof(int32_t), cudaMemcpyHostToDevice,
                                c.stream));
        f->has_perm = true;
    }
    if (n == 0) return f.release();
    PD_CUDA(cudaMemsetAsync(f->ab.p, 0, f->ld * n * sizeof(double), c.stream));
    launch(k_csr_to_band, c.grid_for(n, 256), 256, 0, c.stream, n, A.rowptr.p, A.col.p, A.val.p,
           f->ab.p, kl, ku, f->ld);
    DevBuf<int> info(1);
    PD_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), c.stream));
    const int wlen = kBandNB + kl;
    int nw = (int)std::min<size_t>(8, (200 * 1024) / (wlen * sizeof(double)));
    nw = std::max(nw, 1);
    const size_t smem = (size_t)nw * wlen * sizeof(double);
    if (smem > 48 * 1024)
        PD_CUDA(cudaFuncSetAttribute(k_band_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024));
    for (int64_t k0 = 0; k0 < n; k0 += kBandNB) {
        const int nb = (int)std::min<int64_t>(kBandNB, n - k0);
        launch(k_band_panel, 1, 1024, 0, c.stream, f->ab.p, n, kl, ku, f->ld, k0, nb, f->piv.p,
               info.p);
        const int64_t ncols = std::min<int64_t>(n, k0 + nb + kd) - (k0 + nb);
        if (ncols > 0)
            launch(k_band_cols, (unsigned)((ncols + nw - 1) / nw), nw * 32, smem, c.stream, f->ab.p,
                   n, kl, ku, f->ld, k0, nb, (const int32_t*)f->piv.p, ncols);
    }
    PD_LAUNCH_CHECK();
    int h = 0;
    PD_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    // SuperLU raises "Factor is exactly singular" (spacetime.py:154-195 lets it propagate)
    if (h != 0) throw SolverError("banded LU: matrix is exactly singular", h - 1);
    return f.release();
}

void band_lu_solve(Ctx& c, BandLU& f, const double* b, double* x) {
    const int64_t n = f.n;
    if (n == 0) return;
    if (b == x && f.has_perm) throw ConfigError("permuted banded solve needs distinct buffers");
    const size_t smem = (size_t)f.R * sizeof(double);
    if (smem > 48 * 1024)
        PD_CUDA(cudaFuncSetAttribute(k_band_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024));
    double* y = f.has_perm ? f.work.p : x;
    launch(k_band_solve, 1, 1024, smem, c.stream, (const double*)f.ab.p, (const int32_t*)f.piv.p, n,
           f.kl, f.ku, f.ld, f.R, f.has_perm ? (const int32_t*)f.perm.p : nullptr, b, y,
           (int64_t)0);
    if (f.has_perm)
        launch(k_band_unpermute, c.grid_for(n, 256), 256, 0, c.stream, (const double*)y,
               (const int32_t*)f.perm.p, x, n);
    PD_LAUNCH_CHECK();
}

void band_lu_destroy(BandLU* f) { delete f; }

}  // namespace pd
