// Structured SpMV for Galerkin space-time operators on 2D grids.
//
// The SMG coarse operators R A P (multigrid.py:224-241) of a 2D FD space-time
// system keep a fixed shape: row (step, m, y, x) couples to the previous step's
// last node and to every node m' of its own step, each through the 3x3
// neighbourhood of (y, x) (boundary rows simply lack the outside neighbours).
// When a CSR has exactly that pattern (checked entry by entry on the host) its
// values are re-laid out as [position k][row] (coalesced across a warp, no
// column indices: 8 instead of 12 bytes per entry) and the product walks the
// positions in the CSR's column order, so every row's sum is bitwise the CSR
// SpMV's.  The copy is refreshed lazily whenever the CSR's values change
// (csr_update_values, spgemm_values, Multigrid::set_fine_values mark it stale).
#include <cuda_runtime.h>

#include <vector>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pd {
using namespace dev;

struct GridSpmv {
    int64_t nt = 0, N = 0;
    int M = 0, n = 0, K = 0;
    DevBuf<double> vals;  // [K][N]
};

namespace {
constexpr int GB = 256;  // 32 x 8 threads

// the row's positions in column order: block 0 = previous step's last node,
// block 1 + m' = node m' of the own step; 3x3 (dy, dx) lexicographic inside
__device__ __forceinline__ bool present(int blk, int step, int y, int x, int dy, int dx, int n) {
    return (blk > 0 || step > 0) && y + dy >= 0 && y + dy < n && x + dx >= 0 && x + dx < n;
}

__global__ void k_gspmv_gather(int64_t N, int M, int n, const int64_t* __restrict__ rp,
                               const double* __restrict__ v, double* vals) {
    const int64_t S = (int64_t)n * n;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t plane = r / S, j = r - plane * S;
        const int step = (int)(plane / M), y = (int)(j / n), x = (int)(j - (int64_t)y * n);
        int64_t p = rp[r];
        int k = 0;
        for (int blk = 0; blk <= M; ++blk)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx, ++k)
                    vals[(int64_t)k * N + r] = present(blk, step, y, x, dy, dx, n) ? v[p++] : 0.0;
    }
}

template <int M, bool REDUCE>
__global__ void __launch_bounds__(GB, 5) k_gspmv(int64_t nt, int n, int gy, int64_t N,
                                              const double* __restrict__ vals,
                                              const double* __restrict__ xv, double* y, int mode,
                                              const double* b, const int* guard, int want,
                                              double* partials, unsigned int* counter,
                                              double* norm2, int* nonfinite) {
    if (guard_off(guard, want)) return;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int xi = blockIdx.x * 32 + threadIdx.x, yi = blockIdx.y * 8 + threadIdx.y;
    const bool inside = xi < n && yi < n;
    const int64_t S = (int64_t)n * n;
    const int j = yi * n + xi;
    double acc2 = 0.0;
    bool bad = false;
    for (int64_t plane = blockIdx.z; inside && plane < nt * M; plane += gridDim.z) {
        const int step = (int)(plane / M);
        const int64_t r = plane * S + j;
        const double* vr = vals + r;
        double s = 0.0;
#pragma unroll
        for (int blk = 0; blk <= M; ++blk) {
            const double* xb = xv + (blk == 0 ? ((int64_t)step * M - 1) * S
                                              : ((int64_t)step * M + blk - 1) * S);
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    const int k = blk * 9 + (dy + 1) * 3 + (dx + 1);
                    if (present(blk, step, yi, xi, dy, dx, n))
                        s = add(s, mul(__ldg(vr + (int64_t)k * N),
                                       __ldg(xb + (int64_t)(yi + dy) * n + (xi + dx))));
                }
        }
        double out = s;
        if (mode == 1) out = sub(b[r], s);
        else if (mode == 2) out = add(b[r], s);
        y[r] = out;
        if (REDUCE) {
            acc2 = fma(out, out, acc2);
            if (nonfinite && !isfinite(xv[r])) bad = true;
        }
    }
    if (REDUCE) {
        if (bad) atomicOr(nonfinite, 1);
        __shared__ double sh[GB / 32];
        __shared__ bool last;
        const double sblk = block_sum_flat<GB>(acc2, sh, tid);
        const unsigned int bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const unsigned int nb = gridDim.x * gridDim.y * gridDim.z;
        if (tid == 0) {
            partials[bid] = sblk;
            __threadfence();
            last = (atomicAdd(counter, 1u) == nb - 1);
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        double t = 0.0;
        for (unsigned int i = tid; i < nb; i += GB) t += __ldcg(partials + i);
        t = block_sum_flat<GB>(t, sh, tid);
        if (tid == 0) {
            *norm2 = t;
            *counter = 0u;
        }
    }
}

template <int M>
void launch_gspmv(Ctx& c, const GridSpmv& g, const double* x, double* y, int mode,
                  const double* b, const int* guard, int want, double* norm2, int* nonfinite) {
    const int gx = (g.n + 31) / 32, gy = (g.n + 7) / 8;
    const int64_t planes = g.nt * M;
    int64_t gz = std::min<int64_t>(planes, std::max<int64_t>(1, (int64_t)c.sms * 32 / (gx * gy)));
    if (norm2) gz = std::max<int64_t>(1, std::min<int64_t>(gz, kReduceMaxBlocks / (gx * gy)));
    const dim3 grid(gx, gy, (unsigned)gz), block(32, GB / 32);
    if (norm2) {
        if ((int64_t)gx * gy * gz > kReduceMaxBlocks) throw ConfigError("grid SpMV: too many blocks");
        launch(k_gspmv<M, true>, grid, block, 0, c.stream, g.nt, g.n, gy, g.N, g.vals.p, x, y,
               mode, b, guard, want, c.red_partials.p, c.red_counter.p, norm2, nonfinite);
    } else {
        launch(k_gspmv<M, false>, grid, block, 0, c.stream, g.nt, g.n, gy, g.N, g.vals.p, x, y,
               mode, b, guard, want, (double*)nullptr, (unsigned int*)nullptr, (double*)nullptr,
               (int*)nullptr);
    }
}
}  // namespace

static void gspmv_gather(Ctx& c, const Csr& A, GridSpmv& g) {
    launch(k_gspmv_gather, c.grid_for(g.N, 256), 256, 0, c.stream, g.N, g.M, g.n, A.rowptr.p,
           (const double*)A.val.p, g.vals.p);
    PD_LAUNCH_CHECK();
}

bool csr_attach_grid(Ctx& c, Csr& A, int64_t nt, int M, int64_t n) {
    ++c.epoch;
    A.grid.reset();
    A.grid_stale = false;
    if (getenv("PD_NO_GRID_SPMV") || M < 1 || M > 5 || n < 3 || nt < 1) return false;
    const int64_t S = n * n, N = nt * M * S;
    if (A.nrows != N || A.ncols != N || N >= INT32_MAX) return false;
    std::vector<int64_t> rp(N + 1);
    std::vector<int32_t> ci(std::max<int64_t>(A.nnz, 1));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    PD_CUDA(cudaMemcpy(rp.data(), A.rowptr.p, (N + 1) * 8, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(ci.data(), A.col.p, A.nnz * 4, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < N; ++r) {
        const int64_t plane = r / S, j = r - plane * S;
        const int64_t step = plane / M, y = j / n, x = j % n;
        int64_t p = rp[r];
        for (int blk = 0; blk <= M; ++blk) {
            if (blk == 0 && step == 0) continue;
            const int64_t cb = blk == 0 ? (step * M - 1) * S : (step * M + blk - 1) * S;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (y + dy < 0 || y + dy >= n || x + dx < 0 || x + dx >= n) continue;
                    if (p >= rp[r + 1] || ci[p] != cb + (y + dy) * n + (x + dx)) return false;
                    ++p;
                }
        }
        if (p != rp[r + 1]) return false;
    }
    auto g = std::make_shared<GridSpmv>();
    g->nt = nt;
    g->M = M;
    g->n = (int)n;
    g->K = 9 * (M + 1);
    g->N = N;
    g->vals.alloc((int64_t)g->K * N);
    gspmv_gather(c, A, *g);
    A.grid = g;
    return true;
}

bool grid_spmv(Ctx& c, const Csr& A, const double* x, double* y, int mode, const double* b,
               const int* guard, int want, double* norm2, int* nonfinite) {
    if (!A.grid) return false;
    GridSpmv& g = *A.grid;
    if (A.grid_stale) {  // the CSR's values changed since the last gather
        gspmv_gather(c, A, g);
        A.grid_stale = false;
    }
    switch (g.M) {
        case 1: launch_gspmv<1>(c, g, x, y, mode, b, guard, want, norm2, nonfinite); break;
        case 2: launch_gspmv<2>(c, g, x, y, mode, b, guard, want, norm2, nonfinite); break;
        case 3: launch_gspmv<3>(c, g, x, y, mode, b, guard, want, norm2, nonfinite); break;
        case 4: launch_gspmv<4>(c, g, x, y, mode, b, guard, want, norm2, nonfinite); break;
        case 5: launch_gspmv<5>(c, g, x, y, mode, b, guard, want, norm2, nonfinite); break;
        default: return false;
    }
    PD_LAUNCH_CHECK();
    return true;
}

}  // namespace pd
