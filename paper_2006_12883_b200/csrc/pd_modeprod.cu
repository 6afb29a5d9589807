// Mode product of the spectral PFASST node solve (pfasst.py:118-132 solves
// (Mh + dt q Kh) x = b; for a structured FD Kh the exact inverse is
// Phi^(x)d diag(1/lambda) Phi^T(x)d with the 1D eigenvectors Phi):
//
//   out[o, a, r] = sum_i Mat[a, i] * in[o, i, r],   in/out C-order [outer][n][stride],
//   Mat = Phi^T (transpose = 1) or Phi (transpose = 0), phi row-major n x n.
//
// Hand-written FP64 GEMM (no library): every (o, r) pair is a column of an
// n x (outer * stride) matrix; a CTA produces a 128 x 64 output tile from K chunks of
// 16 staged in shared memory (next chunk prefetched into registers during the
// multiply), a thread an 8 x 4 register tile of plain DFMAs.  B200's FP64 tensor rate
// equals its DFMA rate, so there is no tensor-core variant to prefer.  n <= 128 rows
// per CTA tile; larger n loops over row tiles.
#include <cuda_runtime.h>

#include "pd_internal.h"

namespace pd {

namespace {

constexpr int MP_TM = 128, MP_TN = 64, MP_TK = 16, MP_THREADS = 256;

// KCONTIG: stride == 1 (a column's entries are contiguous in memory)
template <bool KCONTIG>
__global__ void __launch_bounds__(MP_THREADS, 2) k_mode_product(
    const double* __restrict__ in, double* __restrict__ out, int64_t ncols, int n, int64_t stride,
    const double* __restrict__ phi, int transpose) {
    __shared__ __align__(16) double As[MP_TK][MP_TM];      // As[k][a] = Mat[a0 + a, k0 + k]
    __shared__ __align__(16) double Xs[MP_TK][MP_TN + 4];  // Xs[k][c] = x_{c0 + c}[k0 + k]
    __shared__ int64_t colbase[MP_TN];
    const int tid = threadIdx.x;
    const int64_t c0 = blockIdx.x * (int64_t)MP_TN;
    const int a0 = blockIdx.y * MP_TM;
    if (tid < MP_TN) {
        const int64_t c = c0 + tid;
        int64_t base = -1;
        if (c < ncols) {
            if (KCONTIG) base = c * n;
            else {
                const int64_t o = c / stride, r = c - o * stride;
                base = o * n * stride + r;
            }
        }
        colbase[tid] = base;
    }
    __syncthreads();
    const int tx = tid & 15, ty = tid >> 4;  // 16 column groups of 4, 16 row groups of 8
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    // staging registers: 8 matrix entries and 4 vector entries per thread and chunk
    double ra[8], rx[4];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid + q * MP_THREADS;  // 0 .. TK*TM
            // consecutive threads walk phi's contiguous index
            int k, a;
            if (transpose) { a = e % MP_TM; k = e / MP_TM; }   // Mat[a, i] = phi[i * n + a]
            else { k = e % MP_TK; a = e / MP_TK; }             // Mat[a, i] = phi[a * n + i]
            const int gi = k0 + k, ga = a0 + a;
            ra[q] = (gi < n && ga < n) ? __ldg(phi + (transpose ? (int64_t)gi * n + ga
                                                                 : (int64_t)ga * n + gi))
                                       : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + q * MP_THREADS;  // 0 .. TK*TN
            int k, cc;
            if (KCONTIG) { k = e % MP_TK; cc = e / MP_TK; }
            else { cc = e % MP_TN; k = e / MP_TN; }
            const int64_t base = colbase[cc];
            const int gi = k0 + k;
            rx[q] = (base >= 0 && gi < n) ? __ldg(in + base + (int64_t)gi * (KCONTIG ? 1 : stride))
                                          : 0.0;
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid + q * MP_THREADS;
            int k, a;
            if (transpose) { a = e % MP_TM; k = e / MP_TM; }
            else { k = e % MP_TK; a = e / MP_TK; }
            As[k][a] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + q * MP_THREADS;
            int k, cc;
            if (KCONTIG) { k = e % MP_TK; cc = e / MP_TK; }
            else { cc = e % MP_TN; k = e / MP_TN; }
            Xs[k][cc] = rx[q];
        }
    };
    fetch(0);
    for (int k0 = 0; k0 < n; k0 += MP_TK) {
        stage();
        __syncthreads();
        if (k0 + MP_TK < n) fetch(k0 + MP_TK);
#pragma unroll
        for (int k = 0; k < MP_TK; ++k) {
            double a[8], b[4];
            const double2* ap = reinterpret_cast<const double2*>(&As[k][ty * 8]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double2 v = ap[i];
                a[2 * i] = v.x;
                a[2 * i + 1] = v.y;
            }
            const double2* bp = reinterpret_cast<const double2*>(&Xs[k][tx * 4]);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double2 v = bp[j];
                b[2 * j] = v.x;
                b[2 * j + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t base = colbase[tx * 4 + j];
        if (base < 0) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int ga = a0 + ty * 8 + i;
            if (ga < n) out[base + (int64_t)ga * (KCONTIG ? 1 : stride)] = acc[i][j];
        }
    }
}

}  // namespace

void mode_product(Ctx& c, const double* in, double* out, int64_t total, int64_t n, int64_t stride,
                  const double* phi, int transpose) {
    if (n <= 0 || total <= 0) return;
    if (total % (n * stride)) throw ConfigError("mode product: array size is not outer*n*stride");
    const int64_t ncols = total / n;
    const dim3 grid((unsigned)((ncols + MP_TN - 1) / MP_TN), (unsigned)((n + MP_TM - 1) / MP_TM));
    if (stride == 1)
        launch(k_mode_product<true>, grid, MP_THREADS, 0, c.stream, in, out, ncols, (int)n, stride,
               phi, transpose);
    else
        launch(k_mode_product<false>, grid, MP_THREADS, 0, c.stream, in, out, ncols, (int)n, stride,
               phi, transpose);
    PD_LAUNCH_CHECK();
}

}  // namespace pd
