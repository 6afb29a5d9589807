// Mode product of the spectral PFASST node solve (pfasst.py:118-132 solves
// (Mh + dt q Kh) x = b; for a structured FD Kh the exact inverse is
// Phi^(x)d diag(1/lambda) Phi^T(x)d with the 1D eigenvectors Phi):
//
//   out[o, a, r] = sum_i Mat[a, i] * in[o, i, r],   in/out C-order [outer][n][stride],
//   Mat = Phi^T (transpose = 1) or Phi (transpose = 0), phi row-major n x n.
//
// Hand-written FP64 GEMM (no library): every (o, r) pair is a column of an
// n x (outer * stride) matrix; a CTA produces a TM x TN output tile (128 or 64 rows, 64
// or 32 columns: small tiles keep the SMs busy on the coarse chain's one-grid launches)
// from K chunks of 16 staged in shared memory (next chunk prefetched into registers
// during the multiply), a thread an 8 x 4 register tile of plain DFMAs.  B200's FP64
// tensor rate equals its DFMA rate, so there is no tensor-core variant to prefer.
#include <cuda_runtime.h>

#include "pd_internal.h"

namespace pd {

namespace {

constexpr int MP_TK = 16;

// KCONTIG: stride == 1 (a column's entries are contiguous in memory).  TM x TN output
// tile per CTA, an 8 x CT register tile per thread: (TM/8) * (TN/CT) threads.
template <int TM, int TN, int CT, bool KCONTIG>
__global__ void __launch_bounds__((TM / 8) * (TN / CT), (TM / 8) * (TN / CT) >= 256 ? 2 : 1) k_mode_product(
    const double* __restrict__ in, double* __restrict__ out, int64_t ncols, int n, int64_t stride,
    const double* __restrict__ phi, int transpose) {
    constexpr int THREADS = (TM / 8) * (TN / CT);
    constexpr int NA = MP_TK * TM / THREADS, NX = MP_TK * TN / THREADS;
    __shared__ __align__(16) double As[MP_TK][TM];      // As[k][a] = Mat[a0 + a, k0 + k]
    __shared__ __align__(16) double Xs[MP_TK][TN + 4];  // Xs[k][c] = x_{c0 + c}[k0 + k]
    __shared__ int64_t colbase[TN];
    const int tid = threadIdx.x;
    const int64_t c0 = blockIdx.x * (int64_t)TN;
    const int a0 = blockIdx.y * TM;
    if (tid < TN) {
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
    const int tx = tid % (TN / CT), ty = tid / (TN / CT);  // column groups of CT, row groups of 8
    double acc[8][CT];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < CT; ++j) acc[i][j] = 0.0;
    // staging registers of the next K chunk
    double ra[NA], rx[NX];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int e = tid + q * THREADS;  // 0 .. TK*TM, walking phi's contiguous index
            int k, a;
            if (transpose) { a = e % TM; k = e / TM; }        // Mat[a, i] = phi[i * n + a]
            else { k = e % MP_TK; a = e / MP_TK; }            // Mat[a, i] = phi[a * n + i]
            const int gi = k0 + k, ga = a0 + a;
            ra[q] = (gi < n && ga < n) ? __ldg(phi + (transpose ? (int64_t)gi * n + ga
                                                                 : (int64_t)ga * n + gi))
                                       : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = tid + q * THREADS;  // 0 .. TK*TN
            int k, cc;
            if (KCONTIG) { k = e % MP_TK; cc = e / MP_TK; }
            else { cc = e % TN; k = e / TN; }
            const int64_t base = colbase[cc];
            const int gi = k0 + k;
            rx[q] = (base >= 0 && gi < n) ? __ldg(in + base + (int64_t)gi * (KCONTIG ? 1 : stride))
                                          : 0.0;
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int e = tid + q * THREADS;
            int k, a;
            if (transpose) { a = e % TM; k = e / TM; }
            else { k = e % MP_TK; a = e / MP_TK; }
            As[k][a] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = tid + q * THREADS;
            int k, cc;
            if (KCONTIG) { k = e % MP_TK; cc = e / MP_TK; }
            else { cc = e % TN; k = e / TN; }
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
            double a[8], b[CT];
            const double2* ap = reinterpret_cast<const double2*>(&As[k][ty * 8]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double2 v = ap[i];
                a[2 * i] = v.x;
                a[2 * i + 1] = v.y;
            }
            const double2* bp = reinterpret_cast<const double2*>(&Xs[k][tx * CT]);
#pragma unroll
            for (int j = 0; j < CT / 2; ++j) {
                const double2 v = bp[j];
                b[2 * j] = v.x;
                b[2 * j + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < CT; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < CT; ++j) {
        const int64_t base = colbase[tx * CT + j];
        if (base < 0) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int ga = a0 + ty * 8 + i;
            if (ga < n) out[base + (int64_t)ga * (KCONTIG ? 1 : stride)] = acc[i][j];
        }
    }
}

template <int TM, int TN, int CT>
void launch_mode_product(Ctx& c, const double* in, double* out, int64_t ncols, int n, int64_t stride,
                         const double* phi, int transpose) {
    const dim3 grid((unsigned)((ncols + TN - 1) / TN), (unsigned)((n + TM - 1) / TM));
    constexpr int threads = (TM / 8) * (TN / CT);
    if (stride == 1)
        launch(k_mode_product<TM, TN, CT, true>, grid, threads, 0, c.stream, in, out, ncols, n, stride,
               phi, transpose);
    else
        launch(k_mode_product<TM, TN, CT, false>, grid, threads, 0, c.stream, in, out, ncols, n, stride,
               phi, transpose);
}

}  // namespace

void mode_product(Ctx& c, const double* in, double* out, int64_t total, int64_t n, int64_t stride,
                  const double* phi, int transpose) {
    if (n <= 0 || total <= 0) return;
    if (total % (n * stride)) throw ConfigError("mode product: array size is not outer*n*stride");
    const int64_t ncols = total / n;
    // tile choice: rows padded to 64 or 128; narrow column tiles when wide ones would leave
    // SMs idle (the serial coarse chain runs one worker's 63^3 grid per launch)
    const bool tall = n > 64;
    const int64_t row_tiles = tall ? (n + 127) / 128 : 1;
    const bool wide = ((ncols + 63) / 64) * row_tiles >= 2 * (int64_t)c.sms;
    // (an 8 x 8 register tile was measured too: 10.2 vs 13.7 TFLOP/s at 127^3 x 32 — spills)
    if (tall) {
        if (wide) launch_mode_product<128, 64, 4>(c, in, out, ncols, (int)n, stride, phi, transpose);
        else launch_mode_product<128, 32, 4>(c, in, out, ncols, (int)n, stride, phi, transpose);
    } else {
        if (wide) launch_mode_product<64, 64, 4>(c, in, out, ncols, (int)n, stride, phi, transpose);
        else launch_mode_product<64, 32, 4>(c, in, out, ncols, (int)n, stride, phi, transpose);
    }
    PD_LAUNCH_CHECK();
}

}  // namespace pd
