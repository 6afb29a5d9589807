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

#include <cstdlib>

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

// Large products (many columns) on the FP64 tensor path: mma.sync m8n8k4 (DMMA).  CTA tile
// 128 rows x 64 columns, 8 warps as 4 x 2, a warp 32 x 32 = 4 x 4 MMA tiles (32
// accumulators per lane); K chunks of 16 staged through registers like the DFMA kernel.
// Fragment layout (PTX ISA, m8n8k4 .f64): A[row = lane / 4][k = lane % 4],
// B[k = lane % 4][col = lane / 4], C[row = lane / 4][col = 2 (lane % 4) + {0, 1}].
constexpr int MM_THREADS = 256;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// MM_TM = 128 (4 x 2 warps, 64 columns) or 64 (2 x 4 warps, 128 columns)
template <int MM_TM, bool KCONTIG>
__global__ void __launch_bounds__(MM_THREADS, 2) k_mode_product_mma(
    const double* __restrict__ in, double* __restrict__ out, int64_t ncols, int n, int64_t stride,
    const double* __restrict__ phi, int transpose) {
    constexpr int WR = MM_TM / 32, MM_TN = (8 / WR) * 32, MM_LDA = MM_TM + 8, MM_LDX = MM_TN + 8;
    __shared__ __align__(16) double As[MP_TK][MM_LDA];  // As[k][a] = Mat[a0 + a, k0 + k]
    __shared__ __align__(16) double Xs[MP_TK][MM_LDX];  // Xs[k][c] = x_{c0 + c}[k0 + k]
    __shared__ int64_t colbase[MM_TN];
    const int tid = threadIdx.x;
    const int64_t c0 = blockIdx.x * (int64_t)MM_TN;
    const int a0 = blockIdx.y * MM_TM;
    if (tid < MM_TN) {
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
    constexpr int NA = MP_TK * MM_TM / MM_THREADS, NX = MP_TK * MM_TN / MM_THREADS;
    double ra[NA], rx[NX];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int e = tid + q * MM_THREADS;
            int k, a;
            if (transpose) { a = e % MM_TM; k = e / MM_TM; }
            else { k = e % MP_TK; a = e / MP_TK; }
            const int gi = k0 + k, ga = a0 + a;
            ra[q] = (gi < n && ga < n) ? __ldg(phi + (transpose ? (int64_t)gi * n + ga
                                                                 : (int64_t)ga * n + gi))
                                       : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = tid + q * MM_THREADS;
            int k, cc;
            if (KCONTIG) { k = e % MP_TK; cc = e / MP_TK; }
            else { cc = e % MM_TN; k = e / MM_TN; }
            const int64_t base = colbase[cc];
            const int gi = k0 + k;
            rx[q] = (base >= 0 && gi < n) ? __ldg(in + base + (int64_t)gi * (KCONTIG ? 1 : stride))
                                          : 0.0;
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            const int e = tid + q * MM_THREADS;
            int k, a;
            if (transpose) { a = e % MM_TM; k = e / MM_TM; }
            else { k = e % MP_TK; a = e / MP_TK; }
            As[k][a] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            const int e = tid + q * MM_THREADS;
            int k, cc;
            if (KCONTIG) { k = e % MP_TK; cc = e / MP_TK; }
            else { cc = e % MM_TN; k = e / MM_TN; }
            Xs[k][cc] = rx[q];
        }
    };
    const int lane = tid & 31, warp = tid >> 5;
    const int wr = (warp % WR) * 32, wc = (warp / WR) * 32;  // warp tile origin (rows, cols)
    const int g = lane >> 2, t = lane & 3;
    double acc[4][4][2];  // [row tile][col tile][2 columns]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    fetch(0);
    for (int k0 = 0; k0 < n; k0 += MP_TK) {
        stage();
        __syncthreads();
        if (k0 + MP_TK < n) fetch(k0 + MP_TK);
#pragma unroll
        for (int ks = 0; ks < MP_TK; ks += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[ks + t][wr + 8 * i + g];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Xs[ks + t][wc + 8 * j + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t base = colbase[wc + 8 * j + 2 * t + h];
            if (base < 0) continue;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ga = a0 + wr + 8 * i + g;
                if (ga < n) out[base + (int64_t)ga * (KCONTIG ? 1 : stride)] = acc[i][j][h];
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
    // many columns and a tall matrix: the tensor (DMMA) kernel.  Measured alternatives at
    // 127^3 x 32: DFMA 8 x 4 register tile 13.7 TFLOP/s, 8 x 8 with register staging 10.2
    // (spills), 8 x 8 with cp.async staging 10.4.
    static const bool no_mma = getenv("PD_MODEPROD_NO_MMA") != nullptr;
    const int mm_tm = n > 64 ? 128 : 64, mm_tn = n > 64 ? 64 : 128;
    if (!no_mma && n > 32 &&
        ((ncols + mm_tn - 1) / mm_tn) * ((n + mm_tm - 1) / mm_tm) >= 2 * (int64_t)c.sms) {
        const dim3 grid((unsigned)((ncols + mm_tn - 1) / mm_tn), (unsigned)((n + mm_tm - 1) / mm_tm));
        auto go = [&](auto kernel) {
            launch(kernel, grid, MM_THREADS, 0, c.stream, in, out, ncols, (int)n, stride, phi,
                   transpose);
        };
        if (mm_tm == 128) {
            if (stride == 1) go(k_mode_product_mma<128, true>);
            else go(k_mode_product_mma<128, false>);
        } else {
            if (stride == 1) go(k_mode_product_mma<64, true>);
            else go(k_mode_product_mma<64, false>);
        }
        PD_LAUNCH_CHECK();
        return;
    }
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
