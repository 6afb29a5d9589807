// K1 — matrix-free space-time operator of the DG-in-time system.
//
//   L = I (x) Aqh + S_{-1} (x) Bqh,   Aqh = Kq (x) Mh + dt Mq (x) Kh,
//   Bqh = -(Jq (x) Mh),  Jq = l0 l1^T  (only the last column is nonzero)
//                                                  spacetime.py:77-80,117-124
//   F(u) = L u + gamma (I (x) Mqh) r(u) - rhs      spacetime.py:131-142
//
// The spatial stiffness Kh is an S x S CSR (a few MB, L2-resident) and Mh its
// lumped diagonal; the M x M tableau lives in kernel parameters.  Every
// coefficient is rebuilt with the rounding of the reference's scipy kron/sum
// assembly (fl(Kq*mh) + fl(dt*fl(Mq*k)) on the diagonal, fl(dt*fl(Mq*k)) off
// it, -fl(l0*mh) for the step coupling) and summed in the global CSR's column
// order, so `apply` is bitwise the assembled matrix's SpMV while streaming
// only x and y from HBM (16 + 8/M bytes per dof instead of ~12*nnz_row).
// The `residual` mode follows the reference's blockwise evaluation order.
#include "../../include/paradiff_b200.h"
#include "pd_device.cuh"
#include "pd_stencil.h"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace pd {
using namespace dev;

namespace {
constexpr int SB = 256;

struct Tab {
    double Kq[kStMaxM * kStMaxM], Mq[kStMaxM * kStMaxM], l0[kStMaxM];
};

__device__ __forceinline__ double react_v(int kind, double u) {
    if (kind == 1) return sub(mul(mul(u, u), u), u);
    if (kind == 2) return sub(mul(u, u), u);
    return 0.0;
}

// coef[(m*M + m')*nnzK + p] = the Aqh CSR value of entry p of Kh's row j in
// block (m, m'), with scipy's rounding: fl(dt*fl(Mq*k)) off the diagonal,
// fl(fl(Kq*mh_j) + fl(dt*fl(Mq*k))) on it (spacetime.py:78, linalg.py:55-60)
__global__ void k_st_coef(int M, int64_t S, double dt, Tab T, const int64_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const double* __restrict__ kv,
                          const double* __restrict__ mh, int64_t nnzK, double* coef) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < S;
         j += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t p = rp[j]; p < rp[j + 1]; ++p)
            for (int mm = 0; mm < M * M; ++mm) {
                double cval = mul(dt, mul(T.Mq[mm], kv[p]));
                if (ci[p] == j) cval = add(mul(T.Kq[mm], mh[j]), cval);
                coef[(int64_t)mm * nnzK + p] = cval;
            }
    }
}

// y = L x (global CSR order) with mode 0 set, 1 b - Lx, 2 b + Lx; halo = x of
// the previous step's last node for the first local step (null: none).
// Grid: x over spatial rows j, y over planes (n, m): no index divisions.
template <bool REDUCE>
__global__ void __launch_bounds__(SB) k_st_apply(int64_t Nt, int M, int64_t S, Tab T,
                                                 const int64_t* __restrict__ rp,
                                                 const int32_t* __restrict__ ci,
                                                 const double* __restrict__ coef, int64_t nnzK,
                                                 const double* __restrict__ mh,
                                                 const double* __restrict__ x,
                                                 const double* __restrict__ halo, double* y,
                                                 int mode, const double* b, const int* guard,
                                                 int want, double* partials,
                                                 unsigned int* counter, double* norm2,
                                                 int* nonfinite) {
    if (guard_off(guard, want)) return;
    const int64_t MS = (int64_t)M * S;
    double acc2 = 0.0;
    bool bad = false;
    for (int64_t plane = blockIdx.y; plane < Nt * M; plane += gridDim.y) {
        const int64_t n = plane / M;
        const int m = (int)(plane - n * M);
        const double* xprev = n > 0 ? x + (n - 1) * MS + (int64_t)(M - 1) * S : halo;
        const double* xn = x + n * MS;
        const double l0m = T.l0[m];
        const double* cm = coef + (int64_t)m * M * nnzK;
        for (int64_t j = blockIdx.x * (int64_t)SB + threadIdx.x; j < S;
             j += (int64_t)gridDim.x * SB) {
            const int64_t r = plane * S + j;
            double s = 0.0;
            if (xprev && l0m != 0.0) s = add(s, mul(-mul(l0m, mh[j]), xprev[j]));
            const int64_t p0 = rp[j], p1 = rp[j + 1];
            for (int mp = 0; mp < M; ++mp) {
                const double* xm = xn + (int64_t)mp * S;
                const double* cmp = cm + (int64_t)mp * nnzK;
                for (int64_t p = p0; p < p1; ++p) s = add(s, mul(cmp[p], __ldg(xm + ci[p])));
            }
            double out = s;
            if (mode == 1) out = sub(b[r], s);
            else if (mode == 2) out = add(b[r], s);
            y[r] = out;
            if (REDUCE) {
                acc2 = fma(out, out, acc2);
                if (nonfinite && !isfinite(x[r])) bad = true;
            }
        }
    }
    if (REDUCE) {
        if (bad) atomicOr(nonfinite, 1);
        // 2D grid: flatten the block index for the deterministic finish
        __shared__ double sh[SB / 32];
        __shared__ bool last;
        double sblk = block_sum<SB>(acc2, sh);
        const unsigned int bid = blockIdx.y * gridDim.x + blockIdx.x;
        const unsigned int nb = gridDim.x * gridDim.y;
        if (threadIdx.x == 0) {
            partials[bid] = sblk;
            __threadfence();
            last = (atomicAdd(counter, 1u) == nb - 1);
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        double t = 0.0;
        for (unsigned int i = threadIdx.x; i < nb; i += SB) t += __ldcg(partials + i);
        t = block_sum<SB>(t, sh);
        if (threadIdx.x == 0) {
            *norm2 = t;
            *counter = 0u;
        }
    }
}

// F(u) in the reference's blockwise order (spacetime.py:135-141):
// res = Aqh u_n ; res += gamma*(Mqh r(u_n)) ; res += Bqh u_{n-1} (n>0) ; res -= rhs
__global__ void __launch_bounds__(SB) k_st_residual(int64_t Nt, int M, int64_t S, double dt,
                                                    Tab T, const int64_t* __restrict__ rp,
                                                    const int32_t* __restrict__ ci,
                                                    const double* __restrict__ coef, int64_t nnzK,
                                                    const double* __restrict__ mh,
                                                    const double* __restrict__ u,
                                                    const double* __restrict__ rhs,
                                                    double* __restrict__ out, double gamma,
                                                    int kind) {
    const int64_t MS = (int64_t)M * S;
    for (int64_t plane = blockIdx.y; plane < Nt * M; plane += gridDim.y) {
        const int64_t n = plane / M;
        const int m = (int)(plane - n * M);
        const double* un = u + n * MS;
        const double* cm = coef + (int64_t)m * M * nnzK;
        for (int64_t j = blockIdx.x * (int64_t)SB + threadIdx.x; j < S;
             j += (int64_t)gridDim.x * SB) {
            const int64_t r = plane * S + j;
            const double mj = mh[j];
            const int64_t p0 = rp[j], p1 = rp[j + 1];
            double s = 0.0;
            for (int mp = 0; mp < M; ++mp) {
                const double* um = un + (int64_t)mp * S;
                const double* cmp = cm + (int64_t)mp * nnzK;
                for (int64_t p = p0; p < p1; ++p) s = add(s, mul(cmp[p], um[ci[p]]));
            }
            if (gamma != 0.0) {
                // (Mqh r(U_n))_j ; Mqh = dt * (Mq (x) Mh): entries fl(dt*fl(Mq*mh))
                double t = 0.0;
                for (int mp = 0; mp < M; ++mp)
                    t = add(t, mul(mul(dt, mul(T.Mq[m * M + mp], mj)),
                                   react_v(kind, un[(int64_t)mp * S + j])));
                s = add(s, mul(gamma, t));
            }
            if (n > 0 && T.l0[m] != 0.0)
                s = add(s, mul(-mul(T.l0[m], mj), u[(n - 1) * MS + (int64_t)(M - 1) * S + j]));
            if (n == 0) s = sub(s, rhs[r]);
            out[r] = s;
        }
    }
}

// ---- structured-grid K1 (Dirichlet 1D/2D/3D constant-coefficient stencils) ----
// When Kh is the (2*DIM+1)-point stencil on an n^DIM grid with one value per
// stencil position and Mh is constant, every coefficient of L depends only on
// (m, m', position): a table of M*M*(2*DIM+1) values (scipy's rounding, built
// by k_st_coef on the grid's first interior row) replaces the per-entry coef/ci
// gathers.  A thread owns one point of one step and produces its M rows from
// the (2*DIM+1)*M neighbour values (coalesced along x, reused through L1), each
// row summed in the global CSR's column order (previous step's last node, then
// per node m' the stencil positions -z,-y,-x,c,+x,+y,+z); a missing boundary
// entry contributes c * 0, which leaves the sum unchanged: bitwise the CSR SpMV.
// The coefficient table travels as a kernel parameter and a block handles one step
// (no step loop): the unrolled multiplies take their coefficients from uniform
// registers / the constant bank — no shared-memory loads (round 1 spent 48 LDS per
// point on them), 0.075 -> 0.054 ms on C2.  With a step loop the compiler hoisted the
// 48 coefficients into 96 registers (spills) or, behind an opaque pointer, re-read
// them by generic loads (0.084 ms).

template <int DIM, int M>
struct GridTabP {
    double c[M * M * (2 * DIM + 1) + M];  // [m][m'][pos], then the step coupling per m
};

template <int DIM, int M, bool REDUCE>
__global__ void __launch_bounds__(SB, M <= 3 ? 3 : 2) k_st_grid(int64_t Nt, int n, int gy,
                                                const __grid_constant__ GridTabP<DIM, M> T,
                                                const double* __restrict__ x,
                                                const double* __restrict__ halo, double* y,
                                                int mode, const double* b, const int* guard,
                                                int want, double* partials,
                                                unsigned int* counter, double* norm2,
                                                int* nonfinite) {
    if (guard_off(guard, want)) return;
    constexpr int NP = 2 * DIM + 1;  // stencil positions, column order
    // the M*M*NP + M coefficients are kernel parameters: with the loops unrolled every
    // use is a constant-bank operand of the multiply (no shared-memory or global loads)
    const double* c = T.c;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    // block (32 x 8) tiles x and y; blockIdx.y = (z, y-tile); blockIdx.z = the time step
    const int zi = DIM == 3 ? (int)(blockIdx.y / gy) : 0;
    const int yt = DIM == 3 ? (int)(blockIdx.y - zi * gy) : (int)blockIdx.y;
    const int xi = blockIdx.x * 32 + threadIdx.x;
    const int yi = DIM >= 2 ? yt * 8 + threadIdx.y : 0;
    const bool inside = xi < n && (DIM < 2 || yi < n);
    const int64_t S = DIM == 1 ? n : DIM == 2 ? (int64_t)n * n : (int64_t)n * n * n;
    const int64_t MS = (int64_t)M * S;
    const int j = (zi * n + yi) * n + xi;  // S < 2^31 (checked at plan time)
    int off[NP];
    bool has[NP];
    {
        int k = 0;
        if (DIM == 3) { off[k] = -n * n; has[k++] = zi > 0; }
        if (DIM >= 2) { off[k] = -n; has[k++] = yi > 0; }
        off[k] = -1; has[k++] = xi > 0;
        off[k] = 0; has[k++] = true;
        off[k] = 1; has[k++] = xi < n - 1;
        if (DIM >= 2) { off[k] = n; has[k++] = yi < n - 1; }
        if (DIM == 3) { off[k] = n * n; has[k++] = zi < n - 1; }
    }
    const int Si = (int)S;
    double acc2 = 0.0;
    bool bad = false;
    // one step per block (gridDim.z = Nt): without a loop the coefficients stay
    // constant-bank operands of the multiplies instead of being hoisted into registers
    const int64_t step = blockIdx.z;
    if (inside && step < Nt) {
        const double* xs = x + step * MS + j;
        double v[M][NP];
#pragma unroll
        for (int mp = 0; mp < M; ++mp)
#pragma unroll
            for (int k = 0; k < NP; ++k)
                v[mp][k] = has[k] ? __ldg(xs + (mp * Si + off[k])) : 0.0;
        const double* xp = step > 0 ? xs - MS + (M - 1) * Si : (halo ? halo + j : nullptr);
        const double vprev = xp ? __ldg(xp) : 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            double sacc = 0.0;
            if (xp && c[M * M * NP + m] != 0.0) sacc = add(sacc, mul(c[M * M * NP + m], vprev));
#pragma unroll
            for (int mp = 0; mp < M; ++mp)
#pragma unroll
                for (int k = 0; k < NP; ++k)  // an absent entry adds c * 0: bitwise a no-op
                    sacc = add(sacc, mul(c[(m * M + mp) * NP + k], v[mp][k]));
            const int64_t r = step * MS + j + m * Si;
            double out = sacc;
            if (mode == 1) out = sub(b[r], sacc);
            else if (mode == 2) out = add(b[r], sacc);
            y[r] = out;
            if (REDUCE) {
                acc2 = fma(out, out, acc2);
                if (nonfinite && !isfinite(v[m][DIM])) bad = true;
            }
        }
    }
    if (REDUCE) {
        if (bad) atomicOr(nonfinite, 1);
        __shared__ double sh[SB / 32];
        __shared__ bool last;
        // block_sum needs a flat thread index: reduce over tid order
        double sblk = block_sum_flat<SB>(acc2, sh, tid);
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
        for (unsigned int i = tid; i < nb; i += SB) t += __ldcg(partials + i);
        t = block_sum_flat<SB>(t, sh, tid);
        if (tid == 0) {
            *norm2 = t;
            *counter = 0u;
        }
    }
}

// ---- periodic 2D grids (BASELINE config 3) ----
// The same kernel for the 5-point stencil with wrap-around neighbours.  Every point has
// all five entries; what changes at the grid's edges is their COLUMN ORDER in the CSR
// row (a wrapped neighbour's column sorts to the other end), and the sum must follow it
// to stay bitwise scipy's.  Products are formed in the interior order (y-1, x-1, c, x+1,
// y+1) and added in the order of the point's case: x interior / first / last column
// times y interior / first / last line — nine fully unrolled variants, divergent only in
// the warps that touch an edge.
template <int XC, int YC>
__device__ __forceinline__ double add_periodic5(double s, const double (&p)[5]) {
    // x group in column order
    auto xg = [&](double a) {
        if (XC == 0) { a = add(a, p[1]); a = add(a, p[2]); a = add(a, p[3]); }        // x-1, c, x+1
        else if (XC == 1) { a = add(a, p[2]); a = add(a, p[3]); a = add(a, p[1]); }   // x = 0
        else { a = add(a, p[3]); a = add(a, p[1]); a = add(a, p[2]); }                // x = n-1
        return a;
    };
    if (YC == 0) { s = add(s, p[0]); s = xg(s); s = add(s, p[4]); }        // y-1, X, y+1
    else if (YC == 1) { s = xg(s); s = add(s, p[4]); s = add(s, p[0]); }   // y = 0: y-1 wraps last
    else { s = add(s, p[4]); s = add(s, p[0]); s = xg(s); }                // y = n-1: y+1 wraps first
    return s;
}

template <int M, int XC, int YC>
__device__ __forceinline__ void rows_periodic(const double* c, const double (&v)[M][5], bool prev,
                                              double vprev, double (&out)[M]) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
        double sacc = 0.0;
        if (prev && c[M * M * 5 + m] != 0.0) sacc = add(sacc, mul(c[M * M * 5 + m], vprev));
#pragma unroll
        for (int mp = 0; mp < M; ++mp) {
            double p[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) p[k] = mul(c[(m * M + mp) * 5 + k], v[mp][k]);
            sacc = add_periodic5<XC, YC>(sacc, p);
        }
        out[m] = sacc;
    }
}

template <int M, bool REDUCE>
__global__ void __launch_bounds__(SB, M <= 3 ? 3 : 2) k_st_grid_per(
    int64_t Nt, int n, const __grid_constant__ GridTabP<2, M> T, const double* __restrict__ x,
    const double* __restrict__ halo, double* y, int mode, const double* b, const int* guard,
    int want, double* partials, unsigned int* counter, double* norm2, int* nonfinite) {
    if (guard_off(guard, want)) return;
    const double* c = T.c;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int xi = blockIdx.x * 32 + threadIdx.x;
    const int yi = (int)blockIdx.y * 8 + threadIdx.y;
    const bool inside = xi < n && yi < n;
    const int Si = n * n;
    const int64_t MS = (int64_t)M * Si;
    const int j = yi * n + xi;
    double acc2 = 0.0;
    bool bad = false;
    const int64_t step = blockIdx.z;
    if (inside && step < Nt) {
        const int xc = xi == 0 ? 1 : (xi == n - 1 ? 2 : 0), yc = yi == 0 ? 1 : (yi == n - 1 ? 2 : 0);
        int off[5];
        off[0] = yc == 1 ? (n - 1) * n : -n;
        off[1] = xc == 1 ? n - 1 : -1;
        off[2] = 0;
        off[3] = xc == 2 ? -(n - 1) : 1;
        off[4] = yc == 2 ? -(n - 1) * n : n;
        const double* xs = x + step * MS + j;
        double v[M][5];
#pragma unroll
        for (int mp = 0; mp < M; ++mp)
#pragma unroll
            for (int k = 0; k < 5; ++k) v[mp][k] = __ldg(xs + (mp * Si + off[k]));
        const double* xp = step > 0 ? xs - MS + (M - 1) * Si : (halo ? halo + j : nullptr);
        const double vprev = xp ? __ldg(xp) : 0.0;
        double rows[M];
        switch (yc * 3 + xc) {
            case 0: rows_periodic<M, 0, 0>(c, v, xp != nullptr, vprev, rows); break;
            case 1: rows_periodic<M, 1, 0>(c, v, xp != nullptr, vprev, rows); break;
            case 2: rows_periodic<M, 2, 0>(c, v, xp != nullptr, vprev, rows); break;
            case 3: rows_periodic<M, 0, 1>(c, v, xp != nullptr, vprev, rows); break;
            case 4: rows_periodic<M, 1, 1>(c, v, xp != nullptr, vprev, rows); break;
            case 5: rows_periodic<M, 2, 1>(c, v, xp != nullptr, vprev, rows); break;
            case 6: rows_periodic<M, 0, 2>(c, v, xp != nullptr, vprev, rows); break;
            case 7: rows_periodic<M, 1, 2>(c, v, xp != nullptr, vprev, rows); break;
            default: rows_periodic<M, 2, 2>(c, v, xp != nullptr, vprev, rows); break;
        }
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int64_t r = step * MS + j + m * Si;
            double out = rows[m];
            if (mode == 1) out = sub(b[r], rows[m]);
            else if (mode == 2) out = add(b[r], rows[m]);
            y[r] = out;
            if (REDUCE) {
                acc2 = fma(out, out, acc2);
                if (nonfinite && !isfinite(v[m][2])) bad = true;
            }
        }
    }
    if (REDUCE) {
        if (bad) atomicOr(nonfinite, 1);
        __shared__ double sh[SB / 32];
        __shared__ bool last;
        double sblk = block_sum_flat<SB>(acc2, sh, tid);
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
        for (unsigned int i = tid; i < nb; i += SB) t += __ldcg(partials + i);
        t = block_sum_flat<SB>(t, sh, tid);
        if (tid == 0) {
            *norm2 = t;
            *counter = 0u;
        }
    }
}

// the grid table from the coefficient table of one interior row (k_st_coef's
// rounding) and the step coupling -fl(l0[m]*mh)
__global__ void k_st_grid_tab(int M, int NP, int64_t nnzK, const int64_t* __restrict__ rp,
                              int64_t jrow, const double* __restrict__ coef, Tab T,
                              const double* __restrict__ mh, double* tab) {
    const int64_t p0 = rp[jrow];
    for (int i = threadIdx.x; i < M * M * NP; i += blockDim.x) {
        const int mm = i / NP, k = i - mm * NP;
        tab[i] = coef[(int64_t)mm * nnzK + p0 + k];
    }
    for (int m = threadIdx.x; m < M; m += blockDim.x) tab[M * M * NP + m] = -mul(T.l0[m], mh[jrow]);
}

}  // namespace

static Tab make_tab_raw(const double* Kq, const double* Mq, const double* l0, int M) {
    Tab T;
    std::memset(&T, 0, sizeof(T));
    std::memcpy(T.Kq, Kq, sizeof(double) * M * M);
    std::memcpy(T.Mq, Mq, sizeof(double) * M * M);
    std::memcpy(T.l0, l0, sizeof(double) * M);
    return T;
}

StOp::StOp(Ctx& c_, int64_t Nt_, int M_, int64_t S_, const double* Kq_, const double* Mq_,
           const double* l0_, double dt_, const Csr& Kh_, const double* mh_host)
    : c(c_), Nt(Nt_), M(M_), S(S_), dt(dt_) {
    if (M < 1 || M > kStMaxM) throw ConfigError("node count out of range for the stencil operator");
    if (Kh_.nrows != S || Kh_.ncols != S) throw ConfigError("Kh must be S x S");
    std::memcpy(Kq, Kq_, sizeof(double) * M * M);
    std::memcpy(Mq, Mq_, sizeof(double) * M * M);
    std::memcpy(l0, l0_, sizeof(double) * M);
    std::vector<int64_t> rp(S + 1);
    PD_CUDA(cudaMemcpy(rp.data(), Kh_.rowptr.p, (S + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    Kh = csr_upload(c, S, S, Kh_.nnz, Kh_.rowptr.p, Kh_.col.p, Kh_.val.p, true);
    mh.alloc(S);
    PD_CUDA(cudaMemcpy(mh.p, mh_host, S * sizeof(double), cudaMemcpyHostToDevice));
    nnzK = Kh->nnz;
    coef.alloc(std::max<int64_t>((int64_t)M * M * nnzK, 1));
    Tab T = make_tab_raw(Kq, Mq, l0, M);
    launch(k_st_coef, c.grid_for(S, SB), SB, 0, c.stream, M, S, dt, T, Kh->rowptr.p, Kh->col.p,
           Kh->val.p, mh.p, nnzK, coef.p);
    PD_LAUNCH_CHECK();
    PD_CUDA(cudaStreamSynchronize(c.stream));
    detect_grid(rp, mh_host);
}

// Kh is exactly the Dirichlet (2d+1)-point stencil on an n^d grid (d = 2, 3)
// with one value per stencil position (positions in CSR column order: -z, -y,
// -x, centre, +x, +y, +z; boundary rows simply lack the outside neighbours).
// Checked entry by entry on a host copy.  jc = a centre row with every entry.
bool detect_dirichlet_stencil(const Csr& K, int& dim, int& n_out, double tv[7], int64_t& jc_out) {
    const int64_t S = K.nrows;
    dim = 0;
    if (S < 27 || K.ncols != S || getenv("PD_NO_GRID_STENCIL")) return false;
    std::vector<int64_t> rp(S + 1);
    std::vector<int32_t> ci(std::max<int64_t>(K.nnz, 1));
    std::vector<double> kv(std::max<int64_t>(K.nnz, 1));
    PD_CUDA(cudaMemcpy(rp.data(), K.rowptr.p, (S + 1) * 8, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(ci.data(), K.col.p, K.nnz * 4, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(kv.data(), K.val.p, K.nnz * 8, cudaMemcpyDeviceToHost));
    for (int d = 2; d <= 3; ++d) {
        const int64_t n = (int64_t)llround(std::pow((double)S, 1.0 / d));
        const int64_t Sd = d == 2 ? n * n : n * n * n;
        if (Sd != S || n < 3 || S >= INT_MAX / 8) continue;
        const int NP = 2 * d + 1;
        const int64_t mid = n / 2, jc = d == 2 ? mid * n + mid : (mid * n + mid) * n + mid;
        if (rp[jc + 1] - rp[jc] != NP) continue;
        for (int k = 0; k < NP; ++k) tv[k] = kv[rp[jc] + k];
        bool ok = true;
        for (int64_t j = 0; j < S && ok; ++j) {
            const int64_t xi = j % n, yi = (j / n) % n, zi = d == 3 ? j / (n * n) : 0;
            int64_t off[7];
            bool has[7];
            int k = 0;
            if (d == 3) { off[k] = -n * n; has[k++] = zi > 0; }
            off[k] = -n; has[k++] = yi > 0;
            off[k] = -1; has[k++] = xi > 0;
            off[k] = 0; has[k++] = true;
            off[k] = 1; has[k++] = xi < n - 1;
            off[k] = n; has[k++] = yi < n - 1;
            if (d == 3) { off[k] = n * n; has[k++] = zi < n - 1; }
            int64_t p = rp[j];
            for (k = 0; k < NP && ok; ++k) {
                if (!has[k]) continue;
                if (p >= rp[j + 1] || ci[p] != j + off[k] || kv[p] != tv[k]) ok = false;
                ++p;
            }
            if (p != rp[j + 1]) ok = false;
        }
        if (getenv("PD_STENCIL_VERBOSE"))
            fprintf(stderr, "[stencil] S=%lld d=%d n=%lld %s\n", (long long)S, d, (long long)n,
                    ok ? "structured" : "not constant-coefficient");
        if (!ok) continue;
        dim = d;
        n_out = (int)n;
        jc_out = jc;
        return true;
    }
    return false;
}

// Kh is exactly the periodic 5-point stencil on an n x n grid (n >= 3): every row has
// its five wrapped neighbours, in sorted column order, with one value per position.
// tv = values by position (y-1, x-1, c, x+1, y+1) of an interior row jc.
static bool detect_periodic_stencil2d(const Csr& K, int& n_out, int64_t& jc_out) {
    const int64_t S = K.nrows;
    if (S < 9 || K.ncols != S || K.nnz != 5 * S || getenv("PD_NO_GRID_STENCIL")) return false;
    const int64_t n = (int64_t)llround(std::sqrt((double)S));
    if (n * n != S || n < 3 || S >= INT_MAX / 8) return false;
    std::vector<int64_t> rp(S + 1);
    std::vector<int32_t> ci(K.nnz);
    std::vector<double> kv(K.nnz);
    PD_CUDA(cudaMemcpy(rp.data(), K.rowptr.p, (S + 1) * 8, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(ci.data(), K.col.p, K.nnz * 4, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(kv.data(), K.val.p, K.nnz * 8, cudaMemcpyDeviceToHost));
    const int64_t mid = n / 2, jc = mid * n + mid;
    if (n < 5 || rp[jc + 1] - rp[jc] != 5) return false;
    double tv[5];
    for (int k = 0; k < 5; ++k) tv[k] = kv[rp[jc] + k];
    for (int64_t j = 0; j < S; ++j) {
        if (rp[j + 1] - rp[j] != 5) return false;
        const int64_t xi = j % n, yi = j / n;
        // (column, position) of the five wrapped neighbours, sorted by column
        std::pair<int64_t, int> e[5] = {
            {((yi + n - 1) % n) * n + xi, 0}, {yi * n + (xi + n - 1) % n, 1}, {j, 2},
            {yi * n + (xi + 1) % n, 3}, {((yi + 1) % n) * n + xi, 4}};
        std::sort(e, e + 5);
        for (int k = 0; k < 5; ++k)
            if (ci[rp[j] + k] != e[k].first || kv[rp[j] + k] != tv[e[k].second]) return false;
    }
    n_out = (int)n;
    jc_out = jc;
    return true;
}

// Structured K1 mode: Kh a Dirichlet constant-coefficient stencil, Mh constant,
// and a kernel instantiated for M.
void StOp::detect_grid(const std::vector<int64_t>& rp, const double* mh_host) {
    (void)rp;
    grid_dim = 0;
    if (getenv("PD_NO_GRID_K1") || M < 2 || M > 5) return;
    for (int64_t j = 1; j < S; ++j)
        if (mh_host[j] != mh_host[0]) return;
    int d = 0, n = 0;
    double tv[7];
    int64_t jc = 0;
    if (S * M >= INT_MAX) return;
    if (!detect_dirichlet_stencil(*Kh, d, n, tv, jc)) {
        if (!detect_periodic_stencil2d(*Kh, n, jc)) return;
        d = 2;
        grid_periodic = true;
    }
    grid_tab.alloc(kGridMaxTabHost);
    Tab T = make_tab_raw(Kq, Mq, l0, (int)M);
    launch(k_st_grid_tab, 1, 128, 0, c.stream, (int)M, 2 * d + 1, nnzK, Kh->rowptr.p, jc, coef.p,
           T, mh.p, grid_tab.p);
    PD_LAUNCH_CHECK();
    {  // blocks of one structured apply: x tiles * line tiles (* planes) * steps
        const int64_t gx = (n + 31) / 32, gy = (n + 7) / 8;
        const int64_t per_step = gx * (d == 3 ? gy * n : gy);
        if (Nt > 65535 || per_step * Nt > ((int64_t)1 << 26)) return;  // general kernel instead
        grid_blocks_max = std::max<int64_t>(kGridMaxBlocks, per_step * Nt);
    }
    grid_partials.alloc((size_t)grid_blocks_max);
    grid_counter.alloc(1);
    PD_CUDA(cudaMemsetAsync(grid_counter.p, 0, sizeof(unsigned int), c.stream));
    // host copy: the coefficients travel to k_st_grid as kernel parameters
    grid_tab_host.assign((size_t)M * M * (2 * d + 1) + M, 0.0);
    PD_CUDA(cudaMemcpyAsync(grid_tab_host.data(), grid_tab.p, grid_tab_host.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, c.stream));
    PD_CUDA(cudaStreamSynchronize(c.stream));
    grid_dim = d;
    grid_n = n;
}

static Tab make_tab(const StOp& op) { return make_tab_raw(op.Kq, op.Mq, op.l0, (int)op.M); }

static dim3 st_grid(const Ctx& c, int64_t S, int64_t planes, bool reduce) {
    int64_t gx = (S + SB - 1) / SB;
    int64_t gy = planes;
    const int64_t cap = reduce ? kReduceMaxBlocks : (int64_t)c.sms * 16;
    if (gx > cap) gx = cap;
    if (gx * gy > cap) gy = std::max<int64_t>(1, cap / gx);
    return dim3((unsigned)gx, (unsigned)gy);
}

template <int DIM, int MM>
static void launch_grid(const StOp& op, const double* x, double* y, int mode, const double* b,
                        const int* guard, int want, double* norm2_out, int* nonfinite,
                        const double* halo) {
    Ctx& c = op.c;
    const int n = op.grid_n;
    const int gx = (n + 31) / 32, gy = DIM >= 2 ? (n + 7) / 8 : 1;
    const int gyz = DIM == 3 ? gy * n : gy;
    // one step per block (blockIdx.z): the kernel has no step loop, so its M*M*NP + M
    // coefficients stay constant-bank operands; the fused norm keeps one partial per block
    // (grid_partials is sized for it at plan time)
    const int64_t per_step = (int64_t)gx * gyz;
    const int64_t gz = op.Nt;
    if (gz > 65535 || per_step * gz > op.grid_blocks_max)
        throw ConfigError("grid K1: too many blocks");
    const dim3 grid((unsigned)gx, (unsigned)gyz, (unsigned)gz), block(32, SB / 32);
    GridTabP<DIM, MM> T;
    if (op.grid_tab_host.size() != sizeof(T.c) / sizeof(double))
        throw ConfigError("grid K1: coefficient table size mismatch");
    std::memcpy(T.c, op.grid_tab_host.data(), sizeof(T.c));
    if constexpr (DIM == 2) {
        if (op.grid_periodic) {
            if (norm2_out)
                launch(k_st_grid_per<MM, true>, grid, block, 0, c.stream, op.Nt, n, T, x, halo, y,
                       mode, b, guard, want, op.grid_partials.p, op.grid_counter.p, norm2_out,
                       nonfinite);
            else
                launch(k_st_grid_per<MM, false>, grid, block, 0, c.stream, op.Nt, n, T, x, halo, y,
                       mode, b, guard, want, (double*)nullptr, (unsigned int*)nullptr,
                       (double*)nullptr, (int*)nullptr);
            return;
        }
    }
    if (norm2_out) {
        launch(k_st_grid<DIM, MM, true>, grid, block, 0, c.stream, op.Nt, n, gy, T, x,
               halo, y, mode, b, guard, want, op.grid_partials.p, op.grid_counter.p, norm2_out,
               nonfinite);
    } else {
        launch(k_st_grid<DIM, MM, false>, grid, block, 0, c.stream, op.Nt, n, gy, T,
               x, halo, y, mode, b, guard, want, (double*)nullptr, (unsigned int*)nullptr,
               (double*)nullptr, (int*)nullptr);
    }
}

template <int DIM>
static bool launch_grid_m(const StOp& op, const double* x, double* y, int mode, const double* b,
                          const int* guard, int want, double* norm2_out, int* nonfinite,
                          const double* halo) {
    switch (op.M) {
        case 2: launch_grid<DIM, 2>(op, x, y, mode, b, guard, want, norm2_out, nonfinite, halo); return true;
        case 3: launch_grid<DIM, 3>(op, x, y, mode, b, guard, want, norm2_out, nonfinite, halo); return true;
        case 4: launch_grid<DIM, 4>(op, x, y, mode, b, guard, want, norm2_out, nonfinite, halo); return true;
        case 5: launch_grid<DIM, 5>(op, x, y, mode, b, guard, want, norm2_out, nonfinite, halo); return true;
        default: return false;
    }
}

void StOp::apply(const double* x, double* y, int mode, const double* b, const int* guard,
                 int want, double* norm2_out, int* nonfinite, const double* halo) const {
    const int64_t N = size();
    if (N <= 0) return;
    if (grid_dim == 2 || grid_dim == 3) {
        const bool done = grid_dim == 2
            ? launch_grid_m<2>(*this, x, y, mode, b, guard, want, norm2_out, nonfinite, halo)
            : launch_grid_m<3>(*this, x, y, mode, b, guard, want, norm2_out, nonfinite, halo);
        if (done) {
            PD_LAUNCH_CHECK();
            return;
        }
    }
    const Tab T = make_tab(*this);
    if (norm2_out) {
        launch(k_st_apply<true>, st_grid(c, S, Nt * M, true), SB, 0, c.stream, Nt, (int)M, S, T,
               Kh->rowptr.p, Kh->col.p, coef.p, nnzK, mh.p, x, halo, y, mode, b, guard, want,
               c.red_partials.p, c.red_counter.p, norm2_out, nonfinite);
    } else {
        launch(k_st_apply<false>, st_grid(c, S, Nt * M, false), SB, 0, c.stream, Nt, (int)M, S,
               T, Kh->rowptr.p, Kh->col.p, coef.p, nnzK, mh.p, x, halo, y, mode, b, guard, want,
               (double*)nullptr, (unsigned int*)nullptr, (double*)nullptr, (int*)nullptr);
    }
    PD_LAUNCH_CHECK();
}

void StOp::residual(const double* u, const double* rhs, double* out, double gamma, int kind) const {
    const int64_t N = size();
    if (N <= 0) return;
    const Tab T = make_tab(*this);
    launch(k_st_residual, st_grid(c, S, Nt * M, false), SB, 0, c.stream, Nt, (int)M, S, dt, T,
           Kh->rowptr.p, Kh->col.p, coef.p, nnzK, mh.p, u, rhs, out, gamma, kind);
    PD_LAUNCH_CHECK();
}

}  // namespace pd

namespace {
template <class F>
int guarded_st(F&& f) {
    try {
        f();
        return PD_OK;
    } catch (const pd::ConfigError& e) {
        pd_set_error_(e.what(), -1);
        return PD_ERR_CONFIG;
    } catch (const std::exception& e) {
        pd_set_error_(e.what(), -1);
        return PD_ERR_CUDA;
    }
}
}  // namespace

extern "C" {

int pd_stop_create(void* ctx, int64_t Nt, int M, int64_t S, const double* Kq, const double* Mq,
                   const double* l0, double dt, void* Kh, const double* mh_host, void** out) {
    return guarded_st([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        if (!Kh) throw pd::ConfigError("null Kh");
        *out = new pd::StOp(c, Nt, M, S, Kq, Mq, l0, dt, *static_cast<pd::Csr*>(Kh), mh_host);
    });
}

int pd_stop_destroy(void* op) {
    return guarded_st([&] { delete static_cast<pd::StOp*>(op); });
}

int pd_stop_apply(void* op, const double* x, double* y, int mode, const double* b,
                  const double* halo) {
    return guarded_st([&] {
        if (mode < 0 || mode > 2) throw pd::ConfigError("bad apply mode");
        static_cast<pd::StOp*>(op)->apply(x, y, mode, b, nullptr, 0, nullptr, nullptr, halo);
    });
}

int pd_stop_residual(void* op, const double* u, const double* rhs, double* out, double gamma,
                     int kind) {
    return guarded_st(
        [&] { static_cast<pd::StOp*>(op)->residual(u, rhs, out, gamma, kind); });
}

}  // extern "C"
