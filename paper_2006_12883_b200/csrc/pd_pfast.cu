// P-fast: matrix-free block-Jacobi-in-time smoother with inner spatial V-cycles
// (SURVEY §7.1 "(P-fast) north_star matrix-free profile", §7.2 item 7).
//
// The space-time system is the reference's L = I⊗Aqh + S₋₁⊗Bqh
// (spacetime.py:77-80,117-124) on a structured FD grid: Kh = κ h^{d-2}(2d·I − Σ
// neighbours), Mh = h^d I, Aqh = Kq⊗Mh + dt·Mq⊗Kh, Bqh = −Jq⊗Mh (only the last
// node couples, Jq[:, M-1] = l(0)).  One outer sweep (structure of
// multigrid.py:243-305, time blocks as linalg.py:152-189 with one block per
// step):
//     r = b − L x;  e_t ≈ Aqh⁻¹ r_t for every step t by ONE spatial V-cycle;
//     x += ω_t e.
// The V-cycle is batched over all steps: point-block damped Jacobi (the M×M
// diagonal block of Aqh inverted on the host), full-weighting restriction
// R = Pᵀ, bilinear/trilinear prolongation, coarse operators rediscretised at
// 2h (non-Galerkin), the coarsest level smoothed `coarse_sweeps` times.
// There is no reference counterpart; parity is against the CPU restatement in
// oracle/pfast_oracle.py.
//
// Layout: (nt, M, n^d) C-order fp64, the last grid axis fastest — the layout
// of every other kernel of the library.  Every kernel is one pass over HBM
// with the neighbour planes served from L1/L2 (algorithmic bytes in DESIGN §4).
#include "../../include/paradiff_b200.h"
#include "pd_internal.h"

#include <cmath>
#include <cstdlib>
#include <memory>
#include <vector>

namespace pd {
namespace {

constexpr int PFB = 256;
constexpr int kPfMaxM = 5;
constexpr int kPfNormBlocks = 1024;

struct PfCoef {  // one level's point-block operator (row-major M×M each)
    double Ac[kPfMaxM * kPfMaxM];    // Kq·h^d + dt·Mq·κh^{d-2}·2d (centre)
    double Ao[kPfMaxM * kPfMaxM];    // −dt·Mq·κh^{d-2} (per neighbour)
    double Dinv[kPfMaxM * kPfMaxM];  // ω·Ac⁻¹
    double cprev[kPfMaxM];           // −l0[m]·h^d (level 0 time coupling)
    double omega_t;                  // outer damping (MODE 4)
};

// per-axis neighbour of coordinate v (−1 = outside a Dirichlet grid)
template <bool PER>
__device__ __forceinline__ int nb(int v, int d, int n) {
    const int w = v + d;
    if (PER) return w < 0 ? w + n : (w >= n ? w - n : w);
    return (w < 0 || w >= n) ? -1 : w;
}

// MODE 0: out = x + Dinv(b − A x)     (damped point-block Jacobi)
// MODE 1: out = Dinv b                (first sweep from a zero guess)
// MODE 2: out = b − A x               (level residual)
// MODE 3: out = b − A x − cprev·x[t-1, M-1]  (space-time residual, level 0;
//         at t = 0 the coupling uses `halo` when non-null)
// MODE 4: out += ω_t (x + Dinv(b − A x))  (MODE 0 fused with the outer update)
template <int DIM, int M, int MODE, bool PER>
__global__ void __launch_bounds__(PFB) k_pf_point(PfCoef C, int n, int64_t nt,
                                                 const double* __restrict__ x,
                                                 const double* __restrict__ b, double* out,
                                                 const double* __restrict__ halo) {
    // one warp per (step, grid row, 32-point x tile): 32-bit index math only
    const unsigned nn = (unsigned)n;
    const unsigned R = DIM == 2 ? nn : nn * nn;  // rows per step
    const unsigned xt = (nn + 31u) / 32u;
    const unsigned items = (unsigned)nt * R * xt;  // < 2^31 (checked at plan time)
    const int64_t S = (int64_t)R * nn;
    const unsigned lane = threadIdx.x & 31u;
    for (unsigned w = blockIdx.x * (PFB / 32) + (threadIdx.x >> 5); w < items;
         w += gridDim.x * (PFB / 32)) {
        const unsigned row = w / xt;
        const unsigned ix_u = (w - row * xt) * 32u + lane;
        if (ix_u >= nn) continue;
        const unsigned t_u = row / R;
        const unsigned rr = row - t_u * R;
        const int64_t t = t_u;
        const int64_t j = (int64_t)rr * nn + ix_u;
        const int64_t base = t * M * S + j;
        double bv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) bv[m] = b[base + m * S];
        if (MODE == 1) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(C.Dinv[m * M + k], bv[k], acc);
                out[base + m * S] = acc;
            }
            continue;
        }
        const int ix = (int)ix_u;
        const int iy = DIM == 2 ? (int)rr : (int)(rr % nn);
        const int iz = DIM == 3 ? (int)(rr / nn) : 0;
        // neighbour offsets (relative to j); 0 marks "outside" for Dirichlet
        int64_t off[2 * DIM];
        bool ok[2 * DIM];
        {
            int k = 0;
            int w;
            w = nb<PER>(ix, -1, n); ok[k] = w >= 0; off[k++] = (int64_t)(w - ix);
            w = nb<PER>(ix, 1, n); ok[k] = w >= 0; off[k++] = (int64_t)(w - ix);
            w = nb<PER>(iy, -1, n); ok[k] = w >= 0; off[k++] = (int64_t)(w - iy) * n;
            w = nb<PER>(iy, 1, n); ok[k] = w >= 0; off[k++] = (int64_t)(w - iy) * n;
            if (DIM == 3) {
                w = nb<PER>(iz, -1, n); ok[k] = w >= 0; off[k++] = (int64_t)(w - iz) * n * n;
                w = nb<PER>(iz, 1, n); ok[k] = w >= 0; off[k++] = (int64_t)(w - iz) * n * n;
            }
        }
        double xc[M], ns[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const double* xm = x + base + m * S;
            xc[m] = xm[0];
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 2 * DIM; ++k) s += ok[k] ? xm[off[k]] : 0.0;
            ns[m] = s;
        }
        double r[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            double ax = 0.0;
#pragma unroll
            for (int k = 0; k < M; ++k) {
                ax = fma(C.Ac[m * M + k], xc[k], ax);
                ax = fma(C.Ao[m * M + k], ns[k], ax);
            }
            r[m] = bv[m] - ax;
        }
        if (MODE == 3 && (t > 0 || halo)) {
            // x[t-1, M-1, j]; the first step of a time slab reads the previous
            // slab's last node (halo) when the steps are sharded over ranks
            const double xp = t > 0 ? x[base - S] : halo[j];
#pragma unroll
            for (int m = 0; m < M; ++m) r[m] = fma(-C.cprev[m], xp, r[m]);
        }
        if (MODE == 2 || MODE == 3) {
#pragma unroll
            for (int m = 0; m < M; ++m) out[base + m * S] = r[m];
        } else {
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double acc = xc[m];
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(C.Dinv[m * M + k], r[k], acc);
                if (MODE == 4)  // last level-0 sweep: straight into the solution
                    out[base + m * S] = fma(C.omega_t, acc, out[base + m * S]);
                else
                    out[base + m * S] = acc;
            }
        }
    }
}

// per-axis restriction stencil: fine coordinates feeding coarse c, weights 1/2,1,1/2
template <bool PER>
__device__ __forceinline__ void rstencil(int c, int nf, int f[3]) {
    const int ctr = PER ? 2 * c : 2 * c + 1;
    f[0] = nb<PER>(ctr, -1, nf);
    f[1] = ctr;
    f[2] = nb<PER>(ctr, 1, nf);
}

// coarse = Pᵀ fine over planes (nt·M of them).  One warp per coarse row: the
// row's plane/y/z decomposition and its 3×3 fine source rows once per row,
// lanes across x.
template <int DIM, bool PER>
__global__ void __launch_bounds__(PFB) k_pf_restrict(int nc, int nf, int64_t planes,
                                                    const double* __restrict__ fine,
                                                    double* coarse) {
    const int64_t Sc = DIM == 2 ? (int64_t)nc * nc : (int64_t)nc * nc * nc;
    const int64_t Sf = DIM == 2 ? (int64_t)nf * nf : (int64_t)nf * nf * nf;
    const double w[3] = {0.5, 1.0, 0.5};
    const unsigned R = DIM == 2 ? (unsigned)nc : (unsigned)nc * nc;  // coarse rows per plane
    const unsigned rows = (unsigned)planes * R;
    const int lane = threadIdx.x & 31;
    for (unsigned row = blockIdx.x * (PFB / 32) + (threadIdx.x >> 5); row < rows;
         row += gridDim.x * (PFB / 32)) {
        const unsigned p_u = row / R;
        const unsigned rr = row - p_u * R;
        const int cy = DIM == 2 ? (int)rr : (int)(rr % (unsigned)nc);
        const int cz = DIM == 3 ? (int)(rr / (unsigned)nc) : 0;
        int fy[3], fz[3] = {0, -1, -1};
        rstencil<PER>(cy, nf, fy);
        if (DIM == 3) rstencil<PER>(cz, nf, fz);
        const double* src = fine + (int64_t)p_u * Sf;
        // up to 9 source rows with their weights (missing rows: weight 0, row 0)
        const double* rp[9];
        double rw[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
                const bool ok = (DIM == 3 ? fz[a] >= 0 : a == 1) && fy[bb] >= 0;
                const int zz = DIM == 3 ? fz[a] : 0;
                rp[a * 3 + bb] = src + (ok ? ((int64_t)zz * nf + fy[bb]) * nf : 0);
                rw[a * 3 + bb] = ok ? (DIM == 3 ? w[a] : 1.0) * w[bb] : 0.0;
            }
        double* dst = coarse + (int64_t)p_u * Sc + (int64_t)rr * nc;
        for (int cx = lane; cx < nc; cx += 32) {
            int fx[3];
            rstencil<PER>(cx, nf, fx);
            const bool okl = fx[0] >= 0;  // Dirichlet: always; periodic: wrapped
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                if (rw[k] == 0.0) continue;
                const double* r = rp[k];
                double v = okl ? 0.5 * __ldg(r + fx[0]) : 0.0;
                v = fma(1.0, __ldg(r + fx[1]), v);
                v = fma(0.5, __ldg(r + fx[2]), v);
                acc = fma(rw[k], v, acc);
            }
            dst[cx] = acc;
        }
    }
}

// per-axis interpolation: coarse sources of fine f (index −1 = none) and weights
template <bool PER>
__device__ __forceinline__ void pstencil(int f, int nc, int c[2], double w[2]) {
    if (PER) {
        if ((f & 1) == 0) { c[0] = f >> 1; w[0] = 1.0; c[1] = -1; w[1] = 0.0; }
        else { c[0] = f >> 1; c[1] = (c[0] + 1 == nc) ? 0 : c[0] + 1; w[0] = w[1] = 0.5; }
    } else {
        if (f & 1) { c[0] = f >> 1; w[0] = 1.0; c[1] = -1; w[1] = 0.0; }
        else {
            c[0] = (f >> 1) - 1; c[1] = f >> 1; w[0] = w[1] = 0.5;
            if (c[0] < 0) c[0] = -1;
            if (c[1] >= nc) c[1] = -1;
        }
    }
}

// fine += P coarse over planes.  One warp per fine row: its (≤ 2×2) coarse
// source rows and weights once per row, lanes across x.
template <int DIM, bool PER>
__global__ void __launch_bounds__(PFB) k_pf_prolong_add(int nc, int nf, int64_t planes,
                                                       const double* __restrict__ coarse,
                                                       double* fine) {
    const int64_t Sc = DIM == 2 ? (int64_t)nc * nc : (int64_t)nc * nc * nc;
    const int64_t Sf = DIM == 2 ? (int64_t)nf * nf : (int64_t)nf * nf * nf;
    const unsigned R = DIM == 2 ? (unsigned)nf : (unsigned)nf * nf;  // fine rows per plane
    const unsigned rows = (unsigned)planes * R;
    const int lane = threadIdx.x & 31;
    for (unsigned row = blockIdx.x * (PFB / 32) + (threadIdx.x >> 5); row < rows;
         row += gridDim.x * (PFB / 32)) {
        const unsigned p_u = row / R;
        const unsigned rr = row - p_u * R;
        const int fy = DIM == 2 ? (int)rr : (int)(rr % (unsigned)nf);
        const int fz = DIM == 3 ? (int)(rr / (unsigned)nf) : 0;
        int cy[2], cz[2] = {0, -1};
        double wy[2], wz[2] = {1.0, 0.0};
        pstencil<PER>(fy, nc, cy, wy);
        if (DIM == 3) pstencil<PER>(fz, nc, cz, wz);
        const double* src = coarse + (int64_t)p_u * Sc;
        const double* rp[4];
        double rw[4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const bool ok = cz[a] >= 0 && cy[bb] >= 0;
                rp[a * 2 + bb] = src + (ok ? ((int64_t)cz[a] * nc + cy[bb]) * nc : 0);
                rw[a * 2 + bb] = ok ? wz[a] * wy[bb] : 0.0;
            }
        double* dst = fine + (int64_t)p_u * Sf + (int64_t)rr * nf;
        // 8 x tiles per pass: the fine loads of all eight are in flight together
        for (int fx0 = lane; fx0 < nf; fx0 += 256) {
            double fv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) fv[u] = fx0 + 32 * u < nf ? dst[fx0 + 32 * u] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int fx = fx0 + 32 * u;
                if (fx >= nf) break;
                int cx[2];
                double wx[2];
                pstencil<PER>(fx, nc, cx, wx);
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (rw[k] == 0.0) continue;
                    const double* r = rp[k];
                    double v = cx[0] >= 0 ? wx[0] * __ldg(r + cx[0]) : 0.0;
                    if (cx[1] >= 0) v = fma(wx[1], __ldg(r + cx[1]), v);
                    acc = fma(rw[k], v, acc);
                }
                dst[fx] = fv[u] + acc;
            }
        }
    }
}

__global__ void __launch_bounds__(PFB) k_pf_axpy(int64_t n, double a, const double* __restrict__ e,
                                                double* x) {
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PFB)
        x[i] = fma(a, e[i], x[i]);
}

// deterministic two-pass |v|^2 (fixed grid, fixed partial order)
__global__ void __launch_bounds__(PFB) k_pf_norm_part(int64_t n, const double* __restrict__ v,
                                                     double* part) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PFB)
        acc = fma(v[i], v[i], acc);
    __shared__ double sh[PFB];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = PFB / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_pf_norm_final(const double* __restrict__ part, double* out) {
    __shared__ double sh[PFB];
    double acc = 0.0;
    for (int i = threadIdx.x; i < kPfNormBlocks; i += PFB) acc += part[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = PFB / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// host M×M inverse (Gauss-Jordan, partial pivoting)
bool invert(const double* A, double* Ai, int M) {
    double a[kPfMaxM][2 * kPfMaxM];
    for (int i = 0; i < M; ++i)
        for (int k = 0; k < 2 * M; ++k) a[i][k] = k < M ? A[i * M + k] : (k - M == i ? 1.0 : 0.0);
    for (int c = 0; c < M; ++c) {
        int p = c;
        for (int i = c + 1; i < M; ++i)
            if (std::fabs(a[i][c]) > std::fabs(a[p][c])) p = i;
        if (a[p][c] == 0.0) return false;
        for (int k = 0; k < 2 * M; ++k) std::swap(a[c][k], a[p][k]);
        const double d = a[c][c];
        for (int k = 0; k < 2 * M; ++k) a[c][k] /= d;
        for (int i = 0; i < M; ++i) {
            if (i == c) continue;
            const double f = a[i][c];
            for (int k = 0; k < 2 * M; ++k) a[i][k] -= f * a[c][k];
        }
    }
    for (int i = 0; i < M; ++i)
        for (int k = 0; k < M; ++k) Ai[i * M + k] = a[i][M + k];
    return true;
}

}  // namespace

struct PfastPlan {
    Ctx& c;
    int dim, M, levels, nu, coarse_sweeps;
    bool periodic;
    int64_t nt;
    double omega_t;
    std::vector<int> n;            // grid points per axis per level
    std::vector<int64_t> len;      // nt·M·n^d per level
    std::vector<PfCoef> coef;
    std::vector<DevBuf<double>> B, E, T;  // level rhs, iterate, ping-pong
    DevBuf<double> part, norm;
    double* pinned = nullptr;
    const double* halo = nullptr;  // previous slab's last node (sharded steps)
    PfastPlan(Ctx& c_) : c(c_) {}
    ~PfastPlan() {
        if (pinned) cudaFreeHost(pinned);
    }
};

namespace {

// One wave of resident blocks (grid-stride kernels): a grid of sms x 8 blocks
// with only 6 resident per SM left a second, mostly empty wave (ncu: achieved
// occupancy 52% of a theoretical 75%).
template <class K>
int one_wave(const PfastPlan& P, K kernel, int64_t threads) {
    int occ = 0;
    PD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, PFB, 0));
    static const int cap = getenv("PD_PF_BLOCKS") ? atoi(getenv("PD_PF_BLOCKS")) : 0;
    if (cap > 0) occ = std::min(occ, cap);  // probe knob: fewer resident rows per SM
    return P.c.grid_for(threads, PFB, std::max(occ, 1));
}

template <int DIM, int M, bool PER>
void launch_point(PfastPlan& P, int l, int mode, const double* x, const double* b, double* out) {
    const int64_t nl = P.n[l];
    const int64_t rows = P.nt * (P.dim == 2 ? nl : nl * nl);
    const int64_t threads = rows * ((nl + 31) / 32) * 32;
    const PfCoef& C = P.coef[l];
    auto go = [&](auto kernel, const double* halo) {
        launch(kernel, one_wave(P, kernel, threads), PFB, 0, P.c.stream, C, P.n[l], P.nt, x, b, out,
               halo);
    };
    switch (mode) {
        case 0: go(k_pf_point<DIM, M, 0, PER>, nullptr); break;
        case 1: go(k_pf_point<DIM, M, 1, PER>, nullptr); break;
        case 2: go(k_pf_point<DIM, M, 2, PER>, nullptr); break;
        case 4: go(k_pf_point<DIM, M, 4, PER>, nullptr); break;
        default: go(k_pf_point<DIM, M, 3, PER>, P.halo);
    }
    PD_LAUNCH_CHECK();
}

template <int DIM, int M, bool PER>
void point_op(PfastPlan& P, int l, int mode, const double* x, const double* b, double* out) {
    launch_point<DIM, M, PER>(P, l, mode, x, b, out);
}

using PointFn = void (*)(PfastPlan&, int, int, const double*, const double*, double*);

template <int DIM, bool PER>
PointFn pick_m(int M) {
    switch (M) {
        case 1: return point_op<DIM, 1, PER>;
        case 2: return point_op<DIM, 2, PER>;
        case 3: return point_op<DIM, 3, PER>;
        case 4: return point_op<DIM, 4, PER>;
        default: return point_op<DIM, 5, PER>;
    }
}

PointFn pick(const PfastPlan& P) {
    if (P.dim == 2) return P.periodic ? pick_m<2, true>(P.M) : pick_m<2, false>(P.M);
    return P.periodic ? pick_m<3, true>(P.M) : pick_m<3, false>(P.M);
}

void restrict_to(PfastPlan& P, int l, const double* fine, double* coarse) {
    const int64_t planes = P.nt * P.M;
    const int nc = P.n[l + 1], nf = P.n[l];
    const int64_t rows = planes * (P.dim == 2 ? nc : (int64_t)nc * nc);
    if (P.dim == 2) {
        if (P.periodic) launch(k_pf_restrict<2, true>, one_wave(P, k_pf_restrict<2, true>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, fine, coarse);
        else launch(k_pf_restrict<2, false>, one_wave(P, k_pf_restrict<2, false>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, fine, coarse);
    } else {
        if (P.periodic) launch(k_pf_restrict<3, true>, one_wave(P, k_pf_restrict<3, true>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, fine, coarse);
        else launch(k_pf_restrict<3, false>, one_wave(P, k_pf_restrict<3, false>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, fine, coarse);
    }
    PD_LAUNCH_CHECK();
}

void prolong_add(PfastPlan& P, int l, const double* coarse, double* fine) {
    const int64_t planes = P.nt * P.M;
    const int nc = P.n[l + 1], nf = P.n[l];
    const int64_t rows = planes * (P.dim == 2 ? nf : (int64_t)nf * nf);
    if (P.dim == 2) {
        if (P.periodic) launch(k_pf_prolong_add<2, true>, one_wave(P, k_pf_prolong_add<2, true>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, coarse, fine);
        else launch(k_pf_prolong_add<2, false>, one_wave(P, k_pf_prolong_add<2, false>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, coarse, fine);
    } else {
        if (P.periodic) launch(k_pf_prolong_add<3, true>, one_wave(P, k_pf_prolong_add<3, true>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, coarse, fine);
        else launch(k_pf_prolong_add<3, false>, one_wave(P, k_pf_prolong_add<3, false>, rows * 32), PFB, 0, P.c.stream, nc, nf, planes, coarse, fine);
    }
    PD_LAUNCH_CHECK();
}

// e_l ≈ A_l⁻¹ B_l from a zero guess; result in P.E[l] (T[l] is scratch).
// With xupd (level 0) the last smoothing sweep, when it is a MODE 0 sweep,
// adds ω_t·e straight into xupd instead of storing e (returns true then).
bool vcycle(PfastPlan& P, int l, double* xupd = nullptr) {
    bool fused = false;
    const PointFn op = pick(P);
    const int sweeps = (l == P.levels - 1) ? P.coarse_sweeps : P.nu;
    double* e = P.E[l].p;
    double* t = P.T[l].p;
    const double* b = P.B[l].p;
    bool last = false;  // the smoothing pass that ends this level's work
    auto smooth = [&](int count, bool from_zero) {
        for (int s = 0; s < count; ++s) {
            if (from_zero && s == 0) {
                op(P, l, 1, nullptr, b, e);
            } else if (last && xupd && s == count - 1) {
                op(P, l, 4, e, b, xupd);
                fused = true;
            } else {
                op(P, l, 0, e, b, t);
                std::swap(e, t);
            }
        }
    };
    last = l == P.levels - 1;
    smooth(sweeps, true);
    if (l < P.levels - 1) {
        op(P, l, 2, e, b, t);  // t = b − A e
        restrict_to(P, l, t, P.B[l + 1].p);
        vcycle(P, l + 1);
        prolong_add(P, l, P.E[l + 1].p, e);
        last = true;
        smooth(P.nu, false);
    }
    if (e != P.E[l].p) std::swap(P.E[l].p, P.T[l].p);  // current iterate back in E[l]
    return fused;
}

void norm2(PfastPlan& P, const double* v, int64_t n, double* out_dev) {
    launch(k_pf_norm_part, kPfNormBlocks, PFB, 0, P.c.stream, n, v, P.part.p);
    launch(k_pf_norm_final, 1, PFB, 0, P.c.stream, (const double*)P.part.p, out_dev);
    PD_LAUNCH_CHECK();
}

}  // namespace
}  // namespace pd

namespace {
template <class F>
int guarded_pf(F&& f) {
    try {
        f();
        return PD_OK;
    } catch (const pd::ConfigError& e) {
        pd_set_error_(e.what(), -1);
        return PD_ERR_CONFIG;
    } catch (const pd::SolverError& e) {
        pd_set_error_(e.what(), e.index);
        return PD_ERR_SOLVER;
    } catch (const std::exception& e) {
        pd_set_error_(e.what(), -1);
        return PD_ERR_CUDA;
    }
}
}  // namespace

extern "C" {

int pd_pfast_create(void* ctx, int dim, int64_t n, int bc_periodic, double kappa, int M, int64_t nt,
                    double dt, const double* Kq, const double* Mq, const double* l0, int levels,
                    int nu, int coarse_sweeps, double omega_s, double omega_t, void** out) {
    return guarded_pf([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        if (dim != 2 && dim != 3) throw pd::ConfigError("P-fast needs a 2D or 3D grid");
        if (M < 1 || M > pd::kPfMaxM) throw pd::ConfigError("P-fast supports 1..5 nodes");
        if (nt < 1 || n < 1) throw pd::ConfigError("P-fast needs nt >= 1 and n >= 1");
        if (levels < 1 || nu < 1 || coarse_sweeps < 1)
            throw pd::ConfigError("P-fast needs levels, nu and coarse_sweeps >= 1");
        auto P = std::make_unique<pd::PfastPlan>(c);
        P->dim = dim;
        P->M = M;
        P->nt = nt;
        P->levels = levels;
        P->nu = nu;
        P->coarse_sweeps = coarse_sweeps;
        P->periodic = bc_periodic != 0;
        P->omega_t = omega_t;
        int64_t nl = n;
        for (int l = 0; l < levels; ++l) {
            if (l > 0) {
                if (P->periodic) {
                    if (nl % 2 || nl < 4) throw pd::ConfigError("cannot coarsen the periodic grid");
                    nl /= 2;
                } else {
                    if (nl % 2 == 0 || nl < 3) throw pd::ConfigError("cannot coarsen the Dirichlet grid");
                    nl = (nl - 1) / 2;
                }
            }
            if (nl > (1 << 20)) throw pd::ConfigError("grid too large");
            if (nt * M * nl * (dim == 3 ? nl : 1) * ((nl + 31) / 32) >= (int64_t(1) << 31))
                throw pd::ConfigError("P-fast grid x steps too large for one plan");
            P->n.push_back((int)nl);
            int64_t S = nl * nl * (dim == 3 ? nl : 1);
            P->len.push_back(nt * M * S);
            // h of this level (StencilSpec.h: Dirichlet 1/(n+1), periodic 1/n)
            const double h = P->periodic ? 1.0 / (double)nl : 1.0 / (double)(nl + 1);
            const double mh = std::pow(h, dim);
            const double ks = kappa * std::pow(h, dim - 2);
            pd::PfCoef C{};
            double D[pd::kPfMaxM * pd::kPfMaxM];
            for (int i = 0; i < M; ++i)
                for (int k = 0; k < M; ++k) {
                    C.Ac[i * M + k] = Kq[i * M + k] * mh + dt * Mq[i * M + k] * (ks * 2.0 * dim);
                    C.Ao[i * M + k] = -dt * Mq[i * M + k] * ks;
                    D[i * M + k] = C.Ac[i * M + k];
                }
            double Di[pd::kPfMaxM * pd::kPfMaxM];
            if (!pd::invert(D, Di, M)) throw pd::ConfigError("singular point block");
            for (int i = 0; i < M * M; ++i) C.Dinv[i] = omega_s * Di[i];
            for (int m = 0; m < M; ++m) C.cprev[m] = -l0[m] * mh;
            C.omega_t = omega_t;
            P->coef.push_back(C);
        }
        P->B.resize(levels);
        P->E.resize(levels);
        P->T.resize(levels);
        for (int l = 0; l < levels; ++l) {
            P->B[l].alloc(P->len[l]);
            P->E[l].alloc(P->len[l]);
            P->T[l].alloc(P->len[l]);
        }
        P->part.alloc(pd::kPfNormBlocks);
        P->norm.alloc(1);
        PD_CUDA(cudaMallocHost(&P->pinned, sizeof(double)));
        *out = P.release();
    });
}

/* r = b − L x (the space-time residual at level 0); |r|^2 into *norm2_dev when non-null */
int pd_pfast_residual(void* plan, const double* x, const double* b, double* r, double* norm2_dev) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        pd::pick(P)(P, 0, 3, x, b, r);
        if (norm2_dev) pd::norm2(P, r, P.len[0], norm2_dev);
    });
}

/* one outer block-Jacobi-in-time sweep: x += ω_t · Vcycle(b − L x) */
int pd_pfast_sweep(void* plan, const double* b, double* x) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        pd::pick(P)(P, 0, 3, x, b, P.B[0].p);
        if (!pd::vcycle(P, 0, x)) {
            pd::launch(pd::k_pf_axpy, P.c.grid_for(P.len[0], pd::PFB, 8), pd::PFB, 0, P.c.stream,
                       P.len[0], P.omega_t, (const double*)P.E[0].p, x);
            PD_LAUNCH_CHECK();
        }
    });
}

/* sweeps until |b − L x| <= max(tol_abs, tol_rel |b − L x0|) (multigrid.py:275-305
 * stopping and divergence rules); hist (host, max_sweeps + 1) optional */
int pd_pfast_solve(void* plan, const double* b, double* x, double tol_rel, double tol_abs,
                   int max_sweeps, pd_solve_report* rep, double* hist) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        const auto op = pd::pick(P);
        auto resid = [&]() {
            op(P, 0, 3, x, b, P.B[0].p);
            pd::norm2(P, P.B[0].p, P.len[0], P.norm.p);
            PD_CUDA(cudaMemcpyAsync(P.pinned, P.norm.p, sizeof(double), cudaMemcpyDeviceToHost,
                                    P.c.stream));
            PD_CUDA(cudaStreamSynchronize(P.c.stream));
            return std::sqrt(*P.pinned);
        };
        double r = resid();
        if (!std::isfinite(r)) throw pd::SolverError("non-finite initial residual", -1);
        const double thr = std::max(tol_abs, tol_rel * r);
        double lowest = r;
        int it = 0, conv = 0, div = 0;
        if (hist) hist[0] = r;
        while (true) {
            if (r <= thr) { conv = 1; break; }
            if (it >= max_sweeps) { div = 1; break; }
            if (!pd::vcycle(P, 0, x)) {
                pd::launch(pd::k_pf_axpy, P.c.grid_for(P.len[0], pd::PFB, 8), pd::PFB, 0,
                           P.c.stream, P.len[0], P.omega_t, (const double*)P.E[0].p, x);
                PD_LAUNCH_CHECK();
            }
            ++it;
            r = resid();
            if (hist) hist[it] = r;
            if (!std::isfinite(r)) throw pd::SolverError("non-finite residual in P-fast sweep", it);
            lowest = std::min(lowest, r);
            if (r > 10.0 * lowest) { div = 1; break; }
        }
        rep->iterations = it;
        rep->converged = conv;
        rep->diverged = div;
        rep->hist_len = hist ? it + 1 : 0;
    });
}

int pd_pfast_set_halo(void* plan, const double* halo) {
    return guarded_pf([&] { static_cast<pd::PfastPlan*>(plan)->halo = halo; });
}

int pd_pfast_destroy(void* plan) {
    return guarded_pf([&] { delete static_cast<pd::PfastPlan*>(plan); });
}

}  // extern "C"
