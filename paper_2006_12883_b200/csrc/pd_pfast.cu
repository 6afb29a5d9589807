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
// Round 2: (a) the Newton linearisation J = L + γ(I⊗Mqh)diag(r'(u))
// (spacetime.py:126-129,144-151) enters the point blocks through a per-point
// weight array W = γ·dt·h^d·r'(u) (NL kernels: block = Ac(I + G·diag(w)), G = Ac⁻¹Mq,
// solved per point in registers) and MODE 5 evaluates the nonlinear residual
// (spacetime.py:131-142); (b) `PfastSt`: the space-time V-cycle around the
// smoother — time halved on every level, space while μ = κ·dt/h² allows it
// (schedule built by the host, pfast.st_schedule), rediscretised operators,
// time transfers = the coarse element's polynomial at the fine elements' nodes.
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
    double Ainv[kPfMaxM * kPfMaxM];  // Ac⁻¹ (NL: first half of the block solve)
    double G[kPfMaxM * kPfMaxM];     // Ac⁻¹·Mq (NL: block = Ac(I + G·diag(w)))
    double Mq[kPfMaxM * kPfMaxM];    // NL apply / MODE 5: Σ_k Mq[m,k]·(w_k x_k | r(x_k))
    double omega_s;                  // spatial damping (NL)
    double rs;                       // MODE 5: γ·dt·h^d
    int kind;                        // MODE 5: 0 cubic u³−u, 1 Fisher u²−u
};

struct PfTime {  // time transfers between space-time levels (row-major M×M)
    double P1[kPfMaxM * kPfMaxM];  // coarse polynomial at the first fine element's nodes
    double P2[kPfMaxM * kPfMaxM];  // ... at the second fine element's nodes
    double E[kPfMaxM * kPfMaxM];   // fine cardinal values at coarse node m
    int half[kPfMaxM];             // coarse node m lies in fine element 2tc + half[m]
};

// d = ω_s (I + G diag(w))⁻¹ Ac⁻¹ r: unrolled elimination without pivoting (the host
// checks ‖G‖∞·max|w| < 1, so the matrix is strictly diagonally dominant)
template <int M>
__device__ __forceinline__ void nl_block_solve(const PfCoef& C, const double (&w)[M],
                                               const double (&r)[M], double (&d)[M]) {
    double B[M][M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            acc = fma(C.Ainv[m * M + k], r[k], acc);
            B[m][k] = fma(C.G[m * M + k], w[k], m == k ? 1.0 : 0.0);
        }
        d[m] = acc;
    }
#pragma unroll
    for (int c = 0; c < M; ++c) {
        const double inv = 1.0 / B[c][c];
#pragma unroll
        for (int i = c + 1; i < M; ++i) {
            const double f = B[i][c] * inv;
#pragma unroll
            for (int k = c + 1; k < M; ++k) B[i][k] = fma(-f, B[c][k], B[i][k]);
            d[i] = fma(-f, d[c], d[i]);
        }
    }
#pragma unroll
    for (int c = M - 1; c >= 0; --c) {
        double acc = d[c];
#pragma unroll
        for (int k = c + 1; k < M; ++k) acc = fma(-B[c][k], d[k], acc);
        d[c] = acc / B[c][c];
    }
#pragma unroll
    for (int m = 0; m < M; ++m) d[m] *= C.omega_s;
}

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
// MODE 5: out = b − A x − cprev·x[t-1, M-1] − rs·Mq r(x)  (nonlinear residual −F(x))
// NL: A and the point block carry the linearisation weights W (same layout as x)
template <int DIM, int M, int MODE, bool PER, bool NL>
__global__ void __launch_bounds__(PFB) k_pf_point(PfCoef C, int n, int64_t nt,
                                                 const double* __restrict__ x,
                                                 const double* __restrict__ b, double* out,
                                                 const double* __restrict__ halo,
                                                 const double* __restrict__ W) {
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
        double wv[M];
        if (NL) {
#pragma unroll
            for (int m = 0; m < M; ++m) wv[m] = W[base + m * S];
        }
        if (MODE == 1) {
            if (NL) {
                double d[M];
                nl_block_solve<M>(C, wv, bv, d);
#pragma unroll
                for (int m = 0; m < M; ++m) out[base + m * S] = d[m];
                continue;
            }
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
                if (NL) ax = fma(C.Mq[m * M + k], wv[k] * xc[k], ax);
            }
            r[m] = bv[m] - ax;
        }
        if (MODE == 5) {
            double rx[M];
#pragma unroll
            for (int k = 0; k < M; ++k)
                rx[k] = C.kind == 0 ? xc[k] * xc[k] * xc[k] - xc[k] : xc[k] * xc[k] - xc[k];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(C.Mq[m * M + k], rx[k], acc);
                r[m] = fma(-C.rs, acc, r[m]);
            }
        }
        if ((MODE == 3 || MODE == 5) && (t > 0 || halo)) {
            // x[t-1, M-1, j]; the first step of a time slab reads the previous
            // slab's last node (halo) when the steps are sharded over ranks
            const double xp = t > 0 ? x[base - S] : halo[j];
#pragma unroll
            for (int m = 0; m < M; ++m) r[m] = fma(-C.cprev[m], xp, r[m]);
        }
        if (MODE == 2 || MODE == 3 || MODE == 5) {
#pragma unroll
            for (int m = 0; m < M; ++m) out[base + m * S] = r[m];
        } else {
            double d[M];
            if (NL) nl_block_solve<M>(C, wv, r, d);
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double acc = xc[m];
                if (NL) {
                    acc += d[m];
                } else {
#pragma unroll
                    for (int k = 0; k < M; ++k) acc = fma(C.Dinv[m * M + k], r[k], acc);
                }
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

// ---- periodic grids with nc a multiple of 32: pair-per-lane transfers ----
// A lane owns the fine pair (2cx, 2cx+1) of its coarse point cx: one 16-byte access per
// fine row and pair, the x neighbour from the adjacent lane by shuffle (the edge lane
// loads it, wrapping around the row).  The general kernels above issue up to 8 scalar
// coarse loads per fine point (prolongation) / 27 scalar fine loads per coarse point
// (restriction): they run at the L1 request rate, not at the HBM rate.

// fine += P coarse.  A warp takes the coarse cell (cz, cy) x one 32-point chunk of cx and
// updates its 2 x 2 fine rows (2D: 2 fine rows) from the 2 x 2 coarse rows read once.
template <int DIM>
__global__ void __launch_bounds__(PFB) k_pf_prolong_add_pp(int nc, int64_t planes,
                                                          const double* __restrict__ coarse,
                                                          double* fine) {
    const int nf = 2 * nc;
    const int64_t Sc = DIM == 2 ? (int64_t)nc * nc : (int64_t)nc * nc * nc;
    const int64_t Sf = DIM == 2 ? (int64_t)nf * nf : (int64_t)nf * nf * nf;
    const unsigned chunks = (unsigned)nc >> 5;
    const unsigned G = (DIM == 2 ? (unsigned)nc : (unsigned)nc * nc) * chunks;  // units per plane
    const unsigned units = (unsigned)planes * G;
    const int lane = threadIdx.x & 31;
    constexpr int NZ = DIM == 3 ? 2 : 1;
    for (unsigned unit = blockIdx.x * (PFB / 32) + (threadIdx.x >> 5); unit < units;
         unit += gridDim.x * (PFB / 32)) {
        const unsigned p_u = unit / G;
        unsigned rr = unit - p_u * G;
        const int ch = (int)(rr % chunks);
        rr /= chunks;
        const int cy = DIM == 2 ? (int)rr : (int)(rr % (unsigned)nc);
        const int cz = DIM == 3 ? (int)(rr / (unsigned)nc) : 0;
        const int cy1 = cy + 1 == nc ? 0 : cy + 1, cz1 = cz + 1 == nc ? 0 : cz + 1;
        const int cx = ch * 32 + lane;
        const int cxn = cx + 1 == nc ? 0 : cx + 1;
        const double* src = coarse + (int64_t)p_u * Sc;
        // coarse rows [z][y] at cx, and at cx + 1 (neighbour lane; the last lane loads it)
        double c[NZ][2], cn[NZ][2];
#pragma unroll
        for (int a = 0; a < NZ; ++a)
#pragma unroll
            for (int bb = 0; bb < 2; ++bb) {
                const double* row = src + ((int64_t)(a ? cz1 : cz) * (DIM == 3 ? nc : 0) +
                                           (bb ? cy1 : cy)) * nc;
                c[a][bb] = __ldg(row + cx);
                cn[a][bb] = __shfl_down_sync(0xffffffffu, c[a][bb], 1);
                if (lane == 31) cn[a][bb] = __ldg(row + cxn);
            }
        double* dst = fine + (int64_t)p_u * Sf;
#pragma unroll
        for (int j = 0; j < NZ; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                // interpolated coarse row for fine (z = 2cz + j, y = 2cy + i) at cx and cx + 1
                double r, rn;
                if (DIM == 2 || j == 0) {
                    r = i ? 0.5 * (c[0][0] + c[0][1]) : c[0][0];
                    rn = i ? 0.5 * (cn[0][0] + cn[0][1]) : cn[0][0];
                } else {
                    r = i ? 0.25 * ((c[0][0] + c[0][1]) + (c[NZ - 1][0] + c[NZ - 1][1]))
                          : 0.5 * (c[0][0] + c[NZ - 1][0]);
                    rn = i ? 0.25 * ((cn[0][0] + cn[0][1]) + (cn[NZ - 1][0] + cn[NZ - 1][1]))
                           : 0.5 * (cn[0][0] + cn[NZ - 1][0]);
                }
                double2* q = reinterpret_cast<double2*>(
                    dst + ((int64_t)(2 * cz + j) * (DIM == 3 ? nf : 0) + (2 * cy + i)) * nf + 2 * cx);
                double2 v = *q;
                v.x += r;
                v.y += 0.5 * (r + rn);
                *q = v;
            }
    }
}

// coarse = P^T fine.  A warp takes the coarse row (cz, cy) x one 32-point chunk of cx: the
// 3 x 3 (2D: 3) fine rows are combined per lane pair first, then in x with one shuffle.
template <int DIM>
__global__ void __launch_bounds__(PFB) k_pf_restrict_pp(int nc, int64_t planes,
                                                       const double* __restrict__ fine,
                                                       double* coarse) {
    const int nf = 2 * nc;
    const int64_t Sc = DIM == 2 ? (int64_t)nc * nc : (int64_t)nc * nc * nc;
    const int64_t Sf = DIM == 2 ? (int64_t)nf * nf : (int64_t)nf * nf * nf;
    const unsigned chunks = (unsigned)nc >> 5;
    const unsigned G = (DIM == 2 ? (unsigned)nc : (unsigned)nc * nc) * chunks;
    const unsigned units = (unsigned)planes * G;
    const int lane = threadIdx.x & 31;
    constexpr int NZ = DIM == 3 ? 3 : 1;
    for (unsigned unit = blockIdx.x * (PFB / 32) + (threadIdx.x >> 5); unit < units;
         unit += gridDim.x * (PFB / 32)) {
        const unsigned p_u = unit / G;
        unsigned rr = unit - p_u * G;
        const int ch = (int)(rr % chunks);
        rr /= chunks;
        const int cy = DIM == 2 ? (int)rr : (int)(rr % (unsigned)nc);
        const int cz = DIM == 3 ? (int)(rr / (unsigned)nc) : 0;
        const int cx = ch * 32 + lane;
        const int fxm = cx == 0 ? nf - 1 : 2 * cx - 1;  // wrapped left neighbour of the pair
        int fy[3], fz[3];
        fy[0] = cy == 0 ? nf - 1 : 2 * cy - 1; fy[1] = 2 * cy; fy[2] = 2 * cy + 1;
        fz[0] = cz == 0 ? nf - 1 : 2 * cz - 1; fz[1] = 2 * cz; fz[2] = 2 * cz + 1;
        const double* src = fine + (int64_t)p_u * Sf;
        const double w3[3] = {0.5, 1.0, 0.5};
        double ax = 0.0, ay = 0.0, am = 0.0;  // combined rows at 2cx, 2cx+1 and 2cx-1
#pragma unroll
        for (int a = 0; a < NZ; ++a)
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
                const double w = (DIM == 3 ? w3[a] : 1.0) * w3[bb];
                const double* row = src + ((int64_t)(DIM == 3 ? fz[a] : 0) * nf + fy[bb]) * nf;
                const double2 v = __ldg(reinterpret_cast<const double2*>(row + 2 * cx));
                double left = __shfl_up_sync(0xffffffffu, v.y, 1);
                if (lane == 0) left = __ldg(row + fxm);
                ax = fma(w, v.x, ax);
                ay = fma(w, v.y, ay);
                am = fma(w, left, am);
            }
        coarse[(int64_t)p_u * Sc + ((int64_t)cz * (DIM == 3 ? nc : 0) + cy) * nc + cx] =
            fma(0.5, am, fma(0.5, ay, ax));
    }
}

__global__ void __launch_bounds__(PFB) k_pf_axpy(int64_t n, double a, const double* __restrict__ e,
                                                double* x) {
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PFB)
        x[i] = fma(a, e[i], x[i]);
}

// W = rs·r'(u) (linearisation weights, spacetime.py:48-50,126-129) and max|W|
// (bit pattern of a non-negative double orders like an unsigned integer)
__global__ void __launch_bounds__(PFB) k_pf_weights(int64_t n, double rs, int kind,
                                                   const double* __restrict__ u, double* W,
                                                   unsigned long long* wmax) {
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PFB) {
        const double v = u[i];
        const double w = rs * (kind == 0 ? fma(3.0 * v, v, -1.0) : fma(2.0, v, -1.0));
        W[i] = w;
        mx = fmax(mx, fabs(w));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(wmax, (unsigned long long)__double_as_longlong(mx));
}

__global__ void __launch_bounds__(PFB) k_pf_absmax(int64_t n, const double* __restrict__ w,
                                                  unsigned long long* wmax) {
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PFB)
        mx = fmax(mx, fabs(w[i]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(wmax, (unsigned long long)__double_as_longlong(mx));
}

// Time transfers between space-time levels; vectors (nt, M, S), one thread per
// (coarse step, point).
// KIND 0 (residual restriction):  out[tc,m] = Σ_k P1[k,m]·in[2tc,k] + P2[k,m]·in[2tc+1,k]
// KIND 1 (weights):               out[tc,m] = 2 Σ_k E[m,k]·in[2tc+half[m],k]
template <int M, int KIND>
__global__ void __launch_bounds__(PFB) k_pf_tcombine(PfTime T, int64_t ntc, int64_t S,
                                                    const double* __restrict__ in, double* out) {
    const int64_t total = ntc * S;
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * PFB) {
        const int64_t tc = i / S, j = i - tc * S;
        double a[M], c[M];
#pragma unroll
        for (int k = 0; k < M; ++k) {
            a[k] = in[((2 * tc) * M + k) * S + j];
            c[k] = in[((2 * tc + 1) * M + k) * S + j];
        }
#pragma unroll
        for (int m = 0; m < M; ++m) {
            double acc = 0.0;
            if (KIND == 0) {
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(T.P1[k * M + m], a[k], acc);
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(T.P2[k * M + m], c[k], acc);
            } else {
#pragma unroll
                for (int k = 0; k < M; ++k) acc = fma(T.E[m * M + k], T.half[m] ? c[k] : a[k], acc);
                acc *= 2.0;
            }
            out[(tc * M + m) * S + j] = acc;
        }
    }
}

// prolongation in time: fine[2tc+s, m] (+)= Σ_k P{s}[m,k]·coarse[tc,k], s = 0, 1
template <int M, bool ADD>
__global__ void __launch_bounds__(PFB) k_pf_texpand(PfTime T, int64_t ntc, int64_t S,
                                                   const double* __restrict__ coarse,
                                                   double* fine) {
    const int64_t total = ntc * S;
    for (int64_t i = blockIdx.x * (int64_t)PFB + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * PFB) {
        const int64_t tc = i / S, j = i - tc * S;
        double e[M];
#pragma unroll
        for (int k = 0; k < M; ++k) e[k] = coarse[(tc * M + k) * S + j];
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < M; ++k)
                    acc = fma(s ? T.P2[m * M + k] : T.P1[m * M + k], e[k], acc);
                double* dst = fine + ((2 * tc + s) * M + m) * S + j;
                *dst = ADD ? *dst + acc : acc;
            }
    }
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
    double omega_t, dt, kappa, ginf = 0.0;  // ginf = ‖Ac⁻¹Mq‖∞ of level 0
    std::vector<int> n;            // grid points per axis per level
    std::vector<int64_t> len;      // nt·M·n^d per level
    std::vector<PfCoef> coef;
    std::vector<DevBuf<double>> B, E, T;  // level rhs, iterate, ping-pong
    std::vector<DevBuf<double>> W;        // linearisation weights per level (lazily allocated)
    bool nl = false;                      // weights active
    DevBuf<double> part, norm;
    DevBuf<unsigned long long> wmax;
    double* pinned = nullptr;
    PfastPlan(Ctx& c_) : c(c_) {}
    ~PfastPlan() {
        if (pinned) cudaFreeHost(pinned);
    }
    int64_t S(int l) const { return dim == 2 ? (int64_t)n[l] * n[l] : (int64_t)n[l] * n[l] * n[l]; }
};

namespace {

// One wave of resident blocks (grid-stride kernels): a grid of sms x 8 blocks
// with only 6 resident per SM left a second, mostly empty wave (ncu: achieved
// occupancy 52% of a theoretical 75%).
template <class K>
int one_wave(Ctx& c, K kernel, int64_t threads) {
    int occ = 0;
    PD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, PFB, 0));
    static const int cap = getenv("PD_PF_BLOCKS") ? atoi(getenv("PD_PF_BLOCKS")) : 0;
    if (cap > 0) occ = std::min(occ, cap);  // probe knob: fewer resident rows per SM
    return c.grid_for(threads, PFB, std::max(occ, 1));
}

template <int DIM, int M, bool PER, bool NL>
void launch_point(PfastPlan& P, int l, int mode, const double* x, const double* b, double* out,
                  const double* halo) {
    const int64_t nl = P.n[l];
    const int64_t rows = P.nt * (P.dim == 2 ? nl : nl * nl);
    const int64_t threads = rows * ((nl + 31) / 32) * 32;
    const PfCoef& C = P.coef[l];
    const double* W = NL ? P.W[l].p : nullptr;
    auto go = [&](auto kernel, const double* h) {
        launch(kernel, one_wave(P.c, kernel, threads), PFB, 0, P.c.stream, C, P.n[l], P.nt, x, b, out,
               h, W);
    };
    switch (mode) {
        case 0: go(k_pf_point<DIM, M, 0, PER, NL>, nullptr); break;
        case 1: go(k_pf_point<DIM, M, 1, PER, NL>, nullptr); break;
        case 2: go(k_pf_point<DIM, M, 2, PER, NL>, nullptr); break;
        case 4: go(k_pf_point<DIM, M, 4, PER, NL>, nullptr); break;
        case 5:
            if constexpr (!NL) go(k_pf_point<DIM, M, 5, PER, false>, halo);
            break;
        default: go(k_pf_point<DIM, M, 3, PER, NL>, halo);
    }
    PD_LAUNCH_CHECK();
}

// mode 5 (nonlinear residual) never uses the weights
template <int DIM, int M, bool PER>
void point_op(PfastPlan& P, int l, int mode, const double* x, const double* b, double* out,
              const double* halo) {
    if (P.nl && mode != 5) launch_point<DIM, M, PER, true>(P, l, mode, x, b, out, halo);
    else launch_point<DIM, M, PER, false>(P, l, mode, x, b, out, halo);
}

using PointFn = void (*)(PfastPlan&, int, int, const double*, const double*, double*,
                         const double*);

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

// coarse = Pᵀ fine over `planes` grids (nf → nc points per axis)
void restrict_planes(Ctx& c, int dim, bool periodic, int nc, int nf, int64_t planes,
                     const double* fine, double* coarse) {
    const int64_t rows = planes * (dim == 2 ? nc : (int64_t)nc * nc);
    auto go = [&](auto kernel) {
        launch(kernel, one_wave(c, kernel, rows * 32), PFB, 0, c.stream, nc, nf, planes, fine, coarse);
    };
    static const bool no_pp = getenv("PD_PF_NO_PAIR_TRANSFERS") != nullptr;
    if (periodic && nf == 2 * nc && nc % 32 == 0 && !no_pp) {
        auto gp = [&](auto kernel) {
            launch(kernel, one_wave(c, kernel, rows * 32), PFB, 0, c.stream, nc, planes, fine, coarse);
        };
        if (dim == 2) gp(k_pf_restrict_pp<2>);
        else gp(k_pf_restrict_pp<3>);
        PD_LAUNCH_CHECK();
        return;
    }
    if (dim == 2) {
        if (periodic) go(k_pf_restrict<2, true>);
        else go(k_pf_restrict<2, false>);
    } else {
        if (periodic) go(k_pf_restrict<3, true>);
        else go(k_pf_restrict<3, false>);
    }
    PD_LAUNCH_CHECK();
}

// fine += P coarse over `planes` grids
void prolong_add_planes(Ctx& c, int dim, bool periodic, int nc, int nf, int64_t planes,
                        const double* coarse, double* fine) {
    const int64_t rows = planes * (dim == 2 ? nf : (int64_t)nf * nf);
    auto go = [&](auto kernel) {
        launch(kernel, one_wave(c, kernel, rows * 32), PFB, 0, c.stream, nc, nf, planes, coarse, fine);
    };
    static const bool no_pp = getenv("PD_PF_NO_PAIR_TRANSFERS") != nullptr;
    if (periodic && nf == 2 * nc && nc % 32 == 0 && !no_pp) {
        const int64_t crows = planes * (dim == 2 ? nc : (int64_t)nc * nc);
        auto gp = [&](auto kernel) {
            launch(kernel, one_wave(c, kernel, crows * 32), PFB, 0, c.stream, nc, planes, coarse,
                   fine);
        };
        if (dim == 2) gp(k_pf_prolong_add_pp<2>);
        else gp(k_pf_prolong_add_pp<3>);
        PD_LAUNCH_CHECK();
        return;
    }
    if (dim == 2) {
        if (periodic) go(k_pf_prolong_add<2, true>);
        else go(k_pf_prolong_add<2, false>);
    } else {
        if (periodic) go(k_pf_prolong_add<3, true>);
        else go(k_pf_prolong_add<3, false>);
    }
    PD_LAUNCH_CHECK();
}

void restrict_to(PfastPlan& P, int l, const double* fine, double* coarse) {
    restrict_planes(P.c, P.dim, P.periodic, P.n[l + 1], P.n[l], P.nt * P.M, fine, coarse);
}

void prolong_add(PfastPlan& P, int l, const double* coarse, double* fine) {
    prolong_add_planes(P.c, P.dim, P.periodic, P.n[l + 1], P.n[l], P.nt * P.M, coarse, fine);
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
                op(P, l, 1, nullptr, b, e, nullptr);
            } else if (last && xupd && s == count - 1) {
                op(P, l, 4, e, b, xupd, nullptr);
                fused = true;
            } else {
                op(P, l, 0, e, b, t, nullptr);
                std::swap(e, t);
            }
        }
    };
    last = l == P.levels - 1;
    smooth(sweeps, true);
    if (l < P.levels - 1) {
        op(P, l, 2, e, b, t, nullptr);  // t = b − A e
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

// x += ω_t · Vcycle(b − L x); the residual is left in B[0]
void sweep(PfastPlan& P, const double* b, double* x, const double* halo) {
    pick(P)(P, 0, 3, x, b, P.B[0].p, halo);
    if (!vcycle(P, 0, x)) {
        launch(k_pf_axpy, P.c.grid_for(P.len[0], PFB, 8), PFB, 0, P.c.stream, P.len[0], P.omega_t,
               (const double*)P.E[0].p, x);
        PD_LAUNCH_CHECK();
    }
}

double read_scalar(PfastPlan& P, const double* dev) {
    PD_CUDA(cudaMemcpyAsync(P.pinned, dev, sizeof(double), cudaMemcpyDeviceToHost, P.c.stream));
    PD_CUDA(cudaStreamSynchronize(P.c.stream));
    return *P.pinned;
}

// max|W[0]| of a plan (synchronising)
double weights_absmax(PfastPlan& P) {
    PD_CUDA(cudaMemsetAsync(P.wmax.p, 0, sizeof(unsigned long long), P.c.stream));
    launch(k_pf_absmax, P.c.grid_for(P.len[0], PFB, 8), PFB, 0, P.c.stream, P.len[0],
           (const double*)P.W[0].p, P.wmax.p);
    PD_LAUNCH_CHECK();
    static_assert(sizeof(double) == sizeof(unsigned long long), "bit copy");
    return read_scalar(P, reinterpret_cast<const double*>(P.wmax.p));
}

void alloc_weights(PfastPlan& P) {
    if (!P.W.empty()) return;
    P.W.resize(P.levels);
    for (int l = 0; l < P.levels; ++l) P.W[l].alloc(P.len[l]);
}

// W[0] is set: restrict it down the spatial levels (Pᵀ W), check the point blocks
// stay diagonally dominant, switch the NL kernels on
void weights_ready(PfastPlan& P) {
    for (int l = 0; l + 1 < P.levels; ++l) restrict_to(P, l, P.W[l].p, P.W[l + 1].p);
    const double wm = weights_absmax(P);
    if (!(P.ginf * wm < 1.0))
        throw ConfigError("P-fast: reaction too stiff for the point-block solve "
                          "(|Ac^-1 Mq| max|gamma dt h^d r'(u)| >= 1); use fewer time levels");
    P.nl = true;
}

std::unique_ptr<PfastPlan> make_plan(Ctx& c, int dim, int64_t n, int bc_periodic, double kappa, int M,
                                     int64_t nt, double dt, const double* Kq, const double* Mq,
                                     const double* l0, int levels, int nu, int coarse_sweeps,
                                     double omega_s, double omega_t) {
    if (dim != 2 && dim != 3) throw ConfigError("P-fast needs a 2D or 3D grid");
    if (M < 1 || M > kPfMaxM) throw ConfigError("P-fast supports 1..5 nodes");
    if (nt < 1 || n < 1) throw ConfigError("P-fast needs nt >= 1 and n >= 1");
    if (levels < 1 || nu < 1 || coarse_sweeps < 1)
        throw ConfigError("P-fast needs levels, nu and coarse_sweeps >= 1");
    auto P = std::make_unique<PfastPlan>(c);
    P->dim = dim;
    P->M = M;
    P->nt = nt;
    P->dt = dt;
    P->kappa = kappa;
    P->levels = levels;
    P->nu = nu;
    P->coarse_sweeps = coarse_sweeps;
    P->periodic = bc_periodic != 0;
    P->omega_t = omega_t;
    int64_t nl = n;
    for (int l = 0; l < levels; ++l) {
        if (l > 0) {
            if (P->periodic) {
                if (nl % 2 || nl < 4) throw ConfigError("cannot coarsen the periodic grid");
                nl /= 2;
            } else {
                if (nl % 2 == 0 || nl < 3) throw ConfigError("cannot coarsen the Dirichlet grid");
                nl = (nl - 1) / 2;
            }
        }
        if (nl > (1 << 20)) throw ConfigError("grid too large");
        if (nt * M * nl * (dim == 3 ? nl : 1) * ((nl + 31) / 32) >= (int64_t(1) << 31))
            throw ConfigError("P-fast grid x steps too large for one plan");
        P->n.push_back((int)nl);
        int64_t S = nl * nl * (dim == 3 ? nl : 1);
        P->len.push_back(nt * M * S);
        // h of this level (StencilSpec.h: Dirichlet 1/(n+1), periodic 1/n)
        const double h = P->periodic ? 1.0 / (double)nl : 1.0 / (double)(nl + 1);
        const double mh = std::pow(h, dim);
        const double ks = kappa * std::pow(h, dim - 2);
        PfCoef C{};
        double D[kPfMaxM * kPfMaxM];
        for (int i = 0; i < M; ++i)
            for (int k = 0; k < M; ++k) {
                C.Ac[i * M + k] = Kq[i * M + k] * mh + dt * Mq[i * M + k] * (ks * 2.0 * dim);
                C.Ao[i * M + k] = -dt * Mq[i * M + k] * ks;
                C.Mq[i * M + k] = Mq[i * M + k];
                D[i * M + k] = C.Ac[i * M + k];
            }
        double Di[kPfMaxM * kPfMaxM];
        if (!invert(D, Di, M)) throw ConfigError("singular point block");
        double ginf = 0.0;
        for (int i = 0; i < M; ++i) {
            double rowsum = 0.0;
            for (int k = 0; k < M; ++k) {
                C.Dinv[i * M + k] = omega_s * Di[i * M + k];
                C.Ainv[i * M + k] = Di[i * M + k];
                double g = 0.0;
                for (int q = 0; q < M; ++q) g += Di[i * M + q] * Mq[q * M + k];
                C.G[i * M + k] = g;
                rowsum += std::fabs(g);
            }
            ginf = std::max(ginf, rowsum);
        }
        if (l == 0) P->ginf = ginf;
        for (int m = 0; m < M; ++m) C.cprev[m] = -l0[m] * mh;
        C.omega_t = omega_t;
        C.omega_s = omega_s;
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
    P->part.alloc(kPfNormBlocks);
    P->norm.alloc(1);
    P->wmax.alloc(1);
    PD_CUDA(cudaMallocHost(&P->pinned, sizeof(double)));
    return P;
}

// stopping / divergence rules of multigrid.py:275-305 around `step`
template <class Resid, class Step>
void iterate(Resid&& resid, Step&& step, double tol_rel, double tol_abs, int max_it,
             pd_solve_report* rep, double* hist) {
    double r = resid();
    int it = 0, conv = 0, div = 0;
    if (hist) hist[0] = r;
    if (!std::isfinite(r)) {
        div = 1;  // a non-finite residual reports divergence (multigrid.py:296-300), no throw
    } else {
        const double thr = std::max(tol_abs, tol_rel * r);
        double lowest = r;
        while (true) {
            if (r <= thr) { conv = 1; break; }
            if (it >= max_it) { div = 1; break; }
            step();
            ++it;
            r = resid();
            if (hist) hist[it] = r;
            if (!std::isfinite(r)) { div = 1; break; }
            lowest = std::min(lowest, r);
            if (r > 10.0 * lowest) { div = 1; break; }
        }
    }
    rep->iterations = it;
    rep->converged = conv;
    rep->diverged = div;
    rep->hist_len = hist ? it + 1 : 0;
}

}  // namespace

// Space-time multigrid around the smoother: level l has nt_l = nt_0 / 2^l steps of
// dt_l = 2^l dt_0 on an n_l^d grid (n_{l+1} = n_l or its 2:1 coarsening).
struct PfastSt {
    Ctx& c;
    int M = 0, dim = 0, nu_t = 1, coarse_t_sweeps = 1;
    bool periodic = false;
    PfTime T{};
    std::vector<std::unique_ptr<PfastPlan>> sm;  // one smoother (spatial hierarchy) per level
    std::vector<int> space;                      // space coarsened between l and l+1
    std::vector<DevBuf<double>> X, Bv;           // level iterates / right-hand sides, l >= 1
    explicit PfastSt(Ctx& c_) : c(c_) {}
};

namespace {

template <class F>
void for_m(int M, F&& f) {
    switch (M) {
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 3: f(std::integral_constant<int, 3>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        default: f(std::integral_constant<int, 5>{});
    }
}

// in (level l layout, or already space-restricted) -> level l+1, KIND as k_pf_tcombine
template <int KIND>
void time_combine(PfastSt& S, int l, const double* in, double* out) {
    PfastPlan& C = *S.sm[l + 1];
    const int64_t Sc = C.S(0), total = C.nt * Sc;
    for_m(S.M, [&](auto m) {
        constexpr int MM = decltype(m)::value;
        launch(k_pf_tcombine<MM, KIND>, S.c.grid_for(total, PFB, 8), PFB, 0, S.c.stream, S.T, C.nt, Sc,
               in, out);
    });
    PD_LAUNCH_CHECK();
}

// b_{l+1} = Rt Rs r_l; r_l = the level-l smoother's B[0]; T[0] is scratch
void st_restrict(PfastSt& S, int l, double* bc) {
    PfastPlan& F = *S.sm[l];
    const double* r = F.B[0].p;
    if (S.space[l]) {
        restrict_planes(S.c, S.dim, S.periodic, S.sm[l + 1]->n[0], F.n[0], F.nt * F.M, r, F.T[0].p);
        r = F.T[0].p;
    }
    time_combine<0>(S, l, r, bc);
}

// x_l += Ps Pt e_{l+1}
void st_prolong(PfastSt& S, int l, const double* ec, double* x) {
    PfastPlan& F = *S.sm[l];
    PfastPlan& C = *S.sm[l + 1];
    const int64_t Sc = C.S(0), total = C.nt * Sc;
    const bool sp = S.space[l] != 0;
    double* dst = sp ? F.T[0].p : x;
    for_m(S.M, [&](auto m) {
        constexpr int MM = decltype(m)::value;
        if (sp)
            launch(k_pf_texpand<MM, false>, S.c.grid_for(total, PFB, 8), PFB, 0, S.c.stream, S.T, C.nt,
                   Sc, ec, dst);
        else
            launch(k_pf_texpand<MM, true>, S.c.grid_for(total, PFB, 8), PFB, 0, S.c.stream, S.T, C.nt,
                   Sc, ec, dst);
    });
    PD_LAUNCH_CHECK();
    if (sp) prolong_add_planes(S.c, S.dim, S.periodic, C.n[0], F.n[0], F.nt * F.M, dst, x);
}

void st_cycle(PfastSt& S, int l, const double* b, double* x) {
    PfastPlan& P = *S.sm[l];
    const int L = (int)S.sm.size();
    if (l == L - 1) {
        for (int s = 0; s < S.coarse_t_sweeps; ++s) sweep(P, b, x, nullptr);
        return;
    }
    for (int s = 0; s < S.nu_t; ++s) sweep(P, b, x, nullptr);
    pick(P)(P, 0, 3, x, b, P.B[0].p, nullptr);
    st_restrict(S, l, S.Bv[l + 1].p);
    PD_CUDA(cudaMemsetAsync(S.X[l + 1].p, 0, S.sm[l + 1]->len[0] * sizeof(double), S.c.stream));
    st_cycle(S, l + 1, S.Bv[l + 1].p, S.X[l + 1].p);
    st_prolong(S, l, S.X[l + 1].p, x);
    for (int s = 0; s < S.nu_t; ++s) sweep(P, b, x, nullptr);
}

// weights of level 0 are set: all coarser space-time levels and spatial levels
void st_weights_ready(PfastSt& S) {
    const int L = (int)S.sm.size();
    for (int l = 0; l < L; ++l) {
        PfastPlan& F = *S.sm[l];
        if (l + 1 < L) {
            PfastPlan& C = *S.sm[l + 1];
            alloc_weights(C);
            const double* w = F.W[0].p;
            if (S.space[l]) {  // T[0] is scratch outside a sweep
                restrict_planes(S.c, S.dim, S.periodic, C.n[0], F.n[0], F.nt * F.M, w, F.T[0].p);
                w = F.T[0].p;
            }
            time_combine<1>(S, l, w, C.W[0].p);
        }
        weights_ready(F);
    }
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
        *out = pd::make_plan(c, dim, n, bc_periodic, kappa, M, nt, dt, Kq, Mq, l0, levels, nu,
                             coarse_sweeps, omega_s, omega_t)
                   .release();
    });
}

/* r = b − L x (or b − J x with weights set) at level 0; |r|^2 into *norm2_dev when
 * non-null; halo: the previous slab's last node (NULL: none) */
int pd_pfast_residual(void* plan, const double* x, const double* b, double* r, const double* halo,
                      double* norm2_dev) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        pd::pick(P)(P, 0, 3, x, b, r, halo);
        if (norm2_dev) pd::norm2(P, r, P.len[0], norm2_dev);
    });
}

/* out = rhs − L u − γ(I⊗Mqh) r(u) = −F(u) (spacetime.py:131-142); kind 0 cubic, 1 Fisher */
int pd_pfast_nl_residual(void* plan, const double* u, const double* rhs, double* out,
                         const double* halo, double gamma, int kind, double* norm2_dev) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        if (kind != 0 && kind != 1) throw pd::ConfigError("unknown reaction kind");
        const double h = P.periodic ? 1.0 / P.n[0] : 1.0 / (P.n[0] + 1);
        P.coef[0].rs = gamma * P.dt * std::pow(h, P.dim);
        P.coef[0].kind = kind;
        pd::pick(P)(P, 0, 5, u, rhs, out, halo);
        if (norm2_dev) pd::norm2(P, out, P.len[0], norm2_dev);
    });
}

/* Linearisation state: W = γ·dt·h^d·r'(u) on every spatial level (NULL u: back to
 * the linear operator).  Synchronising (checks the point blocks). */
int pd_pfast_set_state(void* plan, const double* u, double gamma, int kind) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        if (!u) {
            P.nl = false;
            return;
        }
        if (kind != 0 && kind != 1) throw pd::ConfigError("unknown reaction kind");
        pd::alloc_weights(P);
        const double h = P.periodic ? 1.0 / P.n[0] : 1.0 / (P.n[0] + 1);
        PD_CUDA(cudaMemsetAsync(P.wmax.p, 0, sizeof(unsigned long long), P.c.stream));
        pd::launch(pd::k_pf_weights, P.c.grid_for(P.len[0], pd::PFB, 8), pd::PFB, 0, P.c.stream,
                   P.len[0], gamma * P.dt * std::pow(h, P.dim), kind, u, P.W[0].p, P.wmax.p);
        PD_LAUNCH_CHECK();
        pd::weights_ready(P);
    });
}

/* one outer block-Jacobi-in-time sweep: x += ω_t · Vcycle(b − L x) */
int pd_pfast_sweep(void* plan, const double* b, double* x, const double* halo) {
    return guarded_pf([&] { pd::sweep(*static_cast<pd::PfastPlan*>(plan), b, x, halo); });
}

/* sweeps until |b − L x| <= max(tol_abs, tol_rel |b − L x0|) (multigrid.py:275-305
 * stopping and divergence rules); hist (host, max_sweeps + 1) optional */
int pd_pfast_solve(void* plan, const double* b, double* x, const double* halo, double tol_rel,
                   double tol_abs, int max_sweeps, pd_solve_report* rep, double* hist) {
    return guarded_pf([&] {
        auto& P = *static_cast<pd::PfastPlan*>(plan);
        auto resid = [&]() {
            pd::pick(P)(P, 0, 3, x, b, P.B[0].p, halo);
            pd::norm2(P, P.B[0].p, P.len[0], P.norm.p);
            return std::sqrt(pd::read_scalar(P, P.norm.p));
        };
        // the residual of resid() is still in B[0]: the sweep's V-cycle starts from it
        auto step = [&]() {
            if (!pd::vcycle(P, 0, x)) {
                pd::launch(pd::k_pf_axpy, P.c.grid_for(P.len[0], pd::PFB, 8), pd::PFB, 0,
                           P.c.stream, P.len[0], P.omega_t, (const double*)P.E[0].p, x);
                PD_LAUNCH_CHECK();
            }
        };
        pd::iterate(resid, step, tol_rel, tol_abs, max_sweeps, rep, hist);
    });
}

int pd_pfast_destroy(void* plan) {
    return guarded_pf([&] { delete static_cast<pd::PfastPlan*>(plan); });
}

/* ---- space-time multigrid around the smoother ---- */
int pd_pfast_st_create(void* ctx, int dim, int bc_periodic, double kappa, int M, const double* Kq,
                       const double* Mq, const double* l0, int nlevels, const int64_t* nt,
                       const int64_t* n, const double* dt, const int* space_levels,
                       const double* P1, const double* P2, const double* E, const int* half,
                       int nu_t, int coarse_t_sweeps, int nu, int coarse_sweeps, double omega_s,
                       double omega_t, void** out) {
    return guarded_pf([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        if (nlevels < 1 || nu_t < 1 || coarse_t_sweeps < 1)
            throw pd::ConfigError("P-fast STMG needs nlevels, nu_t and coarse_t_sweeps >= 1");
        auto S = std::make_unique<pd::PfastSt>(c);
        S->M = M;
        S->dim = dim;
        S->periodic = bc_periodic != 0;
        S->nu_t = nu_t;
        S->coarse_t_sweeps = coarse_t_sweeps;
        if (M < 1 || M > pd::kPfMaxM) throw pd::ConfigError("P-fast supports 1..5 nodes");
        for (int i = 0; i < M * M; ++i) {
            S->T.P1[i] = P1[i];
            S->T.P2[i] = P2[i];
            S->T.E[i] = E[i];
        }
        for (int m = 0; m < M; ++m) S->T.half[m] = half[m];
        S->X.resize(nlevels);
        S->Bv.resize(nlevels);
        for (int l = 0; l < nlevels; ++l) {
            const bool last = l == nlevels - 1;
            if (l > 0) {
                if (nt[l] * 2 != nt[l - 1]) throw pd::ConfigError("time levels must halve the steps");
                const int64_t nf = n[l - 1];
                const int64_t nc = S->periodic ? nf / 2 : (nf - 1) / 2;
                if (n[l] != nf && n[l] != nc) throw pd::ConfigError("bad space-time level grid");
                S->space.push_back(n[l] != nf);
            }
            // the coarsest level sweeps undamped (exact after nt sweeps for exact blocks)
            S->sm.push_back(pd::make_plan(c, dim, n[l], bc_periodic, kappa, M, nt[l], dt[l], Kq, Mq,
                                          l0, space_levels[l], nu, coarse_sweeps, omega_s,
                                          last ? 1.0 : omega_t));
            if (l > 0) {
                S->X[l].alloc(S->sm[l]->len[0]);
                S->Bv[l].alloc(S->sm[l]->len[0]);
            }
        }
        S->space.push_back(0);
        *out = S.release();
    });
}

int pd_pfast_st_destroy(void* st) {
    return guarded_pf([&] { delete static_cast<pd::PfastSt*>(st); });
}

/* linearisation state on every space-time and spatial level (NULL u: linear) */
int pd_pfast_st_set_state(void* st, const double* u, double gamma, int kind) {
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        if (!u) {
            for (auto& p : S.sm) p->nl = false;
            return;
        }
        if (kind != 0 && kind != 1) throw pd::ConfigError("unknown reaction kind");
        pd::PfastPlan& P = *S.sm[0];
        pd::alloc_weights(P);
        const double h = P.periodic ? 1.0 / P.n[0] : 1.0 / (P.n[0] + 1);
        PD_CUDA(cudaMemsetAsync(P.wmax.p, 0, sizeof(unsigned long long), P.c.stream));
        pd::launch(pd::k_pf_weights, P.c.grid_for(P.len[0], pd::PFB, 8), pd::PFB, 0, P.c.stream,
                   P.len[0], gamma * P.dt * std::pow(h, P.dim), kind, u, P.W[0].p, P.wmax.p);
        PD_LAUNCH_CHECK();
        pd::st_weights_ready(S);
    });
}

/* one V(nu_t, nu_t) space-time cycle on level 0 */
int pd_pfast_st_cycle(void* st, const double* b, double* x) {
    return guarded_pf([&] { pd::st_cycle(*static_cast<pd::PfastSt*>(st), 0, b, x); });
}

/* cycles until |b − J x| <= max(tol_abs, tol_rel |b − J x0|) (multigrid.py:275-305) */
int pd_pfast_st_solve(void* st, const double* b, double* x, double tol_rel, double tol_abs,
                      int max_cycles, pd_solve_report* rep, double* hist) {
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        pd::PfastPlan& P = *S.sm[0];
        auto resid = [&]() {
            pd::pick(P)(P, 0, 3, x, b, P.B[0].p, nullptr);
            pd::norm2(P, P.B[0].p, P.len[0], P.norm.p);
            return std::sqrt(pd::read_scalar(P, P.norm.p));
        };
        pd::iterate(resid, [&]() { pd::st_cycle(S, 0, b, x); }, tol_rel, tol_abs, max_cycles, rep,
                    hist);
    });
}

/* Level primitives for the time-slab sharded cycle (driven by pfast.py): b / x NULL
 * select the level's own vectors (levels >= 1). */
int pd_pfast_st_level_plan(void* st, int level, void** plan_out) { /* borrowed smoother */
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        if (level < 0 || level >= (int)S.sm.size()) throw pd::ConfigError("bad level");
        *plan_out = S.sm[level].get();
    });
}

int pd_pfast_st_level_sweep(void* st, int level, const double* b, double* x, const double* halo) {
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        if (level < 0 || level >= (int)S.sm.size()) throw pd::ConfigError("bad level");
        if (level == 0 && (!b || !x)) throw pd::ConfigError("level 0 vectors are the caller's");
        pd::sweep(*S.sm[level], b ? b : S.Bv[level].p, x ? x : S.X[level].p, halo);
    });
}

/* residual of the level into the smoother's B[0], restricted into level+1's right-hand
 * side; level+1's iterate is zeroed */
int pd_pfast_st_level_restrict(void* st, int level, const double* b, const double* x,
                               const double* halo) {
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        if (level < 0 || level + 1 >= (int)S.sm.size()) throw pd::ConfigError("bad level");
        if (level == 0 && (!b || !x)) throw pd::ConfigError("level 0 vectors are the caller's");
        pd::PfastPlan& P = *S.sm[level];
        pd::pick(P)(P, 0, 3, x ? x : S.X[level].p, b ? b : S.Bv[level].p, P.B[0].p, halo);
        pd::st_restrict(S, level, S.Bv[level + 1].p);
        PD_CUDA(cudaMemsetAsync(S.X[level + 1].p, 0, S.sm[level + 1]->len[0] * sizeof(double),
                                S.c.stream));
    });
}

int pd_pfast_st_level_prolong(void* st, int level, double* x) {
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        if (level < 0 || level + 1 >= (int)S.sm.size()) throw pd::ConfigError("bad level");
        if (level == 0 && !x) throw pd::ConfigError("level 0 vectors are the caller's");
        pd::st_prolong(S, level, S.X[level + 1].p, x ? x : S.X[level].p);
    });
}

/* copy the last node of the level's iterate (n_l^d doubles) into out (device) */
int pd_pfast_st_level_last(void* st, int level, const double* x, double* out) {
    return guarded_pf([&] {
        auto& S = *static_cast<pd::PfastSt*>(st);
        if (level < 0 || level >= (int)S.sm.size()) throw pd::ConfigError("bad level");
        if (level == 0 && !x) throw pd::ConfigError("level 0 vectors are the caller's");
        pd::PfastPlan& P = *S.sm[level];
        const double* src = (x ? x : S.X[level].p) + P.len[0] - P.S(0);
        PD_CUDA(cudaMemcpyAsync(out, src, P.S(0) * sizeof(double), cudaMemcpyDeviceToDevice,
                                S.c.stream));
    });
}

}  // extern "C"
