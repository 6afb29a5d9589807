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
#include <cstring>

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

void StOp::apply(const double* x, double* y, int mode, const double* b, const int* guard,
                 int want, double* norm2_out, int* nonfinite, const double* halo) const {
    const int64_t N = size();
    if (N <= 0) return;
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
