// Pointwise kernels of the space-time residual/Jacobian (spacetime.py:44-50,
// 131-151): reactions r(u) and r'(u) and the fused residual assembly
//   F = L u + gamma * (I (x) Mqh) r(u) - rhs
// on CSR operators (the general, operator-agnostic path; the matrix-free
// stencil path lives in pd_stencil.cu).
#include "../../include/paradiff_b200.h"
#include "pd_device.cuh"
#include "pd_internal.h"

namespace pd {
using namespace dev;

// kind 0: none, 1: cubic u^3 - u (reference), 2: Fisher u^2 - u (BASELINE C3)
__device__ __forceinline__ double react(int kind, double u) {
    if (kind == 1) return sub(mul(mul(u, u), u), u);
    if (kind == 2) return sub(mul(u, u), u);
    return 0.0;
}
__device__ __forceinline__ double react_deriv(int kind, double u) {
    if (kind == 1) return sub(mul(3.0, mul(u, u)), 1.0);
    if (kind == 2) return sub(mul(2.0, u), 1.0);
    return 0.0;
}

__global__ void k_reaction(int kind, int deriv, const double* u, double* out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = deriv ? react_deriv(kind, u[i]) : react(kind, u[i]);
}

// out = out + gamma * t   (residual accumulation, reference `res += gamma*(...)`)
__global__ void k_add_scaled(double* out, const double* t, double gamma, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = add(out[i], mul(gamma, t[i]));
}

// y = x + s * d   (Newton trial point u + step*delta)
__global__ void k_axpy_to(double* y, const double* x, const double* d, double s, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = add(x[i], mul(s, d[i]));
}

__global__ void k_scale(double* y, const double* x, double s, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = mul(s, x[i]);
}

}  // namespace pd

namespace {
template <class F>
int guarded_vec(F&& f) {
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

int pd_reaction(void* ctx, int kind, int deriv, const double* u, double* out, int64_t n) {
    return guarded_vec([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        if (kind < 0 || kind > 2) throw pd::ConfigError("unknown reaction kind");
        if (n > 0) pd::launch(pd::k_reaction, c.grid_for(n, 256), 256, 0, c.stream, kind, deriv, u, out, n);
        PD_LAUNCH_CHECK();
    });
}

// F = L u - rhs + gamma * MR r(u); tmp holds n doubles of scratch.
int pd_st_residual_csr(void* ctx, void* L, void* MR, double gamma, int kind, const double* u,
                       const double* rhs, double* out, double* tmp) {
    return guarded_vec([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        auto& A = *static_cast<pd::Csr*>(L);
        const int64_t n = A.nrows;
        pd::csr_spmv(c, A, u, out, pd::SPMV_SET, nullptr);
        // out = L u - rhs  (as  -(rhs - L u) would round identically)
        if (gamma != 0.0 && MR) {
            auto& R = *static_cast<pd::Csr*>(MR);
            pd::launch(pd::k_reaction, c.grid_for(n, 256), 256, 0, c.stream, kind, 0, u, tmp, n);
            pd::csr_spmv(c, R, tmp, tmp + n, pd::SPMV_SET, nullptr);
            pd::launch(pd::k_add_scaled, c.grid_for(n, 256), 256, 0, c.stream, out, tmp + n, gamma, n);
        }
        pd::launch(pd::k_add_scaled, c.grid_for(n, 256), 256, 0, c.stream, out, rhs, -1.0, n);
        PD_LAUNCH_CHECK();
    });
}

int pd_axpy_to(void* ctx, double* y, const double* x, const double* d, double s, int64_t n) {
    return guarded_vec([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        if (n > 0) pd::launch(pd::k_axpy_to, c.grid_for(n, 256), 256, 0, c.stream, y, x, d, s, n);
        PD_LAUNCH_CHECK();
    });
}

}  // extern "C"

extern "C" {

// host_out = ||x||_2 (deterministic device reduction; synchronising)
int pd_norm(void* ctx, const double* x, int64_t n, double* host_out) {
    return guarded_vec([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        *host_out = pd::vec_norm_host(c, x, n);
    });
}

// host_out = x . y (the same deterministic two-stage reduction; synchronising)
int pd_dot(void* ctx, const double* x, const double* y, int64_t n, double* host_out) {
    return guarded_vec([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        double h = 0.0;
        if (n > 0) {
            pd::vec_dot(c, x, y, n, c.scalars.p);
            PD_CUDA(cudaMemcpyAsync(&h, c.scalars.p, sizeof(double), cudaMemcpyDeviceToHost,
                                    c.stream));
            PD_CUDA(cudaStreamSynchronize(c.stream));
        }
        *host_out = h;
    });
}

// y = s * x
int pd_scale(void* ctx, double* y, const double* x, double s, int64_t n) {
    return guarded_vec([&] {
        auto& c = *static_cast<pd::Ctx*>(ctx);
        if (n > 0) pd::launch(pd::k_scale, c.grid_for(n, 256), 256, 0, c.stream, y, x, s, n);
        PD_LAUNCH_CHECK();
    });
}

}  // extern "C"
