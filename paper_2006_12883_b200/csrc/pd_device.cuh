// Device-side helpers shared by the paradiff-b200 kernels (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace pd {
namespace dev {

// Guarded kernels: the device-resident solver state decides whether a
// launched kernel does anything, so whole V-cycles run without host syncs
// (and can be captured into CUDA graphs).
__device__ __forceinline__ bool guard_off(const int* guard, int want) {
    return guard != nullptr && *((volatile const int*)guard) != want;
}

// Loads that bypass L1 (values produced by other SMs inside the same launch).
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int64_t ldcg(const int64_t* p) {
    return (int64_t)__ldcg((const long long*)p);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Wait until every row in cols[p0, p1) has flag >= target.  The polls are
// independent relaxed loads (issued back to back, one L2 round trip per
// sweep over the dependencies) followed by a single acquire fence, instead of
// one acquire round trip per dependency.
__device__ __forceinline__ void wait_all(const int* flag, const int32_t* cols, int64_t p0,
                                         int64_t p1, int target) {
    unsigned int ns = 32;
    for (;;) {
        int ok = 1;
        for (int64_t p = p0; p < p1; ++p) ok &= (ld_relaxed(flag + cols[p]) >= target);
        if (ok) break;
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
    fence_acq_rel();
}

// Wait until flag >= target (monotone epochs).
__device__ __forceinline__ void wait_flag(const int* f, int target) {
    if (ld_acquire(f) >= target) return;
    unsigned int ns = 32;
    while (ld_acquire(f) < target) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

// Separately rounded multiply/subtract/add: keeps the reference's (non-FMA)
// rounding so CSR products and ILU factors reproduce scipy/numba bitwise.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// Deterministic block reduction (fixed tree) of one double.
template <int BS>
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (w == 0) {
        s = (lane < BS / 32) ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    }
    __syncthreads();
    return s;  // valid in thread 0
}

// block_sum for multi-dimensional blocks: `tid` is the linear thread index
template <int BS>
__device__ __forceinline__ double block_sum_flat(double v, double* sh, int tid) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = tid & 31, w = tid >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (w == 0) {
        s = (lane < BS / 32) ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    }
    __syncthreads();
    return s;  // valid in tid 0
}

// Grid-wide deterministic sum: each block writes its partial; the last block
// to arrive sums the partials in index order and stores *out (then resets the
// counter so the slot can be reused by the next kernel on the stream).
template <int BS>
__device__ __forceinline__ void grid_sum_finish(double v, double* partials, unsigned int* counter,
                                                double* out) {
    __shared__ double sh[BS / 32];
    __shared__ bool last;
    double s = block_sum<BS>(v, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = s;
        __threadfence();
        unsigned int prev = atomicAdd(counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = 0.0;
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += BS) t += __ldcg(partials + i);
    t = block_sum<BS>(t, sh);
    if (threadIdx.x == 0) {
        *out = t;
        *counter = 0u;
    }
}

// Value-as-flag words: a sweep output starts as this signalling-NaN payload and
// is published with one single-copy-atomic 64-bit store (pd_sparse.cu).
constexpr unsigned long long kPending = 0x7ff4a5a55a5a0001ull;  // signalling-NaN payload

__device__ __forceinline__ unsigned long long ld_strong_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_strong(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v))
                 : "memory");
}
__device__ __forceinline__ void st_pending(double* p) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(kPending) : "memory");
}


}  // namespace dev
}  // namespace pd
