// Microbenchmark: per-step cost of the wavefront executor's skeleton pieces on
// one CTA of 768 threads (64 CTAs, like the C2 fine-level lower sweep).
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(768, 1) k(double* y, const unsigned char* blob, size_t bytes,
                                            int steps, long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long bar[3];
    const int t = threadIdx.x;
    if (t == 0) for (int i = 0; i < 3; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const long long c0 = clock64();
    double acc = t;
    auto issue = [&](int s) {
        unsigned st = s % 3;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"((unsigned)bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + st * bytes)), "l"(blob + ((size_t)blockIdx.x * steps + s) % 64 * bytes), "r"((unsigned)bytes), "r"(smem_u32(&bar[st])) : "memory");
    };
    if (MODE & 4) { if (t == 0) { issue(0); issue(1); } }
    for (int s = 0; s < steps; ++s) {
        if (MODE & 4) {
            if (t == 0 && s + 2 < steps) issue(s + 2);
            unsigned st = s % 3, par = (s / 3) & 1;
            asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar[st])), "r"(par) : "memory");
            acc += reinterpret_cast<const double*>(sm + st * bytes)[t];
        }
        if (MODE & 2) {
            double* p = y + ((size_t)blockIdx.x * 765 + t) * 257 + s;
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(acc)) : "memory");
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p + 100000000), "l"(__double_as_longlong(acc)) : "memory");
        }
        if (MODE & 8) {  // 13-entry dependent fp64 chain with smem loads
            double* r = reinterpret_cast<double*>(sm + 160000);
#pragma unroll
            for (int k2 = 0; k2 < 13; ++k2) acc = __dadd_rn(acc, -__dmul_rn(r[(t + k2 * 37) % 1024], 1.0000001));
            r[t] = acc;
        }
        if (MODE & 1) __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = clock64() - c0;
    if (acc == 12345.0) y[0] = acc;
}

int main() {
    const int steps = 513, ctas = 64;
    const size_t bytes = 50560;
    double* y; unsigned char* blob; long long* out;
    cudaMalloc(&y, 2ull * 100000000 * 8 + 64ull * 765 * 257 * 8 * 2);
    cudaMalloc(&blob, 64 * bytes);
    cudaMemset(blob, 0, 64 * bytes);
    cudaMalloc(&out, ctas * 8);
    size_t smem = 3 * bytes + 1024 * 8 + 16384;
    long long h[64];
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int rep = 0; rep < 3; ++rep) kern<<<ctas, 768, smem>>>(y, blob, bytes, steps, out);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<ctas, 768, smem>>>(y, blob, bytes, steps, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-34s %8.1f ns/step  (%lld cycles/step) err=%s\n", name, ms * 1e6 / steps, h[0] / steps,
               cudaGetErrorString(cudaGetLastError()));
    };
    run(k<1>, "barrier");
    run(k<3>, "barrier+2 strong stores");
    run(k<5>, "barrier+TMA 50KB/step");
    run(k<9>, "barrier+13-entry fp64 chain");
    run(k<15>, "all");
    run(k<13>, "barrier+TMA+chain");
    return 0;
}
