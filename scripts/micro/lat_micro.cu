// Single-warp latency microbenchmark for the wavefront step critical path:
// cycles per iteration of dependent fp64 add / mul+add / div chains and
// dependent shared-memory loads on B200 (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, long long* cyc) {
    __shared__ double sm[1024];
    __shared__ int si[1024];
    const int t = threadIdx.x;
    for (int i = t; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; si[i] = (i * 7 + 1) & 1023; }
    __syncthreads();
    double acc = t * 1e-3 + 1.0, d = 1.0000001;
    int idx = t;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) acc = __dadd_rn(acc, d);                       // dependent DADD
        if (MODE == 1) acc = __dsub_rn(acc, __dmul_rn(d, acc));       // dependent DMUL+DADD
        if (MODE == 2) acc = __dsub_rn(acc, __dmul_rn(d, sm[i & 1023]));  // independent loads, dep add
        if (MODE == 3) acc = acc / d;                                  // dependent DDIV
        if (MODE == 4) idx = si[idx];                                  // dependent LDS
        if (MODE == 5) { acc = __dadd_rn(acc, d); __syncthreads(); }   // add + barrier
        if (MODE == 6) acc = __fma_rn(acc, d, 1e-9);                   // dependent DFMA
    }
    const long long c1 = clock64();
    if (t == 0) *cyc = c1 - c0;
    out[t] = acc + idx;
}

int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    const int iters = 100000;
    auto run = [&](auto kern, const char* name) {
        kern<<<1, 32>>>(out, iters, cyc);
        kern<<<1, 32>>>(out, iters, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %6.1f cycles/iter  %s\n", name, (double)h / iters, cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0>, "dependent DADD");
    run(k<1>, "dependent DMUL+DSUB");
    run(k<2>, "LDS + DMUL + dep DSUB");
    run(k<3>, "dependent DDIV");
    run(k<4>, "dependent LDS");
    run(k<5>, "DADD + bar.sync (1 warp)");
    run(k<6>, "dependent DFMA");
    return 0;
}
