// Skewed-wavefront ILU(0) sweeps for structured 2D space-time levels (v2).
//
// Rows of one time step are [node m][line y][point x] (paradiff/spacetime.py:
// 117-124 layout).  On the levels this kernel serves, every factor entry of row
// (m, y, x) couples to a compile-time template of neighbours:
//   FINE5  (fine level, 5-point Kh (x) dense M x M time block):
//          lower = prev step (M-1, y, x) | m' < m: 5-point | m' = m: (-1,0),(0,-1)
//   GAL9   (SMG Galerkin levels, 9-point (x) M x M, 3 x 3 coupling to the previous step):
//          lower = prev step 3 x 3 | m' < m: 3 x 3 | m' = m: (-1,-1),(-1,0),(-1,1),(0,-1)
// (the upper sweep mirrors both).  The host checks every row's entries against the
// template in CSR order; missing entries (grid boundary, block-Jacobi mask) are
// stored as zero factors, which leave the accumulation bitwise unchanged.
//
// Schedule: one CTA per time step, ONE THREAD PER LINE running all M nodes; row
// (m, y, x) runs at step s = x + SIG*y + KAP*m (sweep coordinates; the upper sweep
// mirrors x, y and m), with SIG/KAP chosen so that every source of a row was
// produced at an earlier step.  So the M rows a thread runs per step are
// independent, their sources come from a shared-memory ring (slot x mod R) written
// in earlier steps, and a step needs one __syncthreads.  Entries are evaluated in
// CSR order with separately rounded multiply/subtract (linalg.py:104-113): results
// are bitwise those of the numba reference.  Every source address is a ring base
// plus a compile-time immediate; factor values arrive per step by TMA bulk copies
// ([line][entry] rows with an odd stride: conflict-free LDS.64 at immediate offsets).
// The upper sweep's division uses a reciprocal computed off the chain plus one
// FMA correction (Markstein), which equals IEEE division for normal operands; zero,
// subnormal, huge and non-finite cases take the IEEE path.
//
// The previous time step's last node grid (lower sweep only, block-Jacobi
// partitions permitting) is produced by another CTA: it is polled from global
// memory with the value-as-flag protocol of pd_sparse.cu, two steps ahead, into a
// pseudo-node region of the ring.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pd {
using namespace dev;

namespace {

enum { kFine5 = 0, kGal9 = 1 };
constexpr int kMaxStages2 = 4;
constexpr int kPD = 4;  // previous-step values are loaded this many steps before use
constexpr int kStartLag = 0;  // extra steps a time step's CTA trails its predecessor
constexpr int kPB = kPD;  // right-hand-side values are loaded this many steps before use

struct TE {
    int node, dy, dx;  // sweep coordinates; node == M: previous-step pseudo node
};

__host__ __device__ constexpr int sig_of(int kind) { return kind == kFine5 ? 1 : 2; }
__host__ __device__ constexpr int kap_of(int kind) { return kind == kFine5 ? 2 : 4; }
__host__ __device__ constexpr int nb_of(int kind) { return kind == kFine5 ? 5 : 9; }
__host__ __device__ constexpr int nsame_of(int kind) { return kind == kFine5 ? 2 : 4; }
__host__ __device__ constexpr int nprev_of(int kind) { return kind == kFine5 ? 1 : 9; }
// pseudo values are written D steps before the row of the same (line, x) runs
__host__ __device__ constexpr int lead_of(int kind) { return kind == kFine5 ? 1 : 2 + sig_of(kind); }

// entries of a row at sweep node mb
__host__ __device__ constexpr int tmpl_len(bool upper, int kind, int M, int mb) {
    return upper ? nsame_of(kind) + mb * nb_of(kind)
                 : nprev_of(kind) + mb * nb_of(kind) + nsame_of(kind);
}
// padded row stride in the step block (odd: conflict-free 8-byte loads); the upper
// sweep stores the diagonal and its reciprocal after its entries
__host__ __device__ constexpr int tmpl_pad(bool upper, int kind, int M, int mb) {
    return (tmpl_len(upper, kind, M, mb) + (upper ? 2 : 0)) | 1;
}

__host__ __device__ constexpr TE block_entry(int kind, int k) {
    // k-th entry of an off-node block in ORIGINAL coordinates, CSR (dy, dx) order
    return kind == kFine5 ? (k == 0   ? TE{0, -1, 0}
                             : k == 1 ? TE{0, 0, -1}
                             : k == 2 ? TE{0, 0, 0}
                             : k == 3 ? TE{0, 0, 1}
                                      : TE{0, 1, 0})
                          : TE{0, k / 3 - 1, k % 3 - 1};
}

// j-th template entry of sweep node mb, in SWEEP coordinates
__host__ __device__ constexpr TE tmpl_entry(bool upper, int kind, int M, int mb, int j) {
    if (!upper) {
        const int np = nprev_of(kind), nb = nb_of(kind);
        if (j < np) return kind == kFine5 ? TE{M, 0, 0} : TE{M, j / 3 - 1, j % 3 - 1};
        const int jj = j - np;
        if (jj < mb * nb) {
            const TE e = block_entry(kind, jj % nb);
            return TE{jj / nb, e.dy, e.dx};
        }
        const int k = jj - mb * nb;  // same node, entries before the diagonal
        if (kind == kFine5) return k == 0 ? TE{mb, -1, 0} : TE{mb, 0, -1};
        return k < 3 ? TE{mb, -1, k - 1} : TE{mb, 0, -1};
    }
    // upper: original node m = M-1-mb; same node after the diagonal, then the
    // blocks of original nodes m+1 .. M-1 (sweep nodes mb-1 .. 0); mirrored offsets
    const int ns = nsame_of(kind), nb = nb_of(kind);
    if (j < ns) {
        TE o = kind == kFine5 ? (j == 0 ? TE{0, 0, 1} : TE{0, 1, 0})
                              : (j == 0 ? TE{0, 0, 1} : TE{0, 1, j - 2});
        return TE{mb, -o.dy, -o.dx};
    }
    const int jj = j - ns;
    const TE e = block_entry(kind, jj % nb);
    return TE{mb - 1 - jj / nb, -e.dy, -e.dx};
}

__host__ __device__ constexpr int imax(int a, int b) { return a > b ? a : b; }
// ring depth (power of two) > the longest lifetime of a ring slot in steps
__host__ __device__ constexpr int ring_need(bool upper, int kind, int M) {
    // regular node m': last read by node M-1 at (dy, dx) = (-1, -1) relative
    //   -> 1 + SIG + KAP (M-1) steps after it was written (m' = 0)
    // pseudo: written lead steps before its first reader; last read as above
    return upper ? 1 + sig_of(kind) + kap_of(kind) * (M - 1)
                 : (kind == kFine5 ? imax(1 + sig_of(kind) + kap_of(kind) * (M - 1),
                                          lead_of(kind) + kap_of(kind) * (M - 1))
                                   : imax(1 + sig_of(kind) + kap_of(kind) * (M - 1),
                                          lead_of(kind) + 1 + sig_of(kind) + kap_of(kind) * (M - 1)));
}
__host__ __device__ constexpr int pow2_above(int v) {  // smallest power of two > v
    int r = 1;
    while (r <= v) r <<= 1;
    return r;
}
__host__ __device__ constexpr int ring_depth(bool upper, int kind, int M) {
    return pow2_above(ring_need(upper, kind, M));
}

struct Wf2Dev {
    int* prog;                  // per task: last completed step (lower sweep), -1 before
    unsigned long long* trace;  // PD_WF2_TRACE: per task {t0, t1, wait_stage, wait_bar, wait_poll}
    const double* blob;
    const int32_t* stepoff;
    const unsigned char* hasprev;
    int64_t task_stride;
    int ntask, NS, NL, NX, S, stages;
    unsigned stage_bytes;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_copy(unsigned dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    constexpr unsigned kPieces = 4;
    const unsigned piece = ((bytes + kPieces - 1) / kPieces + 15) & ~15u;
    for (unsigned o = 0; o < bytes; o += piece) {
        const unsigned nb = min(piece, bytes - o);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(dst + o),
            "l"(static_cast<const char*>(src) + o), "r"(nb), "r"(smem_u32(bar))
            : "memory");
    }
}
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
    if (bytes)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes)
                     : "memory");
}

// a / d with r = RN(1/d) precomputed: one Markstein correction step; IEEE division
// where its preconditions (normal, mid-range operands and quotient) do not hold
__device__ __forceinline__ double div_fast(double a, double d, double r) {
    const double q0 = __dmul_rn(a, r);
    const double e = __fma_rn(-q0, d, a);
    const double q1 = __fma_rn(e, r, q0);
    const double aq = fabs(q1), aa = fabs(a);
    if (!(aq > 0x1p-900 && aq < 0x1p900 && aa > 0x1p-900 && aa < 0x1p900)) return a / d;
    return q1;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
__device__ __forceinline__ int lo_line(int a, int NX, int sig) {
    const int v = a - NX + 1;
    return v <= 0 ? 0 : (v + sig - 1) / sig;
}
__device__ __forceinline__ int hi_line(int a, int NL, int sig) {
    return a < 0 ? -1 : min(NL - 1, a / sig);
}

// one row: CSR-ordered accumulation over the compile-time template of sweep node MB
// (sources from the ring, factors from the staged step block), then the division
// for the upper sweep
template <bool UPPER, int KIND, int M, int NLR, unsigned kSlot, int MB>
__device__ __forceinline__ double row_value(unsigned fa, unsigned sb0, unsigned sb1, unsigned sb2,
                                           double acc) {
    constexpr int E = tmpl_len(UPPER, KIND, M, MB);
    double v[E], f[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const TE e = tmpl_entry(UPPER, KIND, M, MB, j);
        const unsigned base = e.dx < 0 ? sb0 : e.dx == 0 ? sb1 : sb2;
        v[j] = lds_f64(base + (unsigned)(e.node * NLR + e.dy) * 8u);
        f[j] = lds_f64(fa + 8u * (unsigned)j);
    }
#pragma unroll
    for (int j = 0; j < E; ++j) acc = sub(acc, mul(f[j], v[j]));
    if (UPPER)  // diagonal and its reciprocal follow the entries
        acc = div_fast(acc, lds_f64(fa + 8u * (unsigned)E), lds_f64(fa + 8u * (unsigned)(E + 1)));
    return acc;
}

template <bool UPPER, int KIND, int M, int NLR, unsigned kSlot, int MB>
__device__ __forceinline__ double row_dispatch(int g, unsigned fa, unsigned sb0, unsigned sb1,
                                              unsigned sb2, double acc) {
    if constexpr (MB + 1 < M) {
        if (g != MB) return row_dispatch<UPPER, KIND, M, NLR, kSlot, MB + 1>(g, fa, sb0, sb1, sb2, acc);
    }
    return row_value<UPPER, KIND, M, NLR, kSlot, MB>(fa, sb0, sb1, sb2, acc);
}

// Thread (g, t) = (sweep node g, line t): one row per step.  Warps are 32 lines of
// one node, so the node's template is warp-uniform (a switch over compile-time nodes).
template <bool UPPER, int KIND, int M, int NLP>
__global__ void __launch_bounds__(M * NLP, 1)
    k_wf2(Wf2Dev P, const double* __restrict__ b, double* y, unsigned long long* counter,
          const int* guard, int want) {
    if (guard_off(guard, want)) return;
    constexpr int SIG = sig_of(KIND), KAP = kap_of(KIND), LEAD = lead_of(KIND);
    constexpr int NN = UPPER ? M : M + 1;  // ring nodes (+ the previous-step pseudo node)
    constexpr int R = ring_depth(UPPER, KIND, M);
    constexpr int NLR = NLP + 2;  // lines -1 .. NLP (the outer two stay zero)
    constexpr unsigned kSlot = (unsigned)NN * NLR * 8u;  // bytes per ring slot
    constexpr int NT = M * NLP;
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long bar[kMaxStages2];
    __shared__ int s_ticket;
    const int tid = threadIdx.x, g = tid / NLP, t = tid % NLP;
    const int NL = P.NL, NX = P.NX, S = P.S, NS = P.NS;
    const unsigned sb = P.stage_bytes, nst = (unsigned)P.stages;
    const unsigned u0 = smem_u32(sm);
    const unsigned u_ring = u0 + nst * sb;
    constexpr unsigned ring_bytes = (unsigned)R * kSlot;
    // per step: node block offsets (doubles) so[s*(M+1) + m], m = 0..M (M: step end)
    int32_t* so = reinterpret_cast<int32_t*>(sm + nst * sb + ring_bytes);
    double* ring = reinterpret_cast<double*>(sm + nst * sb);
    const bool lane = t < NL;
    for (int i = tid; i < NS * (M + 1); i += NT) so[i] = P.stepoff[i];
    if (tid == 0)
        for (unsigned k = 0; k < nst; ++k) mbar_init(&bar[k]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned ist = 0, wst = 0, wpar = 0;  // running stage indices (issue / consume)
    const int EP = tmpl_pad(UPPER, KIND, M, g);
    for (;;) {
        __syncthreads();
        if (tid == 0) s_ticket = (int)atomicAdd(counter, 1ull);
        // every ring slot starts finite: template entries absent from a row read an
        // arbitrary slot with a zero factor
        for (unsigned i = tid; i < ring_bytes / 8u; i += NT) ring[i] = 0.0;
        __syncthreads();
        const int task = s_ticket;
        if (task >= P.ntask) return;
        long long c_stage = 0, c_bar = 0, c_poll = 0;
        if (P.trace && tid == 0) P.trace[5 * task] = globaltimer_ns();
        const double* blob = P.blob + (int64_t)task * P.task_stride;
        const int64_t rbase = (int64_t)task * M * S;
        auto step_bytes = [&](int s) {
            return (unsigned)(so[s * (M + 1) + M] - so[s * (M + 1)]) * 8u;
        };
        auto issue = [&](int s) {
            bulk_copy(u0 + ist * sb, blob + so[s * (M + 1)], step_bytes(s), &bar[ist]);
            ist = ist + 1 == nst ? 0u : ist + 1;
        };
        if (tid == 0) {
            for (int s = 0; s < (int)nst - 1 && s < NS; ++s) issue(s);
            for (int s = (int)nst - 1; s < (int)nst + 5 && s < NS; ++s)
                prefetch_l2(blob + so[s * (M + 1)], step_bytes(s));
        }
        // previous step's last node grid, line t (lower sweep; node-0 threads): value
        // x is stored into the ring at step x + SIG*t - LEAD.  Values are published
        // by the producing CTA with plain stores into a buffer armed with the
        // pending sentinel (value-as-flag, pd_sparse.cu) and loaded kPD steps ahead
        // with L2 loads; a pending value is re-polled.  Before its first step the
        // CTA waits until the producer is kStartLag steps further than strictly
        // needed, so the early loads normally find their values.
        const bool hp_task = !UPPER && task > 0 && P.hasprev[task] != 0;
        const bool hp = hp_task && g == 0 && lane;
        const double* prevp = y + rbase - S + (int64_t)t * NX;
        auto poll = [&](int x, unsigned long long cur) -> double {
            if (cur == kPending) {
                unsigned ns = 32;
                do {
                    __nanosleep(ns);
                    if (ns < 256) ns <<= 1;
                    cur = ld_strong_u64(prevp + x);
                } while (cur == kPending);
            }
            return __longlong_as_double((long long)cur);
        };
        auto put = [&](int xp, double v) {
            sts_f64(u_ring + (unsigned)(xp & (R - 1)) * kSlot + (unsigned)(M * NLR + t + 1) * 8u, v);
        };
        unsigned long long q[kPD];
#pragma unroll
        for (int k = 0; k < kPD; ++k) q[k] = kPending;
        long long c_pro = 0, n_hit = 0;
        if (hp_task) {
            const long long cp = P.trace ? clock64() : 0;
            if (tid == 0) {
                const int xg = min(NX - 1, LEAD + kPD + kStartLag);
                poll(xg, ld_strong_u64(prevp + xg));
            }
            __syncthreads();
            if (P.trace) c_pro += clock64() - cp;
        }
        if (hp) {
            // values consumed before step 0 would have stored them: stored now
            for (int x = -SIG * t; x < LEAD - SIG * t; ++x)
                if (x >= 0 && x < NX) put(x, poll(x, ld_strong_u64(prevp + x)));
#pragma unroll
            for (int k = 0; k < kPD; ++k) {
                const int x = k - SIG * t + LEAD;
                if (x >= 0 && x < NX) q[k] = ld_strong_u64(prevp + x);
            }
        }
        if (!UPPER) __syncthreads();
        // right-hand side along x, kPB steps ahead in a register queue
        auto row_of = [&](int x) -> int64_t {
            const int64_t rel = (int64_t)g * S + (int64_t)t * NX + x;
            return UPPER ? rbase + (int64_t)M * S - 1 - rel : rbase + rel;
        };
        double qb[kPB];
#pragma unroll
        for (int k = 0; k < kPB; ++k) {
            const int x = k - SIG * t - KAP * g;
            qb[k] = (lane && x >= 0 && x < NX) ? __ldg(b + row_of(x)) : 0.0;
        }
        // steps in groups of kPB: queue slot k belongs to step s0 + k, so the
        // prefetch queues rotate by renaming (a register move would wait on its load)
        for (int s0 = 0; s0 < NS; s0 += kPB) {
#pragma unroll
            for (int k = 0; k < kPB; ++k) {
                const int s = s0 + k;
                if (s >= NS) break;
                if (tid == 0) {
                    if (s + (int)nst - 1 < NS) issue(s + (int)nst - 1);
                    const int sp = s + (int)nst + 5;
                    if (sp < NS) prefetch_l2(blob + so[sp * (M + 1)], step_bytes(sp));
                }
                if (!UPPER && hp) {
                    const long long cp = P.trace ? clock64() : 0;
                    const int xp = s - SIG * t + LEAD;
                    const unsigned long long cur = q[k];
                    const int xn = xp + kPD;
                    if (xn >= 0 && xn < NX) q[k] = ld_strong_u64(prevp + xn);
                    if (P.trace && xp >= 0 && xp < NX && cur == kPending) ++n_hit;
                    if (xp >= 0 && xp < NX) put(xp, poll(xp, cur));
                    if (P.trace) c_poll += clock64() - cp;
                }
                // this step's factor block
                long long c0 = P.trace ? clock64() : 0;
                mbar_wait(&bar[wst], wpar);
                if (P.trace) c_stage += clock64() - c0;
                const unsigned stg = u0 + wst * sb;
                if (++wst == nst) {
                    wst = 0;
                    wpar ^= 1u;
                }
                const int a = s - KAP * g;  // = x + SIG * line
                const int lo = lo_line(a, NX, SIG), hi = hi_line(a, NL, SIG);
                const int x = a - SIG * t;
                if (lane && t >= lo && t <= hi) {
                    const unsigned fa =
                        stg + (unsigned)(so[s * (M + 1) + g] - so[s * (M + 1)] + (t - lo) * EP) * 8u;
                    const unsigned sb0 = u_ring + (unsigned)((x - 1) & (R - 1)) * kSlot + (unsigned)(t + 1) * 8u;
                    const unsigned sb1 = u_ring + (unsigned)(x & (R - 1)) * kSlot + (unsigned)(t + 1) * 8u;
                    const unsigned sb2 = u_ring + (unsigned)((x + 1) & (R - 1)) * kSlot + (unsigned)(t + 1) * 8u;
                    const double acc =
                        row_dispatch<UPPER, KIND, M, NLR, kSlot, 0>(g, fa, sb0, sb1, sb2, qb[k]);
                    sts_f64(sb1 + (unsigned)(g * NLR) * 8u, acc);
                    if (!UPPER && g == M - 1)
                        st_strong(y + row_of(x), acc);  // polled by the next time step's CTA
                    else
                        y[row_of(x)] = acc;
                }
                const int xn = x + kPB;
                if (lane && xn >= 0 && xn < NX) qb[k] = __ldg(b + row_of(xn));
                if (P.trace) c0 = clock64();
                __syncthreads();
                if (P.trace) c_bar += clock64() - c0;

            }
        }
        if (P.trace && tid == 0) {
            P.trace[5 * task + 1] = globaltimer_ns();
            P.trace[5 * task + 2] = c_stage;
            P.trace[5 * task + 3] = c_bar;
            P.trace[5 * task + 4] = (unsigned long long)c_poll | ((unsigned long long)n_hit << 40) |
                                    ((unsigned long long)(c_pro >> 10) << 52);
        }
    }
}

// factor values into the step blocks (one thread per row; template slots in CSR
// order, absent entries zero)
template <bool UPPER>
__global__ void k_wf2_gather(int64_t n, int64_t MS, int64_t S, int M, int64_t task_stride,
                             const int32_t* rowslot, const uint64_t* mask, const int32_t* E,
                             const int64_t* rp, const int64_t* diag, const double* fac,
                             double* blob) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t task = r / MS, rel = r % MS;
        const int m = (int)(rel / S);
        const int mb = UPPER ? M - 1 - m : m;
        double* dst = blob + task * task_stride + rowslot[rel];
        int64_t p = UPPER ? diag[r] + 1 : rp[r];
        const uint64_t msk = mask[r];
        const int e = E[mb];
        for (int j = 0; j < e; ++j) dst[j] = (msk >> j) & 1ull ? fac[p++] : 0.0;
        if (UPPER) {
            const double d = fac[diag[r]];
            dst[e] = d;
            dst[e + 1] = 1.0 / d;  // IEEE reciprocal for the sweep's one-step division
        }
    }
}

__global__ void k_wf2_begin(unsigned long long* c, int* prog, int ntask, const int* guard,
                            int want) {
    if (guard_off(guard, want)) return;
    if (threadIdx.x == 0) *c = 0ull;
    for (int i = threadIdx.x; i < ntask; i += blockDim.x) prog[i] = -1;
}

}  // namespace

struct Wf2Plan {
    bool upper = false;
    int kind = 0, M = 0, NLP = 0, NL = 0, NX = 0, ntask = 0, NS = 0, stages = 2, blocks = 0;
    int64_t S = 0, n = 0, task_stride = 0;
    size_t smem = 0, stage_bytes = 0;
    bool any_prev = false;
    DevBuf<double> blob;
    DevBuf<int32_t> stepoff, rowslot, E;
    DevBuf<unsigned char> hasprev;
    DevBuf<uint64_t> mask;
    DevBuf<unsigned long long> trace;
    DevBuf<int> prog;
};

namespace {

bool w2_fail(const char* why) {
    if (getenv("PD_WF_VERBOSE")) fprintf(stderr, "[wf2] not applicable: %s\n", why);
    return false;
}

int host_lo(int a, int NX, int sig) {
    const int v = a - NX + 1;
    return v <= 0 ? 0 : (v + sig - 1) / sig;
}
int host_hi(int a, int NL, int sig) { return a < 0 ? -1 : std::min(NL - 1, a / sig); }

template <bool UPPER, int KIND, int M, int NLP>
void w2_set_attr(size_t) {
    // per kernel and device, shared by every plan: always the device maximum (the
    // launch's own size decides occupancy), so plans of different sizes coexist
    int dev = 0, dev_max = 0;
    PD_CUDA(cudaGetDevice(&dev));
    PD_CUDA(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    PD_CUDA(cudaFuncGetAttributes(&fa, k_wf2<UPPER, KIND, M, NLP>));
    PD_CUDA(cudaFuncSetAttribute(k_wf2<UPPER, KIND, M, NLP>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 dev_max - (int)fa.sharedSizeBytes));
}

template <bool UPPER, int KIND, int M>
bool w2_dispatch(Wf2Plan& p, bool set_attr, Ctx* c, const double* b, double* y,
                 unsigned long long* ctr, const int* guard, int want) {
    Wf2Dev d{p.prog.p, p.trace.p, p.blob.p, p.stepoff.p, p.hasprev.p, p.task_stride, p.ntask, p.NS, p.NL, p.NX,
             (int)p.S, p.stages, (unsigned)p.stage_bytes};
    switch (p.NLP) {
#define PD_W2_CASE(NLP_)                                                                        \
    case NLP_:                                                                                  \
        if (set_attr)                                                                           \
            w2_set_attr<UPPER, KIND, M, NLP_>(p.smem);                                          \
        else                                                                                    \
            launch(k_wf2<UPPER, KIND, M, NLP_>, p.blocks, M * NLP_, p.smem, c->stream, d, b, y, ctr, \
                   guard, want);                                                                \
        return true;
        PD_W2_CASE(32)
        PD_W2_CASE(64)
        PD_W2_CASE(128)
        PD_W2_CASE(256)
#undef PD_W2_CASE
        default:
            return false;
    }
}

bool w2_call(Wf2Plan& p, bool set_attr, Ctx* c = nullptr, const double* b = nullptr,
             double* y = nullptr, unsigned long long* ctr = nullptr, const int* guard = nullptr,
             int want = 0) {
    if (p.M == 3) {
        if (p.kind == kFine5)
            return p.upper ? w2_dispatch<true, kFine5, 3>(p, set_attr, c, b, y, ctr, guard, want)
                           : w2_dispatch<false, kFine5, 3>(p, set_attr, c, b, y, ctr, guard, want);
        return p.upper ? w2_dispatch<true, kGal9, 3>(p, set_attr, c, b, y, ctr, guard, want)
                       : w2_dispatch<false, kGal9, 3>(p, set_attr, c, b, y, ctr, guard, want);
    }
    return false;
}

template <bool UPPER, int KIND>
TE host_tmpl(int M, int mb, int j) {
    return tmpl_entry(UPPER, KIND, M, mb, j);
}

// Build the schedule of one sweep; false when the factor pattern does not fit a template.
bool w2_build(Ctx& c, const std::vector<int64_t>& rp, const std::vector<int32_t>& ci,
              const std::vector<int64_t>& dg, int64_t n, int M, int64_t NL64, int64_t NX64,
              bool upper, int kind, Wf2Plan& p) {
    const int64_t S = NL64 * NX64, MS = (int64_t)M * S;
    if (M != 3) return w2_fail("M != 3");
    if (NL64 < 3 || NX64 < 3 || NL64 > 256 || NX64 > 65535 || n % MS != 0) return w2_fail("geometry");
    const int NL = (int)NL64, NX = (int)NX64;
    const int NLP = NL <= 32 ? 32 : NL <= 64 ? 64 : NL <= 128 ? 128 : 256;
    const int sig = sig_of(kind), kap = kap_of(kind);
    const int64_t ntask = n / MS;
    if (ntask > INT32_MAX) return w2_fail("tasks");
    int E[8], EP[8];
    for (int mb = 0; mb < M; ++mb) {
        E[mb] = tmpl_len(upper, kind, M, mb);
        EP[mb] = tmpl_pad(upper, kind, M, mb);
        if (E[mb] > 63) return w2_fail("template too long");
    }
    // template in ORIGINAL coordinates (tp = -1: previous step), per original node
    struct OE { int tp, m, dy, dx; };
    std::vector<std::vector<OE>> tm(M);
    for (int m = 0; m < M; ++m) {
        const int mb = upper ? M - 1 - m : m;
        for (int j = 0; j < E[mb]; ++j) {
            const TE e = upper ? host_tmpl<true, kFine5>(M, mb, j) : host_tmpl<false, kFine5>(M, mb, j);
            const TE g = upper ? host_tmpl<true, kGal9>(M, mb, j) : host_tmpl<false, kGal9>(M, mb, j);
            const TE te = kind == kFine5 ? e : g;
            OE o;
            if (te.node == M) {
                o = {-1, M - 1, te.dy, te.dx};
            } else {
                o.tp = 0;
                o.m = upper ? M - 1 - te.node : te.node;
                o.dy = upper ? -te.dy : te.dy;
                o.dx = upper ? -te.dx : te.dx;
            }
            tm[m].push_back(o);
        }
    }
    // per row: template bits present (CSR order must follow the template order)
    std::vector<uint64_t> mask(n, 0);
    std::vector<unsigned char> hasprev(ntask, 0);
    const int nth = std::max(1, std::min(16, (int)std::thread::hardware_concurrency()));
    std::vector<int> bad(nth, 0);
    std::vector<std::thread> th;
    for (int w = 0; w < nth; ++w)
        th.emplace_back([&, w]() {
            for (int64_t task = w; task < ntask && !bad[w]; task += nth) {
                bool any = false;
                for (int64_t rel = 0; rel < MS; ++rel) {
                    const int64_t r = task * MS + rel;
                    const int m = (int)(rel / S);
                    const int yy = (int)((rel % S) / NX), xx = (int)(rel % NX);
                    const int64_t p0 = upper ? dg[r] + 1 : rp[r], p1 = upper ? rp[r + 1] : dg[r];
                    const auto& T = tm[m];
                    size_t j = 0;
                    uint64_t msk = 0;
                    for (int64_t q = p0; q < p1; ++q) {
                        const int64_t col = ci[q];
                        const int64_t tc = col / MS, rc = col % MS;
                        const int mc = (int)(rc / S), yc = (int)((rc % S) / NX), xc = (int)(rc % NX);
                        const int tp = (int)(tc - task), dy = yc - yy, dx = xc - xx;
                        while (j < T.size() && !(T[j].tp == tp && T[j].m == mc && T[j].dy == dy &&
                                                 T[j].dx == dx))
                            ++j;
                        if (j == T.size()) {
                            bad[w] = 1;
                            break;
                        }
                        if (tp < 0) any = true;
                        msk |= 1ull << j;
                        ++j;
                    }
                    if (bad[w]) break;
                    mask[r] = msk;
                }
                hasprev[task] = any ? 1 : 0;
            }
        });
    for (auto& x : th) x.join();
    for (int w = 0; w < nth; ++w)
        if (bad[w]) return w2_fail("pattern outside the template");
    if (!upper && hasprev[0]) return w2_fail("first task couples to a previous step");
    // step blocks: [node][line - lo][EP] per step, 16-byte aligned; so[s*(M+1) + m] =
    // first double of node m's rows in step s, so[s*(M+1) + M] = end of the step
    const int NS = NX + sig * (NL - 1) + kap * (M - 1);
    std::vector<int32_t> stepoff((size_t)NS * (M + 1), 0);
    size_t maxblk = 0;
    int64_t off = 0;
    for (int s = 0; s < NS; ++s) {
        const int64_t start = off;
        for (int mb = 0; mb < M; ++mb) {
            stepoff[(size_t)s * (M + 1) + mb] = (int32_t)off;
            const int a = s - kap * mb;
            const int lo = host_lo(a, NX, sig), hi = host_hi(a, NL, sig);
            if (hi >= lo) off += (int64_t)(hi - lo + 1) * EP[mb];
        }
        off = (off + 1) & ~1ll;
        stepoff[(size_t)s * (M + 1) + M] = (int32_t)off;
        maxblk = std::max(maxblk, (size_t)(off - start) * 8);
        if (off > INT32_MAX / 2) return w2_fail("task too large");
    }
    const int64_t task_stride = (off + 15) & ~15ll;  // 128-byte aligned tasks
    std::vector<int32_t> rowslot(MS);
    for (int64_t rel = 0; rel < MS; ++rel) {
        const int m = (int)(rel / S);
        const int yy = (int)((rel % S) / NX), xx = (int)(rel % NX);
        const int mb = upper ? M - 1 - m : m, tb = upper ? NL - 1 - yy : yy,
                  xb = upper ? NX - 1 - xx : xx;
        const int s = xb + sig * tb + kap * mb;
        const int a = s - kap * mb;
        rowslot[rel] = stepoff[(size_t)s * (M + 1) + mb] + (tb - host_lo(a, NX, sig)) * EP[mb];
    }
    // launch configuration: ring + stages + step table in shared memory
    const int NN = upper ? M : M + 1;
    const int R = ring_depth(upper, kind, M);
    const size_t ring_bytes = (size_t)R * NN * (NLP + 2) * 8;
    const size_t stage_bytes = (maxblk + 127) & ~(size_t)127;
    const size_t fixed = ring_bytes + (size_t)NS * (M + 1) * 4 + 64;
    int dev_max = 0;
    PD_CUDA(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    const size_t budget = (size_t)dev_max - 256;  // static shared memory (barriers, ticket)
    if (fixed + 2 * stage_bytes > budget) return w2_fail("shared memory");
    int stages = (int)std::min<size_t>(kMaxStages2, (budget - fixed) / stage_bytes);
    if (const char* e = getenv("PD_WF2_STAGES")) stages = std::max(2, std::min(stages, atoi(e)));
    p.upper = upper;
    p.kind = kind;
    p.M = M;
    p.NLP = NLP;
    p.NL = NL;
    p.NX = NX;
    p.S = S;
    p.n = n;
    p.ntask = (int)ntask;
    p.NS = NS;
    p.stages = stages;
    p.stage_bytes = stage_bytes;
    p.task_stride = task_stride;
    p.smem = (size_t)stages * stage_bytes + fixed;
    p.any_prev = false;
    for (auto h : hasprev) p.any_prev = p.any_prev || h;
    if (!w2_call(p, true)) return w2_fail("no instantiation");
    p.blocks = (int)std::min<int64_t>(ntask, c.sms);
    auto up = [](auto& dst, const auto& src) {
        dst.alloc(std::max<size_t>(src.size(), 1));
        if (!src.empty())
            PD_CUDA(cudaMemcpy(dst.p, src.data(), src.size() * sizeof(src[0]),
                               cudaMemcpyHostToDevice));
    };
    up(p.stepoff, stepoff);
    p.prog.alloc((size_t)ntask);
    up(p.rowslot, rowslot);
    up(p.hasprev, hasprev);
    up(p.mask, mask);
    std::vector<int32_t> ev(E, E + M);
    up(p.E, ev);
    p.blob.alloc((size_t)(task_stride * ntask));
    PD_CUDA(cudaMemset(p.blob.p, 0, (size_t)(task_stride * ntask) * 8));
    if (getenv("PD_WF_VERBOSE"))
        fprintf(stderr, "[wf2] %s kind=%d NL=%d NX=%d tasks=%d NS=%d stage=%zu x%d smem=%zu prev=%d\n",
                upper ? "upper" : "lower", kind, NL, NX, p.ntask, NS, stage_bytes, stages, p.smem,
                (int)p.any_prev);
    return true;
}

bool w2_disabled() {
    const char* e = getenv("PD_WF2");
    return e && *e == '0';
}

}  // namespace

bool wf2_lower_preferred(const Ilu0& f) {
    // measured on C2 (scripts/wf2_probe.py): the template lower sweep wins on the
    // Galerkin levels (3x3 coupling to the previous step); on the fine level the
    // pattern-table lower sweep is faster (its one-point time coupling pipelines
    // with a shorter lag).  PD_WF2_LOWER=all|none overrides.
    const char* e = getenv("PD_WF2_LOWER");
    if (e && !strcmp(e, "all")) return true;
    if (e && !strcmp(e, "none")) return false;
    return f.w2_lo && f.w2_lo->kind == kGal9;
}

void wf2_drop_lower(Ilu0& f) { f.w2_lo.reset(); }

void wf2_gather(Ctx& c, Ilu0& f) {
    if (!f.w2_up) return;
    const Csr& P = f.pat();
    for (int upper = 0; upper < 2; ++upper) {
        if (!upper && !f.w2_lo) continue;
        Wf2Plan& p = upper ? *f.w2_up : *f.w2_lo;
        const int g = c.grid_for(p.n, 256);
        if (upper)
            launch(k_wf2_gather<true>, g, 256, 0, c.stream, p.n, (int64_t)p.M * p.S, p.S, p.M,
                   p.task_stride, p.rowslot.p, p.mask.p, p.E.p, P.rowptr.p, f.diag.p, f.fac.p,
                   p.blob.p);
        else
            launch(k_wf2_gather<false>, g, 256, 0, c.stream, p.n, (int64_t)p.M * p.S, p.S, p.M,
                   p.task_stride, p.rowslot.p, p.mask.p, p.E.p, P.rowptr.p, f.diag.p, f.fac.p,
                   p.blob.p);
        PD_LAUNCH_CHECK();
    }
}

bool ilu0_set_wf2(Ctx& c, Ilu0& f, int M, int64_t nline, int64_t npoint) {
    f.w2_lo.reset();
    f.w2_up.reset();
    if (w2_disabled() || f.n == 0) return false;
    const Csr& P = f.pat();
    const int64_t n = f.n;
    PD_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int64_t> rp(n + 1), dg(n);
    std::vector<int32_t> ci(std::max<int64_t>(P.nnz, 1));
    PD_CUDA(cudaMemcpy(rp.data(), P.rowptr.p, (n + 1) * 8, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(ci.data(), P.col.p, P.nnz * 4, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(dg.data(), f.diag.p, n * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i)
        if (dg[i] < rp[i] || dg[i] >= rp[i + 1] || ci[dg[i]] != i) return false;
    auto lo = std::make_shared<Wf2Plan>();
    auto up = std::make_shared<Wf2Plan>();
    bool ok = false;
    for (int kind : {kFine5, kGal9}) {
        if (w2_build(c, rp, ci, dg, n, M, nline, npoint, false, kind, *lo) &&
            w2_build(c, rp, ci, dg, n, M, nline, npoint, true, kind, *up)) {
            ok = true;
            break;
        }
    }
    if (!ok) return false;
    ++c.epoch;
    f.w2_lo = lo;
    f.w2_up = up;
    wf2_gather(c, f);
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return true;
}

static void w2_trace_report(Ctx& c, Wf2Plan& p, const char* name) {
    PD_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<unsigned long long> tr(5 * (size_t)p.ntask);
    PD_CUDA(cudaMemcpy(tr.data(), p.trace.p, tr.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull, t1 = 0;
    double st = 0, sb = 0, sp = 0, dur = 0, hits = 0, pro = 0;
    for (int k = 0; k < p.ntask; ++k) {
        t0 = std::min(t0, tr[5 * k]);
        t1 = std::max(t1, tr[5 * k + 1]);
        dur += (double)(tr[5 * k + 1] - tr[5 * k]);
        st += (double)tr[5 * k + 2];
        sb += (double)tr[5 * k + 3];
        sp += (double)(tr[5 * k + 4] & ((1ull << 40) - 1));
        hits += (double)((tr[5 * k + 4] >> 40) & 0xfff);
        pro += (double)((tr[5 * k + 4] >> 52) << 10);
    }
    const double n = p.ntask;
    fprintf(stderr,
            "[wf2 %s] NL=%d NS=%d tasks=%d span=%.1fus mean task=%.1fus (%.0f ns/step) per task "
            "clk: stage-wait %.0f barrier %.0f poll %.0f (per step %.0f/%.0f/%.0f) thread-0 "
            "pending hits %.1f, start wait %.0f clk\n",
            name, p.NL, p.NS, p.ntask, (t1 - t0) * 1e-3, dur / n * 1e-3, dur / n / p.NS, st / n,
            sb / n, sp / n, st / n / p.NS, sb / n / p.NS, sp / n / p.NS, hits / n, pro / n);
}

void wf2_solve_upper(Ctx& c, Ilu0& f, double* x, const int* guard, int want) {
    Wf2Plan& up = *f.w2_up;
    static const bool trace = getenv("PD_WF2_TRACE") != nullptr;
    if (trace && !up.trace.p) up.trace.alloc(5 * (size_t)up.ntask);
    launch(k_wf2_begin, 1, 256, 0, c.stream, f.counter.p, up.prog.p, up.ntask, guard, want);
    w2_call(up, false, &c, f.scratch.p, x, f.counter.p, guard, want);
    PD_LAUNCH_CHECK();
    if (trace) w2_trace_report(c, up, "upper");
}

void wf2_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard, int want) {
    Wf2Plan& lo = *f.w2_lo;
    Wf2Plan& up = *f.w2_up;
    static const bool trace = getenv("PD_WF2_TRACE") != nullptr;
    if (trace && !lo.trace.p) {
        lo.trace.alloc(5 * (size_t)lo.ntask);
        up.trace.alloc(5 * (size_t)up.ntask);
    }
    if (lo.any_prev) arm_pending(c, f.scratch.p, f.n, guard, want);
    launch(k_wf2_begin, 1, 256, 0, c.stream, f.counter.p, lo.prog.p, lo.ntask, guard, want);
    w2_call(lo, false, &c, b, f.scratch.p, f.counter.p, guard, want);
    launch(k_wf2_begin, 1, 256, 0, c.stream, f.counter.p, up.prog.p, up.ntask, guard, want);
    w2_call(up, false, &c, f.scratch.p, x, f.counter.p, guard, want);
    PD_LAUNCH_CHECK();
    if (trace) {
        w2_trace_report(c, lo, "lower");
        w2_trace_report(c, up, "upper");
    }
}

}  // namespace pd
