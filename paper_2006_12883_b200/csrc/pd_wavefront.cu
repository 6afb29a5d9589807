// Structured wavefront ILU(0) sweeps for grid-ordered space-time systems.
//
// The level-scheduled sweeps in pd_sparse.cu pay one L2 round trip per
// dependency level (~1,060 levels per C2 fine-level solve, ~2.9 us each).  For
// 2D FD space-time operators the rows of one time step are [node m][line y]
// [point x] (paradiff/spacetime.py:117-124 layout); all couplings inside a time
// step (the 5/9-point stencil of Kh and the dense node coupling Kq (x) Mh +
// dt Mq (x) Kh) follow a wavefront that one CTA walks with one thread per
// (node, line) and one __syncthreads per step.  In-task results live in a
// shared-memory ring; only the Jq coupling to the previous time step (another
// CTA) is read from global memory with the value-as-flag protocol of
// pd_sparse.cu, one step ahead.
//
// Data per step (one contiguous block, staged into shared memory by TMA bulk
// copies kStages-1 steps ahead): per node group the active line range, a
// 16-bit pattern id per row (the row's entry sources, deduplicated into a
// table: ring slot relative to (thread, x) or global column relative to the
// row) and the row's factor values.  Column indices are never streamed.
//
// Arithmetic is unchanged: every row accumulates its factor entries in CSR
// order with separately rounded multiply/subtract (linalg.py:104-113), so the
// results are bitwise those of the level-scheduled sweeps and of the numba
// reference.  The schedule is built once on the host from the factor pattern
// and verified; when it does not apply the level-scheduled sweeps stay.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pd {
using namespace dev;

namespace {

constexpr int kMaxStages = 16;  // staged step blocks (TMA bulk copies stages-1 ahead)
constexpr int kMinStages = 2, kDefStages = 3;
constexpr int kMaxGroups = 24;  // node grids per task (M nodes x time steps)
// cross-task (global) entries per row, prefetched one step ahead: kNgFine for
// fine-level stencils (Jq couples one point), kNgWide for Galerkin levels
// (R Mh P couples a 3x3 neighbourhood of the previous time step)
constexpr int kNgFine = 2, kNgWide = 10;
// step-block header: per group int4 {lo, cnt, pid_off, val_off}, then dval_off[G] (16-B padded)
constexpr int hdr_ints(int G) { return (5 * G + 3) & ~3; }
constexpr uint16_t kIdle = 0xFFFF;
constexpr int kChunk = 4;       // entries loaded together before their multiply/subtract chain
// Patterns: header [len, ng, goff[NG]] (int32) and, per ring phase (x mod R),
// the shared-memory offset of every entry's source relative to the thread's
// ring column (int16; ring is slot-major [R + NG][Tp]): ((x + dx) mod R)*Tp +
// dthread for in-task results, (R + j)*Tp for the thread's polled cross-task
// slots.  Every entry is then one conflict-free shared load.
constexpr int kRmax = 16;
constexpr int kOffPad = 4;      // offset rows: a multiple of 4 entries (8-byte loads)
constexpr unsigned kBulkPieces = 8;  // bulk copy requests per step block     // entry offsets of the next row held in registers

struct WfDev {
    const int32_t* nsteps;
    const int64_t* boff;     // per task: first index into bofs
    const int64_t* bofs;     // byte offset of every step block (+1 sentinel per task)
    const int64_t* q0;       // per task: sweep position of its first row
    const int32_t* pattern;  // [npat][2 + NG]
    const int16_t* offs;     // [npat][R][pwo]
    const unsigned char* blob;
    unsigned long long* trace;
    int64_t n;
    int ntask, T, nline, npoint, R, pwo, maxS, npat, G, stages, gfirst, win;
    size_t stage_bytes;
};

WfDev wf_dev(WfPlan& p) {
    WfDev d;
    d.nsteps = p.nsteps.p;
    d.boff = p.boff.p;
    d.bofs = p.bofs.p;
    d.q0 = p.q0.p;
    d.pattern = p.pattern.p;
    d.offs = p.offs.p;
    d.blob = p.blob.p;
    d.trace = p.trace.p;
    d.n = p.n;
    d.ntask = p.ntask;
    d.T = p.T;
    d.nline = p.nline;
    d.npoint = p.npoint;
    d.R = p.R;
    d.pwo = p.pwo;
    d.maxS = p.maxS;
    d.npat = p.npat;
    d.G = p.T / p.nline;
    d.stages = p.stages;
    d.gfirst = p.gfirst ? 1 : 0;
    d.win = p.win ? 1 : 0;

    d.stage_bytes = p.stage_bytes;
    return d;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
// relaxed gpu-scope load issued only when `pred`; otherwise the register keeps
// its value (no select on the load result, no dummy-address hot spot)
__device__ __forceinline__ unsigned long long ld_strong_if(bool pred, const double* p,
                                                           unsigned long long v) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q ld.relaxed.gpu.global.b64 %0, [%1];\n}\n"
        : "+l"(v)
        : "l"(p), "r"((unsigned)pred)
        : "memory");
    return v;
}
// weak (L1-cacheable) load issued only when `pred`
__device__ __forceinline__ unsigned long long ld_weak_if(bool pred, const double* p,
                                                         unsigned long long v) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q ld.global.b64 %0, [%1];\n}\n"
        : "+l"(v)
        : "l"(p), "r"((unsigned)pred)
        : "memory");
    return v;
}
__device__ __forceinline__ void st_strong4(double* p, double a, double b, double c, double d) {
    asm volatile("st.relaxed.gpu.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)),
                 "l"(__double_as_longlong(c)), "l"(__double_as_longlong(d))
                 : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
    // the stage being refilled was only read through the generic proxy before
    // the __syncthreads that precedes this call: no proxy fence is needed (a
    // fence.proxy.async here costs a CTA-wide MEMBAR on the issuing thread)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    // several requests in flight per block
    const unsigned piece = ((bytes + kBulkPieces - 1) / kBulkPieces + 15) & ~15u;
    for (unsigned o = 0; o < bytes; o += piece) {
        const unsigned nb = min(piece, bytes - o);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(static_cast<char*>(dst) + o)),
            "l"(static_cast<const char*>(src) + o), "r"(nb), "r"(smem_u32(bar))
            : "memory");
    }
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 32-bit shared-memory accessors: LDS/STS on shared-window addresses (no
// generic-address conversion, no 64-bit address arithmetic).  volatile keeps
// them ordered against __syncthreads / mbarrier waits.
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_u16(unsigned a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int2 lds_v2s32(unsigned a) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds_v4s32(unsigned a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds_v2u32(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds_v4s16(unsigned a, int& o0, int& o1, int& o2, int& o3) {
    short x0, x1, x2, x3;
    asm volatile("ld.shared.v4.s16 {%0, %1, %2, %3}, [%4];"
                 : "=h"(x0), "=h"(x1), "=h"(x2), "=h"(x3)
                 : "r"(a));
    o0 = x0;
    o1 = x1;
    o2 = x2;
    o3 = x3;
}
__device__ __forceinline__ void sts_f64(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// One CTA per task (up to kMaxGroups node grids: the M nodes of one or more
// time steps), tickets in topological order so a CTA only waits on tasks
// already claimed by running CTAs.  Thread t = g*nline + line walks points
// x = 0.. of line `line` of grid g (in sweep order), one row per wavefront step.
// (A thread running the M node rows of its line measured slower on every C2
// level: the per-step chain lengthens.)  Shared memory is addressed through
// 32-bit shared-window offsets.
template <bool UPPER, int NG, bool PAD, bool WIN = false>
__global__ void __launch_bounds__(NG <= kNgFine ? 768 : 512, 1)
    k_wf_sweep(WfDev P, const double* __restrict__ b, double* y, unsigned long long* counter,
               const int* guard, int want) {
    if (guard_off(guard, want)) return;
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long bar[kMaxStages];
    __shared__ unsigned long long bar_tab;
    __shared__ int s_ticket;
    constexpr int kPatHdr = 2 + NG;
    constexpr int NGA = NG > 0 ? NG : 1;
    const int T = P.T, R = P.R, pwo = P.pwo, G = P.G, t = threadIdx.x;
    const bool gf = P.gfirst != 0;  // polled values folded from registers, no ring slots
    const unsigned Tp = (unsigned)(T + 31) & ~31u, RW = (unsigned)(R + (gf ? 0 : NG));
    const unsigned sb = (unsigned)P.stage_bytes;
    // layout (bytes from sm): stages | ring [RW(+1)][Tp] f64 | block offsets | patterns | offsets
    const unsigned nst = (unsigned)P.stages;
    const unsigned o_ring = nst * sb;
    // PAD plans read an extra all-zero slot row; unpadded plans skip it (every KB
    // counts: above 196 KB of shared memory the SM keeps no L1 for the b loads)
    const unsigned o_bofs = o_ring + Tp * (RW + (PAD ? 1u : 0u)) * 8u;
    const unsigned o_pat = (o_bofs + (unsigned)(P.maxS + 1) * 4u + 15u) & ~15u;
    const unsigned pat_bytes = ((unsigned)(P.npat * kPatHdr) * 4u + 15u) & ~15u;
    const unsigned off_bytes = ((unsigned)(P.npat * R * pwo) * 2u + 15u) & ~15u;
    const unsigned o_off = o_pat + pat_bytes;
    int32_t* sbofs = reinterpret_cast<int32_t*>(sm + o_bofs);  // block offsets in the task
    const unsigned u0 = smem_u32(sm);
    const unsigned u_pat = u0 + o_pat, u_off = u0 + o_off;
    const bool lane = t < T;
    const int g = lane ? t / P.nline : 0, line = lane ? t % P.nline : 0;
    const unsigned my_ring = u0 + o_ring + (lane ? (unsigned)t : 0u) * 8u;
    const unsigned ring_step = Tp * 8u;             // bytes between ring slots
    const unsigned off_row = (unsigned)pwo * 2u;    // bytes per (pattern, phase) offset row
    const unsigned off_pat = (unsigned)R * off_row;  // bytes per pattern
    if (PAD)
        for (unsigned i = t; i < Tp; i += blockDim.x)  // the zero slot row
            reinterpret_cast<double*>(sm + o_ring)[RW * Tp + i] = 0.0;
    if (t == 0) {
        for (unsigned k = 0; k < nst; ++k) mbar_init(&bar[k]);
        mbar_init(&bar_tab);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // pattern and offset tables: two bulk copies (a per-thread copy loop costs
    // ~100 us of dependent load->store latency on small CTAs)
    if (t == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&bar_tab)),
                     "r"(pat_bytes + off_bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(u_pat),
            "l"(P.pattern), "r"(pat_bytes), "r"(smem_u32(&bar_tab))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(u_off),
            "l"(P.offs), "r"(off_bytes), "r"(smem_u32(&bar_tab))
            : "memory");
    }
    mbar_wait(&bar_tab, 0);
    unsigned ist = 0;             // stage of the next bulk copy (thread 0)
    unsigned wst = 0, wpar = 0;   // stage and mbarrier parity of the next block consumed
    const int n = (int)P.n;
    const bool y32 = (reinterpret_cast<uintptr_t>(y) & 31) == 0;
    for (;;) {
        __syncthreads();
        if (t == 0) s_ticket = (int)atomicAdd(counter, 1ull);
        __syncthreads();
        const int task = s_ticket;
        if (task >= P.ntask) return;
        if (P.trace && t == 0) P.trace[2 * task] = globaltimer();
        const int S = P.nsteps[task];
        const int64_t bo = P.boff[task];
        const int64_t base = P.bofs[bo];
        for (int s = t; s <= S; s += blockDim.x) sbofs[s] = (int32_t)(P.bofs[bo + s] - base);
        __syncthreads();
        // blocks are issued and consumed in order, once each: running stage
        // indices (no runtime division by the stage count)
        auto issue = [&](int s) {
            bulk_load(sm + ist * sb, P.blob + base + sbofs[s], (unsigned)(sbofs[s + 1] - sbofs[s]),
                      &bar[ist]);
            ist = ist + 1 == nst ? 0u : ist + 1;
        };
        if (t == 0)
            for (int s = 0; s < (int)nst - 1 && s < S; ++s) issue(s);
        auto next_block = [&]() -> unsigned {
            mbar_wait(&bar[wst], wpar);
            const unsigned a = u0 + wst * sb;
            if (++wst == nst) {
                wst = 0;
                wpar ^= 1u;
            }
            return a;
        };
        const int qline = (int)P.q0[task] + t * P.npoint;  // sweep position of x = 0
        int seq = 0;                  // rows done on this line
        unsigned phase_b = 0, ring_ph = 0;  // ring phase: offset-row and slot byte offsets
        // results are published per aligned 4-row sector (one 32-byte store instead
        // of four scattered 8-byte ones); a line's last rows are flushed at its end
        double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
        int wcnt = 0;
        // the thread's next row, prepared one step ahead: descriptor, right-hand
        // side and cross-task values (loads land while this step computes)
        bool n_act = false;
        unsigned n_val = 0, n_stride = 0, n_dval = 0, n_pat = 0, n_ph = 0;
        int n_len = 0, n_ng = 0;
        double bn = 0.0, xn[NGA];
        // WIN: sliding 3x3 window of the previous step's last node grid around
        // (line, x): wv[dy+1][dx+1]; nc / nc0 = next column(s) loaded ahead
        double wv[3][3], nc[3], nc0[3], cnc[3], cnc0[3];
        const int Sg = P.nline * P.npoint;
        const double* prevp = y + ((int64_t)qline - (int64_t)(g + 1) * Sg);  // (line, x=0)
        auto wload = [&](int dy, int col) -> double {
            const bool ok = lane && line + dy >= 0 && line + dy < P.nline && col >= 0 &&
                            col < P.npoint;
            return __longlong_as_double((long long)ld_weak_if(
                ok, prevp + (int64_t)dy * P.npoint + (ok ? col : 0), (unsigned long long)kPending));
        };
        auto wresolve = [&](double v, int dy, int col) -> double {
            unsigned long long u = (unsigned long long)__double_as_longlong(v);
            if (u == kPending && line + dy >= 0 && line + dy < P.nline && col >= 0 &&
                col < P.npoint) {
                unsigned int ns = 32;
                do {
                    __nanosleep(ns);
                    if (ns < 256) ns <<= 1;
                    u = ld_strong_u64(prevp + (int64_t)dy * P.npoint + col);
                } while (u == kPending);
            }
            return __longlong_as_double((long long)u);
        };
        if (WIN) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                nc[d] = nc0[d] = cnc[d] = cnc0[d] = 0.0;
                wv[d][0] = wv[d][1] = wv[d][2] = 0.0;
            }
        }
        auto view = [&](unsigned blk, int q) {
            const int4 h = lds_v4s32(blk + 16u * (unsigned)g);  // lo, cnt, pid_off, val_off
            const int i = line - h.x;
            bool act = lane && (unsigned)i < (unsigned)h.y;
            unsigned pid = kIdle;
            if (act) pid = lds_u16(blk + (unsigned)h.z + 2u * (unsigned)i);
            act = act && pid != kIdle;
            n_act = act;
            n_val = blk + (unsigned)h.w + 8u * (unsigned)i;
            n_stride = 8u * (unsigned)h.y;
            if (UPPER) n_dval = blk + (unsigned)lds_s32(blk + 16u * G + 4u * g) + 8u * (unsigned)i;
            n_len = 0;
            n_ng = 0;
            int row = 0;
            const unsigned pat = u_pat + pid * (unsigned)(kPatHdr * 4);
            n_ph = pat;
            n_pat = u_off + pid * off_pat;
            if (act) {
                const int2 lg = lds_v2s32(pat);
                n_len = lg.x;
                n_ng = lg.y;
                row = UPPER ? n - 1 - q : q;
            }
            const double* yrow = y + row;
            if (WIN) {
                if (act && n_ng > 0) {
                    const int xq = q - qline;  // the next row's point on this line
                    if (xq == 0) {
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            nc0[d] = wload(d - 1, 0);
                            nc[d] = wload(d - 1, 1);
                        }
                    } else {
#pragma unroll
                        for (int d = 0; d < 3; ++d) nc[d] = wload(d - 1, xq + 1);
                    }
                }
                bn = __ldg(b + row);
                return;
            }
#pragma unroll
            for (int k = 0; k < NG; ++k) {
                const bool pk = k < n_ng;
                const int go = pk ? lds_s32(pat + 8u + 4u * k) : 0;
                // first look with a weak (L1-cacheable) load: each word goes from the
                // sentinel to its final value exactly once per launch (L1 starts clean),
                // so a weak load sees one or the other; pending values are re-polled
                // with strong loads below
                xn[k] = __longlong_as_double(
                    (long long)ld_weak_if(pk, yrow + go, (unsigned long long)kPending));
            }
            bn = __ldg(b + row);
        };
        view(next_block(), qline);
        for (int s = 0; s < S; ++s) {
            // refill the stage freed by step s-1 (everyone passed the barrier)
            if (t == 0 && s + (int)nst - 1 < S) issue(s + (int)nst - 1);
            const bool act = n_act;
            const unsigned val = n_val, stride = n_stride, dval = n_dval, pat = n_pat, ph = n_ph;
            const int len = n_len, ng = n_ng;
            const double bb = bn;
            double xs[NGA];
#pragma unroll
            for (int k = 0; k < NG; ++k) xs[k] = xn[k];
            if (WIN) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    cnc[d] = nc[d];
                    cnc0[d] = nc0[d];
                }
            }
            if (s + 1 < S) view(next_block(), qline + seq + (act ? 1 : 0));
            if (act) {
                const int q = qline + seq;
                const int row = UPPER ? n - 1 - q : q;
                double acc = bb;
                unsigned fa = val;
                if (WIN && ng > 0) {
                    // slide the window to x = seq and fold the present 3x3 entries in
                    // CSR order ((dy, dx) lexicographic = column order)
                    const int xq = seq;
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        if (xq == 0) {
                            wv[d][0] = 0.0;
                            wv[d][1] = wresolve(cnc0[d], d - 1, 0);
                        } else {
                            wv[d][0] = wv[d][1];
                            wv[d][1] = wv[d][2];
                        }
                        wv[d][2] = wresolve(cnc[d], d - 1, xq + 1);
                    }
                    int k = 0;
#pragma unroll
                    for (int d = 0; d < 3; ++d)
#pragma unroll
                        for (int e = 0; e < 3; ++e) {
                            const bool pr = line + d - 1 >= 0 && line + d - 1 < P.nline &&
                                            xq + e - 1 >= 0 && xq + e - 1 < P.npoint;
                            if (pr) {
                                acc = sub(acc, mul(lds_f64(fa + (unsigned)k * stride), wv[d][e]));
                                ++k;
                            }
                        }
                    fa += (unsigned)ng * stride;
                } else if (NG > 0 && ng > 0) {
                    // cross-task values: resolve the (rare) pending ones by strong polls
                    unsigned long long u[NGA];
#pragma unroll
                    for (int k = 0; k < NG; ++k) {
                        u[k] = (unsigned long long)__double_as_longlong(xs[k]);
                        if (k < ng) {
                            if (P.trace) {  // diagnostics: polls, and polls found pending
                                atomicAdd(P.trace + 2 * P.ntask + 1, 1ull);
                                if (u[k] == kPending) atomicAdd(P.trace + 2 * P.ntask, 1ull);
                            }
                            if (u[k] == kPending) {
                                const int go = lds_s32(ph + 8u + 4u * k);
                                unsigned int ns = 32;
                                do {
                                    __nanosleep(ns);
                                    if (ns < 256) ns <<= 1;
                                    u[k] = ld_strong_u64(y + row + go);
                                } while (u[k] == kPending);
                            }
                        }
                    }
                    if (gf) {  // CSR order: the previous-step entries come first
                        double fg[NGA];
#pragma unroll
                        for (int k = 0; k < NG; ++k)
                            if (k < ng) fg[k] = lds_f64(fa + (unsigned)k * stride);
#pragma unroll
                        for (int k = 0; k < NG; ++k)
                            if (k < ng)
                                acc = sub(acc, mul(fg[k], __longlong_as_double((long long)u[k])));
                        fa += (unsigned)ng * stride;
                    } else {
#pragma unroll
                        for (int k = 0; k < NG; ++k)
                            if (k < ng)
                                sts_f64(my_ring + (unsigned)(R + k) * ring_step,
                                        __longlong_as_double((long long)u[k]));
                    }
                }
                const unsigned orow = pat + phase_b;
                // PAD: len is padded to kChunk with zero entries, no per-entry predicates
                // each chunk's offsets are loaded one chunk ahead: the ring loads of a
                // chunk then wait on nothing but their own issue
                uint2 onext = lds_v2u32(orow);
#pragma unroll 1
                for (int k0 = 0; k0 < len; k0 += kChunk) {
                    const uint2 oc = onext;
                    if (k0 + kChunk < len) onext = lds_v2u32(orow + 2u * (unsigned)(k0 + kChunk));
                    const int oi[kChunk] = {(int)(short)(oc.x & 0xffffu), (int)oc.x >> 16,
                                            (int)(short)(oc.y & 0xffffu), (int)oc.y >> 16};
                    double v[kChunk], f[kChunk];
#pragma unroll
                    for (int k = 0; k < kChunk; ++k)
                        if (PAD || k0 + k < len) {
                            v[k] = lds_f64(my_ring + 8u * (unsigned)oi[k]);
                            f[k] = lds_f64(fa + (unsigned)k * stride);
                        }
#pragma unroll
                    for (int k = 0; k < kChunk; ++k)
                        if (PAD || k0 + k < len) acc = sub(acc, mul(f[k], v[k]));
                    fa += kChunk * stride;
                }
                if (UPPER) acc = acc / lds_f64(dval);
                {
                    const int sl = row & 3;
                    w0 = sl == 0 ? acc : w0;
                    w1 = sl == 1 ? acc : w1;
                    w2 = sl == 2 ? acc : w2;
                    w3 = sl == 3 ? acc : w3;
                    ++wcnt;
                    if ((UPPER ? sl == 0 : sl == 3) || seq + 1 == P.npoint) {
                        double* g0 = y + (row & ~3);
                        if (wcnt == 4 && y32) {
                            st_strong4(g0, w0, w1, w2, w3);
                        } else {  // partial sector: rows [lo, hi] of this group
                            const int lo = UPPER ? sl : sl - wcnt + 1;
                            const int hi = UPPER ? sl + wcnt - 1 : sl;
                            if (lo <= 0 && 0 <= hi) st_strong(g0, w0);
                            if (lo <= 1 && 1 <= hi) st_strong(g0 + 1, w1);
                            if (lo <= 2 && 2 <= hi) st_strong(g0 + 2, w2);
                            if (lo <= 3 && 3 <= hi) st_strong(g0 + 3, w3);
                        }
                        wcnt = 0;
                    }
                }
                sts_f64(my_ring + ring_ph, acc);
                ++seq;
                const bool wrap = phase_b + off_row == off_pat;
                phase_b = wrap ? 0u : phase_b + off_row;
                ring_ph = wrap ? 0u : ring_ph + ring_step;
            }
            __syncthreads();
        }
        if (P.trace && t == 0) P.trace[2 * task + 1] = globaltimer();
    }
}

// factor values into the step blocks: one slot per row (first value index,
// stride between its entries, entry count, diagonal index), built with the plan
template <bool UPPER>
__global__ void k_wf_gather(int64_t nslot, const int32_t* srow, const int64_t* sval,
                            const int32_t* sstride, const int64_t* sdiag, const int32_t* scount,
                            const int64_t* rp, const double* fac, const int64_t* diag,
                            double* blobd) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslot;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = srow[i];
        const int64_t src = UPPER ? diag[r] + 1 : rp[r];
        const int cnt = scount[i], st = sstride[i];
        const int64_t v0 = sval[i];
        for (int k = 0; k < cnt; ++k) blobd[v0 + (int64_t)k * st] = fac[src + k];
        if (UPPER) blobd[sdiag[i]] = fac[diag[r]];
    }
}

struct HostPlan {
    std::vector<int32_t> S;
    std::vector<int64_t> boff, bofs, q0;
    std::vector<int32_t> pattern;
    std::vector<int16_t> offs;
    int R = 0, pwo = 0, ng = 0;
    bool gfirst = false;
    bool win = false;  // cross-task entries are the previous step's 3x3 neighbourhood
    std::vector<unsigned char> blob;
    std::vector<int32_t> srow, sstride, scount;
    std::vector<int64_t> sval, sdiag;
    int maxS = 0;
    size_t stage_bytes = 0;
};

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool plan_fail(const char* why) {
    if (getenv("PD_WF_VERBOSE")) fprintf(stderr, "[wf] schedule rejected (check %s)\n", why);
    return false;
}

// Host schedule for one sweep.  Sweep position q runs over rows in solve order
// (row = q for the lower sweep, n-1-q for the upper), so both sweeps share one
// builder: task = q / (G*nline*npoint), thread = (group, line), x = point.
bool build_plan(const std::vector<int64_t>& rp, const std::vector<int32_t>& ci,
                const std::vector<int64_t>& dg, int64_t n, int G, int64_t nline, int64_t npoint,
                bool upper, int NG, bool pad, HostPlan& hp) {
    const int kPatHdr = 2 + NG;
    const int64_t TR = (int64_t)G * nline * npoint, T = (int64_t)G * nline;
    if (G < 1 || G > kMaxGroups || TR <= 0 || n % TR != 0 || n >= INT_MAX || T > 4096)
        return plan_fail("1");
    const int64_t ntask = n / TR;
    auto row_of = [&](int64_t q) { return upper ? n - 1 - q : q; };
    auto q_of = [&](int64_t r) { return upper ? n - 1 - r : r; };
    auto ent = [&](int64_t r, int64_t& p0, int64_t& p1) {
        if (upper) { p0 = dg[r] + 1; p1 = rp[r + 1]; }
        else { p0 = rp[r]; p1 = dg[r]; }
    };
    std::vector<int32_t> step(n);
    hp.S.assign(ntask, 0);
    for (int64_t q = 0; q < n; ++q) {
        const int64_t task = q / TR, x = (q % TR) % npoint;
        int64_t p0, p1;
        ent(row_of(q), p0, p1);
        int32_t s = x > 0 ? step[q - 1] + 1 : 0;
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t qc = q_of(ci[p]);
            if (qc >= q) return plan_fail("2");  // not triangular in sweep order
            if (qc / TR == task) s = std::max(s, step[qc] + 1);
        }
        step[q] = s;
        hp.S[task] = std::max(hp.S[task], s + 1);
    }
    // ring depth: a producer's slot is rewritten R points later on its line;
    // that must happen strictly after every step reading it
    auto need_of = [&](int64_t q, int64_t qc) -> int64_t {
        const int64_t xc = (qc % TR) % npoint;
        int64_t r = 1;
        while (xc + r < npoint && step[qc + r] <= step[q]) ++r;
        return r;
    };
    int64_t R = 4;  // >= 4: an in-task entry read back from global memory is flushed
    for (int64_t q = 0; q < n; ++q) {
        int64_t p0, p1;
        ent(row_of(q), p0, p1);
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t qc = q_of(ci[p]);
            if (qc / TR != q / TR) continue;
            const int64_t r = need_of(q, qc);
            if (r <= kRmax) R = std::max(R, r);
        }
    }
    const int64_t Tp = (T + 31) / 32 * 32;
    hp.R = (int)R;
    hp.ng = NG;
    if ((R + NG + 1) * Tp + Tp > 32767) return plan_fail("3");  // int16 offsets
    // entry-source patterns, deduplicated: key = [len, ng, goff[NG], (dth, dx | global j)...]
    std::unordered_map<std::string, int> pid_of;
    std::vector<std::vector<int32_t>> pats;
    std::vector<uint16_t> pid(n);
    std::vector<int32_t> nent(n);
    std::vector<int32_t> d;
    for (int64_t q = 0; q < n; ++q) {
        const int64_t task = q / TR, o = q % TR, th = o / npoint, x = o % npoint;
        const int64_t r = row_of(q);
        int64_t p0, p1;
        ent(r, p0, p1);
        d.assign(kPatHdr, 0);
        int nglob = 0;
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t c = ci[p], qc = q_of(c);
            if (qc / TR == task && need_of(q, qc) <= R) {
                const int64_t oc = qc % TR;
                const int64_t dth = oc / npoint - th, dx = oc % npoint - x;
                d.push_back((int32_t)dth);
                d.push_back((int32_t)dx);
            } else {  // polled from global memory into the thread's slot R + j
                if (nglob >= NG || c - r < INT_MIN || c - r > INT_MAX) return plan_fail("4");
                d[2 + nglob] = (int32_t)(c - r);
                d.push_back(INT_MIN);
                d.push_back(nglob);
                ++nglob;
            }
        }
        d[0] = (int32_t)((d.size() - kPatHdr) / 2);
        d[1] = nglob;
        nent[q] = d[0];
        std::string key(reinterpret_cast<const char*>(d.data()), d.size() * sizeof(int32_t));
        auto it = pid_of.find(key);
        int id;
        if (it == pid_of.end()) {
            id = (int)pats.size();
            if (id >= kIdle) return plan_fail("5");
            pid_of.emplace(std::move(key), id);
            pats.push_back(d);
        } else {
            id = it->second;
        }
        pid[q] = (uint16_t)id;
    }
    // globals first: every pattern's cross-task entries precede its ring entries
    // (the lower sweep's previous-step columns come first in CSR order).  Then the
    // kernel folds polled values straight from registers and the ring needs no
    // global slots; otherwise they go through slots R + j.
    bool gfirst = true;
    for (auto& pt : pats)
        for (int e = pt[1]; e < pt[0]; ++e)
            if (pt[kPatHdr + 2 * e] == INT_MIN) gfirst = false;
    hp.gfirst = gfirst;
    // Window eligibility (lower sweep, one time step per task, 2D grid): every
    // polled row (g, y, x) reads exactly the present part of the 3x3 neighbourhood
    // of (y, x) in the previous step's last node grid, in (dy, dx) order, i.e.
    // global offsets -(g+1)*S + dy*npoint + dx.  The kernel then keeps a sliding
    // 3x3 register window per thread (3 new values per row instead of 9 polls).
    hp.win = false;
    if (!upper && gfirst && NG == kNgWide && G * nline * npoint == TR && nline == npoint &&
        !getenv("PD_WF_NO_WINDOW")) {
        bool ok = true;
        const int64_t S = nline * npoint;
        for (int64_t q = 0; q < n && ok; ++q) {
            const auto& pt = pats[pid[q]];
            const int ngq = pt[1];
            if (ngq == 0) continue;
            const int64_t o = q % TR, th = o / npoint, x = o % npoint;
            const int64_t gg = th / nline, yl = th % nline;
            int k = 0;
            for (int dy = -1; dy <= 1 && ok; ++dy)
                for (int dx = -1; dx <= 1 && ok; ++dx) {
                    if (yl + dy < 0 || yl + dy >= nline || x + dx < 0 || x + dx >= npoint) continue;
                    if (k >= ngq || pt[2 + k] != -(gg + 1) * S + dy * npoint + dx) ok = false;
                    ++k;
                }
            if (k != ngq) ok = false;
        }
        hp.win = ok;
    }
    const int64_t RW = R + (gfirst ? 0 : NG);
    int maxlen = 1;
    for (auto& pt : pats) maxlen = std::max(maxlen, pt[0] - (gfirst ? pt[1] : 0));
    const int pwo = (int)align_up(std::max(maxlen, kOffPad), kOffPad);
    hp.pwo = pwo;
    hp.pattern.assign(pats.size() * kPatHdr, 0);
    hp.offs.assign(pats.size() * R * pwo, 0);
    // Entry lists are padded to a multiple of kChunk with (zero slot, +0.0 factor)
    // entries: acc - (+0)*(+0) == acc bitwise for every acc, so the chunk loop
    // needs no per-entry predication.  The pattern header stores the padded length.
    const int16_t zero_off = (int16_t)(RW * Tp);
    for (size_t k = 0; k < pats.size(); ++k) {
        const auto& pt = pats[k];
        std::copy(pt.begin(), pt.begin() + kPatHdr, hp.pattern.begin() + k * kPatHdr);
        const int e0 = gfirst ? pt[1] : 0;  // first entry taken from the ring
        const int nr = pt[0] - e0;
        const int lenp = pad ? (int)align_up(nr, kChunk) : nr;
        hp.pattern[k * kPatHdr] = lenp;
        for (int64_t ph = 0; ph < R; ++ph)
            for (int e = 0; e < pwo; ++e) {
                int64_t off = zero_off;
                if (e < nr) {
                    const int32_t a = pt[kPatHdr + 2 * (e0 + e)], b2 = pt[kPatHdr + 2 * (e0 + e) + 1];
                    off = a == INT_MIN ? (R + b2) * Tp : ((((ph + b2) % R) + R) % R) * Tp + a;
                }
                hp.offs[(k * R + ph) * pwo + e] = (int16_t)off;
            }
        (void)lenp;
    }
    // step blocks: rows of (task, step) grouped per node grid, line-contiguous
    hp.boff.assign(ntask, 0);
    hp.q0.assign(ntask, 0);
    hp.maxS = 0;
    size_t maxblock = 0;
    std::vector<std::vector<int64_t>> at;  // per step: sweep positions
    for (int64_t task = 0; task < ntask; ++task) {
        const int S = hp.S[task];
        hp.maxS = std::max(hp.maxS, S);
        hp.boff[task] = (int64_t)hp.bofs.size();
        hp.q0[task] = task * TR;
        at.assign(S, {});
        for (int64_t q = task * TR; q < (task + 1) * TR; ++q) at[step[q]].push_back(q);
        for (int s = 0; s < S; ++s) {
            int32_t lo[kMaxGroups], hi[kMaxGroups], W[kMaxGroups], cnt[kMaxGroups];
            for (int gg = 0; gg < kMaxGroups; ++gg) { lo[gg] = INT_MAX; hi[gg] = -1; W[gg] = 0; }
            for (int64_t q : at[s]) {
                const int64_t th = (q % TR) / npoint;
                const int gg = (int)(th / nline), ln = (int)(th % nline);
                lo[gg] = std::min<int32_t>(lo[gg], ln);
                hi[gg] = std::max<int32_t>(hi[gg], ln);
                const int32_t ngq = gfirst ? pats[pid[q]][1] : 0;
                W[gg] = std::max(W[gg], pad ? ngq + (int32_t)align_up(nent[q] - ngq, kChunk)
                                            : nent[q]);
            }
            // header: per group int4 {lo, cnt, pid_off, val_off}, then dval_off[G]
            std::vector<int32_t> hdr(hdr_ints(G), 0);
            size_t off = hdr.size() * 4;
            for (int gg = 0; gg < G; ++gg) {
                cnt[gg] = hi[gg] >= lo[gg] ? hi[gg] - lo[gg] + 1 : 0;
                hdr[4 * gg] = cnt[gg] ? lo[gg] : 0;
                hdr[4 * gg + 1] = cnt[gg];
                hdr[4 * gg + 2] = (int32_t)off;
                off += (size_t)cnt[gg] * 2;
            }
            off = align_up(off, 8);
            for (int gg = 0; gg < G; ++gg) {
                hdr[4 * gg + 3] = (int32_t)off;
                off += (size_t)cnt[gg] * W[gg] * 8;
            }
            for (int gg = 0; gg < G; ++gg) {
                hdr[4 * G + gg] = (int32_t)off;
                if (upper) off += (size_t)cnt[gg] * 8;
            }
            const size_t bytes = align_up(off, 16);
            maxblock = std::max(maxblock, bytes);
            const size_t base = hp.blob.size();
            hp.bofs.push_back((int64_t)base);
            hp.blob.resize(base + bytes, 0);
            unsigned char* blk = hp.blob.data() + base;
            std::memcpy(blk, hdr.data(), hdr.size() * 4);
            for (int gg = 0; gg < G; ++gg)
                for (int i = 0; i < cnt[gg]; ++i)
                    reinterpret_cast<uint16_t*>(blk + hdr[4 * gg + 2])[i] = kIdle;
            for (int64_t q : at[s]) {
                const int64_t th = (q % TR) / npoint;
                const int gg = (int)(th / nline), i = (int)(th % nline) - lo[gg];
                reinterpret_cast<uint16_t*>(blk + hdr[4 * gg + 2])[i] = pid[q];
                hp.srow.push_back((int32_t)row_of(q));
                hp.sval.push_back((int64_t)(base + hdr[4 * gg + 3]) / 8 + i);
                hp.sstride.push_back(cnt[gg]);
                hp.scount.push_back(nent[q]);
                hp.sdiag.push_back((int64_t)(base + hdr[4 * G + gg]) / 8 + i);
            }
        }
        hp.bofs.push_back((int64_t)hp.blob.size());
    }
    hp.stage_bytes = align_up(maxblock, 128);
    return true;
}

template <bool UPPER, int NG, bool PAD>
bool configure_launch_pad(Ctx& c, WfPlan& p) {
    constexpr int kPatHdr = 2 + NG;
    const size_t fixed = (size_t)((p.T + 31) / 32 * 32) *
                             (p.R + (p.gfirst ? 0 : NG) + (PAD ? 1 : 0)) * sizeof(double) +
                         (size_t)(p.maxS + 1) * sizeof(int32_t) + 16 +
                         align_up((size_t)p.npat * kPatHdr * sizeof(int32_t), 16) +
                         align_up((size_t)p.npat * p.R * p.pwo * sizeof(int16_t), 16);
    int dev_max = 0;
    PD_CUDA(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    // kDefStages staged step blocks (a block is requested stages-1 steps before its
    // use); deeper staging measured no faster on any C2 level (the step is bound by
    // its own dependency chain, not the copy).  Two when three do not fit.
    const size_t budget = (size_t)dev_max - 1024;
    int stages = kDefStages;
    if (const char* e = getenv("PD_WF_STAGES")) stages = atoi(e);
    if (budget > fixed)
        stages = std::min<int>(stages, (int)((budget - fixed) / std::max<size_t>(p.stage_bytes, 1)));
    stages = std::max(kMinStages, std::min(kMaxStages, stages));
    const size_t smem = stages * p.stage_bytes + fixed;
    p.stages = stages;
    const int threads = (p.T + 31) / 32 * 32;
    const int max_threads = NG <= kNgFine ? 768 : 512;
    if (getenv("PD_WF_VERBOSE"))
        fprintf(stderr, "[wf] %s NG=%d PAD=%d T=%d R=%d npat=%d pwo=%d stage=%zu smem=%zu (max %d)\n",
                UPPER ? "upper" : "lower", NG, (int)PAD, p.T, p.R, p.npat, p.pwo, p.stage_bytes, smem,
                dev_max);
    if (smem + 1024 > (size_t)dev_max || threads > max_threads) return false;
    p.smem = smem;
    // the attribute is per kernel, shared by every plan: only ever raise it
    static size_t attr_max = 0;
    if (smem > attr_max) {
        PD_CUDA(cudaFuncSetAttribute(k_wf_sweep<UPPER, NG, PAD>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (!UPPER && NG == kNgWide)
            PD_CUDA(cudaFuncSetAttribute(k_wf_sweep<false, kNgWide, PAD, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_max = smem;
    }
    int per_sm = 0;
    PD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wf_sweep<UPPER, NG, PAD>,
                                                          threads, smem));
    if (per_sm < 1) return false;
    p.blocks = std::min(p.ntask, per_sm * c.sms);
    p.pad = PAD;
    p.threads = threads;
    return true;
}

template <bool UPPER, int NG>
bool configure_launch(Ctx& c, WfPlan& p, bool pad) {
    return pad ? configure_launch_pad<UPPER, NG, true>(c, p)
               : configure_launch_pad<UPPER, NG, false>(c, p);
}

void upload(WfPlan& p, HostPlan& hp, int64_t n, int G, int64_t nline, int64_t npoint) {
    p.n = n;
    p.ntask = (int)hp.S.size();
    p.T = (int)(G * nline);
    p.nline = (int)nline;
    p.npoint = (int)npoint;
    p.R = hp.R;
    p.pwo = hp.pwo;
    p.ng = hp.ng;
    p.npat = (int)(hp.pattern.size() / (2 + hp.ng));
    p.gfirst = hp.gfirst;
    p.win = hp.win;
    // tables are bulk-copied into shared memory: 16-byte multiples
    hp.pattern.resize(align_up(hp.pattern.size() * 4, 16) / 4, 0);
    hp.offs.resize(align_up(hp.offs.size() * 2, 16) / 2, 0);
    p.maxS = hp.maxS;
    p.stage_bytes = hp.stage_bytes;
    auto up = [](auto& dst, auto& src) {
        dst.alloc(std::max<size_t>(src.size(), 1));
        if (!src.empty())
            PD_CUDA(cudaMemcpy(dst.p, src.data(), src.size() * sizeof(src[0]),
                               cudaMemcpyHostToDevice));
    };
    up(p.nsteps, hp.S);
    up(p.boff, hp.boff);
    up(p.bofs, hp.bofs);
    up(p.q0, hp.q0);
    up(p.pattern, hp.pattern);
    up(p.offs, hp.offs);
    up(p.blob, hp.blob);
    up(p.srow, hp.srow);
    up(p.sval, hp.sval);
    up(p.sstride, hp.sstride);
    up(p.scount, hp.scount);
    up(p.sdiag, hp.sdiag);
    p.nslot = (int64_t)hp.srow.size();
}

bool wavefront_disabled() {
    const char* e = getenv("PD_NO_WAVEFRONT");
    return e && *e && *e != '0';
}

}  // namespace

bool ilu0_set_wavefront(Ctx& c, Ilu0& f, int64_t ngroup, int64_t nline, int64_t npoint,
                        int64_t ngroup_lower) {
    ++c.epoch;
    f.wf_lo.reset();
    f.wf_up.reset();
    if (wavefront_disabled() || f.n == 0) return false;
    // template-structured sweeps first (one time step per task, pd_wf2.cu); where its
    // lower sweep is not the faster one (wf2_lower_preferred) the pattern-table lower
    // sweep below runs with the template upper sweep
    const bool w2 = ngroup > 0 && ngroup <= 8 && ilu0_set_wf2(c, f, (int)ngroup, nline, npoint);
    if (w2 && wf2_lower_preferred(f)) return true;
    // the lower sweep's tasks may span several time steps (in-task time coupling
    // through the ring instead of cross-CTA polls); the upper factor has no time
    // coupling, so its tasks stay one step each
    const int64_t glo = ngroup_lower > 0 ? ngroup_lower : ngroup;
    const Csr& P = f.pat();
    const int64_t n = f.n;
    PD_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int64_t> rp(n + 1), dg(n);
    std::vector<int32_t> ci(std::max<int64_t>(P.nnz, 1));
    PD_CUDA(cudaMemcpy(rp.data(), P.rowptr.p, (n + 1) * 8, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(ci.data(), P.col.p, P.nnz * 4, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemcpy(dg.data(), f.diag.p, n * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i)  // factor must have a stored diagonal
        if (dg[i] < rp[i] || dg[i] >= rp[i + 1] || ci[dg[i]] != i) return false;
    auto lo = std::make_unique<WfPlan>();
    auto up = std::make_unique<WfPlan>();
    auto build = [&](bool upper, int64_t G, WfPlan& plan) -> bool {
        // zero-padded entry lists first (no predication); unpadded when the
        // padded step blocks do not fit three stages
        // Padding trades issue slots (extra zero entries) for a shorter per-entry
        // critical path: it pays on latency-bound CTAs (<= 12 warps: C2 127^2..7^2
        // levels) and costs on the 24-warp fine level (upper sweep 631 -> 770 us).
        const char* pe = getenv("PD_WF_PAD");  // experiments: 0 = never, 1 = always
        const bool try_pad = pe && *pe ? *pe == '1' : G * nline <= 384;
        for (bool pad : {true, false})
            for (int NG : {0, kNgFine, kNgWide}) {
                if (pad && !try_pad) continue;
                HostPlan hp;
                if (!build_plan(rp, ci, dg, n, (int)G, nline, npoint, upper, NG, pad, hp))
                    continue;
                upload(plan, hp, n, (int)G, nline, npoint);
                const bool ok = NG == 0 ? (upper ? configure_launch<true, 0>(c, plan, pad)
                                                 : configure_launch<false, 0>(c, plan, pad))
                    : NG == kNgFine ? (upper ? configure_launch<true, kNgFine>(c, plan, pad)
                                             : configure_launch<false, kNgFine>(c, plan, pad))
                                    : (upper ? configure_launch<true, kNgWide>(c, plan, pad)
                                             : configure_launch<false, kNgWide>(c, plan, pad));
                if (ok && (plan.stages >= kDefStages || !pad)) return true;
            }
        return false;
    };
    if (w2) {
        if (!build(false, glo, *lo)) return true;  // template sweeps for both
        f.wf_lo = std::move(lo);
        wf2_drop_lower(f);
        wf_gather(c, f);
        PD_CUDA(cudaStreamSynchronize(c.stream));
        return true;
    }
    if (!build(false, glo, *lo) || !build(true, ngroup, *up)) return false;
    f.wf_lo = std::move(lo);
    f.wf_up = std::move(up);
    wf_gather(c, f);
    PD_CUDA(cudaStreamSynchronize(c.stream));
    return true;
}

void wf_gather(Ctx& c, Ilu0& f) {
    if (!f.wf_lo) return;
    const Csr& P = f.pat();
    for (int upper = 0; upper < 2; ++upper) {
        if (upper && !f.wf_up) continue;
        WfPlan& p = upper ? *f.wf_up : *f.wf_lo;
        const int g = c.grid_for(p.nslot, 256);
        double* blobd = reinterpret_cast<double*>(p.blob.p);
        if (upper)
            launch(k_wf_gather<true>, g, 256, 0, c.stream, p.nslot, p.srow.p, p.sval.p,
                   p.sstride.p, p.sdiag.p, p.scount.p, P.rowptr.p, f.fac.p, f.diag.p, blobd);
        else
            launch(k_wf_gather<false>, g, 256, 0, c.stream, p.nslot, p.srow.p, p.sval.p,
                   p.sstride.p, p.sdiag.p, p.scount.p, P.rowptr.p, f.fac.p, f.diag.p, blobd);
        PD_LAUNCH_CHECK();
    }
}

__global__ void k_wf_begin(unsigned long long* c, const int* guard, int want) {
    if (guard_off(guard, want)) return;
    *c = 0ull;
}

static void wf_trace_report(Ctx& c, WfPlan& p, const char* name) {
    PD_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<unsigned long long> tr(2 * (size_t)p.ntask + 2);
    std::vector<int32_t> S(p.ntask);
    PD_CUDA(cudaMemcpy(tr.data(), p.trace.p, tr.size() * 8, cudaMemcpyDeviceToHost));
    PD_CUDA(cudaMemset(p.trace.p + 2 * (size_t)p.ntask, 0, 16));
    fprintf(stderr, "[wf %s] polls=%llu pending=%llu\n", name, tr[2 * (size_t)p.ntask + 1],
            tr[2 * (size_t)p.ntask]);
    PD_CUDA(cudaMemcpy(S.data(), p.nsteps.p, S.size() * 4, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<double> per_step, start;
    for (int k = 0; k < p.ntask; ++k) {
        t0 = std::min(t0, tr[2 * k]);
        t1 = std::max(t1, tr[2 * k + 1]);
    }
    for (int k = 0; k < p.ntask; ++k) {
        per_step.push_back((tr[2 * k + 1] - tr[2 * k]) / std::max(1.0, (double)S[k]));
        start.push_back((tr[2 * k] - t0) * 1e-3);
    }
    auto q = [](std::vector<double> v, double f) {
        std::sort(v.begin(), v.end());
        return v[(size_t)(f * (v.size() - 1))];
    };
    fprintf(stderr,
            "[wf %s] tasks=%d blocks=%d T=%d S=%d npat=%d stage=%zuBx%d smem=%zuB span=%.1fus "
            "ns/step min/med/max=%.0f/%.0f/%.0f start(us) med/max=%.1f/%.1f\n",
            name, p.ntask, p.blocks, p.T, p.maxS, p.npat, p.stage_bytes, p.stages, p.smem,
            (t1 - t0) * 1e-3, q(per_step, 0), q(per_step, 0.5), q(per_step, 1), q(start, 0.5),
            q(start, 1));
}

template <bool UPPER, int NG>
static void launch_sweep_ng(Ctx& c, WfPlan& p, const double* b, double* y,
                            unsigned long long* ctr, const int* guard, int want) {
    if (!UPPER && NG == kNgWide && p.win) {
        if (p.pad)
            launch(k_wf_sweep<false, kNgWide, true, true>, p.blocks, p.threads, p.smem, c.stream,
                   wf_dev(p), b, y, ctr, guard, want);
        else
            launch(k_wf_sweep<false, kNgWide, false, true>, p.blocks, p.threads, p.smem,
                   c.stream, wf_dev(p), b, y, ctr, guard, want);
        return;
    }
    if (p.pad)
        launch(k_wf_sweep<UPPER, NG, true>, p.blocks, p.threads, p.smem, c.stream, wf_dev(p), b,
               y, ctr, guard, want);
    else
        launch(k_wf_sweep<UPPER, NG, false>, p.blocks, p.threads, p.smem, c.stream, wf_dev(p),
               b, y, ctr, guard, want);
}

template <bool UPPER>
static void launch_sweep(Ctx& c, WfPlan& p, const double* b, double* y, unsigned long long* ctr,
                         const int* guard, int want) {
    if (p.ng == 0)
        launch_sweep_ng<UPPER, 0>(c, p, b, y, ctr, guard, want);
    else if (p.ng == kNgFine)
        launch_sweep_ng<UPPER, kNgFine>(c, p, b, y, ctr, guard, want);
    else
        launch_sweep_ng<UPPER, kNgWide>(c, p, b, y, ctr, guard, want);
}

void wf_solve_lower(Ctx& c, Ilu0& f, const double* b, const int* guard, int want) {
    WfPlan& lo = *f.wf_lo;
    if (lo.ng > 0) arm_pending(c, f.scratch.p, f.n, guard, want);
    launch(k_wf_begin, 1, 1, 0, c.stream, f.counter.p, guard, want);
    launch_sweep<false>(c, lo, b, f.scratch.p, f.counter.p, guard, want);
    PD_LAUNCH_CHECK();
}

void wf_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard, int want) {
    WfPlan& lo = *f.wf_lo;
    WfPlan& up = *f.wf_up;
    static const bool trace = getenv("PD_WF_TRACE") != nullptr;
    if (trace && !lo.trace.p) {
        lo.trace.alloc(2 * (size_t)lo.ntask + 2);
        up.trace.alloc(2 * (size_t)up.ntask + 2);
    }
    // outputs are armed with the pending sentinel only when a sweep polls them
    if (lo.ng > 0) arm_pending(c, f.scratch.p, f.n, guard, want);
    launch(k_wf_begin, 1, 1, 0, c.stream, f.counter.p, guard, want);
    launch_sweep<false>(c, lo, b, f.scratch.p, f.counter.p, guard, want);
    if (up.ng > 0) arm_pending(c, x, f.n, guard, want);
    launch(k_wf_begin, 1, 1, 0, c.stream, f.counter.p, guard, want);
    launch_sweep<true>(c, up, f.scratch.p, x, f.counter.p, guard, want);
    PD_LAUNCH_CHECK();
    if (trace) {
        wf_trace_report(c, lo, "lower");
        wf_trace_report(c, up, "upper");
    }
}

}  // namespace pd
