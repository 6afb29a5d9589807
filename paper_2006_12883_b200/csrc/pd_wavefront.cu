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

constexpr int kStages = 3;      // staged step blocks (TMA bulk copies kStages-1 ahead)
constexpr int kMaxGroups = 8;   // node grids per task
// cross-task (global) entries per row, prefetched one step ahead: kNgFine for
// fine-level stencils (Jq couples one point), kNgWide for Galerkin levels
// (R Mh P couples a 3x3 neighbourhood of the previous time step)
constexpr int kNgFine = 2, kNgWide = 10;
constexpr int kHdrInts = 6 * kMaxGroups;  // lo, cnt, W, pid_off, val_off, dval_off per group
constexpr uint16_t kIdle = 0xFFFF;
constexpr int kChunk = 4;       // entries loaded together before their multiply/subtract chain
// Patterns: header [len, ng, goff[NG]] (int32) and, per ring phase (x mod R),
// the shared-memory offset of every entry's source relative to the thread's
// ring column (int16; ring is slot-major [R + NG][Tp]): ((x + dx) mod R)*Tp +
// dthread for in-task results, (R + j)*Tp for the thread's polled cross-task
// slots.  Every entry is then one conflict-free shared load.
constexpr int kRmax = 16;
constexpr int kOffPad = 16;     // offset rows: at least this many entries, multiple of 8
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
    int ntask, T, nline, npoint, R, pwo, maxS, npat;
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

struct RowView {  // this thread's slot in one step block
    bool active;
    int W, cnt, i;
    const double* val;   // entry k at val[k * cnt]
    const double* dval;  // upper diagonal
    int pid;
};

__device__ __forceinline__ RowView view_row(const unsigned char* blk, int g, int line) {
    const int32_t* h = reinterpret_cast<const int32_t*>(blk);
    RowView v;
    const int lo = h[g], cnt = h[kMaxGroups + g];
    v.active = false;
    v.cnt = cnt;
    v.W = 0;
    v.i = 0;
    v.pid = kIdle;
    v.val = v.dval = nullptr;
    if (line < lo || line >= lo + cnt) return v;
    v.i = line - lo;
    v.pid = reinterpret_cast<const uint16_t*>(blk + h[3 * kMaxGroups + g])[v.i];
    if (v.pid == kIdle) return v;
    v.active = true;
    v.W = h[2 * kMaxGroups + g];
    v.val = reinterpret_cast<const double*>(blk + h[4 * kMaxGroups + g]) + v.i;
    v.dval = reinterpret_cast<const double*>(blk + h[5 * kMaxGroups + g]) + v.i;
    return v;
}

// One CTA per task (a time step: up to kMaxGroups node grids), tickets in
// topological order so a CTA only waits on tasks already claimed by running
// CTAs.  Thread t = g*nline + line walks points x = 0.. of line `line` of node
// grid g (in sweep order).
template <bool UPPER, int NG>
__global__ void __launch_bounds__(NG <= kNgFine ? 768 : 512, 1) k_wf_sweep(WfDev P, const double* b, double* y,
                                                     unsigned long long* counter,
                                                     const int* guard, int want) {
    if (guard_off(guard, want)) return;
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long bar[kStages];
    __shared__ int s_ticket;
    constexpr int kPatHdr = 2 + NG;
    const int T = P.T, R = P.R, RW = P.R + NG, pwo = P.pwo, t = threadIdx.x;
    unsigned char* stage = sm;  // kStages * stage_bytes
    const int Tp = (T + 31) & ~31;
    // ring, slot-major [RW][Tp]: lanes of a warp always hit distinct banks
    double* ring = reinterpret_cast<double*>(sm + kStages * P.stage_bytes);
    int64_t* sbofs = reinterpret_cast<int64_t*>(ring + (size_t)Tp * RW);    // [maxS + 1]
    int32_t* spat = reinterpret_cast<int32_t*>(                           // [npat][kPatHdr]
        (reinterpret_cast<uintptr_t>(sbofs + P.maxS + 1) + 15) & ~(uintptr_t)15);
    int16_t* soff = reinterpret_cast<int16_t*>(spat + P.npat * kPatHdr);   // [npat][R][pwo]
    for (int i = t; i < P.npat * kPatHdr; i += blockDim.x) spat[i] = P.pattern[i];
    for (int i = t; i < P.npat * R * pwo; i += blockDim.x) soff[i] = P.offs[i];
    const bool lane = t < T;
    const int g = lane ? t / P.nline : 0, line = lane ? t % P.nline : -1;
    double* myring = ring + (lane ? t : 0);
    if (t == 0)
        for (int k = 0; k < kStages; ++k) mbar_init(&bar[k]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned uses = 0;  // blocks consumed by this CTA so far (stage = uses % kStages)
    for (;;) {
        __syncthreads();
        if (t == 0) s_ticket = (int)atomicAdd(counter, 1ull);
        __syncthreads();
        const int task = s_ticket;
        if (task >= P.ntask) return;
        if (P.trace && t == 0) P.trace[2 * task] = globaltimer();
        const int S = P.nsteps[task];
        const int64_t bo = P.boff[task];
        for (int s = t; s <= S; s += blockDim.x) sbofs[s] = P.bofs[bo + s];
        __syncthreads();
        auto issue = [&](int s) {
            const unsigned st = (uses + s) % kStages;
            bulk_load(stage + st * P.stage_bytes, P.blob + sbofs[s],
                      (unsigned)(sbofs[s + 1] - sbofs[s]), &bar[st]);
        };
        if (t == 0)
            for (int s = 0; s < kStages - 1 && s < S; ++s) issue(s);
        auto block_of = [&](int s) -> const unsigned char* {
            const unsigned k = uses + s;
            mbar_wait(&bar[k % kStages], (k / kStages) & 1u);
            return stage + (k % kStages) * P.stage_bytes;
        };
        const int64_t qline = P.q0[task] + (int64_t)t * P.npoint;  // sweep position of x = 0
        int seq = 0, phase = 0;  // rows done on this line, and seq mod R
        // results are published per aligned 4-row sector (one 32-byte store instead
        // of four scattered 8-byte ones); a line's last rows are flushed at its end
        double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
        int wcnt = 0;
        const bool y32 = (reinterpret_cast<uintptr_t>(y) & 31) == 0;
        double xs[NG], xn[NG];
        double bn = 0.0;
        // The thread's next row, prepared one step ahead: right-hand side and
        // cross-task values (loads that land while the current step computes;
        // unconditional or predicated inside one instruction, so no select
        // waits on them) and its entry counts.
        int n_len = 0, n_ng = 0;
        auto prefetch = [&](const RowView& v, int64_t q) {
            int64_t row = 0;
            const int32_t* pat = spat;
            n_len = 0;
            n_ng = 0;
            if (v.active) {
                row = UPPER ? P.n - 1 - q : q;
                pat = spat + v.pid * kPatHdr;
                n_len = pat[0];
                n_ng = pat[1];
            }
            bn = b[row];
#pragma unroll
            for (int j = 0; j < NG; ++j)
                xn[j] = __longlong_as_double((long long)ld_strong_if(
                    j < n_ng, y + row + (j < n_ng ? pat[2 + j] : 0),
                    (unsigned long long)kPending));
        };
        RowView nv = view_row(block_of(0), g, line);
        nv.active = nv.active && lane;
        prefetch(nv, qline);
        for (int s = 0; s < S; ++s) {
            // refill the stage freed by step s-1 (everyone passed the barrier)
            if (t == 0 && s + kStages - 1 < S) issue(s + kStages - 1);
            const RowView cv = nv;
            const double bb = bn;
            const int len = n_len, ng = n_ng;
#pragma unroll
            for (int j = 0; j < NG; ++j) xs[j] = xn[j];
            if (s + 1 < S) {
                nv = view_row(block_of(s + 1), g, line);
                nv.active = nv.active && lane;
                prefetch(nv, qline + seq + (cv.active ? 1 : 0));
            }
            if (cv.active) {
                const int64_t q = qline + seq;
                const int64_t row = UPPER ? P.n - 1 - q : q;
                // cross-task values: wait until published, then into the own slots
                if (ng > 0) {
                    const int32_t* pat = spat + cv.pid * kPatHdr;
#pragma unroll
                    for (int j = 0; j < NG; ++j)
                        if (j < ng) {
                            unsigned long long u =
                                (unsigned long long)__double_as_longlong(xs[j]);
                            unsigned int ns = 32;
                            while (u == kPending) {
                                __nanosleep(ns);
                                if (ns < 256) ns <<= 1;
                                u = ld_strong_u64(y + row + pat[2 + j]);
                            }
                            myring[(R + j) * Tp] = __longlong_as_double((long long)u);
                        }
                }
                double acc = bb;
                const int16_t* off = soff + ((size_t)cv.pid * R + phase) * pwo;
                for (int k0 = 0; k0 < len; k0 += kChunk) {
                    const short4 o = *reinterpret_cast<const short4*>(off + k0);
                    const int oi[kChunk] = {o.x, o.y, o.z, o.w};
                    double v[kChunk], f[kChunk];
#pragma unroll
                    for (int k = 0; k < kChunk; ++k)
                        if (k0 + k < len) {
                            v[k] = myring[oi[k]];
                            f[k] = cv.val[(size_t)(k0 + k) * cv.cnt];
                        }
#pragma unroll
                    for (int k = 0; k < kChunk; ++k)
                        if (k0 + k < len) acc = sub(acc, mul(f[k], v[k]));
                }
                if (UPPER) acc = acc / cv.dval[0];
                {
                    const int sl = (int)(row & 3);
                    w0 = sl == 0 ? acc : w0;
                    w1 = sl == 1 ? acc : w1;
                    w2 = sl == 2 ? acc : w2;
                    w3 = sl == 3 ? acc : w3;
                    ++wcnt;
                    if ((UPPER ? sl == 0 : sl == 3) || seq + 1 == P.npoint) {
                        const int64_t g0 = row & ~(int64_t)3;
                        if (wcnt == 4 && y32) {
                            st_strong4(y + g0, w0, w1, w2, w3);
                        } else {  // partial sector: rows [lo, hi] of this group
                            const int lo = UPPER ? sl : sl - wcnt + 1;
                            const int hi = UPPER ? sl + wcnt - 1 : sl;
                            if (lo <= 0 && 0 <= hi) st_strong(y + g0, w0);
                            if (lo <= 1 && 1 <= hi) st_strong(y + g0 + 1, w1);
                            if (lo <= 2 && 2 <= hi) st_strong(y + g0 + 2, w2);
                            if (lo <= 3 && 3 <= hi) st_strong(y + g0 + 3, w3);
                        }
                        wcnt = 0;
                    }
                }
                myring[phase * Tp] = acc;
                ++seq;
                phase = (phase + 1 == R) ? 0 : phase + 1;
            }
            __syncthreads();
        }
        uses += (unsigned)S;
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
                bool upper, int NG, HostPlan& hp) {
    const int kPatHdr = 2 + NG;
    const int64_t TR = (int64_t)G * nline * npoint, T = (int64_t)G * nline;
    if (G < 1 || G > kMaxGroups || TR <= 0 || n % TR != 0 || n >= INT_MAX ||
        T > (NG <= kNgFine ? 768 : 512))
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
    const int64_t RW = R + NG, Tp = (T + 31) / 32 * 32;
    hp.R = (int)R;
    hp.ng = NG;
    if (RW * Tp + Tp > 32767) return plan_fail("3");  // int16 offsets
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
    int maxlen = 1;
    for (auto& pt : pats) maxlen = std::max(maxlen, pt[0]);
    const int pwo = (int)align_up(std::max(maxlen, kOffPad), 8);
    hp.pwo = pwo;
    hp.pattern.assign(pats.size() * kPatHdr, 0);
    hp.offs.assign(pats.size() * R * pwo, 0);
    for (size_t k = 0; k < pats.size(); ++k) {
        const auto& pt = pats[k];
        std::copy(pt.begin(), pt.begin() + kPatHdr, hp.pattern.begin() + k * kPatHdr);
        for (int64_t ph = 0; ph < R; ++ph)
            for (int e = 0; e < pt[0]; ++e) {
                const int32_t a = pt[kPatHdr + 2 * e], b2 = pt[kPatHdr + 2 * e + 1];
                const int64_t off =
                    a == INT_MIN ? (R + b2) * Tp : ((((ph + b2) % R) + R) % R) * Tp + a;
                hp.offs[(k * R + ph) * pwo + e] = (int16_t)off;
            }
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
                W[gg] = std::max(W[gg], nent[q]);
            }
            int32_t hdr[kHdrInts] = {0};
            size_t off = kHdrInts * 4;
            for (int gg = 0; gg < kMaxGroups; ++gg) {
                cnt[gg] = hi[gg] >= lo[gg] ? hi[gg] - lo[gg] + 1 : 0;
                hdr[gg] = cnt[gg] ? lo[gg] : 0;
                hdr[kMaxGroups + gg] = cnt[gg];
                hdr[2 * kMaxGroups + gg] = W[gg];
                hdr[3 * kMaxGroups + gg] = (int32_t)off;
                off += (size_t)cnt[gg] * 2;
            }
            off = align_up(off, 8);
            for (int gg = 0; gg < kMaxGroups; ++gg) {
                hdr[4 * kMaxGroups + gg] = (int32_t)off;
                off += (size_t)cnt[gg] * W[gg] * 8;
            }
            for (int gg = 0; gg < kMaxGroups; ++gg) {
                hdr[5 * kMaxGroups + gg] = (int32_t)off;
                if (upper) off += (size_t)cnt[gg] * 8;
            }
            const size_t bytes = align_up(off, 16);
            maxblock = std::max(maxblock, bytes);
            const size_t base = hp.blob.size();
            hp.bofs.push_back((int64_t)base);
            hp.blob.resize(base + bytes, 0);
            unsigned char* blk = hp.blob.data() + base;
            std::memcpy(blk, hdr, sizeof(hdr));
            for (int gg = 0; gg < kMaxGroups; ++gg)
                for (int i = 0; i < cnt[gg]; ++i)
                    reinterpret_cast<uint16_t*>(blk + hdr[3 * kMaxGroups + gg])[i] = kIdle;
            for (int64_t q : at[s]) {
                const int64_t th = (q % TR) / npoint;
                const int gg = (int)(th / nline), i = (int)(th % nline) - lo[gg];
                reinterpret_cast<uint16_t*>(blk + hdr[3 * kMaxGroups + gg])[i] = pid[q];
                hp.srow.push_back((int32_t)row_of(q));
                hp.sval.push_back((int64_t)(base + hdr[4 * kMaxGroups + gg]) / 8 + i);
                hp.sstride.push_back(cnt[gg]);
                hp.scount.push_back(nent[q]);
                hp.sdiag.push_back((int64_t)(base + hdr[5 * kMaxGroups + gg]) / 8 + i);
            }
        }
        hp.bofs.push_back((int64_t)hp.blob.size());
    }
    hp.stage_bytes = align_up(maxblock, 128);
    return true;
}

template <bool UPPER, int NG>
bool configure_launch(Ctx& c, WfPlan& p) {
    constexpr int kPatHdr = 2 + NG;
    const size_t smem = kStages * p.stage_bytes +
                        (size_t)((p.T + 31) / 32 * 32) * (p.R + NG) * sizeof(double) +
                        (size_t)(p.maxS + 1) * sizeof(int64_t) + 16 +
                        (size_t)p.npat * kPatHdr * sizeof(int32_t) +
                        align_up((size_t)p.npat * p.R * p.pwo * sizeof(int16_t), 16);
    int dev_max = 0;
    PD_CUDA(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c.device));
    if (smem + 1024 > (size_t)dev_max) return false;
    p.smem = smem;
    // the attribute is per kernel, shared by every plan: only ever raise it
    static size_t attr_max = 0;
    if (smem > attr_max) {
        PD_CUDA(cudaFuncSetAttribute(k_wf_sweep<UPPER, NG>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_max = smem;
    }
    const int threads = (p.T + 31) / 32 * 32;
    int per_sm = 0;
    PD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wf_sweep<UPPER, NG>, threads,
                                                          smem));
    if (per_sm < 1) return false;
    p.blocks = std::min(p.ntask, per_sm * c.sms);
    return true;
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
                        int ring) {
    f.wf_lo.reset();
    f.wf_up.reset();
    if (wavefront_disabled() || f.n == 0) return false;
    (void)ring;  // ring depth is derived from the schedule (kept for the ABI)
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
    auto build = [&](int NG) -> bool {
        {
            HostPlan hp;
            if (!build_plan(rp, ci, dg, n, (int)ngroup, nline, npoint, false, NG, hp)) return false;
            upload(*lo, hp, n, (int)ngroup, nline, npoint);
        }
        HostPlan hp;
        if (!build_plan(rp, ci, dg, n, (int)ngroup, nline, npoint, true, NG, hp)) return false;
        upload(*up, hp, n, (int)ngroup, nline, npoint);
        if (NG == kNgFine)
            return configure_launch<false, kNgFine>(c, *lo) && configure_launch<true, kNgFine>(c, *up);
        return configure_launch<false, kNgWide>(c, *lo) && configure_launch<true, kNgWide>(c, *up);
    };
    if (!build(kNgFine) && !build(kNgWide)) return false;
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
    std::vector<unsigned long long> tr(2 * (size_t)p.ntask);
    std::vector<int32_t> S(p.ntask);
    PD_CUDA(cudaMemcpy(tr.data(), p.trace.p, tr.size() * 8, cudaMemcpyDeviceToHost));
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
            "[wf %s] tasks=%d blocks=%d T=%d S=%d npat=%d stage=%zuB smem=%zuB span=%.1fus "
            "ns/step min/med/max=%.0f/%.0f/%.0f start(us) med/max=%.1f/%.1f\n",
            name, p.ntask, p.blocks, p.T, p.maxS, p.npat, p.stage_bytes, p.smem,
            (t1 - t0) * 1e-3, q(per_step, 0), q(per_step, 0.5), q(per_step, 1), q(start, 0.5),
            q(start, 1));
}

void wf_solve(Ctx& c, Ilu0& f, const double* b, double* x, const int* guard, int want) {
    WfPlan& lo = *f.wf_lo;
    WfPlan& up = *f.wf_up;
    static const bool trace = getenv("PD_WF_TRACE") != nullptr;
    if (trace && !lo.trace.p) {
        lo.trace.alloc(2 * (size_t)lo.ntask);
        up.trace.alloc(2 * (size_t)up.ntask);
    }
    const int threads = (lo.T + 31) / 32 * 32;
    arm_pending(c, f.scratch.p, f.n, guard, want);
    launch(k_wf_begin, 1, 1, 0, c.stream, f.counter.p, guard, want);
    if (lo.ng == kNgFine)
        launch(k_wf_sweep<false, kNgFine>, lo.blocks, threads, lo.smem, c.stream, wf_dev(lo), b,
               f.scratch.p, f.counter.p, guard, want);
    else
        launch(k_wf_sweep<false, kNgWide>, lo.blocks, threads, lo.smem, c.stream, wf_dev(lo), b,
               f.scratch.p, f.counter.p, guard, want);
    arm_pending(c, x, f.n, guard, want);
    launch(k_wf_begin, 1, 1, 0, c.stream, f.counter.p, guard, want);
    if (up.ng == kNgFine)
        launch(k_wf_sweep<true, kNgFine>, up.blocks, threads, up.smem, c.stream, wf_dev(up),
               (const double*)f.scratch.p, x, f.counter.p, guard, want);
    else
        launch(k_wf_sweep<true, kNgWide>, up.blocks, threads, up.smem, c.stream, wf_dev(up),
               (const double*)f.scratch.p, x, f.counter.p, guard, want);
    PD_LAUNCH_CHECK();
    if (trace) {
        wf_trace_report(c, lo, "lower");
        wf_trace_report(c, up, "upper");
    }
}

}  // namespace pd
