// blocked.cu -- GCM_ALGO_BLOCKED: the chain-shortened single-factor path.
//
// The paper's sweep (CholeskyModifyA, PAPER.md 24-30) has a serial chain of
// n + k - 1 Compute links (each a sqrt/div) because row block b cannot start
// before the V entries of its columns have been rotated by every earlier row.
// Those V states have a closed form:
//
//   P = L^{-T} V,  G_b = P_{<b}^T P_{<b},  U_b = chol_lower(I + sigma G_b),
//   V-state of column m at the start of row block b  =  U_b^{-1} r_m^{(b)},
//   r_m^{(b)} = v_m - sum_{i < bD} L_{i,m} p_i  (the forward-substitution residual),
//
// which is exact (U_b^{-1} is the product of the lower-triangular k x k maps the
// rotations of rows < bD induce on V, the unique one with U^{-T}... = (I+sigma G)^{-1}).
// So every diagonal block runs the paper's Compute/Apply sweep INDEPENDENTLY
// (same rotations, same V_exit up to rounding) and every off-diagonal D x D tile
// is an independent Apply task.  The only serial chain left is the triangular
// solve for P, whose links are one FMA + one MUL instead of a sqrt/div chain.
//
// Kernels (one pass per <= 32 update columns; k > 32 runs ceil(k/32) passes =
// sequential rank-32 modifications, R3):
//   trsv_kernel   persistent, cooperative (one CTA per SM): CTAs 0..NC-1 = the chains
//                 (P in 32-row blocks, kRPC right-hand sides each, operands N/M/X
//                 precomputed), CTA NC = the Gram prefix sums, the rest = strip owners
//                 (J1 operands, then right-looking residual updates + Apply checkpoints),
//                 which take diagonal-sweep tickets once their strips are done (worker
//                 mode: bdiag_body per 64-row block, in parallel as the chain advances).
//   btma_kernel   Apply of each block's panel to 64 x 256 off-diagonal tiles (TMA boxes,
//                 scaled 2-FMA rotations from the checkpointed V states); launched as a
//                 programmatic dependent of trsv_kernel, waiting on per-block flags.
//   btile_kernel / bapply_kernel: the Apply as a plain launch after the TRSV kernel
//                 (unaligned L or odd ldl, or checkpoint interval CI > 1).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "bparts.cuh"
#include "internal.h"
#include "rot.cuh"
#include "tma.cuh"

namespace gcm {

namespace {

constexpr int kDT = 32;            // rows per triangular-solve block
constexpr int kTrsvThreads = 288;  // chain CTA: 2 critical + 6 prep + loader warps;
                                   // helper CTA: 8 compute warps + 1 feeder warp
constexpr int kBKMax = 32;         // update columns per pass
constexpr int kApplyT = 64;        // threads per apply CTA (= kD columns)
constexpr int kLdT = kDT + 1;
constexpr int kLdR = kDT + 4;  // column stride of a helper's ring tiles (conflict-free MMA fragments)
#ifndef GCM_LOOKC
#define GCM_LOOKC 4
#endif
constexpr int kLookC = GCM_LOOKC;       // blocks of lookahead the chain absorbs
constexpr int kSeg = (kLookC - 1) * kDT;  // rows of the prepared part of a lookahead segment (lags 2..kLookC)
constexpr int kLdN = kSeg + 1;            // row stride of N (odd: lane = j reads are conflict-free)
// Per 32-row block tb the helpers precompute (J1), contiguous so one bulk copy stages it:
//   N   [kDT][kLdN]  N(j, R) = sum_q X(q, j) L(rs + R, tb*32 + q),  rs = (tb - kLookC) * 32
//   M^T [kDT][kDT]   M = X^T L_{tb-1,tb}^T
//   X   [kDT][kDT]   X = L_{tb,tb}^{-1} (row-major)
// so the chain's prepared value is  prepX_tb = X^T r^{hand} - N p_seg  (no X matvec after the sums).
constexpr int kMXN = kDT * kLdN;
constexpr int kMXStride = ((kMXN + 2 * kDT * kDT) + 1) / 2 * 2;  // doubles per block (16-byte multiple)

#ifndef GCM_POLL_NS
#define GCM_POLL_NS 20
#endif

struct Layout {
    int64_t n;
    int k;
    int NT, NB, CI;
    int64_t nchk;
    size_t P, rcur, rchain, pfast, MX, chk, G, Q, U, panels, flags, hprog, total;
};


// chk_count_before for CI = 2^CIlog without a 64-bit division (device hot loop)
__device__ __forceinline__ int64_t chk_count_before_pow2(int s, int CIlog) {
    const int S = s - 1;
    if (S <= 0) return 0;
    const int64_t q = S >> CIlog, r = S & ((1 << CIlog) - 1);
    return ((q * (q + 1) / 2) << CIlog) + (q + 1) * r;
}

// rank padding of a pass (the kernels' template KB)
__host__ __device__ constexpr int kb_of(int k) { return k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32; }

Layout make_layout(int64_t n, int k, size_t chk_budget) {
    Layout l{};
    l.n = n;
    l.k = k;
    l.NT = (int)((n + kDT - 1) / kDT);
    l.NB = (int)((n + kD - 1) / kD);
    l.CI = 1;
    for (;;) {
        l.nchk = chk_count_before(l.NB, l.CI);
        if ((size_t)l.nchk * kD * k * sizeof(double) <= chk_budget || l.CI >= l.NB) break;
        l.CI *= 2;
    }
    size_t o = 0;
    auto take = [&](size_t doubles) {
        const size_t at = o;
        o += ((doubles * sizeof(double) + 255) / 256) * 256;
        return at;
    };
    l.P = take((size_t)l.NT * kDT * k);  // padded to whole 32-row blocks (bulk copies)
    l.rcur = take((size_t)l.NT * kDT * k);
    l.rchain = take((size_t)l.NT * kDT * k);
    // rchain .. hprog are armed by ONE memset (all-ones) at the start of every pass: the
    // hand-off slots and pfast start empty, the ticket counter at -1, and no flag or
    // progress word can equal the pass's epoch (never 0 or all-ones) before it is published
    l.pfast = take((size_t)l.NT * kDT * k + 2);  // + ticket counter
    l.flags = take(((2ull * l.NT + 2ull * l.NB) * sizeof(unsigned) + 7) / 8);  // lflag, qflag, uflag, bflag
    l.hprog = take((size_t)l.NT + 1);
    l.MX = take((size_t)l.NT * kMXStride);
    l.chk = take((size_t)l.nchk * kD * k);
    l.G = take((size_t)l.NB * kb_of(k) * kb_of(k));     // Gram prefixes G_b (KB x KB)
    l.Q = take((size_t)l.NT * kb_of(k) * kb_of(k));     // per 32-row block P_tb^T P_tb (helpers)
    l.U = take((size_t)l.NB * kb_of(k) * kb_of(k));       // U_b^{-1}, KB x KB, zero padded
    l.panels = take((size_t)l.NB * panel_doubles(kb_of(k)));  // coefficient panels, stride KB
    l.total = o;
    return l;
}


#ifdef GCM_TRACE
__device__ __forceinline__ long long gtime() {
    long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
__device__ long long g_htrace[4096 * 8];  // hand-off timeline in globaltimer ns, indexed by strip s
#define HTRACE(slot, s) (g_htrace[(s) * 8 + (slot)] = gtime())
#define CTRACE(slot, s) (g_trace[(s) * 8 + (slot)] = clock64())
// kernel timeline (globaltimer ns, max over CTAs): 0 trsv entry, 1 J1 done, 2 chain start, 3 chain end, 4 btma end
#define JMARK(slot) (g_htrace[2001 * 8 + (slot)] = gtime())
#define TLINE(slot) atomicMax(reinterpret_cast<unsigned long long *>(&g_htrace[2000 * 8 + (slot)]), (unsigned long long)gtime())
// one helper's per-tile phases (clock64), rows = tile sequence number
#define HPT(slot, val) ((h == 100 && t == 0 && seq < 2900) ? (void)(g_htrace[seq * 8 + (slot)] = (val)) : (void)0)
__device__ long long g_trace[4096 * 8];
#define TRACE(slot, tb) (blockIdx.x == 0 ? (void)(g_trace[(tb) * 8 + (slot)] = clock64()) : (void)0)
#else
#define TRACE(slot, tb) ((void)0)
#define HTRACE(slot, s) ((void)0)
#define CTRACE(slot, s) ((void)0)
#define HPT(slot, val) ((void)0)
#define TLINE(slot) ((void)0)
#define JMARK(slot) ((void)0)
#endif

// Bytes of Apply checkpoints before the checkpoint interval CI doubles (2 GiB;
// GCM_CHK_BUDGET overrides it per call -- the tests use it to exercise CI > 1).
Layout make_layout(int64_t n, int k, size_t chk_budget);
size_t chk_budget(int64_t n, int kc) {
    const char *e = std::getenv("GCM_CHK_BUDGET");
    if (e) return (size_t)std::strtoull(e, nullptr, 10);
    // at least 2 GiB, up to a quarter of the free device memory when more lets the checkpoint
    // interval drop to 1 (n = 100000: 20 GB of checkpoints next to its 80 GB factor, and the
    // TMA Apply path). Sticky: the cached workspace keeps what it was granted, and
    // cudaMemGetInfo (milliseconds) is only asked when the current budget gives CI > 1.
    static size_t high_water = (size_t)(2ull << 30);
    if (make_layout(n, kc, high_water).CI > 1) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) high_water = std::max(high_water, free_b / 4);
    }
    return high_water;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    chaos_delay();
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Hand-off values are self-validating: rchain starts all-ones (a NaN no
// producer writes, see handoff_value) and each chain thread polls its own
// 8-byte value, so the hand-off needs no flag, no fence and no second round trip.
__device__ __forceinline__ double handoff_value(double v) {
    return v == v ? v : __longlong_as_double(0x7ff8000000000000ll);  // NaNs canonicalised
}
__device__ __forceinline__ void st_handoff(double *p, double v) {
    chaos_delay();
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(handoff_value(v)) : "memory");
}
__device__ __forceinline__ double ld_handoff(double *p) {
    chaos_delay();
    unsigned long long u;
    do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(u) : "l"(p) : "memory");
    } while (u == kEmpty);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(kEmpty) : "memory");  // re-arm for the next call
    return __longlong_as_double((long long)u);
}
__device__ __forceinline__ void st_release64(unsigned long long *p, unsigned long long v) {
    chaos_delay();
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    chaos_delay();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// CTA-wide publish: every thread's prior global stores, then *f = epoch.
__device__ __forceinline__ void cta_publish(unsigned *f, unsigned epoch) {
    chaos_delay();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release(f, epoch);
    }
}

struct TrsvArgs {
    const double *L;
    int64_t n, ldl;
    const double *V;  // this pass's first column (ld n)
    int k;
    double *P, *rcur, *rchain, *pfast, *chk;  // pfast: self-validating copy of P for the hand-off tiles
    double *MX;       // per 32-block (kMXStride doubles): N, M^T, X (see kMXN)
    bool bulk_ok;     // L 16-byte aligned and ldl even (the Apply's TMA path)
    int CI, CIlog;  // checkpoint interval (a power of two) and its log2
    int NC;           // chain CTAs (each solves kRPC right-hand sides)
    unsigned *lflag;
    unsigned epoch;
    double *G, *Ui;   // Gram prefixes G_b = P_{<b}^T P_{<b} and U_b^{-1} (U_b = chol_lower(I + sigma G_b))
    double *Q;        // per 32-row block Q_tb = P_tb^T P_tb (KB x KB), by the helper of strip tb+1
    unsigned *qflag;  // [NT] epoch when Q_tb is stored
    int sigma;
    // fused diagonal sweeps: helpers whose strips are done run bdiag tasks (ticket order)
    double *Vw;               // this pass's V (V_exit written by the sweeps)
    double *panels;           // coefficient panels
    unsigned long long *key;  // first-failure key
    int64_t ebase;            // first update column of this pass
    unsigned *uflag;          // [NB] epoch when what block b's sweep needs from the Gram CTA is stored
    unsigned *taskctr;        // ticket counter (armed to all-ones by the pass's memset)
    int publish;              // 1: publish sweep flags and helper tile-row progress (overlapped Apply)
    int own_cap;              // strip residuals a helper keeps in shared memory (<= help_max_own(KB))
    int H;                    // helper CTAs (strip s is owned by helper s % H)
    unsigned *bflag;          // [NB] epoch when block b's sweep (panel, U_b^{-1}) is stored
    unsigned long long *hprog;  // [H] (epoch << 32) | tile rows a helper has finished (published by its feeder)
};

constexpr int kRPC = 2;                 // right-hand sides per chain CTA
constexpr int kPrepWarps = 6;           // chain CTA warps: 0..kRPC-1 critical, then prep, then the loader
constexpr int kPrepThreads = kPrepWarps * 32;
constexpr int kSvcWarp = kRPC + kPrepWarps;  // loader warp
constexpr int kWin = kLookC <= 4 ? 128 : kLookC <= 8 ? 256 : 512;  // rows of the chain's p window (pow2 >= kLookC*kDT)
static_assert(kWin >= kLookC * kDT && kLookC <= 16, "p window indexed by row & (kWin - 1)");
// strips whose residual a helper keeps in shared memory (the rest round-trip through L2 on
// every tile): at large n a helper owns ~n/(32*139) strips (24 at n = 100000)
// (GCM_HELP_OWN_CAP=<m> lowers it at run time: the tests use it to drive the spill path,
// which the default only reaches at n > ~50k (KB = 32) / ~107k (KB <= 16))
__host__ __device__ constexpr int help_max_own(int KB) { return KB <= 16 ? 24 : 12; }
#ifndef GCM_HELP_RING
#define GCM_HELP_RING 3
#endif
constexpr int kHelpRing = GCM_HELP_RING;  // tiles (L tile + P block) a helper's feeder keeps in flight
// (3: a deeper ring bulk-copies P blocks before the chains have written them, and the compute
// warps then re-poll every value; profiles/r02ar_ab_helper_ring.txt)
#ifndef GCM_FASTBACK
#define GCM_FASTBACK 2
#endif
constexpr int kFastBack = GCM_FASTBACK;         // tiles before the hand-off tile that also read P from pfast
constexpr int kHelpCompute = 256;       // helper compute threads (warps 0..7); warp 8 feeds
static_assert((kSvcWarp + 1) * 32 <= kTrsvThreads, "chain CTA needs a loader warp");

// Tile (tb, s) takes P_tb from pfast (no progress word, no bulk copy) when it is
// the strip's hand-off tile or one of the kFastBack before it: those sit on the
// chain's critical loop, the earlier ones have slack for the published path.
__device__ __forceinline__ bool fast_tile(int tb, int s) {
    return tb + 1 <= s - kLookC && tb + 1 >= s - kLookC - kFastBack;
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// Shared-memory plan of a chain CTA (doubles).  A "stage" holds block tb's
// precomputed operands (N, M^T, X: one bulk copy of kMXStride doubles); three
// stages rotate.
struct ChainSmem {
    static constexpr int stage = kMXStride;
    static constexpr int off_stage = 0;                                   // [3][stage]
    static constexpr int off_pwin = off_stage + 3 * stage;                // [kWin][kRPC]  p by row & (kWin-1)
    static constexpr int off_part = off_pwin + kWin * kRPC;               // [kPrepWarps][kDT][kRPC]
    static constexpr int off_hand = off_part + kPrepWarps * kDT * kRPC;   // [kDT][kRPC]  hand-off residual
    static constexpr int off_prepx = off_hand + kDT * kRPC;               // [2][kDT][kRPC]
    static constexpr int off_bar = off_prepx + 2 * kDT * kRPC;            // 3 mbarriers (u64) + pcount
    static constexpr int total = off_bar + 4;
};

// ---------------------------------------------------------------- chain CTA
// CTA c solves L^T p = v for the right-hand sides e = kRPC*c .. kRPC*c+kRPC-1,
// 32 rows (one block tb) per step:
//   critical warps (one per RHS, lane = row j):  p_tb = prepX_tb - M_tb p_{tb-1}
//        with M_tb = X_tb^T L_{tb-1,tb}^T precomputed by the helpers (X_tb = L_tb,tb^{-1});
//   prep warps: prepX_{tb+1} = X_{tb+1}^T r^{(tb+1-kLookC)} - N_{tb+1} p_{rows of blocks tb-kLookC+2 .. tb-1},
//        r^{(.)} handed over by the helper owning strip tb+1 (its load is issued first),
//        N = X^T L_seg^T precomputed, the rows split evenly over the prep warps;
//   loader warp: streams block tb+3's operands (one bulk copy) on a per-stage mbarrier.
// The k right-hand sides are independent, so chain CTAs never talk to each other;
// the helpers read p from the self-validating copy pfast (no progress words).
__device__ void trsv_chain(const TrsvArgs &a, double *smem, int c) {
    using S = ChainSmem;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int NT = (int)((a.n + kDT - 1) / kDT);
    const int k = a.k;
    const int e0 = c * kRPC;
    double *pwin = smem + S::off_pwin;
    double *part = smem + S::off_part;
    double *hand = smem + S::off_hand;
    double *prepx = smem + S::off_prepx;
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + S::off_bar);
    auto stage_of = [&](int tb) { return smem + S::off_stage + (tb % 3) * S::stage; };

    // loader warp: bring block tb's operands into stage tb % 3
    auto issue_loads = [&](int tb) {
        if (lane == 0) {
            while (ld_acquire(a.lflag + tb) != a.epoch) {
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");  // helpers' generic stores -> bulk read
            unsigned long long *bar = bars + (tb % 3);
            mbar_arrive_expect_tx(bar, (unsigned)kMXStride * 8u);
            bulk_g2s(stage_of(tb), a.MX + (int64_t)tb * kMXStride, (unsigned)kMXStride * 8u, bar);
        }
        __syncwarp();
    };

    // critical warps count published p blocks here (monotonic; a named barrier
    // could be overrun because the critical warps may run two steps ahead of the
    // loader warp)
    volatile unsigned *pcount = reinterpret_cast<volatile unsigned *>(bars + 3);
    if (t == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(bars + i, 1u);
        *pcount = 0u;
    }
    for (int i = t; i < kWin * kRPC; i += blockDim.x) pwin[i] = 0.0;  // rows < 0 of early segments (N is 0 there)
    __syncthreads();
    if (warp == kSvcWarp)
        for (int tb = 0; tb < 3 && tb < NT; ++tb) issue_loads(tb);

    // prep warps: prepX for block tb (needs p up to tb-2, i.e. <= step tb-1 of the critical warps)
    const int pt = t - kRPC * 32;
    auto do_prep = [&](int tb) {
        const double *st = stage_of(tb);
        // the hand-off value is usually stored before it is needed: issue its load
        // first so its L2 round trip overlaps the stage wait and the partial sums
        double *hptr = nullptr;
        unsigned long long hv = 0ull;  // rows past n / padded RHS: 0
        if (pt < kDT * kRPC) {
            const int jj = pt / kRPC, w = pt % kRPC;
            const int e = e0 + w;
            const int64_t row = (int64_t)tb * kDT + jj;
            if (e < k && row < a.n) {
                hptr = a.rchain + (int64_t)tb * kDT * k + (int64_t)jj * k + e;
                hv = ld_relaxed_u64(hptr);
            }
        }
        mbar_wait(bars + (tb % 3), (unsigned)((tb / 3) & 1));
        if (pt == 0) TRACE(3, tb - 1);
        const int pw = pt >> 5, j = lane;
        const int rs = (tb - kLookC) * kDT;  // first segment row (may be < 0: N is zero there)
        double acc0[kRPC], acc1[kRPC];
#pragma unroll
        for (int w = 0; w < kRPC; ++w) acc0[w] = acc1[w] = 0.0;
        {  // - N p over this warp's share of the kSeg segment rows: every shared load of the
           // share issued before the first FMA (a load-FMA loop left each iteration waiting on
           // its own loads: ~1.3k cycles per step, the chain's largest phase)
            constexpr int kPer = (kSeg + kPrepWarps - 1) / kPrepWarps;
            const int r0 = pw * kPer;
            const double *nrow = st + j * kLdN;
            double l[kPer];
            double2 pv[kPer];
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int R = r0 + q;
                const bool in = kSeg % kPrepWarps == 0 || R < kSeg;
                l[q] = in ? nrow[R] : 0.0;
                pv[q] = in ? *reinterpret_cast<const double2 *>(pwin + ((rs + R) & (kWin - 1)) * kRPC)
                           : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                if (q & 1) {
                    acc1[0] = fma(-l[q], pv[q].x, acc1[0]);
                    acc1[1] = fma(-l[q], pv[q].y, acc1[1]);
                } else {
                    acc0[0] = fma(-l[q], pv[q].x, acc0[0]);
                    acc0[1] = fma(-l[q], pv[q].y, acc0[1]);
                }
            }
        }
        if (pt == 0) TRACE(4, tb - 1);
        if (hptr) {
            if (pt == 0 && c == 0) HTRACE(0, 3500 + tb);
            if (hv == kEmpty) {
                hv = __double_as_longlong(ld_handoff(hptr));
            } else {  // prefetched: re-arm the slot for the next call
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(hptr), "l"(kEmpty) : "memory");
            }
            if (pt == 0 && c == 0) HTRACE(6, 3000 + tb);
        }
        if (pt < kDT * kRPC) hand[pt] = __longlong_as_double((long long)hv);
        if (pt == 0) TRACE(5, tb - 1);
        named_bar(2, kPrepThreads);
        {  // + X^T r^{hand} over this warp's share of the 32 rows q
            constexpr int kPerX = (kDT + kPrepWarps - 1) / kPrepWarps;
            const double *X = st + kMXN + kDT * kDT;
            double x[kPerX];
            double2 hvv[kPerX];
#pragma unroll
            for (int u = 0; u < kPerX; ++u) {  // loads first (as above)
                const int q = pw * kPerX + u;
                x[u] = q <= j ? X[q * kDT + j] : 0.0;
                hvv[u] = q <= j ? *reinterpret_cast<const double2 *>(hand + q * kRPC) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < kPerX; ++u) {
                const int q = pw * kPerX + u;
                // X = L_tb,tb^{-1} is upper triangular: X(q, j) = 0 for q > j is skipped, not
                // multiplied -- a NaN residual of a later row must not reach row j (0 * NaN),
                // or a NaN input would be reported at an earlier row (R5, R6)
                if (q <= j) {
                    acc0[0] = fma(x[u], hvv[u].x, acc0[0]);
                    acc0[1] = fma(x[u], hvv[u].y, acc0[1]);
                }
            }
        }
#pragma unroll
        for (int w = 0; w < kRPC; ++w) part[(pw * kDT + j) * kRPC + w] = acc0[w] + acc1[w];
        named_bar(2, kPrepThreads);
        if (pt < kDT * kRPC) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < kPrepWarps; ++q) acc += part[q * kDT * kRPC + pt];
            prepx[(tb & 1) * kDT * kRPC + pt] = acc;
        }
    };
    static_assert(kRPC == 2, "prep vectorises the two right-hand sides");

    double mrow[kDT];  // critical warps: row j of M_tb in registers
    if (warp >= kRPC && warp < kSvcWarp) do_prep(0);
    if (warp < kRPC) {
        const double *st = stage_of(0);
        mbar_wait(bars + 0, 0u);
#pragma unroll
        for (int m = 0; m < kDT; ++m) mrow[m] = st[kMXN + m * kDT + lane];  // M^T stored: (m, j)
    }
    if (warp < kSvcWarp) named_bar(1, kSvcWarp * 32);  // B_0

    if (warp == kSvcWarp) {  // loader: block tb+3 into stage tb%3 once step tb is under way
        for (int tb = 0; tb + 3 < NT; ++tb) {
            if (lane == 0) {
                while (*pcount < (unsigned)(kRPC * (tb + 1))) {
                }
            }
            __syncwarp();
            issue_loads(tb + 3);
            if (lane == 0) TRACE(7, tb);
        }
        return;
    }
    if (warp > kSvcWarp) return;
    if (t == 0) TLINE(2);
    for (int tb = 0; tb < NT; ++tb) {
        if (warp < kRPC) {
            const int w = warp, j = lane;
            if (t == 0) TRACE(0, tb);
            double a0 = prepx[(tb & 1) * kDT * kRPC + j * kRPC + w], a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (t == 0 && c == 0) HTRACE(7, 3000 + tb);
            if (tb > 0) {
                const double *pprev = pwin + (((tb - 1) * kDT) & (kWin - 1)) * kRPC + w;
#pragma unroll
                for (int m = 0; m < kDT; m += 4) {
                    a0 = fma(-mrow[m], pprev[m * kRPC], a0);
                    a1 = fma(-mrow[m + 1], pprev[(m + 1) * kRPC], a1);
                    a2 = fma(-mrow[m + 2], pprev[(m + 2) * kRPC], a2);
                    a3 = fma(-mrow[m + 3], pprev[(m + 3) * kRPC], a3);
                }
            }
            const double p = (a0 + a1) + (a2 + a3);
            pwin[(((tb * kDT) & (kWin - 1)) + j) * kRPC + w] = p;
            const int e = e0 + w;
            const int64_t row = (int64_t)tb * kDT + j;
            if (e < k && row < a.n) {
                st_handoff(a.pfast + row * k + e, p);  // polled by the helpers (every tile) and the Gram path
                a.P[row * k + e] = p;
                if (t == 0 && c == 0) HTRACE(0, 3000 + tb + kLookC + 1);
            }
            if (t == 0) TRACE(1, tb);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                atomicAdd(const_cast<unsigned *>(pcount), 1u);
            }
            if (tb + 1 < NT) {  // M_{tb+1} row into registers while the prep warps finish
                const double *st = stage_of(tb + 1);
                mbar_wait(bars + ((tb + 1) % 3), (unsigned)(((tb + 1) / 3) & 1));
#pragma unroll
                for (int m = 0; m < kDT; ++m) mrow[m] = st[kMXN + m * kDT + lane];
            }
        } else if (tb + 1 < NT) {
            if (pt == 0) TRACE(2, tb);
            do_prep(tb + 1);
            if (pt == 0) TRACE(6, tb);
        }
        named_bar(1, kSvcWarp * 32);  // B_{tb+1}: p_tb and prepX_{tb+1} ready
    }
    if (t == 0) TLINE(3);
}

// ---------------------------------------------------------------- helper CTAs
template <int KB>
__device__ unsigned long long *trsv_helper(const TrsvArgs &a, double *smem, int h, int H) {
    double *Lb = smem;                      // [kDT][kLdT]
    double *Pt = Lb + kDT * kLdT;           // [kDT][max(KB, kLdT)]  (P block; X during J1)
    constexpr int kHelpMaxOwn = help_max_own(KB);
    double *rs = Pt + kDT * (KB > kLdT ? KB : kLdT);  // [kHelpMaxOwn][kDT][KB] residuals of owned strips
    const int t = threadIdx.x;
    const int k = a.k;
    const int NT = (int)((a.n + kDT - 1) / kDT);

    // J2 set-up first (residual = V of every owned strip, the early hand-offs and the tile
    // (0, s) checkpoints): the chain's first steps wait on those hand-offs, which used to come
    // after all of this helper's J1 blocks.  Column strips s = h, h+H, ...
    auto rptr = [&](int i, int s) -> double * {  // residual of owned strip #i (smem or global)
        return i < a.own_cap ? rs + i * kDT * KB : a.rcur + (int64_t)s * kDT * k;
    };
    auto rstride = [&](int i) { return i < a.own_cap ? KB : k; };
    int last = -1, i = 0;
    for (int s = h; s < NT; s += H, ++i) {
        last = s;
        const int64_t c0 = (int64_t)s * kDT;
        const int nc = (int)imin64(kDT, a.n - c0);
        double *r = rptr(i, s);
        const int ld = rstride(i);
        for (int o = t; o < kDT * k; o += kTrsvThreads) {
            const int cc = o / k, e = o % k;
            const double v = cc < nc ? a.V[(c0 + cc) + (int64_t)e * a.n] : 0.0;
            r[cc * ld + e] = v;
            if (s - kLookC <= 0 && cc < nc) st_handoff(a.rchain + c0 * k + o, v);
            const int s64 = s / 2;
            if (s64 >= 1 && cc < nc)
                a.chk[((int64_t)chk_count_before(s64, a.CI)) * kD * k + ((s % 2) * kDT + cc) * k + e] = v;
        }
    }
    __syncthreads();
    // J1: per 32-block tb: X = L_tb,tb^{-1} (upper) and M = X^T L_{tb-1,tb}^T, the
    // operands of the chain's critical step  p_tb = X^T prep - M p_{tb-1}.
    for (int tb = h; tb < NT; tb += H) {
        if (t == 0 && h == 0 && tb == 0) JMARK(0);
        const int64_t r0 = (int64_t)tb * kDT;
        const int nr = (int)imin64(kDT, a.n - r0);
        double *Xs = Pt;  // reuse: [kDT][kLdT]  Xs[q][j] = X(q, j)   (needs kDT*kLdT <= kDT*KB + ... see smem plan)
        for (int idx = t; idx < kDT * kDT; idx += kTrsvThreads) {
            const int c = idx / kDT, m = idx % kDT;
            double v = 0.0;
            if (c < nr && m <= c) v = a.L[(r0 + m) + (r0 + c) * a.ldl];
            else if (c >= nr && m == c) v = 1.0;  // identity padding
            Lb[c * kLdT + m] = v;
        }
        __syncthreads();
        if (t == 0 && h == 0 && tb == 0) JMARK(1);
        // X column c by back substitution in column (axpy) form: x_j = acc_j / L_jj, then
        // acc_i -= L(i, j) x_j for i < j -- 32 independent running sums per thread, so the
        // dependent chain is one multiply + one FMA per row (the row form chained ~16 FMAs and
        // a division per row: 15 us of the kernel's start-up).  Columns j > c are skipped, not
        // multiplied by zero (NaN inputs).
        double *rd = rs + kHelpMaxOwn * kDT * KB + kDT * kLdN;  // [kDT] in the idle ring, after the segment
        if (t < kDT) rd[t] = 1.0 / Lb[t * kLdT + t];
        __syncthreads();
        if (t < kDT) {
            const int c = t;
            double acc[kDT];
#pragma unroll
            for (int i = 0; i < kDT; ++i) acc[i] = i == c ? 1.0 : 0.0;
#pragma unroll
            for (int j = kDT - 1; j >= 0; --j) {
                if (j <= c) {
                    acc[j] *= rd[j];
#pragma unroll
                    for (int i = 0; i < j; ++i) acc[i] = fma(-Lb[j * kLdT + i], acc[j], acc[i]);
                }
            }
#pragma unroll
            for (int j = 0; j < kDT; ++j) Xs[j * kLdT + c] = j <= c ? acc[j] : 0.0;
        }
        __syncthreads();
        if (t == 0 && h == 0 && tb == 0) JMARK(2);
        // Lb <- L tile (rows of block tb-1, columns of block tb):  Lb[q][m] = L(row (tb-1)*32+m, col tb*32+q)
        for (int idx = t; idx < kDT * kDT; idx += kTrsvThreads) {
            const int q = idx / kDT, m = idx % kDT;
            Lb[q * kLdT + m] = (tb > 0 && q < nr) ? a.L[(r0 - kDT + m) + (r0 + q) * a.ldl] : 0.0;
        }
        // segment (rows rs .. rs+kSeg-1 = blocks tb-kLookC .. tb-2, columns of block tb) into the
        // (still idle) tile ring:  sg[q][R] = L(rs + R, tb*32 + q), zero above row 0
        double *sg = rs + kHelpMaxOwn * kDT * KB;
        const int64_t rseg = r0 - (int64_t)kLookC * kDT;
        for (int idx = t; idx < kDT * kSeg; idx += kTrsvThreads) {
            const int q = idx / kSeg, R = idx % kSeg;
            sg[q * kLdN + R] = (q < nr && rseg + R >= 0) ? a.L[(rseg + R) + (r0 + q) * a.ldl] : 0.0;
        }
        __syncthreads();
        if (t == 0 && h == 0 && tb == 0) JMARK(3);
        double *mx = a.MX + (int64_t)tb * kMXStride;
        for (int idx = t; idx < kDT * kDT; idx += kTrsvThreads) {
            const int m = idx / kDT, j = idx % kDT;  // M(j, m) = sum_{q <= j} X(q, j) L(m, q)
            // X is upper triangular: the q > j terms are skipped, not multiplied by zero, so a
            // NaN entry of a later column cannot reach row j (R5, R6)
            // (fully unrolled with the q > j FMAs predicated off: the loads pipeline)
            double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < kDT; ++q) {
                const double xv = Xs[q * kLdT + j], lv = Lb[q * kLdT + m];
                if (q <= j) s[q & 3] = fma(xv, lv, s[q & 3]);
            }
            mx[kMXN + m * kDT + j] = (s[0] + s[1]) + (s[2] + s[3]);  // M^T row-major: (m, j)
            mx[kMXN + kDT * kDT + m * kDT + j] = Xs[m * kLdT + j];   // X row-major: (q=m, j)
        }
        for (int idx = t; idx < kDT * kSeg; idx += kTrsvThreads) {
            const int j = idx / kSeg, R = idx % kSeg;  // N(j, R) = sum_{q <= j} X(q, j) L(rs + R, q)
            double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < kDT; ++q) {
                const double xv = Xs[q * kLdT + j], lv = sg[q * kLdN + R];
                if (q <= j) s[q & 3] = fma(xv, lv, s[q & 3]);
            }
            mx[j * kLdN + R] = (s[0] + s[1]) + (s[2] + s[3]);
        }
        cta_publish(a.lflag + tb, a.epoch);
        if (t == 0 && h == 0 && tb == 0) JMARK(4);
    }
    if (t == 0) TLINE(1);

    // Tiles (tb, s), s owned and > tb, in tb-major order, flow through a ring of
    // kHelpRing shared-memory slots (L tile + P block).  Warp 8 (the feeder) runs
    // ahead: it issues the static L tile as soon as a slot is free, waits until
    // every chain has published P_tb, copies P_tb, and the slot's mbarrier completes
    // when both cp.async batches land.  Warps 0..7 only compute, so a helper's
    // tile throughput is its GEMM, not its memory and polling latency.
    int nown = 0;
    for (int s = h; s < NT; s += H) ++nown;

    struct It {
        int tb, ii;
    };
    auto first_owned_after = [&](int tb) { return tb < h ? 0 : (tb - h) / H + 1; };
    auto valid = [&](const It &x) { return x.tb < last && x.ii < nown; };
    auto advance = [&](It &x) {
        if (++x.ii >= nown) {
            ++x.tb;
            x.ii = first_owned_after(x.tb);
        }
    };
    constexpr int kSlot = kDT * kLdR + kDT * KB;  // L tile [32][kLdR] + P block [32][k] (dense, bulk copy)
    double *ring = rs + kHelpMaxOwn * kDT * KB;  // [kHelpRing][kSlot]
    unsigned long long *full = reinterpret_cast<unsigned long long *>(ring + kHelpRing * kSlot);
    unsigned long long *empty = full + kHelpRing;
    if (t == 0) {
        for (int i = 0; i < kHelpRing; ++i) {
            mbar_init(full + i, 33u);  // 1 noinc arrival per feeder lane (L batch) + the P bulk copy's arrive
            mbar_init(empty + i, kHelpCompute / 32);
        }
    }
    __syncthreads();
    const int warp = t >> 5, lane = t & 31;
    if (warp == kHelpCompute / 32) {
        // ------------------------------------------------------------ feeder
        // progress for the fused Apply tiles: once a slot's previous tile is consumed, the
        // tile rows it completed are published (a ring's lag behind the compute warps)
        int slot_row[kHelpRing];
#pragma unroll
        for (int i = 0; i < kHelpRing; ++i) slot_row[i] = -1;
        // each publication is a release (the feeder stalls until the checkpoints are out), so
        // publish every 64 rows for KB = 16 and every 128 for smaller ranks (same-box A/B)
        constexpr int kPubEvery = KB >= 16 ? 1 : 3;
        auto publish = [&](int rows) {
            if (lane == 0) st_release64(a.hprog + h, ((unsigned long long)a.epoch << 32) | (unsigned)rows);
        };
        int seq = 0;
        for (It it{0, first_owned_after(0)}; valid(it); advance(it), ++seq) {
            const int slot = seq % kHelpRing, use = seq / kHelpRing;
            if (use > 0) mbar_wait(empty + slot, (unsigned)((use - 1) & 1));
#pragma unroll
            for (int i = 0; i < kHelpRing; ++i)
                if (i == slot) {
                    if (use > 0 && slot_row[i] >= 0 && a.publish && (slot_row[i] & kPubEvery) == kPubEvery) publish(slot_row[i] + 1);
                    slot_row[i] = it.ii == nown - 1 ? it.tb : -1;
                }
            double *stg = ring + slot * kSlot;
            const int s = h + it.ii * H;
            const int64_t c0 = (int64_t)s * kDT;
            const int nc = (int)imin64(kDT, a.n - c0);
            for (int cc = 0; cc < nc; ++cc)  // lane = row: coalesced 256-byte column segments
                cp_async8(stg + cc * kLdR + lane, a.L + ((int64_t)it.tb * kDT + lane) + (c0 + cc) * a.ldl);
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(full + slot)) : "memory");
            if (fast_tile(it.tb, s)) {  // tiles next to the hand-off: the compute warps poll pfast themselves
                if (lane == 0) mbar_arrive(full + slot);
                continue;
            }
            if (lane == 0) {  // P_tb (32 x k, contiguous) from pfast with one bulk copy; values still
                              // empty on arrival are polled by the compute warps
                asm volatile("fence.proxy.async.global;" ::: "memory");
                const unsigned bytes = (unsigned)(kDT * k) * 8u;
                mbar_arrive_expect_tx(full + slot, bytes);
                bulk_g2s(stg + kDT * kLdR, a.pfast + (int64_t)it.tb * kDT * k, bytes, full + slot);
            }
        }
        cp_async_wait_all();
        if (a.publish) {  // every tile consumed: all rows
            for (int q = seq - kHelpRing > 0 ? seq - kHelpRing : 0; q < seq; ++q)
                mbar_wait(empty + q % kHelpRing, (unsigned)((q / kHelpRing) & 1));
            publish(NT);
        }
        return full;
    }
    // ---------------------------------------------------------------- compute warps
    int seq = 0;
    for (It pit{0, first_owned_after(0)}; valid(pit); advance(pit), ++seq) {
        const int tb = pit.tb;
        const int slot = seq % kHelpRing;
        HPT(0, clock64());
        mbar_wait(full + slot, (unsigned)((seq / kHelpRing) & 1));
        HPT(1, clock64());
        HPT(6, (long long)pit.tb);
        HPT(7, (long long)(h + pit.ii * H));
        if (t == 0 && pit.tb + 1 == h + pit.ii * H - kLookC) HTRACE(1, 3000 + h + pit.ii * H);
        const int ii = pit.ii;
        const int s = h + ii * H;
        const double *Lt = ring + slot * kSlot;
        const double *Pt = Lt + kDT * kLdR;
        const int64_t c0 = (int64_t)s * kDT;
        const int nc = (int)imin64(kDT, a.n - c0);
        double *r = rptr(ii, s);
        const int ld = rstride(ii);
        // r[c][e] -= sum_m L(m, c) P[m][e], register-blocked 2 columns x 2 update
        // columns per thread (EG = KB/2 e-pairs, 16 * EG threads): per row m one
        // L pair and one P pair feed four FMAs, so the tile costs ~kDT*(3 LDS +
        // 4 FMA) per thread -- this tile is on the hand-off's critical path and
        // shared-memory wavefronts, not FMAs, set its latency.
        const bool chain_handoff = (tb + 1 == s - kLookC);
        const int b64 = (tb + 1) / 2, s64 = s / 2;
        const bool checkpoint = ((tb + 1) % 2 == 0) && b64 < s64 && (b64 & (a.CI - 1)) == 0;
        const bool direct = fast_tile(tb, s);
        if (!direct) {  // bulk-copied P_tb: poll the values that were still empty
            double *Pw = const_cast<double *>(Pt);
            const double *src = a.pfast + (int64_t)tb * kDT * k;
            constexpr int kPerV = (kDT * KB + kHelpCompute - 1) / kHelpCompute;
            unsigned long long u[kPerV];
            unsigned miss = 0u;
#pragma unroll
            for (int q = 0; q < kPerV; ++q) {  // every missing value's load in flight at once
                const int o = t + q * kHelpCompute;
                u[q] = 0ull;
                if (o < kDT * k && __double_as_longlong(Pw[o]) == (long long)kEmpty) {
                    u[q] = ld_relaxed_u64(src + o);
                    miss |= 1u << q;
                }
            }
#pragma unroll
            for (int q = 0; q < kPerV; ++q) {
                if (miss >> q & 1u) {
                    const int o = t + q * kHelpCompute;
                    if (u[q] == kEmpty) u[q] = (unsigned long long)__double_as_longlong(ld_value(src + o));
                    Pw[o] = __longlong_as_double((long long)u[q]);
                }
            }
            named_bar(1, kHelpCompute);
        }
        if (direct) {  // P_tb straight from the chains' self-validating copy
            double *Pw = const_cast<double *>(Pt);
            const double *src = a.pfast + (int64_t)tb * kDT * k;
            constexpr int kPer = (kDT * KB + kHelpCompute - 1) / kHelpCompute;
            unsigned long long u[kPer];
#pragma unroll
            for (int q = 0; q < kPer; ++q) {  // issue every load first: one round trip, not kPer
                const int o = t + q * kHelpCompute;
                u[q] = o < kDT * k ? ld_relaxed_u64(src + o) : 0ull;
            }
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int o = t + q * kHelpCompute;
                if (o < kDT * k) {
                    if (u[q] == kEmpty) u[q] = __double_as_longlong(ld_value(src + o));
                    Pw[o] = __longlong_as_double((long long)u[q]);
                }
            }
            if (t == 0 && chain_handoff) HTRACE(2, 3000 + s);
            named_bar(1, kHelpCompute);
            if (t == 0 && chain_handoff) HTRACE(3, 3000 + s);
        }
        HPT(2, clock64());
        if constexpr (KB >= 8) {
            // r[c][e] -= sum_m L(m, c) P[m][e] on the FP64 tensor cores (DMMA m8n8k4: M = strip
            // columns, N = update columns, K = rows; warp = 8 columns x 8 * TPW update columns):
            // 8 dependent MMAs per output tile instead of ~32 DFMA rounds on shared loads
            constexpr int ET = KB / 8, TPW = ET >= 2 ? ET / 2 : 1;
            const int cw = warp % 4, eg = warp / 4;
            if (eg * TPW < ET) {
                const int gi = lane >> 2, tg = lane & 3;
                const int c = cw * 8 + gi;
                double acc[TPW][2];
#pragma unroll
                for (int v = 0; v < TPW; ++v) acc[v][0] = acc[v][1] = 0.0;
                const double *la = Lt + c * kLdR + tg;
#pragma unroll
                for (int m0 = 0; m0 < kDT; m0 += 4) {
                    const double af = la[m0];
#pragma unroll
                    for (int v = 0; v < TPW; ++v) {
                        const int e = (eg * TPW + v) * 8 + gi;
                        dmma_884(acc[v], af, e < k ? Pt[(m0 + tg) * k + e] : 0.0);
                    }
                }
                HPT(3, clock64());
                if (t == 0 && chain_handoff) HTRACE(4, 3000 + s);
                double *ck = checkpoint ? a.chk + (chk_count_before_pow2(s64, a.CIlog) + (b64 >> a.CIlog)) * kD * k +
                                              ((s % 2) * kDT + c) * k
                                        : nullptr;
#pragma unroll
                for (int v = 0; v < TPW; ++v)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int ee = (eg * TPW + v) * 8 + 2 * tg + hh;
                        if (c < nc && ee < k) {
                            double *rr = r + c * ld + ee;
                            const double nv = *rr - acc[v][hh];
                            *rr = nv;
                            if (chain_handoff) st_handoff(a.rchain + c0 * k + (int64_t)c * k + ee, nv);
                            if (chain_handoff && t == 0 && v == 0 && hh == 0) HTRACE(5, 3000 + s);
                            if (ck) ck[ee] = nv;  // the chain does not wait for these
                        }
                    }
            }
        } else {
            constexpr int EG = KB / 2;
            constexpr int kGemmT = 16 * EG;
            static_assert(kGemmT <= kHelpCompute, "helper GEMM threads");
            if (t < kGemmT) {
                const int cq = t / EG, eg = t % EG;
                const int ca = 2 * cq, e = 2 * eg;
                // four interleaved partial sums per output: FMA chains 8 deep, not 32
                double acc[4][4];
    #pragma unroll
                for (int q = 0; q < 4; ++q)
    #pragma unroll
                    for (int o = 0; o < 4; ++o) acc[q][o] = 0.0;
                if (e < k) {
                    const double *La = Lt + ca * kLdR, *Lb2 = La + kLdR;
                    if ((k & 1) == 0) {
    #pragma unroll
                        for (int m = 0; m < kDT; ++m) {
                            const double2 pv = *reinterpret_cast<const double2 *>(Pt + m * k + e);
                            const double la = La[m], lb = Lb2[m];
                            acc[m & 3][0] = fma(la, pv.x, acc[m & 3][0]);
                            acc[m & 3][1] = fma(la, pv.y, acc[m & 3][1]);
                            acc[m & 3][2] = fma(lb, pv.x, acc[m & 3][2]);
                            acc[m & 3][3] = fma(lb, pv.y, acc[m & 3][3]);
                        }
                    } else {
                        const bool e1 = e + 1 < k;
    #pragma unroll
                        for (int m = 0; m < kDT; ++m) {
                            const double p0 = Pt[m * k + e], p1 = e1 ? Pt[m * k + e + 1] : 0.0;
                            const double la = La[m], lb = Lb2[m];
                            acc[m & 3][0] = fma(la, p0, acc[m & 3][0]);
                            acc[m & 3][1] = fma(la, p1, acc[m & 3][1]);
                            acc[m & 3][2] = fma(lb, p0, acc[m & 3][2]);
                            acc[m & 3][3] = fma(lb, p1, acc[m & 3][3]);
                        }
                    }
                }
                const double s00 = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
                const double s01 = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
                const double s10 = (acc[0][2] + acc[1][2]) + (acc[2][2] + acc[3][2]);
                const double s11 = (acc[0][3] + acc[1][3]) + (acc[2][3] + acc[3][3]);
                const double sv[2][2] = {{s00, s01}, {s10, s11}};
                HPT(3, clock64());
                if (t == 0 && chain_handoff) HTRACE(4, 3000 + s);
                double vout[2][2];
    #pragma unroll
                for (int i = 0; i < 2; ++i) {
    #pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int c = ca + i, ee = e + j;
                        double v = 0.0;
                        if (c < nc && ee < k) {
                            double *rr = r + c * ld + ee;
                            *rr = v = *rr - sv[i][j];
                            if (chain_handoff) st_handoff(a.rchain + c0 * k + (int64_t)c * k + ee, v);
                            if (chain_handoff && t == 0 && i == 0 && j == 0) HTRACE(5, 3000 + s);
                        }
                        vout[i][j] = v;
                    }
                }
                if (checkpoint) {  // the chain does not wait for these
    #pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int c = ca + i;
                        double *ck = a.chk + (chk_count_before_pow2(s64, a.CIlog) + (b64 >> a.CIlog)) * kD * k +
                                     ((s % 2) * kDT + c) * k;
    #pragma unroll
                        for (int j = 0; j < 2; ++j)
                            if (c < nc && e + j < k) ck[e + j] = vout[i][j];
                    }
                }
            }
        }
        if (s == tb + 1) {  // this strip's last tile: the Gram contribution of P_tb for the Gram CTA
            for (int o = t; o < KB * KB; o += kHelpCompute) {
                const int e1 = o / KB, e2 = o % KB;
                double acc0 = 0.0, acc1 = 0.0;
                if (e1 < k && e2 < k) {
#pragma unroll 8
                    for (int m = 0; m < kDT; m += 2) {
                        acc0 = fma(Pt[m * k + e1], Pt[m * k + e2], acc0);
                        acc1 = fma(Pt[(m + 1) * k + e1], Pt[(m + 1) * k + e2], acc1);
                    }
                }
                a.Q[(int64_t)tb * KB * KB + o] = acc0 + acc1;
            }
            named_bar(1, kHelpCompute);
            if (t == 0) {
                __threadfence();
                st_release(a.qflag + tb, a.epoch);
            }
        }
        HPT(4, clock64());
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
    }
    return full;
}


// ---------------------------------------------------------------- Gram CTA
// Accumulates G = P^T P block by block as the helpers publish per-block Grams (warps 0..3)
// and stores the prefix G_b at every 64-row boundary (no Gram/scan kernels).  U_b^{-1}
// (chol_lower(I + sigma G_b), inverted) is formed by block b's diagonal sweep in its
// coefficient warp (in parallel over blocks, while the column threads form w): one
// Gram-CTA warp per block could not keep pace with the chains.

template <int KB>
__device__ void trsv_gram(const TrsvArgs &a, double *smem) {
    const int t = threadIdx.x, warp = t >> 5;
    const int NB = (int)((a.n + kD - 1) / kD);
    constexpr int kAccT = 128;
    for (int o = t; o < KB * KB; o += blockDim.x) a.Ui[o] = (o / KB == o % KB) ? 1.0 : 0.0;  // U_0 = I
    __syncthreads();
    if (t == 0) {
        __threadfence();
        st_release(a.uflag, a.epoch);
    }
    if (warp < kAccT / 32) {
        // prefix sums of the helpers' per-block Grams Q_tb (thread t owns entries t + 128u)
        constexpr int EPB = (KB * KB + kAccT - 1) / kAccT;
        double g[EPB];
#pragma unroll
        for (int u = 0; u < EPB; ++u) g[u] = 0.0;
        const int NT = (int)((a.n + kDT - 1) / kDT);
        for (int tb = 0; tb + 1 < NT; ++tb) {  // Q of the last 32-row block never enters a G_b (b < NB)
            if (t == 0)
                while (ld_acquire(a.qflag + tb) != a.epoch) __nanosleep(GCM_POLL_NS);
            named_bar(1, kAccT);
            const double *Qt = a.Q + (int64_t)tb * KB * KB;
#pragma unroll
            for (int u = 0; u < EPB; ++u) {
                const int o = t + kAccT * u;
                if (o < KB * KB) g[u] += __ldcg(Qt + o);
            }
            const int bn = tb / 2 + 1;
            if ((tb & 1) && bn < NB) {  // G_bn = P_{<bn}^T P_{<bn}
#pragma unroll
                for (int u = 0; u < EPB; ++u) {
                    const int o = t + kAccT * u;
                    if (o < KB * KB) a.G[(int64_t)bn * KB * KB + o] = g[u];
                }
                named_bar(1, kAccT);
                if (t == 0) {
                    __threadfence();
                    st_release(a.uflag + bn, a.epoch);
                }
            }
        }
        return;
    }
}





// One CTA per (checkpoint segment g, 64-column strip s): tiles b in
// [g*CI, min(g*CI+CI, s)).  Thread = column; the tile streams through shared
// memory in kRC-row chunks (cp.async, double-buffered, coalesced both ways);
// the V state stays in registers, the coefficient panel in shared memory.
constexpr int kRC = 16;
constexpr int kLdC = kRC + 1;

template <int KB>
__global__ void __launch_bounds__(kApplyT) bapply_kernel(double *__restrict__ L, int64_t n, int64_t ldl, int k,
                                                         const double *__restrict__ chk, int CI,
                                                         const double *__restrict__ U,
                                                         const double *__restrict__ panels) {
    const int s = blockIdx.x + 1;
    const int g = blockIdx.y;
    const int b0 = g * CI;
    if (b0 >= s) return;
    const int b1 = min(b0 + CI, s);
    extern __shared__ double2 smem_bapply[];
    double2 *cs = smem_bapply;                               // [kD * KB]
    double *rho = reinterpret_cast<double *>(cs + kD * KB);  // [kD]
    double *nu = rho + kD;                                  // [KB]
    double *Us = nu + KB;                                   // [KB * KB]
    double *buf = Us + KB * KB;                             // [2][kD cols][kLdC]
    const int t = threadIdx.x;
    const int64_t c0 = (int64_t)s * kD;
    const int nc = (int)imin64(kD, n - c0);
    double v[KB];
    constexpr int NCH = kD / kRC;

    auto issue = [&](int b, int ch) {
        double *bb = buf + (ch & 1) * kD * kLdC;
        for (int idx = t; idx < kD * kRC; idx += kApplyT) {
            const int c = idx / kRC, j = idx % kRC;
            if (c < nc) cp_async8(bb + c * kLdC + j, L + ((int64_t)b * kD + ch * kRC + j) + (c0 + c) * ldl);
        }
        cp_async_commit();
    };
    for (int b = b0; b < b1; ++b) {
        issue(b, 0);
        const double *panel = panels + (int64_t)b * panel_doubles(KB);
        for (int i = t; i < kD * KB; i += kApplyT) cs[i] = make_double2(panel[2 * i], panel[2 * i + 1]);
        for (int i = t; i < kD; i += kApplyT) rho[i] = panel[2ll * kD * KB + i];
        for (int i = t; i < KB; i += kApplyT) nu[i] = panel[2ll * kD * KB + kD + i];
        if (b == b0)
            for (int i = t; i < KB * KB; i += kApplyT) Us[i] = U[(int64_t)b * KB * KB + i];
        __syncthreads();
        if (b == b0 && t < nc) {  // V-state = U_b^{-1} r
            const double *r = chk + (chk_count_before(s, CI) + g) * kD * k + (int64_t)t * k;
            double rr[KB];
#pragma unroll
            for (int e = 0; e < KB; ++e) rr[e] = e < k ? r[e] : 0.0;
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                double acc = 0.0;
#pragma unroll
                for (int ep = 0; ep <= e; ++ep) acc = fma(Us[e * KB + ep], rr[ep], acc);
                v[e] = acc;
            }
        }
        for (int ch = 0; ch < NCH; ++ch) {
            if (ch + 1 < NCH) {
                issue(b, ch + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                cp_async_wait_all();
            }
            __syncthreads();
            double *bb = buf + (ch & 1) * kD * kLdC;
            if (t < nc) {
                double *col = bb + t * kLdC;
#pragma unroll 4
                for (int j = 0; j < kRC; ++j)
                    col[j] = apply_row<KB>(col[j], v, cs + (ch * kRC + j) * KB, rho[ch * kRC + j], KB);
            }
            __syncthreads();
            for (int idx = t; idx < kD * kRC; idx += kApplyT) {
                const int c = idx / kRC, j = idx % kRC;
                if (c < nc) L[((int64_t)b * kD + ch * kRC + j) + (c0 + c) * ldl] = bb[c * kLdC + j];
            }
        }
        if (t < nc) {
#pragma unroll
            for (int e = 0; e < KB; ++e) v[e] *= nu[e];
        }
        __syncthreads();
    }
}

// CI == 1 (every tile has its own checkpoint): one CTA per (row block b, group of
// kStripsPerCta strips right of it).  The coefficient panel of block b is loaded
// once per CTA; thread (q, c) owns column c of strip q: its V state starts at
// U_b^{-1} r (the checkpointed residual), and the tile streams through shared
// memory in kRC-row chunks (cp.async double buffer, coalesced loads and stores).
constexpr int kStripsPerCta = 4;
constexpr int kTileThreads = kStripsPerCta * kD;

template <int KB>
__global__ void __launch_bounds__(kTileThreads, KB >= 32 ? 1 : 2) btile_kernel(double *__restrict__ L, int64_t n, int64_t ldl, int k,
                                                                const double *__restrict__ chk,
                                                                const double *__restrict__ U,
                                                                const double *__restrict__ panels, int NB) {
    const int b = blockIdx.x;
    const int s0 = b + 1 + kStripsPerCta * blockIdx.y;  // first strip of this CTA
    if (s0 >= NB) return;
    extern __shared__ double2 smem_btile[];
    double2 *cs = smem_btile;                                // [kD * KB]
    double *rho = reinterpret_cast<double *>(cs + kD * KB);  // [kD]
    double *nu = rho + kD;                                  // [KB]
    double *Us = nu + KB;                                   // [KB * KB]
    double *buf = Us + KB * KB;                             // [2][kStripsPerCta * kD][kLdC]
    const int t = threadIdx.x;
    const int q = t / kD, c = t % kD;
    const int s = s0 + q;
    const int64_t c0 = (int64_t)s * kD;
    const int nstr = min(kStripsPerCta, NB - s0);  // strips in this CTA
    const int64_t ncols_cta = imin64((int64_t)nstr * kD, n - (int64_t)s0 * kD);
    constexpr int NCH = kD / kRC;
    const int64_t rb = (int64_t)b * kD;
    auto issue = [&](int ch) {
        double *bb = buf + (ch & 1) * kStripsPerCta * kD * kLdC;
        for (int idx = t; idx < kStripsPerCta * kD * kRC; idx += kTileThreads) {
            const int col = idx / kRC, j = idx % kRC;
            if (col < ncols_cta)
                cp_async8(bb + col * kLdC + j, L + (rb + ch * kRC + j) + ((int64_t)s0 * kD + col) * ldl);
        }
        cp_async_commit();
    };
    issue(0);
    const double *panel = panels + (int64_t)b * panel_doubles(KB);  // stride KB, padding = identities
    for (int i = t; i < kD * KB; i += kTileThreads) cs[i] = make_double2(panel[2 * i], panel[2 * i + 1]);
    for (int i = t; i < kD; i += kTileThreads) rho[i] = panel[2ll * kD * KB + i];
    for (int i = t; i < KB * KB; i += kTileThreads) Us[i] = U[(int64_t)b * KB * KB + i];
    __syncthreads();
    const bool act = q < nstr && c0 + c < n;
    double v[KB];
    if (act) {  // V-state = U_b^{-1} r
        const double *r = chk + (chk_count_before(s, 1) + b) * kD * k + (int64_t)c * k;
        double rr[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) rr[e] = e < k ? r[e] : 0.0;
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            double acc = 0.0;
#pragma unroll
            for (int ep = 0; ep <= e; ++ep) acc = fma(Us[e * KB + ep], rr[ep], acc);
            v[e] = acc;
        }
    }
    for (int ch = 0; ch < NCH; ++ch) {
        if (ch + 1 < NCH) {
            issue(ch + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        double *bb = buf + (ch & 1) * kStripsPerCta * kD * kLdC;
        if (act) {
            // rows held in registers and the (row, e) loops fully unrolled: row j+1's
            // rotation e only waits for row j's rotation e, so rows pipeline
            // instead of serialising on the 2k-deep chain of one row
            constexpr int RG = KB <= 8 ? kRC : kRC / 2;
            double *col = bb + t * kLdC;
#pragma unroll
            for (int g = 0; g < kRC; g += RG) {
                double l[RG];
#pragma unroll
                for (int j = 0; j < RG; ++j) l[j] = col[g + j];
                const double2 *cc = cs + (ch * kRC + g) * KB;
#pragma unroll
                for (int j = 0; j < RG; ++j) {
#pragma unroll
                    for (int e = 0; e < KB; ++e) {
                        const double2 gd = cc[j * KB + e];
                        l[j] = fma(gd.x, v[e], l[j]);
                        v[e] = fma(-gd.y, l[j], v[e]);
                    }
                }
#pragma unroll
                for (int j = 0; j < RG; ++j) col[g + j] = l[j] * rho[ch * kRC + g + j];
            }
        }
        __syncthreads();
        for (int idx = t; idx < kStripsPerCta * kD * kRC; idx += kTileThreads) {
            const int col = idx / kRC, j = idx % kRC;
            if (col < ncols_cta) L[(rb + ch * kRC + j) + ((int64_t)s0 * kD + col) * ldl] = bb[col * kLdC + j];
        }
    }
}


// Flags an Apply grid launched while the TRSV kernel still runs (programmatic dependent
// launch) waits on: tile (b, s0..) needs sweep b, the strip owners past tile rows 2b, 2b+1
// (checkpoints written, L rows of block b read) and J1 done with the rows of block b.
struct ApplyWait {
    const unsigned *bflag;  // nullptr: plain stream order, no waits
    const unsigned long long *hprog;
    const unsigned *lflag;
    unsigned epoch;
    int H, NT;
};
// polite spin (no timeout: every flag waited on is published unconditionally by a CTA of the
// co-resident TRSV grid, and a trap would poison the whole CUDA context under a debugger or
// time-slicing; GCM_SPIN_TRAP_NS=<ns> builds a debug variant that traps instead of hanging)
__device__ __forceinline__ void spin_wait(bool (*ok)(const void *, unsigned, int), const void *p, unsigned epoch,
                                          int need) {
#ifdef GCM_SPIN_TRAP_NS
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
    while (!ok(p, epoch, need)) {
        __nanosleep(256);
#ifdef GCM_SPIN_TRAP_NS
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > (long long)(GCM_SPIN_TRAP_NS)) __trap();
#endif
    }
}
__device__ bool flag_ok(const void *p, unsigned epoch, int) { return ld_acquire((const unsigned *)p) == epoch; }
__device__ bool prog_ok(const void *p, unsigned epoch, int need) {
    const unsigned long long v = ld_acquire64((const unsigned long long *)p);
    return (unsigned)(v >> 32) == epoch && (int)(unsigned)v >= need;
}

template <int KB>
__global__ void __launch_bounds__(kT2Threads, 2) btma_kernel(const __grid_constant__ CUtensorMap tm, int64_t n, int k,
                                                              const double *__restrict__ chk,
                                                              const double *__restrict__ Ui,
                                                              const double *__restrict__ panels, int NB,
                                                              ApplyWait w) {
    const int s0 = blockIdx.x + 1 + t2_strips(KB) * blockIdx.y;
    if (s0 >= NB) return;
    if (w.bflag) {
        const int b = blockIdx.x;
        if (threadIdx.x == 0) {
            spin_wait(flag_ok, w.bflag + b, w.epoch, 0);
            const int slo = 2 * s0, shi = min(w.NT, 2 * (s0 + t2_strips(KB)));
            for (int s32 = slo; s32 < shi; ++s32) spin_wait(prog_ok, w.hprog + s32 % w.H, w.epoch, 2 * b + 2);
            for (int tb = 2 * b + 2; tb <= min(w.NT - 1, 2 * b + 1 + kLookC); ++tb)
                spin_wait(flag_ok, w.lflag + tb, w.epoch, 0);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // sweep's generic stores -> bulk copies
        }
        __syncthreads();
    }
    extern __shared__ __align__(16) unsigned char smem_t2[];
    btma_body<KB>(tm, n, k, chk, Ui, panels, NB, blockIdx.x, s0, smem_t2, 0);
    if (threadIdx.x == 0) TLINE(4);
}

// ---------------------------------------------------------------- worker mode
// A helper whose strips are all done takes tickets for the diagonal sweeps (block b =
// ticket, so every sweep waits only on the chains, the Gram CTA and strip owners --
// never on a later ticket): block b needs U_b^{-1} (or G_b for KB = 32) from the Gram
// CTA and the owner of strip 2b+1 past its last tile (2b, 2b+1), the only other reader
// of L_bb; P_b is polled from the self-validating copy.
static_assert(kDiagThreads == kTrsvThreads, "helpers run the diagonal sweep with all their threads");
template <int KB>
__device__ void trsv_worker(const TrsvArgs &a, double *smem, unsigned long long *ring_bars) {
    __shared__ unsigned s_task;
    const int t = threadIdx.x;
    const int NB = (int)((a.n + kD - 1) / kD);
    const int NT = (int)((a.n + kDT - 1) / kDT);
    __syncthreads();
    if (t < 2 * kHelpRing)
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(ring_bars + t)) : "memory");
    for (;;) {
        __syncthreads();
        if (t == 0) {
            const unsigned task = atomicAdd(a.taskctr, 1u) + 1u;  // armed to all-ones: first ticket 0
            s_task = task < (unsigned)NB ? task : 0xffffffffu;  // tickets in block order
        }
        __syncthreads();
        const unsigned task = s_task;
        if (task == 0xffffffffu) break;
        const int b = (int)task;
        {  // the diagonal sweep of block b
            if (t == 0) {
#ifdef GCM_TRACE
                g_htrace[(1000 + b) * 8 + 0] = gtime();
                g_htrace[(1000 + b) * 8 + 3] = blockIdx.x;
#endif
                while (ld_acquire(a.uflag + b) != a.epoch) __nanosleep(64);
#ifdef GCM_TRACE
                g_htrace[(1000 + b) * 8 + 4] = gtime();
#endif
                if (2 * b + 1 < NT)
                    while (ld_acquire(a.qflag + 2 * b) != a.epoch) __nanosleep(64);
#ifdef GCM_TRACE
                g_htrace[(1000 + b) * 8 + 1] = gtime();
#endif
            }
            __syncthreads();
            bdiag_body<KB>(const_cast<double *>(a.L), a.n, a.ldl, a.Vw, a.n, a.k, a.sigma, a.pfast, true, a.Ui, a.G,
                           a.panels, a.key, a.ebase, b, smem);
            __syncthreads();
            if (t == 0) {
#ifdef GCM_TRACE
                g_htrace[(1000 + b) * 8 + 2] = gtime();
#endif
                if (a.publish) {
                    __threadfence();
                    st_release(a.bflag + b, a.epoch);
                }
            }
        }
    }
}

template <int KB>
__global__ void __launch_bounds__(kTrsvThreads, 1) trsv_kernel(const __grid_constant__ TrsvArgs a) {
    extern __shared__ __align__(128) double smem_trsv[];
    // every CTA is resident (cooperative launch): the Apply grid may be scheduled onto SMs
    // as our CTAs exit (programmatic dependent launch); it waits on our flags, not on us
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) TLINE(0);
    if ((int)blockIdx.x < a.NC)
        trsv_chain(a, smem_trsv, blockIdx.x);
    else if ((int)blockIdx.x == a.NC) {
        trsv_gram<KB>(a, smem_trsv);
    } else {
        unsigned long long *bars = trsv_helper<KB>(a, smem_trsv, blockIdx.x - a.NC - 1, gridDim.x - a.NC - 1);
        trsv_worker<KB>(a, smem_trsv, bars);
    }
}

bool encode_tmap(CUtensorMap *m, const double *L, int64_t n, int64_t ldl, unsigned box_rows, unsigned box_cols,
                 CUtensorMapSwizzle swz) {
    return encode_tmap_f64(m, L, 2, n, n, ldl, 1, 0, box_rows, box_cols, swz);
}

template <int KB>
gcm_status_t blocked_pass(double *L, int64_t n, int64_t ldl, double *V, int k, int sigma, unsigned long long *key,
                          int64_t ebase, char *wsbase, const Layout &lay, unsigned epoch, cudaStream_t stream) {
    TrsvArgs a;
    a.L = L;
    a.n = n;
    a.ldl = ldl;
    a.V = V;
    a.k = k;
    a.P = reinterpret_cast<double *>(wsbase + lay.P);
    a.rcur = reinterpret_cast<double *>(wsbase + lay.rcur);
    a.rchain = reinterpret_cast<double *>(wsbase + lay.rchain);
    a.pfast = reinterpret_cast<double *>(wsbase + lay.pfast);
    a.MX = reinterpret_cast<double *>(wsbase + lay.MX);
    a.bulk_ok = (ldl % 2 == 0) && ((reinterpret_cast<uintptr_t>(L) & 15) == 0) && n <= 0x7fffffff;
    a.chk = reinterpret_cast<double *>(wsbase + lay.chk);
    a.CI = lay.CI;
    a.CIlog = 0;
    while ((1 << a.CIlog) < lay.CI) ++a.CIlog;
    unsigned *flags = reinterpret_cast<unsigned *>(wsbase + lay.flags);
    a.lflag = flags;
    a.qflag = a.lflag + lay.NT;
    a.Q = reinterpret_cast<double *>(wsbase + lay.Q);
    a.epoch = epoch;

    a.NC = (k + kRPC - 1) / kRPC;
    a.Vw = V;
    a.panels = reinterpret_cast<double *>(wsbase + lay.panels);
    a.key = key;
    a.ebase = ebase;
    a.uflag = a.qflag + lay.NT;
    a.taskctr = reinterpret_cast<unsigned *>(a.pfast + (size_t)lay.NT * kDT * k);
    // the diagonal sweeps always run inside the TRSV kernel (worker mode; KB = 32 alone:
    // 1.39 ms at k = 64 with the sweeps after the solve, 1.17 ms fused -- same-box A/B)
    a.bflag = a.uflag + lay.NB;
    a.hprog = reinterpret_cast<unsigned long long *>(wsbase + lay.hprog);
    a.own_cap = help_max_own(KB);
    if (const char *e = std::getenv("GCM_HELP_OWN_CAP")) a.own_cap = std::max(0, std::min(a.own_cap, std::atoi(e)));
    // Overlapped Apply: btma_kernel is launched as a programmatic dependent of the TRSV
    // kernel and takes SMs as TRSV CTAs exit, each tile waiting on its sweep's flag and the
    // strip owners' progress -- so the Apply of the early blocks runs under the last
    // diagonal sweeps instead of after them.  (Apply tiles as worker tickets inside the
    // TRSV kernel were measured slower, 0.52 vs 0.43 ms at n=5000, k=16: their 200 MB
    // stream competes with the helpers' latency-bound tile loads.)
    CUtensorMap tm2;
    const bool pdl = lay.NB > 1 && lay.CI == 1 && a.bulk_ok &&
                     encode_tmap(&tm2, L, n, ldl, (unsigned)kT2Rows, (unsigned)kT2Box, CU_TENSOR_MAP_SWIZZLE_64B);
    a.publish = pdl;
    a.G = reinterpret_cast<double *>(wsbase + lay.G);
    a.Ui = reinterpret_cast<double *>(wsbase + lay.U);
    a.sigma = sigma;
    int dev = 0, nsm = 0;
    gcm_status_t st = check_cuda(cudaGetDevice(&dev));
    if (st == GCM_OK) st = check_cuda(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (st != GCM_OK) return st;
    const size_t smem_chain = (size_t)ChainSmem::total * sizeof(double);
    const size_t smem_help = (size_t)(kDT * kLdT + kDT * std::max(KB, kLdT) + help_max_own(KB) * kDT * KB +
                                      kHelpRing * (kDT * kLdR + kDT * (KB + 1)) + 3 * kHelpRing) *
                             sizeof(double);
    const size_t smem_diag = (size_t)bdiag_smem_doubles(KB) * sizeof(double);
    size_t smem = std::max(std::max(smem_chain, smem_help), smem_diag);
    st = check_cuda(cudaFuncSetAttribute(trsv_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (st != GCM_OK) return st;
    int per_sm = 0;
    st = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trsv_kernel<KB>, kTrsvThreads, smem));
    if (st != GCM_OK) return st;
    if (per_sm < 1) return GCM_ECUDA;
    const int grid = (int)std::min<int64_t>((int64_t)nsm * per_sm, a.NC + 1 + lay.NT);
    if (grid <= a.NC + 1) return GCM_ECUDA;
    a.H = grid - a.NC - 1;
    void *args[] = {&a};
    // hand-off slots, pfast, the ticket counter, flags and progress words: all-ones (see
    // make_layout; hand-off consumers also re-arm what they read)
    st = check_cuda(cudaMemsetAsync(wsbase + lay.rchain, 0xff, lay.MX - lay.rchain, stream));
    if (st != GCM_OK) return st;
    double *U = reinterpret_cast<double *>(wsbase + lay.U);
    double *panels = reinterpret_cast<double *>(wsbase + lay.panels);
    if (pdl) {  // one profiling scope: an event between the two launches would serialise them
        const size_t smem_t2 = t2_smem_bytes(KB);
        st = check_cuda(
            cudaFuncSetAttribute(btma_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t2));
        if (st != GCM_OK) return st;
        ProfScope ps("blocked", stream);
        st = check_cuda(cudaLaunchCooperativeKernel((const void *)trsv_kernel<KB>, dim3(grid), dim3(kTrsvThreads),
                                                    args, smem, stream));
        if (st != GCM_OK) return st;
        ApplyWait w{a.bflag, a.hprog, a.lflag, epoch, a.H, lay.NT};
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(lay.NB - 1, (lay.NB - 1 + t2_strips(KB) - 1) / t2_strips(KB));
        cfg.blockDim = dim3(kT2Threads);
        cfg.dynamicSmemBytes = smem_t2;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const double *chk = a.chk;
        count_launch(2);  // the TRSV kernel above and this Apply grid
        return check_cuda(cudaLaunchKernelEx(&cfg, btma_kernel<KB>, tm2, n, k, chk, (const double *)U,
                                             (const double *)panels, (int)lay.NB, w));
    }
    {
        ProfScope ps("trsv", stream);
        st = check_cuda(cudaLaunchCooperativeKernel((const void *)trsv_kernel<KB>, dim3(grid), dim3(kTrsvThreads),
                                                    args, smem, stream));
        count_launch();
    }
    if (st != GCM_OK) return st;

    if (lay.NB > 1) {  // the Apply after the TRSV kernel (unaligned L or CI > 1)
        const size_t smem_apply = (size_t)(2 * kD * KB + kD + KB + KB * KB + 2 * kD * kLdC) * sizeof(double);
        st = check_cuda(
            cudaFuncSetAttribute(bapply_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_apply));
        if (st != GCM_OK) return st;
        if (lay.CI == 1) {
            const size_t smem_tile =
                (size_t)(2 * kD * KB + kD + KB + KB * KB + 2 * kStripsPerCta * kD * kLdC) * sizeof(double);
            st = check_cuda(
                cudaFuncSetAttribute(btile_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tile));
            if (st != GCM_OK) return st;
            const dim3 gridt(lay.NB - 1, (lay.NB - 1 + kStripsPerCta - 1) / kStripsPerCta);
            ProfScope ps("bapply", stream);
            btile_kernel<KB><<<gridt, kTileThreads, smem_tile, stream>>>(L, n, ldl, k, a.chk, U, panels, lay.NB);
            count_launch();
            return check_cuda(cudaGetLastError());
        }
        const dim3 grid2(lay.NB - 1, (lay.NB - 1 + lay.CI - 1) / lay.CI);
        ProfScope ps("bapply", stream);
        bapply_kernel<KB><<<grid2, kApplyT, smem_apply, stream>>>(L, n, ldl, k, a.chk, lay.CI, U, panels);
        count_launch();
    }
    return check_cuda(cudaGetLastError());
}

}  // namespace

#ifdef GCM_TRACE
extern "C" int gcm_debug_trace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(long long) * count);
}
#ifdef GCM_SWEEP_TRACE
extern "C" int gcm_debug_sweep_trace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, gcm::gcm_sweep_trace, sizeof(long long) * count);
}
#endif
extern "C" int gcm_debug_htrace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, g_htrace, sizeof(long long) * count);
}
extern "C" int gcm_debug_dtrace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, g_dtrace, sizeof(long long) * count);
}
#endif

size_t blocked_workspace_bytes(int64_t n, int64_t k) {
    const int kc = (int)std::min<int64_t>(k, kBKMax);
    return make_layout(n, kc, chk_budget(n, kc)).total;
}

gcm_status_t modify_blocked(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                            unsigned long long *key, Workspace *ws, cudaStream_t stream) {
    gcm_status_t st = GCM_OK;
    char *base = reinterpret_cast<char *>(ws->panels);
    for (int64_t e0 = 0; e0 < k; e0 += kBKMax) {
        const int kc = (int)std::min<int64_t>(kBKMax, k - e0);
        // the layout must fit the workspace sized earlier (free memory may have changed since)
        size_t budget = chk_budget(n, kc);
        Layout lay = make_layout(n, kc, budget);
        const size_t cap = ws->bytes - (size_t)(reinterpret_cast<char *>(ws->panels) - reinterpret_cast<char *>(ws->key));
        while (lay.total > cap && lay.CI < lay.NB) {
            budget /= 2;
            lay = make_layout(n, kc, budget);
        }
        if (lay.total > cap) return GCM_ENOMEM;
        // flags are armed to all-ones each pass: the epoch is never 0 or all-ones
        if (++ws->epoch == 0xffffffffu) ws->epoch = 1;
        const unsigned epoch = ws->epoch;
        double *Vc = V + e0 * n;
        if (kc <= 4) st = blocked_pass<4>(L, n, ldl, Vc, kc, sigma, key, e0, base, lay, epoch, stream);
        else if (kc <= 8) st = blocked_pass<8>(L, n, ldl, Vc, kc, sigma, key, e0, base, lay, epoch, stream);
        else if (kc <= 16) st = blocked_pass<16>(L, n, ldl, Vc, kc, sigma, key, e0, base, lay, epoch, stream);
        else st = blocked_pass<32>(L, n, ldl, Vc, kc, sigma, key, e0, base, lay, epoch, stream);
        if (st != GCM_OK) return st;
    }
    return GCM_OK;
}

}  // namespace gcm
