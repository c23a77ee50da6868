// bparts.cuh -- device building blocks shared by the blocked single-factor path
// (blocked.cu) and the column-sharded / large-n path (panel.cu): the self-validating
// value reads, the checkpoint layout, the KB x KB Cholesky inverse of I + sigma G_b, the
// diagonal-block sweep (bdiag_body) and the TMA Apply of one 64-row panel to a 64 x 256
// tile (btma_body).  (Moved out of blocked.cu unchanged except for the parameters noted.)
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "diag.cuh"
#include "internal.h"
#include "rot.cuh"
#include "tma.cuh"

namespace gcm {
namespace {

__host__ __device__ inline int64_t chk_count_before(int64_t s, int CI) {
    // sum_{s'=1}^{s-1} ceil(s'/CI)
    const int64_t S = s - 1;
    if (S <= 0) return 0;
    const int64_t q = S / CI, r = S % CI;
    return CI * q * (q + 1) / 2 + (q + 1) * r;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double *p) {
    unsigned long long u;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(u) : "l"(p) : "memory");
    return u;
}
// same, for values several consumers read (no re-arm; the pass's memset arms them)
__device__ __forceinline__ double ld_value(const double *p) {
    chaos_delay();
    unsigned long long u;
    do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(u) : "l"(p) : "memory");
    } while (u == kEmpty);
    return __longlong_as_double((long long)u);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// U^{-1} for U = chol_lower(A), A a KB x KB SPD matrix, in one warp: Gaussian elimination
// on [A | I] with lane i holding row i (A part in a[], identity part in w[]); step c
// broadcasts the pivot row by shuffles and every lower lane eliminates with one
// multiply by the pivot's reciprocal, leaving A = D U'^T and w = U'^{-1} (U' unit
// lower); then U^{-1} = D^{-1/2} U'^{-1}.  Writes U^{-1} row-major to out[KB*KB]
// (lane i writes row i).  A non-positive pivot gives NaNs (the sweep reports it).
template <int KB>
__device__ __forceinline__ void warp_chol_inv(double (&a)[KB], double *out) {
    const int i = threadIdx.x & 31;
    double w[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) w[j] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int c = 0; c < KB - 1; ++c) {
        // rows above the pivot are left untouched (selected, not multiplied by f = 0): a NaN
        // in a later row (a NaN update column, R5/R6) must not reach the rows of
        // the earlier update columns through 0 * NaN, or the failure report would name
        // the wrong (lexicographically smaller) column
        const bool below = i > c;
        const double rp = 1.0 / __shfl_sync(kFull, a[c], c);
        const double f = a[c] * rp;
#pragma unroll
        for (int j = c + 1; j < KB; ++j) {
            const double x = __shfl_sync(kFull, a[j], c);
            if (below) a[j] = fma(-f, x, a[j]);
        }
#pragma unroll
        for (int j = 0; j <= c; ++j) {
            const double x = __shfl_sync(kFull, w[j], c);
            if (below) w[j] = fma(-f, x, w[j]);
        }
    }
    double di = 0.0;
#pragma unroll
    for (int j = 0; j < KB; ++j)
        if (j == i) di = a[j];
    const double s = rsqrt(di);
    if (i < KB)
#pragma unroll
        for (int j = 0; j < KB; ++j) out[i * KB + j] = w[j] * s;
}

// One CTA per 64-row diagonal block, all blocks in parallel.
#ifndef GCM_DIAG_NQ
#define GCM_DIAG_NQ 4
#endif
constexpr int kDiagNQ = GCM_DIAG_NQ;  // threads per column in the diagonal sweep
constexpr int kDiagThreads = 4 * kD + 32;  // up to 4 column parts + the coefficient warp
static_assert(kDiagNQ == 1 || kDiagNQ == 2 || kDiagNQ == 4, "kDiagNQ * kD + 32 <= kDiagThreads");

#ifdef GCM_TRACE  // per-block phase times of the diagonal sweep (globaltimer ns; tools/trace_chain.py)
__device__ long long g_dtrace[256 * 8];
#define DT_MARK(b, slot)                                                                        \
    do {                                                                                        \
        if (threadIdx.x == 0 && (b) < 256) {                                                    \
            long long v_;                                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_));                             \
            g_dtrace[(b) * 8 + (slot)] = v_;                                                    \
        }                                                                                       \
    } while (0)
#else
#define DT_MARK(b, slot) ((void)0)
#endif

// the diagonal sweep's form: the closed form (diag.cuh) for rank buckets <= 16 (its KB x KB
// per-row eliminations fit the worker's shared memory), the wave for 32
#ifndef GCM_DIAG_CLOSED
#define GCM_DIAG_CLOSED 1
#endif
__host__ __device__ constexpr bool bdiag_closed(int KB) { return GCM_DIAG_CLOSED && KB <= 16; }
__host__ __device__ constexpr int bdiag_smem_doubles(int KB) {
    return kD * (kD + 1) + kD * (KB + 1) + KB * (KB + 1) + 2 + wave_panel_doubles(KB) + 1 + 4 * kD * KB + 2 * kD +
           (bdiag_closed(KB) ? kD * (KB + 1) + diag_closed_scratch(KB) : 0);
}

// The sweep of diagonal block b by one CTA of kDiagThreads threads (a TRSV helper in
// worker mode; P is read from the self-validating copy when p_poll).
template <int KB>
__device__ void bdiag_body(double *__restrict__ L, int64_t n, int64_t ldl, double *__restrict__ V, int64_t ldv, int k,
                           int sigma,
                           const double *__restrict__ P, bool p_poll, double *__restrict__ Ui,
                           const double *__restrict__ G, double *__restrict__ panels, unsigned long long *key,
                           int64_t ebase, int b, double *smem_bdiag) {
    double(*Ls)[kD + 1] = reinterpret_cast<double(*)[kD + 1]>(smem_bdiag);               // [kD][kD+1]
    double(*Ps)[KB + 1] = reinterpret_cast<double(*)[KB + 1]>(smem_bdiag + kD * (kD + 1)); // [kD][KB+1]
    double(*M)[KB + 1] = reinterpret_cast<double(*)[KB + 1]>(smem_bdiag + kD * (kD + 1) + kD * (KB + 1));
    double *pan = smem_bdiag + kD * (kD + 1) + kD * (KB + 1) + KB * (KB + 1);  // panel (16-byte aligned below)
    pan += (reinterpret_cast<uintptr_t>(pan) & 15) ? 1 : 0;
    double *vx = pan + wave_panel_doubles(KB) + 1;
    double *dinv = vx + kD * KB;
    double *vt = dinv + kD;
    double *imx = vt + kD * (KB + 1);
    double *Vs = imx + kD * KB;
    const int t = threadIdx.x;
    const int64_t r0 = (int64_t)b * kD;
    const int Db = (int)imin64(kD, n - r0);
    DT_MARK(b, 0);
#ifdef GCM_SWEEP_TRACE
    if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[1000] = clock64();
#endif

    // U_b^{-1} from G_b, by the coefficient warp (idle until the sweep) while the column
    // threads form w
    double *Uis = reinterpret_cast<double *>(M);  // [KB][KB] in the (KB x KB+1) slot
    {  // every load in flight before the first use (one memory latency, not one per element)
        constexpr int kLI = (kD * kD + kDiagThreads - 1) / kDiagThreads;
        double lv[kLI];
#pragma unroll
        for (int q = 0; q < kLI; ++q) {
            const int idx = t + q * kDiagThreads, m = idx / kD, j = idx % kD;
            lv[q] = (idx < kD * kD && m < Db && j <= m) ? L[(r0 + j) + (r0 + m) * ldl] : 0.0;
        }
        constexpr int kPI = (kD * KB + kDiagThreads - 1) / kDiagThreads;
        unsigned long long pv[kPI];
#pragma unroll
        for (int q = 0; q < kPI; ++q) {
            const int o = t + q * kDiagThreads, m = k > 0 ? o / k : 0;
            pv[q] = 0ull;
            if (o < kD * k && m < Db)
                pv[q] = p_poll ? ld_relaxed_u64(P + (r0 + m) * k + o % k)
                               : (unsigned long long)__double_as_longlong(P[(r0 + m) * k + o % k]);
        }
#pragma unroll
        for (int q = 0; q < kLI; ++q) {
            const int idx = t + q * kDiagThreads, m = idx / kD, j = idx % kD;
            if (idx < kD * kD && m < Db && j <= m) Ls[m][j] = lv[q];
        }
#pragma unroll
        for (int q = 0; q < kPI; ++q) {
            const int o = t + q * kDiagThreads;
            if (o < kD * k) {
                const int m = o / k, e = o % k;
                if (p_poll && m < Db && pv[q] == kEmpty) pv[q] = __double_as_longlong(ld_value(P + (r0 + m) * k + e));
                Ps[m][e] = __longlong_as_double((long long)pv[q]);
            }
        }
    }
    __syncthreads();
    DT_MARK(b, 1);
#ifdef GCM_SWEEP_TRACE
    if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[1003] = clock64();
#endif
    constexpr int EPT = KB / kDiagNQ;
    if (t < kDiagNQ * kD) {
        // column threads (m, q): w = (L_bb^T P_b)[m] for update columns q*EPT .. (into vt)
        const int cm = t % kD, cq = t / kD;
        double w[EPT];
#pragma unroll
        for (int i = 0; i < EPT; ++i) w[i] = 0.0;
        if (cm < Db) {
            for (int j = 0; j <= cm; ++j) {
                const double l = Ls[cm][j];
#pragma unroll
                for (int i = 0; i < EPT; ++i) w[i] = fma(l, Ps[j][cq * EPT + i], w[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i) vt[cm * (KB + 1) + cq * EPT + i] = w[i];  // odd stride: no bank conflicts
#ifdef GCM_SWEEP_TRACE
        if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[1005] = clock64();
#endif
    } else {

        const int lane = t & 31;
        if (b == 0) {
            for (int o = lane; o < KB * KB; o += 32) Uis[o] = (o / KB == o % KB) ? 1.0 : 0.0;
        } else {
            const double *Gb = G + (int64_t)b * KB * KB;
            double row[KB];
#pragma unroll
            for (int j = 0; j < KB; ++j)
                row[j] = (lane < k && j < k) ? (lane == j ? 1.0 : 0.0) + (sigma > 0 ? Gb[lane * KB + j] : -Gb[lane * KB + j])
                                             : (lane == j ? 1.0 : 0.0);
            warp_chol_inv<KB>(row, Uis);
        }
        __syncwarp();
        for (int o = lane; o < KB * KB; o += 32) Ui[(int64_t)b * KB * KB + o] = Uis[o];
    }
    __syncthreads();
    DT_MARK(b, 2);
#ifdef GCM_SWEEP_TRACE
    if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[1006] = clock64();
#endif
    // closed-form block (diag.cuh, R20) for KB <= 16: q_m = U_b^{-1} p_m (the block's
    // L^{-T} of the V states, no solve needed), every row's rotations in parallel
    constexpr bool kClosed = bdiag_closed(KB);
    double *qv = Vs + kD * KB;  // [kD][KB+1] (closed form only), then diag_closed's scratch
    if (t < kDiagNQ * kD) {  // V state y = U^{-1} w (and q = U^{-1} p)
        const int cm = t % kD, cq = t / kD;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int e = cq * EPT + i;
            double acc = 0.0, aq = 0.0;
#pragma unroll
            for (int ep = 0; ep < KB; ++ep) {  // U^{-1} lower triangular; vt past column k is scratch
                if (ep <= e) acc = fma(Uis[e * KB + ep], vt[cm * (KB + 1) + ep], acc);
                if (kClosed && ep <= e && ep < k) aq = fma(Uis[e * KB + ep], Ps[cm][ep], aq);
            }
            Vs[cm * KB + e] = (cm < Db && e < k) ? acc : 0.0;
            if (kClosed) qv[cm * (KB + 1) + e] = (cm < Db && e < k) ? aq : 0.0;
        }
    }
    __syncthreads();  // the sweep reads Vs from other threads before its own first barrier
#ifdef GCM_SWEEP_TRACE
    if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[1001] = clock64();
#endif
    DT_MARK(b, 3);
    if constexpr (kClosed) {
        diag_closed<KB>(Ls, qv, KB + 1, Db, k, sigma, r0, pan, V + r0, ldv, key, ebase, qv + kD * (KB + 1));
        DT_MARK(b, 4);
        if (t < Db && t > 0) {  // the block's own triangle, column t from its block-start state
            double y[KB];
#pragma unroll
            for (int e = 0; e < KB; ++e) y[e] = Vs[t * KB + e];
            diag_triangle<KB>(Ls, t, y, pan);
        }
        __syncthreads();
    } else {
        wave_sweep<KB, kDiagNQ, kD + 1>(Ls, Vs, Db, k, sigma, r0, pan, V + r0, ldv, key, ebase, vx, dinv, vt, imx,
                                        0, kDiagNQ * kD / 32);
    }
#ifdef GCM_SWEEP_TRACE
    if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[1002] = clock64();
#endif
    DT_MARK(b, 5);
    // panel out in the blocked path's stride-KB layout (padding rotations are identities)
    double *panel = panels + (int64_t)b * panel_doubles(KB);
    for (int i = t; i < (int)panel_doubles(KB); i += kDiagThreads) panel[i] = pan[i];
    for (int idx = t; idx < kD * kD; idx += kDiagThreads) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) L[(r0 + j) + (r0 + m) * ldl] = Ls[m][j];
    }
}

// Inverse of one 64x64 upper-triangular block U (U(i, j) = Lb[i + j * ldl], i <= j < D), by 64
// threads: thread m computes column m of U^{-1} by back substitution (U w = e_m), its 64 running
// sums in registers at compile-time indices, every U entry a shared-memory broadcast; the
// partial sums of rows j > m are never formed, so a NaN in U reaches exactly the entries
// substitution would reach.  Stored by rows: w[j * 64 + m] = (U^{-1})(j, m), zero for j > m and
// for m >= D.  Us: [kD][kD] shared scratch, rd: [kD].
__device__ __forceinline__ void pinv_block(const double *__restrict__ Lb, int64_t ldl, int D, double *w,
                                           double (*Us)[kD], double *rd) {
    const int m = threadIdx.x;
    // the block by asynchronous copies, all 64 per thread in flight at once (zero-filled outside
    // the triangle); a load-then-store loop waited one memory latency per few elements
    for (int idx = m; idx < kD * kD; idx += kD) {
        const int j = idx / kD, i = idx % kD;  // consecutive threads: consecutive rows of column j
        const bool ok = i <= j && j < D;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(&Us[j][i])),
                     "l"(ok ? Lb + i + (int64_t)j * ldl : Lb), "r"(ok ? 8 : 0)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    rd[m] = m < D ? 1.0 / Us[m][m] : 0.0;
    __syncthreads();
    const bool act = m < D;
    double acc[kD];
#pragma unroll
    for (int i = 0; i < kD; ++i) acc[i] = i == m ? 1.0 : 0.0;
#pragma unroll
    for (int j = kD - 1; j >= 0; --j) {
        if (act && j <= m) {
            acc[j] *= rd[j];  // w_j
#pragma unroll
            for (int i = 0; i < j; ++i) acc[i] = fma(-Us[j][i], acc[j], acc[i]);
        }
    }
#pragma unroll
    for (int j = 0; j < kD; ++j) w[j * kD + m] = (act && j <= m) ? acc[j] : 0.0;
}

// One FP64 tensor-core step (DMMA, mma.sync m8n8k4 .f64): c(8x8) += a(8x4) b(4x8), lane l
// holding a[l/4][l%4], b[l%4][l/4] and c[l/4][2(l%4) .. 2(l%4)+1] (PTX ISA fragment layout).
__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// CI == 1 Apply through TMA (L 16-byte aligned, ldl even): one CTA of 128 threads per
// (row block b, 2C column strips = 128*C columns); thread t owns columns t + 128q
// (q < C, C = 4 for KB <= 16, else 2), so each broadcast (gamma, delta) load feeds 2C
// FMAs and the shared-memory pipe stops being the limit.  The 64-row tile streams
// through a 3-stage ring of 8-row chunks (one 8 x 256 TMA box per 256 columns, 64-byte
// rows, 64B swizzle: a lane's row pair is one conflict-free 16-byte load), is rotated
// in place and leaves by TMA stores; the panel and U_b^{-1} arrive by two bulk copies.
// DRAM traffic is the tile read + write once; the V states start at U_b^{-1} r from
// the checkpoints.
#ifndef GCM_T2_STAGES
#define GCM_T2_STAGES 4
#endif
constexpr int kT2Threads = 128;
constexpr int kT2Box = 256;  // columns per TMA box
constexpr int kT2Rows = 8;
constexpr int kT2Stages = GCM_T2_STAGES;
constexpr int kT2Chunks = kD / kT2Rows;
constexpr unsigned kT2BoxBytes = kT2Rows * kT2Box * 8;

#ifndef GCM_T2_C
#define GCM_T2_C 2
#endif
#ifndef GCM_T2_UNROLL
#define GCM_T2_UNROLL 4
#endif
constexpr int kT2Unroll = GCM_T2_UNROLL;
__host__ __device__ constexpr int t2_cols_per_thread(int KB) { return KB <= 16 ? GCM_T2_C : 2; }
__host__ __device__ constexpr int t2_strips(int KB) { return kT2Threads * t2_cols_per_thread(KB) / kD; }
__host__ __device__ constexpr size_t t2_smem_bytes(int KB) {
    return 1024 + (size_t)kT2Stages * kT2BoxBytes * (t2_cols_per_thread(KB) / 2) +
           ((size_t)panel_doubles(KB) + KB * KB) * 8 + 8 * (2 * kT2Stages + 1);
}

// Apply of panel b to the 64 x 256 tile at 64-column strip s0 by threads 0..kT2Threads-1
// (a btma_kernel CTA, or a TRSV helper in worker mode: then `bar` is a named barrier id
// for those threads only; tm must be a __grid_constant__ parameter).
// Column map of an Apply: gstrip == nullptr is the single-factor layout (strip s = global
// 64-column strip s, checkpoint of tile (b, s) at chk_count_before(s, 1) + b); otherwise the
// tile's columns are LOCAL strips s of a column-sharded factor (panel.cu): global strip
// gstrip[s], checkpoint at chkoff[s] + b, ncols local columns.
struct ApplyMap {
    const int *gstrip;
    const int64_t *chkoff;
    int64_t ncols;
};

template <int KB>
__device__ void btma_body(const CUtensorMap &tm, int64_t n, int k, const double *__restrict__ chk,
                          const double *__restrict__ Ui, const double *__restrict__ panels, int NB, int b, int s0,
                          unsigned char *smem_t2, int bar, const ApplyMap &map = ApplyMap{nullptr, nullptr, 0}) {
    constexpr int C = t2_cols_per_thread(KB);
    constexpr int NBOX = C / 2;  // TMA boxes per chunk
    constexpr unsigned kStage = kT2BoxBytes * NBOX;
    auto sync = [&]() {
        if (bar == 0) __syncthreads();
        else named_bar(bar, kT2Threads);
    };
    const unsigned sbase = smem_u32(smem_t2);
    unsigned char *st = smem_t2 + (((sbase + 1023u) & ~1023u) - sbase);  // swizzled boxes: 1 KB aligned
    double2 *cs = reinterpret_cast<double2 *>(st + kT2Stages * kStage);   // [kD][KB] (gamma, delta)
    const double *rho = reinterpret_cast<const double *>(cs + kD * KB);    // [kD]
    double *Us = reinterpret_cast<double *>(st + kT2Stages * kStage) + panel_doubles(KB);  // [KB][KB]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(Us + KB * KB);     // full[stages], panel
    const int t = threadIdx.x;
    const int rb = b * kD, col0 = s0 * kD;
    auto load_chunk = [&](int ch) {  // thread 0
        const int sg = ch % kT2Stages;
        mbar_arrive_expect_tx(bars + sg, kStage);
#pragma unroll
        for (int x = 0; x < NBOX; ++x)
            tma_load_2d(st + sg * kStage + x * kT2BoxBytes, &tm, rb + ch * kT2Rows, col0 + x * kT2Box, bars + sg);
    };
    if (t == 0) {
        for (int i = 0; i <= kT2Stages; ++i) mbar_init(bars + i, 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    sync();
    if (t == 0) {
        const unsigned pbytes = (unsigned)panel_doubles(KB) * 8u, ubytes = (unsigned)(KB * KB) * 8u;
        mbar_arrive_expect_tx(bars + kT2Stages, pbytes + ubytes);
        bulk_g2s(cs, panels + (int64_t)b * panel_doubles(KB), pbytes, bars + kT2Stages);
        bulk_g2s(Us, Ui + (int64_t)b * KB * KB, ubytes, bars + kT2Stages);
        for (int ch = 0; ch < kT2Stages; ++ch) load_chunk(ch);
    }
    // V states = U_b^{-1} r (checkpointed residuals), the C columns together so each
    // U entry is loaded once and consumed at once
    double v[C][KB];
    const double *pr[C];
    bool act[C];
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const int c = t + kT2Threads * q;
        const int s = s0 + c / kD;
        if (map.gstrip) {
            act[q] = (int64_t)col0 + c < map.ncols && map.gstrip[min(s, (int)((map.ncols - 1) / kD))] > b;
            pr[q] = chk + (map.chkoff[act[q] ? s : s0] + b) * kD * k + (int64_t)(c % kD) * k;
        } else {
            act[q] = s < NB && (int64_t)col0 + c < n;
            pr[q] = chk + (chk_count_before(act[q] ? s : s0, 1) + b) * kD * k + (int64_t)(c % kD) * k;
        }
#pragma unroll
        for (int e = 0; e < KB; ++e) v[q][e] = 0.0;
    }
    mbar_wait(bars + kT2Stages, 0u);
#pragma unroll
    for (int ep = 0; ep < KB; ++ep) {
        double rv[C];
#pragma unroll
        for (int q = 0; q < C; ++q) rv[q] = (act[q] && ep < k) ? pr[q][ep] : 0.0;
#pragma unroll
        for (int e = ep; e < KB; ++e) {
            const double u = Us[e * KB + ep];
#pragma unroll
            for (int q = 0; q < C; ++q) v[q][e] = fma(u, rv[q], v[q][e]);
        }
    }
    for (int ch = 0; ch < kT2Chunks; ++ch) {
        const int sg = ch % kT2Stages;
        mbar_wait(bars + sg, (unsigned)((ch / kT2Stages) & 1));
        unsigned char *buf = st + sg * kStage;
#pragma unroll kT2Unroll
        for (int jp = 0; jp < kT2Rows / 2; ++jp) {
            double2 *p[C];
            double2 x[C];
#pragma unroll
            for (int q = 0; q < C; ++q) {
                const int c = t + kT2Threads * q, cc = c % kT2Box;
                p[q] = reinterpret_cast<double2 *>(buf + (c / kT2Box) * kT2BoxBytes + cc * 64 +
                                                   ((jp ^ ((cc >> 1) & 3)) << 4));
                x[q] = *p[q];
            }
            const int j = ch * kT2Rows + 2 * jp;
            const double2 *g0 = cs + j * KB, *g1 = g0 + KB;
#pragma unroll
            for (int e = 0; e < KB; ++e) {  // row j
                const double2 gd = g0[e];
#pragma unroll
                for (int q = 0; q < C; ++q) {
                    x[q].x = fma(gd.x, v[q][e], x[q].x);
                    v[q][e] = fma(-gd.y, x[q].x, v[q][e]);
                }
            }
#pragma unroll
            for (int e = 0; e < KB; ++e) {  // row j + 1
                const double2 gd = g1[e];
#pragma unroll
                for (int q = 0; q < C; ++q) {
                    x[q].y = fma(gd.x, v[q][e], x[q].y);
                    v[q][e] = fma(-gd.y, x[q].y, v[q][e]);
                }
            }
            const double ra = rho[j], rbb = rho[j + 1];
#pragma unroll
            for (int q = 0; q < C; ++q) {
                x[q].x *= ra;
                x[q].y *= rbb;
                *p[q] = x[q];
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> TMA store
        sync();
        if (t == 0) {
#pragma unroll
            for (int x = 0; x < NBOX; ++x) tma_store_2d(&tm, rb + ch * kT2Rows, col0 + x * kT2Box, buf + x * kT2BoxBytes);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            const int nx = ch + kT2Stages - 1;  // refill the stage of chunk ch-1 once its store has read it
            if (ch >= 1 && nx < kT2Chunks) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                load_chunk(nx);
            }
        }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    sync();  // the shared memory (and its mbarriers) may be reused by the caller
    if (t <= kT2Stages) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bars + t)) : "memory");
}

}  // namespace
}  // namespace gcm
