// batched.cu -- gcm_modify_batched: many independent factors of one shape
// (BASELINE.json configs[4]: 4096 factors, n = 512, k = 8).
//
// One CTA runs one factor through the paper's panel order (PAPER.md 76-77):
// for each 64-row block b, the owner warps of the block's columns run the
// diagonal Compute chain (rot.cuh block_sweep) into a shared-memory coefficient
// panel, then every thread applies that panel to the rows of block b of its own
// columns (PAPER.md 91-106).  Column c is owned by thread c mod blockDim for the
// whole call, so its k V entries live in registers from the first panel to its
// own diagonal block; the factor's L is read and written exactly once.  Factors
// are independent, so the grid is simply the batch (many CTAs per SM hide one
// CTA's serial diagonal chain behind the others' Apply streams).
#include <algorithm>
#include <cstdlib>

#include "diag.cuh"
#include "internal.h"
#include "rot.cuh"
#include "tma.cuh"

namespace gcm {

namespace {

constexpr int kBT = 256;          // threads per factor CTA
constexpr int kMaxSlotsAll = 4;   // columns per thread -> n <= kBT * kMaxSlotsAll
constexpr int kRows = 8;          // rows of a column loaded per register batch
constexpr int kBatchNQ = 2;       // threads per column in the diagonal sweep (+ one coefficient warp)

template <int KB, int kMaxSlots>
__global__ void __launch_bounds__(kBT, 3) batched_kernel(double *__restrict__ Lall, int64_t n, int64_t ldl,
                                                      int64_t strideL, double *__restrict__ Vall, int64_t strideV,
                                                      int k, int sigma, unsigned long long *__restrict__ keys) {
    extern __shared__ double smem_b[];
    double(*Ls)[kD + 1] = reinterpret_cast<double(*)[kD + 1]>(smem_b);  // [kD][kD+1]
    double *panel = smem_b + kD * (kD + 1);                              // panel_doubles(k)
    double *vx = panel + wave_panel_doubles(KB) + 1;                     // [kD*KB] wave_sweep scratch
    double *dinv = vx + kD * KB;                                         // [kD]
    double *vt = dinv + kD;                                              // [kD*KB]
    double *imx = vt + kD * KB;                                          // [kD*KB]
    double *Vs = imx + kD * KB;                                          // [kD*KB]

    const int t = threadIdx.x;
    const int64_t f = blockIdx.x;
    double *L = Lall + f * strideL;
    double *V = Vall + f * strideV;
    unsigned long long *key = keys + f;
    const int nb = (int)((n + kD - 1) / kD);

    double v[kMaxSlots][KB];
#pragma unroll
    for (int s = 0; s < kMaxSlots; ++s) {
        const int64_t c = t + (int64_t)s * kBT;
#pragma unroll
        for (int e = 0; e < KB; ++e) v[s][e] = (c < n && e < k) ? V[c + (int64_t)e * n] : 0.0;
    }
    if (t == 0) *key = kInfoNone;

    for (int b = 0; b < nb; ++b) {
        const int64_t r0 = (int64_t)b * kD;
        const int Db = (int)(n - r0 < kD ? n - r0 : kD);
        // ---- diagonal block b: the owner threads of its columns run the chain
        for (int idx = t; idx < kD * kD; idx += kBT) {
            const int m = idx / kD, j = idx % kD;
            if (m < Db && j <= m) Ls[m][j] = L[(r0 + j) + (r0 + m) * ldl];
        }
        // owner threads hand their V state of the block's columns to the sweep
        const int slot_b = (int)(r0 / kBT);
        const int tbase = (int)(r0 % kBT);
        if (t >= tbase && t < tbase + kD) {
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                double x = 0.0;
#pragma unroll
                for (int s = 0; s < kMaxSlots; ++s)
                    if (s == slot_b) x = v[s][e];
                Vs[(t - tbase) * KB + e] = x;
            }
        }
        __syncthreads();
        wave_sweep<KB, kBatchNQ, kD + 1>(Ls, Vs, Db, k, sigma, r0, panel, V + r0, n, key, 0, vx, dinv, vt, imx, 0,
                                         kBatchNQ * kD / 32);
        for (int idx = t; idx < kD * kD; idx += kBT) {
            const int m = idx / kD, j = idx % kD;
            if (m < Db && j <= m) L[(r0 + j) + (r0 + m) * ldl] = Ls[m][j];
        }
        if (b + 1 == nb) break;
        // ---- Apply panel b to rows r0.. of every column to the right of the block
        const double2 *pcs = reinterpret_cast<const double2 *>(panel);  // stride KB (padded rank)
        const double *prho = panel + 2 * kD * KB;
        const double *pnu = prho + kD;
#pragma unroll
        for (int s = 0; s < kMaxSlots; ++s) {
            const int64_t c = t + (int64_t)s * kBT;
            if (c < r0 + kD || c >= n) continue;
            double *col = L + c * ldl + r0;
            double buf[kRows];
#pragma unroll
            for (int q = 0; q < kRows; ++q) buf[q] = col[q];
            for (int j0 = 0; j0 < kD; j0 += kRows) {
                double nxt[kRows];
                if (j0 + kRows < kD) {
#pragma unroll
                    for (int q = 0; q < kRows; ++q) nxt[q] = col[j0 + kRows + q];
                }
#pragma unroll
                for (int q = 0; q < kRows; ++q)
                    col[j0 + q] = apply_row<KB>(buf[q], v[s], pcs + (j0 + q) * KB, prho[j0 + q], KB);
                if (j0 + kRows < kD) {
#pragma unroll
                    for (int q = 0; q < kRows; ++q) buf[q] = nxt[q];
                }
            }
#pragma unroll
            for (int e = 0; e < KB; ++e) v[s][e] *= (e < k) ? pnu[e] : 1.0;
        }
        __syncthreads();  // panel and Ls reused by the next block
    }
}

// ---------------------------------------------------------------- TMA batched kernel
// One CTA (256 threads) per factor, thread t owning columns t + 256 s (V state in
// registers, as above); per 64-row block b:
//   diagonal block: closed form (diag.cuh) -- q = L_bb^{-T} Y (one short in-block solve),
//     every row's V state and rotations in parallel, the panel, V_exit, L~_bb -- instead of
//     the D + k - 1 tick wavefront (rot.cuh wave_sweep: ~36 us per block at k = 8);
//   Apply of panel b (PAPER.md 52-54) to the rows of block b of every column right of it:
//     8-row chunks arrive as 8 x 64 TMA boxes (one per 64-column strip; 64B swizzle, so a
//     thread's row pair is one conflict-free 16-byte shared load) in a 2-stage ring, are
//     rotated in place and leave by TMA stores -- every L element is read and written once,
//     in full 128-byte lines.
// The diagonal block's shared memory aliases the ring (they are never live together), so
// three factors share an SM and one's diagonal block overlaps the others' streams.
constexpr unsigned kBBox = 8 * kD * 8;  // bytes of one 8-row x 64-column box

#ifdef GCM_BT_TRACE  // phase clocks of two CTAs (tools/batched_trace.py)
__device__ long long g_bt_trace[2 * 16 * 8];
#define BT_MARK(b, slot)                                                                          \
    do {                                                                                          \
        if (t == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2) && (b) < 16)               \
            g_bt_trace[((blockIdx.x == 0 ? 0 : 1) * 16 + (b)) * 8 + (slot)] = clock64();         \
    } while (0)
#else
#define BT_MARK(b, slot) ((void)0)
#endif

template <int KB>
__host__ __device__ constexpr int bt_diag_doubles() {
    return kD * (kD + 1) + kD * (KB + 1) + diag_closed_scratch(KB) + kD;
}

#ifndef GCM_BT_INTERLEAVE
#define GCM_BT_INTERLEAVE 0  // 1: a thread's columns rotate in one loop (measured slower)
#endif
#ifndef GCM_BT_STAGES
#define GCM_BT_STAGES 3
#endif
constexpr int kBTStages = GCM_BT_STAGES;  // ring depth: chunks ch+1, ch+2 land while ch is rotated

#ifndef GCM_BT_MINB
#define GCM_BT_MINB 2
#endif
template <int KB, int SLOTS>
__global__ void __launch_bounds__(kBT, KB <= 8 ? GCM_BT_MINB : 2) batched_tma_kernel(const __grid_constant__ CUtensorMap tm,
                                                          double *__restrict__ Lall, int64_t n, int64_t ldl,
                                                          int64_t strideL, double *__restrict__ Vall, int64_t strideV,
                                                          int k, int sigma, unsigned long long *__restrict__ keys,
                                                          unsigned stage_bytes) {
    extern __shared__ __align__(1024) unsigned char smem_bt[];
    const unsigned sbase = smem_u32(smem_bt);
    unsigned char *ring = smem_bt + (((sbase + 1023u) & ~1023u) - sbase);  // swizzled boxes: 1 KB aligned
    const unsigned region = max(kBTStages * stage_bytes, (unsigned)(bt_diag_doubles<KB>() * 8));
    double *pan = reinterpret_cast<double *>(ring + ((region + 15) & ~15u));  // panel_doubles(KB)
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(pan + ((panel_doubles(KB) + 1) & ~1));
    // the diagonal block's scratch (aliases the ring)
    double(*Ls)[kD + 1] = reinterpret_cast<double(*)[kD + 1]>(ring);
    double *qv = reinterpret_cast<double *>(ring) + kD * (kD + 1);  // [kD][KB+1]: Y, then q
    double *scr = qv + kD * (KB + 1);
    double *rinv = scr + diag_closed_scratch(KB);
    constexpr int LQ = KB + 1;

    const int t = threadIdx.x;
    const int64_t f = blockIdx.x;
    double *L = Lall + f * strideL;
    double *V = Vall + f * strideV;
    unsigned long long *key = keys + f;
    const int NB = (int)((n + kD - 1) / kD);
    const int NS = NB;  // 64-column strips

    double v[SLOTS][KB];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int64_t c = t + (int64_t)s * kBT;
#pragma unroll
        for (int e = 0; e < KB; ++e) v[s][e] = (c < n && e < k) ? V[c + (int64_t)e * n] : 0.0;
    }
    if (t == 0) {
        *key = kInfoNone;
        for (int i = 0; i < kBTStages; ++i) mbar_init(bars + i, 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned phase = 0;  // bit i: parity of ring stage i's next completion

    for (int b = 0; b < NB; ++b) {
        const int64_t r0 = (int64_t)b * kD;
        const int Db = (int)(n - r0 < kD ? n - r0 : kD);
        const int slot_b = (int)(r0 / kBT), tb = (int)(r0 % kBT);
        const bool owner = t >= tb && t < tb + Db;
        __syncthreads();  // the ring's last stores have read shared memory (thread 0 waited)
        BT_MARK(b, 0);
        // ---- diagonal block b: every element's copy in flight at once (cp.async, no registers)
        for (int idx = t; idx < kD * kD; idx += kBT) {
            const int m = idx / kD, j = idx % kD;
            if (m < Db && j <= m) {
                const unsigned d = smem_u32(&Ls[m][j]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(L + (r0 + j) + (r0 + m) * ldl)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        double y[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            double x = 0.0;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s)
                if (s == slot_b) x = v[s][e];
            y[e] = x;
        }
        if (owner)
#pragma unroll
            for (int e = 0; e < KB; ++e) qv[(t - tb) * LQ + e] = y[e];
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        BT_MARK(b, 1);
        block_trsv<KB>(Ls, qv, LQ, Db, rinv);
        BT_MARK(b, 2);
        diag_closed<KB>(Ls, qv, LQ, Db, k, sigma, r0, pan, V + r0, n, key, 0, scr);
        BT_MARK(b, 3);
        if (owner) diag_triangle<KB>(Ls, t - tb, y, pan);
        __syncthreads();
        BT_MARK(b, 4);
        for (int idx = t; idx < kD * kD; idx += kBT) {
            const int m = idx / kD, j = idx % kD;
            if (m < Db && j <= m) L[(r0 + j) + (r0 + m) * ldl] = Ls[m][j];
        }
        if (b + 1 == NB) break;
        __syncthreads();  // Ls read out before the ring overwrites it
        BT_MARK(b, 5);
        // ---- Apply panel b to strips b+1 .. NS-1 (rows r0 .. r0+63)
        const int s1 = b + 1, nstr = NS - s1;
        const unsigned chunk_bytes = (unsigned)nstr * kBBox;
        auto issue = [&](int ch) {  // thread 0
            unsigned long long *bar = bars + ch % kBTStages;
            unsigned char *st = ring + (ch % kBTStages) * stage_bytes;
            mbar_arrive_expect_tx(bar, chunk_bytes);
            for (int s = 0; s < nstr; ++s)
                tma_load_3d(st + s * kBBox, &tm, (int)r0 + 8 * ch, (s1 + s) * kD, (int)f, bar);
        };
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem use -> TMA writes
            for (int ch = 0; ch < kBTStages; ++ch) issue(ch);
        }
        const double2 *cs = reinterpret_cast<const double2 *>(pan);
        const double *rho = pan + 2 * kD * KB;
        constexpr int NCH = kD / 8;
        static_assert(NCH >= kBTStages, "ring deeper than a block's chunks");
        for (int ch = 0; ch < NCH; ++ch) {
            const int sg = ch % kBTStages;
            mbar_wait(bars + sg, (phase >> sg) & 1u);
            phase ^= 1u << sg;
            unsigned char *st = ring + sg * stage_bytes;
#if GCM_BT_INTERLEAVE
            // the thread's columns rotate together: each (gamma, delta) load feeds every slot,
            // and the slots' independent FMA chains interleave
            bool act[SLOTS];
            double2 *col[SLOTS];
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int c = t + s * kBT;
                const int strip = c / kD;
                act[s] = strip >= s1 && c < n;
                const int cc = c % kD;
                col[s] = reinterpret_cast<double2 *>(st + (act[s] ? strip - s1 : 0) * kBBox + cc * 64);
            }
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) {
                double2 x[SLOTS];
                double2 *pp[SLOTS];
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) {
                    const int cc = (t + s * kBT) % kD;
                    pp[s] = col[s] + (jp ^ ((cc >> 1) & 3));
                    x[s] = act[s] ? *pp[s] : make_double2(0.0, 0.0);
                }
                const int j = 8 * ch + 2 * jp;
                const double2 *g0 = cs + j * KB, *g1 = g0 + KB;
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    const double2 gd = g0[e];
#pragma unroll
                    for (int s = 0; s < SLOTS; ++s) {
                        x[s].x = fma(gd.x, v[s][e], x[s].x);
                        v[s][e] = fma(-gd.y, x[s].x, v[s][e]);
                    }
                }
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    const double2 gd = g1[e];
#pragma unroll
                    for (int s = 0; s < SLOTS; ++s) {
                        x[s].y = fma(gd.x, v[s][e], x[s].y);
                        v[s][e] = fma(-gd.y, x[s].y, v[s][e]);
                    }
                }
                const double ra = rho[j], rb = rho[j + 1];
#pragma unroll
                for (int s = 0; s < SLOTS; ++s)
                    if (act[s]) *pp[s] = make_double2(x[s].x * ra, x[s].y * rb);
            }
#else
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int c = t + s * kBT;
                const int strip = c / kD;
                if (strip < s1 || c >= n) continue;
                const int cc = c % kD;
                unsigned char *col = st + (strip - s1) * kBBox + cc * 64;
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {
                    double2 *p = reinterpret_cast<double2 *>(col + ((jp ^ ((cc >> 1) & 3)) << 4));
                    double2 x = *p;
                    const int j = 8 * ch + 2 * jp;
                    const double2 *g0 = cs + j * KB, *g1 = g0 + KB;
#pragma unroll
                    for (int e = 0; e < KB; ++e) {
                        const double2 gd = g0[e];
                        x.x = fma(gd.x, v[s][e], x.x);
                        v[s][e] = fma(-gd.y, x.x, v[s][e]);
                    }
#pragma unroll
                    for (int e = 0; e < KB; ++e) {
                        const double2 gd = g1[e];
                        x.y = fma(gd.x, v[s][e], x.y);
                        v[s][e] = fma(-gd.y, x.y, v[s][e]);
                    }
                    x.x *= rho[j];
                    x.y *= rho[j + 1];
                    *p = x;
                }
            }
#endif
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> TMA store
            __syncthreads();
            if (t == 0) {
                for (int s = 0; s < nstr; ++s) tma_store_3d(&tm, (int)r0 + 8 * ch, (s1 + s) * kD, (int)f, st + s * kBBox);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // refill the stage of chunk ch-1 (its store had a whole chunk to drain; the
                // store just committed may still be reading)
                if (ch >= 1 && ch + kBTStages - 1 < NCH) {
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    issue(ch + kBTStages - 1);
                }
            }
        }
        if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        BT_MARK(b, 6);
        // V states back to true values at the block end (rot.cuh: V = Vt * nu)
        const double *nu = rho + kD;
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int c = t + s * kBT;
            if (c / kD >= s1 && c < n)
#pragma unroll
                for (int e = 0; e < KB; ++e) v[s][e] *= nu[e];
        }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores globally done
}

template <int KB, int SLOTS>
bool batched_tma_launch(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V, int64_t strideV, int k,
                        int sigma, int64_t batch, unsigned long long *keys, cudaStream_t stream, gcm_status_t *st) {
    CUtensorMap tm;
    if (!encode_tmap_f64(&tm, L, 3, n, n, ldl, batch, strideL, 8u, (unsigned)kD, CU_TENSOR_MAP_SWIZZLE_64B))
        return false;
    const int NB = (int)((n + kD - 1) / kD);
    const unsigned stage = (unsigned)std::max(NB - 1, 1) * kBBox;
    const size_t region = std::max<size_t>((size_t)kBTStages * stage, (size_t)bt_diag_doubles<KB>() * 8);
    const size_t smem = 1024 + ((region + 15) & ~(size_t)15) + (size_t)((panel_doubles(KB) + 1) & ~1) * 8 + 8 * kBTStages;
    *st = check_cuda(
        cudaFuncSetAttribute(batched_tma_kernel<KB, SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (*st != GCM_OK) return true;
    for (int64_t f0 = 0; f0 < batch; f0 += 0x7fffffff) {
        const unsigned grid = (unsigned)std::min<int64_t>(batch - f0, 0x7fffffff);
        ProfScope ps("batched", stream);
        // factor index f0 + blockIdx.x goes through the tensor map's batch coordinate: one
        // launch covers < 2^31 factors, the map is re-encoded for the next range
        if (f0 > 0 && !encode_tmap_f64(&tm, L + f0 * strideL, 3, n, n, ldl, batch - f0, strideL, 8u, (unsigned)kD,
                                       CU_TENSOR_MAP_SWIZZLE_64B)) {
            *st = GCM_ECUDA;
            return true;
        }
        batched_tma_kernel<KB, SLOTS><<<grid, kBT, smem, stream>>>(tm, L + f0 * strideL, n, ldl, strideL,
                                                                   V + f0 * strideV, strideV, k, sigma, keys + f0,
                                                                   stage);
        count_launch();
    }
    *st = check_cuda(cudaGetLastError());
    return true;
}

template <int KB, int SLOTS>
gcm_status_t batched_launch_s(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V, int64_t strideV, int k,
                              int sigma, int64_t batch, unsigned long long *keys, cudaStream_t stream) {
    const size_t smem = (size_t)(kD * (kD + 1) + wave_panel_doubles(KB) + 1 + 4 * kD * KB + kD) * sizeof(double);
    gcm_status_t st = check_cuda(
        cudaFuncSetAttribute(batched_kernel<KB, SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (st != GCM_OK) return st;
    for (int64_t f0 = 0; f0 < batch; f0 += 0x7fffffff) {
        const unsigned grid = (unsigned)std::min<int64_t>(batch - f0, 0x7fffffff);
        ProfScope ps("batched", stream);
        batched_kernel<KB, SLOTS><<<grid, kBT, smem, stream>>>(L + f0 * strideL, n, ldl, strideL, V + f0 * strideV,
                                                               strideV, k, sigma, keys + f0);
        count_launch();
    }
    return check_cuda(cudaGetLastError());
}

template <int KB>
gcm_status_t batched_launch(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V, int64_t strideV, int k,
                            int sigma, int64_t batch, unsigned long long *keys, cudaStream_t stream) {
    // TMA path: rank buckets <= 16, n <= 512 (two columns per thread), L 16-byte aligned with an
    // even ldl and strideL (tensor-map strides); else the register-column kernel below
    if constexpr (KB <= 16) {
        if (n <= 2 * kBT && std::getenv("GCM_BATCHED_LEGACY") == nullptr) {
            gcm_status_t st = GCM_OK;
            if (batched_tma_launch<KB, 2>(L, n, ldl, strideL, V, strideV, k, sigma, batch, keys, stream, &st))
                return st;
        }
    }
    if (n <= kBT) return batched_launch_s<KB, 1>(L, n, ldl, strideL, V, strideV, k, sigma, batch, keys, stream);
    if (n <= 2 * kBT) return batched_launch_s<KB, 2>(L, n, ldl, strideL, V, strideV, k, sigma, batch, keys, stream);
    return batched_launch_s<KB, 4>(L, n, ldl, strideL, V, strideV, k, sigma, batch, keys, stream);
}

}  // namespace

gcm_status_t modify_batched(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V, int64_t strideV,
                            int64_t k, int sigma, int64_t batch, gcm_info_t *d_info, cudaStream_t stream) {
    Workspace *ws = nullptr;
    if (n <= (int64_t)kBT * kMaxSlotsAll && k <= 32) {
        gcm_status_t st = get_workspace(stream, 256, (size_t)batch, &ws);
        if (st != GCM_OK) return st;
        // the kernel resets each factor's failure key itself
        const int kc = (int)k;
        if (kc <= 4) st = batched_launch<4>(L, n, ldl, strideL, V, strideV, kc, sigma, batch, ws->key, stream);
        else if (kc <= 8) st = batched_launch<8>(L, n, ldl, strideL, V, strideV, kc, sigma, batch, ws->key, stream);
        else if (kc <= 16) st = batched_launch<16>(L, n, ldl, strideL, V, strideV, kc, sigma, batch, ws->key, stream);
        else st = batched_launch<32>(L, n, ldl, strideL, V, strideV, kc, sigma, batch, ws->key, stream);
        if (st != GCM_OK) return st;
        return finalize_info(ws->key, d_info, batch, stream);
    }
    // larger factors: one single-factor call per factor on the same stream (each
    // already fills the GPU), each reporting into its own failure slot
    gcm_algo_t algo = pick_algo(n, k, GCM_ALGO_AUTO);
    if (algo == GCM_ALGO_PANEL) algo = GCM_ALGO_BLOCKED;  // the per-factor loop runs on one workspace
    gcm_status_t st = get_workspace(stream, single_workspace_bytes(n, k, algo), (size_t)batch, &ws);
    if (st != GCM_OK) return st;
    for (int64_t f = 0; f < batch; ++f) {
        st = run_single(L + f * strideL, n, ldl, V + f * strideV, k, sigma, algo, ws->key + f, ws, stream);
        if (st != GCM_OK) return st;
    }
    return finalize_info(ws->key, d_info, batch, stream);
}

}  // namespace gcm

#ifdef GCM_BT_TRACE
extern "C" int gcm_debug_bt_trace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, gcm::g_bt_trace, sizeof(long long) * count);
}
extern "C" int gcm_debug_dc_trace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, gcm::g_dc_trace, sizeof(long long) * count);
}
#endif
