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

#include "internal.h"
#include "rot.cuh"

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
    }
    return check_cuda(cudaGetLastError());
}

template <int KB>
gcm_status_t batched_launch(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V, int64_t strideV, int k,
                            int sigma, int64_t batch, unsigned long long *keys, cudaStream_t stream) {
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
    const gcm_algo_t algo = pick_algo(n, k, GCM_ALGO_AUTO);
    gcm_status_t st = get_workspace(stream, single_workspace_bytes(n, k, algo), (size_t)batch, &ws);
    if (st != GCM_OK) return st;
    for (int64_t f = 0; f < batch; ++f) {
        st = run_single(L + f * strideL, n, ldl, V + f * strideV, k, sigma, algo, ws->key + f, ws, stream);
        if (st != GCM_OK) return st;
    }
    return finalize_info(ws->key, d_info, batch, stream);
}

}  // namespace gcm
