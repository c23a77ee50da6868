// sweep.cu -- GCM_ALGO_SWEEP: the paper's panel order (PAPER.md lines 76-77:
// diagonal block, then the off-diagonal panel to its right, then the next
// diagonal block ...) with BOTH roles on the GPU:
//   diag_chain_kernel : the serial Compute chain of one D-row diagonal block
//                       (the paper ran it on the CPU)
//   panel_apply_kernel: the data-parallel Apply of that block's k*D rotations
//                       to every column to its right:
//                       one thread per L column, its k V entries in registers,
//                       all k rotations applied per L read, each L element read
//                       and written once per pass.
#include <algorithm>

#include "internal.h"
#include "rot.cuh"

namespace gcm {

namespace {

constexpr int kApplyThreads = 128;

// One CTA of kD threads: thread m owns column m of the diagonal block.
// Lb points at element (r0, first column of the block); L(r0+j, col m) = Lb[j + m*ldl].
// Vb points at the V row of the block's first column; V(col m, e) = Vb[m + e*ldv].
template <int KMAX>
__global__ void __launch_bounds__(kD) diag_chain_kernel(double *__restrict__ Lb, int64_t ldl, int Db,
                                                        double *__restrict__ Vb, int64_t ldv, int k, int sigma,
                                                        int64_t grow0, double *__restrict__ panel,
                                                        unsigned long long *key, int64_t ebase) {
    __shared__ double Ls[kD][kD + 1];  // Ls[m][j] = L(r0 + j, col m)
    __shared__ double vrow[KMAX];
    __shared__ double IM[KMAX];
    __shared__ double2 cs[KMAX];
    __shared__ double rho_s;

    const int t = threadIdx.x;
    // load the block's upper triangle (coalesced: consecutive threads -> consecutive rows)
    for (int idx = t; idx < kD * kD; idx += kD) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) Ls[m][j] = Lb[j + m * ldl];
    }
    double v[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e) v[e] = (t < Db && e < k) ? Vb[t + (int64_t)e * ldv] : 0.0;
    __syncthreads();

    block_sweep<KMAX, kD + 1>(Ls, v, Db, k, sigma, grow0, panel, Vb, ldv, key, ebase, vrow, IM, cs, &rho_s);
    for (int idx = t; idx < kD * kD; idx += kD) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) Lb[j + m * ldl] = Ls[m][j];
    }
}

// Apply a panel (Db rows) to ncols columns, one thread per column.
// Lr points at element (r0, first column); Vc at the first column's V row (ld ldv).
template <int KMAX>
__global__ void __launch_bounds__(kApplyThreads) panel_apply_kernel(double *__restrict__ Lr, int64_t ldl, int Db,
                                                                    int64_t ncols, double *__restrict__ Vc,
                                                                    int64_t ldv, int k,
                                                                    const double *__restrict__ panel) {
    extern __shared__ double2 smem_apply[];
    double2 *cs = smem_apply;                                // [kD * k]
    double *rho = reinterpret_cast<double *>(cs + kD * k);   // [kD]
    double *nu = rho + kD;                                   // [k]
    const int t = threadIdx.x;
    for (int i = t; i < Db * k; i += kApplyThreads)
        cs[i] = make_double2(panel[2 * i], panel[2 * i + 1]);
    for (int i = t; i < Db; i += kApplyThreads) rho[i] = panel[2ll * kD * k + i];
    for (int i = t; i < k; i += kApplyThreads) nu[i] = panel[2ll * kD * k + kD + i];
    __syncthreads();

    const int64_t m = (int64_t)blockIdx.x * kApplyThreads + t;
    if (m >= ncols) return;
    double v[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e) v[e] = e < k ? Vc[m + (int64_t)e * ldv] : 0.0;
    double *col = Lr + m * ldl;
    for (int j = 0; j < Db; ++j) col[j] = apply_row<KMAX>(col[j], v, cs + j * k, rho[j], k);
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
        if (e < k) Vc[m + (int64_t)e * ldv] = v[e] * nu[e];
}

template <int KMAX>
gcm_status_t diag_launch(double *Lb, int64_t ldl, int Db, double *Vb, int64_t ldv, int k, int sigma, int64_t grow0,
                         double *panel, unsigned long long *key, int64_t ebase, cudaStream_t stream) {
    ProfScope ps("diag_chain", stream);
    diag_chain_kernel<KMAX><<<1, kD, 0, stream>>>(Lb, ldl, Db, Vb, ldv, k, sigma, grow0, panel, key, ebase);
    count_launch();
    return check_cuda(cudaGetLastError());
}

template <int KMAX>
gcm_status_t apply_launch(double *Lr, int64_t ldl, int Db, int64_t ncols, double *Vc, int64_t ldv, int k,
                          const double *panel, cudaStream_t stream) {
    if (ncols <= 0) return GCM_OK;
    // per device context; cheap, so set on every call rather than cache per device
    cudaError_t err = cudaFuncSetAttribute(panel_apply_kernel<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(panel_doubles(KMAX) * sizeof(double)));
    if (err != cudaSuccess) return check_cuda(err);
    const size_t smem = panel_doubles(k) * sizeof(double);
    const unsigned grid = (unsigned)((ncols + kApplyThreads - 1) / kApplyThreads);
    ProfScope ps("panel_apply", stream);
    panel_apply_kernel<KMAX><<<grid, kApplyThreads, smem, stream>>>(Lr, ldl, Db, ncols, Vc, ldv, k, panel);
    count_launch();
    return check_cuda(cudaGetLastError());
}

#define GCM_KMAX_DISPATCH(k, CALL)                 \
    ((k) <= 1    ? CALL(1)                         \
     : (k) <= 4  ? CALL(4)                         \
     : (k) <= 8  ? CALL(8)                         \
     : (k) <= 16 ? CALL(16)                        \
     : (k) <= 32 ? CALL(32)                        \
                 : CALL(64))

}  // namespace

gcm_status_t sweep_diag(double *Lb, int64_t ldl, int Db, double *Vb, int64_t ldv, int k, int sigma, int64_t grow0,
                        double *panel, unsigned long long *key, int64_t ebase, cudaStream_t stream) {
#define CALL(KM) diag_launch<KM>(Lb, ldl, Db, Vb, ldv, k, sigma, grow0, panel, key, ebase, stream)
    return GCM_KMAX_DISPATCH(k, CALL);
#undef CALL
}

gcm_status_t sweep_apply(double *Lr, int64_t ldl, int Db, int64_t ncols, double *Vc, int64_t ldv, int k,
                         const double *panel, cudaStream_t stream) {
#define CALL(KM) apply_launch<KM>(Lr, ldl, Db, ncols, Vc, ldv, k, panel, stream)
    return GCM_KMAX_DISPATCH(k, CALL);
#undef CALL
}

gcm_status_t modify_sweep(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                          unsigned long long *key, double *panels, cudaStream_t stream) {
    const int64_t nb = (n + kD - 1) / kD;
    for (int64_t e0 = 0; e0 < k; e0 += kKMax) {
        const int kc = (int)std::min<int64_t>(kKMax, k - e0);
        double *Vc = V + e0 * n;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t r0 = b * kD;
            const int Db = (int)std::min<int64_t>(kD, n - r0);
            double *panel = panels + b * panel_doubles(kc);
            gcm_status_t st = sweep_diag(L + r0 + r0 * ldl, ldl, Db, Vc + r0, n, kc, sigma, r0, panel, key, e0, stream);
            if (st != GCM_OK) return st;
            const int64_t c0 = r0 + kD;
            if (c0 < n) st = sweep_apply(L + r0 + c0 * ldl, ldl, Db, n - c0, Vc + c0, n, kc, panel, stream);
            if (st != GCM_OK) return st;
        }
    }
    return GCM_OK;
}

}  // namespace gcm
