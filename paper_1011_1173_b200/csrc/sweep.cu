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

// One CTA of kD threads: thread m owns column r0+m of the diagonal block.
template <int KMAX>
__global__ void __launch_bounds__(kD) diag_chain_kernel(double *__restrict__ L, int64_t n, int64_t ldl,
                                                        double *__restrict__ V, int k, int sigma, int64_t r0,
                                                        double *__restrict__ panel, unsigned long long *key,
                                                        int64_t ebase) {
    __shared__ double Ls[kD][kD + 1];  // Ls[m][j] = L(r0 + j, r0 + m)
    __shared__ double vrow[KMAX];
    __shared__ double IM[KMAX];
    __shared__ double2 cs[KMAX];
    __shared__ double rho_s;

    const int t = threadIdx.x;
    const int Db = (int)(n - r0 < kD ? n - r0 : kD);

    // load the block's upper triangle (coalesced: consecutive threads -> consecutive rows)
    for (int idx = t; idx < kD * kD; idx += kD) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) Ls[m][j] = L[(r0 + j) + (r0 + m) * ldl];
    }
    double v[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e) v[e] = (t < Db && e < k) ? V[(r0 + t) + (int64_t)e * n] : 0.0;
    __syncthreads();

    block_sweep<KMAX, kD + 1>(Ls, v, Db, k, sigma, r0, panel, V + r0, n, key, ebase, vrow, IM, cs, &rho_s);
    for (int idx = t; idx < kD * kD; idx += kD) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) L[(r0 + j) + (r0 + m) * ldl] = Ls[m][j];
    }
}

// Apply panel (rows r0 .. r0+Db-1) to columns c0 .. n-1, one thread per column.
template <int KMAX>
__global__ void __launch_bounds__(kApplyThreads) panel_apply_kernel(double *__restrict__ L, int64_t n, int64_t ldl,
                                                                    double *__restrict__ V, int k, int64_t r0,
                                                                    int64_t c0, const double *__restrict__ panel) {
    extern __shared__ double2 smem_apply[];
    double2 *cs = smem_apply;                                // [kD * k]
    double *rho = reinterpret_cast<double *>(cs + kD * k);   // [kD]
    double *nu = rho + kD;                                   // [k]
    const int t = threadIdx.x;
    const int Db = (int)(n - r0 < kD ? n - r0 : kD);
    for (int i = t; i < Db * k; i += kApplyThreads)
        cs[i] = make_double2(panel[2 * i], panel[2 * i + 1]);
    for (int i = t; i < Db; i += kApplyThreads) rho[i] = panel[2ll * kD * k + i];
    for (int i = t; i < k; i += kApplyThreads) nu[i] = panel[2ll * kD * k + kD + i];
    __syncthreads();

    const int64_t m = c0 + (int64_t)blockIdx.x * kApplyThreads + t;
    if (m >= n) return;
    double v[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e) v[e] = e < k ? V[m + (int64_t)e * n] : 0.0;
    double *col = L + m * ldl + r0;
    for (int j = 0; j < Db; ++j) col[j] = apply_row<KMAX>(col[j], v, cs + j * k, rho[j], k);
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
        if (e < k) V[m + (int64_t)e * n] = v[e] * nu[e];
}

template <int KMAX>
gcm_status_t sweep_pass(double *L, int64_t n, int64_t ldl, double *V, int k, int sigma,
                        unsigned long long *key, double *panels, int64_t ebase, cudaStream_t stream) {
    const int64_t nb = (n + kD - 1) / kD;
    const int64_t pstride = panel_doubles(k);
    const size_t smem = panel_doubles(k) * sizeof(double);
    // per device context; cheap, so set on every call rather than cache per device
    cudaError_t err = cudaFuncSetAttribute(panel_apply_kernel<KMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(panel_doubles(KMAX) * sizeof(double)));
    if (err != cudaSuccess) return check_cuda(err);
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t r0 = b * kD;
        double *panel = panels + b * pstride;
        {
            ProfScope ps("diag_chain", stream);
            diag_chain_kernel<KMAX><<<1, kD, 0, stream>>>(L, n, ldl, V, k, sigma, r0, panel, key, ebase);
        }
        const int64_t c0 = r0 + kD;
        if (c0 < n) {
            const unsigned grid = (unsigned)((n - c0 + kApplyThreads - 1) / kApplyThreads);
            ProfScope ps("panel_apply", stream);
            panel_apply_kernel<KMAX><<<grid, kApplyThreads, smem, stream>>>(L, n, ldl, V, k, r0, c0, panel);
        }
    }
    return check_cuda(cudaGetLastError());
}

}  // namespace

gcm_status_t modify_sweep(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                          unsigned long long *key, double *panels, cudaStream_t stream) {
    for (int64_t e0 = 0; e0 < k; e0 += kKMax) {
        const int kc = (int)std::min<int64_t>(kKMax, k - e0);
        double *Vc = V + e0 * n;
        gcm_status_t st;
        if (kc <= 1) st = sweep_pass<1>(L, n, ldl, Vc, kc, sigma, key, panels, e0, stream);
        else if (kc <= 4) st = sweep_pass<4>(L, n, ldl, Vc, kc, sigma, key, panels, e0, stream);
        else if (kc <= 8) st = sweep_pass<8>(L, n, ldl, Vc, kc, sigma, key, panels, e0, stream);
        else if (kc <= 16) st = sweep_pass<16>(L, n, ldl, Vc, kc, sigma, key, panels, e0, stream);
        else if (kc <= 32) st = sweep_pass<32>(L, n, ldl, Vc, kc, sigma, key, panels, e0, stream);
        else st = sweep_pass<64>(L, n, ldl, Vc, kc, sigma, key, panels, e0, stream);
        if (st != GCM_OK) return st;
    }
    return GCM_OK;
}

}  // namespace gcm
