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
// (templated on the element type T: double, or float for the single-precision entry point
// gcm_modify_f32 -- PAPER.md 111 ran both precisions)
template <int KMAX, typename T>
__global__ void __launch_bounds__(kD) diag_chain_kernel(T *__restrict__ Lb, int64_t ldl, int Db, T *__restrict__ Vb,
                                                        int64_t ldv, int k, int sigma, int64_t grow0,
                                                        T *__restrict__ panel, unsigned long long *key,
                                                        int64_t ebase) {
    __shared__ T Ls[kD][kD + 1];  // Ls[m][j] = L(r0 + j, col m)
    __shared__ T vrow[KMAX];
    __shared__ T IM[KMAX];
    __shared__ typename V2<T>::type cs[KMAX];
    __shared__ T rho_s;

    const int t = threadIdx.x;
    // load the block's upper triangle (coalesced: consecutive threads -> consecutive rows)
    for (int idx = t; idx < kD * kD; idx += kD) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) Ls[m][j] = Lb[j + m * ldl];
    }
    T v[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e) v[e] = (t < Db && e < k) ? Vb[t + (int64_t)e * ldv] : T(0);
    __syncthreads();

    block_sweep<KMAX, kD + 1>(Ls, v, Db, k, sigma, grow0, panel, Vb, ldv, key, ebase, vrow, IM, cs, &rho_s);
    for (int idx = t; idx < kD * kD; idx += kD) {
        const int m = idx / kD, j = idx % kD;
        if (m < Db && j <= m) Lb[j + m * ldl] = Ls[m][j];
    }
}

// Apply a panel (Db rows) to ncols columns, one thread per column.
// Lr points at element (r0, first column); Vc at the first column's V row (ld ldv).
template <int KMAX, typename T>
__global__ void __launch_bounds__(kApplyThreads) panel_apply_kernel(T *__restrict__ Lr, int64_t ldl, int Db,
                                                                    int64_t ncols, T *__restrict__ Vc, int64_t ldv,
                                                                    int k, const T *__restrict__ panel) {
    using T2 = typename V2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_apply_raw[];
    T2 *cs = reinterpret_cast<T2 *>(smem_apply_raw);  // [kD * k]
    T *rho = reinterpret_cast<T *>(cs + kD * k);       // [kD]
    T *nu = rho + kD;                                  // [k]
    const int t = threadIdx.x;
    for (int i = t; i < Db * k; i += kApplyThreads) cs[i] = V2<T>::make(panel[2 * i], panel[2 * i + 1]);
    for (int i = t; i < Db; i += kApplyThreads) rho[i] = panel[2ll * kD * k + i];
    for (int i = t; i < k; i += kApplyThreads) nu[i] = panel[2ll * kD * k + kD + i];
    __syncthreads();

    const int64_t m = (int64_t)blockIdx.x * kApplyThreads + t;
    if (m >= ncols) return;
    T v[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e) v[e] = e < k ? Vc[m + (int64_t)e * ldv] : T(0);
    T *col = Lr + m * ldl;
    for (int j = 0; j < Db; ++j) col[j] = apply_row<KMAX>(col[j], v, cs + j * k, rho[j], k);
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
        if (e < k) Vc[m + (int64_t)e * ldv] = v[e] * nu[e];
}

template <int KMAX, typename T>
gcm_status_t diag_launch(T *Lb, int64_t ldl, int Db, T *Vb, int64_t ldv, int k, int sigma, int64_t grow0, T *panel,
                         unsigned long long *key, int64_t ebase, cudaStream_t stream) {
    ProfScope ps("diag_chain", stream);
    diag_chain_kernel<KMAX, T><<<1, kD, 0, stream>>>(Lb, ldl, Db, Vb, ldv, k, sigma, grow0, panel, key, ebase);
    count_launch();
    return check_cuda(cudaGetLastError());
}

template <int KMAX, typename T>
gcm_status_t apply_launch(T *Lr, int64_t ldl, int Db, int64_t ncols, T *Vc, int64_t ldv, int k, const T *panel,
                          cudaStream_t stream) {
    if (ncols <= 0) return GCM_OK;
    // per device context; cheap, so set on every call rather than cache per device
    cudaError_t err = cudaFuncSetAttribute(panel_apply_kernel<KMAX, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(panel_doubles(KMAX) * sizeof(T)));
    if (err != cudaSuccess) return check_cuda(err);
    const size_t smem = panel_doubles(k) * sizeof(T);
    const unsigned grid = (unsigned)((ncols + kApplyThreads - 1) / kApplyThreads);
    ProfScope ps("panel_apply", stream);
    panel_apply_kernel<KMAX, T><<<grid, kApplyThreads, smem, stream>>>(Lr, ldl, Db, ncols, Vc, ldv, k, panel);
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


template <typename T>
gcm_status_t sweep_diag_t(T *Lb, int64_t ldl, int Db, T *Vb, int64_t ldv, int k, int sigma, int64_t grow0, T *panel,
                          unsigned long long *key, int64_t ebase, cudaStream_t stream) {
#define CALL(KM) diag_launch<KM, T>(Lb, ldl, Db, Vb, ldv, k, sigma, grow0, panel, key, ebase, stream)
    return GCM_KMAX_DISPATCH(k, CALL);
#undef CALL
}

template <typename T>
gcm_status_t sweep_apply_t(T *Lr, int64_t ldl, int Db, int64_t ncols, T *Vc, int64_t ldv, int k, const T *panel,
                           cudaStream_t stream) {
#define CALL(KM) apply_launch<KM, T>(Lr, ldl, Db, ncols, Vc, ldv, k, panel, stream)
    return GCM_KMAX_DISPATCH(k, CALL);
#undef CALL
}

template <typename T>
gcm_status_t modify_sweep_t(T *L, int64_t n, int64_t ldl, T *V, int64_t k, int sigma, unsigned long long *key,
                            T *panels, cudaStream_t stream) {
    const int64_t nb = (n + kD - 1) / kD;
    for (int64_t e0 = 0; e0 < k; e0 += kKMax) {
        const int kc = (int)std::min<int64_t>(kKMax, k - e0);
        T *Vc = V + e0 * n;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t r0 = b * kD;
            const int Db = (int)std::min<int64_t>(kD, n - r0);
            T *panel = panels + b * panel_doubles(kc);
            gcm_status_t st =
                sweep_diag_t<T>(L + r0 + r0 * ldl, ldl, Db, Vc + r0, n, kc, sigma, r0, panel, key, e0, stream);
            if (st != GCM_OK) return st;
            const int64_t c0 = r0 + kD;
            if (c0 < n) st = sweep_apply_t<T>(L + r0 + c0 * ldl, ldl, Db, n - c0, Vc + c0, n, kc, panel, stream);
            if (st != GCM_OK) return st;
        }
    }
    return GCM_OK;
}

}  // namespace

gcm_status_t sweep_diag(double *Lb, int64_t ldl, int Db, double *Vb, int64_t ldv, int k, int sigma, int64_t grow0,
                        double *panel, unsigned long long *key, int64_t ebase, cudaStream_t stream) {
    return sweep_diag_t<double>(Lb, ldl, Db, Vb, ldv, k, sigma, grow0, panel, key, ebase, stream);
}
gcm_status_t sweep_apply(double *Lr, int64_t ldl, int Db, int64_t ncols, double *Vc, int64_t ldv, int k,
                         const double *panel, cudaStream_t stream) {
    return sweep_apply_t<double>(Lr, ldl, Db, ncols, Vc, ldv, k, panel, stream);
}
gcm_status_t modify_sweep(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                          unsigned long long *key, double *panels, cudaStream_t stream) {
    return modify_sweep_t<double>(L, n, ldl, V, k, sigma, key, panels, stream);
}
gcm_status_t modify_sweep_f32(float *L, int64_t n, int64_t ldl, float *V, int64_t k, int sigma,
                              unsigned long long *key, float *panels, cudaStream_t stream) {
    return modify_sweep_t<float>(L, n, ldl, V, k, sigma, key, panels, stream);
}

}  // namespace gcm
