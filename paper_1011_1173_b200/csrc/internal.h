// internal.h -- shared host/device declarations of the gcm library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gcm.h"

namespace gcm {

// Row-block height D of the sweep: one diagonal chain block / one Apply panel
// covers D rows (the paper's fixed BlocksPerKernel x
// ThreadsPerBlock = 896, is Fermi-era prior art).
constexpr int kD = 64;
// Widest rank handled in one pass; larger k runs as ceil(k/kKMax) sequential
// passes over the same L (k sequential rank-1 sweeps, R3).
constexpr int kKMax = 64;

// Per-row-block coefficient panel (fp64, in global memory, L2-resident):
//   gd[(j*k + e)*2 + 0] = gamma_{j,e}   gd[(j*k + e)*2 + 1] = delta_{j,e}
//   rho[j]  at offset 2*D*k,  nu[e] at offset 2*D*k + D.
// gamma/delta/rho/nu are the rotation (c_{j,e}, s_{j,e}) of PAPER.md 44-49
// restated for the scaled 2-FMA Apply.
__host__ __device__ constexpr int64_t panel_doubles(int k) { return 2ll * kD * k + kD + k; }

// Failure key: atomicMin over ((e << 41) | (row << 1) | (code == 2 ? 0 : 1)),
// i.e. lexicographic (e, row) with code 2 first at equal (e, row).
__host__ __device__ inline unsigned long long info_key(int64_t e, int64_t row, int code) {
    return ((unsigned long long)e << 41) | ((unsigned long long)row << 1) | (code == 2 ? 0ull : 1ull);
}
constexpr unsigned long long kInfoNone = ~0ull;

struct Workspace {
    double *panels = nullptr;          // NB panels
    unsigned long long *key = nullptr; // failure key (batched: one per factor)
    void *extra = nullptr;             // algorithm-specific scratch
    size_t bytes = 0;
    unsigned epoch = 0;                // device-flag epoch of the last call (flags start zeroed)
};

// Returns a workspace of at least `bytes` bytes (+ key) for (current device, stream).
gcm_status_t get_workspace(cudaStream_t stream, size_t bytes, size_t nkeys, Workspace **ws);

gcm_status_t check_cuda(cudaError_t e);
// consume an error a previous failed call left behind (called at every ABI entry point)
void clear_stale_error();

// Profiling hook (gcm_profile_enable): bracket a launch with events on `stream`.
// Usage: { ProfScope ps("trsv", stream); kernel<<<..., stream>>>(...); }
extern bool g_profile_on;
// kernels this library launched while profiling is on (gcm_profile_launches)
void count_launch(int n = 1);
void prof_record(const char *name, cudaStream_t stream, bool begin);
struct ProfScope {
    const char *name;
    cudaStream_t stream;
    ProfScope(const char *n, cudaStream_t s) : name(n), stream(s) {
        if (g_profile_on) prof_record(name, stream, true);
    }
    ~ProfScope() {
        if (g_profile_on) prof_record(name, stream, false);
    }
};

// algorithms (enqueue only; arguments already validated, n > 0, k > 0)
// Sweep building blocks on arbitrary (local) column ranges, k <= kKMax:
//  sweep_diag : the Compute chain of one diagonal block (Db rows/columns); Lb -> element
//               (r0, first column), Vb -> V row of the first column (ld ldv); grow0 = r0
//               (global row index, for failure reports); writes the coefficient panel.
//  sweep_apply: that panel applied to ncols columns (Lr -> element (r0, first column)).
gcm_status_t sweep_diag(double *Lb, int64_t ldl, int Db, double *Vb, int64_t ldv, int k, int sigma, int64_t grow0,
                        double *panel, unsigned long long *key, int64_t ebase, cudaStream_t stream);
gcm_status_t sweep_apply(double *Lr, int64_t ldl, int Db, int64_t ncols, double *Vc, int64_t ldv, int k,
                         const double *panel, cudaStream_t stream);
gcm_status_t modify_sweep(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                          unsigned long long *key, double *panels, cudaStream_t stream);
gcm_status_t modify_sweep_f32(float *L, int64_t n, int64_t ldl, float *V, int64_t k, int sigma,
                              unsigned long long *key, float *panels, cudaStream_t stream);
gcm_status_t modify_blocked(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                            unsigned long long *key, Workspace *ws, cudaStream_t stream);
// Bytes of scratch one single-factor call needs (either algorithm), and the
// dispatcher that runs it on an already-sized workspace (no allocation).
size_t single_workspace_bytes(int64_t n, int64_t k, gcm_algo_t algo);
gcm_algo_t pick_algo(int64_t n, int64_t k, gcm_algo_t algo);
gcm_status_t run_single(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_algo_t algo,
                        unsigned long long *key, Workspace *ws, cudaStream_t stream);
size_t blocked_workspace_bytes(int64_t n, int64_t k);
gcm_status_t modify_batched(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V,
                            int64_t strideV, int64_t k, int sigma, int64_t batch,
                            gcm_info_t *d_info, cudaStream_t stream);
gcm_status_t modify_panel(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_info_t *d_info,
                          cudaStream_t stream);
gcm_status_t finalize_info(const unsigned long long *key, gcm_info_t *d_info, int64_t count,
                           cudaStream_t stream);

}  // namespace gcm
