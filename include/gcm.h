/*
 * gcm.h -- C ABI of the B200-native rank-k Cholesky up/down-date library
 * (arXiv 1011.1173, Walder 2010, "gpucholmodV0.2").
 *
 * The operation (Sec. 1): given an upper-triangular factor L
 * with A = L^T L and V in R^{n x k}, overwrite L with the upper-triangular
 * L~ (positive diagonal) such that
 *
 *        L~^T L~ = L^T L + sigma V V^T,      sigma = +1 (update) or -1 (downdate),
 *
 * computed with the hyperbolic/Givens row sweep of Algorithm 1
 * (CholeskyModifyA; Compute lines 44-49; Apply lines
 * 52-54) in O(k n^2) fp64 work, on the GPU, with no CPU fallback.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All matrices are IEEE fp64.  All pointers are DEVICE pointers unless an
 *    entry point says otherwise.  The library never synchronises the stream
 *    except in gcm_modify_host; work is enqueued on `stream` and the call
 *    returns.  The caller owns L, V and d_info and must not touch them until
 *    the stream work completes.
 *  - L: column-major, leading dimension ldl >= max(1, n).  Factor entry (i, j),
 *    i <= j, is L[i + j*ldl].  Only the upper triangle including the diagonal
 *    is read or written; the strictly lower part and rows n..ldl-1 are never
 *    touched.  (Storage is unstated in the paper; reading R7.)
 *  - V: column-major n x k with leading dimension n (update vector e is
 *    V[e*n .. e*n+n-1]).  V is overwritten: on exit V[i + e*n] holds the value
 *    Compute(i, e) consumed, i.e. update vector e rotated by all rows < i
 *    ("write the elements of V ... back"; R8).
 *  - Rank k is k sequential rank-1 modifications in column order e = 0..k-1
 *    (R3).
 *  - Synchronous errors (returned, nothing enqueued): GCM_EINVAL for n < 0,
 *    k < 0, ldl < max(1, n), sigma not in {+1, -1}, a NULL L or V with
 *    n*k > 0, batch < 0, or strides smaller than the footprint.  n == 0 or
 *    k == 0 is a successful no-op.  GCM_ECUDA reports a failed launch or
 *    allocation (cudaGetLastError is consumed), GCM_ENCCL a failed NCCL call.
 *  - Numerical failure is ASYNCHRONOUS, reported through d_info (like
 *    cuSOLVER's devInfo): code 1 = indefinite downdate, i.e. Compute found
 *    !(L_ii^2 + sigma V_i^2 > 0) (R5); code 2 =
 *    !(L_ii > 0) on entry to row i.  (col, row) is the lexicographically first
 *    failing (e, i) -- what k sequential rank-1 calls would report first
 *    (R6).  After a failure the contents of L and V are
 *    unspecified (NaN propagates) but the call always terminates.
 */
#ifndef GCM_H
#define GCM_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *gcm_stream_t; /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
    GCM_OK = 0,
    GCM_EINVAL = 1,
    GCM_ECUDA = 2,
    GCM_ENOMEM = 3,
    GCM_ENCCL = 4,
    GCM_ENOTSUP = 5 /* feature not compiled in (e.g. NCCL absent) */
} gcm_status_t;

typedef struct {
    int32_t code; /* 0 ok, 1 indefinite downdate, 2 non-positive pivot on entry */
    int32_t col;  /* update column e of the first failure (lexicographic (e, row)) */
    int64_t row;  /* row index i of the first failure */
} gcm_info_t;

/* Algorithm selector for gcm_modify_ex (all compute the same L~ and V_exit). */
typedef enum {
    GCM_ALGO_AUTO = 0,     /* library's choice for the shape          */
    GCM_ALGO_SWEEP = 1,    /* per-row-block launches: diagonal chain, then Apply panel */
    GCM_ALGO_BLOCKED = 2,  /* chain-shortened: block-parallel diagonal sweeps seeded by
                              P = L^{-T} V             */
    GCM_ALGO_PANEL = 3     /* the column-sharded algorithm of gcm_modify_dist on one GPU:
                              right-looking column blocks of 512, separate Apply
                              (large n)                   */
} gcm_algo_t;

/* In-place rank-k modification L~^T L~ = L^T L + sigma V V^T.
 * L: device, n x n upper (column-major, ldl).  V: device, n x k (ld n), overwritten
 * with V_exit.  sigma: +1 update, -1 downdate.  Numerical failures are not
 * reported (use gcm_modify_info).  Enqueued on `stream`. */
gcm_status_t gcm_modify(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                        gcm_stream_t stream);

/* As gcm_modify, plus the asynchronous failure report.  d_info: device pointer
 * to ONE gcm_info_t, or NULL; it is fully written by the call (code 0 on success). */
gcm_status_t gcm_modify_info(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                             gcm_info_t *d_info, gcm_stream_t stream);

/* As gcm_modify_info with an explicit algorithm. */
gcm_status_t gcm_modify_ex(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                           gcm_info_t *d_info, gcm_algo_t algo, gcm_stream_t stream);

/* Single precision: as gcm_modify_info with L, V in fp32 (float, same layouts).  The paper's
 * experiments ran both precisions (PAPER.md 111, Figs. 2-3); this is the paper's panel-order
 * sweep (diagonal Compute chain kernel, then the panel Apply kernel, per 64-row block)
 * instantiated for float.  Failure semantics as in fp64 (the tests are in fp32). */
gcm_status_t gcm_modify_f32(float *L, int64_t n, int64_t ldl, float *V, int64_t k, int sigma,
                            gcm_info_t *d_info, gcm_stream_t stream);

/* End-to-end convenience: L_host (n x n, ldl) and V_host (n x k) are HOST
 * pointers (pinned memory gives full PCIe bandwidth); the call copies the upper
 * triangle's columns and V to the device, runs gcm_modify_info on an internal
 * stream, copies L and V back, synchronises, and writes *h_info (host pointer,
 * nullable).  Device buffers are cached per device between calls. */
gcm_status_t gcm_modify_host(double *L_host, int64_t n, int64_t ldl, double *V_host, int64_t k,
                             int sigma, gcm_info_t *h_info);

/* Bytes gcm_modify_host moves in EACH direction for (n, k): the upper triangle
 * as column blocks of 256 columns (block [j0, j1) carries rows 0..j1-1, so a
 * little of the strictly lower part near the diagonal rides along and is
 * written back unchanged) plus V.  Host-only, no CUDA call; -1 if n or k < 0. */
int64_t gcm_modify_host_bytes(int64_t n, int64_t k);

/* Batched variant: `batch` independent factors of the same n, k, sigma.
 * Factor b is L + b*strideL (n x n, ldl) and V + b*strideV (n x k, ld n).
 * strideL >= ldl*n, strideV >= n*k (the footprints must not overlap).
 * d_info: device array of `batch` gcm_info_t, or NULL.  One CTA runs each
 * factor (its diagonal chain and its Apply panels) -- DESIGN.md "batched". */
gcm_status_t gcm_modify_batched(double *L, int64_t n, int64_t ldl, int64_t strideL, double *V,
                                int64_t strideV, int64_t k, int sigma, int64_t batch,
                                gcm_info_t *d_info, gcm_stream_t stream);

/* ---- multi-GPU, one process per GPU (column-block sharding) ----
 * The NCCL unique id is exchanged by the caller (e.g. torch.distributed).
 * Layout: 1-D block-cyclic over columns with block width nb: global column
 * block g = j / nb lives on rank g % nranks at local column block g / nranks.
 * L_local is n x n_local column-major (ldl_local >= n), n_local = the number
 * of columns this rank owns; V_local holds the V rows of those columns
 * (n_local x k, ld n_local), overwritten with their V_exit rows.  Every rank
 * calls gcm_modify_dist with identical (n, nb, k, sigma); it is collective.
 * nb must be a positive multiple of 64 (a multiple of 256 lets the Apply use
 * 256-column TMA tiles), nranks <= 8, n < 2^31, else GCM_EINVAL.
 * Algorithm (PAPER.md 24-30/44-54 restated as in
 * GCM_ALGO_BLOCKED): per column block the owner solves its rows of P = L^{-T} V,
 * which reach every rank (ncclBroadcast here; device-initiated stores in the
 * virtual-rank entry below), every rank updates its own residuals; then each
 * rank sweeps its own diagonal blocks, the coefficient panels reach every rank,
 * and every rank applies them to its own tiles.  d_info (device, nullable)
 * receives the global first failure on every rank.  Built without NCCL:
 * GCM_ENOTSUP. */
typedef struct gcm_comm *gcm_comm_t;
gcm_status_t gcm_comm_unique_id(void *host_id_out /* 128 bytes */);
gcm_status_t gcm_comm_init(gcm_comm_t *comm, const void *host_id, int nranks, int rank);
gcm_status_t gcm_comm_destroy(gcm_comm_t comm);
/* on != 0: later gcm_modify_dist calls on this communicator exchange P rows and coefficient
 * panels by DEVICE-INITIATED stores into the other ranks' memory (CUDA IPC windows mapped at
 * the first call, NVLink peer stores, system-scope release flags / counters that the
 * consumers' kernels acquire) instead of ncclBroadcast; NCCL is then used only to exchange
 * the IPC handles, for one barrier per pass and the final failure all-reduce.  Collective:
 * every rank sets the same mode.  (Verified on one GPU with one rank.) */
gcm_status_t gcm_comm_set_peer(gcm_comm_t comm, int on);
/* Number of columns rank `rank` owns (block-cyclic, width nb), or -1 on bad arguments. Host only. */
int64_t gcm_dist_local_cols(int64_t n, int64_t nb, int nranks, int rank);
/* Global column index of local column `local_col` of rank `rank`, or -1. Host only. */
int64_t gcm_dist_global_col(int64_t nb, int nranks, int rank, int64_t local_col);
gcm_status_t gcm_modify_dist(gcm_comm_t comm, double *L_local, int64_t n, int64_t nb,
                             int64_t ldl_local, double *V_local, int64_t k, int sigma,
                             gcm_info_t *d_info, gcm_stream_t stream);
/* Host only (no CUDA call): the work rank `rank` does in gcm_modify_dist.  what = 0:
 * its Apply tiles as (row block b, global 64-column strip s) pairs, 2 entries each;
 * what = 1: its 64-row diagonal blocks b; what = 2: the column blocks g whose rows of P
 * it solves.  Writes min(count, cap) entries of out and returns count (-1 on bad
 * arguments).  The union over ranks covers every tile (b < s), diagonal block and
 * column block exactly once (tests/test_dist_host.py). */
int64_t gcm_dist_plan(int64_t n, int64_t nb, int nranks, int rank, int what, int64_t *out, int64_t cap);

/* Virtual ranks: the same column-sharded algorithm for `nranks` ranks whose shards all
 * live on the CURRENT device, run by one call on one stream (the ranks' kernels are
 * ordered by the stream, never waiting on each other).  L_local[r], ldl_local[r],
 * V_local[r] are HOST arrays of nranks entries holding rank r's device pointers and
 * leading dimension, laid out as for gcm_modify_dist.  The owner of each column block
 * writes its P rows, and each rank its coefficient panels, straight into every other
 * rank's buffers (device-initiated stores: the multi-GPU exchange with peer pointers).
 * nranks in 1..8.  d_info: one gcm_info_t (device, nullable), the global first failure. */
gcm_status_t gcm_modify_dist_virtual(int nranks, double *const *L_local, int64_t n, int64_t nb,
                                     const int64_t *ldl_local, double *const *V_local, int64_t k,
                                     int sigma, gcm_info_t *d_info, gcm_stream_t stream);

/* ---- measurement hooks (used by bench.py; off by default, no cost when off) ----
 * When enabled, every kernel launch of the library on any stream is bracketed by
 * a pair of CUDA events recorded on that stream.  gcm_profile_read synchronises
 * the recorded events and returns, per kernel family (e.g. "trsv", "bapply"),
 * the number of launches and the summed event time in milliseconds, then clears
 * the record.  names: caller buffer of max_entries * 32 chars (NUL-terminated
 * strings, 32 bytes each); counts/ms: arrays of max_entries.  Returns the number
 * of entries written (or -1 on a CUDA error). */
gcm_status_t gcm_profile_enable(int on);
int gcm_profile_read(char *names, int64_t *counts, double *ms, int max_entries);
/* Number of kernels the library launched (all streams) while profiling was enabled, since the
 * last call; resets the count. */
int64_t gcm_profile_launches(void);

/* Human-readable status. */
const char *gcm_status_string(gcm_status_t s);

/* Frees every cached per-(device, stream) workspace.  Must not race with
 * in-flight calls. */
gcm_status_t gcm_release_workspace(void);

/* Library version string (e.g. "gcm 0.1 sm_100a"). */
const char *gcm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GCM_H */
