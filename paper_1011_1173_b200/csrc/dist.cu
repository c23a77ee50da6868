// dist.cu -- column-sharded multi-GPU modification (BASELINE.json configs[3],
// SURVEY.md 8(e)), one process per GPU, NCCL over NVLink/NVSwitch.
//
// Layout: 1-D block-cyclic over columns with block width nb (a multiple of the
// 64-row panel height): global column block g = j / nb lives on rank g % P at
// local block g / P.  Each rank holds all n rows of its columns, so:
//   for every 64-row block b (rows r0 .. r0+63):
//     the owner of columns r0.. runs the diagonal Compute chain on its local copy
//       of the diagonal block (PAPER.md 44-49) -> coefficient panel b;
//     ncclBroadcast(panel b, root = owner)  -- the only exchange step, ~17 KB;
//     every rank applies panel b to its local columns right of the block
//       (PAPER.md 52-54), V rows of those columns live on the same rank.
// Failures: each rank records the first failing (e, row) of its own diagonal
// blocks; an all-reduce(min) of the 64-bit key gives every rank the global one.
#include <cstring>
#include <new>

#include "internal.h"

#ifdef GCM_WITH_NCCL
#include <nccl.h>
#endif

struct gcm_comm {
#ifdef GCM_WITH_NCCL
    ncclComm_t nc = nullptr;
#endif
    int rank = 0;
    int nranks = 1;
};

namespace gcm {
namespace {

int64_t local_cols(int64_t n, int64_t nb, int P, int r) {
    if (n <= 0 || nb <= 0 || P <= 0 || r < 0 || r >= P) return -1;
    const int64_t nblk = (n + nb - 1) / nb;
    int64_t cols = 0;
    for (int64_t g = r; g < nblk; g += P) cols += std::min<int64_t>(nb, n - g * nb);
    return cols;
}

// first local column of rank r whose global index is >= c
int64_t local_start(int64_t n, int64_t nb, int P, int r, int64_t c) {
    if (c >= n) return local_cols(n, nb, P, r);
    const int64_t g = c / nb;
    const int64_t lb_first = (g <= r) ? 0 : (g - r + P - 1) / P;  // first local block with global block >= g
    const int64_t gg = lb_first * P + r;
    if (gg == g) return lb_first * nb + (c - g * nb);
    return lb_first * nb;
}

}  // namespace
}  // namespace gcm

using namespace gcm;

extern "C" {

int64_t gcm_dist_local_cols(int64_t n, int64_t nb, int nranks, int rank) { return local_cols(n, nb, nranks, rank); }

int64_t gcm_dist_global_col(int64_t nb, int nranks, int rank, int64_t local_col) {
    if (nb <= 0 || nranks <= 0 || rank < 0 || rank >= nranks || local_col < 0) return -1;
    const int64_t lb = local_col / nb;
    return (lb * nranks + rank) * nb + local_col % nb;
}

#ifdef GCM_WITH_NCCL

static gcm_status_t check_nccl(ncclResult_t r) { return r == ncclSuccess ? GCM_OK : GCM_ENCCL; }

gcm_status_t gcm_comm_unique_id(void *host_id_out) {
    if (!host_id_out) return GCM_EINVAL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    ncclUniqueId id;
    gcm_status_t st = check_nccl(ncclGetUniqueId(&id));
    if (st == GCM_OK) std::memcpy(host_id_out, &id, sizeof(id));
    return st;
}

gcm_status_t gcm_comm_init(gcm_comm_t *comm, const void *host_id, int nranks, int rank) {
    if (!comm || !host_id || nranks <= 0 || rank < 0 || rank >= nranks) return GCM_EINVAL;
    gcm_comm *c = new (std::nothrow) gcm_comm;
    if (!c) return GCM_ENOMEM;
    ncclUniqueId id;
    std::memcpy(&id, host_id, sizeof(id));
    gcm_status_t st = check_nccl(ncclCommInitRank(&c->nc, nranks, id, rank));
    if (st != GCM_OK) {
        delete c;
        return st;
    }
    c->rank = rank;
    c->nranks = nranks;
    *comm = c;
    return GCM_OK;
}

gcm_status_t gcm_comm_destroy(gcm_comm_t comm) {
    if (!comm) return GCM_EINVAL;
    gcm_status_t st = check_nccl(ncclCommDestroy(comm->nc));
    delete comm;
    return st;
}

gcm_status_t gcm_modify_dist(gcm_comm_t comm, double *L_local, int64_t n, int64_t nb, int64_t ldl_local,
                             double *V_local, int64_t k, int sigma, gcm_info_t *d_info, gcm_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (!comm || n < 0 || k < 0 || nb <= 0 || nb % kD != 0 || (sigma != 1 && sigma != -1)) return GCM_EINVAL;
    if (ldl_local < std::max<int64_t>(1, n)) return GCM_EINVAL;
    const int P = comm->nranks, r = comm->rank;
    const int64_t nloc = local_cols(n, nb, P, r);
    if (n > 0 && k > 0 && nloc > 0 && (L_local == nullptr || V_local == nullptr)) return GCM_EINVAL;
    if (n == 0 || k == 0) {
        if (d_info) return check_cuda(cudaMemsetAsync(d_info, 0, sizeof(gcm_info_t), stream));
        return GCM_OK;
    }
    Workspace *ws = nullptr;
    gcm_status_t st = get_workspace(stream, (size_t)panel_doubles((int)std::min<int64_t>(k, kKMax)) * sizeof(double), 1,
                                    &ws);
    if (st != GCM_OK) return st;
    st = check_cuda(cudaMemsetAsync(ws->key, 0xff, sizeof(unsigned long long), stream));
    if (st != GCM_OK) return st;
    double *panel = ws->panels;
    const int64_t nblocks = (n + kD - 1) / kD;
    const int64_t ldv = std::max<int64_t>(nloc, 1);
    for (int64_t e0 = 0; e0 < k; e0 += kKMax) {
        const int kc = (int)std::min<int64_t>(kKMax, k - e0);
        double *Vc = V_local + e0 * ldv;
        for (int64_t b = 0; b < nblocks; ++b) {
            const int64_t r0 = b * kD;
            const int Db = (int)std::min<int64_t>(kD, n - r0);
            const int owner = (int)((r0 / nb) % P);
            if (owner == r) {
                const int64_t lc0 = local_start(n, nb, P, r, r0);
                st = sweep_diag(L_local + r0 + lc0 * ldl_local, ldl_local, Db, Vc + lc0, ldv, kc, sigma, r0, panel,
                                ws->key, e0, stream);
                if (st != GCM_OK) return st;
            }
            {
                ProfScope ps("bcast", stream);
                st = check_nccl(ncclBroadcast(panel, panel, (size_t)panel_doubles(kc), ncclDouble, owner, comm->nc,
                                              stream));
            }
            if (st != GCM_OK) return st;
            const int64_t ls = local_start(n, nb, P, r, r0 + kD);
            if (ls < nloc) {
                st = sweep_apply(L_local + r0 + ls * ldl_local, ldl_local, Db, nloc - ls, Vc + ls, ldv, kc, panel,
                                 stream);
                if (st != GCM_OK) return st;
            }
        }
    }
    // global first failure: min over ranks of the lexicographic key
    st = check_nccl(ncclAllReduce(ws->key, ws->key, 1, ncclUint64, ncclMin, comm->nc, stream));
    if (st != GCM_OK) return st;
    return finalize_info(ws->key, d_info, 1, stream);
}

#else  // built without NCCL

gcm_status_t gcm_comm_unique_id(void *) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_init(gcm_comm_t *, const void *, int, int) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_destroy(gcm_comm_t) { return GCM_ENOTSUP; }
gcm_status_t gcm_modify_dist(gcm_comm_t, double *, int64_t, int64_t, int64_t, double *, int64_t, int, gcm_info_t *,
                             gcm_stream_t) {
    return GCM_ENOTSUP;
}

#endif

}  // extern "C"
