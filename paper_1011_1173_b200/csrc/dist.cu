// dist.cu -- multi-GPU column-sharded path. Not yet built.
#include "internal.h"
extern "C" {
gcm_status_t gcm_comm_unique_id(void *) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_init(gcm_comm_t *, const void *, int, int) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_destroy(gcm_comm_t) { return GCM_ENOTSUP; }
int64_t gcm_dist_local_cols(int64_t, int64_t, int, int) { return -1; }
gcm_status_t gcm_modify_dist(gcm_comm_t, double *, int64_t, int64_t, int64_t, double *, int64_t, int, gcm_info_t *,
                             gcm_stream_t) {
    return GCM_ENOTSUP;
}
}
