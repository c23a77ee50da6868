// batched.cu -- gcm_modify_batched. Not yet built.
#include "internal.h"
namespace gcm {
gcm_status_t modify_batched(double *, int64_t, int64_t, int64_t, double *, int64_t, int64_t, int, int64_t,
                            gcm_info_t *, cudaStream_t) {
    return GCM_ENOTSUP;
}
}  // namespace gcm
