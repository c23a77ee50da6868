// blocked.cu -- GCM_ALGO_BLOCKED (chain-shortened single-factor path). Not yet built.
#include "internal.h"
namespace gcm {
size_t blocked_workspace_bytes(int64_t, int64_t) { return 0; }
gcm_status_t modify_blocked(double *, int64_t, int64_t, double *, int64_t, int, unsigned long long *, cudaStream_t) {
    return GCM_ENOTSUP;
}
}  // namespace gcm
