// oom.cu — out-of-memory mode (§5): workload-aware partition scheduling.
#include "internal.h"

namespace csaw {

csaw_status run_mdrw_oom(const csaw_graph* g, const csaw_bias& b, int32_t length, const uint32_t* d_seeds, int64_t n,
                         uint64_t base, uint64_t seed, uint32_t* d_path, cudaStream_t st) {
    (void)g; (void)b; (void)length; (void)d_seeds; (void)n; (void)base; (void)seed; (void)d_path; (void)st;
    return fail(CSAW_ERR_UNSUPPORTED, "OOM mode: not implemented yet");
}

}  // namespace csaw
