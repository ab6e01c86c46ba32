// tc.cu -- tcgen05 screening assign (placeholder until the TC path lands).
#include "common.cuh"

namespace ftk {
int tc_assign_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t,
                  int64_t, int32_t *, void *, cudaStream_t) {
    set_error("tc variant not built");
    return FTK_ERR_UNSUPPORTED;
}
}  // namespace ftk
