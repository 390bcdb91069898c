// cdist_tc.cu -- tcgen05 3xTF32 distance tile for large feature counts
// (BASELINE config 4, d = 1024).  Placeholder dispatch until the UMMA kernel
// lands: nothing is eligible, the FFMA tile in cdist.cu serves every shape.
#include "common.cuh"

namespace dndc {

bool cdist_tc_eligible(int64_t, int64_t, int64_t) { return false; }

void cdist_tile_tc_f32(dndc_ctx*, const float*, const float*, int64_t, const float*, const float*,
                       int64_t, int64_t, float*, int64_t, int64_t, int64_t, cudaStream_t) {
    throw Error(DNDC_EINTERNAL, "cdist_tc: tcgen05 path not built");
}

}  // namespace dndc
