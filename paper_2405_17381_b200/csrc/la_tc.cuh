// la_tc.cuh -- host-side entry points of the TMA + tcgen05 backend (la_tc.cu).
#pragma once
#include "la_common.cuh"

namespace la {
bool tc_supported(int dtype, int d, const int64_t* strides);
bool tc_pointers_ok(const PassDesc& p);
const char* tc_detail();  // thread-local detail of the last host-side failure
Plan tc_plan(int64_t bh, int64_t n, int d, int64_t want_segments);
// one launch of the main pass kernel (state_only = false) or of the per-segment summary kernel
cudaError_t tc_launch(const PassDesc& p, bool state_only, cudaStream_t st);
}  // namespace la
