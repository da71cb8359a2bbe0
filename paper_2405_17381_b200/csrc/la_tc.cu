// la_tc.cu -- placeholder until the tcgen05 kernel lands.
#include "la_tc.cuh"

namespace la {
bool tc_supported(int, int, const int64_t*) { return false; }
Plan tc_plan(int64_t bh, int64_t n, int, int64_t want) { return make_plan(bh, n, 128, want, kNumSMs, 4); }
size_t tc_workspace_bytes(int64_t, int, int) { return 0; }
cudaError_t tc_pass(const PassDesc&, void*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t tc_state(const PassDesc&, void*, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace la
