// la_simt.cuh -- host-side entry points of the CUDA-core backend (la_simt.cu).
#pragma once
#include "la_common.cuh"

namespace la {
int simt_chunk(int dtype);
// one launch of the main pass kernel (state_only = false) or of the per-segment summary kernel
cudaError_t simt_launch(int dtype, const PassDesc& p, bool state_only, cudaStream_t st);
}  // namespace la
