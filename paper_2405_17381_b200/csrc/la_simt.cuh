// la_simt.cuh -- host-side entry points of the CUDA-core backend (la_simt.cu).
#pragma once
#include "la_common.cuh"

namespace la {
int simt_chunk(int dtype);
size_t simt_workspace_bytes(int dtype, int64_t bh, int nseg, int d);
cudaError_t simt_pass(int dtype, const PassDesc& p, void* ws, cudaStream_t st);
cudaError_t simt_state(int dtype, const PassDesc& p, void* ws, cudaStream_t st);
}  // namespace la
