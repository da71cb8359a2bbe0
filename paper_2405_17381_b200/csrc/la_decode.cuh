// la_decode.cuh -- recurrent decode step (la_decode.cu).
#pragma once
#include "la_common.cuh"

namespace la {
// kv <- lam kv + k v^T; o = q . kv, for every (batch, head); q, k, v, o at base b*sb + h*sh
cudaError_t decode_launch(int dtype, int batch, int heads, int d, int64_t sb, int64_t sh, const void* q,
                          const void* k, const void* v, const double* lam, void* kv, void* o, cudaStream_t st);
}  // namespace la
