// la_gla.cuh -- element-wise stages of the GLA layer around the attention core (la_gla.cu).
#pragma once
#include "la_common.cuh"

namespace la {
struct GlaRows {
  int64_t rows;    // batch * n
  int n;           // positions per sequence (LRPE position = row % n + offset)
  int width;       // heads * d
  int d;           // head dim (LRPE pairs within a head)
  int dtype;       // la_dtype
  int act;         // la_act
  int64_t offset;  // LRPE position of each sequence's first row
};
size_t gla_prologue_bwd_partial_bytes(const GlaRows& g);
cudaError_t gla_prologue(const GlaRows& g, const void* qp, const void* kp, const double* theta, void* q, void* k,
                         cudaStream_t st);
cudaError_t gla_prologue_bwd(const GlaRows& g, const void* qp, const void* kp, const double* theta, const void* dq,
                             const void* dk, void* dqp, void* dkp, void* partial, double* dtheta, cudaStream_t st);
cudaError_t gla_epilogue(const GlaRows& g, const void* a, const void* u, void* gated, void* rawnorm, double eps,
                         cudaStream_t st);
cudaError_t gla_epilogue_bwd(const GlaRows& g, const void* dgated, const void* a, const void* u, const void* rawnorm,
                             void* da, void* du, double eps, cudaStream_t st);
// tensor-parallel GLA: gated = a * u (u nullable) + per-row sum of squares of a at rowsq[row * stride]
cudaError_t gla_gate_rowsq(const GlaRows& g, const void* a, const void* u, void* gated, void* rowsq,
                           int64_t rowsq_stride, cudaStream_t st);
// y[r, :] = red[r, :out_w] sqrt(out_w) / max(sqrt(red[r, out_w]), eps); red / y in the accumulation type
cudaError_t gla_rowscale(bool acc_double, const void* red, void* y, int64_t rows, int out_w, double eps,
                         cudaStream_t st);
}  // namespace la
