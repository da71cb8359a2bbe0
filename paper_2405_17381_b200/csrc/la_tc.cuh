// la_tc.cuh -- host-side entry points of the TMA + tcgen05 backend (la_tc.cu).
#pragma once
#include <cuda.h>

#include "la_common.cuh"

namespace la {
// bf16, d = 128, and every stride of the `count` (batch, head, position) triples a multiple of 16 bytes
bool tc_supported(int dtype, int d, const int64_t* strides, int count);
bool tc_pointers_ok(const PassDesc& p);
const char* tc_detail();  // thread-local detail of the last host-side failure
// 4-D TMA descriptor (d, n, heads, batch) over a bf16 [.., .., .., 128] tensor with the desc's strides,
// box 64 x box_rows, 128-byte swizzle
bool tc_make_map(CUtensorMap* map, const void* base, const PassDesc& p, const Strides3& s, int box_rows = 128);
struct GlaPrologue;
// the segment-summary pass (la_summary.cu): p.delta_out, sub-segment geometry, g_lo..g_hi; with `gla`, B is
// the pre-activation kp and the pass summarises rot(act(kp)) (the GLA core's segmented forward)
cudaError_t tc_summary_launch(const PassDesc& p, cudaStream_t st, const GlaPrologue* gla = nullptr);
Plan tc_plan(int64_t bh, int64_t n, int d, int64_t want_segments, int sms);
// the fused reverse sweep of the backward: dK and dV in one pass over q, k, v, do (p.state_in = the
// entering adjoint state in dkv orientation; p.state_out = dkv_out, written by segment 0)
// s[6]: strides of q, k, v, do, dk, dv
struct GlaEpilogue;
cudaError_t tc_dkdv_launch(const PassDesc& p, const void* q, const void* k, const void* v, const void* dout,
                           void* dk, void* dv, const Strides3* s, cudaStream_t st, const GlaEpilogue* epi = nullptr);
// one launch of the main pass kernel (state_only = false) or of the per-segment summary kernel
cudaError_t tc_launch(const PassDesc& p, bool state_only, cudaStream_t st);
// GLA core forward (la_tc.cu GLA mode): the pass on (rot(act(a)), rot(act(b)), c) with the prologue
// applied in shared memory; q_out / k_out (nullable together) receive the transformed tiles (strides sa / sbb)
struct GlaPrologue {
  const double* theta;  // [d/2] or nullptr
  int act;
  int64_t offset;
  void* q_out;
  void* k_out;
};
cudaError_t tc_gla_fwd_launch(const PassDesc& p, const GlaPrologue& gla, cudaStream_t st);
// GLA core backward: the prologue's backward applied to a pass's output tile (dq -> dqp) or the dK/dV sweep's
// dK tile (dk -> dkp), with x the pre-activation rows (qp / kp: the output's geometry, strides sx)
struct GlaEpilogue {
  const void* xp;
  Strides3 sx;
  const double* theta;  // [d/2] or nullptr
  int act;
  int64_t offset;
};
cudaError_t tc_epi_launch(const PassDesc& p, const GlaEpilogue& epi, cudaStream_t st);
// the fp32 pass (la_tc32.cu): three-term bf16 split on tcgen05, d = 128, 16-byte strides
bool tc32_supported(int dtype, int d, const int64_t* strides, int count);
Plan tc32_plan(int64_t bh, int64_t n, int64_t want_segments, int sms);
cudaError_t tc32_launch(const PassDesc& p, bool state_only, cudaStream_t st);
}  // namespace la
