// la_scan.cuh -- decayed exclusive scan of sub-segment state summaries (la_scan.cu).
#pragma once
#include "la_common.cuh"

namespace la {
// fwd: in[0] = user (or 0);    in[g+1] = decayed in[g] + the summaries of segment g's sub-segments
// rev: in[last] = user (or 0); in[g-1] = the same, walking down
// Geometry (n, seg_len, nseg, sub_len, sub_per_seg, g_lo..g_hi, rev) comes from the summary pass's desc.
// seg_in / final_out nullable; seg_in is [bh][nseg][d][d], delta [bh][nseg * sub_per_seg][d][d]
// (double if acc_double, else float).
cudaError_t launch_segment_scan(bool acc_double, const void* delta, void* seg_in, const void* user_in, int user_T,
                                void* final_out, int final_T, const double* lam, int bh, int heads, int d,
                                const PassDesc& p, cudaStream_t st);
}  // namespace la
