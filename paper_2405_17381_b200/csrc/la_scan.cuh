// la_scan.cuh -- decayed exclusive scan of per-segment state summaries (la_scan.cu).
#pragma once
#include "la_common.cuh"

namespace la {
// fwd: in[0] = user (or 0);    in[s+1] = lam^len(s) in[s] + delta[s]
// rev: in[last] = user (or 0); in[s-1] = lam^len(s) in[s] + delta[s]
// seg_in / final_out nullable; states are [bh][nseg][d][d] (double if acc_double, else float).
cudaError_t launch_segment_scan(bool acc_double, const void* delta, void* seg_in, const void* user_in, int user_T,
                                void* final_out, int final_T, const double* lam, int bh, int heads, int d, int n,
                                int seg_len, int nseg, int rev, cudaStream_t st);
}  // namespace la
