// la_scan.cu -- combine per-segment state summaries into each segment's entering state.
#include "la_scan.cuh"

namespace la {

namespace {

// Exclusive decayed scan of the per-segment summaries along the sequence:
//   fwd: in[0] = user (or 0);   in[s+1] = lam^len(s) in[s] + delta[s]
//   rev: in[last] = user (or 0); in[s-1] = lam^len(s) in[s] + delta[s]
// `final_out` (nullable) receives the inclusive total (F(n) / R(0)).
template <typename Tacc>
__global__ void __launch_bounds__(256) segment_scan_kernel(
    const Tacc* __restrict__ delta, Tacc* __restrict__ seg_in, const void* user_in, int user_T,
    Tacc* final_out, int final_T, const double* lam, int heads, int d, int n, int seg_len, int nseg,
    int rev) {
  const int e = blockIdx.x * 256 + threadIdx.x;
  const int bh = blockIdx.y;
  if (e >= d * d) return;
  const int r = e / d, c = e % d;
  const double l = lam[bh % heads];
  Tacc s = 0;
  if (user_in != nullptr) {
    const Tacc* u = reinterpret_cast<const Tacc*>(user_in) + (int64_t)bh * d * d;
    s = user_T ? u[c * d + r] : u[e];
  }
  const Tacc full_decay = (Tacc)pow(l, (double)seg_len);                     // every segment but the last
  const Tacc last_decay = (Tacc)pow(l, (double)(n - (nseg - 1) * seg_len));  // the (possibly short) last one
  for (int k = 0; k < nseg; ++k) {
    const int sgi = rev ? (nseg - 1 - k) : k;
    const int64_t off = ((int64_t)bh * nseg + sgi) * d * d + e;
    if (seg_in != nullptr) seg_in[off] = s;
    s = (sgi == nseg - 1 ? last_decay : full_decay) * s + delta[off];
  }
  if (final_out != nullptr) final_out[(int64_t)bh * d * d + (final_T ? c * d + r : e)] = s;
}

}  // namespace

cudaError_t launch_segment_scan(bool acc_double, const void* delta, void* seg_in, const void* user_in, int user_T,
                                void* final_out, int final_T, const double* lam, int bh, int heads, int d, int n,
                                int seg_len, int nseg, int rev, cudaStream_t st) {
  dim3 grid((unsigned)((d * d + 255) / 256), bh);
  if (acc_double)
    segment_scan_kernel<double><<<grid, 256, 0, st>>>(reinterpret_cast<const double*>(delta),
                                                      reinterpret_cast<double*>(seg_in), user_in, user_T,
                                                      reinterpret_cast<double*>(final_out), final_T, lam, heads, d, n,
                                                      seg_len, nseg, rev);
  else
    segment_scan_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(delta),
                                                     reinterpret_cast<float*>(seg_in), user_in, user_T,
                                                     reinterpret_cast<float*>(final_out), final_T, lam, heads, d, n,
                                                     seg_len, nseg, rev);
  return cudaGetLastError();
}

}  // namespace la
