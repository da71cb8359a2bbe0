// la_scan.cu -- combine sub-segment state summaries into each segment's entering state.
#include "la_scan.cuh"

namespace la {

namespace {

// Exclusive decayed scan along the sequence.  Summary slot (g, j) = sub-segment j of segment g, its rows
// [g seg_len + j sub_len, min(.. + sub_len, (g + 1) seg_len, n)); segments g_lo..g_hi were summarised.
//   fwd: in[0] = user (or 0);    walking g, j upwards:   s = lam^len(g,j) s + delta[g][j]
//   rev: in[last] = user (or 0); walking g, j downwards: same
// seg_in[g] = s on entering segment g.  `final_out` (nullable; needs every segment summarised) receives
// the inclusive total (F(n) / R(0)).
template <typename Tacc>
__global__ void __launch_bounds__(256) segment_scan_kernel(
    const Tacc* __restrict__ delta, Tacc* __restrict__ seg_in, const void* user_in, int user_T,
    Tacc* final_out, int final_T, const double* lam, int heads, int d, int n, int seg_len, int nseg,
    int sub_len, int sub_per_seg, int g_lo, int g_hi, int rev) {
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
  const Tacc full_decay = (Tacc)pow(l, (double)sub_len);
  const int nsub = nseg * sub_per_seg;
  for (int k = 0; k < nseg; ++k) {
    const int g = rev ? (nseg - 1 - k) : k;
    if (seg_in != nullptr) seg_in[((int64_t)bh * nseg + g) * d * d + e] = s;
    if (g < g_lo || g > g_hi) continue;
    const int seg_end = min(n, (g + 1) * seg_len);
    for (int m = 0; m < sub_per_seg; ++m) {
      const int j = rev ? (sub_per_seg - 1 - m) : m;
      const int p0 = g * seg_len + j * sub_len;
      const int p1 = min(seg_end, p0 + sub_len);
      if (p0 >= p1) continue;  // past the end of the sequence: empty, never written
      const Tacc dec = (p1 - p0 == sub_len) ? full_decay : (Tacc)pow(l, (double)(p1 - p0));
      s = dec * s + delta[((int64_t)bh * nsub + g * sub_per_seg + j) * d * d + e];
    }
  }
  if (final_out != nullptr) final_out[(int64_t)bh * d * d + (final_T ? c * d + r : e)] = s;
}

}  // namespace

cudaError_t launch_segment_scan(bool acc_double, const void* delta, void* seg_in, const void* user_in, int user_T,
                                void* final_out, int final_T, const double* lam, int bh, int heads, int d,
                                const PassDesc& p, cudaStream_t st) {
  dim3 grid((unsigned)((d * d + 255) / 256), bh);
  if (acc_double)
    segment_scan_kernel<double><<<grid, 256, 0, st>>>(
        reinterpret_cast<const double*>(delta), reinterpret_cast<double*>(seg_in), user_in, user_T,
        reinterpret_cast<double*>(final_out), final_T, lam, heads, d, p.n, p.seg_len, p.nseg, p.sub_len,
        p.sub_per_seg, p.g_lo, p.g_hi, p.rev);
  else
    segment_scan_kernel<float><<<grid, 256, 0, st>>>(
        reinterpret_cast<const float*>(delta), reinterpret_cast<float*>(seg_in), user_in, user_T,
        reinterpret_cast<float*>(final_out), final_T, lam, heads, d, p.n, p.seg_len, p.nseg, p.sub_len,
        p.sub_per_seg, p.g_lo, p.g_hi, p.rev);
  return cudaGetLastError();
}

}  // namespace la
