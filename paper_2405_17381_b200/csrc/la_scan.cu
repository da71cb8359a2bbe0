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
constexpr int kScanThreads = 256;
constexpr int kScanElems = 8;  // state elements per thread (consecutive)

template <typename Tacc>
__global__ void __launch_bounds__(kScanThreads) segment_scan_kernel(
    const Tacc* __restrict__ delta, Tacc* __restrict__ seg_in, const void* user_in, int user_T,
    Tacc* final_out, int final_T, const double* lam, int heads, int d, int n, int seg_len, int nseg,
    int sub_len, int sub_per_seg, int g_lo, int g_hi, int rev) {
  extern __shared__ unsigned char scan_smem[];
  Tacc* s_dec = reinterpret_cast<Tacc*>(scan_smem);  // lam^len of every sub-segment, once per block
  const int bh = blockIdx.y;
  const int nsub = nseg * sub_per_seg;
  {
    const double l = lam[bh % heads];
    for (int kk = threadIdx.x; kk < nsub; kk += blockDim.x) {
      const int g = kk / sub_per_seg, j = kk % sub_per_seg;
      const int p0 = g * seg_len + j * sub_len;
      const int p1 = min(min(n, (g + 1) * seg_len), p0 + sub_len);
      s_dec[kk] = p1 > p0 ? (Tacc)pow(l, (double)(p1 - p0)) : (Tacc)1;
    }
    __syncthreads();
  }
  // a thread owns kScanElems consecutive state elements: few, fat blocks (the scan is latency-bound)
  const int e0 = (blockIdx.x * kScanThreads + threadIdx.x) * kScanElems;
  const int dd = d * d;
  if (e0 >= dd) return;
  const int ne = min(kScanElems, dd - e0);
  Tacc s[kScanElems];
#pragma unroll
  for (int q = 0; q < kScanElems; ++q) {
    s[q] = 0;
    const int e = e0 + q;
    if (user_in != nullptr && q < ne) {
      const Tacc* u = reinterpret_cast<const Tacc*>(user_in) + (int64_t)bh * dd;
      s[q] = user_T ? u[(e % d) * d + e / d] : u[e];
    }
  }
  const Tacc* dcol = delta + (int64_t)bh * nsub * dd + e0;
  Tacc* scol = seg_in != nullptr ? seg_in + (int64_t)bh * nseg * dd + e0 : nullptr;
  // Walk the sub-segments in scan order (k -> segment g, sub-segment j); their loads are independent:
  // issue a batch, then fold it in order.
  constexpr int kBatch = 4;
  for (int k0 = 0; k0 < nsub; k0 += kBatch) {
    Tacc x[kBatch][kScanElems];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int k = k0 + u;
      const int kk = rev ? nsub - 1 - k : k;
      const int g = kk / sub_per_seg, j = kk % sub_per_seg;
      const bool live = k < nsub && g >= g_lo && g <= g_hi && g * seg_len + j * sub_len < min(n, (g + 1) * seg_len);
#pragma unroll
      for (int q = 0; q < kScanElems; ++q) x[u][q] = (live && q < ne) ? dcol[(int64_t)kk * dd + q] : (Tacc)0;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int k = k0 + u;
      if (k >= nsub) break;
      const int kk = rev ? nsub - 1 - k : k;
      const int g = kk / sub_per_seg, j = kk % sub_per_seg;
      // entering segment g: its first sub-segment in scan order
      if (scol != nullptr && j == (rev ? sub_per_seg - 1 : 0)) {
#pragma unroll
        for (int q = 0; q < kScanElems; ++q)
          if (q < ne) scol[(int64_t)g * dd + q] = s[q];
      }
      if (g < g_lo || g > g_hi) continue;
      const int p0 = g * seg_len + j * sub_len;
      if (p0 >= min(min(n, (g + 1) * seg_len), p0 + sub_len)) continue;  // past the end: never written
      const Tacc dec = s_dec[kk];
#pragma unroll
      for (int q = 0; q < kScanElems; ++q) s[q] = dec * s[q] + x[u][q];
    }
  }
  if (final_out != nullptr) {
#pragma unroll
    for (int q = 0; q < kScanElems; ++q) {
      const int e = e0 + q;
      if (q < ne) final_out[(int64_t)bh * dd + (final_T ? (e % d) * d + e / d : e)] = s[q];
    }
  }
}

}  // namespace

cudaError_t launch_segment_scan(bool acc_double, const void* delta, void* seg_in, const void* user_in, int user_T,
                                void* final_out, int final_T, const double* lam, int bh, int heads, int d,
                                const PassDesc& p, cudaStream_t st) {
  dim3 grid((unsigned)((d * d + kScanThreads * kScanElems - 1) / (kScanThreads * kScanElems)), bh);
  const size_t smem = (size_t)p.nseg * p.sub_per_seg * (acc_double ? sizeof(double) : sizeof(float));
  if (acc_double)
    segment_scan_kernel<double><<<grid, kScanThreads, smem, st>>>(
        reinterpret_cast<const double*>(delta), reinterpret_cast<double*>(seg_in), user_in, user_T,
        reinterpret_cast<double*>(final_out), final_T, lam, heads, d, p.n, p.seg_len, p.nseg, p.sub_len,
        p.sub_per_seg, p.g_lo, p.g_hi, p.rev);
  else
    segment_scan_kernel<float><<<grid, kScanThreads, smem, st>>>(
        reinterpret_cast<const float*>(delta), reinterpret_cast<float*>(seg_in), user_in, user_T,
        reinterpret_cast<float*>(final_out), final_T, lam, heads, d, p.n, p.seg_len, p.nseg, p.sub_len,
        p.sub_per_seg, p.g_lo, p.g_hi, p.rev);
  return cudaGetLastError();
}

}  // namespace la
