// la_scan.cu -- combine sub-segment state summaries into each segment's entering state.
#include "la_ptx.cuh"
#include "la_scan.cuh"

namespace la {

namespace {

// Exclusive decayed scan along the sequence.  Summary slot (g, j) = sub-segment j of segment g, its rows
// [g seg_len + j sub_len, min(.. + sub_len, (g + 1) seg_len, n)); segments g_lo..g_hi were summarised.
//   fwd: in[0] = user (or 0);    walking g, j upwards:   s = lam^len(g,j) s + delta[g][j]
//   rev: in[last] = user (or 0); walking g, j downwards: same
// seg_in[g] = s on entering segment g.  `final_out` (nullable; needs every segment summarised) receives
// the inclusive total (F(n) / R(0)).  Sub-segments whose contribution a later factor lam^len == 0 discards
// exactly (sub_dead, la_common.cuh) are neither summarised nor read: they count as zero.
constexpr int kScanThreads = 128;
constexpr int kBatch = 8;  // sub-segment loads in flight per thread

template <typename Tacc, int V> struct alignas(16) VecA {
  Tacc x[V];
};

// One thread owns V consecutive state elements (one 16-byte vector): many small blocks, every load of a
// batch of sub-segments issued before the first is folded in (the scan is latency-bound, ~nsub loads deep).
template <typename Tacc, int V>
__global__ void __launch_bounds__(kScanThreads) segment_scan_kernel(
    const Tacc* __restrict__ delta, Tacc* __restrict__ seg_in, const void* user_in, int user_T,
    Tacc* final_out, int final_T, const double* lam, int heads, int d, int n, int seg_len, int nseg,
    int sub_len, int sub_per_seg, int g_lo, int g_hi, int rev) {
  using Vec = VecA<Tacc, V>;
  ptx::griddep_wait();    // PDL: the summaries of the previous kernel are complete and visible
  ptx::griddep_launch();  // tiny kernel: let the main pass start its prologue right away
  // lam^len of a sub-segment: len is sub_len, a segment's short last sub-segment, or the sequence's
  // short last one -- three pow()s per block instead of one per sub-segment
  __shared__ Tacc s_pow[3];
  __shared__ int s_len[3];
  __shared__ int s_last_full, s_last_seq, s_gl;  // last sub-segment index of a full segment / of the last one
  const int bh = blockIdx.y;
  const int nsub = nseg * sub_per_seg;
  auto sub_range = [&](int kk, int& p0, int& p1) {
    const int g = kk / sub_per_seg, j = kk % sub_per_seg;
    p0 = g * seg_len + j * sub_len;
    p1 = min(min(n, (g + 1) * seg_len), p0 + sub_len);
  };
  if (threadIdx.x < 3) {
    const int last_in_seg = (seg_len - 1) / sub_len;  // index of a full segment's last sub-segment
    int len = sub_len;
    if (threadIdx.x == 1) len = seg_len - last_in_seg * sub_len;
    if (threadIdx.x == 2) {
      int p0, p1;
      const int gl = (n - 1) / seg_len;
      sub_range(gl * sub_per_seg + ((n - 1 - gl * seg_len) / sub_len), p0, p1);
      len = p1 - p0;
    }
    s_len[threadIdx.x] = len;
    s_pow[threadIdx.x] = (Tacc)pow(load_decay(lam, bh % heads), (double)len);
    if (threadIdx.x == 0) {
      s_last_full = last_in_seg;
      s_gl = (n - 1) / seg_len;
      s_last_seq = (n - 1 - s_gl * seg_len) / sub_len;
    }
  }
  __syncthreads();
  const bool zero_full = s_pow[0] == (Tacc)0;
  // slot kk contributes nothing (never summarised) -- see sub_dead
  auto dead = [&](int kk) {
    const int g = kk / sub_per_seg, j = kk % sub_per_seg;
    const bool lastseg = g == s_gl;
    const int last = lastseg ? s_last_seq : s_last_full;
    const bool zero_last = (lastseg ? s_pow[2] : s_pow[1]) == (Tacc)0;
    return sub_dead(j, last, rev, zero_full, zero_last);
  };
  const int dd = d * d;
  const int e0 = (blockIdx.x * kScanThreads + threadIdx.x) * V;
  if (e0 >= dd) return;
  Tacc s[V];
#pragma unroll
  for (int q = 0; q < V; ++q) {
    s[q] = 0;
    if (user_in != nullptr) {
      const Tacc* u = reinterpret_cast<const Tacc*>(user_in) + (int64_t)bh * dd;
      const int e = e0 + q;
      s[q] = user_T ? u[(e % d) * d + e / d] : u[e];
    }
  }
  const Tacc* dcol = delta + (int64_t)bh * nsub * dd + e0;
  Tacc* scol = seg_in != nullptr ? seg_in + (int64_t)bh * nseg * dd + e0 : nullptr;
  for (int k0 = 0; k0 < nsub; k0 += kBatch) {
    Vec x[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int k = k0 + u;
      const int kk = rev ? nsub - 1 - k : k;
      const int g = kk / sub_per_seg;
      int p0, p1;
      sub_range(kk, p0, p1);
      if (k < nsub && g >= g_lo && g <= g_hi && p1 > p0 && !dead(kk))
        x[u] = *reinterpret_cast<const Vec*>(dcol + (int64_t)kk * dd);
      else
#pragma unroll
        for (int q = 0; q < V; ++q) x[u].x[q] = 0;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int k = k0 + u;
      if (k >= nsub) break;
      const int kk = rev ? nsub - 1 - k : k;
      const int g = kk / sub_per_seg, j = kk % sub_per_seg;
      // entering segment g: its first sub-segment in scan order
      if (scol != nullptr && j == (rev ? sub_per_seg - 1 : 0)) {
        Vec o;
#pragma unroll
        for (int q = 0; q < V; ++q) o.x[q] = s[q];
        *reinterpret_cast<Vec*>(scol + (int64_t)g * dd) = o;
      }
      int p0, p1;
      sub_range(kk, p0, p1);
      if (g < g_lo || g > g_hi || p1 <= p0) continue;  // not summarised / past the end
      const int len = p1 - p0;
      const Tacc dec = len == s_len[0] ? s_pow[0] : len == s_len[1] ? s_pow[1] : s_pow[2];
#pragma unroll
      for (int q = 0; q < V; ++q) s[q] = dec * s[q] + x[u].x[q];
    }
  }
  if (final_out != nullptr) {
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int e = e0 + q;
      final_out[(int64_t)bh * dd + (final_T ? (e % d) * d + e / d : e)] = s[q];
    }
  }
}

}  // namespace

cudaError_t launch_segment_scan(bool acc_double, const void* delta, void* seg_in, const void* user_in, int user_T,
                                void* final_out, int final_T, const double* lam, int bh, int heads, int d,
                                const PassDesc& p, cudaStream_t st) {
  const int dd = d * d;
  auto grid = [&](int v) { return dim3((unsigned)((dd / v + kScanThreads - 1) / kScanThreads), bh); };
#define LA_SCAN_ARGS(T)                                                                                          \
  reinterpret_cast<const T*>(delta), reinterpret_cast<T*>(seg_in), user_in, user_T, reinterpret_cast<T*>(final_out), \
      final_T, lam, heads, d, p.n, p.seg_len, p.nseg, p.sub_len, p.sub_per_seg, p.g_lo, p.g_hi, p.rev
  if (acc_double) {
    if (dd % 2 == 0) return launch_pdl(segment_scan_kernel<double, 2>, grid(2), dim3(kScanThreads), 0, st,
                                       LA_SCAN_ARGS(double));
    return launch_pdl(segment_scan_kernel<double, 1>, grid(1), dim3(kScanThreads), 0, st, LA_SCAN_ARGS(double));
  }
  if (dd % 4 == 0)
    return launch_pdl(segment_scan_kernel<float, 4>, grid(4), dim3(kScanThreads), 0, st, LA_SCAN_ARGS(float));
  return launch_pdl(segment_scan_kernel<float, 1>, grid(1), dim3(kScanThreads), 0, st, LA_SCAN_ARGS(float));
#undef LA_SCAN_ARGS
  return cudaGetLastError();
}

}  // namespace la
