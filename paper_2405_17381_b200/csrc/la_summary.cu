// la_summary.cu -- the segment-summary pass on tcgen05: a lean kernel for the long-sequence path.
//
// For a sub-segment [p0, p1) of one (batch, head) it computes the local carried state (la_common.cuh)
//   fwd: sum_s lam^(p1-1-s) b[s] c[s]^T        rev: sum_s lam^(s-p0+1) b[s] c[s]^T
// with each row's decay to the sub-segment's far edge folded into B~ = w * B, so chunks accumulate
// straight into one fp32 TMEM state: per chunk one SS-MMA state += B~^T C (M = N = d = 128, K = 64
// rows) -- no per-chunk state round trip.
//
// The summary reads two rows per position and does one MMA per chunk, so what bounds it is how many
// bytes each SM keeps in flight.  Hence 64-row chunks (16 KB tiles), a 3-deep {B, C} ring (96 KB of
// SMEM) and 128 TMEM columns per CTA: two CTAs share an SM, and a launch of ~2 x 148 sub-segments
// keeps the whole GPU streaming (the main-pass kernel's 224 KB / 512-column footprint allowed one).
//
// Warps: 0 TMA producer (one lane), 1 MMA issuer (+ TMEM owner), 2-5 B scaling (in place, swizzle-
// order, conflict-free) and, at the end, the TMEM -> global export (one warp per TMEM lane quadrant).
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <type_traits>

#include "la_common.cuh"
#include "la_ptx.cuh"
#include "la_tc.cuh"

namespace la {

namespace {

using namespace ptx;

constexpr int SC = 64;                // chunk rows
constexpr int SD = 128;               // head dim
constexpr int STILE = SC * SD * 2;    // 16 KB bf16 tile
constexpr int SHALF = STILE / 2;      // [64 rows][64 cols] = 8 KB, one 128B-swizzle column block
constexpr int SNST = 3;               // ring depth
constexpr int S_WARPS = 6, S_THREADS = S_WARPS * 32;
constexpr uint32_t S_TM_COLS = 128;
constexpr size_t S_SMEM_BYTES = (size_t)SNST * 2 * STILE + 1024;
constexpr uint32_t S_IDESC = idesc_bf16(128, 128, 1, 1);  // A (B~^T) and B (C) both MN-major

struct SumBars {
  uint64_t full[SNST], empty[SNST], scaled[SNST];
  uint64_t done;
  uint32_t tmem_base;
};

struct SumArgs {
  int heads, n, seg_len, nseg, rev;
  int sub_len, sub_per_seg, g_lo;
  int d;  // head dim (64 or 128): features past d are zero (TMA out-of-bounds fill); deltas are d x d
  const double* lam;
  float* delta_out;  // [bh][nseg * sub_per_seg][d][d]
  // GLA mode: B is the pre-activation kp; the B warps apply rot(act(.)) before the decay weight
  const double* theta;  // [d/2] or nullptr
  int act;
  int64_t offset;
};

template <bool GLA>
__global__ void __launch_bounds__(S_THREADS, 2)
    tc_summary_kernel(const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_c,
                      const SumArgs args) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ SumBars bars;
  __shared__ float2 anchor_s[GLA ? SD / 2 : 1];  // GLA: (cos, sin) of theta_j (chunk row 0 + offset)
  const uint32_t smem = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem - smem_u32(smem_raw));
  auto tile_b = [smem](int s) { return smem + (uint32_t)(s * 2 * STILE); };
  auto tile_c = [smem](int s) { return smem + (uint32_t)(s * 2 * STILE + STILE); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int bi = bh / args.heads, hi = bh % args.heads;
  const int g = args.g_lo + (int)blockIdx.x / args.sub_per_seg, j = (int)blockIdx.x % args.sub_per_seg;
  const int slot = g * args.sub_per_seg + j;
  const int p0 = g * args.seg_len + j * args.sub_len;
  const int p1 = min(min(args.n, (g + 1) * args.seg_len), p0 + args.sub_len);
  const int nchunks_all = p1 > p0 ? (p1 - p0 + SC - 1) / SC : 0;
  const int rev = args.rev;
  if (nchunks_all == 0) return;  // uniform across the CTA: an empty sub-segment (past n) writes nothing
  // Work whose contribution is exactly zero is skipped (the same arithmetic result, uniform across the CTA):
  // a sub-segment that a later factor lam^len == 0 discards in the scan (sub_dead: its slot is never read),
  // and, in a live one, the chunks whose largest weight rounds to zero in bf16 (their B~ rows are all zero).
  // Short-memory heads thereby summarise ~one chunk per segment instead of the whole segment.
  griddep_wait();  // PDL: the previous kernel of the stream has completed (inputs written, outputs free)
  const double lamv = load_decay(args.lam, hi);
  int t_beg = 0, t_end = nchunks_all;
  {
    const int seg_end = min(args.n, (g + 1) * args.seg_len);
    const int last = (seg_end - 1 - g * args.seg_len) / args.sub_len;
    const int last_len = seg_end - (g * args.seg_len + last * args.sub_len);
    const bool zero_full = (float)pow(lamv, (double)args.sub_len) == 0.f;
    const bool zero_last = (float)pow(lamv, (double)last_len) == 0.f;
    if (sub_dead(j, last, rev, zero_full, zero_last)) return;
    // largest weight of chunk t: fwd at its last row, lam^(p1 - min(p1, r0 + SC)); rev at its first, lam^(r0 - p0 + 1)
    auto live = [&](int t) {
      const int r0 = p0 + t * SC;
      const int e = rev ? r0 - p0 + 1 : p1 - min(p1, r0 + SC);
      return (__bfloat16_as_ushort(__float2bfloat16_rn((float)pow(lamv, (double)e))) & 0x7fff) != 0;
    };
    // live(t) is monotone in t (rising for fwd, falling for rev): bisect the boundary
    if (!rev) {
      int lo = 0, hi2 = nchunks_all - 1;  // the last chunk is always live (weight 1 at the edge)
      while (lo < hi2) {
        const int mid = (lo + hi2) >> 1;
        if (live(mid)) hi2 = mid; else lo = mid + 1;
      }
      t_beg = lo;
    } else {
      int lo = 0, hi2 = nchunks_all - 1;  // chunk 0 is always live
      while (lo < hi2) {
        const int mid = (lo + hi2 + 1) >> 1;
        if (live(mid)) lo = mid; else hi2 = mid - 1;
      }
      t_end = lo + 1;
    }
  }
  const int nchunks = t_end - t_beg;          // the chunks walked: t_beg .. t_end - 1
  const int q0 = p0 + t_beg * SC;             // first row walked

  if (threadIdx.x == 0) {
    for (int s = 0; s < SNST; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], 1);
      mbar_init(&bars.scaled[s], 4);
    }
    mbar_init(&bars.done, 1);
    fence_mbar_init();
  }
  const int early = nchunks < SNST ? nchunks : SNST;  // ring stages loaded before the CTA-wide sync
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_b);
    tma_prefetch(&map_c);
    for (int t = 0; t < early; ++t) {  // no empty-slot wait for the first stages
      const int r0 = q0 + t * SC;
      mbar_arrive_expect_tx(&bars.full[t], 2 * STILE);
      uint8_t* gb = smem_gen + (size_t)t * 2 * STILE;
      tma_load_4d(&map_b, &bars.full[t], gb, 0, r0, hi, bi);
      tma_load_4d(&map_b, &bars.full[t], gb + SHALF, 64, r0, hi, bi);
      tma_load_4d(&map_c, &bars.full[t], gb + STILE, 0, r0, hi, bi);
      tma_load_4d(&map_c, &bars.full[t], gb + STILE + SHALF, 64, r0, hi, bi);
    }
  }
  if (warp == 1) tmem_alloc(&bars.tmem_base, S_TM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int t = early; t < nchunks; ++t) {
        const int s = t % SNST;
        if (t >= SNST) mbar_wait(&bars.empty[s], ((t / SNST) - 1) & 1);
        const int r0 = q0 + t * SC;
        mbar_arrive_expect_tx(&bars.full[s], 2 * STILE);
        uint8_t* gb = smem_gen + (size_t)s * 2 * STILE;
        tma_load_4d(&map_b, &bars.full[s], gb, 0, r0, hi, bi);
        tma_load_4d(&map_b, &bars.full[s], gb + SHALF, 64, r0, hi, bi);
        tma_load_4d(&map_c, &bars.full[s], gb + STILE, 0, r0, hi, bi);
        tma_load_4d(&map_c, &bars.full[s], gb + STILE + SHALF, 64, r0, hi, bi);
      }
      griddep_launch();  // every load of this CTA issued: the next kernel may start its prologue
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % SNST;
        mbar_wait(&bars.scaled[s], (t / SNST) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < SC / 16; ++kk)
          mma_bf16_ss(tmem, smem_desc_sw128(tile_b(s) + kk * 2048, SHALF, 1024),
                      smem_desc_sw128(tile_c(s) + kk * 2048, SHALF, 1024), S_IDESC, t > 0 || kk > 0);
        mma_commit(&bars.empty[s]);
      }
      mma_commit(&bars.done);
      // the last commits must land before the CTA retires (their barriers die with its SMEM)
      for (int t = max(0, nchunks - SNST); t < nchunks; ++t) mbar_wait(&bars.empty[t % SNST], (t / SNST) & 1);
      mbar_wait(&bars.done, 0);
    }
  } else {
    // warps 2..5: B~ = w * B in place; thread -> (row, 64-column half)
    const int tid = threadIdx.x - 64;     // 0..127
    const int i = tid & (SC - 1);         // chunk row
    const int hh = tid >> 6;              // column half
    const double lam = lamv;
    for (int t = 0; t < nchunks; ++t) {
      const int s = t % SNST;
      const int r0 = q0 + t * SC;
      const int b = min(SC, p1 - r0);
      mbar_wait(&bars.full[s], (t / SNST) & 1);
      // fwd lam^(p1-1-s), rev lam^(s-p0+1); rows past the sub-segment (tail) contribute nothing
      const int row = r0 + i;
      float w = i < b ? (float)(pow(lam, (double)(rev ? row - p0 + 1 : p1 - 1 - row)) * (lam / lam)) : 0.f;
#ifdef LA_MUTATE_DKV
      if (rev) w = -w;  // fault injection: the reference's `_dkv_step` sign flip (test_kernels.py:249-268)
#endif
      const uint32_t w2 = pack_bf16x2(w, w);
      const uint32_t base = tile_b(s) + hh * SHALF + i * 128;
      if (GLA) {
        // k = rot(act(kp)) first (as la_tc.cu's GLA mode), then the decay weight
        const bool rot = args.theta != nullptr;
        if (rot) {
          named_bar_sync(1, 128);  // the previous chunk's anchors are no longer read
          if (tid < SD / 2) {
            float c0, s0;
            lrpe_cs(args.theta[tid], (int64_t)r0 + args.offset, &c0, &s0);
            anchor_s[tid] = make_float2(c0, s0);
          }
          named_bar_sync(1, 128);
        }
        const bool valid = row < args.n;
        auto tile = [&](auto act_tag) {
          constexpr int ACT = decltype(act_tag)::value;
#pragma unroll 1
          for (int m = 0; m < 8; ++m) {
            const uint32_t a = base + ((m ^ (i & 7)) << 4);
            const uint4 x = lds128(a);
            uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float cs = 1.f, sn = 0.f;
              if (rot) {
                const int jp = hh * 32 + 4 * m + e;
                float cl, sl;
                __sincosf((float)args.theta[jp] * (float)i, &sl, &cl);
                const float2 an = anchor_s[jp];
                cs = an.x * cl - an.y * sl;
                sn = an.y * cl + an.x * sl;
              }
              wv[e] = mul_bf16x2(gla_pair<ACT>(wv[e], cs, sn, valid), w2);
            }
            sts128(a, make_uint4(wv[0], wv[1], wv[2], wv[3]));
          }
        };
        if (args.act == LA_ACT_SWISH) tile(std::integral_constant<int, LA_ACT_SWISH>{});
        else if (args.act == LA_ACT_ONE_PLUS_ELU) tile(std::integral_constant<int, LA_ACT_ONE_PLUS_ELU>{});
        else tile(std::integral_constant<int, LA_ACT_NONE>{});
      } else {
        uint4 x[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = lds128(base + ((m ^ (i & 7)) << 4));
#pragma unroll
        for (int m = 0; m < 8; ++m) sts128(base + ((m ^ (i & 7)) << 4), mul_bf16x2(x[m], w2));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.scaled[s]);
    }
    // export: warp w reads TMEM lanes 32 (w % 4) .. +31 (the state rows), all 128 columns
    mbar_wait(&bars.done, 0);
    tc_fence_after();
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int dS = args.d;
    float* dst = args.delta_out + ((int64_t)bh * args.nseg * args.sub_per_seg + slot) * dS * dS + (int64_t)r * dS;
#pragma unroll 1
    for (int cb = 0; cb < (r < dS ? dS / 32 : 0); ++cb) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + cb * 32, v);
      tmem_ld_wait();
      float4* d4 = reinterpret_cast<float4*>(dst + cb * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, S_TM_COLS);
  }
}

}  // namespace

cudaError_t tc_summary_launch(const PassDesc& p, cudaStream_t st, const GlaPrologue* gla) {
  CUtensorMap mb, mc;
  if (!tc_make_map(&mb, p.b, p, p.sbb, SC) || !tc_make_map(&mc, p.c, p, p.sc, SC)) return cudaErrorInvalidValue;
  SumArgs a;
  std::memset(&a, 0, sizeof(a));
  a.heads = p.heads;
  a.n = p.n;
  a.seg_len = p.seg_len;
  a.nseg = p.nseg;
  a.rev = p.rev;
  a.sub_len = p.sub_len;
  a.sub_per_seg = p.sub_per_seg;
  a.g_lo = p.g_lo;
  a.d = p.d;
  a.lam = p.lam;
  a.delta_out = reinterpret_cast<float*>(p.delta_out);
  dim3 grid((p.g_hi - p.g_lo + 1) * p.sub_per_seg, p.batch * p.heads);
  if (gla == nullptr) {
    static std::atomic<bool> smem_set[64] = {};
    cudaError_t err = set_smem_once(tc_summary_kernel<false>, (int)S_SMEM_BYTES, smem_set);
    if (err != cudaSuccess) return err;
    return launch_pdl(tc_summary_kernel<false>, grid, dim3(S_THREADS), S_SMEM_BYTES, st, mb, mc, a);
  }
  a.theta = gla->theta;
  a.act = gla->act;
  a.offset = gla->offset;
  static std::atomic<bool> smem_set_gla[64] = {};
  cudaError_t err = set_smem_once(tc_summary_kernel<true>, (int)S_SMEM_BYTES, smem_set_gla);
  if (err != cudaSuccess) return err;
  return launch_pdl(tc_summary_kernel<true>, grid, dim3(S_THREADS), S_SMEM_BYTES, st, mb, mc, a);
}

}  // namespace la
