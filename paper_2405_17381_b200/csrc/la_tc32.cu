// la_tc32.cu -- the fp32 pass on tcgen05: the reference's "working" precision (float32, kernels.py:66)
// at <= 1e-4 relative on the tensor cores, by a three-term bf16 split.
//
// Every fp32 operand x is split into x = hi + lo + r with hi = bf16(x), lo = bf16(x - hi), |r| <= 2^-17 |x|,
// and each product of the pass (la_common.cuh algebra) becomes three bf16 MMAs accumulating in fp32:
//     a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi          (dropped: a_lo.b_lo + residuals, ~2^-16 |a||b|)
// That covers the operands (A, B, C from HBM) AND the two quantities the pass rounds internally: the
// masked scores P = S * M (fp32 in TMEM, split in place) and the bf16 copy of the carried state (split
// into a hi and a lo tile).  TF32 alone measured 5.6e-4 .. 8.5e-4, over the bar.
//
// One CTA per (batch, head, segment), chunks of C = 128 rows, 8 warps that all take part in every phase
// (thread = chunk row i and a 64-column half hh; warp w owns TMEM lanes 32 (w % 4) ..):
//
//   TMA  A, B, C fp32 tiles (4 boxes of [128 rows][32 fp32], 128B swizzle) into 64 KB regions
//   cvt  each region in place -> its bf16 hi tile | lo tile (the MMA's K-major / MN-major 128B-swizzle
//        layout); A~ = out_scale * A split straight into TMEM from the same registers
//   S    = A B^T                                 3 x 8 SS-MMAs (M = N = K = 128)       -> TMEM S
//   P    = S * M, split in place (per 32-key block: 16 hi columns | 16 lo columns)
//   B~   = in_scale * B, recombined from hi + lo, re-split in place (after S read B)
//   for value half h = 0, 1 (the state's bf16 hi + lo copy of one half fits the 32 KB left):
//     publish state[:, h] (hi, lo) to SMEM, pre-scale the TMEM state half by lam^b
//     X_h  O[:, h] = A~ state[:, h]              3 x 8 TS-MMAs (M = 128, N = 64)
//     U_h  state[:, h] += B~^T C[:, h]           3 x 8 SS-MMAs (M = 128, N = 64)
//   Y    O += P C                                3 x 8 TS-MMAs (M = N = 128)
//   out  TMEM O -> fp32 rows -> global
//
// SMEM: 3 x 64 KB operand regions + 32 KB state half = 224 KB.  TMEM: S | A~ | O | state = 512 columns.
// S is issued once A and B are split, and runs while C is split and the first state half published.  The
// A region is refilled as soon as S has read it, B and C once chunk t's MMAs are done.  State-only
// mode (segment summaries, la_api.cu segment_states) runs B~ and U only.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "la_common.cuh"
#include "la_ptx.cuh"
#include "la_tc.cuh"

namespace la {

namespace {

using namespace ptx;

constexpr int C = 128;
constexpr int D = 128;
constexpr int BOX = C * 32 * 4;        // 16 KB: one TMA box, 32 fp32 columns
constexpr int REGION = 4 * BOX;        // 64 KB: one fp32 operand tile = its bf16 hi + lo tiles
constexpr int HALF = C * 64 * 2;       // 16 KB: [128 rows][64 bf16], one 128B-swizzle column block
constexpr int BF_TILE = 2 * HALF;      // 32 KB: one bf16 tile (hi or lo)
constexpr int NTHREADS = 256;
constexpr uint32_t TM_S = 0, TM_AT = 128, TM_O = 256, TM_ST = 384, TM_COLS = 512;
constexpr uint32_t R_A = 0, R_B = REGION, R_C = 2 * REGION, R_ST = 3 * REGION;
constexpr size_t SMEM_BYTES = 3 * (size_t)REGION + 2 * HALF + 1024;

constexpr uint32_t IDESC_S = idesc_bf16(128, 128, 0, 0);    // A, B K-major
constexpr uint32_t IDESC_X = idesc_bf16(128, 64, 0, 1);     // A from TMEM, B (state half) MN-major
constexpr uint32_t IDESC_U = idesc_bf16(128, 64, 1, 1);     // A = B~^T MN-major, B = C half MN-major
constexpr uint32_t IDESC_U128 = idesc_bf16(128, 128, 1, 1); // state-only: the whole state at once
constexpr uint32_t IDESC_Y = idesc_bf16(128, 128, 0, 1);    // A = P from TMEM, B = C MN-major

struct Bars {
  uint64_t full[3];   // TMA: A, B, C fp32 tiles landed
  uint64_t s_done;    // MMA: S read A, B
  uint64_t x0_done;   // MMA: X_0 / U_0 done (the state-half SMEM copy is reusable)
  uint64_t all_done;  // MMA: every product of the chunk done
  uint32_t tmem_base;
};

struct Tc32Args {
  int heads, n, seg_len, nseg, rev;
  const double* lam;
  float* out;
  Strides3 so;
  const float* state_in;
  int64_t in_bh_stride, in_seg_stride;
  int in_T;
  float* state_out;
  int out_T;
  float* delta_out;  // state-only: [bh][nseg][d][d]
};

__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// this thread's 64 fp32 features [64 hh, 64 hh + 64) of row i of a TMA-landed fp32 region
__device__ __forceinline__ void read_f32_row(uint32_t region, int i, int hh, float (&x)[64]) {
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
    const uint32_t base = region + (uint32_t)((2 * hh + kb) * BOX) + (uint32_t)(i * 128);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 v = lds128(base + ((c ^ (i & 7)) << 4));
      x[kb * 32 + 4 * c + 0] = __uint_as_float(v.x);
      x[kb * 32 + 4 * c + 1] = __uint_as_float(v.y);
      x[kb * 32 + 4 * c + 2] = __uint_as_float(v.z);
      x[kb * 32 + 4 * c + 3] = __uint_as_float(v.w);
    }
  }
}

// (x0, x1) -> packed bf16x2 hi and lo words: hi = bf16(x), lo = bf16(x - hi)
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& h, uint32_t& l) {
  h = pack_bf16x2(x0, x1);
  l = pack_bf16x2(x0 - bf16lo(h), x1 - bf16hi(h));
}

// hi / lo words (feature pairs of this thread's 64 columns) into the bf16 tiles of a region
__device__ __forceinline__ void write_split(uint32_t region, int i, int hh, const uint32_t (&h)[32],
                                            const uint32_t (&l)[32]) {
  const uint32_t hb = region + (uint32_t)(hh * HALF), lb = region + BF_TILE + (uint32_t)(hh * HALF);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    sts128(hb + sw128(i, c), make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]));
    sts128(lb + sw128(i, c), make_uint4(l[4 * c], l[4 * c + 1], l[4 * c + 2], l[4 * c + 3]));
  }
}

template <bool STATE_ONLY>
__global__ void __launch_bounds__(NTHREADS, 1)
    tc32_pass_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ CUtensorMap map_c, const Tc32Args args) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;
  __shared__ __align__(16) float pw[C + 8];  // lam^0 .. lam^128
  const uint32_t smem = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem - smem_u32(smem_raw));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = tid & 127;   // chunk row == TMEM lane (warp w owns lanes 32 (w % 4) ..)
  const int hh = tid >> 7;   // 64-column half
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int seg = blockIdx.x, bh = blockIdx.y;
  const int bi = bh / args.heads, hi = bh % args.heads;
  const int p0 = seg * args.seg_len;
  const int p1 = min(args.n, p0 + args.seg_len);
  const int nchunks = p1 > p0 ? (p1 - p0 + C - 1) / C : 0;
  const int rev = args.rev;
  auto chunk_row0 = [&](int t) { return p0 + (rev ? (nchunks - 1 - t) : t) * C; };
  auto chunk_len = [&](int t) { return min(C, p1 - chunk_row0(t)); };
  (void)lane;

  if (tid == 0) {
    for (int x = 0; x < 3; ++x) mbar_init(&bars.full[x], 1);
    mbar_init(&bars.s_done, 1);
    mbar_init(&bars.x0_done, 1);
    mbar_init(&bars.all_done, 1);
    fence_mbar_init();
  }
  griddep_wait();  // PDL: the previous kernel of the stream has completed
  if (tid <= C) {
    const double l = load_decay(args.lam, hi);
    pw[tid] = (float)(pow_int(l, tid) * (l / l));
  }
  auto load = [&](int x, int t) {  // fp32 tile x (0 A, 1 B, 2 C) of chunk t: four 32-column boxes
    const CUtensorMap* map = x == 0 ? &map_a : (x == 1 ? &map_b : &map_c);
    mbar_arrive_expect_tx(&bars.full[x], REGION);
    uint8_t* g = smem_gen + x * REGION;
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) tma_load_4d(map, &bars.full[x], g + kb * BOX, 32 * kb, chunk_row0(t), hi, bi);
  };
  if (tid == 0 && nchunks > 0) {
    if (!STATE_ONLY) tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    tma_prefetch(&map_c);
    for (int x = STATE_ONLY ? 1 : 0; x < 3; ++x) load(x, 0);
  }
  if (warp == 0) tmem_alloc(&bars.tmem_base, TM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t st_cols = tmem + lane_off + TM_ST + 64 * hh;  // this thread's 64 state columns, row i

  // entering state (row i = the b-feature, columns = c-features), or zero
  if (nchunks > 0) {
#pragma unroll 1
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t w[16];
      if (!STATE_ONLY && args.state_in != nullptr) {
        const float* src = args.state_in + (int64_t)bh * args.in_bh_stride + (int64_t)seg * args.in_seg_stride;
        if (args.in_T) {
#pragma unroll
          for (int j = 0; j < 16; ++j) w[j] = __float_as_uint(src[(64 * hh + 16 * q4 + j) * D + i]);
        } else {
          const float4* s4 = reinterpret_cast<const float4*>(src + i * D + 64 * hh + 16 * q4);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 v = s4[j];
            w[4 * j] = __float_as_uint(v.x), w[4 * j + 1] = __float_as_uint(v.y);
            w[4 * j + 2] = __float_as_uint(v.z), w[4 * j + 3] = __float_as_uint(v.w);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = 0u;
      }
      tmem_st16(st_cols + 16 * q4, w);
    }
  }
  tmem_st_wait();  // the state columns are read back by other threads (publish_half): order the stores
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const uint32_t A_HI = smem + R_A, A_LO = A_HI + BF_TILE;
  const uint32_t B_HI = smem + R_B, B_LO = B_HI + BF_TILE;
  const uint32_t C_HI = smem + R_C, C_LO = C_HI + BF_TILE;
  const uint32_t ST_HI = smem + R_ST, ST_LO = ST_HI + HALF;

  // all threads: make generic SMEM writes and TMEM stores visible to the tensor core, then sync
  auto handoff = [&]() {
    fence_proxy_async_smem();
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  };
  // publish bf16 hi / lo of state columns [64 h + 32 hh, +32) (row i) and pre-scale them by `decay`
  auto publish_half = [&](int h, float decay) {
    float x[32];
    tmem_ld32(tmem + lane_off + TM_ST + 64 * h + 32 * hh, x);
    tmem_ld_wait();
    uint32_t hw[16], lw[16], sc[32];
#pragma unroll
    for (int q = 0; q < 16; ++q) split2(x[2 * q], x[2 * q + 1], hw[q], lw[q]);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      sts128(ST_HI + sw128(i, 4 * hh + c), make_uint4(hw[4 * c], hw[4 * c + 1], hw[4 * c + 2], hw[4 * c + 3]));
      sts128(ST_LO + sw128(i, 4 * hh + c), make_uint4(lw[4 * c], lw[4 * c + 1], lw[4 * c + 2], lw[4 * c + 3]));
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) sc[j] = __float_as_uint(x[j] * decay);
    tmem_st16(tmem + lane_off + TM_ST + 64 * h + 32 * hh, *reinterpret_cast<uint32_t(*)[16]>(sc));
    tmem_st16(tmem + lane_off + TM_ST + 64 * h + 32 * hh + 16, *reinterpret_cast<uint32_t(*)[16]>(sc + 16));
  };

  for (int t = 0; t < nchunks; ++t) {
    const uint32_t ph = t & 1;
    const int r0 = chunk_row0(t);
    const int b = chunk_len(t);
    const float decay = pw[b];
    float isc = i < b ? (rev ? pw[i + 1] : pw[b - 1 - i]) : 0.f;
#ifdef LA_MUTATE_DKV
    if (rev) isc = -isc;  // fault injection: the reference's `_dkv_step` sign flip (test_kernels.py:249-268)
#endif
    // ---------------------------------------------------------------- split the landed fp32 tiles
    if (!STATE_ONLY) {
      mbar_wait(&bars.full[0], ph);
      float x[64];
      read_f32_row(smem + R_A, i, hh, x);
      {  // A~ = out_scale * A straight into TMEM: hi columns [32 hh, +32), lo columns [64 + 32 hh, +32)
        const float osc = rev ? pw[max(b - 1 - i, 0)] : pw[i + 1];
        uint32_t th[32], tl[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) split2(osc * x[2 * q], osc * x[2 * q + 1], th[q], tl[q]);
        const uint32_t at = tmem + lane_off + TM_AT + 32 * hh;
        tmem_st16(at, *reinterpret_cast<uint32_t(*)[16]>(th));
        tmem_st16(at + 16, *reinterpret_cast<uint32_t(*)[16]>(th + 16));
        tmem_st16(at + 64, *reinterpret_cast<uint32_t(*)[16]>(tl));
        tmem_st16(at + 80, *reinterpret_cast<uint32_t(*)[16]>(tl + 16));
      }
      uint32_t h[32], l[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) split2(x[2 * q], x[2 * q + 1], h[q], l[q]);
      __syncthreads();  // every thread has read the fp32 region
      write_split(smem + R_A, i, hh, h, l);
    }
    {
      mbar_wait(&bars.full[1], ph);
      float x[64];
      read_f32_row(smem + R_B, i, hh, x);
      const float s = STATE_ONLY ? isc : 1.f;  // state-only: B~ directly (B is needed by no score)
      uint32_t h[32], l[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) split2(s * x[2 * q], s * x[2 * q + 1], h[q], l[q]);
      __syncthreads();
      write_split(smem + R_B, i, hh, h, l);
    }
    auto convert_c = [&]() {
      mbar_wait(&bars.full[2], ph);
      float x[64];
      read_f32_row(smem + R_C, i, hh, x);
      uint32_t h[32], l[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) split2(x[2 * q], x[2 * q + 1], h[q], l[q]);
      __syncthreads();
      write_split(smem + R_C, i, hh, h, l);
    };
    if (STATE_ONLY) {
      convert_c();
      // pre-scale the state by lam^b, then state += B~^T C (whole width)
      float x[32];
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        tmem_ld32(st_cols + 32 * part, x);
        tmem_ld_wait();
        uint32_t w[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(x[j] * decay);
        tmem_st16(st_cols + 32 * part, *reinterpret_cast<uint32_t(*)[16]>(w));
        tmem_st16(st_cols + 32 * part + 16, *reinterpret_cast<uint32_t(*)[16]>(w + 16));
      }
      handoff();
      if (tid == 0) {
#pragma unroll 1
        for (int g = 0; g < 3; ++g) {
          const uint32_t a = g == 2 ? B_LO : B_HI, c = g == 1 ? C_LO : C_HI;
#pragma unroll
          for (int kk = 0; kk < C / 16; ++kk)
            mma_bf16_ss(tmem + TM_ST, smem_desc_sw128(a + kk * 2048, HALF, 1024),
                        smem_desc_sw128(c + kk * 2048, HALF, 1024), IDESC_U128, 1);
        }
        mma_commit(&bars.all_done);
      }
      mbar_wait(&bars.all_done, ph);
      tc_fence_after();
      if (tid == 0 && t + 1 < nchunks) {
        load(1, t + 1);
        load(2, t + 1);
      }
      continue;
    }
    handoff();
    // ---------------------------------------------------------------- S = A B^T (C's split and the first
    // state publish overlap it)
    if (tid == 0) {
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t a = g == 2 ? A_LO : A_HI, bb = g == 1 ? B_LO : B_HI;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
          mma_bf16_ss(tmem + TM_S, smem_desc_sw128(a + off, 0, 1024), smem_desc_sw128(bb + off, 0, 1024), IDESC_S,
                      (g | kk) != 0);
        }
      }
      mma_commit(&bars.s_done);
    }
    convert_c();
    publish_half(0, decay);
    mbar_wait(&bars.s_done, ph);
    tc_fence_after();
    if (tid == 0 && t + 1 < nchunks) load(0, t + 1);  // A's tiles are consumed (A~ lives in TMEM)
    // ---------------------------------------------------------------- P = S * M, split in place
#pragma unroll 1
    for (int cbi = 0; cbi < 2; ++cbi) {
      const int cb = 2 * hh + cbi;
      float v[32];
      tmem_ld32(tmem + lane_off + TM_S + 32 * cb, v);
      tmem_ld_wait();
      uint32_t hw[16], lw[16];
#pragma unroll
      for (int jj = 0; jj < 32; jj += 2) {
        const int j = 32 * cb + jj;
        const int d0 = rev ? j - i : i - j, d1 = rev ? j + 1 - i : i - j - 1;
        const float p0 = d0 >= 0 ? v[jj] * pw[d0] : 0.f;
        const float p1v = d1 >= 0 ? v[jj + 1] * pw[d1] : 0.f;
        split2(p0, p1v, hw[jj >> 1], lw[jj >> 1]);
      }
      tmem_st16(tmem + lane_off + TM_S + 32 * cb, hw);
      tmem_st16(tmem + lane_off + TM_S + 32 * cb + 16, lw);
    }
    // ---------------------------------------------------------------- B~ = in_scale * B, in place
    {
      const uint32_t hb = B_HI + (uint32_t)(hh * HALF), lb = B_LO + (uint32_t)(hh * HALF);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 xh = lds128(hb + sw128(i, c)), xl = lds128(lb + sw128(i, c));
        const uint32_t hs[4] = {xh.x, xh.y, xh.z, xh.w}, ls[4] = {xl.x, xl.y, xl.z, xl.w};
        uint32_t ho[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          split2(isc * (bf16lo(hs[e]) + bf16lo(ls[e])), isc * (bf16hi(hs[e]) + bf16hi(ls[e])), ho[e], lo[e]);
        sts128(hb + sw128(i, c), make_uint4(ho[0], ho[1], ho[2], ho[3]));
        sts128(lb + sw128(i, c), make_uint4(lo[0], lo[1], lo[2], lo[3]));
      }
    }
    handoff();
    // ---------------------------------------------------------------- X_0, U_0
    auto issue_xu = [&](int h) {
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t at = TM_AT + (g == 2 ? 64 : 0), st = g == 1 ? ST_LO : ST_HI;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts(tmem + TM_O + 64 * h, tmem + at + kk * 8, smem_desc_sw128(st + kk * 2048, HALF, 1024), IDESC_X,
                      (g | kk) != 0);
      }
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t a = g == 2 ? B_LO : B_HI, c = (g == 1 ? C_LO : C_HI) + h * HALF;
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk)
          mma_bf16_ss(tmem + TM_ST + 64 * h, smem_desc_sw128(a + kk * 2048, HALF, 1024),
                      smem_desc_sw128(c + kk * 2048, HALF, 1024), IDESC_U, 1);
      }
    };
    if (tid == 0) {
      issue_xu(0);
      mma_commit(&bars.x0_done);
    }
    mbar_wait(&bars.x0_done, ph);
    tc_fence_after();
    publish_half(1, decay);
    handoff();
    // ---------------------------------------------------------------- X_1, U_1, Y = P C
    if (tid == 0) {
      issue_xu(1);
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t pofs = g == 2 ? 16 : 0, c = g == 1 ? C_LO : C_HI;
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk) {
          const uint32_t pcol = 32 * (kk >> 1) + pofs + 8 * (kk & 1);
          mma_bf16_ts(tmem + TM_O, tmem + TM_S + pcol, smem_desc_sw128(c + kk * 2048, HALF, 1024), IDESC_Y, 1);
        }
      }
      mma_commit(&bars.all_done);
    }
    mbar_wait(&bars.all_done, ph);
    tc_fence_after();
    if (tid == 0 && t + 1 < nchunks) {
      load(1, t + 1);
      load(2, t + 1);
    }
    // ---------------------------------------------------------------- out = O (fp32 rows)
    {
      float* orow = args.out + (int64_t)bi * args.so.b + (int64_t)hi * args.so.h + (int64_t)(r0 + i) * args.so.n +
                    64 * hh;
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        float y[32];
        tmem_ld32(tmem + lane_off + TM_O + 64 * hh + 32 * part, y);
        tmem_ld_wait();
        if (i < b) {
          float4* o4 = reinterpret_cast<float4*>(orow + 32 * part);
#pragma unroll
          for (int q = 0; q < 8; ++q) o4[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        }
      }
    }
    tc_fence_before();
  }
  if (tid == 0) griddep_launch();

  // ---------------------------------------------------------------- final state export
  if (nchunks > 0) {
    float* dst = nullptr;
    int T = 0;
    if (STATE_ONLY) {
      dst = args.delta_out + ((int64_t)bh * args.nseg + seg) * D * D;
    } else if (args.state_out != nullptr && (rev ? seg == 0 : seg == args.nseg - 1)) {
      dst = args.state_out + (int64_t)bh * D * D;
      T = args.out_T;
    }
    if (dst != nullptr) {
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        float x[32];
        tmem_ld32(st_cols + 32 * part, x);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = 64 * hh + 32 * part + j;
          dst[T ? (col * D + i) : (i * D + col)] = x[j];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, TM_COLS);
  }
}

thread_local char g_detail32[256];

// 4-D TMA descriptor (d, n, heads, batch) over an fp32 [.., .., .., 128] tensor: box 32 x 128, 128B swizzle
bool tc32_make_map(CUtensorMap* map, const void* base, const PassDesc& p, const Strides3& s) {
  static const PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  if (enc == nullptr) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p.d, (cuuint64_t)p.n, (cuuint64_t)p.heads, (cuuint64_t)p.batch};
  cuuint64_t strides[3] = {(cuuint64_t)s.n * 4, (cuuint64_t)s.h * 4, (cuuint64_t)s.b * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)C, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  if (p.heads == 1) strides[1] = strides[0] * (cuuint64_t)p.n;
  if (p.batch == 1) strides[2] = strides[1] * (cuuint64_t)p.heads;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    snprintf(g_detail32, sizeof(g_detail32), "fp32 cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool tc32_supported(int dtype, int d, const int64_t* strides, int count) {
  if (dtype != LA_F32 || d != D) return false;
  for (int x = 0; x < 3 * count; ++x)
    if ((strides[x] * 4) % 16 != 0) return false;
  return true;
}

// One wave of 1-CTA-per-SM segments when batch * heads leaves SMs idle (as tc_plan); the summaries are
// whole segments (state-only mode of the same kernel), so sub_per_seg = 1.
Plan tc32_plan(int64_t bh, int64_t n, int64_t want_segments, int sms) {
  if (sms < 1) sms = kNumSMs;
  if (want_segments > 0) return make_plan(bh, n, C, want_segments, sms, 1);
  const int64_t nchunks = (n + C - 1) / C;
  const int64_t cap = std::max<int64_t>(1, sms / bh);
  int64_t nseg = 1;
  if (bh * 10 < (int64_t)sms * 6) nseg = std::min<int64_t>(cap, std::max<int64_t>(1, nchunks / 2));
  Plan p = make_plan(bh, n, C, nseg, sms, 1);
  p.nseg_ws = (int)std::max<int64_t>(cap, p.nseg);
  p.nsub_ws = p.nseg_ws;
  return p;
}

cudaError_t tc32_launch(const PassDesc& p, bool state_only, cudaStream_t st) {
  CUtensorMap ma, mb, mc;
  std::memset(&ma, 0, sizeof(ma));
  if (!tc32_make_map(&mb, p.b, p, p.sbb) || !tc32_make_map(&mc, p.c, p, p.sc)) return cudaErrorInvalidValue;
  if (!state_only && !tc32_make_map(&ma, p.a, p, p.sa)) return cudaErrorInvalidValue;
  Tc32Args a;
  std::memset(&a, 0, sizeof(a));
  a.heads = p.heads;
  a.n = p.n;
  a.seg_len = p.seg_len;
  a.nseg = p.nseg;
  a.rev = p.rev;
  a.lam = p.lam;
  a.out = reinterpret_cast<float*>(p.out);
  a.so = p.so;
  a.state_in = reinterpret_cast<const float*>(p.state_in);
  a.in_bh_stride = p.state_in_bh_stride;
  a.in_seg_stride = p.state_in_seg_stride;
  a.in_T = p.state_in_T;
  a.state_out = reinterpret_cast<float*>(p.state_out);
  a.out_T = p.state_out_T;
  a.delta_out = reinterpret_cast<float*>(p.delta_out);
  dim3 grid(p.nseg, p.batch * p.heads);
  if (state_only) {
    static std::atomic<bool> set[64] = {};
    cudaError_t err = set_smem_once(tc32_pass_kernel<true>, (int)SMEM_BYTES, set);
    if (err != cudaSuccess) return err;
    return launch_pdl(tc32_pass_kernel<true>, grid, dim3(NTHREADS), SMEM_BYTES, st, ma, mb, mc, a);
  }
  static std::atomic<bool> set[64] = {};
  cudaError_t err = set_smem_once(tc32_pass_kernel<false>, (int)SMEM_BYTES, set);
  if (err != cudaSuccess) return err;
  return launch_pdl(tc32_pass_kernel<false>, grid, dim3(NTHREADS), SMEM_BYTES, st, ma, mb, mc, a);
}

}  // namespace la
