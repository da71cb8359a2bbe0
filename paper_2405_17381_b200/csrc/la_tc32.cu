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
// One CTA per (batch, head, segment), chunks of C = 128 rows.  Warps 0-7 are workers (thread = chunk row i
// and a 64-column half hh; warp w owns TMEM lanes 32 (w % 4) ..); warp 8 issues: lane 0 every MMA, lane 1
// every TMA load / store, between mbarrier hand-offs with the workers:
//
//   TMA  A, B, C fp32 tiles (4 boxes of [128 rows][32 fp32], 128B swizzle) into 64 KB regions
//   cvt  each region in place -> its bf16 hi tile | lo tile (the MMA's K-major / MN-major 128B-swizzle
//        layout); A~ = out_scale * A split straight into TMEM from the same registers
//   S    = A B^T                                 3 x 8 SS-MMAs (M = N = K = 128)       -> TMEM S
//   P    = S * M, split in place (per 32-key block: 16 hi columns | 16 lo columns)
//   B~   = in_scale * B, recombined from hi + lo, re-split in place (after S read B)
//   X_h  O[:, h] = A~ state[:, h] for value half h = 0, 1 (the bf16 hi + lo copy of one state half fits the
//        32 KB left; half 1's copy waits in registers until X_0 read half 0's)
//                                                3 x 8 TS-MMAs each (M = 128, N = 64)
//   U    state = lam^b state + B~^T C           TMEM state pre-scaled by the workers; 3 x 8 SS-MMAs (N = 128)
//   Y    O = P C (issued before X_0 / X_1, which accumulate onto it)   3 x 8 TS-MMAs (M = N = 128)
//   out  TMEM O -> fp32 rows staged in C's region -> TMA store
//
// SMEM: 3 x 64 KB operand regions + 32 KB state half = 224 KB.  TMEM: S | A~ | O | state = 512 columns.
// Overlap: the state is published while S runs; B~ and C's split come right after S so the state update
// (B's last reader) runs while the scores are converted and B's refill for the next chunk is issued early;
// the next chunk's A is split while X_1 and Y run.  The A region is refilled as soon as S has read it,
// B after the state update, C once the output rows staged in it are stored.  State-only mode (segment summaries, la_api.cu segment_states) runs B~ and
// U only.
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

#ifdef LA_TRACE
// debug build only: thread 0 of CTA (0, 0) stamps the phases of its first 32 chunks ([chunk][16 events])
__device__ unsigned long long* g_tc32_trace = nullptr;
#define T32(t, ev)                                                               \
  do {                                                                           \
    if (t32p != nullptr && tid == 0 && (t) < 32) t32p[(t) * 16 + (ev)] = clock64(); \
  } while (0)
#else
#define T32(t, ev) \
  do {             \
  } while (0)
#endif

constexpr int C = 128;
constexpr int D = 128;
constexpr int BOX = C * 32 * 4;        // 16 KB: one TMA box, 32 fp32 columns
constexpr int REGION = 4 * BOX;        // 64 KB: one fp32 operand tile = its bf16 hi + lo tiles
constexpr int HALF = C * 64 * 2;       // 16 KB: [128 rows][64 bf16], one 128B-swizzle column block
constexpr int BF_TILE = 2 * HALF;      // 32 KB: one bf16 tile (hi or lo)
constexpr int NUM_WORKERS = 8;                  // warps 0-7: conversions (thread = row i, half hh)
constexpr int WARP_ISSUE = NUM_WORKERS;          // warp 8: lane 0 issues the MMAs, lane 1 the TMA loads / stores
constexpr int NTHREADS = (NUM_WORKERS + 1) * 32;
constexpr uint32_t TM_S = 0, TM_AT = 128, TM_O = 256, TM_ST = 384, TM_COLS = 512;
constexpr uint32_t R_A = 0, R_B = REGION, R_C = 2 * REGION, R_ST = 3 * REGION;
constexpr size_t SMEM_BYTES = 3 * (size_t)REGION + 2 * HALF + 1024;

constexpr uint32_t IDESC_S = idesc_bf16(128, 128, 0, 0);    // A, B K-major
constexpr uint32_t IDESC_X = idesc_bf16(128, 64, 0, 1);     // A from TMEM, B (state half) MN-major
constexpr uint32_t IDESC_U128 = idesc_bf16(128, 128, 1, 1); // A = B~^T MN-major, B = C MN-major: the whole state
constexpr uint32_t IDESC_Y = idesc_bf16(128, 128, 0, 1);    // A = P from TMEM, B = C MN-major

struct Bars {
  uint64_t full[3];   // TMA: A, B, C fp32 tiles landed
  uint64_t s_done;    // MMA: S read A, B
  uint64_t x0_done;   // MMA: X_0 done (the state-half SMEM copy is reusable)
  uint64_t u1_done;   // MMA: the state update done (the last reader of B)
  uint64_t x1_done;   // MMA: X_1 done (A~'s last reader)
  uint64_t all_done;  // MMA: every product of the chunk done
  uint64_t go_s, go_u, go_x0, go_x1;  // workers -> issuer: operands of S / of U / of X_0 / of X_1, Y ready
  uint64_t o_staged;            // workers -> issuer: O(t) staged in C's region for the TMA store
  uint32_t tmem_base;
};

struct Tc32Args {
  int heads, n, seg_len, nseg, rev;
  int d;  // head dim (a multiple of 32, <= 128): features past d are zero (TMA out-of-bounds fill), states d x d
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
                     const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_o,
                     const Tc32Args args) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;
  __shared__ __align__(16) float pw[C + 8];  // lam^0 .. lam^128
  const uint32_t smem = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem - smem_u32(smem_raw));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool worker = warp < NUM_WORKERS;
  const int i = tid & 127;   // worker: chunk row == TMEM lane (warp w owns lanes 32 (w % 4) ..)
  const int hh = (tid >> 7) & 1;  // worker: 64-column half
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int seg = blockIdx.x, bh = blockIdx.y;
  const int bi = bh / args.heads, hi = bh % args.heads;
  const int p0 = seg * args.seg_len;
  const int p1 = min(args.n, p0 + args.seg_len);
  const int nchunks = p1 > p0 ? (p1 - p0 + C - 1) / C : 0;
  const int rev = args.rev;
  auto chunk_row0 = [&](int t) { return p0 + (rev ? (nchunks - 1 - t) : t) * C; };
  auto chunk_len = [&](int t) { return min(C, p1 - chunk_row0(t)); };
#ifdef LA_TRACE
  unsigned long long* const t32p = (blockIdx.x == 0 && blockIdx.y == 0) ? g_tc32_trace : nullptr;
#endif

  if (tid == 0) {
    for (int x = 0; x < 3; ++x) mbar_init(&bars.full[x], 1);
    mbar_init(&bars.s_done, 1);
    mbar_init(&bars.x0_done, 1);
    mbar_init(&bars.u1_done, 1);
    mbar_init(&bars.x1_done, 1);
    mbar_init(&bars.all_done, 1);
    mbar_init(&bars.go_s, NUM_WORKERS);
    mbar_init(&bars.go_u, NUM_WORKERS);
    mbar_init(&bars.go_x0, NUM_WORKERS);
    mbar_init(&bars.go_x1, NUM_WORKERS);
    mbar_init(&bars.o_staged, NUM_WORKERS);
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
  const bool issuer = warp == WARP_ISSUE && lane == 0;
  if (tid == 0 && nchunks > 0) {  // the thread that initialised the barriers: chunk 0's loads before the sync
    if (!STATE_ONLY) {
      tma_prefetch(&map_a);
      tma_prefetch(&map_o);
    }
    tma_prefetch(&map_b);
    tma_prefetch(&map_c);
    for (int x = STATE_ONLY ? 1 : 0; x < 3; ++x) load(x, 0);
  }
  if (warp == WARP_ISSUE) tmem_alloc(&bars.tmem_base, TM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t st_cols = tmem + lane_off + TM_ST + 64 * hh;  // worker: its 64 state columns, row i

  const uint32_t A_HI = smem + R_A, A_LO = A_HI + BF_TILE;
  const uint32_t B_HI = smem + R_B, B_LO = B_HI + BF_TILE;
  const uint32_t C_HI = smem + R_C, C_LO = C_HI + BF_TILE;
  const uint32_t ST_HI = smem + R_ST, ST_LO = ST_HI + HALF;

  if (warp == WARP_ISSUE && lane == 1) {
    // ------------------------------------------------------------------ TMA lane (warp 8, lane 1): refills and
    // the output stores, each as soon as its region is free (decoupled from the MMA lane, whose issue
    // blocks while the tensor core's queue is full)
    for (int t = 0; t < nchunks; ++t) {
      if (STATE_ONLY) {
        mbar_wait(&bars.all_done, t & 1);
        if (t + 1 < nchunks) {
          load(1, t + 1);
          load(2, t + 1);
        }
        continue;
      }
      mbar_wait(&bars.s_done, t & 1);
      if (t + 1 < nchunks) load(0, t + 1);  // A's SMEM tiles consumed by S
      mbar_wait(&bars.u1_done, t & 1);
      if (t + 1 < nchunks) load(1, t + 1);  // B's by the state update
      // out(t): staged by the workers in C's region once the chunk's products are done; store it, then
      // refill C with the next chunk's tile
      mbar_wait(&bars.o_staged, t & 1);
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) tma_store_4d(&map_o, smem_gen + R_C + kb * BOX, 32 * kb, chunk_row0(t), hi, bi);
      tma_store_commit();
      tma_store_wait_read();
      if (t + 1 < nchunks) load(2, t + 1);
    }
    tma_store_wait_all();
    griddep_launch();
  } else if (issuer) {
    // ------------------------------------------------------------------ MMA lane (warp 8, lane 0)
    auto go = [&](uint64_t* bar, int t) {
      mbar_wait(bar, t & 1);
      tc_fence_after();
    };
    auto issue_x = [&](int h) {  // O[:, h] += A~ state[:, h]  (Y initialised O)
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t at = TM_AT + (g == 2 ? 64 : 0), st = g == 1 ? ST_LO : ST_HI;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts(tmem + TM_O + 64 * h, tmem + at + kk * 8, smem_desc_sw128(st + kk * 2048, HALF, 1024),
                      IDESC_X, 1);
      }
    };
    auto issue_u = [&]() {  // state += B~^T C, both halves
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t a = g == 2 ? B_LO : B_HI, c = g == 1 ? C_LO : C_HI;
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk)
          mma_bf16_ss(tmem + TM_ST, smem_desc_sw128(a + kk * 2048, HALF, 1024),
                      smem_desc_sw128(c + kk * 2048, HALF, 1024), IDESC_U128, 1);
      }
    };
    for (int t = 0; t < nchunks; ++t) {
      if (STATE_ONLY) {
        go(&bars.go_s, t);  // B~, C split; state pre-scaled
        issue_u();
        mma_commit(&bars.all_done);
        continue;
      }
      // S = A B^T
      go(&bars.go_s, t);  // A(t), B(t) split, A~(t) in TMEM; Y(t-1) done with P's columns (workers saw all_done)
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
      // the state update first (B's last reader: B's refill for the next chunk starts as early as possible;
      // X reads the SMEM copy of the state taken before it, so the TMEM update does not disturb X)
      go(&bars.go_u, t);  // B~, C split; the TMEM state pre-scaled
      issue_u();
      mma_commit(&bars.u1_done);
      // Y = P C first (it initialises O; both X halves accumulate onto it), then X_0 = A~ state[:, 0:64]
      go(&bars.go_x0, t);  // P, the first state half's copy; O(t-1) drained
#pragma unroll 1
      for (int g = 0; g < 3; ++g) {
        const uint32_t pofs = g == 2 ? 16 : 0, c = g == 1 ? C_LO : C_HI;
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk) {
          const uint32_t pcol = 32 * (kk >> 1) + pofs + 8 * (kk & 1);
          mma_bf16_ts(tmem + TM_O, tmem + TM_S + pcol, smem_desc_sw128(c + kk * 2048, HALF, 1024), IDESC_Y,
                      (g | kk) != 0);
        }
      }
      issue_x(0);
      mma_commit(&bars.x0_done);
      // X_1 (A~'s last reader, the chunk's last product)
      go(&bars.go_x1, t);  // the second state half's copy in SMEM
      issue_x(1);
      mma_commit(&bars.x1_done);
      mma_commit(&bars.all_done);
    }
    // drain: every commit must land before the CTA retires
    if (nchunks > 0) mbar_wait(&bars.all_done, (nchunks - 1) & 1);
  } else if (worker) {
    // ------------------------------------------------------------------ workers (warps 0-7): conversions
    auto wbar = [&]() { named_bar_sync(1, NUM_WORKERS * 32); };
    auto signal = [&](uint64_t* bar) {  // generic SMEM writes + TMEM stores -> the tensor core, then arrive
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    auto await = [&](uint64_t* bar, int t) {
      mbar_wait(bar, t & 1);
      tc_fence_after();
    };
    // entering state (row i = the b-feature, columns = c-features), or zero
    if (nchunks > 0) {
#pragma unroll 1
      for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t w[16];
        if (!STATE_ONLY && args.state_in != nullptr && i < args.d && 64 * hh + 16 * q4 < args.d) {
          const int dS = args.d;
          const float* src = args.state_in + (int64_t)bh * args.in_bh_stride + (int64_t)seg * args.in_seg_stride;
          if (args.in_T) {
#pragma unroll
            for (int j = 0; j < 16; ++j) w[j] = __float_as_uint(src[(64 * hh + 16 * q4 + j) * dS + i]);
          } else {
            const float4* s4 = reinterpret_cast<const float4*>(src + i * dS + 64 * hh + 16 * q4);
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
    tmem_st_wait();  // the state columns are read back by other workers (take_half): order the stores
    tc_fence_before();
    wbar();
    tc_fence_after();
    // fp32 region x -> its bf16 hi / lo tiles, every element scaled by `sc`
    auto split_region = [&](uint32_t region, int x, int t, float sc) {
      mbar_wait(&bars.full[x], t & 1);
      float v[64];
      read_f32_row(smem + region, i, hh, v);
      uint32_t h[32], l[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) split2(sc * v[2 * q], sc * v[2 * q + 1], h[q], l[q]);
      wbar();  // every worker has read the fp32 region
      write_split(smem + region, i, hh, h, l);
    };
    // B of chunk t: SMEM hi / lo tiles for S; B~ = in_scale B's words kept in registers (bt_h / bt_l) and
    // written over B's tiles once S has read them -- no second pass over B in shared memory
    auto split_b = [&](int t, float isc, uint32_t (&bth)[32], uint32_t (&btl)[32]) {
      mbar_wait(&bars.full[1], t & 1);
      float v[64];
      read_f32_row(smem + R_B, i, hh, v);
      uint32_t h[32], l[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        split2(v[2 * q], v[2 * q + 1], h[q], l[q]);
        split2(isc * v[2 * q], isc * v[2 * q + 1], bth[q], btl[q]);
      }
      wbar();  // every worker has read the fp32 region
      write_split(smem + R_B, i, hh, h, l);
    };
    // A of chunk t: SMEM hi / lo tiles; A~ = out_scale A's words returned for TMEM
    auto convert_a = [&](int t, uint32_t (&th)[32], uint32_t (&tl)[32]) {
      const int b = chunk_len(t);
      mbar_wait(&bars.full[0], t & 1);
      float x[64];
      read_f32_row(smem + R_A, i, hh, x);
      const float osc = rev ? pw[max(b - 1 - i, 0)] : pw[i + 1];
#pragma unroll
      for (int q = 0; q < 32; ++q) split2(osc * x[2 * q], osc * x[2 * q + 1], th[q], tl[q]);
      uint32_t h[32], l[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) split2(x[2 * q], x[2 * q + 1], h[q], l[q]);
      wbar();
      write_split(smem + R_A, i, hh, h, l);
    };
    auto store_at = [&](const uint32_t (&th)[32], const uint32_t (&tl)[32]) {
      const uint32_t at = tmem + lane_off + TM_AT + 32 * hh;  // hi columns [32 hh, +32), lo [64 + 32 hh, +32)
      tmem_st16(at, *reinterpret_cast<const uint32_t(*)[16]>(th));
      tmem_st16(at + 16, *reinterpret_cast<const uint32_t(*)[16]>(th + 16));
      tmem_st16(at + 64, *reinterpret_cast<const uint32_t(*)[16]>(tl));
      tmem_st16(at + 80, *reinterpret_cast<const uint32_t(*)[16]>(tl + 16));
    };
    // bf16 hi / lo of state columns [64 h + 32 hh, +32) (row i) -> hw / lw; the TMEM copy pre-scaled by `decay`
    auto take_half = [&](int h, float decay, uint32_t (&hw)[16], uint32_t (&lw)[16]) {
      float x[32];
      tmem_ld32(tmem + lane_off + TM_ST + 64 * h + 32 * hh, x);
      tmem_ld_wait();
      uint32_t sc[32];
#pragma unroll
      for (int q = 0; q < 16; ++q) split2(x[2 * q], x[2 * q + 1], hw[q], lw[q]);
#pragma unroll
      for (int j = 0; j < 32; ++j) sc[j] = __float_as_uint(x[j] * decay);
      tmem_st16(tmem + lane_off + TM_ST + 64 * h + 32 * hh, *reinterpret_cast<uint32_t(*)[16]>(sc));
      tmem_st16(tmem + lane_off + TM_ST + 64 * h + 32 * hh + 16, *reinterpret_cast<uint32_t(*)[16]>(sc + 16));
    };
    auto publish = [&](const uint32_t (&hw)[16], const uint32_t (&lw)[16]) {  // -> the SMEM state-half copy
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sts128(ST_HI + sw128(i, 4 * hh + c), make_uint4(hw[4 * c], hw[4 * c + 1], hw[4 * c + 2], hw[4 * c + 3]));
        sts128(ST_LO + sw128(i, 4 * hh + c), make_uint4(lw[4 * c], lw[4 * c + 1], lw[4 * c + 2], lw[4 * c + 3]));
      }
    };
    // the state entering chunk t: half 0's bf16 copy to SMEM, half 1's kept in registers (h1w / h1l) until X_0
    // has read the SMEM copy; the TMEM state pre-scaled by lam^b(t) for the chunk's whole-width update
    uint32_t h1w[16], h1l[16];
    auto take_state = [&](int t) {
      const float dec = pw[chunk_len(t)];
      uint32_t hw[16], lw[16];
      take_half(0, dec, hw, lw);
      publish(hw, lw);
      take_half(1, dec, h1w, h1l);
    };
    if (!STATE_ONLY && nchunks > 0) {  // chunk 0's A (later chunks': while the previous one's products run)
      uint32_t th[32], tl[32];
      convert_a(0, th, tl);
      store_at(th, tl);
    }
    // O columns [64 h + 32 hh, +32) of row i -> fp32 TMA-store box 2 h + hh of C's region
    auto stage_o_box = [&](int h) {
      float y[32];
      tmem_ld32(tmem + lane_off + TM_O + 64 * h + 32 * hh, y);
      tmem_ld_wait();
      const uint32_t box = smem + R_C + (uint32_t)((2 * h + hh) * BOX) + (uint32_t)(i * 128);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        sts128(box + ((c ^ (i & 7)) << 4), make_uint4(__float_as_uint(y[4 * c]), __float_as_uint(y[4 * c + 1]),
                                                       __float_as_uint(y[4 * c + 2]), __float_as_uint(y[4 * c + 3])));
    };
    const int quad = warp & 3;
    const uint32_t pw_addr = smem_u32(pw);
    for (int t = 0; t < nchunks; ++t) {
      const int b = chunk_len(t);
      const float decay = pw[b];
      float isc = i < b ? (rev ? pw[i + 1] : pw[b - 1 - i]) : 0.f;
#ifdef LA_MUTATE_DKV
      if (rev) isc = -isc;  // fault injection: the reference's `_dkv_step` sign flip (test_kernels.py:249-268)
#endif
      T32(t, 0);
      if (STATE_ONLY) {
        split_region(R_B, 1, t, isc);  // B~ directly (B feeds no score here)
        split_region(R_C, 2, t, 1.f);
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {  // pre-scale the state by lam^b
          float x[32];
          tmem_ld32(st_cols + 32 * part, x);
          tmem_ld_wait();
          uint32_t w[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(x[j] * decay);
          tmem_st16(st_cols + 32 * part, *reinterpret_cast<uint32_t(*)[16]>(w));
          tmem_st16(st_cols + 32 * part + 16, *reinterpret_cast<uint32_t(*)[16]>(w + 16));
        }
        signal(&bars.go_s);
        await(&bars.all_done, t);
        continue;
      }
      uint32_t bth[32], btl[32];
      split_b(t, isc, bth, btl);
      signal(&bars.go_s);  // A(t), A~(t), B(t)
      T32(t, 1);
      take_state(t);  // while S runs
      await(&bars.s_done, t);
      T32(t, 4);
      // B~ = in_scale * B over B's tiles (S has read them), from the words kept since B's split
      write_split(smem + R_B, i, hh, bth, btl);
      T32(t, 3);
      split_region(R_C, 2, t, 1.f);
      signal(&bars.go_u);  // B~, C: the state update may run while the scores are converted
      T32(t, 2);
      // P = S * M, split in place: per 32-key block, a zero block (causality), an off-diagonal block
      // (lam^|i-j| = per-row base x a broadcast ladder), or the diagonal block
#pragma unroll 1
      for (int cbi = 0; cbi < 2; ++cbi) {
        const int cb = 2 * hh + cbi;
        uint32_t hw[16], lw[16];
        if (rev ? (cb < quad) : (cb > quad)) {
#pragma unroll
          for (int e = 0; e < 16; ++e) hw[e] = lw[e] = 0u;
        } else {
          float v[32];
          tmem_ld32(tmem + lane_off + TM_S + 32 * cb, v);
          if (cb != quad) {
            const float base = rev ? pw[32 * cb - i] : pw[i - 32 * cb - 31];
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              // ladder lam^(31 - jj) (fwd) or lam^jj (rev) for jj = 4q .. 4q+3, one broadcast LDS.128
              const uint4 wq = lds128(pw_addr + 4 * (rev ? 4 * q : 28 - 4 * q));
              float w0 = __uint_as_float(wq.x), w1 = __uint_as_float(wq.y), w2 = __uint_as_float(wq.z),
                    w3 = __uint_as_float(wq.w);
              if (!rev) {
                const float t0 = w0, t1 = w1;
                w0 = w3;
                w1 = w2;
                w2 = t1;
                w3 = t0;
              }
              split2(v[4 * q] * (base * w0), v[4 * q + 1] * (base * w1), hw[2 * q], lw[2 * q]);
              split2(v[4 * q + 2] * (base * w2), v[4 * q + 3] * (base * w3), hw[2 * q + 1], lw[2 * q + 1]);
            }
          } else {
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; jj += 2) {
              const int d0 = rev ? jj - lane : lane - jj, d1 = rev ? jj + 1 - lane : lane - jj - 1;
              split2(d0 >= 0 ? v[jj] * pw[d0] : 0.f, d1 >= 0 ? v[jj + 1] * pw[d1] : 0.f, hw[jj >> 1], lw[jj >> 1]);
            }
          }
        }
        tmem_st16(tmem + lane_off + TM_S + 32 * cb, hw);
        tmem_st16(tmem + lane_off + TM_S + 32 * cb + 16, lw);
      }
      T32(t, 5);
      signal(&bars.go_x0);
      await(&bars.x0_done, t);
      T32(t, 6);
      publish(h1w, h1l);
      signal(&bars.go_x1);
      T32(t, 7);
      // out(t), value half 0: final once X_0 is done (Y, issued before it, and the state update were C's
      // readers), so it is staged in C's region now, box `hh` per thread; half 1 after X_1 below.  The
      // workers' barrier orders the staging after every worker's C split in the CTA's own order too.
      wbar();
      stage_o_box(0);
      // while the state update, X_1 and Y run: the next chunk's A (its SMEM tiles are free since S), its A~
      // once X_1 has read A~
      if (t + 1 < nchunks) {
        uint32_t th[32], tl[32];
        convert_a(t + 1, th, tl);
        T32(t, 8);
        await(&bars.x1_done, t);
        T32(t, 9);
        store_at(th, tl);
      }
      // out(t), value half 1 (final after X_1), then the TMA lane stores the staged rows
      await(&bars.all_done, t);
      T32(t, 10);
      stage_o_box(1);
      signal(&bars.o_staged);
      T32(t, 11);
    }

    // ------------------------------------------------------------------ final state export
    if (nchunks > 0) {
      float* dst = nullptr;
      int T = 0;
      const int dS = args.d;
      if (STATE_ONLY) {
        dst = args.delta_out + ((int64_t)bh * args.nseg + seg) * dS * dS;
      } else if (args.state_out != nullptr && (rev ? seg == 0 : seg == args.nseg - 1)) {
        dst = args.state_out + (int64_t)bh * dS * dS;
        T = args.out_T;
      }
      if (dst != nullptr && i < dS) {
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
          float x[32];
          tmem_ld32(st_cols + 32 * part, x);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = 64 * hh + 32 * part + j;
            if (col < dS) dst[T ? (col * dS + i) : (i * dS + col)] = x[j];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_ISSUE) {
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

#ifdef LA_TRACE
extern "C" __attribute__((visibility("default"))) int la_debug_set_trace32(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(g_tc32_trace, &dev_ptr, sizeof(dev_ptr));
}
#endif

bool tc32_supported(int dtype, int d, const int64_t* strides, int count) {
  // d < 128 runs the d = 128 kernel on zero-padded features (TMA out-of-bounds fill / clipped stores)
  if (dtype != LA_F32 || d < 32 || d > D || d % 32 != 0) return false;
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
  CUtensorMap ma, mb, mc, mo;
  std::memset(&ma, 0, sizeof(ma));
  std::memset(&mo, 0, sizeof(mo));
  if (!tc32_make_map(&mb, p.b, p, p.sbb) || !tc32_make_map(&mc, p.c, p, p.sc)) return cudaErrorInvalidValue;
  if (!state_only && (!tc32_make_map(&ma, p.a, p, p.sa) || !tc32_make_map(&mo, p.out, p, p.so)))
    return cudaErrorInvalidValue;
  Tc32Args a;
  std::memset(&a, 0, sizeof(a));
  a.heads = p.heads;
  a.n = p.n;
  a.d = p.d;
  a.seg_len = p.seg_len;
  a.nseg = p.nseg;
  a.rev = p.rev;
  a.lam = p.lam;
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
    return launch_pdl(tc32_pass_kernel<true>, grid, dim3(NTHREADS), SMEM_BYTES, st, ma, mb, mc, mo, a);
  }
  static std::atomic<bool> set[64] = {};
  cudaError_t err = set_smem_once(tc32_pass_kernel<false>, (int)SMEM_BYTES, set);
  if (err != cudaSuccess) return err;
  return launch_pdl(tc32_pass_kernel<false>, grid, dim3(NTHREADS), SMEM_BYTES, st, ma, mb, mc, mo, a);
}

}  // namespace la
