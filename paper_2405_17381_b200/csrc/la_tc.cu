// la_tc.cu -- the bf16 pass kernel on B200 tensor cores: TMA -> SMEM (128B
// swizzle) -> tcgen05.mma (fp32 accumulators in TMEM) -> tcgen05.ld epilogues.
//
// One CTA owns one (batch, head, segment) and walks its chunks of C = 128 rows
// (fwd) or walks them backwards (rev).  The d x d fp32 state lives in TMEM and
// the tensor core accumulates each chunk's contribution straight into it; a
// bf16 copy in SMEM is the B operand of the inter-chunk product.  Per chunk
// (la_common.cuh algebra):
//
//   S     = A B^T                 SS-MMA  M=N=K=128              -> TMEM S[t%2]
//   P     = bf16(S * M_decay)     P warps: tcgen05.ld S, mask, tcgen05.st -> TMEM (aliases S[t%2])
//   A~    = bf16(out_scale * A)   P warps: SMEM rows -> TMEM (upper half of S[t%2])
//   B~    = in_scale * B          state warps, in place in SMEM once S has consumed B
//   state = lam^b state + B~^T C  state warps pre-scale the TMEM state, SS-MMA accumulates
//   O     = A~ state_bf16 + P C   TS-MMAs (A operands from TMEM)  -> TMEM O
//   out   = bf16(O)               output warps: tcgen05.ld -> registers -> global
//
// Warp roles (26 warps): 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2-9 P/A~
// conversion, 10-17 B scaling + output, 18-25 state publish -- each group two warps per TMEM lane
// quadrant, each warp owning 64 of the 128 columns.  Every hand-off is an mbarrier; a stage is
// handed back to the TMA producer by the tensor core's own commit after its
// last MMA, and the MMA issuer runs one chunk ahead on S so the score
// conversion of chunk t+1 overlaps the products of chunk t.
//
// Shared memory: 2 stages x {A, B, C} tiles (3 x 32 KB) + the bf16 state
// (32 KB) = 224 KB -> one CTA per SM.  TMEM: S0 | S1 | O | state = 512 columns.
//
// GLA mode (template GLA, la_gla_core_fwd): the GLA prologue q = rot(act(qp)),
// k = rot(act(kp)) (model.py:381-397, positional.py:126-150) is applied to each landed A / B tile in
// shared memory by the state warps -- idle for most of a chunk -- before S is issued, so the pre-activation
// projections stream straight into the core (no q / k round trip through HBM); a store lane writes the
// transformed tiles out for the backward when asked.
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "la_common.cuh"
#include "la_ptx.cuh"
#include "la_scan.cuh"
#include "la_tc.cuh"

namespace la {

namespace {

using namespace ptx;

#ifdef LA_TRACE
// debug build only: cycle stamps of pipeline events of CTA (0, 0), [chunk][event].  The buffer pointer is
// read once into `la_trp` at kernel entry (a global load per stamp would distort the timeline).
__device__ unsigned long long* g_la_trace = nullptr;
#define LA_TR(t, ev)                                                          \
  do {                                                                        \
    if (la_trp != nullptr && (t) < 32) la_trp[(t) * 32 + (ev)] = clock64(); \
  } while (0)
// per-P-warp stamps: [chunk][p warp][event 0..7] after the 1024 slots above
#define LA_TRP(t, pw_, ev)                                                                          \
  do {                                                                                              \
    if (la_trp != nullptr && (t) < 32 && (threadIdx.x & 31) == 0)                                   \
      la_trp[1024 + ((t) * 8 + (pw_)) * 8 + (ev)] = clock64();                                       \
  } while (0)
#else
#define LA_TR(t, ev) \
  do {               \
  } while (0)
#define LA_TRP(t, pw_, ev) \
  do {                     \
  } while (0)
#endif


constexpr int C = 128;           // chunk rows
constexpr int D = 128;           // head dim (only d == 128 on this backend)
constexpr int TILE = C * D * 2;  // 32 KB bf16 tile
constexpr int HALF = TILE / 2;   // [128 rows][64 cols] = 16 KB, one 128B-swizzle column block
constexpr int NSTAGE = 2;
#ifndef LA_EARLY_STAGES
#define LA_EARLY_STAGES NSTAGE  // ring stages thread 0 loads before the CTA-wide sync
#endif
constexpr int WARP_TMA = 0, WARP_MMA = 1, WARP_P = 2, NUM_P = 8, WARP_O = 10, NUM_O = 8, WARP_KV = 18, NUM_KV = 8;
constexpr int NUM_WARPS = WARP_KV + NUM_KV;
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr uint32_t TM_S0 = 0, TM_O = 256, TM_ST = 384, TM_COLS = 512;

// kind::f16 instruction descriptors (M = N = 128)
constexpr uint32_t IDESC_KK = idesc_bf16(128, 128, 0, 0);    // A K-major, B K-major
constexpr uint32_t IDESC_KMN = idesc_bf16(128, 128, 0, 1);   // A K-major (or TMEM), B MN-major
constexpr uint32_t IDESC_MNMN = idesc_bf16(128, 128, 1, 1);  // A MN-major, B MN-major

constexpr int NSTAGE_MAX = NSTAGE;

struct Bars {
  uint64_t xf_done[NSTAGE_MAX];   // GLA: A / B tiles of the stage transformed in place -> MMA (S), qk store lane
  uint64_t qk_stored[NSTAGE_MAX]; // GLA: the store lane has read the transformed tiles -> B warps (B~ in place)
  uint64_t out_ready[NSTAGE_MAX]; // EPI: the staged output tile transformed in place -> store lane
  uint64_t full[3][NSTAGE_MAX];   // TMA -> consumers, one ring per operand tile A, B, C (tx bytes)
  uint64_t empty[3][NSTAGE_MAX];  // MMA commit after the tile's last reader -> TMA
  uint64_t s_full[2];      // MMA: S[t%2] done                 -> P warps, state warps
  uint64_t a_full[2];      // A~(t) in TMEM                    -> MMA (per buffer: P warps run a chunk ahead)
  uint64_t p_full[2];      // P(t) in TMEM                     -> MMA
  uint64_t x_done;         // MMA: X(t) = A~ state_bf16 done   -> state warps (SMEM state copy reusable)
  uint64_t y_done[2];      // MMA: O(t) done, per S buffer     -> MMA (before S(t+2) reuses the buffer)
  uint64_t o_full;         // MMA: O done                      -> output warps
  uint64_t o_free;         // output warps read O              -> MMA
  uint64_t o_staged[2];    // bf16 O(t) staged in C's slot t%2 -> store lane (per slot: the output warps
                           // may stage a chunk ahead of the store lane)
  uint64_t b_scaled[NSTAGE_MAX];  // B~ in SMEM (per stage: in state-only mode the B warps are gated by
                                 // the TMA only and may run a stage ahead) -> MMA
  uint64_t ds_full;        // MMA: state += B~^T C done        -> state warps
  uint64_t st_ready;       // bf16 state in SMEM, TMEM state pre-scaled -> MMA
  uint32_t tmem_base;
};

constexpr size_t SMEM_TILES = (size_t)NSTAGE * 3 * TILE + TILE;  // 224 KB
constexpr size_t SMEM_BYTES = SMEM_TILES + 1024 /*align slack*/;

struct TcArgs {
  int heads, n, seg_len, nseg, rev;
  int d;  // head dim (64 or 128): features past d are zero (TMA out-of-bounds fill), states are d x d
  const double* lam;
  uint16_t* out;  // bf16 output (full mode)
  const float* state_in;
  int64_t in_bh_stride, in_seg_stride;
  int in_T;
  float* state_out;
  int out_T;
  // GLA mode
  const double* theta;  // LRPE angles [d/2] (nullable: no rotation)
  int act;              // la_act
  int qk_out;           // store the transformed q / k tiles (map_qo / map_ko)
  int64_t offset;       // LRPE position of row 0
  // EPI mode: the pre-activation rows x (bf16, the output's geometry, strides sx)
  const uint16_t* xp;
  Strides3 sx;
};


// byte offset of 16-byte chunk `c` (0..7) of row `r` inside a [128][64] bf16 block, 128B swizzle
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }


// MODE 0: the plain pass.  1 (GLA): the GLA prologue on the A / B tiles (the fused GLA core forward).
// 2 (EPI): the GLA prologue's backward on the output tile, out = act'(x) * R^T pass(a, b, c) with x the
// pre-activation rows args.xp -- the dq pass of the fused GLA core backward, writing dqp instead of dq.
template <int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_pass_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_o,
                   const __grid_constant__ CUtensorMap map_qo, const __grid_constant__ CUtensorMap map_ko,
                   const TcArgs args) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;
  constexpr bool GLA = MODE == 1, EPI = MODE == 2;
  __shared__ float theta_s[GLA || EPI ? D / 2 : 1];     // LRPE angles (fp32: local angles theta_j * i, i < 128)
  __shared__ float2 anchor_s[GLA || EPI ? D / 2 : 1];   // (cos, sin) of theta_j * (chunk row 0 + offset), fp64-reduced
  __shared__ __align__(16) float pw[C + 8];  // lam^0 .. lam^128
  const uint32_t smem = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem - smem_u32(smem_raw));
  constexpr int NS = NSTAGE;  // ring depth
  auto tile_a = [smem](int s) { return smem + (uint32_t)(s * 3 * TILE); };
  auto tile_b = [smem](int s) { return smem + (uint32_t)(s * 3 * TILE + TILE); };
  auto tile_c = [smem](int s) { return smem + (uint32_t)(s * 3 * TILE + 2 * TILE); };
  const uint32_t st_bf16 = smem + (uint32_t)(NSTAGE * 3 * TILE);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef LA_TRACE
  unsigned long long* const la_trp = (blockIdx.x == 0 && blockIdx.y == 0) ? g_la_trace : nullptr;
#endif
  const int bh = blockIdx.y;
  const int bi = bh / args.heads, hi = bh % args.heads;
  const int seg = blockIdx.x;  // CTA = one segment of one (batch, head)
  const int p0 = seg * args.seg_len;
  const int p1 = min(args.n, p0 + args.seg_len);
  const int nchunks = p1 > p0 ? (p1 - p0 + C - 1) / C : 0;
  const int rev = args.rev;
  auto chunk_row0 = [&](int t) { return p0 + (rev ? (nchunks - 1 - t) : t) * C; };
  auto chunk_len = [&](int t) { return min(C, p1 - chunk_row0(t)); };
  const int early = nchunks < LA_EARLY_STAGES ? nchunks : LA_EARLY_STAGES;  // chunks thread 0 loads before the sync

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      for (int x = 0; x < 3; ++x) {
        mbar_init(&bars.full[x][s], 1);
        // GLA with q / k out: A's slot is also released by the store lane once its TMA store read the tile
        mbar_init(&bars.empty[x][s], (GLA && x == 0 && args.qk_out) ? 2 : 1);
      }
      mbar_init(&bars.b_scaled[s], NUM_KV);
      mbar_init(&bars.xf_done[s], NUM_KV);
      mbar_init(&bars.qk_stored[s], 1);
      mbar_init(&bars.out_ready[s], NUM_KV);
    }
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&bars.s_full[s], 1);
      mbar_init(&bars.p_full[s], NUM_P);
      mbar_init(&bars.a_full[s], NUM_P);
      mbar_init(&bars.y_done[s], 1);
    }
    mbar_init(&bars.o_full, 1);
    mbar_init(&bars.o_free, NUM_O);
    mbar_init(&bars.o_staged[0], NUM_O);
    mbar_init(&bars.o_staged[1], NUM_O);
    mbar_init(&bars.ds_full, 1);
    mbar_init(&bars.x_done, 1);
    mbar_init(&bars.st_ready, NUM_KV);
    fence_mbar_init();
  }
  griddep_wait();  // PDL: the previous kernel of the stream has completed (inputs written, outputs free)
  // lam^0 .. lam^C, one power per thread (binary exponentiation in fp64): a serial ladder here held
  // every warp (and the first TMA loads) back by ~130 dependent multiplies
  if (threadIdx.x <= C) {
    const double l = load_decay(args.lam, hi);
    pw[threadIdx.x] = (float)(pow_int(l, (int)threadIdx.x) * (l / l));
  }
  if ((GLA || EPI) && args.theta != nullptr && threadIdx.x >= 160 && threadIdx.x < 160 + D / 2)
    theta_s[threadIdx.x - 160] = (float)args.theta[threadIdx.x - 160];
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    tma_prefetch(&map_c);
    tma_prefetch(&map_o);
    // the first ring stages need no empty-slot wait: start their loads now, before the CTA-wide sync
    // and the TMEM allocation, so the first tiles are in flight during the setup
    for (int t = 0; t < early; ++t)
      for (int x = 0; x < 3; ++x) {
        const CUtensorMap* map = x == 0 ? &map_a : (x == 1 ? &map_b : &map_c);
        mbar_arrive_expect_tx(&bars.full[x][t], TILE);
        uint8_t* g = smem_gen + (t * 3 + x) * TILE;
        tma_load_4d(map, &bars.full[x][t], g, 0, chunk_row0(t), hi, bi);
        tma_load_4d(map, &bars.full[x][t], g + HALF, 64, chunk_row0(t), hi, bi);
      }
  }
  if (warp == WARP_MMA) tmem_alloc(&bars.tmem_base, TM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;


  if (warp == WARP_TMA) {
    // ------------------------------------------------------------ TMA producer
    // Lanes 0/1/2 each run the ring of one operand tile (A, B, C), so a tile is refilled as soon as
    // its own last reader retires: A after X(t), B after the state update, C after Y(t).
    const int x = lane;
    if (x < 3) {
      const CUtensorMap* map = x == 0 ? &map_a : (x == 1 ? &map_b : &map_c);
      for (int t = early; t < nchunks; ++t) {
        const int s = t % NS;
        if (t >= NS) mbar_wait(&bars.empty[x][s], ((t / NS) - 1) & 1);
        const int r0 = chunk_row0(t);
        mbar_arrive_expect_tx(&bars.full[x][s], TILE);
        if (x == 0) LA_TR(t, 0);
        if (x == 1) LA_TR(t, 16);
        if (x == 2) LA_TR(t, 17);
        uint8_t* g = smem_gen + (s * 3 + x) * TILE;
        tma_load_4d(map, &bars.full[x][s], g, 0, r0, hi, bi);
        tma_load_4d(map, &bars.full[x][s], g + HALF, 64, r0, hi, bi);
      }
      if (x == 0) griddep_launch();  // every load of this CTA issued: the next kernel may start its prologue
    } else if (x == 3) {
      // store lane: bf16 O(t) is staged in C(t)'s slot (C's MMA readers are done by then); TMA-store it
      // and hand the slot back to the C ring once the store has read it
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NSTAGE;
        mbar_wait(EPI ? &bars.out_ready[s] : &bars.o_staged[s], (t / NSTAGE) & 1);
        uint8_t* g = smem_gen + (s * 3 + 2) * TILE;
        const int r0 = chunk_row0(t);
        tma_store_4d(&map_o, g, 0, r0, hi, bi);
        tma_store_4d(&map_o, g + HALF, 64, r0, hi, bi);
        tma_store_commit();
        tma_store_wait_read();
        mbar_arrive(&bars.empty[2][s]);
      }
      tma_store_wait_all();
    } else if (GLA && x == 4 && args.qk_out) {
      // q / k lane: TMA-store each transformed A / B tile, then hand A's slot back to its ring and B's
      // tile to the B warps (which scale it in place)
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NSTAGE;
        mbar_wait(&bars.xf_done[s], (t / NSTAGE) & 1);
        const int r0 = chunk_row0(t);
        uint8_t* ga = smem_gen + (s * 3 + 0) * TILE;
        uint8_t* gb = smem_gen + (s * 3 + 1) * TILE;
        tma_store_4d(&map_qo, ga, 0, r0, hi, bi);
        tma_store_4d(&map_qo, ga + HALF, 64, r0, hi, bi);
        tma_store_4d(&map_ko, gb, 0, r0, hi, bi);
        tma_store_4d(&map_ko, gb + HALF, 64, r0, hi, bi);
        tma_store_commit();
        tma_store_wait_read();
        mbar_arrive(&bars.qk_stored[s]);
        mbar_arrive(&bars.empty[0][s]);
      }
      tma_store_wait_all();
    }
  } else if (warp == WARP_MMA) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      auto issue_s = [&](int t) {  // S[t%2] = A B^T  (both K-major)
        const int s = t % NSTAGE;
        const uint32_t a_addr = tile_a(s), b_addr = tile_b(s);
        if (GLA) {
          mbar_wait(&bars.xf_done[s], (t / NSTAGE) & 1);  // the prologue transform (implies the TMA landed)
        } else {
          mbar_wait(&bars.full[0][s], (t / NSTAGE) & 1);
          mbar_wait(&bars.full[1][s], (t / NSTAGE) & 1);
        }
        // S[t%2] overwrites the TMEM columns P(t-2) / A~(t-2) were read from: those TS-MMAs must have
        // retired (in-order issue alone does not order a TMEM A-operand read before a later D write)
        if (t >= 2) mbar_wait(&bars.y_done[t & 1], ((t - 2) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
          mma_bf16_ss(tmem + TM_S0 + (t & 1) * 128, smem_desc_sw128(a_addr + off, 0, 1024),
                      smem_desc_sw128(b_addr + off, 0, 1024), IDESC_KK, kk > 0);
        }
        mma_commit(&bars.s_full[t & 1]);
        LA_TR(t, 1);
      };
      int s_issued = 0;  // S issued for chunks < s_issued
      if (nchunks > 0) {
        issue_s(0);
        s_issued = 1;
      }
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NS;
        const uint32_t b_addr = tile_b(s), c_addr = tile_c(s);
        const uint32_t sbuf = tmem + TM_S0 + (t & 1) * 128;
        if (s_issued == t + 1 && t + 1 < nchunks &&
            (GLA ? mbar_try_wait(smem_u32(&bars.xf_done[(t + 1) % NSTAGE]), ((t + 1) / NSTAGE) & 1)
                 : (mbar_try_wait(smem_u32(&bars.full[0][(t + 1) % NSTAGE]), ((t + 1) / NSTAGE) & 1) &&
                    mbar_try_wait(smem_u32(&bars.full[1][(t + 1) % NSTAGE]), ((t + 1) / NSTAGE) & 1)))) {
          issue_s(t + 1);  // run ahead: S(t+1) as soon as its operands landed
          s_issued = t + 2;
        }
        // st_ready(t): bf16 state_{t-1} in SMEM and the TMEM state pre-scaled by lam^b.  State-only
        // mode folds the decay into B~ instead and accumulates straight onto the zeroed state.
        mbar_wait(&bars.st_ready, t & 1);
        {
          // X(t) = A~ state_{t-1}  -> O (fresh accumulation)
          if (t >= 1) mbar_wait(&bars.o_free, (t - 1) & 1);
          mbar_wait(&bars.a_full[t & 1], (t >> 1) & 1);
          LA_TR(t, 15);
          tc_fence_after();
#ifndef LA_KO_MMAX
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_bf16_ts(tmem + TM_O, sbuf + 64 + kk * 8, smem_desc_sw128(st_bf16 + kk * 2048, HALF, 1024),
                        IDESC_KMN, kk > 0);
#endif
          mma_commit(&bars.x_done);
          mma_commit(&bars.empty[0][s]);  // A's readers (S(t), the A~ build) are done
        }
        // state += B~^T C
        mbar_wait(&bars.b_scaled[s], (t / NS) & 1);
        mbar_wait(&bars.full[2][s], (t / NS) & 1);
        LA_TR(t, 4);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk)
          mma_bf16_ss(tmem + TM_ST, smem_desc_sw128(b_addr + kk * 2048, HALF, 1024),
                      smem_desc_sw128(c_addr + kk * 2048, HALF, 1024), IDESC_MNMN, 1);
        mma_commit(&bars.ds_full);
        mma_commit(&bars.empty[1][s]);  // B's last reader
        LA_TR(t, 5);
        {
          // Y(t) = P C  -> O (accumulate)
          mbar_wait(&bars.p_full[t & 1], (t >> 1) & 1);
          LA_TR(t, 2);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < C / 16; ++kk) {
            // key block cb = kk / 2 lives at column 32 (cb & 1) + 16 (cb >> 1) (see the P warps)
            const int cb = kk >> 1;
            const uint32_t pcol = 32 * (cb & 1) + 16 * (cb >> 1) + 8 * (kk & 1);
            mma_bf16_ts(tmem + TM_O, sbuf + pcol, smem_desc_sw128(c_addr + kk * 2048, HALF, 1024), IDESC_KMN, 1);
          }
          mma_commit(&bars.o_full);
          mma_commit(&bars.y_done[t & 1]);
          LA_TR(t, 3);
        }
        if (s_issued == t + 1 && t + 1 < nchunks) {
          issue_s(t + 1);
          s_issued = t + 2;
        }
      }
      // Drain: every asynchronous tcgen05.commit arrival must land before this CTA retires, or it
      // would hit the barriers of the next CTA scheduled onto this SM's shared memory.
      for (int t = max(0, nchunks - NS); t < nchunks; ++t) {
        for (int x = 0; x < 3; ++x) mbar_wait(&bars.empty[x][t % NS], (t / NS) & 1);
        mbar_wait(&bars.y_done[t & 1], (t >> 1) & 1);
      }
    }
  } else if (warp < WARP_O) {
    // ------------------------------------------------------------ A~ / P conversion (warps 2..9)
    {
      const int quad = warp & 3;
      const int half = (warp - WARP_P) >> 2;  // A~ columns [64 half, +64); key blocks {half, half + 2}
      const int i = quad * 32 + lane;         // chunk row == TMEM lane
      const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
      const uint32_t pw_addr = smem_u32(pw);
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NSTAGE;
        const int b = chunk_len(t);
        const uint32_t sbuf = tmem + lane_off + TM_S0 + (t & 1) * 128;
        mbar_wait(&bars.s_full[t & 1], (t >> 1) & 1);
        if (warp == WARP_P && lane == 0) LA_TR(t, 6);
        LA_TRP(t, warp - WARP_P, 0);
        tc_fence_after();
        // P = bf16(S * M): fwd keeps j <= i with lam^(i-j), rev keeps j >= i with lam^(j-i).
        // A block of 32 keys is all-zero / all-kept / diagonal depending on the warp's quadrant.
        auto convert_block = [&](int cb, uint32_t (&pk)[16]) {
#ifndef LA_KO_PCONV
          const bool zero = rev ? (cb < quad) : (cb > quad);
#else
          const bool zero = true;
#endif
          if (zero) {
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = 0u;
          } else if (cb != quad) {
            // off-diagonal: lam^|i-j| = lam^(|i - block edge|) * lam^(distance within the block);
            // both factors are >= the product, so no spurious underflow
            float v[32];
            tmem_ld32(sbuf + cb * 32, v);
            const float base = rev ? pw[cb * 32 - i] : pw[i - cb * 32 - 31];
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              // w = lam^(31 - jj) (fwd) or lam^jj (rev) for jj = 4q .. 4q+3: one broadcast LDS.128
              const uint4 wq = lds128(pw_addr + 4 * (rev ? 4 * q : 28 - 4 * q));
              float w0 = __uint_as_float(wq.x), w1 = __uint_as_float(wq.y), w2 = __uint_as_float(wq.z),
                    w3 = __uint_as_float(wq.w);
              if (!rev) {  // fwd wants descending powers
                const float t0 = w0, t1 = w1;
                w0 = w3;
                w1 = w2;
                w2 = t1;
                w3 = t0;
              }
              pk[2 * q] = pack_bf16x2(v[4 * q] * (base * w0), v[4 * q + 1] * (base * w1));
              pk[2 * q + 1] = pack_bf16x2(v[4 * q + 2] * (base * w2), v[4 * q + 3] * (base * w3));
            }
          } else {
            // diagonal block: row i = 32 quad + lane, key j = 32 quad + jj, distance |lane - jj| < 32.
            // fwd needs lam^(lane - jj) = (lam^l of lane l - jj): a shuffle-up by the constant jj;
            // rev needs lam^(jj - lane) = (lam^(31-l) of lane l + 31 - jj): a shuffle-down.
            float v[32];
            tmem_ld32(sbuf + cb * 32, v);
            const float own = rev ? pw[31 - lane] : pw[lane];
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; jj += 2) {
              float x0, x1;
              if (!rev) {
                const float f0 = __shfl_up_sync(0xffffffffu, own, jj);
                const float f1 = __shfl_up_sync(0xffffffffu, own, jj + 1);
                x0 = lane >= jj ? v[jj] * f0 : 0.f;
                x1 = lane >= jj + 1 ? v[jj + 1] * f1 : 0.f;
              } else {
                const float f0 = __shfl_down_sync(0xffffffffu, own, 31 - jj);
                const float f1 = __shfl_down_sync(0xffffffffu, own, 30 - jj);
                x0 = lane <= jj ? v[jj] * f0 : 0.f;
                x1 = lane <= jj + 1 ? v[jj + 1] * f1 : 0.f;
              }
              pk[jj >> 1] = pack_bf16x2(x0, x1);
            }
          }
        };
        // TMEM columns of the buffer: S block cb sits at [32 cb, +32).  Warp `half` reads S blocks half
        // and half + 2 and only ever overwrites those: its A~ goes to [64 + 32 half, +32) (= S block
        // half + 2, read first) and its two P blocks to [32 half, +32) (= S block half): P(half) at
        // 32 half, P(half + 2) at 32 half + 16.  The MMA addresses P per key block accordingly.
        uint32_t p_hi[16];
        convert_block(half + 2, p_hi);
        LA_TRP(t, warp - WARP_P, 1);
        // A~ = bf16(out_scale * A): fwd lam^(i+1), rev lam^(b-1-i); this warp's 64 columns
        {
          const float osc = rev ? pw[max(b - 1 - i, 0)] : pw[i + 1];
          const uint32_t osc2 = pack_bf16x2(osc, osc);
          const uint32_t a_addr = tile_a(s) + half * HALF;
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            uint32_t pk[16];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const uint4 x = mul_bf16x2(lds128(a_addr + sw128(i, part * 4 + m)), osc2);
              pk[4 * m + 0] = x.x;
              pk[4 * m + 1] = x.y;
              pk[4 * m + 2] = x.z;
              pk[4 * m + 3] = x.w;
            }
            tmem_st16(sbuf + 64 + half * 32 + part * 16, pk);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars.a_full[t & 1]);
        }
        LA_TRP(t, warp - WARP_P, 2);
        {
          uint32_t p_lo[16];
          convert_block(half, p_lo);
          tmem_st16(sbuf + 32 * half, p_lo);
          tmem_st16(sbuf + 32 * half + 16, p_hi);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[t & 1]);
        if (warp == WARP_P && lane == 0) LA_TR(t, 7);
        LA_TRP(t, warp - WARP_P, 3);
      }
    }
  } else if (warp < WARP_KV) {
    // ------------------------------------------------------------ B scaling + output (warps 10..17)
    const int quad = warp & 3;
    const int hh = (warp - WARP_O) >> 2;  // 64-column half this warp owns (of B and of O)
    const int i = quad * 32 + lane;       // chunk row == TMEM lane
    const uint32_t o_cols = tmem + ((uint32_t)(quad * 32) << 16) + TM_O + hh * 64;
    for (int t = 0; t < nchunks; ++t) {
      const int s = t % NS;
      const int r0 = chunk_row0(t);
      const int b = chunk_len(t);
      mbar_wait(&bars.s_full[t & 1], (t >> 1) & 1);
      if (warp == WARP_O && lane == 0) LA_TR(t, 11);
      if (GLA && args.qk_out) mbar_wait(&bars.qk_stored[s], (t / NS) & 1);  // k's TMA store read B first
      // B~ = in_scale * B, in place once S has consumed B (row i, this warp's 64 columns):
      // fwd lam^(b-1-i), rev lam^(i+1).  Row scaling is order-free, so visit the row's 16-byte chunks in
      // swizzled order: lane i touches physical chunk m ^ (i & 7), spreading a warp over all 32 banks.
      {
        float isc = (i < b) ? (rev ? pw[i + 1] : pw[b - 1 - i]) : 0.f;
#ifdef LA_MUTATE_DKV
        if (rev) isc = -isc;  // fault injection: the reference's `_dkv_step` sign flip (test_kernels.py:249-268)
#endif
        const uint32_t isc2 = pack_bf16x2(isc, isc);
        const uint32_t base = tile_b(s) + hh * HALF + i * 128;
#ifndef LA_KO_BSCALE  // knock-out experiments only (wrong numerics): tools/gpu/ko_power.sh
        uint4 x[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = lds128(base + ((m ^ (i & 7)) << 4));
#pragma unroll
        for (int m = 0; m < 8; ++m) sts128(base + ((m ^ (i & 7)) << 4), mul_bf16x2(x[m], isc2));
#else
        (void)isc2;
        (void)base;
#endif
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.b_scaled[s]);
      if (warp == WARP_O && lane == 0) LA_TR(t, 12);
      // out = bf16(O): TMEM -> registers (then O's columns are released) -> C's SMEM slot -> TMA store
      (void)r0;
      mbar_wait(&bars.o_full, t & 1);
      if (warp == WARP_O && lane == 0) LA_TR(t, 8);
      tc_fence_after();
      uint32_t pk[32];
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        float y[32];
        tmem_ld32(o_cols + cb * 32, y);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[cb * 16 + e] = pack_bf16x2(y[2 * e], y[2 * e + 1]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.o_free);  // O's TMEM is free; the stores proceed from registers
      {
        const uint32_t base = tile_c(s) + hh * HALF;
#ifndef LA_KO_OSTAGE
#pragma unroll
        for (int m = 0; m < 8; ++m)
          sts128(base + sw128(i, m), make_uint4(pk[4 * m], pk[4 * m + 1], pk[4 * m + 2], pk[4 * m + 3]));
#else
        (void)base;
#endif
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.o_staged[s]);
      if (warp == WARP_O && lane == 0) LA_TR(t, 9);
    }
  } else {
    // ------------------------------------------------------------ state (warps 18..25)
    const int quad = warp & 3;
    const int hh = (warp - WARP_KV) >> 2;  // which 64 state columns
    const int i = quad * 32 + lane;        // state row (d_k index) == TMEM lane
    const uint32_t st_cols = tmem + ((uint32_t)(quad * 32) << 16) + TM_ST + hh * 64;
    // publish bf16(state) to SMEM and pre-scale the TMEM state by `next_decay`
    auto publish = [&](const float (&x)[16], int q4, float next_decay) {
      {
        const uint32_t base = st_bf16 + hh * HALF;
        sts128(base + sw128(i, 2 * q4),
               make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                          pack_bf16x2(x[6], x[7])));
        sts128(base + sw128(i, 2 * q4 + 1),
               make_uint4(pack_bf16x2(x[8], x[9]), pack_bf16x2(x[10], x[11]), pack_bf16x2(x[12], x[13]),
                          pack_bf16x2(x[14], x[15])));
      }
      uint32_t w[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = __float_as_uint(x[j] * next_decay);
      tmem_st16(st_cols + q4 * 16, w);
    };
    auto signal_ready = [&]() {
      tmem_st_wait();
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.st_ready);
    };
    // GLA prologue on chunk t's landed A (qp) and B (kp) tiles, in place: row i, this warp's 64 columns
    // (32 feature pairs (2j, 2j+1), j = 32 hh + 4 c + e); rows past n are zeroed
    auto transform = [&](int t) {
      const int s = t % NS;
      const int r0 = chunk_row0(t);
      const bool rot = args.theta != nullptr;
      // the chunk's LRPE anchors cos / sin(theta_j (r0 + offset)), exact (fp64-reduced); row i then adds the
      // local angle theta_j i < 128 rad in fp32 by the angle-addition formula
      if (rot) {
        named_bar_sync(1, NUM_KV * 32);  // the previous chunk's anchors are no longer read
        if (warp == WARP_KV + 4 || warp == WARP_KV + 5) {
          const int j = (warp - WARP_KV - 4) * 32 + lane;
          float c0, s0;
          lrpe_cs(args.theta[j], (int64_t)r0 + args.offset, &c0, &s0);
          anchor_s[j] = make_float2(c0, s0);
        }
        named_bar_sync(1, NUM_KV * 32);
      }
      mbar_wait(&bars.full[0][s], (t / NS) & 1);
      mbar_wait(&bars.full[1][s], (t / NS) & 1);
      const bool valid = r0 + i < p1;
      const uint32_t arow = tile_a(s) + hh * HALF + i * 128, brow = tile_b(s) + hh * HALF + i * 128;
      auto tile = [&](auto act_tag) {
        constexpr int ACT = decltype(act_tag)::value;
#pragma unroll 2
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = (uint32_t)((c ^ (i & 7)) << 4);
          const uint4 xa = lds128(arow + off), xb = lds128(brow + off);
          const uint32_t wa[4] = {xa.x, xa.y, xa.z, xa.w}, wb[4] = {xb.x, xb.y, xb.z, xb.w};
          uint32_t ya[4], yb[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float cs = 1.f, sn = 0.f;
            if (rot) {
              const int j = hh * 32 + 4 * c + e;
              float cl, sl;
              __sincosf(theta_s[j] * (float)i, &sl, &cl);
              const float2 an = anchor_s[j];
              cs = an.x * cl - an.y * sl;
              sn = an.y * cl + an.x * sl;
            }
            ya[e] = gla_pair<ACT>(wa[e], cs, sn, valid);
            yb[e] = gla_pair<ACT>(wb[e], cs, sn, valid);
          }
          sts128(arow + off, make_uint4(ya[0], ya[1], ya[2], ya[3]));
          sts128(brow + off, make_uint4(yb[0], yb[1], yb[2], yb[3]));
        }
      };
      if (args.act == LA_ACT_SWISH) tile(std::integral_constant<int, LA_ACT_SWISH>{});
      else if (args.act == LA_ACT_ONE_PLUS_ELU) tile(std::integral_constant<int, LA_ACT_ONE_PLUS_ELU>{});
      else tile(std::integral_constant<int, LA_ACT_NONE>{});
      fence_proxy_async_smem();  // the tensor core and the TMA store read the tiles next
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.xf_done[s]);
    };
    // EPI: out(t) = act'(x) * R^T out(t) on the tile the output warps staged in C's slot, in place; row i,
    // this warp's 64 columns (pairs j = 32 hh + 4 c + e); x loaded straight from global (one 128-byte row
    // segment per thread)
    uint4 xr[8];  // EPI: x row segment of the chunk to transform next, loaded a chunk ahead of its use
    auto load_x = [&](int t) {
      const int r0 = chunk_row0(t);
      if (r0 + i < p1) {
        const uint4* src = reinterpret_cast<const uint4*>(args.xp + (int64_t)bi * args.sx.b + (int64_t)hi * args.sx.h +
                                                          (int64_t)(r0 + i) * args.sx.n + hh * 64);
#pragma unroll
        for (int c = 0; c < 8; ++c) xr[c] = __ldg(src + c);
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) xr[c] = make_uint4(0, 0, 0, 0);
      }
    };
    auto transform_out = [&](int t) {
      const int s = t % NS;
      const int r0 = chunk_row0(t);
      const bool rot = args.theta != nullptr;
      if (rot) {
        named_bar_sync(1, NUM_KV * 32);
        if (warp == WARP_KV + 4 || warp == WARP_KV + 5) {
          const int j = (warp - WARP_KV - 4) * 32 + lane;
          float c0, s0;
          lrpe_cs(args.theta[j], (int64_t)r0 + args.offset, &c0, &s0);
          anchor_s[j] = make_float2(c0, s0);
        }
        named_bar_sync(1, NUM_KV * 32);
      }
      mbar_wait(&bars.o_staged[s], (t / NS) & 1);
      const uint32_t row = tile_c(s) + hh * HALF;
      auto tile = [&](auto act_tag) {
        constexpr int ACT = decltype(act_tag)::value;
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // fully unrolled: xr stays in registers
          const uint32_t a = row + sw128(i, c);
          const uint4 dy = lds128(a);
          const uint32_t dw[4] = {dy.x, dy.y, dy.z, dy.w}, xw[4] = {xr[c].x, xr[c].y, xr[c].z, xr[c].w};
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float cs = 1.f, sn = 0.f;
            if (rot) {
              const int j = hh * 32 + 4 * c + e;
              float cl, sl;
              __sincosf(theta_s[j] * (float)i, &sl, &cl);
              const float2 an = anchor_s[j];
              cs = an.x * cl - an.y * sl;
              sn = an.y * cl + an.x * sl;
            }
            o[e] = gla_pair_bwd<ACT>(xw[e], dw[e], cs, sn);
          }
          sts128(a, make_uint4(o[0], o[1], o[2], o[3]));
        }
      };
      if (args.act == LA_ACT_SWISH) tile(std::integral_constant<int, LA_ACT_SWISH>{});
      else if (args.act == LA_ACT_ONE_PLUS_ELU) tile(std::integral_constant<int, LA_ACT_ONE_PLUS_ELU>{});
      else tile(std::integral_constant<int, LA_ACT_NONE>{});
      fence_proxy_async_smem();  // the TMA store reads the tile next
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.out_ready[s]);
    };
    if (GLA && nchunks > 0) transform(0);
    if (EPI && nchunks > 0) load_x(0);
    if (nchunks > 0) {
      const float d0 = pw[chunk_len(0)];
#pragma unroll 1
      for (int q4 = 0; q4 < 4; ++q4) {
        float x[16];
        const int dS = args.d, c0 = hh * 64 + q4 * 16;
        if (args.state_in != nullptr && i < dS && c0 < dS) {
          const float* src = args.state_in + (int64_t)bh * args.in_bh_stride + (int64_t)seg * args.in_seg_stride;
          if (args.in_T) {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = src[(c0 + j) * dS + i];  // lanes: consecutive i
          } else {
            // row i, 16 consecutive columns: four 16-byte loads (the state buffers are 16-byte aligned)
            const float4* s4 = reinterpret_cast<const float4*>(src + i * dS + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 w = s4[j];
              x[4 * j] = w.x, x[4 * j + 1] = w.y, x[4 * j + 2] = w.z, x[4 * j + 3] = w.w;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) x[j] = 0.f;
        }
        publish(x, q4, d0);
      }
      signal_ready();
    }
    for (int t = 0; t < nchunks; ++t) {
      // the tensor core accumulated this chunk: read the state, publish it for chunk t+1 once X(t)
      // has finished reading the previous bf16 copy
      if (GLA && t + 1 < nchunks) transform(t + 1);  // overlaps chunk t's products
      mbar_wait(&bars.ds_full, t & 1);
      mbar_wait(&bars.x_done, t & 1);
      if (warp == WARP_KV && lane == 0) LA_TR(t, 13);
      tc_fence_after();
      if (t + 1 < nchunks) {
        const float next_decay = pw[chunk_len(t + 1)];
#pragma unroll 1
        for (int q4 = 0; q4 < 4; ++q4) {
          float x[16];
          tmem_ld16(st_cols + q4 * 16, x);
          tmem_ld_wait();
          publish(x, q4, next_decay);
        }
        signal_ready();
      }
      if (warp == WARP_KV && lane == 0) LA_TR(t, 14);
      if (EPI) {
        transform_out(t);
        if (t + 1 < nchunks) load_x(t + 1);  // in flight while the next chunk's products run
      }
    }
    if (nchunks > 0 && args.state_out != nullptr && (rev ? seg == 0 : seg == args.nseg - 1)) {
      // the pass's final state F(n) / R(0): kv_out / dkv_out
      const int dS = args.d;
      float* dst = args.state_out + (int64_t)bh * dS * dS;
      const int T = args.out_T;
      {
#pragma unroll 1
        for (int q4 = 0; q4 < 4; ++q4) {
          float x[16];
          tmem_ld16(st_cols + q4 * 16, x);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = hh * 64 + q4 * 16 + j;
            if (i < dS && col < dS) dst[T ? (col * dS + i) : (i * dS + col)] = x[j];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem, TM_COLS);
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // resolved once (a function-local static is initialised thread-safely), at the CUDA 12.0 ABI
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

thread_local char g_detail[256];

}  // namespace

#ifndef LA_L2_PROMO
#define LA_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

bool tc_make_map(CUtensorMap* map, const void* base, const PassDesc& p, const Strides3& s, int box_rows) {
  auto enc = encode_fn();
  if (enc == nullptr) {
    snprintf(g_detail, sizeof(g_detail), "cuTensorMapEncodeTiled entry point unavailable");
    return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)p.d, (cuuint64_t)p.n, (cuuint64_t)p.heads, (cuuint64_t)p.batch};
  cuuint64_t strides[3] = {(cuuint64_t)s.n * 2, (cuuint64_t)s.h * 2, (cuuint64_t)s.b * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  // degenerate strides of size-1 dims must still be valid multiples of 16
  if (p.heads == 1) strides[1] = strides[0] * (cuuint64_t)p.n;
  if (p.batch == 1) strides[2] = strides[1] * (cuuint64_t)p.heads;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)LA_L2_PROMO,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    snprintf(g_detail, sizeof(g_detail), "cuTensorMapEncodeTiled failed (CUresult %d) base=%p dims=%llu,%llu,%llu,%llu "
             "strides=%llu,%llu,%llu", (int)r, base, (unsigned long long)dims[0], (unsigned long long)dims[1],
             (unsigned long long)dims[2], (unsigned long long)dims[3], (unsigned long long)strides[0],
             (unsigned long long)strides[1], (unsigned long long)strides[2]);
  return r == CUDA_SUCCESS;
}

namespace {

// gla: nullptr for the plain pass; else the GLA-mode prologue parameters and the q / k out maps
cudaError_t launch_tc(const PassDesc& p, cudaStream_t st, const GlaPrologue* gla = nullptr,
                      const GlaEpilogue* epi = nullptr) {
  CUtensorMap ma, mb, mc, mo, mqo, mko;
  std::memset(&ma, 0, sizeof(ma));
  std::memset(&mo, 0, sizeof(mo));
  std::memset(&mqo, 0, sizeof(mqo));
  std::memset(&mko, 0, sizeof(mko));
  if (!tc_make_map(&mb, p.b, p, p.sbb) || !tc_make_map(&mc, p.c, p, p.sc)) return cudaErrorInvalidValue;
  if (!tc_make_map(&ma, p.a, p, p.sa) || !tc_make_map(&mo, p.out, p, p.so)) return cudaErrorInvalidValue;
  TcArgs a;
  std::memset(&a, 0, sizeof(a));
  a.out = reinterpret_cast<uint16_t*>(p.out);
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
  const size_t smem_bytes = SMEM_BYTES;
  dim3 grid(p.nseg, p.batch * p.heads);
  if (epi != nullptr) {
    a.theta = epi->theta;
    a.act = epi->act;
    a.offset = epi->offset;
    a.xp = reinterpret_cast<const uint16_t*>(epi->xp);
    a.sx = epi->sx;
    static std::atomic<bool> smem_set_epi[64] = {};
    cudaError_t err = set_smem_once(tc_pass_kernel<2>, (int)smem_bytes, smem_set_epi);
    if (err != cudaSuccess) return err;
    return launch_pdl(tc_pass_kernel<2>, grid, dim3(NUM_THREADS), smem_bytes, st, ma, mb, mc, mo, mqo, mko, a);
  }
  if (gla == nullptr) {
    static std::atomic<bool> smem_set[64] = {};
    cudaError_t err = set_smem_once(tc_pass_kernel<0>, (int)smem_bytes, smem_set);
    if (err != cudaSuccess) return err;
    return launch_pdl(tc_pass_kernel<0>, grid, dim3(NUM_THREADS), smem_bytes, st, ma, mb, mc, mo, mqo, mko, a);
  }
  a.theta = gla->theta;
  a.act = gla->act;
  a.offset = gla->offset;
  a.qk_out = gla->q_out != nullptr;
  if (a.qk_out && (!tc_make_map(&mqo, gla->q_out, p, p.sa) || !tc_make_map(&mko, gla->k_out, p, p.sbb)))
    return cudaErrorInvalidValue;
  static std::atomic<bool> smem_set_gla[64] = {};
  cudaError_t err = set_smem_once(tc_pass_kernel<1>, (int)smem_bytes, smem_set_gla);
  if (err != cudaSuccess) return err;
  return launch_pdl(tc_pass_kernel<1>, grid, dim3(NUM_THREADS), smem_bytes, st, ma, mb, mc, mo, mqo, mko, a);
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

}  // namespace

const char* tc_detail() { return g_detail; }

#ifdef LA_TRACE
extern "C" __attribute__((visibility("default"))) int la_debug_set_trace(void* dev_ptr) {
  return (int)cudaMemcpyToSymbol(g_la_trace, &dev_ptr, sizeof(dev_ptr));
}
void la_debug_set_trace_bwd(void* dev_ptr);
extern "C" __attribute__((visibility("default"))) int la_debug_set_trace_bwd_c(void* dev_ptr) {
  la_debug_set_trace_bwd(dev_ptr);
  return (int)cudaGetLastError();
}
#endif

bool tc_supported(int dtype, int d, const int64_t* strides, int count) {
  // d < 128 runs the d = 128 kernels on zero-padded features: the TMA boxes past d read zeros and stores past
  // d are clipped, states are d x d
  if (dtype != LA_BF16 || d < 32 || d > D || d % 32 != 0) return false;
  for (int i = 0; i < 3 * count; ++i)
    if ((strides[i] * 2) % 16 != 0) return false;
  return true;
}

bool tc_pointers_ok(const PassDesc& p) {
  return aligned16(p.b) && aligned16(p.c) && (p.a == nullptr || aligned16(p.a)) &&
         (p.out == nullptr || aligned16(p.out));
}

// Segment count: when batch*heads fill >= 60% of the SMs, no split (a split costs a summary pass over
// two operands); otherwise the largest count that keeps all CTAs in ONE wave, which measured best on
// B200 at every long-n bench shape (profiles/r01_seg_sweep.txt: multi-wave splits lose to per-CTA
// pipeline fill and partial last waves).  Segments keep >= 2 chunks; the workspace is sized for the
// one-wave cap so it does not depend on n.  `sms` = the device's SM count (device_sms()).
Plan tc_plan(int64_t bh, int64_t n, int d, int64_t want_segments, int sms) {
  (void)d;
  if (sms < 1) sms = kNumSMs;
  if (want_segments > 0) {
    Plan p = make_plan(bh, n, C, want_segments, sms, 1);
    p.nsub_ws = (int)(4 * std::max<int64_t>(p.nseg_ws, sms / bh) + 4);
    plan_subsegments(p, bh, 2 * sms, 2, p.nsub_ws);
    return p;
  }
  const int64_t nchunks = (n + C - 1) / C;
  const int64_t cap = std::max<int64_t>(1, sms / bh);
  int64_t nseg = 1;
  if (bh * 10 < (int64_t)sms * 6) nseg = std::min<int64_t>(cap, std::max<int64_t>(1, nchunks / 2));
  Plan p = make_plan(bh, n, C, nseg, sms, 1);
  p.nseg_ws = (int)cap;
  p.nsub_ws = (int)(4 * cap + 4);
  // summaries: one wave of the two-CTAs-per-SM summary kernel over the segments a scan needs,
  // sub-segments of >= 2 chunks
  plan_subsegments(p, bh, 2 * sms, 2, p.nsub_ws);
  return p;
}

cudaError_t tc_launch(const PassDesc& p, bool state_only, cudaStream_t st) {
  // summaries: the lean two-CTAs-per-SM kernel of la_summary.cu
  return state_only ? tc_summary_launch(p, st) : launch_tc(p, st);
}

cudaError_t tc_epi_launch(const PassDesc& p, const GlaEpilogue& epi, cudaStream_t st) {
  if (!tc_pointers_ok(p) || (reinterpret_cast<uintptr_t>(epi.xp) & 15)) return cudaErrorMisalignedAddress;
  return launch_tc(p, st, nullptr, &epi);
}

cudaError_t tc_gla_fwd_launch(const PassDesc& p, const GlaPrologue& gla, cudaStream_t st) {
  if (p.rev) return cudaErrorInvalidValue;  // the prologue belongs to the forward
  return launch_tc(p, st, &gla);
}

}  // namespace la
