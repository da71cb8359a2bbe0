// la_tc_bwd.cu -- the fused reverse sweep of the backward (kernels.py:320-333) on tcgen05:
// dK and dV of one (batch, head, segment) in ONE pass over Q, K, V, dO.
//
// The two reverse passes of la_api.cu's backward,
//     dv = rev(a=k, b=q, c=do)   state dkv   = sum lam.. q do^T
//     dk = rev(a=v, b=do, c=q)   state dkv^T,
// carry the same adjoint state (kernels.py:331-333), so one sweep reads each
// operand once (4 rows in, 2 out per position instead of 3+1 twice), updates
// the state once, and uses one bf16 copy of it for both inter-chunk products:
// as an MN-major B operand for dV and as a K-major one for dK.  Per chunk:
//
//   Sv = K Q^T, Sk = V dO^T           SS-MMAs -> TMEM SV, SK
//   Pv, Pk, K~ = osc K, V~ = osc V    P warps (rev mask lam^(j-i), osc = lam^(b-1-i)), into SV / SK
//   W = in_scale dO  (lam^(i+1))      BO warps, into K's slot once Sv and K~ consumed K
//   state = lam^b state + Q^T W       SS-MMA into the pre-scaled fp32 TMEM state
//   dV = K~ state + Pv dO             TS-MMAs -> TMEM O -> SMEM (dO's slot) -> TMA store
//   dK = V~ state^T + Pk Q            TS-MMAs -> TMEM O -> SMEM (Q's slot)  -> TMA store
//
// SMEM: Q and dO double-slotted, K and V single-slotted (they are consumed first in a
// chunk, so their refill overlaps the rest of it; the tile after each refill is prefetched
// into L2 so the next refill sees L2 latency), bf16 state: 7 x 32 KB = 224 KB.
// TMEM: SV | SK | O | state = 512 columns.  Warp roles as in la_tc.cu (26 warps).
#include <cudaTypedefs.h>

#include <cstring>
#include <type_traits>

#include "la_common.cuh"
#include "la_ptx.cuh"
#include "la_tc.cuh"

namespace la {

namespace {

using namespace ptx;

#ifndef LA_PFKV_DIST
#define LA_PFKV_DIST 1  // chunks ahead
#endif
#ifndef LA_POLL_NS
#define LA_POLL_NS 0  // back-off of the polling producer when no ring advanced (0: spin)
#endif
#ifndef LA_PFKV
#define LA_PFKV 1  // L2 prefetch of the next K and V tiles (+1.2% on the bench sweep, same-box A/B)
#endif

#ifdef LA_TRACE
// debug build only: cycle stamps of CTA (0, 0), [chunk][event] (tests/tc_trace_bwd.py)
__device__ unsigned long long* g_la_trace_bwd = nullptr;
#define LB_TR(t, ev)                                                         \
  do {                                                                       \
    if (lb_trp != nullptr && (t) < 32) lb_trp[(t) * 32 + (ev)] = clock64(); \
  } while (0)
#else
#define LB_TR(t, ev) \
  do {               \
  } while (0)
#endif

constexpr int C = 128;
constexpr int D = 128;
constexpr int TILE = C * D * 2;
constexpr int HALF = TILE / 2;
constexpr int WARP_TMA = 0, WARP_MMA = 1, WARP_P = 2, NUM_P = 8, WARP_O = 10, NUM_O = 8, WARP_KV = 18, NUM_KV = 8;
constexpr int NUM_WARPS = WARP_KV + NUM_KV;
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr uint32_t TM_SV = 0, TM_SK = 128, TM_O = 256, TM_ST = 384, TM_COLS = 512;

constexpr uint32_t IDESC_KK = idesc_bf16(128, 128, 0, 0);
constexpr uint32_t IDESC_KMN = idesc_bf16(128, 128, 0, 1);
constexpr uint32_t IDESC_MNMN = idesc_bf16(128, 128, 1, 1);

// SMEM slots (32 KB each): Q0 Q1 D0 D1 K V STATE
constexpr int SLOT_Q = 0, SLOT_D = 2, SLOT_K = 4, SLOT_V = 5, SLOT_ST = 6;
constexpr size_t SMEM_BYTES = 7 * (size_t)TILE + 1024;

struct Bars {
  uint64_t full_q[2], empty_q[2], full_d[2], empty_d[2];
  uint64_t full_k, empty_k, full_v, empty_v;
  uint64_t sv_full, sk_full;   // MMA: Sv / Sk done
  uint64_t av_full, pv_full;   // P warps: K~, Pv in TMEM
  uint64_t ak_full, pk_full;   // P warps: V~, Pk in TMEM
  uint64_t w_ready;            // BO warps: W = in_scale dO in K's slot
  uint64_t ds_full;            // MMA: state += Q^T W done
  uint64_t x_done;             // MMA: both inter-chunk products read the bf16 state copy
  uint64_t ov_full, ok_full;   // MMA: O holds dV / dK
  uint64_t o_free;             // BO warps read O (two phases per chunk: dV then dK)
  uint64_t dv_staged[2], dk_staged[2];  // BO warps: bf16 dV / dK staged in slot t%2 -> store lane
                                        // (per slot: the BO warps may stage a chunk ahead of the store lane)
  uint64_t st_scaled, st_pub;  // state warps: TMEM state pre-scaled / bf16 copy published
  uint64_t dk_ready[2];        // EPI: the staged dK tile turned into dkp in place by the state warps -> store lane
  uint32_t tmem_base;
};

struct BwdArgs {
  int heads, n, seg_len, nseg;
  int d;  // head dim (64 or 128): features past d are zero (TMA out-of-bounds fill), states are d x d
  const double* lam;
  const float* state_in;  // entering adjoint state (dkv orientation), nullable
  int64_t in_bh_stride, in_seg_stride;
  float* state_out;       // dkv_out (R(0)), written by segment 0
  // EPI mode (the fused GLA core backward): dK -> dkp = act'(kp) * R^T dK before the store
  const uint16_t* xp;
  Strides3 sx;
  const double* theta;
  int act;
  int64_t offset;
};

__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

template <bool EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_dkdv_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                   const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do,
                   const __grid_constant__ CUtensorMap map_dk, const __grid_constant__ CUtensorMap map_dv,
                   const BwdArgs args) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Bars bars;
  __shared__ __align__(16) float pw[C + 8];
  __shared__ float theta_s[EPI ? D / 2 : 1];
  __shared__ float2 anchor_s[EPI ? D / 2 : 1];
  const uint32_t smem = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem - smem_u32(smem_raw));
  auto slot = [smem](int i) { return smem + (uint32_t)(i * TILE); };
  auto slot_gen = [smem_gen](int i) { return smem_gen + (size_t)i * TILE; };
  const uint32_t st_bf16 = slot(SLOT_ST);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef LA_TRACE
  unsigned long long* const lb_trp = (blockIdx.x == 0 && blockIdx.y == 0) ? g_la_trace_bwd : nullptr;
#endif
  const int seg = blockIdx.x, bh = blockIdx.y;
  const int bi = bh / args.heads, hi = bh % args.heads;
  const int p0 = seg * args.seg_len;
  const int p1 = min(args.n, p0 + args.seg_len);
  const int nchunks = (p1 - p0 + C - 1) / C;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.full_q[s], 1);
      mbar_init(&bars.empty_q[s], 1);
      mbar_init(&bars.full_d[s], 1);
      mbar_init(&bars.empty_d[s], 1);
    }
    mbar_init(&bars.full_k, 1);
    mbar_init(&bars.empty_k, 1);
    mbar_init(&bars.full_v, 1);
    mbar_init(&bars.empty_v, 1);
    mbar_init(&bars.sv_full, 1);
    mbar_init(&bars.sk_full, 1);
    mbar_init(&bars.av_full, NUM_P);
    mbar_init(&bars.pv_full, NUM_P);
    mbar_init(&bars.ak_full, NUM_P);
    mbar_init(&bars.pk_full, NUM_P);
    mbar_init(&bars.w_ready, NUM_O);
    mbar_init(&bars.ds_full, 1);
    mbar_init(&bars.x_done, 1);
    mbar_init(&bars.ov_full, 1);
    mbar_init(&bars.ok_full, 1);
    mbar_init(&bars.o_free, NUM_O);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.dv_staged[s], NUM_O);
      mbar_init(&bars.dk_staged[s], NUM_O);
    }
    mbar_init(&bars.st_scaled, NUM_KV);
    mbar_init(&bars.st_pub, NUM_KV);
    mbar_init(&bars.dk_ready[0], NUM_KV);
    mbar_init(&bars.dk_ready[1], NUM_KV);
    fence_mbar_init();
  }
  griddep_wait();  // PDL: the previous kernel of the stream has completed (inputs written, outputs free)
  // lam^0 .. lam^C, one power per thread (binary exponentiation in fp64): a serial ladder here held
  // every warp (and the first TMA loads) back by ~130 dependent multiplies
  if (threadIdx.x <= C) {
    const double l = load_decay(args.lam, hi);
    pw[threadIdx.x] = (float)(pow_int(l, (int)threadIdx.x) * (l / l));
  }
  if (EPI && args.theta != nullptr && threadIdx.x >= 160 && threadIdx.x < 160 + D / 2)
    theta_s[threadIdx.x - 160] = (float)args.theta[threadIdx.x - 160];
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    tma_prefetch(&map_do);
    tma_prefetch(&map_dk);
    tma_prefetch(&map_dv);
  }
  // reverse sweep: chunk t covers rows [row0(t), row0(t) + len(t))
  auto chunk_row0 = [&](int t) { return p0 + (nchunks - 1 - t) * C; };
  auto chunk_len = [&](int t) { return min(C, p1 - chunk_row0(t)); };
  // the rings' first stage needs no empty-slot wait: thread 0 (the producer lane) starts chunk 0's loads
  // before the CTA-wide sync and the TMEM allocation (+0.3% on the short-n sweep; also starting Q's and
  // dO's second stage here lost 1.2%: it queues ahead of chunk 1's K / V)
  const int early_qd = nchunks < 1 ? nchunks : 1, early_kv = early_qd;
  if (threadIdx.x == 0) {
    const CUtensorMap* maps[4] = {&map_q, &map_do, &map_k, &map_v};
    for (int r = 0; r < 4; ++r)
      for (int t = 0; t < (r < 2 ? early_qd : early_kv); ++t) {
        uint64_t* full = r == 0 ? &bars.full_q[t] : r == 1 ? &bars.full_d[t] : r == 2 ? &bars.full_k : &bars.full_v;
        uint8_t* g = slot_gen(r == 0 ? SLOT_Q + t : r == 1 ? SLOT_D + t : r == 2 ? SLOT_K : SLOT_V);
        mbar_arrive_expect_tx(full, TILE);
        tma_load_4d(maps[r], full, g, 0, chunk_row0(t), hi, bi);
        tma_load_4d(maps[r], full, g + HALF, 64, chunk_row0(t), hi, bi);
#if LA_PFKV
        for (int u = t + 1; r >= 2 && u <= t + LA_PFKV_DIST && u < nchunks; ++u) {
          tma_prefetch_l2_4d(maps[r], 0, chunk_row0(u), hi, bi);
          tma_prefetch_l2_4d(maps[r], 64, chunk_row0(u), hi, bi);
        }
#endif
      }
  }
  if (warp == WARP_MMA) tmem_alloc(&bars.tmem_base, TM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  // W = in_scale dO into K's slot (row i: lam^(i+1), rows past the tail 0), once Sv and K~ are done with K;
  // the B/O warps run it (thread -> row i, 64-column half hh).  (Moving it to the state warps, idle at
  // that point, measured no faster: the pass is bound by shared-memory traffic, not by who issues it.)
  auto build_w = [&](int t, int i, int hh) {
    const int s = t & 1;
    const int b = chunk_len(t);
    mbar_wait(&bars.full_d[s], (t >> 1) & 1);
    mbar_wait(&bars.av_full, t & 1);
#ifndef LA_MUTATE_DKV
    const float isc = i < b ? pw[i + 1] : 0.f;
#else
    const float isc = i < b ? -pw[i + 1] : 0.f;  // fault injection: `_dkv_step` sign flip (test_kernels.py:249-268)
#endif
    const uint32_t isc2 = pack_bf16x2(isc, isc);
    const uint32_t src = slot(SLOT_D + s) + hh * HALF + i * 128;
    const uint32_t dst = slot(SLOT_K) + hh * HALF + i * 128;
    uint4 x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = lds128(src + ((m ^ (i & 7)) << 4));
#pragma unroll
    for (int m = 0; m < 8; ++m) sts128(dst + ((m ^ (i & 7)) << 4), mul_bf16x2(x[m], isc2));
    fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&bars.w_ready);
  };

  if (warp == WARP_TMA) {
    // ------------------------------------------------------------ producers (lanes 0-3) + store lane (4)
    if (lane == 0) {
      // One lane serves all four rings from a polling loop, each ring advancing as soon as ITS slot is
      // free.  (Four lanes running one shared loop reconverge every iteration, so the slowest ring's
      // release gated the loads of the other three.)
      const CUtensorMap* maps[4] = {&map_q, &map_do, &map_k, &map_v};
      int next[4] = {early_qd, early_qd, early_kv, early_kv};
      long long t0 = 0;
      for (uint32_t spins = 1; next[0] < nchunks || next[1] < nchunks || next[2] < nchunks || next[3] < nchunks;
           ++spins) {
#if LA_POLL_NS > 0
        const int issued_before = next[0] + next[1] + next[2] + next[3];
#endif
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int t = next[r];
          if (t >= nchunks) continue;
          const int nslot = r < 2 ? 2 : 1;
          const int s = nslot == 2 ? (t & 1) : 0;
          uint64_t* full = r == 0 ? &bars.full_q[s] : r == 1 ? &bars.full_d[s] : r == 2 ? &bars.full_k : &bars.full_v;
          uint64_t* empty = r == 0 ? &bars.empty_q[s] : r == 1 ? &bars.empty_d[s] : r == 2 ? &bars.empty_k
                                                                                            : &bars.empty_v;
          if (t >= nslot && !mbar_test(smem_u32(empty), ((t / nslot) - 1) & 1)) continue;
          LB_TR(t, r);
          const int r0 = chunk_row0(t);
          mbar_arrive_expect_tx(full, TILE);
          uint8_t* g = slot_gen(r == 0 ? SLOT_Q + s : r == 1 ? SLOT_D + s : r == 2 ? SLOT_K : SLOT_V);
          tma_load_4d(maps[r], full, g, 0, r0, hi, bi);
          tma_load_4d(maps[r], full, g + HALF, 64, r0, hi, bi);
#if LA_PFKV
          // K and V are single-slotted: their next tile can only be loaded once this chunk has consumed
          // the slot, so warm L2 with it now and the later load sees L2 latency, not DRAM latency
          if (r >= 2 && t + LA_PFKV_DIST < nchunks) {
            tma_prefetch_l2_4d(maps[r], 0, chunk_row0(t + LA_PFKV_DIST), hi, bi);
            tma_prefetch_l2_4d(maps[r], 64, chunk_row0(t + LA_PFKV_DIST), hi, bi);
          }
#endif
          next[r] = t + 1;
        }
#if LA_POLL_NS > 0
        if (next[0] + next[1] + next[2] + next[3] == issued_before) __nanosleep(LA_POLL_NS);  // nothing free yet
#endif
        if ((spins & 0xFFFFF) == 0) {  // watchdog, as mbar_wait
          if (t0 == 0) t0 = clock64();
          else if (clock64() - t0 > 40000000000LL) __trap();
        }
      }
      griddep_launch();  // every load of this CTA issued: the next kernel may start its prologue
    } else if (lane == 4) {
      for (int t = 0; t < nchunks; ++t) {
        const int s = t & 1;
        const int r0 = chunk_row0(t);
        mbar_wait(&bars.dv_staged[s], (t >> 1) & 1);
        tma_store_4d(&map_dv, slot_gen(SLOT_D + s), 0, r0, hi, bi);
        tma_store_4d(&map_dv, slot_gen(SLOT_D + s) + HALF, 64, r0, hi, bi);
        tma_store_commit();
        LB_TR(t, 20);
        if (EPI) {  // dK waits for the state warps' transform: hand dO's slot back as soon as dV's store read it
          tma_store_wait_read();
          mbar_arrive(&bars.empty_d[s]);
        }
        mbar_wait(EPI ? &bars.dk_ready[s] : &bars.dk_staged[s], (t >> 1) & 1);
        tma_store_4d(&map_dk, slot_gen(SLOT_Q + s), 0, r0, hi, bi);
        tma_store_4d(&map_dk, slot_gen(SLOT_Q + s) + HALF, 64, r0, hi, bi);
        tma_store_commit();
        tma_store_wait_read();
        LB_TR(t, 21);
        if (!EPI) mbar_arrive(&bars.empty_d[s]);
        mbar_arrive(&bars.empty_q[s]);
      }
      tma_store_wait_all();
    }
  } else if (warp == WARP_MMA) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      for (int t = 0; t < nchunks; ++t) {
        const int s = t & 1;
        const uint32_t q_addr = slot(SLOT_Q + s), d_addr = slot(SLOT_D + s);
        const uint32_t k_addr = slot(SLOT_K), v_addr = slot(SLOT_V);
        // Sv = K Q^T (SV's previous P/K~ consumed by dV(t-1))
        mbar_wait(&bars.full_q[s], (t >> 1) & 1);
        LB_TR(t, 24);
        mbar_wait(&bars.full_k, t & 1);
        LB_TR(t, 22);
        if (t >= 1) mbar_wait(&bars.ov_full, (t - 1) & 1);
        LB_TR(t, 23);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
          mma_bf16_ss(tmem + TM_SV, smem_desc_sw128(k_addr + off, 0, 1024), smem_desc_sw128(q_addr + off, 0, 1024),
                      IDESC_KK, kk > 0);
        }
        mma_commit(&bars.sv_full);
        LB_TR(t, 4);
        // Sk = V dO^T
        mbar_wait(&bars.full_d[s], (t >> 1) & 1);
        mbar_wait(&bars.full_v, t & 1);
        if (t >= 1) mbar_wait(&bars.ok_full, (t - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
          mma_bf16_ss(tmem + TM_SK, smem_desc_sw128(v_addr + off, 0, 1024), smem_desc_sw128(d_addr + off, 0, 1024),
                      IDESC_KK, kk > 0);
        }
        mma_commit(&bars.sk_full);
        LB_TR(t, 5);
        // state += Q^T W  (A = Q^T: MN-major Q tile; B = W in K's slot, MN-major)
        mbar_wait(&bars.st_scaled, t & 1);
        mbar_wait(&bars.w_ready, t & 1);
        LB_TR(t, 6);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk)
          mma_bf16_ss(tmem + TM_ST, smem_desc_sw128(q_addr + kk * 2048, HALF, 1024),
                      smem_desc_sw128(k_addr + kk * 2048, HALF, 1024), IDESC_MNMN, 1);
        mma_commit(&bars.ds_full);
        mma_commit(&bars.empty_k);  // K's slot: Sv, K~ and W all consumed
        // dV = K~ state + Pv dO
        mbar_wait(&bars.st_pub, t & 1);
        if (t >= 1) mbar_wait(&bars.o_free, (2 * t - 1) & 1);
        mbar_wait(&bars.av_full, t & 1);
        LB_TR(t, 7);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16_ts(tmem + TM_O, tmem + TM_SV + 64 + kk * 8, smem_desc_sw128(st_bf16 + kk * 2048, HALF, 1024),
                      IDESC_KMN, kk > 0);
        mbar_wait(&bars.pv_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk) {
          const int cb = kk >> 1;
          const uint32_t pcol = 32 * (cb & 1) + 16 * (cb >> 1) + 8 * (kk & 1);
          mma_bf16_ts(tmem + TM_O, tmem + TM_SV + pcol, smem_desc_sw128(d_addr + kk * 2048, HALF, 1024), IDESC_KMN,
                      1);
        }
        mma_commit(&bars.ov_full);
        LB_TR(t, 8);
        // dK = V~ state^T + Pk Q  (state^T = the same bf16 copy read K-major)
        mbar_wait(&bars.o_free, (2 * t) & 1);
        mbar_wait(&bars.ak_full, t & 1);
        LB_TR(t, 9);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
          mma_bf16_ts(tmem + TM_O, tmem + TM_SK + 64 + kk * 8, smem_desc_sw128(st_bf16 + off, 0, 1024), IDESC_KK,
                      kk > 0);
        }
        mma_commit(&bars.x_done);
        mma_commit(&bars.empty_v);  // V's slot: Sk and V~ consumed
        mbar_wait(&bars.pk_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk) {
          const int cb = kk >> 1;
          const uint32_t pcol = 32 * (cb & 1) + 16 * (cb >> 1) + 8 * (kk & 1);
          mma_bf16_ts(tmem + TM_O, tmem + TM_SK + pcol, smem_desc_sw128(q_addr + kk * 2048, HALF, 1024), IDESC_KMN,
                      1);
        }
        mma_commit(&bars.ok_full);
        LB_TR(t, 10);
      }
      // drain every asynchronous commit before the CTA retires
      if (nchunks > 0) {
        const int t = nchunks - 1;
        mbar_wait(&bars.empty_k, t & 1);
        mbar_wait(&bars.empty_v, t & 1);
        mbar_wait(&bars.ok_full, t & 1);
        mbar_wait(&bars.x_done, t & 1);
        mbar_wait(&bars.ds_full, t & 1);
      if (warp == WARP_KV && lane == 0) LB_TR(t, 18);
      }
    }
  } else if (warp < WARP_O) {
    // ------------------------------------------------------------ P / K~ / V~ conversion (warps 2..9)
    const int quad = warp & 3;
    const int half = (warp - WARP_P) >> 2;
    const int i = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t pw_addr = smem_u32(pw);
    // reverse mask: keep j >= i with lam^(j-i)
    auto convert_block = [&](uint32_t sbuf, int cb, uint32_t (&pk)[16]) {
      if (cb < quad) {
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = 0u;
      } else if (cb != quad) {
        float v[32];
        tmem_ld32(sbuf + cb * 32, v);
        const float base = pw[cb * 32 - i];
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 wq = lds128(pw_addr + 16 * q);  // lam^(4q .. 4q+3)
          pk[2 * q] = pack_bf16x2(v[4 * q] * (base * __uint_as_float(wq.x)),
                                  v[4 * q + 1] * (base * __uint_as_float(wq.y)));
          pk[2 * q + 1] = pack_bf16x2(v[4 * q + 2] * (base * __uint_as_float(wq.z)),
                                      v[4 * q + 3] * (base * __uint_as_float(wq.w)));
        }
      } else {
        float v[32];
        tmem_ld32(sbuf + cb * 32, v);
        const float own = pw[31 - lane];
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
          const float f0 = __shfl_down_sync(0xffffffffu, own, 31 - jj);
          const float f1 = __shfl_down_sync(0xffffffffu, own, 30 - jj);
          pk[jj >> 1] = pack_bf16x2(lane <= jj ? v[jj] * f0 : 0.f, lane <= jj + 1 ? v[jj + 1] * f1 : 0.f);
        }
      }
    };
    // one score buffer: S block (half + 2) first (its columns then take this warp's X~ half), then the
    // two P blocks into S block `half`'s columns -- a warp only overwrites columns it has read
    auto convert = [&](uint32_t tm_s, uint32_t x_addr, float osc, uint64_t* a_bar, uint64_t* p_bar) {
      const uint32_t sbuf = tmem + lane_off + tm_s;
      uint32_t p_hi[16];
      convert_block(sbuf, half + 2, p_hi);
      {
        const uint32_t osc2 = pack_bf16x2(osc, osc);
        const uint32_t a_addr = x_addr + half * HALF;
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
        if (lane == 0) mbar_arrive(a_bar);
      }
      uint32_t p_lo[16];
      convert_block(sbuf, half, p_lo);
      tmem_st16(sbuf + 32 * half, p_lo);
      tmem_st16(sbuf + 32 * half + 16, p_hi);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_bar);
    };
    for (int t = 0; t < nchunks; ++t) {
      const float osc = pw[max(chunk_len(t) - 1 - i, 0)];
      mbar_wait(&bars.sv_full, t & 1);
      if (warp == WARP_P && lane == 0) LB_TR(t, 11);
      tc_fence_after();
      convert(TM_SV, slot(SLOT_K), osc, &bars.av_full, &bars.pv_full);
      if (warp == WARP_P && lane == 0) LB_TR(t, 12);
      mbar_wait(&bars.sk_full, t & 1);
      if (warp == WARP_P && lane == 0) LB_TR(t, 13);
      tc_fence_after();
      convert(TM_SK, slot(SLOT_V), osc, &bars.ak_full, &bars.pk_full);
      if (warp == WARP_P && lane == 0) LB_TR(t, 14);
    }
  } else if (warp < WARP_KV) {
    // ------------------------------------------------------------ W + dV / dK epilogues (warps 10..17)
    const int quad = warp & 3;
    const int hh = (warp - WARP_O) >> 2;
    const int i = quad * 32 + lane;
    const uint32_t o_cols = tmem + ((uint32_t)(quad * 32) << 16) + TM_O + hh * 64;
    auto epilogue = [&](uint64_t* full_bar, uint32_t o_phase, uint32_t dst_slot, uint64_t* staged_bar, int t) {
      mbar_wait(full_bar, t & 1);
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
      if (lane == 0) mbar_arrive(&bars.o_free);
      (void)o_phase;
      const uint32_t base = dst_slot + hh * HALF;
#pragma unroll
      for (int m = 0; m < 8; ++m)
        sts128(base + sw128(i, m), make_uint4(pk[4 * m], pk[4 * m + 1], pk[4 * m + 2], pk[4 * m + 3]));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(staged_bar);
    };
    for (int t = 0; t < nchunks; ++t) {
      const int s = t & 1;
      build_w(t, i, hh);
      if (warp == WARP_O && lane == 0) LB_TR(t, 15);
      epilogue(&bars.ov_full, 2 * t, slot(SLOT_D + s), &bars.dv_staged[s], t);
      if (warp == WARP_O && lane == 0) LB_TR(t, 16);
      epilogue(&bars.ok_full, 2 * t + 1, slot(SLOT_Q + s), &bars.dk_staged[s], t);
      if (warp == WARP_O && lane == 0) LB_TR(t, 17);
    }
  } else {
    // ------------------------------------------------------------ state (warps 18..25)
    const int quad = warp & 3;
    const int hh = (warp - WARP_KV) >> 2;
    const int i = quad * 32 + lane;
    const uint32_t st_cols = tmem + ((uint32_t)(quad * 32) << 16) + TM_ST + hh * 64;
    uint32_t bf[32];  // bf16 copy of this thread's 64 state columns, published once X(t) is done
    auto load_scale = [&](bool from_global, float next_decay) {
#pragma unroll 1
      for (int q4 = 0; q4 < 4; ++q4) {
        float x[16];
        if (from_global) {
          if (args.state_in != nullptr && i < args.d && hh * 64 + q4 * 16 < args.d) {
            const float* src = args.state_in + (int64_t)bh * args.in_bh_stride + (int64_t)seg * args.in_seg_stride +
                               (int64_t)i * args.d + hh * 64 + q4 * 16;
            const float4* s4 = reinterpret_cast<const float4*>(src);  // 16-byte aligned state rows
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 w = s4[j];
              x[4 * j] = w.x, x[4 * j + 1] = w.y, x[4 * j + 2] = w.z, x[4 * j + 3] = w.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = 0.f;
          }
        } else {
          tmem_ld16(st_cols + q4 * 16, x);
          tmem_ld_wait();
        }
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = __float_as_uint(x[j] * next_decay);
        tmem_st16(st_cols + q4 * 16, w);
#pragma unroll
        for (int j = 0; j < 8; ++j) bf[q4 * 8 + j] = pack_bf16x2(x[2 * j], x[2 * j + 1]);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.st_scaled);
    };
    auto publish = [&]() {
      const uint32_t base = st_bf16 + hh * HALF;
#pragma unroll
      for (int m = 0; m < 8; ++m) sts128(base + sw128(i, m), make_uint4(bf[4 * m], bf[4 * m + 1], bf[4 * m + 2], bf[4 * m + 3]));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.st_pub);
    };
    // EPI: dkp(t) = act'(kp) * R^T dK(t) on the tile the B/O warps staged in Q's slot t % 2, in place; row i,
    // this warp's 64 columns; kp loaded straight from global (one 128-byte row segment per thread)
    uint4 xr[8];  // EPI: kp row segment of the chunk to transform next, loaded a chunk ahead of its use
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
    auto transform_dk = [&](int t) {
      const int s = t & 1;
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
      mbar_wait(&bars.dk_staged[s], (t >> 1) & 1);
      const uint32_t row = slot(SLOT_Q + s) + hh * HALF;
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
      if (lane == 0) mbar_arrive(&bars.dk_ready[s]);
    };
    if (nchunks > 0) {
      load_scale(true, pw[chunk_len(0)]);
      publish();
    }
    if (EPI && nchunks > 0) load_x(0);
    for (int t = 0; t < nchunks; ++t) {
      mbar_wait(&bars.ds_full, t & 1);
      tc_fence_after();
      if (t + 1 < nchunks) {
        load_scale(false, pw[chunk_len(t + 1)]);
        mbar_wait(&bars.x_done, t & 1);  // both products of chunk t read the previous copy
        publish();
        if (warp == WARP_KV && lane == 0) LB_TR(t, 19);
      }
      if (EPI) {
        transform_dk(t);
        if (t + 1 < nchunks) load_x(t + 1);  // in flight while the next chunk's products run
      }
    }
    if (nchunks > 0 && args.state_out != nullptr && seg == 0 && i < args.d && hh * 64 < args.d) {
      float* dst = args.state_out + (int64_t)bh * args.d * args.d + (int64_t)i * args.d + hh * 64;
#pragma unroll 1
      for (int q4 = 0; q4 < 4; ++q4) {
        float x[16];
        tmem_ld16(st_cols + q4 * 16, x);
        tmem_ld_wait();
        if (hh * 64 + q4 * 16 < args.d) {
#pragma unroll
          for (int j = 0; j < 16; ++j) dst[q4 * 16 + j] = x[j];
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

}  // namespace

#ifdef LA_TRACE
void la_debug_set_trace_bwd(void* dev_ptr) { cudaMemcpyToSymbol(g_la_trace_bwd, &dev_ptr, sizeof(dev_ptr)); }
#endif

cudaError_t tc_dkdv_launch(const PassDesc& p, const void* q, const void* k, const void* v, const void* dout,
                           void* dk, void* dv, const Strides3* s, cudaStream_t st, const GlaEpilogue* epi) {
  CUtensorMap mq, mk, mv, mdo, mdk, mdv;
  if (!tc_make_map(&mq, q, p, s[0]) || !tc_make_map(&mk, k, p, s[1]) || !tc_make_map(&mv, v, p, s[2]) ||
      !tc_make_map(&mdo, dout, p, s[3]) || !tc_make_map(&mdk, dk, p, s[4]) || !tc_make_map(&mdv, dv, p, s[5]))
    return cudaErrorInvalidValue;
  BwdArgs a;
  std::memset(&a, 0, sizeof(a));
  a.heads = p.heads;
  a.n = p.n;
  a.d = p.d;
  a.seg_len = p.seg_len;
  a.nseg = p.nseg;
  a.lam = p.lam;
  a.state_in = reinterpret_cast<const float*>(p.state_in);
  a.in_bh_stride = p.state_in_bh_stride;
  a.in_seg_stride = p.state_in_seg_stride;
  a.state_out = reinterpret_cast<float*>(p.state_out);
  dim3 grid(p.nseg, p.batch * p.heads);
  if (epi != nullptr) {
    if (reinterpret_cast<uintptr_t>(epi->xp) & 15) return cudaErrorMisalignedAddress;
    a.xp = reinterpret_cast<const uint16_t*>(epi->xp);
    a.sx = epi->sx;
    a.theta = epi->theta;
    a.act = epi->act;
    a.offset = epi->offset;
    static std::atomic<bool> smem_set_epi[64] = {};
    cudaError_t err = set_smem_once(tc_dkdv_kernel<true>, (int)SMEM_BYTES, smem_set_epi);
    if (err != cudaSuccess) return err;
    return launch_pdl(tc_dkdv_kernel<true>, grid, dim3(NUM_THREADS), SMEM_BYTES, st, mq, mk, mv, mdo, mdk, mdv, a);
  }
  static std::atomic<bool> smem_set[64] = {};
  cudaError_t err = set_smem_once(tc_dkdv_kernel<false>, (int)SMEM_BYTES, smem_set);
  if (err != cudaSuccess) return err;
  return launch_pdl(tc_dkdv_kernel<false>, grid, dim3(NUM_THREADS), SMEM_BYTES, st, mq, mk, mv, mdo, mdk, mdv, a);
}

}  // namespace la
