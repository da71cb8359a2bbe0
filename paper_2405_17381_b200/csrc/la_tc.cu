// la_tc.cu -- the bf16 pass kernel on B200 tensor cores: TMA -> SMEM (128B
// swizzle) -> tcgen05.mma (fp32 accumulators in TMEM) -> tcgen05.ld epilogues.
//
// One CTA owns one (batch, head, segment) and walks its chunks of C = 128 rows
// (fwd) or walks them backwards (rev), carrying the d x d state in fp32
// REGISTERS of the state warpgroups and a bf16 copy of it in SMEM (the B
// operand of the inter-chunk product).  Per chunk (la_common.cuh algebra):
//
//   S      = A B^T                  tcgen05  M=128 N=128 K=128  -> TMEM [0,128)
//   X      = A state                tcgen05  M=128 N=128 K=128  -> TMEM [256,384)
//   P      = bf16(S * M_decay)      epilogue warps: tcgen05.ld, mask, -> SMEM (A's slot)
//   Y      = P C                    tcgen05  A = P (SMEM)       -> TMEM [128,256)
//   out    = Y + out_scale * X      epilogue warps -> SMEM (A's slot) -> TMA store
//   B~     = in_scale * B           state warps, in place in SMEM after S consumed B
//   dS     = B~^T C                 tcgen05  A MN-major         -> TMEM [384,512)
//   state  = lam^b state + dS       state warps (fp32 registers) -> bf16 SMEM copy
//
// Warp roles (14 warps): 0 TMA producer, 1 MMA issuer (+ TMEM owner),
// 2-5 score/output epilogue (one TMEM lane quadrant each), 6-13 state update
// (two warpgroups, 64 state columns each).  Everything is chained with
// mbarriers; the only CTA-wide barriers are at setup and teardown.
//
// Shared memory: 2 stages x {A, B, C} tiles (3 x 32 KB) + the bf16 state
// (32 KB) = 224 KB -> one CTA per SM.  TMEM: all 512 columns.
#include <cudaTypedefs.h>

#include <cstring>

#include "la_common.cuh"
#include "la_ptx.cuh"
#include "la_scan.cuh"
#include "la_tc.cuh"

namespace la {

namespace {

using namespace ptx;

constexpr int C = 128;                  // chunk rows
constexpr int D = 128;                  // head dim (only d == 128 on this backend)
constexpr int TILE = C * D * 2;         // 32 KB bf16 tile
constexpr int HALF = TILE / 2;          // [128 rows][64 cols] = 16 KB, one 128B-swizzle column block
constexpr int NSTAGE = 2;
constexpr int NUM_WARPS = 14;
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr int WARP_TMA = 0, WARP_MMA = 1, WARP_SO = 2, WARP_KV = 6;
constexpr uint32_t TM_S = 0, TM_Y = 128, TM_X = 256, TM_DS = 384, TM_COLS = 512;

// kind::f16 instruction descriptors (M = N = 128)
constexpr uint32_t IDESC_KK = idesc_bf16(128, 128, 0, 0);    // A K-major, B K-major
constexpr uint32_t IDESC_KMN = idesc_bf16(128, 128, 0, 1);   // A K-major, B MN-major
constexpr uint32_t IDESC_MNMN = idesc_bf16(128, 128, 1, 1);  // A MN-major, B MN-major

struct Bars {
  uint64_t full[NSTAGE];   // TMA -> MMA        (tx bytes)
  uint64_t empty[NSTAGE];  // MMA commit (+ output store) -> TMA
  uint64_t s_full;         // MMA: S and X done -> epilogue + state warps
  uint64_t s_free;         // epilogue read S   -> MMA
  uint64_t p_full;         // P in SMEM         -> MMA
  uint64_t y_full;         // MMA: Y done       -> epilogue
  uint64_t o_free;         // epilogue read Y,X -> MMA
  uint64_t b_scaled;       // B~ in SMEM        -> MMA
  uint64_t ds_full;        // MMA: dS done      -> state warps
  uint64_t ds_free;        // state warps read dS -> MMA
  uint64_t st_ready;       // bf16 state in SMEM -> MMA
  uint32_t tmem_base;
};

constexpr size_t SMEM_TILES = (size_t)NSTAGE * 3 * TILE + TILE;  // 224 KB
constexpr size_t SMEM_BYTES = SMEM_TILES + 1024 /*bars*/ + 1024 /*pw*/ + 1024 /*align slack*/;

struct TcArgs {
  int heads, n, seg_len, nseg, rev;
  const double* lam;
  const float* state_in;
  int64_t in_bh_stride, in_seg_stride;
  int in_T;
  float* state_out;
  int out_T;
  float* delta_out;
};

// byte offset of 16-byte chunk `c` (0..7) of row `r` inside a [128][64] bf16 block, 128B swizzle
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

template <bool STATE_ONLY>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_pass_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_o,
                   const TcArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto tile_a = [smem](int s) { return smem + (size_t)s * 3 * TILE; };
  auto tile_b = [smem](int s) { return smem + (size_t)s * 3 * TILE + TILE; };
  auto tile_c = [smem](int s) { return smem + (size_t)s * 3 * TILE + 2 * TILE; };
  uint8_t* st_bf16 = smem + (size_t)NSTAGE * 3 * TILE;
  Bars* bars = reinterpret_cast<Bars*>(smem + SMEM_TILES);
  float* pw = reinterpret_cast<float*>(smem + SMEM_TILES + 1024);  // lam^0 .. lam^128

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = blockIdx.x, bh = blockIdx.y;
  const int bi = bh / args.heads, hi = bh % args.heads;
  const int p0 = seg * args.seg_len;
  const int p1 = min(args.n, p0 + args.seg_len);
  const int nchunks = (p1 - p0 + C - 1) / C;
  const int rev = args.rev;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], STATE_ONLY ? 1 : 2);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->s_free, 4);
    mbar_init(&bars->p_full, 4);
    mbar_init(&bars->y_full, 1);
    mbar_init(&bars->o_free, 4);
    mbar_init(&bars->b_scaled, 8);
    mbar_init(&bars->ds_full, 1);
    mbar_init(&bars->ds_free, 8);
    mbar_init(&bars->st_ready, 8);
    fence_mbar_init();
    double x = 1.0;
    const double lam = args.lam[hi];
    for (int k = 0; k <= C; ++k) {
      pw[k] = (float)x;
      x *= lam;
    }
  }
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch(&map_b);
    tma_prefetch(&map_c);
    if (!STATE_ONLY) {
      tma_prefetch(&map_a);
      tma_prefetch(&map_o);
    }
  }
  if (warp == WARP_MMA) tmem_alloc(&bars->tmem_base, TM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  auto chunk_row0 = [&](int t) { return p0 + (rev ? (nchunks - 1 - t) : t) * C; };

  if (warp == WARP_TMA) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint32_t bytes = (STATE_ONLY ? 2 : 3) * TILE;
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NSTAGE;
        if (t >= NSTAGE) mbar_wait(&bars->empty[s], ((t / NSTAGE) - 1) & 1);
        const int r0 = chunk_row0(t);
        mbar_arrive_expect_tx(&bars->full[s], bytes);
        for (int hf = 0; hf < 2; ++hf) {
          if (!STATE_ONLY) tma_load_4d(&map_a, &bars->full[s], tile_a(s) + hf * HALF, hf * 64, r0, hi, bi);
          tma_load_4d(&map_b, &bars->full[s], tile_b(s) + hf * HALF, hf * 64, r0, hi, bi);
          tma_load_4d(&map_c, &bars->full[s], tile_c(s) + hf * HALF, hf * 64, r0, hi, bi);
        }
      }
    }
  } else if (warp == WARP_MMA) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t st_addr = smem_u32(st_bf16);
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NSTAGE;
        const uint32_t a_addr = smem_u32(tile_a(s)), b_addr = smem_u32(tile_b(s)), c_addr = smem_u32(tile_c(s));
        mbar_wait(&bars->full[s], (t / NSTAGE) & 1);
        if (!STATE_ONLY) {
          if (t >= 1) {
            mbar_wait(&bars->s_free, (t - 1) & 1);
            mbar_wait(&bars->o_free, (t - 1) & 1);
          }
          mbar_wait(&bars->st_ready, t & 1);
          tc_fence_after();
          // S = A B^T: A [rows][d] K-major, B [rows][d] K-major
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
            mma_bf16_ss(tmem + TM_S, smem_desc_sw128(a_addr + off, 0, 1024), smem_desc_sw128(b_addr + off, 0, 1024),
                        IDESC_KK, kk > 0);
          }
          // X = A state: state bf16 [d_k][d_v] row-major == B operand MN-major (N = d_v contiguous)
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t aoff = (kk >> 2) * HALF + (kk & 3) * 32;
            mma_bf16_ss(tmem + TM_X, smem_desc_sw128(a_addr + aoff, 0, 1024),
                        smem_desc_sw128(st_addr + kk * 2048, HALF, 1024), IDESC_KMN, kk > 0);
          }
          mma_commit(&bars->s_full);
          // Y = P C: P (in A's slot) [rows][keys] K-major, C [keys][d] MN-major
          mbar_wait(&bars->p_full, t & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < C / 16; ++kk) {
            const uint32_t aoff = (kk >> 2) * HALF + (kk & 3) * 32;
            mma_bf16_ss(tmem + TM_Y, smem_desc_sw128(a_addr + aoff, 0, 1024),
                        smem_desc_sw128(c_addr + kk * 2048, HALF, 1024), IDESC_KMN, kk > 0);
          }
          mma_commit(&bars->y_full);
        }
        // dS = B~^T C: A = B~^T (M = d_k contiguous -> MN-major), B = C MN-major
        mbar_wait(&bars->b_scaled, t & 1);
        if (t >= 1) mbar_wait(&bars->ds_free, (t - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk) {
          mma_bf16_ss(tmem + TM_DS, smem_desc_sw128(b_addr + kk * 2048, HALF, 1024),
                      smem_desc_sw128(c_addr + kk * 2048, HALF, 1024), IDESC_MNMN, kk > 0);
        }
        mma_commit(&bars->ds_full);
        mma_commit(&bars->empty[s]);
      }
    }
  } else if (warp < WARP_KV) {
    // ------------------------------------------------------------ score / output epilogue (warps 2..5)
    if (!STATE_ONLY) {
      const int quad = warp & 3;
      const int i = quad * 32 + lane;  // row within the chunk == TMEM lane
      const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
      for (int t = 0; t < nchunks; ++t) {
        const int s = t % NSTAGE;
        const int r0 = chunk_row0(t);
        const int b = min(C, p1 - r0);
        uint8_t* slot = tile_a(s);
        mbar_wait(&bars->s_full, t & 1);
        tc_fence_after();
        // P = bf16(S * M): fwd keeps j <= i with lam^(i-j); rev keeps j >= i with lam^(j-i)
#pragma unroll 1
        for (int cb = 0; cb < 4; ++cb) {
          float v[32];
          tmem_ld32(lane_addr + TM_S + cb * 32, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int jj = 0; jj < 32; jj += 2) {
            const int j0 = cb * 32 + jj, j1 = j0 + 1;
            const int d0 = rev ? (j0 - i) : (i - j0);
            const int d1 = rev ? (j1 - i) : (i - j1);
            const float x0 = d0 >= 0 ? v[jj] * pw[d0] : 0.f;
            const float x1 = d1 >= 0 ? v[jj + 1] * pw[d1] : 0.f;
            pk[jj >> 1] = pack_bf16x2(x0, x1);
          }
          uint8_t* base = slot + (cb >> 1) * HALF;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int c16 = (cb & 1) * 4 + m;
            *reinterpret_cast<uint4*>(base + sw128(i, c16)) = make_uint4(pk[4 * m], pk[4 * m + 1], pk[4 * m + 2],
                                                                         pk[4 * m + 3]);
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars->s_free);
          mbar_arrive(&bars->p_full);
        }
        // out = Y + out_scale * X  -> bf16 into the same slot -> TMA store
        mbar_wait(&bars->y_full, t & 1);
        tc_fence_after();
        const float osc = rev ? pw[max(b - 1 - i, 0)] : pw[i + 1];
#pragma unroll 1
        for (int cb = 0; cb < 4; ++cb) {
          float y[32], x[32];
          tmem_ld32(lane_addr + TM_Y + cb * 32, y);
          tmem_ld32(lane_addr + TM_X + cb * 32, x);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int jj = 0; jj < 32; jj += 2)
            pk[jj >> 1] = pack_bf16x2(fmaf(osc, x[jj], y[jj]), fmaf(osc, x[jj + 1], y[jj + 1]));
          uint8_t* base = slot + (cb >> 1) * HALF;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int c16 = (cb & 1) * 4 + m;
            *reinterpret_cast<uint4*>(base + sw128(i, c16)) = make_uint4(pk[4 * m], pk[4 * m + 1], pk[4 * m + 2],
                                                                         pk[4 * m + 3]);
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->o_free);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == WARP_SO && lane == 0) {
          tma_store_4d(&map_o, slot, 0, r0, hi, bi);
          tma_store_4d(&map_o, slot + HALF, 64, r0, hi, bi);
          tma_store_commit();
          tma_store_wait_read();
          mbar_arrive(&bars->empty[s]);
        }
      }
      if (warp == WARP_SO && lane == 0) tma_store_wait_all();
    }
  } else {
    // ------------------------------------------------------------ state update (warps 6..13)
    const int quad = warp & 3;
    const int hh = (warp - WARP_KV) >> 2;  // which 64 state columns
    const int i = quad * 32 + lane;        // state row (d_k index) == TMEM lane
    const uint32_t lane_addr = tmem + ((uint32_t)(quad * 32) << 16);
    float kv[64];
    if (!STATE_ONLY && args.state_in != nullptr) {
      const float* src = args.state_in + (int64_t)bh * args.in_bh_stride + (int64_t)seg * args.in_seg_stride;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int col = hh * 64 + j;
        kv[j] = args.in_T ? src[col * D + i] : src[i * D + col];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j) kv[j] = 0.f;
    }
    auto publish_state = [&]() {
      uint8_t* base = st_bf16 + hh * HALF;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const uint4 w = make_uint4(pack_bf16x2(kv[8 * m], kv[8 * m + 1]), pack_bf16x2(kv[8 * m + 2], kv[8 * m + 3]),
                                   pack_bf16x2(kv[8 * m + 4], kv[8 * m + 5]), pack_bf16x2(kv[8 * m + 6], kv[8 * m + 7]));
        *reinterpret_cast<uint4*>(base + sw128(i, m)) = w;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->st_ready);
    };
    if (!STATE_ONLY) publish_state();
    for (int t = 0; t < nchunks; ++t) {
      const int s = t % NSTAGE;
      const int r0 = chunk_row0(t);
      const int b = min(C, p1 - r0);
      if (STATE_ONLY)
        mbar_wait(&bars->full[s], (t / NSTAGE) & 1);
      else
        mbar_wait(&bars->s_full, t & 1);
      // B~ = in_scale * B, in place (row i, this warp's 64 columns): fwd lam^(b-1-i), rev lam^(i+1)
      {
        const float isc = (i < b) ? (rev ? pw[i + 1] : pw[b - 1 - i]) : 0.f;
        uint8_t* base = tile_b(s) + hh * HALF;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          uint4* p = reinterpret_cast<uint4*>(base + i * 128 + m * 16);  // row-local chunks: swizzle irrelevant
          uint4 w = *p;
          uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float lo = __uint_as_float(u[e] << 16) * isc;
            const float hi2 = __uint_as_float(u[e] & 0xFFFF0000u) * isc;
            u[e] = pack_bf16x2(lo, hi2);
          }
          *p = w;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->b_scaled);
      // state = lam^b state + dS
      mbar_wait(&bars->ds_full, t & 1);
      tc_fence_after();
      const float decay = pw[b];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float ds[32];
        tmem_ld32(lane_addr + TM_DS + hh * 64 + half * 32, ds);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) kv[half * 32 + j] = fmaf(decay, kv[half * 32 + j], ds[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->ds_free);
      if (!STATE_ONLY) publish_state();
    }
    if (STATE_ONLY) {
      float* dst = args.delta_out + ((int64_t)bh * args.nseg + seg) * D * D + (int64_t)i * D + hh * 64;
#pragma unroll
      for (int j = 0; j < 64; ++j) dst[j] = kv[j];
    } else if (args.state_out != nullptr && (rev ? seg == 0 : seg == args.nseg - 1)) {
      float* dst = args.state_out + (int64_t)bh * D * D;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int col = hh * 64 + j;
        dst[args.out_T ? (col * D + i) : (i * D + col)] = kv[j];
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
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* map, const void* base, const PassDesc& p) {
  auto enc = encode_fn();
  if (enc == nullptr) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p.d, (cuuint64_t)p.n, (cuuint64_t)p.heads, (cuuint64_t)p.batch};
  cuuint64_t strides[3] = {(cuuint64_t)p.sn * 2, (cuuint64_t)p.sh * 2, (cuuint64_t)p.sb * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)C, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  // degenerate strides of size-1 dims must still be valid multiples of 16
  if (p.heads == 1) strides[1] = strides[0] * (cuuint64_t)p.n;
  if (p.batch == 1) strides[2] = strides[1] * (cuuint64_t)p.heads;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool STATE_ONLY>
cudaError_t launch_tc(const PassDesc& p, cudaStream_t st) {
  CUtensorMap ma, mb, mc, mo;
  std::memset(&ma, 0, sizeof(ma));
  std::memset(&mo, 0, sizeof(mo));
  if (!make_map(&mb, p.b, p) || !make_map(&mc, p.c, p)) return cudaErrorInvalidValue;
  if (!STATE_ONLY && (!make_map(&ma, p.a, p) || !make_map(&mo, p.out, p))) return cudaErrorInvalidValue;
  TcArgs a;
  a.heads = p.heads;
  a.n = p.n;
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
  auto kern = tc_pass_kernel<STATE_ONLY>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
  if (err != cudaSuccess) return err;
  dim3 grid(p.nseg, p.batch * p.heads);
  kern<<<grid, NUM_THREADS, SMEM_BYTES, st>>>(ma, mb, mc, mo, a);
  return cudaGetLastError();
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

}  // namespace

bool tc_supported(int dtype, int d, const int64_t* strides) {
  if (dtype != LA_BF16 || d != D) return false;
  for (int i = 0; i < 3; ++i)
    if ((strides[i] * 2) % 16 != 0) return false;
  return true;
}

bool tc_pointers_ok(const PassDesc& p) {
  return aligned16(p.b) && aligned16(p.c) && (p.a == nullptr || aligned16(p.a)) &&
         (p.out == nullptr || aligned16(p.out));
}

Plan tc_plan(int64_t bh, int64_t n, int d, int64_t want_segments) {
  (void)d;
  return make_plan(bh, n, C, want_segments, kNumSMs, 2);
}

size_t tc_workspace_bytes(int64_t bh, int nseg, int d) {
  if (nseg <= 1) return 0;
  return 2 * sizeof(float) * (size_t)bh * nseg * d * d;
}

cudaError_t tc_pass(PassDesc p, void* ws, cudaStream_t st) {
  const int bh = p.batch * p.heads;
  const size_t dd = (size_t)p.d * p.d;
  if (p.nseg > 1) {
    float* delta = reinterpret_cast<float*>(ws);
    float* seg_in = delta + (size_t)bh * p.nseg * dd;
    PassDesc s = p;
    s.a = nullptr;
    s.out = nullptr;
    s.state_in = nullptr;
    s.state_out = nullptr;
    s.delta_out = delta;
    cudaError_t err = launch_tc<true>(s, st);
    if (err != cudaSuccess) return err;
    err = launch_segment_scan(false, delta, seg_in, p.state_in, p.state_in_T, nullptr, 0, p.lam, bh, p.heads, p.d,
                              p.n, p.seg_len, p.nseg, p.rev, st);
    if (err != cudaSuccess) return err;
    p.state_in = seg_in;
    p.state_in_T = 0;
    p.state_in_bh_stride = (int64_t)p.nseg * dd;
    p.state_in_seg_stride = (int64_t)dd;
  } else {
    p.state_in_bh_stride = (int64_t)dd;
    p.state_in_seg_stride = 0;
  }
  return launch_tc<false>(p, st);
}

cudaError_t tc_state(PassDesc p, void* ws, cudaStream_t st) {
  const int bh = p.batch * p.heads;
  if (p.nseg == 1) {
    p.delta_out = p.state_out;
    return launch_tc<true>(p, st);
  }
  float* delta = reinterpret_cast<float*>(ws);
  p.delta_out = delta;
  cudaError_t err = launch_tc<true>(p, st);
  if (err != cudaSuccess) return err;
  return launch_segment_scan(false, delta, nullptr, nullptr, 0, p.state_out, p.state_out_T, p.lam, bh, p.heads, p.d,
                             p.n, p.seg_len, p.nseg, p.rev, st);
}

}  // namespace la
