// la_decode.cu -- one recurrent decode step over every (batch, head) state (model.py:669-709).
//
// The reference's decode_step updates each (layer, head) summary in place and reads the output
// through it (model.py:697-701):
//     kv <- lam * kv + k v^T        (d x d, state dtype)
//     o   = q . kv                  (after the update: the token attends to itself, as in la_fwd)
// so after a prefill of n tokens with kv_out = F(n) the decode continues exactly where la_fwd
// stopped.  The step is bound by the state traffic (d^2 reads + d^2 writes per head), so one CTA per
// (batch, head) streams its state once: a warp covers 32 consecutive columns of a row (coalesced
// 128-byte accesses), eight warps split the rows, and the per-column partial dot products meet in
// shared memory.
#include "la_common.cuh"
#include "la_decode.cuh"
#include "la_ptx.cuh"

namespace la {

namespace {

constexpr int kDecThreads = 256;  // 8 warps: warp w owns rows w, w + 8, ...

// VW state columns per thread (16-byte accesses when the head dim allows, else 1)
template <typename T, typename Tacc, int VW>
__global__ void __launch_bounds__(kDecThreads) decode_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                             const T* __restrict__ v, const double* __restrict__ lam,
                                                             Tacc* __restrict__ kv, T* __restrict__ o, int heads,
                                                             int d, int64_t sb, int64_t sh) {
  __shared__ Tacc sq[128], sk[128], sv[128];
  __shared__ Tacc part[kDecThreads / 32][128];
  const int bh = blockIdx.x;
  const int bi = bh / heads, hi = bh % heads;
  const int64_t base = (int64_t)bi * sb + (int64_t)hi * sh;
  for (int e = threadIdx.x; e < d; e += kDecThreads) {
    sq[e] = (Tacc)Cvt<T>::to_f(q[base + e]);
    sk[e] = (Tacc)Cvt<T>::to_f(k[base + e]);
    sv[e] = (Tacc)Cvt<T>::to_f(v[base + e]);
  }
  __syncthreads();
  const Tacc l = (Tacc)load_decay(lam, hi);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Tacc* st = kv + (int64_t)bh * d * d;
  constexpr int NC = VW == 1 ? 4 : 1;  // column groups per lane: 4 x 32 scalars, or one 32 x VW vector
  Tacc acc[NC][VW];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int e = 0; e < VW; ++e) acc[c][e] = 0;
  // rows i = warp, warp + 8, ...: issue RB rows' loads before any of their stores, so each warp keeps
  // RB independent 512-byte reads in flight (the row loop alone serialised on load latency)
  constexpr int RB = 8;
  for (int i0 = warp; i0 < d; i0 += RB * (kDecThreads / 32)) {
    Tacc x[RB][NC][VW];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = i0 + rr * (kDecThreads / 32);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j0 = VW == 1 ? lane + 32 * c : lane * VW;
        if (i < d && j0 < d) {
          const Tacc* row = st + (int64_t)i * d;
          if (VW > 1) {
            *reinterpret_cast<uint4*>(x[rr][c]) = *reinterpret_cast<const uint4*>(row + j0);
          } else {
            x[rr][c][0] = row[j0];
          }
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = i0 + rr * (kDecThreads / 32);
      if (i >= d) break;
      const Tacc qi = sq[i], ki = sk[i];
      Tacc* row = st + (int64_t)i * d;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j0 = VW == 1 ? lane + 32 * c : lane * VW;
        if (j0 < d) {
#pragma unroll
          for (int e = 0; e < VW; ++e) {
            x[rr][c][e] = l * x[rr][c][e] + ki * sv[j0 + e];
            acc[c][e] += qi * x[rr][c][e];
          }
          if (VW > 1) {
            *reinterpret_cast<uint4*>(row + j0) = *reinterpret_cast<const uint4*>(x[rr][c]);
          } else {
            row[j0] = x[rr][c][0];
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j0 = VW == 1 ? lane + 32 * c : lane * VW;
#pragma unroll
    for (int e = 0; e < VW; ++e)
      if (j0 + e < d) part[warp][j0 + e] = acc[c][e];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += kDecThreads) {
    Tacc s = 0;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) s += part[w][j];
    o[base + j] = Cvt<T>::from_f(s);
  }
}

// d = 128, fp32 state: the state streams through SMEM by 1-D bulk copies (TMA engine), 64 KB per CTA,
// three CTAs per SM, so each SM keeps ~192 KB of state traffic in flight instead of what its warps'
// registers can hold.  Thread t owns state column c = t % 128 for rows r = t / 128 + 2 k.
template <typename T>
__global__ void __launch_bounds__(256) decode_bulk_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                          const T* __restrict__ v, const double* __restrict__ lam,
                                                          float* __restrict__ kv, T* __restrict__ o, int heads,
                                                          int64_t sb, int64_t sh) {
  constexpr int DD = 128;
  extern __shared__ __align__(128) uint8_t dsm[];
  float* st = reinterpret_cast<float*>(dsm);  // [128][128]
  __shared__ float sq[DD], sk[DD], sv[DD], part[2][DD];
  __shared__ __align__(8) uint64_t bar;
  const int bh = blockIdx.x;
  const int bi = bh / heads, hi = bh % heads;
  const int64_t base = (int64_t)bi * sb + (int64_t)hi * sh;
  float* g = kv + (int64_t)bh * DD * DD;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, DD * DD * 4);
#pragma unroll
    for (int part4 = 0; part4 < 4; ++part4)  // 4 x 16 KB
      ptx::bulk_load(st + part4 * DD * DD / 4, g + part4 * DD * DD / 4, DD * DD, &bar);
  }
  if (threadIdx.x < DD) {
    sq[threadIdx.x] = Cvt<T>::to_f(q[base + threadIdx.x]);
    sk[threadIdx.x] = Cvt<T>::to_f(k[base + threadIdx.x]);
    sv[threadIdx.x] = Cvt<T>::to_f(v[base + threadIdx.x]);
  }
  __syncthreads();
  ptx::mbar_wait(&bar, 0);
  const float l = (float)load_decay(lam, hi);
  const int c = threadIdx.x & (DD - 1), r0 = threadIdx.x >> 7;
  const float vc = sv[c];
  float acc = 0.f;
#pragma unroll 8
  for (int r = r0; r < DD; r += 2) {
    const float x = l * st[r * DD + c] + sk[r] * vc;
    st[r * DD + c] = x;
    acc += sq[r] * x;
  }
  part[r0][c] = acc;
  ptx::fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::bulk_store(g, st, DD * DD * 4);
    ptx::tma_store_commit();
  }
  if (threadIdx.x < DD) o[base + threadIdx.x] = Cvt<T>::from_f(part[0][threadIdx.x] + part[1][threadIdx.x]);
  if (threadIdx.x == 0) ptx::tma_store_wait_read();  // SMEM must stay valid until the store has read it
}

}  // namespace

cudaError_t decode_launch(int dtype, int batch, int heads, int d, int64_t sb, int64_t sh, const void* q,
                          const void* k, const void* v, const double* lam, void* kv, void* o, cudaStream_t st) {
  const dim3 grid((unsigned)(batch * heads));
  static std::atomic<bool> set_f32[64] = {}, set_bf16[64] = {};  // per device: a process may drive several GPUs
  cudaError_t aerr = set_smem_once(decode_bulk_kernel<float>, 128 * 128 * 4, set_f32);
  if (aerr == cudaSuccess) aerr = set_smem_once(decode_bulk_kernel<__nv_bfloat16>, 128 * 128 * 4, set_bf16);
  if (aerr != cudaSuccess) return aerr;
  // 16-byte state accesses when a warp's 32 vectors span exactly one row (d = 128 fp32, d = 64 fp64)
  switch (dtype) {
    case LA_F64:
      if (d == 64)
        decode_kernel<double, double, 2><<<grid, kDecThreads, 0, st>>>(
            static_cast<const double*>(q), static_cast<const double*>(k), static_cast<const double*>(v), lam,
            static_cast<double*>(kv), static_cast<double*>(o), heads, d, sb, sh);
      else
        decode_kernel<double, double, 1><<<grid, kDecThreads, 0, st>>>(
            static_cast<const double*>(q), static_cast<const double*>(k), static_cast<const double*>(v), lam,
            static_cast<double*>(kv), static_cast<double*>(o), heads, d, sb, sh);
      break;
    case LA_F32:
      if (d == 128)
        decode_bulk_kernel<float><<<grid, 256, 128 * 128 * 4, st>>>(
            static_cast<const float*>(q), static_cast<const float*>(k), static_cast<const float*>(v), lam,
            static_cast<float*>(kv), static_cast<float*>(o), heads, sb, sh);
      else
        decode_kernel<float, float, 1><<<grid, kDecThreads, 0, st>>>(
            static_cast<const float*>(q), static_cast<const float*>(k), static_cast<const float*>(v), lam,
            static_cast<float*>(kv), static_cast<float*>(o), heads, d, sb, sh);
      break;
    default:
      if (d == 128)
        decode_bulk_kernel<__nv_bfloat16><<<grid, 256, 128 * 128 * 4, st>>>(
            static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
            static_cast<const __nv_bfloat16*>(v), lam, static_cast<float*>(kv), static_cast<__nv_bfloat16*>(o), heads,
            sb, sh);
      else
        decode_kernel<__nv_bfloat16, float, 1><<<grid, kDecThreads, 0, st>>>(
            static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
            static_cast<const __nv_bfloat16*>(v), lam, static_cast<float*>(kv), static_cast<__nv_bfloat16*>(o), heads,
            d, sb, sh);
  }
  return cudaGetLastError();
}

}  // namespace la
