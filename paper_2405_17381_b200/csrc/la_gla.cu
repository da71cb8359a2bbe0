// la_gla.cu -- the element-wise stages of the GLA layer around the attention core
// (model.py:365-453): everything between the four input projections and the output
// projection, which stay library GEMMs.
//
//   prologue      q = rot(act(qp)), k = rot(act(kp))      act: swish | 1+elu | none (model.py:60-99)
//                 rot: LRPE pair rotation by theta_j (t + offset), positional.py:126-150
//   prologue_bwd  dqp = act'(qp) * rot^-1(dq), same for k; dtheta_j += sum_t (t + offset)
//                 (dy2 y1 - dy1 y2) over q and k (positional.py:153-182, model.py:434-441)
//   epilogue      gated = srmsnorm(a) * u, srmsnorm(x) = x sqrt(W) / max(|x|, eps)  (model.py:106-116)
//   epilogue_bwd  (da, du) from dgated (model.py:118-129, 419-426)
//
// Rows are the (batch, position) pairs of a [batch, n, width] tensor (width = heads * d, the
// model-native layout la_fwd / la_bwd read without a transpose).  All stages are single-pass and
// bound by HBM traffic: each reads its inputs once and writes its outputs once, in the operand
// dtype, accumulating in fp32 (fp64 for the fp64 path).  The norm's row statistic (the raw l2 norm)
// is saved by the forward so the backward does not recompute it.
#include <cmath>

#include "la_common.cuh"
#include "la_gla.cuh"

namespace la {

namespace {

template <typename Tacc>
__device__ __forceinline__ Tacc act_fwd(Tacc x, int act) {
  if (act == LA_ACT_SWISH) return x * (Tacc)0.5 * ((Tacc)1 + tanh((Tacc)0.5 * x));  // tanh form, model.py:57-66
  if (act == LA_ACT_ONE_PLUS_ELU) return x > (Tacc)0 ? x + (Tacc)1 : exp(x);
  return x;
}
template <typename Tacc>
__device__ __forceinline__ Tacc act_grad(Tacc x, int act) {
  if (act == LA_ACT_SWISH) {
    const Tacc s = (Tacc)0.5 * ((Tacc)1 + tanh((Tacc)0.5 * x));
    return s * ((Tacc)1 + x * ((Tacc)1 - s));
  }
  if (act == LA_ACT_ONE_PLUS_ELU) return x > (Tacc)0 ? (Tacc)1 : exp(x);
  return (Tacc)1;
}

// cos / sin of theta (t + offset): the angle is formed and reduced mod 2 pi in fp64, so long
// sequences (t ~ 1e6 rad) keep full fp32 accuracy
template <typename Tacc>
__device__ __forceinline__ void rot_cs(double theta, int64_t pos, Tacc* c, Tacc* s) {
  double ang = theta * (double)pos;
  ang = remainder(ang, 6.283185307179586476925286766559);
  if (sizeof(Tacc) == 8) {
    double cc, ss;
    sincos(ang, &ss, &cc);
    *c = (Tacc)cc;
    *s = (Tacc)ss;
  } else {
    float cc, ss;
    sincosf((float)ang, &ss, &cc);
    *c = (Tacc)cc;
    *s = (Tacc)ss;
  }
}

// one thread per feature pair of one row
template <typename T, typename Tacc>
__global__ void prologue_kernel(const T* __restrict__ qp, const T* __restrict__ kp, const double* __restrict__ theta,
                                T* __restrict__ q, T* __restrict__ k, int64_t rows, int n, int width, int d,
                                int64_t offset, int act) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int half_w = width >> 1;
  if (idx >= rows * half_w) return;
  const int64_t row = idx / half_w;
  const int pc = (int)(idx % half_w);  // pair column within the row
  const int64_t e = row * width + 2 * pc;
  Tacc q1 = act_fwd<Tacc>((Tacc)Cvt<T>::to_f(qp[e]), act), q2 = act_fwd<Tacc>((Tacc)Cvt<T>::to_f(qp[e + 1]), act);
  Tacc k1 = act_fwd<Tacc>((Tacc)Cvt<T>::to_f(kp[e]), act), k2 = act_fwd<Tacc>((Tacc)Cvt<T>::to_f(kp[e + 1]), act);
  if (theta != nullptr) {
    Tacc c, s;
    rot_cs<Tacc>(theta[pc % (d >> 1)], row % n + offset, &c, &s);
    const Tacc a1 = q1 * c - q2 * s, a2 = q1 * s + q2 * c;
    const Tacc b1 = k1 * c - k2 * s, b2 = k1 * s + k2 * c;
    q1 = a1, q2 = a2, k1 = b1, k2 = b2;
  }
  q[e] = Cvt<T>::from_f(q1);
  q[e + 1] = Cvt<T>::from_f(q2);
  k[e] = Cvt<T>::from_f(k1);
  k[e + 1] = Cvt<T>::from_f(k2);
}

constexpr int kRowsPerBlock = 64;

// grid (ceil(width/2 / 256), ceil(rows / 64)); dtheta partials per (row block, x block) land in
// `partial` [gridDim.y * gridDim.x][d/2] (deterministic; summed by reduce_theta_kernel)
template <typename T, typename Tacc>
__global__ void __launch_bounds__(256) prologue_bwd_kernel(const T* __restrict__ qp, const T* __restrict__ kp,
                                                           const double* __restrict__ theta, const T* __restrict__ dq,
                                                           const T* __restrict__ dk, T* __restrict__ dqp,
                                                           T* __restrict__ dkp, double* __restrict__ partial,
                                                           int64_t rows, int n, int width, int d, int64_t offset,
                                                           int act) {
  extern __shared__ double sdt[];  // [d/2]
  const int half_w = width >> 1, hd = d >> 1;
  const int pc = blockIdx.x * blockDim.x + threadIdx.x;
  if (theta != nullptr) {
    for (int j = threadIdx.x; j < hd; j += blockDim.x) sdt[j] = 0.0;
    __syncthreads();
  }
  Tacc acc = 0;
  if (pc < half_w) {
    const double th = theta != nullptr ? theta[pc % hd] : 0.0;
    const int64_t r0 = (int64_t)blockIdx.y * kRowsPerBlock;
    const int64_t r1 = r0 + kRowsPerBlock < rows ? r0 + kRowsPerBlock : rows;
    for (int64_t row = r0; row < r1; ++row) {
      const int64_t e = row * width + 2 * pc;
      const Tacc xq1 = (Tacc)Cvt<T>::to_f(qp[e]), xq2 = (Tacc)Cvt<T>::to_f(qp[e + 1]);
      const Tacc xk1 = (Tacc)Cvt<T>::to_f(kp[e]), xk2 = (Tacc)Cvt<T>::to_f(kp[e + 1]);
      Tacc gq1 = (Tacc)Cvt<T>::to_f(dq[e]), gq2 = (Tacc)Cvt<T>::to_f(dq[e + 1]);
      Tacc gk1 = (Tacc)Cvt<T>::to_f(dk[e]), gk2 = (Tacc)Cvt<T>::to_f(dk[e + 1]);
      if (theta != nullptr) {
        Tacc c, s;
        const int64_t pos = row % n + offset;
        rot_cs<Tacc>(th, pos, &c, &s);
        // rotated activations y (recomputed) for the angle gradient
        const Tacc aq1 = act_fwd<Tacc>(xq1, act), aq2 = act_fwd<Tacc>(xq2, act);
        const Tacc ak1 = act_fwd<Tacc>(xk1, act), ak2 = act_fwd<Tacc>(xk2, act);
        const Tacc yq1 = aq1 * c - aq2 * s, yq2 = aq1 * s + aq2 * c;
        const Tacc yk1 = ak1 * c - ak2 * s, yk2 = ak1 * s + ak2 * c;
        acc += (Tacc)pos * ((gq2 * yq1 - gq1 * yq2) + (gk2 * yk1 - gk1 * yk2));
        // dx = rot^-1 dy
        const Tacc rq1 = gq1 * c + gq2 * s, rq2 = -gq1 * s + gq2 * c;
        const Tacc rk1 = gk1 * c + gk2 * s, rk2 = -gk1 * s + gk2 * c;
        gq1 = rq1, gq2 = rq2, gk1 = rk1, gk2 = rk2;
      }
      dqp[e] = Cvt<T>::from_f(gq1 * act_grad<Tacc>(xq1, act));
      dqp[e + 1] = Cvt<T>::from_f(gq2 * act_grad<Tacc>(xq2, act));
      dkp[e] = Cvt<T>::from_f(gk1 * act_grad<Tacc>(xk1, act));
      dkp[e + 1] = Cvt<T>::from_f(gk2 * act_grad<Tacc>(xk2, act));
    }
  }
  if (theta == nullptr) return;
  if (pc < half_w) atomicAdd(&sdt[pc % hd], (double)acc);  // shared-memory reduction over the heads
  __syncthreads();
  double* dst = partial + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * hd;
  for (int j = threadIdx.x; j < hd; j += blockDim.x) dst[j] = sdt[j];
}

__global__ void reduce_theta_kernel(const double* __restrict__ partial, int64_t nparts, int hd,
                                    double* __restrict__ dtheta) {
  const int j = blockIdx.x;
  double s = 0.0;
  for (int64_t p = threadIdx.x; p < nparts; p += blockDim.x) s += partial[p * hd + j];
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) dtheta[j] += red[0];  // accumulated, like grads["lrpe.theta"] += ...
}

template <typename Tacc>
__device__ __forceinline__ Tacc block_sum(Tacc v, Tacc* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // red reused across calls
  if (lane == 0) red[warp] = v;
  __syncthreads();
  Tacc t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

// one CTA per row
template <typename T, typename Tacc>
__global__ void __launch_bounds__(256) epilogue_kernel(const T* __restrict__ a, const T* __restrict__ u,
                                                       T* __restrict__ gated, Tacc* __restrict__ rawnorm, int width,
                                                       double eps) {
  __shared__ Tacc red[32];
  const int64_t row = blockIdx.x;
  const T* ar = a + row * width;
  Tacc ss = 0;
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    const Tacc x = (Tacc)Cvt<T>::to_f(ar[c]);
    ss += x * x;
  }
  ss = block_sum<Tacc>(ss, red);
  const Tacc raw = sqrt(ss);
  const Tacc scale = sqrt((Tacc)width) / (raw > (Tacc)eps ? raw : (Tacc)eps);
  if (threadIdx.x == 0) rawnorm[row] = raw;
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    Tacc y = (Tacc)Cvt<T>::to_f(ar[c]) * scale;
    if (u != nullptr) y *= (Tacc)Cvt<T>::to_f(u[row * width + c]);
    gated[row * width + c] = Cvt<T>::from_f(y);
  }
}

template <typename T, typename Tacc>
__global__ void __launch_bounds__(256) epilogue_bwd_kernel(const T* __restrict__ dgated, const T* __restrict__ a,
                                                           const T* __restrict__ u, const Tacc* __restrict__ rawnorm,
                                                           T* __restrict__ da, T* __restrict__ du, int width,
                                                           double eps) {
  __shared__ Tacc red[32];
  const int64_t row = blockIdx.x;
  const int64_t off = row * width;
  const Tacc raw = rawnorm[row];
  const Tacc r = raw > (Tacc)eps ? raw : (Tacc)eps;
  const Tacc scale = sqrt((Tacc)width) / r;
  Tacc dot = 0;  // sum_c a_c * dan_c
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    const Tacc x = (Tacc)Cvt<T>::to_f(a[off + c]);
    const Tacc g = (Tacc)Cvt<T>::to_f(dgated[off + c]);
    Tacc dan = g;
    if (u != nullptr) {
      const Tacc uu = (Tacc)Cvt<T>::to_f(u[off + c]);
      dan = g * uu;
      du[off + c] = Cvt<T>::from_f(g * x * scale);  // du = dgated * an
    }
    dot += x * dan;
  }
  dot = block_sum<Tacc>(dot, red);
  // srmsnorm_backward: dx = dan sqrt(W)/r - [raw >= eps] x (x.dan / r^2) sqrt(W)/r
  const Tacc proj = raw >= (Tacc)eps ? dot / (r * r) : (Tacc)0;
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    const Tacc x = (Tacc)Cvt<T>::to_f(a[off + c]);
    Tacc dan = (Tacc)Cvt<T>::to_f(dgated[off + c]);
    if (u != nullptr) dan *= (Tacc)Cvt<T>::to_f(u[off + c]);
    da[off + c] = Cvt<T>::from_f((dan - x * proj) * scale);
  }
}

template <typename T, typename Tacc>
cudaError_t prologue_t(const GlaRows& g, const void* qp, const void* kp, const double* theta, void* q, void* k,
                       cudaStream_t st) {
  const int64_t pairs = g.rows * (g.width / 2);
  const int threads = 256;
  const int64_t blocks = (pairs + threads - 1) / threads;
  prologue_kernel<T, Tacc><<<(unsigned)blocks, threads, 0, st>>>(
      static_cast<const T*>(qp), static_cast<const T*>(kp), theta, static_cast<T*>(q), static_cast<T*>(k), g.rows,
      g.n, g.width, g.d, g.offset, g.act);
  return cudaGetLastError();
}

template <typename T, typename Tacc>
cudaError_t prologue_bwd_t(const GlaRows& g, const void* qp, const void* kp, const double* theta, const void* dq,
                           const void* dk, void* dqp, void* dkp, double* partial, double* dtheta, cudaStream_t st) {
  const int half_w = g.width / 2, hd = g.d / 2;
  const dim3 grid((unsigned)((half_w + 255) / 256), (unsigned)((g.rows + kRowsPerBlock - 1) / kRowsPerBlock));
  const size_t smem = theta != nullptr ? (size_t)hd * sizeof(double) : 0;
  prologue_bwd_kernel<T, Tacc><<<grid, 256, smem, st>>>(
      static_cast<const T*>(qp), static_cast<const T*>(kp), theta, static_cast<const T*>(dq),
      static_cast<const T*>(dk), static_cast<T*>(dqp), static_cast<T*>(dkp), partial, g.rows, g.n, g.width, g.d,
      g.offset, g.act);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess || theta == nullptr) return err;
  reduce_theta_kernel<<<hd, 256, 0, st>>>(partial, (int64_t)grid.x * grid.y, hd, dtheta);
  return cudaGetLastError();
}

template <typename T, typename Tacc>
cudaError_t epilogue_t(const GlaRows& g, const void* a, const void* u, void* gated, void* rawnorm, double eps,
                       cudaStream_t st) {
  epilogue_kernel<T, Tacc><<<(unsigned)g.rows, 256, 0, st>>>(static_cast<const T*>(a), static_cast<const T*>(u),
                                                              static_cast<T*>(gated), static_cast<Tacc*>(rawnorm),
                                                              g.width, eps);
  return cudaGetLastError();
}

template <typename T, typename Tacc>
cudaError_t epilogue_bwd_t(const GlaRows& g, const void* dgated, const void* a, const void* u, const void* rawnorm,
                           void* da, void* du, double eps, cudaStream_t st) {
  epilogue_bwd_kernel<T, Tacc><<<(unsigned)g.rows, 256, 0, st>>>(
      static_cast<const T*>(dgated), static_cast<const T*>(a), static_cast<const T*>(u),
      static_cast<const Tacc*>(rawnorm), static_cast<T*>(da), static_cast<T*>(du), g.width, eps);
  return cudaGetLastError();
}

}  // namespace

size_t gla_prologue_bwd_partial_bytes(const GlaRows& g) {
  const int64_t gx = (g.width / 2 + 255) / 256, gy = (g.rows + kRowsPerBlock - 1) / kRowsPerBlock;
  return (size_t)(gx * gy) * (size_t)(g.d / 2) * sizeof(double);
}

#define LA_DISPATCH(fn, ...)                                                      \
  switch (g.dtype) {                                                              \
    case LA_F64: return fn<double, double>(g, __VA_ARGS__);                       \
    case LA_F32: return fn<float, float>(g, __VA_ARGS__);                         \
    default: return fn<__nv_bfloat16, float>(g, __VA_ARGS__);                    \
  }

cudaError_t gla_prologue(const GlaRows& g, const void* qp, const void* kp, const double* theta, void* q, void* k,
                         cudaStream_t st) {
  LA_DISPATCH(prologue_t, qp, kp, theta, q, k, st)
}
cudaError_t gla_prologue_bwd(const GlaRows& g, const void* qp, const void* kp, const double* theta, const void* dq,
                             const void* dk, void* dqp, void* dkp, void* partial, double* dtheta, cudaStream_t st) {
  LA_DISPATCH(prologue_bwd_t, qp, kp, theta, dq, dk, dqp, dkp, static_cast<double*>(partial), dtheta, st)
}
cudaError_t gla_epilogue(const GlaRows& g, const void* a, const void* u, void* gated, void* rawnorm, double eps,
                         cudaStream_t st) {
  LA_DISPATCH(epilogue_t, a, u, gated, rawnorm, eps, st)
}
cudaError_t gla_epilogue_bwd(const GlaRows& g, const void* dgated, const void* a, const void* u, const void* rawnorm,
                             void* da, void* du, double eps, cudaStream_t st) {
  LA_DISPATCH(epilogue_bwd_t, dgated, a, u, rawnorm, da, du, eps, st)
}
#undef LA_DISPATCH

}  // namespace la
