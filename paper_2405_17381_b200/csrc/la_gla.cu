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

// fp32 accumulation uses the SFU forms (ex2 + rcp approximations, ~2^-21 relative): the stages are
// bound by instruction issue otherwise; fp64 keeps the library functions.  FAST (bf16 operands, whose
// results round to 2^-9 anyway): one SFU op, tanh.approx (~2^-11), instead of two
template <typename Tacc, bool FAST = false>
__device__ __forceinline__ Tacc sigmoid(Tacc x) {
  if constexpr (sizeof(Tacc) == 8) return (Tacc)0.5 * ((Tacc)1 + tanh((Tacc)0.5 * x));  // tanh form, model.py:57-66
  else if constexpr (FAST) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
    return fmaf(0.5f, t, 0.5f);
  } else return __fdividef(1.f, 1.f + __expf(-x));
}
template <typename Tacc>
__device__ __forceinline__ Tacc expo(Tacc x) {
  if constexpr (sizeof(Tacc) == 8) return exp(x);
  else return __expf(x);
}
template <typename Tacc, bool FAST = false>
__device__ __forceinline__ Tacc act_fwd(Tacc x, int act) {
  if (act == LA_ACT_SWISH) return x * sigmoid<Tacc, FAST>(x);
  if (act == LA_ACT_ONE_PLUS_ELU) return x > (Tacc)0 ? x + (Tacc)1 : expo(x);
  return x;
}
// act(x) and act'(x) sharing one sigmoid / exp
template <typename Tacc, bool FAST = false>
__device__ __forceinline__ void act_both(Tacc x, int act, Tacc& a, Tacc& g) {
  if (act == LA_ACT_SWISH) {
    const Tacc s = sigmoid<Tacc, FAST>(x);
    a = x * s;
    g = s * ((Tacc)1 + x * ((Tacc)1 - s));
  } else if (act == LA_ACT_ONE_PLUS_ELU) {
    const Tacc e = expo(x < (Tacc)0 ? x : (Tacc)0);
    a = x > (Tacc)0 ? x + (Tacc)1 : e;
    g = x > (Tacc)0 ? (Tacc)1 : e;
  } else {
    a = x;
    g = (Tacc)1;
  }
}

// cos / sin of theta (t + offset): the angle is formed and reduced mod 2 pi in fp64, so long
// sequences (t ~ 1e6 rad) keep full fp32 accuracy
template <typename Tacc>
__device__ __forceinline__ void rot_cs(double theta, int64_t pos, Tacc* c, Tacc* s) {
  double ang = theta * (double)pos;
  ang = fma(-6.283185307179586476925286766559, rint(ang * 0.15915494309189533576888376337251), ang);
  if (sizeof(Tacc) == 8) {
    double cc, ss;
    sincos(ang, &ss, &cc);
    *c = (Tacc)cc;
    *s = (Tacc)ss;
  } else {
    // |ang| <= pi after the fp64 reduction: the hardware approximation is accurate to ~2^-21 there
    float cc, ss;
    __sincosf((float)ang, &ss, &cc);
    *c = (Tacc)cc;
    *s = (Tacc)ss;
  }
}

// LRPE angles along consecutive rows of one column vector: exact (fp64-reduced) at the first row, at
// every sequence start and every kAnchor rows; in between the angle-addition step
// (c, s) <- (c, s) * (cos th, sin th) (4 FMAs, ~1e-7 relative drift per step).  fp64 is exact per row.
constexpr int kAnchor = 16;
template <typename Tacc, int NP>
struct RotWalk {
  double th[NP];
  Tacc c[NP], s[NP], c1[NP], s1[NP];
  __device__ __forceinline__ void init(const double* theta, int j0, int hd) {
#pragma unroll
    for (int pr = 0; pr < NP; ++pr) {
      th[pr] = theta[(j0 + pr) % hd];
      rot_cs<Tacc>(th[pr], 1, &c1[pr], &s1[pr]);
    }
  }
  // angles of position `pos`; `fresh`: no valid previous position (pos - 1) in registers
  __device__ __forceinline__ void at(int64_t pos, bool fresh) {
#pragma unroll
    for (int pr = 0; pr < NP; ++pr) {
      if (sizeof(Tacc) == 8 || fresh) {
        rot_cs<Tacc>(th[pr], pos, &c[pr], &s[pr]);
      } else {
        const Tacc cn = c[pr] * c1[pr] - s[pr] * s1[pr];
        s[pr] = s[pr] * c1[pr] + c[pr] * s1[pr];
        c[pr] = cn;
      }
    }
  }
};

// 16-byte vectors of the operand type (8 bf16, 4 fp32, 2 fp64 = 4, 2, 1 feature pairs)
template <typename T> struct Vec {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};
template <typename T>
__device__ __forceinline__ Vec<T> ldv(const T* p) {
  Vec<T> r;
  *reinterpret_cast<uint4*>(r.v) = __ldg(reinterpret_cast<const uint4*>(p));
  return r;
}
template <typename T>
__device__ __forceinline__ void stv(T* p, const Vec<T>& r) {
  *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(r.v);
}

// grid (ceil(rows / kRowsFwd), ceil(width/V / blockDim)): a thread owns one 16-byte column vector and walks
// kRowsFwd consecutive rows (its feature pairs' angles advance by one position per row)
constexpr int kRowsFwd = 16;
template <typename T, typename Tacc>
__global__ void __launch_bounds__(256) prologue_kernel(const T* __restrict__ qp, const T* __restrict__ kp,
                                                       const double* __restrict__ theta, T* __restrict__ q,
                                                       T* __restrict__ k, int64_t rows, int n, int width, int d,
                                                       int64_t offset, int act) {
  constexpr int V = Vec<T>::N;
  const int vw = width / V;
  const int vc = blockIdx.y * blockDim.x + threadIdx.x;
  if (vc >= vw) return;
  const int c0 = vc * V;
  RotWalk<Tacc, V / 2> rw;
  if (theta != nullptr) rw.init(theta, c0 >> 1, d >> 1);
  const int64_t r0 = (int64_t)blockIdx.x * kRowsFwd;
  const int64_t r1 = r0 + kRowsFwd < rows ? r0 + kRowsFwd : rows;
#pragma unroll 2
  for (int64_t row = r0; row < r1; ++row) {
    const int64_t e = row * width + c0;
    const Vec<T> xq = ldv(qp + e), xk = ldv(kp + e);
    Vec<T> oq, ok;
    const int64_t tp = row % n;
    if (theta != nullptr) rw.at(tp + offset, row == r0 || tp == 0 || ((row - r0) % kAnchor) == 0);
#pragma unroll
    for (int pr = 0; pr < V / 2; ++pr) {
      constexpr bool FAST = sizeof(T) == 2;
      Tacc q1 = act_fwd<Tacc, FAST>((Tacc)Cvt<T>::to_f(xq.v[2 * pr]), act),
           q2 = act_fwd<Tacc, FAST>((Tacc)Cvt<T>::to_f(xq.v[2 * pr + 1]), act);
      Tacc k1 = act_fwd<Tacc, FAST>((Tacc)Cvt<T>::to_f(xk.v[2 * pr]), act),
           k2 = act_fwd<Tacc, FAST>((Tacc)Cvt<T>::to_f(xk.v[2 * pr + 1]), act);
      if (theta != nullptr) {
        const Tacc c = rw.c[pr], s = rw.s[pr];
        const Tacc a1 = q1 * c - q2 * s, a2 = q1 * s + q2 * c;
        const Tacc b1 = k1 * c - k2 * s, b2 = k1 * s + k2 * c;
        q1 = a1, q2 = a2, k1 = b1, k2 = b2;
      }
      oq.v[2 * pr] = Cvt<T>::from_f(q1);
      oq.v[2 * pr + 1] = Cvt<T>::from_f(q2);
      ok.v[2 * pr] = Cvt<T>::from_f(k1);
      ok.v[2 * pr + 1] = Cvt<T>::from_f(k2);
    }
    stv(q + e, oq);
    stv(k + e, ok);
  }
}

constexpr int kRowsPerBlock = 64;

// grid (ceil(rows / 64), ceil(width/V / 256)) -- row blocks on x (no 65535 cap); a thread owns one 16-byte
// column vector and walks 64 rows.  dtheta partials per (row block, column block) land in `partial`
// [gridDim.x * gridDim.y][d/2] (deterministic; summed by reduce_theta_kernel)
template <typename T, typename Tacc>
__global__ void __launch_bounds__(256) prologue_bwd_kernel(const T* __restrict__ qp, const T* __restrict__ kp,
                                                           const double* __restrict__ theta, const T* __restrict__ dq,
                                                           const T* __restrict__ dk, T* __restrict__ dqp,
                                                           T* __restrict__ dkp, double* __restrict__ partial,
                                                           int64_t rows, int n, int width, int d, int64_t offset,
                                                           int act) {
  constexpr int V = Vec<T>::N;
  extern __shared__ double sdt[];  // [blockDim.x][V / 2]: this block's per-pair partials
  const int vw = width / V, hd = d >> 1;
  const int vc = blockIdx.y * blockDim.x + threadIdx.x;
  Tacc acc[V / 2];
#pragma unroll
  for (int pr = 0; pr < V / 2; ++pr) acc[pr] = 0;
  const int c0 = vc * V;
  if (vc < vw) {
    RotWalk<Tacc, V / 2> rw;
    if (theta != nullptr) rw.init(theta, c0 >> 1, hd);
    const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
    const int64_t r1 = r0 + kRowsPerBlock < rows ? r0 + kRowsPerBlock : rows;
#pragma unroll 2
    for (int64_t row = r0; row < r1; ++row) {
      const int64_t e = row * width + c0;
      const Vec<T> xq = ldv(qp + e), xk = ldv(kp + e), gq = ldv(dq + e), gk = ldv(dk + e);
      Vec<T> oq, ok;
      const int64_t tp = row % n;
      const int64_t pos = tp + offset;
      if (theta != nullptr) rw.at(pos, row == r0 || tp == 0 || ((row - r0) % kAnchor) == 0);
#pragma unroll
      for (int pr = 0; pr < V / 2; ++pr) {
        const Tacc xq1 = (Tacc)Cvt<T>::to_f(xq.v[2 * pr]), xq2 = (Tacc)Cvt<T>::to_f(xq.v[2 * pr + 1]);
        const Tacc xk1 = (Tacc)Cvt<T>::to_f(xk.v[2 * pr]), xk2 = (Tacc)Cvt<T>::to_f(xk.v[2 * pr + 1]);
        Tacc gq1 = (Tacc)Cvt<T>::to_f(gq.v[2 * pr]), gq2 = (Tacc)Cvt<T>::to_f(gq.v[2 * pr + 1]);
        Tacc gk1 = (Tacc)Cvt<T>::to_f(gk.v[2 * pr]), gk2 = (Tacc)Cvt<T>::to_f(gk.v[2 * pr + 1]);
        Tacc aq1, aq2, ak1, ak2, hq1, hq2, hk1, hk2;  // act and act' (one sigmoid each)
        constexpr bool FAST = sizeof(T) == 2;
        act_both<Tacc, FAST>(xq1, act, aq1, hq1);
        act_both<Tacc, FAST>(xq2, act, aq2, hq2);
        act_both<Tacc, FAST>(xk1, act, ak1, hk1);
        act_both<Tacc, FAST>(xk2, act, ak2, hk2);
        if (theta != nullptr) {
          const Tacc c = rw.c[pr], s = rw.s[pr];
          // rotated activations y (recomputed) for the angle gradient
          const Tacc yq1 = aq1 * c - aq2 * s, yq2 = aq1 * s + aq2 * c;
          const Tacc yk1 = ak1 * c - ak2 * s, yk2 = ak1 * s + ak2 * c;
          acc[pr] += (Tacc)pos * ((gq2 * yq1 - gq1 * yq2) + (gk2 * yk1 - gk1 * yk2));
          // dx = rot^-1 dy
          const Tacc rq1 = gq1 * c + gq2 * s, rq2 = -gq1 * s + gq2 * c;
          const Tacc rk1 = gk1 * c + gk2 * s, rk2 = -gk1 * s + gk2 * c;
          gq1 = rq1, gq2 = rq2, gk1 = rk1, gk2 = rk2;
        }
        oq.v[2 * pr] = Cvt<T>::from_f(gq1 * hq1);
        oq.v[2 * pr + 1] = Cvt<T>::from_f(gq2 * hq2);
        ok.v[2 * pr] = Cvt<T>::from_f(gk1 * hk1);
        ok.v[2 * pr + 1] = Cvt<T>::from_f(gk2 * hk2);
      }
      stv(dqp + e, oq);
      stv(dkp + e, ok);
    }
  }
  if (theta == nullptr) return;
#pragma unroll
  for (int pr = 0; pr < V / 2; ++pr) sdt[threadIdx.x * (V / 2) + pr] = vc < vw ? (double)acc[pr] : 0.0;
  __syncthreads();
  // fold the heads: pair p of the row belongs to angle p % hd; each angle sums its block-local pairs in
  // increasing order (no atomics, so dtheta is bitwise reproducible)
  const int npairs = blockDim.x * (V / 2);
  const int base = blockIdx.y * npairs;  // row pair index of this block's first pair
  double* dst = partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * hd;
  for (int j = threadIdx.x; j < hd; j += blockDim.x) {
    double sum = 0.0;
    for (int lp = ((j - base) % hd + hd) % hd; lp < npairs; lp += hd) sum += sdt[lp];
    dst[j] = sum;
  }
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
__device__ __forceinline__ Tacc warp_sum(Tacc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kEpiWarps = 8;  // rows per CTA, one warp each

// one warp per row; 16-byte vectors; the second sweep over the row hits L1
template <typename T, typename Tacc>
__global__ void __launch_bounds__(32 * kEpiWarps) epilogue_kernel(const T* __restrict__ a, const T* __restrict__ u,
                                                                  T* __restrict__ gated, Tacc* __restrict__ rawnorm,
                                                                  int64_t rows, int width, double eps) {
  constexpr int V = Vec<T>::N;
  const int64_t row = (int64_t)blockIdx.x * kEpiWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t off = row * width;
  Tacc ss = 0;
  for (int c = lane * V; c < width; c += 32 * V) {
    const Vec<T> x = ldv(a + off + c);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const Tacc f = (Tacc)Cvt<T>::to_f(x.v[e]);
      ss += f * f;
    }
  }
  ss = warp_sum(ss);
  const Tacc raw = sqrt(ss);
  const Tacc scale = sqrt((Tacc)width) / (raw > (Tacc)eps ? raw : (Tacc)eps);
  if (lane == 0) rawnorm[row] = raw;
  for (int c = lane * V; c < width; c += 32 * V) {
    const Vec<T> x = ldv(a + off + c);
    Vec<T> y;
    if (u != nullptr) {
      const Vec<T> g = ldv(u + off + c);
#pragma unroll
      for (int e = 0; e < V; ++e)
        y.v[e] = Cvt<T>::from_f((Tacc)Cvt<T>::to_f(x.v[e]) * scale * (Tacc)Cvt<T>::to_f(g.v[e]));
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) y.v[e] = Cvt<T>::from_f((Tacc)Cvt<T>::to_f(x.v[e]) * scale);
    }
    stv(gated + off + c, y);
  }
}

template <typename T, typename Tacc>
__global__ void __launch_bounds__(32 * kEpiWarps) epilogue_bwd_kernel(const T* __restrict__ dgated,
                                                                      const T* __restrict__ a, const T* __restrict__ u,
                                                                      const Tacc* __restrict__ rawnorm,
                                                                      T* __restrict__ da, T* __restrict__ du,
                                                                      int64_t rows, int width, double eps) {
  constexpr int V = Vec<T>::N;
  const int64_t row = (int64_t)blockIdx.x * kEpiWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t off = row * width;
  const Tacc raw = rawnorm[row];
  const Tacc r = raw > (Tacc)eps ? raw : (Tacc)eps;
  const Tacc scale = sqrt((Tacc)width) / r;
  Tacc dot = 0;  // sum_c a_c * dan_c
  for (int c = lane * V; c < width; c += 32 * V) {
    const Vec<T> x = ldv(a + off + c), g = ldv(dgated + off + c);
    if (u != nullptr) {
      const Vec<T> uu = ldv(u + off + c);
      Vec<T> o;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const Tacc xf = (Tacc)Cvt<T>::to_f(x.v[e]), gf = (Tacc)Cvt<T>::to_f(g.v[e]);
        dot += xf * gf * (Tacc)Cvt<T>::to_f(uu.v[e]);
        o.v[e] = Cvt<T>::from_f(gf * xf * scale);  // du = dgated * an
      }
      stv(du + off + c, o);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) dot += (Tacc)Cvt<T>::to_f(x.v[e]) * (Tacc)Cvt<T>::to_f(g.v[e]);
    }
  }
  dot = warp_sum(dot);
  // srmsnorm_backward: dx = dan sqrt(W)/r - [raw >= eps] x (x.dan / r^2) sqrt(W)/r
  const Tacc proj = raw >= (Tacc)eps ? dot / (r * r) : (Tacc)0;
  for (int c = lane * V; c < width; c += 32 * V) {
    const Vec<T> x = ldv(a + off + c), g = ldv(dgated + off + c);
    Vec<T> o;
    if (u != nullptr) {
      const Vec<T> uu = ldv(u + off + c);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const Tacc dan = (Tacc)Cvt<T>::to_f(g.v[e]) * (Tacc)Cvt<T>::to_f(uu.v[e]);
        o.v[e] = Cvt<T>::from_f((dan - (Tacc)Cvt<T>::to_f(x.v[e]) * proj) * scale);
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e)
        o.v[e] = Cvt<T>::from_f(((Tacc)Cvt<T>::to_f(g.v[e]) - (Tacc)Cvt<T>::to_f(x.v[e]) * proj) * scale);
    }
    stv(da + off + c, o);
  }
}

// the same with the row held in registers (width = NV x 32 lanes x V): one read of a, u, dgated
template <typename T, typename Tacc, int NV>
__global__ void __launch_bounds__(32 * kEpiWarps) epilogue_bwd_reg_kernel(const T* __restrict__ dgated,
                                                                          const T* __restrict__ a,
                                                                          const T* __restrict__ u,
                                                                          const Tacc* __restrict__ rawnorm,
                                                                          T* __restrict__ da, T* __restrict__ du,
                                                                          int64_t rows, int width, double eps) {
  constexpr int V = Vec<T>::N;
  const int64_t row = (int64_t)blockIdx.x * kEpiWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t off = row * width;
  Vec<T> xs[NV], gs[NV], us[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * V;
    xs[i] = ldv(a + off + c);
    gs[i] = ldv(dgated + off + c);
    if (u != nullptr) us[i] = ldv(u + off + c);
  }
  const Tacc raw = rawnorm[row];
  const Tacc r = raw > (Tacc)eps ? raw : (Tacc)eps;
  const Tacc scale = sqrt((Tacc)width) / r;
  Tacc dot = 0;  // sum_c a_c * dan_c
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * V;
    if (u != nullptr) {
      Vec<T> o;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const Tacc xf = (Tacc)Cvt<T>::to_f(xs[i].v[e]), gf = (Tacc)Cvt<T>::to_f(gs[i].v[e]);
        dot += xf * gf * (Tacc)Cvt<T>::to_f(us[i].v[e]);
        o.v[e] = Cvt<T>::from_f(gf * xf * scale);  // du = dgated * an
      }
      stv(du + off + c, o);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) dot += (Tacc)Cvt<T>::to_f(xs[i].v[e]) * (Tacc)Cvt<T>::to_f(gs[i].v[e]);
    }
  }
  dot = warp_sum(dot);
  const Tacc proj = raw >= (Tacc)eps ? dot / (r * r) : (Tacc)0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 32 + lane) * V;
    Vec<T> o;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const Tacc dan = (Tacc)Cvt<T>::to_f(gs[i].v[e]) * (u != nullptr ? (Tacc)Cvt<T>::to_f(us[i].v[e]) : (Tacc)1);
      o.v[e] = Cvt<T>::from_f((dan - (Tacc)Cvt<T>::to_f(xs[i].v[e]) * proj) * scale);
    }
    stv(da + off + c, o);
  }
}

// tensor-parallel GLA (parallel.py:138-178): gated = a * u (no norm) and the row's sum of squares
// of this shard's attention output, written as the last column of an augmented [rows, out_w + 1]
// buffer row (the all-reduce payload); the output projection fills columns [0, out_w)
template <typename T, typename Tacc>
__global__ void __launch_bounds__(32 * kEpiWarps) gate_rowsq_kernel(const T* __restrict__ a, const T* __restrict__ u,
                                                                    T* __restrict__ gated, Tacc* __restrict__ rowsq,
                                                                    int64_t rowsq_stride, int64_t rows, int width) {
  constexpr int V = Vec<T>::N;
  const int64_t row = (int64_t)blockIdx.x * kEpiWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t off = row * width;
  Tacc ss = 0;
  for (int c = lane * V; c < width; c += 32 * V) {
    const Vec<T> x = ldv(a + off + c);
    Vec<T> y;
    if (u != nullptr) {
      const Vec<T> g = ldv(u + off + c);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const Tacc f = (Tacc)Cvt<T>::to_f(x.v[e]);
        ss += f * f;
        y.v[e] = Cvt<T>::from_f(f * (Tacc)Cvt<T>::to_f(g.v[e]));
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const Tacc f = (Tacc)Cvt<T>::to_f(x.v[e]);
        ss += f * f;
        y.v[e] = x.v[e];
      }
    }
    stv(gated + off + c, y);
  }
  ss = warp_sum(ss);
  if (lane == 0) rowsq[row * rowsq_stride] = ss;
}

// y[row, :] = red[row, :out_w] * sqrt(out_w) / max(sqrt(red[row, out_w]), eps)   (parallel.py:176-178)
template <typename Tacc>
__global__ void __launch_bounds__(256) rowscale_kernel(const Tacc* __restrict__ red, Tacc* __restrict__ y,
                                                       int64_t rows, int out_w, double eps) {
  const int64_t row = blockIdx.x;
  if (row >= rows) return;
  const Tacc* r = red + row * (int64_t)(out_w + 1);
  const Tacc raw = sqrt(r[out_w]);
  const Tacc scale = sqrt((Tacc)out_w) / (raw > (Tacc)eps ? raw : (Tacc)eps);
  for (int c = threadIdx.x; c < out_w; c += blockDim.x) y[row * out_w + c] = r[c] * scale;
}

template <typename T, typename Tacc>
cudaError_t prologue_t(const GlaRows& g, const void* qp, const void* kp, const double* theta, void* q, void* k,
                       cudaStream_t st) {
  const int vw = g.width / Vec<T>::N;
  const int threads = vw >= 256 ? 256 : (vw + 31) / 32 * 32;
  const dim3 grid((unsigned)((g.rows + kRowsFwd - 1) / kRowsFwd), (unsigned)((vw + threads - 1) / threads));
  prologue_kernel<T, Tacc><<<grid, threads, 0, st>>>(
      static_cast<const T*>(qp), static_cast<const T*>(kp), theta, static_cast<T*>(q), static_cast<T*>(k), g.rows,
      g.n, g.width, g.d, g.offset, g.act);
  return cudaGetLastError();
}

template <typename T, typename Tacc>
cudaError_t prologue_bwd_t(const GlaRows& g, const void* qp, const void* kp, const double* theta, const void* dq,
                           const void* dk, void* dqp, void* dkp, double* partial, double* dtheta, cudaStream_t st) {
  const int vw = g.width / Vec<T>::N, hd = g.d / 2;
  const dim3 grid((unsigned)((g.rows + kRowsPerBlock - 1) / kRowsPerBlock), (unsigned)((vw + 255) / 256));
  const size_t smem = theta != nullptr ? (size_t)256 * (Vec<T>::N / 2) * sizeof(double) : 0;
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
  epilogue_kernel<T, Tacc><<<(unsigned)((g.rows + kEpiWarps - 1) / kEpiWarps), 32 * kEpiWarps, 0, st>>>(
      static_cast<const T*>(a), static_cast<const T*>(u), static_cast<T*>(gated), static_cast<Tacc*>(rawnorm), g.rows,
      g.width, eps);
  return cudaGetLastError();
}

template <typename T, typename Tacc>
cudaError_t epilogue_bwd_t(const GlaRows& g, const void* dgated, const void* a, const void* u, const void* rawnorm,
                           void* da, void* du, double eps, cudaStream_t st) {
  const unsigned blocks = (unsigned)((g.rows + kEpiWarps - 1) / kEpiWarps);
  const int per = 32 * Vec<T>::N;
  const int nv = g.width % per == 0 ? g.width / per : 0;
#define LA_EPI_BWD_ARGS                                                                                      \
  static_cast<const T*>(dgated), static_cast<const T*>(a), static_cast<const T*>(u),                        \
      static_cast<const Tacc*>(rawnorm), static_cast<T*>(da), static_cast<T*>(du), g.rows, g.width, eps
  switch (nv) {
    case 1: epilogue_bwd_reg_kernel<T, Tacc, 1><<<blocks, 32 * kEpiWarps, 0, st>>>(LA_EPI_BWD_ARGS); break;
    case 2: epilogue_bwd_reg_kernel<T, Tacc, 2><<<blocks, 32 * kEpiWarps, 0, st>>>(LA_EPI_BWD_ARGS); break;
    case 4: epilogue_bwd_reg_kernel<T, Tacc, 4><<<blocks, 32 * kEpiWarps, 0, st>>>(LA_EPI_BWD_ARGS); break;
    case 8: epilogue_bwd_reg_kernel<T, Tacc, 8><<<blocks, 32 * kEpiWarps, 0, st>>>(LA_EPI_BWD_ARGS); break;
    default: epilogue_bwd_kernel<T, Tacc><<<blocks, 32 * kEpiWarps, 0, st>>>(LA_EPI_BWD_ARGS);
  }
#undef LA_EPI_BWD_ARGS
  return cudaGetLastError();
}

template <typename T, typename Tacc>
cudaError_t gate_rowsq_t(const GlaRows& g, const void* a, const void* u, void* gated, void* rowsq,
                         int64_t rowsq_stride, cudaStream_t st) {
  gate_rowsq_kernel<T, Tacc><<<(unsigned)((g.rows + kEpiWarps - 1) / kEpiWarps), 32 * kEpiWarps, 0, st>>>(
      static_cast<const T*>(a), static_cast<const T*>(u), static_cast<T*>(gated), static_cast<Tacc*>(rowsq),
      rowsq_stride, g.rows, g.width);
  return cudaGetLastError();
}

}  // namespace

size_t gla_prologue_bwd_partial_bytes(const GlaRows& g) {
  // sized for the narrowest vector (fp64: one pair per thread), so it covers every dtype
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

cudaError_t gla_gate_rowsq(const GlaRows& g, const void* a, const void* u, void* gated, void* rowsq,
                           int64_t rowsq_stride, cudaStream_t st) {
  switch (g.dtype) {
    case LA_F64: return gate_rowsq_t<double, double>(g, a, u, gated, rowsq, rowsq_stride, st);
    case LA_F32: return gate_rowsq_t<float, float>(g, a, u, gated, rowsq, rowsq_stride, st);
    default: return gate_rowsq_t<__nv_bfloat16, float>(g, a, u, gated, rowsq, rowsq_stride, st);
  }
}

cudaError_t gla_rowscale(bool acc_double, const void* red, void* y, int64_t rows, int out_w, double eps,
                         cudaStream_t st) {
  if (acc_double)
    rowscale_kernel<double><<<(unsigned)rows, 256, 0, st>>>(static_cast<const double*>(red), static_cast<double*>(y),
                                                             rows, out_w, eps);
  else
    rowscale_kernel<float><<<(unsigned)rows, 256, 0, st>>>(static_cast<const float*>(red), static_cast<float*>(y),
                                                            rows, out_w, eps);
  return cudaGetLastError();
}

}  // namespace la
