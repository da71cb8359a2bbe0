// la_simt.cu -- CUDA-core (FFMA / DFMA) kernels for every dtype and d <= 128.
//
// This is the precision path: fp64 ("reference" precision, kernels.py:66) and
// fp32 ("working") must meet the reference's 1e-10 / 1e-4 bars, which TF32
// tensor-core math cannot (SURVEY.md §7 hard part 5).  It is also the generic
// fallback *inside CUDA* for shapes the tcgen05 kernels do not cover (d != 128),
// never a CPU path.
//
// One CTA owns one (batch, head, segment); it walks the segment's chunks in
// order (fwd) or reverse order (rev), keeping the d x d state in shared memory
// in the accumulation type.  Per chunk (see la_common.cuh for the algebra):
//   S   = (A B^T) * M                                   (b x b)
//   out = S C + out_scale * (A state)                   (b x d)
//   state = lam^b state + sum_j in_scale[j] B[j]^T C[j] (d x d)
#include "la_common.cuh"
#include "la_scan.cuh"
#include "la_simt.cuh"

namespace la {

namespace {

constexpr int kThreads = 256;

template <typename Tacc>
__device__ __forceinline__ Tacc load_state(const void* base, int64_t off, int d, int r, int c, int T) {
  const Tacc* p = reinterpret_cast<const Tacc*>(base) + off;
  return T ? p[(int64_t)c * d + r] : p[(int64_t)r * d + c];
}

template <typename Tin, typename Tacc, int C, bool STATE_ONLY>
__global__ void __launch_bounds__(kThreads) simt_pass_kernel(PassDesc p) {
  constexpr int RP = C / 16;                      // chunk rows (and keys) per thread
  constexpr int CP = 8;                           // feature columns per thread: 16 x 8 = 128 >= d
  constexpr int SU = sizeof(Tacc) == 8 ? 2 : 4;   // state rows per thread per pass
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = p.d;
  const int ld = d + 1;  // padded row stride of the chunk tiles
  Tacc* sKV = reinterpret_cast<Tacc*>(smem_raw);
  Tacc* sA = sKV + d * d;
  Tacc* sB = sA + C * ld;
  Tacc* sC = sB + C * ld;
  Tacc* sS = sC + C * ld;
  Tacc* pw = sS + C * (C + 1);  // lam^0 .. lam^C

  const int tid = threadIdx.x;
  const int seg = blockIdx.x;
  const int bh = blockIdx.y;
  const int bi = bh / p.heads, hi = bh % p.heads;
  const int p0 = seg * p.seg_len;
  const int p1 = min(p.n, p0 + p.seg_len);
  const int nchunks = (p1 - p0 + C - 1) / C;
  const double lam = load_decay(p.lam, hi);

  auto base = [&](const Strides3& s) { return (int64_t)bi * s.b + (int64_t)hi * s.h; };
  const Tin* A = STATE_ONLY ? nullptr : reinterpret_cast<const Tin*>(p.a) + base(p.sa);
  const Tin* Bm = reinterpret_cast<const Tin*>(p.b) + base(p.sbb);
  const Tin* Cm = reinterpret_cast<const Tin*>(p.c) + base(p.sc);
  Tin* O = STATE_ONLY ? nullptr : reinterpret_cast<Tin*>(p.out) + base(p.so);

  // Power ladder in fp64 by repeated multiplication, then cast
  // (the reference builds its ladders the same way: matrixops.py:104-119).
  if (tid == 0) {
    double x = lam / lam;  // 1, or NaN for an invalid lam (load_decay)
    for (int k = 0; k <= C; ++k) {
      pw[k] = (Tacc)x;
      x *= lam;
    }
  }
  // State entering this segment.
  const bool have_in = (!STATE_ONLY) && p.state_in != nullptr;
  const int64_t in_off = (int64_t)bh * p.state_in_bh_stride + (int64_t)seg * p.state_in_seg_stride;
  for (int e = tid; e < d * d; e += kThreads) {
    const int r = e / d, c = e % d;
    sKV[e] = have_in ? load_state<Tacc>(p.state_in, in_off, d, r, c, p.state_in_T) : (Tacc)0;
  }
  __syncthreads();

  for (int ci = 0; ci < nchunks; ++ci) {
    const int t = p.rev ? (nchunks - 1 - ci) : ci;
    const int r0 = p0 + t * C;
    const int b = min(C, p1 - r0);

    for (int idx = tid; idx < b * d; idx += kThreads) {
      const int i = idx / d, k = idx % d;
      const int64_t r = r0 + i;
      if (!STATE_ONLY) sA[i * ld + k] = (Tacc)Cvt<Tin>::to_f(A[r * p.sa.n + k]);
      sB[i * ld + k] = (Tacc)Cvt<Tin>::to_f(Bm[r * p.sbb.n + k]);
      sC[i * ld + k] = (Tacc)Cvt<Tin>::to_f(Cm[r * p.sc.n + k]);
    }
    __syncthreads();

    // Register tiles (a 16 x 16 thread grid): each thread owns RP rows x up to CP columns of every
    // product and reuses each shared-memory operand it loads across the whole tile.
    const int tr = tid >> 4, tc = tid & 15;
    if (!STATE_ONLY) {
      // S = (A B^T) * M: rows tr*RP .. +RP, keys tc*RP .. +RP
      {
        Tacc acc[RP][RP];
#pragma unroll
        for (int x = 0; x < RP; ++x)
#pragma unroll
          for (int y = 0; y < RP; ++y) acc[x][y] = 0;
        for (int k = 0; k < d; ++k) {
          Tacc av[RP], bv[RP];
#pragma unroll
          for (int x = 0; x < RP; ++x) av[x] = sA[(tr * RP + x) * ld + k];
#pragma unroll
          for (int y = 0; y < RP; ++y) bv[y] = sB[(tc * RP + y) * ld + k];
#pragma unroll
          for (int x = 0; x < RP; ++x)
#pragma unroll
            for (int y = 0; y < RP; ++y) acc[x][y] += av[x] * bv[y];
        }
#pragma unroll
        for (int x = 0; x < RP; ++x)
#pragma unroll
          for (int y = 0; y < RP; ++y) {
            const int i = tr * RP + x, j = tc * RP + y;
            const bool keep = i < b && j < b && (p.rev ? (j >= i) : (j <= i));
            sS[i * (C + 1) + j] = keep ? acc[x][y] * pw[p.rev ? (j - i) : (i - j)] : (Tacc)0;
          }
      }
      __syncthreads();
      // out = S C + out_scale * (A state): rows tr*RP .. +RP, columns tc + 16 q
      {
        Tacc intra[RP][CP], inter[RP][CP];
#pragma unroll
        for (int x = 0; x < RP; ++x)
#pragma unroll
          for (int q = 0; q < CP; ++q) intra[x][q] = inter[x][q] = 0;
        // S is zero outside the causal band, so the key range only needs to cover this tile's rows
        const int jlo = p.rev ? min(tr * RP, b) : 0;
        const int jhi = p.rev ? b : min(tr * RP + RP, b);
        for (int j = jlo; j < jhi; ++j) {
          Tacc sv[RP], cv[CP];
#pragma unroll
          for (int x = 0; x < RP; ++x) sv[x] = sS[(tr * RP + x) * (C + 1) + j];
#pragma unroll
          for (int q = 0; q < CP; ++q) cv[q] = (tc + 16 * q < d) ? sC[j * ld + tc + 16 * q] : (Tacc)0;
#pragma unroll
          for (int x = 0; x < RP; ++x)
#pragma unroll
            for (int q = 0; q < CP; ++q) intra[x][q] += sv[x] * cv[q];
        }
        for (int k = 0; k < d; ++k) {
          Tacc av[RP], kv[CP];
#pragma unroll
          for (int x = 0; x < RP; ++x) av[x] = sA[(tr * RP + x) * ld + k];
#pragma unroll
          for (int q = 0; q < CP; ++q) kv[q] = (tc + 16 * q < d) ? sKV[k * d + tc + 16 * q] : (Tacc)0;
#pragma unroll
          for (int x = 0; x < RP; ++x)
#pragma unroll
            for (int q = 0; q < CP; ++q) inter[x][q] += av[x] * kv[q];
        }
#pragma unroll
        for (int x = 0; x < RP; ++x) {
          const int i = tr * RP + x;
          if (i >= b) continue;
          const Tacc osc = pw[p.rev ? (b - 1 - i) : (i + 1)];
#pragma unroll
          for (int q = 0; q < CP; ++q) {
            const int col = tc + 16 * q;
            if (col < d) O[(int64_t)(r0 + i) * p.so.n + col] = Cvt<Tin>::from_f(intra[x][q] + osc * inter[x][q]);
          }
        }
      }
      __syncthreads();
    }
    // state <- lam^b state + sum_j in_scale[j] B[j]^T C[j]: state rows tr + 16 u, columns tc + 16 q,
    // in row passes of SU rows per thread (bounded registers for fp64 at d = 128)
    {
      const Tacc decay = pw[b];
      for (int u0 = 0; u0 * 16 < d; u0 += SU) {
        Tacc acc[SU][CP];
#pragma unroll
        for (int u = 0; u < SU; ++u)
#pragma unroll
          for (int q = 0; q < CP; ++q) acc[u][q] = 0;
        for (int j = 0; j < b; ++j) {
          const Tacc isc = pw[p.rev ? (j + 1) : (b - 1 - j)];
          Tacc bv[SU], cv[CP];
#pragma unroll
          for (int u = 0; u < SU; ++u) {
            const int k = tr + 16 * (u0 + u);
            bv[u] = k < d ? isc * sB[j * ld + k] : (Tacc)0;
          }
#pragma unroll
          for (int q = 0; q < CP; ++q) cv[q] = (tc + 16 * q < d) ? sC[j * ld + tc + 16 * q] : (Tacc)0;
#pragma unroll
          for (int u = 0; u < SU; ++u)
#pragma unroll
            for (int q = 0; q < CP; ++q) acc[u][q] += bv[u] * cv[q];
        }
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          const int k = tr + 16 * (u0 + u);
          if (k >= d) continue;
#pragma unroll
          for (int q = 0; q < CP; ++q) {
            const int col = tc + 16 * q;
            if (col >= d) continue;
            Tacc a = acc[u][q];
#ifdef LA_MUTATE_DKV
            if (p.rev) a = -a;  // fault injection: the reference's `_dkv_step` sign flip (test_kernels.py:249-268)
#endif
            sKV[k * d + col] = decay * sKV[k * d + col] + a;
          }
        }
      }
    }
    __syncthreads();
  }

  if (STATE_ONLY) {
    Tacc* dst = reinterpret_cast<Tacc*>(p.delta_out) + ((int64_t)bh * p.nseg + seg) * d * d;
    for (int e = tid; e < d * d; e += kThreads) dst[e] = sKV[e];
  } else if (p.state_out != nullptr) {
    const bool last = p.rev ? (seg == 0) : (seg == p.nseg - 1);
    if (last) {
      Tacc* dst = reinterpret_cast<Tacc*>(p.state_out) + (int64_t)bh * d * d;
      for (int e = tid; e < d * d; e += kThreads) {
        const int r = e / d, c = e % d;
        dst[p.state_out_T ? (c * d + r) : e] = sKV[e];
      }
    }
  }
}

template <typename Tacc, int C>
size_t simt_smem_bytes(int d) {
  return sizeof(Tacc) * ((size_t)d * d + 3 * (size_t)C * (d + 1) + (size_t)C * (C + 1) + C + 1);
}

template <typename Tin, typename Tacc, int C, bool STATE_ONLY>
cudaError_t launch_simt(const PassDesc& p, cudaStream_t st) {
  auto kern = simt_pass_kernel<Tin, Tacc, C, STATE_ONLY>;
  const size_t smem = simt_smem_bytes<Tacc, C>(p.d);
  static std::atomic<bool> smem_set[64] = {};  // raised once to the d = 128 footprint, which covers every d <= 128
  cudaError_t err = set_smem_once(kern, (int)simt_smem_bytes<Tacc, C>(128), smem_set);
  if (err != cudaSuccess) return err;
  dim3 grid(p.nseg, p.batch * p.heads);
  kern<<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

template <typename Tin> struct SimtTraits;
template <> struct SimtTraits<double> { using Acc = double; static constexpr int C = 16; };
template <> struct SimtTraits<float> { using Acc = float; static constexpr int C = 32; };
template <> struct SimtTraits<__nv_bfloat16> { using Acc = float; static constexpr int C = 32; };

template <typename Tin>
cudaError_t simt_launch_t(const PassDesc& p, bool state_only, cudaStream_t st) {
  using Acc = typename SimtTraits<Tin>::Acc;
  constexpr int C = SimtTraits<Tin>::C;
  return state_only ? launch_simt<Tin, Acc, C, true>(p, st) : launch_simt<Tin, Acc, C, false>(p, st);
}

}  // namespace

int simt_chunk(int dtype) { return dtype == LA_F64 ? SimtTraits<double>::C : SimtTraits<float>::C; }

cudaError_t simt_launch(int dtype, const PassDesc& p, bool state_only, cudaStream_t st) {
  switch (dtype) {
    case LA_F64: return simt_launch_t<double>(p, state_only, st);
    case LA_F32: return simt_launch_t<float>(p, state_only, st);
    case LA_BF16: return simt_launch_t<__nv_bfloat16>(p, state_only, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace la
