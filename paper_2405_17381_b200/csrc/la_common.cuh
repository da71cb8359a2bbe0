// la_common.cuh -- shared types for the Lightning Attention CUDA path.
//
// Every kernel in this library implements ONE primitive, a "pass" of causal
// decayed linear attention over a (batch, head) sequence:
//
//   fwd  (rev = 0):  out[t] = sum_{s<=t} lam^(t-s) (a[t].b[s]) c[s]
//                    state F(p) = sum_{s<p}  lam^(p-1-s) b[s] c[s]^T
//   rev  (rev = 1):  out[s] = sum_{t>=s} lam^(t-s) (a[s].b[t]) c[t]
//                    state R(p) = sum_{t>=p} lam^(t-p+1) b[t] c[t]^T
//
// The reference's forward is the fwd pass on (q, k, v) (kernels.py:253-284).
// Its backward (kernels.py:287-334) is three passes:
//   dq = fwd(a=do, b=v, c=k)   state = kv^T   (sweep 1, kernels.py:309-318)
//   dk = rev(a=v,  b=do, c=q)  state = dkv^T  (sweep 2, dk line kernels.py:331)
//   dv = rev(a=k,  b=q,  c=do) state = dkv    (sweep 2, dv line kernels.py:332)
// and the reverse pass's state R is exactly the reference's `state.dkv`,
// updated after use (kernels.py:333).  Per chunk of b rows (local i, j):
//   fwd: mask M[i][j] = lam^(i-j) (j <= i); out-scale lam^(i+1);  in-scale lam^(b-1-j)
//   rev: mask M[i][j] = lam^(j-i) (j >= i); out-scale lam^(b-1-i); in-scale lam^(j+1)
//   state <- lam^b * state + sum_j in_scale[j] b[j] c[j]^T
#pragma once
#include <atomic>

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/lightning_attn.h"

namespace la {

constexpr int kNumSMs = 148;  // B200: the planner's default when the device cannot be queried

// SM count of the calling thread's current device (cached per device ordinal); the segment planners
// size their grids from it, so a MIG slice or another part plans for what it has
int device_sms();

// The decay of head h.  A lam outside (0, 1] or NaN -- which the reference rejects with DomainError
// (matrixops.py:72-77) -- is read as NaN, so every output of the call comes out NaN instead of silently
// wrong: the ABI takes lam on the device and does not read it back per call (LA_FLAG_CHECK_DECAY and
// la_check_decay report it as LA_ERR_DOMAIN).  Ladders multiply lam^0 by `lam / lam` (exactly 1 for a
// valid lam, NaN otherwise) so even the diagonal terms are poisoned.
__device__ __forceinline__ double load_decay(const double* lam, int h) {
  const double l = lam[h];
  return (l > 0.0 && l <= 1.0) ? l : __longlong_as_double(0x7ff8000000000000LL);
}

// Load/convert helpers for the three operand dtypes.
template <typename T> struct Cvt;
template <> struct Cvt<float> {
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct Cvt<double> {
  __device__ __forceinline__ static double to_f(double x) { return x; }
  __device__ __forceinline__ static double from_f(double x) { return x; }
};
template <> struct Cvt<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// Scan-order liveness of summary sub-segment j of a segment whose last sub-segment is `last` (la_scan.cu):
// a sub-segment reaches an entering state only through the decays lam^len of the sub-segments after it in
// scan order (fwd: higher j, rev: lower j) within its segment.  When one of those factors is exactly 0 in
// the accumulation type, the scan's  s = dec * s + delta  discards it exactly (states are finite), so
// neither the summary pass nor the scan touch it.  zero_full: (Tacc)lam^sub_len == 0 (every sub-segment but
// a segment's last is full); zero_last: (Tacc)lam^len(last) == 0.  Short-memory heads (e.g. TNL's lower
// layers, lam <= 0.63) thereby summarise only the tail of each segment -- the same arithmetic result.
__device__ __forceinline__ bool sub_dead(int j, int last, int rev, bool zero_full, bool zero_last) {
  if (rev) return j > 0 && zero_full;
  if (j >= last) return false;
  return (j + 1 < last && zero_full) || zero_last;
}

// Element strides of one operand: batch, head, position (the feature stride is 1).
struct Strides3 {
  int64_t b, h, n;
};

// One pass over all (batch, head) sequences, split into `nseg` segments of
// `seg_len` positions (a multiple of the kernel's chunk).  Every operand has its
// own strides; the feature stride is 1.
struct PassDesc {
  const void* a;
  const void* b;
  const void* c;
  void* out;              // nullptr in state-only mode
  Strides3 sa, sbb, sc, so;  // strides of a, b, c, out
  int batch, heads, n, d;
  const double* lam;      // device [heads]
  int rev;
  int seg_len, nseg;
  // state entering each segment (fwd: at its left edge, rev: at its right edge)
  const void* state_in;   // nullable
  int64_t state_in_bh_stride, state_in_seg_stride;
  int state_in_T;         // 1: stored transposed
  // final state of the pass (fwd: F(n), rev: R(0)), written by the last segment processed
  void* state_out;        // nullable
  int state_out_T;
  // state-only mode: local summaries of sub-segments, [bh][nseg * sub_per_seg][d][d].  Sub-segment j of
  // segment g covers [g seg_len + j sub_len, min(.. + sub_len, (g + 1) seg_len, n)); only segments
  // g_lo..g_hi are summarised (the forward never needs the last segment's, the reverse pass never the
  // first's), so the summary work spreads over all SMs and covers only the rows a scan needs.
  void* delta_out;
  int sub_len, sub_per_seg, g_lo, g_hi;
};

// Segment plan shared by host code of every backend.
// Raise a kernel's dynamic shared-memory limit once per (kernel, device) instead of on every launch
// (cudaFuncSetAttribute costs microseconds of host time).  `done` is the caller's per-kernel flag
// array, indexed by device ordinal.
template <typename K>
inline cudaError_t set_smem_once(K kernel, int bytes, std::atomic<bool> (&done)[64]) {
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev >= 0 && dev < 64 && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
  err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);  // idempotent
  if (err == cudaSuccess && dev >= 0 && dev < 64) done[dev].store(true, std::memory_order_release);
  return err;
}

#ifndef LA_PDL
#define LA_PDL 1
#endif
// Launch with programmatic stream serialization (PDL, see griddep_wait in la_ptx.cuh) so the kernel's prologue
// overlaps the previous kernel's tail; LA_PDL=0 builds plain launches (A/B).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = LA_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct Plan {
  int chunk;        // rows per chunk in the kernel
  int nseg;         // segments per (b, h)
  int seg_len;      // positions per segment (multiple of chunk)
  int nseg_ws;      // segments the workspace is sized for: independent of n (kernels.py:342-368 c05)
  int sub_per_seg;  // summary sub-segments per segment (1: one summary per segment)
  int sub_len;      // positions per summary sub-segment (multiple of chunk)
  int nsub_ws;      // summary slots per (b, h) the workspace is sized for (>= nseg * sub_per_seg)
};

inline Plan make_plan(int64_t bh, int64_t n, int chunk, int64_t want_segments, int64_t target_ctas,
                      int64_t min_chunks_per_seg) {
  Plan p;
  p.chunk = chunk;
  int64_t nchunks = (n + chunk - 1) / chunk;
  int64_t nseg = want_segments;
  if (nseg <= 0) {
    nseg = (target_ctas + bh - 1) / bh;
    int64_t max_seg = nchunks / (min_chunks_per_seg > 0 ? min_chunks_per_seg : 1);
    if (max_seg < 1) max_seg = 1;
    if (nseg > max_seg) nseg = max_seg;
  }
  if (nseg < 1) nseg = 1;
  if (nseg > nchunks) nseg = nchunks;
  int64_t cap = want_segments > 0 ? want_segments : (target_ctas + bh - 1) / bh;
  p.nseg_ws = (int)(cap < 1 ? 1 : cap);
  int64_t chunks_per_seg = (nchunks + nseg - 1) / nseg;
  p.seg_len = (int)(chunks_per_seg * chunk);
  p.nseg = (int)((n + p.seg_len - 1) / p.seg_len);
  p.sub_per_seg = 1;
  p.sub_len = p.seg_len;
  p.nsub_ws = p.nseg_ws;
  return p;
}

// Split each segment into summary sub-segments so that one summary launch over the segments a scan
// needs (all but one) puts about `target_ctas` CTAs of >= `min_chunks` chunks each on the GPU.
// `nsub_cap` bounds nseg * sub_per_seg (the workspace's summary slots).
inline void plan_subsegments(Plan& p, int64_t bh, int64_t target_ctas, int64_t min_chunks, int64_t nsub_cap) {
  p.sub_per_seg = 1;
  p.sub_len = p.seg_len;
  if (p.nseg <= 1) return;
  const int64_t cps = p.seg_len / p.chunk;
  int64_t sps = target_ctas / (bh * (p.nseg - 1));
  const int64_t max_sps = cps / (min_chunks > 0 ? min_chunks : 1);
  if (sps > max_sps) sps = max_sps;
  if (sps * p.nseg > nsub_cap) sps = nsub_cap / p.nseg;
  if (sps < 1) sps = 1;
  const int64_t sub_chunks = (cps + sps - 1) / sps;
  p.sub_len = (int)(sub_chunks * p.chunk);
  p.sub_per_seg = (int)((cps + sub_chunks - 1) / sub_chunks);
}

}  // namespace la
