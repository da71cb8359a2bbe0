// la_api.cu -- the C ABI (include/lightning_attn.h): validation, planning and
// the pass orchestration that maps the reference's forward/backward onto the
// single "pass" primitive (la_common.cuh).
//
// Validation mirrors the reference's error classes:
//   LA_ERR_DOMAIN  n/d < 1, B < 1, bad precision      (kernels.py:84-91)
//   LA_ERR_SHAPE   missing operands, bad strides      (kernels.py:137-146)
// lam in (0, 1] (matrixops.py:72-77): the ABI takes a device array so calls stay
// asynchronous and graph-capturable; every kernel reads lam through load_decay,
// which turns an invalid value into NaN outputs (never silently wrong ones), and
// la_check_decay / LA_FLAG_CHECK_DECAY report it as LA_ERR_DOMAIN.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <string>

#include <vector>

#include <cuda.h>

#include "la_common.cuh"
#include "la_decode.cuh"
#include "la_gla.cuh"
#include "la_scan.cuh"
#include "la_simt.cuh"
#include "la_tc.cuh"

namespace la {

int device_sms() {
  static std::atomic<int> cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSMs;
  const int hit = cache[dev].load(std::memory_order_relaxed);
  if (hit > 0) return hit;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) return kNumSMs;
  cache[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

}  // namespace la

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t err, const char* where) {
  return fail(LA_ERR_CUDA, "%s: %s (%s) %s", where, cudaGetErrorName(err), cudaGetErrorString(err), la::tc_detail());
}

int validate(const la_desc* desc) {
  if (desc == nullptr) return fail(LA_ERR_SHAPE, "null descriptor");
  if (desc->n < 1 || desc->d < 1)
    return fail(LA_ERR_DOMAIN, "need n >= 1 and d >= 1, got n=%lld, d=%lld", (long long)desc->n,
                (long long)desc->d);
  if (desc->batch < 1 || desc->heads < 1)
    return fail(LA_ERR_SHAPE, "need batch >= 1 and heads >= 1, got batch=%lld, heads=%lld",
                (long long)desc->batch, (long long)desc->heads);
  if (desc->block < 0) return fail(LA_ERR_DOMAIN, "block size must be >= 1, got %lld", (long long)desc->block);
  if (desc->dtype != LA_F32 && desc->dtype != LA_F64 && desc->dtype != LA_BF16)
    return fail(LA_ERR_DOMAIN, "dtype must be LA_F32, LA_F64 or LA_BF16, got %d", desc->dtype);
  if (desc->backend < LA_BACKEND_AUTO || desc->backend > LA_BACKEND_TCGEN05)
    return fail(LA_ERR_DOMAIN, "unknown backend %d", desc->backend);
  if (desc->segments < 0) return fail(LA_ERR_DOMAIN, "segments must be >= 0");
  if (desc->segments > 65535) return fail(LA_ERR_UNSUPPORTED, "segments %lld > 65535", (long long)desc->segments);
  for (int i = 0; i < 3; ++i)
    if (desc->stride[i] < 0) return fail(LA_ERR_SHAPE, "negative stride");
  if (desc->stride[2] < desc->d) return fail(LA_ERR_SHAPE, "position stride %lld < d", (long long)desc->stride[2]);
  if (desc->n > (int64_t)INT32_MAX || desc->batch * desc->heads > 65535)
    return fail(LA_ERR_UNSUPPORTED, "n or batch*heads beyond this build's grid limits");
  if (desc->d > 128) return fail(LA_ERR_UNSUPPORTED, "head dim d=%lld > 128 is not implemented", (long long)desc->d);
  return LA_OK;
}

// Every operand's (batch, head, position) strides: the desc's triple unless the caller passed its own.
struct OpStrides {
  la::Strides3 s[8];
};

// `used`: bitmask of the la_operand slots this call reads or writes
int op_strides(const la_desc* desc, const la_tensor_strides* ts, unsigned used, OpStrides* out) {
  for (int i = 0; i < 8; ++i) {
    const int64_t* src = ts != nullptr ? ts->s[i] : desc->stride;
    out->s[i] = la::Strides3{src[0], src[1], src[2]};
  }
  if (ts != nullptr)
    for (int i = 0; i < 8; ++i) {
      if (!(used >> i & 1u)) continue;
      const la::Strides3& x = out->s[i];
      if (x.b < 0 || x.h < 0 || x.n < 0) return fail(LA_ERR_SHAPE, "operand %d: negative stride", i);
      if (x.n < desc->d) return fail(LA_ERR_SHAPE, "operand %d: position stride %lld < d", i, (long long)x.n);
    }
  return LA_OK;
}

// Which backend serves this descriptor (and, for the _ex calls, these operand strides).
// tensor-core eligibility: bf16 (la_tc.cu) or fp32 (la_tc32.cu), d = 128, 16-byte strides
bool tc_eligible(int dtype, int64_t d, const int64_t* strides) {
  return la::tc_supported(dtype, (int)d, strides, 1) || la::tc32_supported(dtype, (int)d, strides, 1);
}

int pick_backend(const la_desc* desc, int* backend, const OpStrides* ops = nullptr, unsigned used = 0) {
  bool tc_ok = tc_eligible(desc->dtype, desc->d, desc->stride);
  if (ops != nullptr)
    for (int i = 0; i < 8; ++i) {
      if (!(used >> i & 1u)) continue;
      const int64_t t[3] = {ops->s[i].b, ops->s[i].h, ops->s[i].n};
      tc_ok = tc_ok && tc_eligible(desc->dtype, desc->d, t);
    }
  if (desc->backend == LA_BACKEND_TCGEN05) {
    if (!tc_ok)
      return fail(LA_ERR_UNSUPPORTED,
                  "tcgen05 backend needs bf16 or fp32, d = 128, 16-byte aligned strides (dtype=%d d=%lld)",
                  desc->dtype, (long long)desc->d);
    *backend = LA_BACKEND_TCGEN05;
  } else if (desc->backend == LA_BACKEND_SIMT) {
    *backend = LA_BACKEND_SIMT;
  } else {
    *backend = tc_ok ? LA_BACKEND_TCGEN05 : LA_BACKEND_SIMT;
  }
  return LA_OK;
}

#ifndef LA_SIMT_MIN_CHUNKS
#define LA_SIMT_MIN_CHUNKS 1  // chunks per segment on the SIMT path (latency-bound: more CTAs win)
#endif

la::Plan plan_for(const la_desc* desc, int backend) {
  const int64_t bh = desc->batch * desc->heads;
  const int sms = la::device_sms();
  if (backend == LA_BACKEND_TCGEN05 && desc->dtype == LA_F32) return la::tc32_plan(bh, desc->n, desc->segments, sms);
  if (backend == LA_BACKEND_TCGEN05) return la::tc_plan(bh, desc->n, (int)desc->d, desc->segments, sms);
  return la::make_plan(bh, desc->n, la::simt_chunk(desc->dtype), desc->segments, 2 * sms, LA_SIMT_MIN_CHUNKS);
}

size_t acc_bytes(int dtype) { return dtype == LA_F64 ? sizeof(double) : sizeof(float); }

// Workspace: per-segment summaries | per-segment entering states, each [bh][nseg][d][d] in the
// accumulation type; sized for the plan's segment cap so it does not depend on n.
size_t ws_bytes_for(const la_desc* desc, int backend, const la::Plan& plan) {
  (void)backend;
  if (plan.nseg_ws <= 1) return 0;
  return acc_bytes(desc->dtype) * (size_t)(desc->batch * desc->heads) * (plan.nsub_ws + plan.nseg_ws) * desc->d *
         desc->d;
}

la::PassDesc base_pass(const la_desc* desc, const la::Plan& plan, const double* lam) {
  la::PassDesc p;
  std::memset(&p, 0, sizeof(p));
  p.sa = p.sbb = p.sc = p.so = la::Strides3{desc->stride[0], desc->stride[1], desc->stride[2]};
  p.batch = (int)desc->batch;
  p.heads = (int)desc->heads;
  p.n = (int)desc->n;
  p.d = (int)desc->d;
  p.lam = lam;
  p.seg_len = plan.seg_len;
  p.nseg = plan.nseg;
  p.sub_len = plan.sub_len;
  p.sub_per_seg = plan.sub_per_seg;
  p.g_lo = 0;
  p.g_hi = plan.nseg - 1;
  return p;
}

cudaError_t launch(int backend, int dtype, const la::PassDesc& p, bool state_only, cudaStream_t st) {
  if (backend == LA_BACKEND_TCGEN05) {
    if (!la::tc_pointers_ok(p)) return cudaErrorMisalignedAddress;  // TMA needs 16-byte aligned bases
    return dtype == LA_F32 ? la::tc32_launch(p, state_only, st) : la::tc_launch(p, state_only, st);
  }
  return la::simt_launch(dtype, p, state_only, st);
}

// Entering state of every segment of a pass (p.b, p.c, p.rev; p.state_in = the caller's state at the
// sequence edge, p.state_in_T its orientation): sub-segment summaries into `delta`, then the decayed
// scan into `seg_in` ([bh][nseg][d][d], kernel orientation).  The segment at the far end of the pass
// (fwd: the last, rev: the first) feeds no entering state, so it is not summarised.
// `resume`: the summaries are already in `delta` (left there by la_fwd_state / la_bwd_state, which
// summarise every segment with the same plan), only the scan runs.
cudaError_t segment_states(int backend, int dtype, const la::PassDesc& p, void* delta, void* seg_in, cudaStream_t st,
                           bool resume = false) {
  la::PassDesc s = p;
  s.a = nullptr;
  s.out = nullptr;
  s.state_in = nullptr;
  s.state_out = nullptr;
  s.delta_out = delta;
  s.g_lo = p.rev ? 1 : 0;
  s.g_hi = p.rev ? p.nseg - 1 : p.nseg - 2;
  cudaError_t err = resume ? cudaSuccess : launch(backend, dtype, s, true, st);
  if (err != cudaSuccess) return err;
  return la::launch_segment_scan(dtype == LA_F64, delta, seg_in, p.state_in, p.state_in_T, nullptr, 0, p.lam,
                                 p.batch * p.heads, p.heads, p.d, s, st);
}

// The main pass.  With one segment the caller's edge state is used as is; with several, the entering
// states `seg_in` (orientation seg_T) must already be computed.
cudaError_t main_pass(int backend, int dtype, la::PassDesc p, const void* seg_in, int seg_T, cudaStream_t st,
                      const la::GlaEpilogue* epi = nullptr) {
  const int64_t dd = (int64_t)p.d * p.d;
  if (p.nseg > 1) {
    p.state_in = seg_in;
    p.state_in_T = seg_T;
    p.state_in_bh_stride = (int64_t)p.nseg * dd;
    p.state_in_seg_stride = dd;
  } else {
    p.state_in_bh_stride = dd;
    p.state_in_seg_stride = 0;
  }
  if (epi != nullptr) return la::tc_epi_launch(p, *epi, st);  // the fused GLA core backward's dq pass
  return launch(backend, dtype, p, false, st);
}

// delta / seg_in regions of the workspace
void* ws_delta(void* ws) { return ws; }
void* ws_seg_in(void* ws, const la_desc* desc, const la::Plan& plan) {
  return static_cast<char*>(ws) + acc_bytes(desc->dtype) * (size_t)(desc->batch * desc->heads) * plan.nsub_ws *
                                      desc->d * desc->d;
}

// This library carries its own (static) CUDA runtime.  A caller's thread may have selected its device
// only through another runtime instance (e.g. torch's autograd worker threads), so every entry binds
// the context that owns the caller's stream before touching the runtime.  The driver entry points
// are requested at the CUDA 12.0 ABI: the default cuStreamGetCtx is the three-argument _v2, and
// calling it with two arguments (an earlier version did) corrupted memory -- it crashed under CUDA
// graph capture.  (cudaStreamGetDevice would be simpler but invalidates a capture in progress.)
template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

void bind_stream_context(cudaStream_t st) {
  using GetCtx = CUresult (*)(CUstream, CUcontext*);
  using CurCtx = CUresult (*)(CUcontext*);
  using SetCtx = CUresult (*)(CUcontext);
  static GetCtx get_ctx = driver_fn<GetCtx>("cuStreamGetCtx");
  static CurCtx cur_ctx = driver_fn<CurCtx>("cuCtxGetCurrent");
  static SetCtx set_ctx = driver_fn<SetCtx>("cuCtxSetCurrent");
  if (!get_ctx || !cur_ctx || !set_ctx) return;
  CUcontext want = nullptr, have = nullptr;
  if (st != nullptr && get_ctx(reinterpret_cast<CUstream>(st), &want) == CUDA_SUCCESS && want != nullptr) {
    if (cur_ctx(&have) == CUDA_SUCCESS && have != want) set_ctx(want);
  } else if (cur_ctx(&have) == CUDA_SUCCESS && have == nullptr) {
    cudaFree(nullptr);  // legacy stream and no context: initialise the runtime's current device
  }
}

// A side stream (+ fork / join events) per device and calling thread, for independent passes that
// can share the GPU: the backward's adjoint summaries run beside its dq pass.  Stream-ordered
// fork / join, so it composes with the caller's stream and with CUDA graph capture.
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

cudaError_t side_stream(SideStream** out) {
  thread_local SideStream res[64];
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  SideStream& r = res[dev];
  if (r.stream == nullptr) {
    // high priority: the side stream carries the backward's critical chain (summaries, scan, dK/dV sweep)
    int least = 0, greatest = 0;
    if ((err = cudaDeviceGetStreamPriorityRange(&least, &greatest)) != cudaSuccess) return err;
    if ((err = cudaStreamCreateWithPriority(&r.stream, cudaStreamNonBlocking, greatest)) != cudaSuccess) return err;
    if ((err = cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming)) != cudaSuccess) return err;
    if ((err = cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming)) != cudaSuccess) return err;
  }
  *out = &r;
  return cudaSuccess;
}

// State buffers (d x d rows in the accumulation type) and GLA rows are read and written as 16-byte vectors.
bool states_aligned(std::initializer_list<const void*> ptrs) {
  for (const void* p : ptrs)
    if (p != nullptr && (reinterpret_cast<uintptr_t>(p) & 15) != 0) return false;
  return true;
}

struct Prepared {
  int backend;
  la::Plan plan;
  size_t need;
};

int prepare(const la_desc* desc, size_t ws_bytes, const void* ws, Prepared* out, const OpStrides* ops = nullptr,
            unsigned used = 0) {
  int rc = validate(desc);
  if (rc != LA_OK) return rc;
  rc = pick_backend(desc, &out->backend, ops, used);
  if (rc != LA_OK) return rc;
  out->plan = plan_for(desc, out->backend);
  out->need = ws_bytes_for(desc, out->backend, out->plan);
  if (out->need > 0 && (ws == nullptr || ws_bytes < out->need))
    return fail(LA_ERR_SHAPE, "workspace too small: need %zu bytes, got %zu", out->need, ws_bytes);
  return LA_OK;
}

// LA_FLAG_CHECK_DECAY: read lam back (synchronous) and validate it like check_decay (matrixops.py:72-77)
int check_decay_device(const double* lam, int64_t heads, cudaStream_t st) {
  std::vector<double> host((size_t)heads);
  cudaError_t err = cudaMemcpyAsync(host.data(), lam, sizeof(double) * (size_t)heads, cudaMemcpyDeviceToHost, st);
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  if (err != cudaSuccess) return cuda_fail(err, "lam read-back");
  return la_check_decay(host.data(), heads);
}

// LA_FLAG_CHECK_FINITE: the reference's ensure_finite on every input (kernels.py:148-149)
template <typename T>
__global__ void count_nonfinite_kernel(const T* x, la::Strides3 s, int64_t batch, int64_t heads, int64_t n, int64_t d,
                                       unsigned long long* bad) {
  const int64_t total = batch * heads * n * d;
  unsigned long long mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i % d, t = (i / d) % n, h = (i / (d * n)) % heads, b = i / (d * n * heads);
    const double v = (double)la::Cvt<T>::to_f(x[b * s.b + h * s.h + t * s.n + f]);
    if (!isfinite(v)) ++mine;
  }
  if (mine) atomicAdd(bad, mine);
}

int check_finite(const la_desc* desc, std::initializer_list<std::pair<const void*, la::Strides3>> ins,
                 std::initializer_list<const char*> names, cudaStream_t st) {
  unsigned long long* bad = nullptr;
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(unsigned long long) * ins.size(), st);
  if (err == cudaSuccess) err = cudaMemsetAsync(bad, 0, sizeof(unsigned long long) * ins.size(), st);
  int i = 0;
  for (const auto& in : ins) {
    if (err != cudaSuccess) break;
    const dim3 grid(4 * la::device_sms()), block(256);
    if (desc->dtype == LA_F64)
      count_nonfinite_kernel<double><<<grid, block, 0, st>>>(reinterpret_cast<const double*>(in.first), in.second,
                                                              desc->batch, desc->heads, desc->n, desc->d, bad + i);
    else if (desc->dtype == LA_F32)
      count_nonfinite_kernel<float><<<grid, block, 0, st>>>(reinterpret_cast<const float*>(in.first), in.second,
                                                             desc->batch, desc->heads, desc->n, desc->d, bad + i);
    else
      count_nonfinite_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(
          reinterpret_cast<const __nv_bfloat16*>(in.first), in.second, desc->batch, desc->heads, desc->n, desc->d,
          bad + i);
    err = cudaGetLastError();
    ++i;
  }
  std::vector<unsigned long long> host(ins.size(), 0);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(host.data(), bad, sizeof(unsigned long long) * ins.size(), cudaMemcpyDeviceToHost, st);
  if (bad != nullptr) cudaFreeAsync(bad, st);
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  if (err != cudaSuccess) return cuda_fail(err, "finiteness check");
  i = 0;
  for (const char* name : names) {
    if (host[i] != 0) return fail(LA_ERR_DOMAIN, "%s: contains NaN or Inf (%llu entries)", name, host[i]);
    ++i;
  }
  return LA_OK;
}

// The fused dK/dV sweep (la_tc_bwd.cu): q, k, v, do read once, one state update.  seg_in: the
// adjoint state entering every segment (split sequences), else the caller's dkv_in.
int dkdv(const la::PassDesc& base, const OpStrides& os, const void* q, const void* k, const void* v, const void* dout,
         void* dk, void* dv, const void* dkv_in, void* dkv_out, const void* seg_in, cudaStream_t st,
         const la::GlaEpilogue* epi = nullptr) {
  la::PassDesc p = base;
  p.rev = 1;
  p.b = q;
  p.c = dout;
  p.a = k;
  p.out = dv;
  p.state_out = dkv_out;
  const int64_t dd = (int64_t)p.d * p.d;
  if (seg_in != nullptr) {
    p.state_in = seg_in;
    p.state_in_bh_stride = (int64_t)p.nseg * dd;
    p.state_in_seg_stride = dd;
  } else {
    p.state_in = dkv_in;
    p.state_in_bh_stride = dd;
    p.state_in_seg_stride = 0;
  }
  if (!la::tc_pointers_ok(p) || (reinterpret_cast<uintptr_t>(v) & 15) || (reinterpret_cast<uintptr_t>(dk) & 15))
    return cuda_fail(cudaErrorMisalignedAddress, "la_bwd dkdv");
  const la::Strides3 s6[6] = {os.s[LA_T_Q], os.s[LA_T_K], os.s[LA_T_V], os.s[LA_T_DO], os.s[LA_T_DK], os.s[LA_T_DV]};
  cudaError_t err = la::tc_dkdv_launch(p, q, k, v, dout, dk, dv, s6, st, epi);
  if (err != cudaSuccess) return cuda_fail(err, "la_bwd dkdv");
  return LA_OK;
}

constexpr uint32_t kKnownFlags =
    LA_FLAG_RESUME | LA_FLAG_CHECK_DECAY | LA_FLAG_CHECK_FINITE | LA_FLAG_NO_DQ | LA_FLAG_NO_DKDV;

}  // namespace

extern "C" {

size_t la_workspace_bytes(const la_desc* desc) {
  if (validate(desc) != LA_OK) return 0;
  int backend;
  if (pick_backend(desc, &backend) != LA_OK) return 0;
  // an _ex call whose operand strides rule out the tensor cores runs the SIMT plan: cover both
  size_t need = ws_bytes_for(desc, backend, plan_for(desc, backend));
  if (backend == LA_BACKEND_TCGEN05) {
    const size_t simt = ws_bytes_for(desc, LA_BACKEND_SIMT, plan_for(desc, LA_BACKEND_SIMT));
    if (simt > need) need = simt;
  }
  return need;
}

int la_segment_count(const la_desc* desc) {
  if (validate(desc) != LA_OK) return -1;
  int backend;
  if (pick_backend(desc, &backend) != LA_OK) return -1;
  return plan_for(desc, backend).nseg;
}

int la_check_decay(const double* lam_host, int64_t heads) {
  if (lam_host == nullptr || heads < 1) return fail(LA_ERR_SHAPE, "la_check_decay: null lam or heads < 1");
  for (int64_t h = 0; h < heads; ++h)
    if (!(lam_host[h] > 0.0 && lam_host[h] <= 1.0))
      return fail(LA_ERR_DOMAIN, "decay rate must lie in (0, 1], got %.17g (head %lld)", lam_host[h], (long long)h);
  return LA_OK;
}

int la_fwd_ex(const la_desc* desc, const la_tensor_strides* strides, uint32_t flags, const void* q, const void* k,
              const void* v, const double* lam, const void* kv_in, void* o, void* kv_out, void* seg_states_out,
              void* workspace, size_t workspace_bytes, void* stream) {
  if (flags & ~kKnownFlags) return fail(LA_ERR_DOMAIN, "la_fwd_ex: unknown flags 0x%x", flags);
  if (flags & (LA_FLAG_NO_DQ | LA_FLAG_NO_DKDV)) return fail(LA_ERR_DOMAIN, "la_fwd_ex: backward-only flags");
  if (desc == nullptr) return fail(LA_ERR_SHAPE, "null descriptor");
  OpStrides os;
  const unsigned used = 1u << LA_T_Q | 1u << LA_T_K | 1u << LA_T_V | 1u << LA_T_O;
  int rc = op_strides(desc, strides, used, &os);
  if (rc != LA_OK) return rc;
  Prepared pr;
  rc = prepare(desc, workspace_bytes, workspace, &pr, &os, used);
  if (rc != LA_OK) return rc;
  if (!q || !k || !v || !o || !lam) return fail(LA_ERR_SHAPE, "la_fwd: null q/k/v/o/lam");
  if (!states_aligned({kv_in, kv_out, seg_states_out}))
    return fail(LA_ERR_SHAPE, "la_fwd: state buffers must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  if ((flags & LA_FLAG_CHECK_DECAY) && (rc = check_decay_device(lam, desc->heads, st)) != LA_OK) return rc;
  if ((flags & LA_FLAG_CHECK_FINITE) &&
      (rc = check_finite(desc, {{q, os.s[LA_T_Q]}, {k, os.s[LA_T_K]}, {v, os.s[LA_T_V]}}, {"Q", "K", "V"}, st)) !=
          LA_OK)
    return rc;
  la::PassDesc p = base_pass(desc, pr.plan, lam);
  p.a = q;
  p.b = k;
  p.c = v;
  p.out = o;
  p.sa = os.s[LA_T_Q];
  p.sbb = os.s[LA_T_K];
  p.sc = os.s[LA_T_V];
  p.so = os.s[LA_T_O];
  p.rev = 0;
  p.state_in = kv_in;
  p.state_out = kv_out;
  cudaError_t err = cudaSuccess;
  void* seg_in = nullptr;
  if (pr.plan.nseg > 1) {
    seg_in = seg_states_out != nullptr ? seg_states_out : ws_seg_in(workspace, desc, pr.plan);
    err = segment_states(pr.backend, desc->dtype, p, ws_delta(workspace), seg_in, st, (flags & LA_FLAG_RESUME) != 0);
  }
  if (err == cudaSuccess) err = main_pass(pr.backend, desc->dtype, p, seg_in, 0, st);
  if (err != cudaSuccess) return cuda_fail(err, "la_fwd");
  return LA_OK;
}

int la_fwd(const la_desc* desc, const void* q, const void* k, const void* v, const double* lam, const void* kv_in,
           void* o, void* kv_out, void* seg_states_out, void* workspace, size_t workspace_bytes, void* stream) {
  return la_fwd_ex(desc, nullptr, 0, q, k, v, lam, kv_in, o, kv_out, seg_states_out, workspace, workspace_bytes,
                   stream);
}

// the backward; epi_q / epi_k (the fused GLA core backward, bf16 tcgen05 only): dq -> dqp, dk -> dkp
static int bwd_impl(const la_desc* desc, const la_tensor_strides* strides, uint32_t flags, const void* q, const void* k,
                    const void* v, const void* dout, const double* lam, const void* kv_in, const void* dkv_in,
                    const void* fwd_seg_states, void* dq, void* dk, void* dv, void* dkv_out, void* workspace,
                    size_t workspace_bytes, void* stream, const la::GlaEpilogue* epi_q, const la::GlaEpilogue* epi_k) {
  if (flags & ~kKnownFlags) return fail(LA_ERR_DOMAIN, "la_bwd_ex: unknown flags 0x%x", flags);
  if (desc == nullptr) return fail(LA_ERR_SHAPE, "null descriptor");
  const bool want_dq = !(flags & LA_FLAG_NO_DQ), want_dkdv = !(flags & LA_FLAG_NO_DKDV);
  OpStrides os;
  const unsigned used = 1u << LA_T_Q | 1u << LA_T_K | 1u << LA_T_V | 1u << LA_T_DO | (want_dq ? 1u << LA_T_DQ : 0u) |
                        (want_dkdv ? (1u << LA_T_DK | 1u << LA_T_DV) : 0u);
  int rc = op_strides(desc, strides, used, &os);
  if (rc != LA_OK) return rc;
  Prepared pr;
  rc = prepare(desc, workspace_bytes, workspace, &pr, &os, used);
  if (rc != LA_OK) return rc;
  if (!q || !k || !v || !dout || !lam || (want_dq && !dq) || (want_dkdv && (!dk || !dv)))
    return fail(LA_ERR_SHAPE, "la_bwd: null q/k/v/do/lam or a requested dq/dk/dv");
  if (!states_aligned({kv_in, dkv_in, fwd_seg_states, dkv_out}))
    return fail(LA_ERR_SHAPE, "la_bwd: state buffers must be 16-byte aligned");
  const bool split = pr.plan.nseg > 1;
  const bool resume = (flags & LA_FLAG_RESUME) != 0;
  if (resume && split && want_dq && fwd_seg_states == nullptr)
    return fail(LA_ERR_SHAPE, "la_bwd_ex: LA_FLAG_RESUME with a split sequence needs fwd_seg_states (sweep 1 would "
                              "overwrite the resumed summaries)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  if ((flags & LA_FLAG_CHECK_DECAY) && (rc = check_decay_device(lam, desc->heads, st)) != LA_OK) return rc;
  if ((flags & LA_FLAG_CHECK_FINITE) &&
      (rc = check_finite(desc, {{q, os.s[LA_T_Q]}, {k, os.s[LA_T_K]}, {v, os.s[LA_T_V]}, {dout, os.s[LA_T_DO]}},
                         {"Q", "K", "V", "dO"}, st)) != LA_OK)
    return rc;
  const la::PassDesc base = base_pass(desc, pr.plan, lam);
  // sweep 2 as the fused dK/dV kernel (bf16 on tcgen05) or as two reverse passes (fp32 on tcgen05, SIMT)
  const bool fused = pr.backend == LA_BACKEND_TCGEN05 && desc->dtype == LA_BF16;
  void* delta = split ? ws_delta(workspace) : nullptr;
  void* seg_in = split ? ws_seg_in(workspace, desc, pr.plan) : nullptr;
  cudaError_t err = cudaSuccess;
  // sweep 1 (kernels.py:309-318): dq = fwd(do, v, k); its state is kv^T, so the forward's segment
  // states serve it transposed when the caller kept them
  la::PassDesc p = base;
  p.a = dout;
  p.b = v;
  p.c = k;
  p.out = dq;
  p.sa = os.s[LA_T_DO];
  p.sbb = os.s[LA_T_V];
  p.sc = os.s[LA_T_K];
  p.so = os.s[LA_T_DQ];
  p.rev = 0;
  p.state_in = kv_in;
  p.state_in_T = 1;
  auto run_dq = [&](cudaStream_t s) -> cudaError_t {
    if (split && fwd_seg_states != nullptr) return main_pass(pr.backend, desc->dtype, p, fwd_seg_states, 1, s, epi_q);
    cudaError_t e = split ? segment_states(pr.backend, desc->dtype, p, delta, seg_in, s) : cudaSuccess;
    return e == cudaSuccess ? main_pass(pr.backend, desc->dtype, p, seg_in, 0, s, epi_q) : e;
  };
  // sweep 2 (kernels.py:320-333): dk = rev(v, do, q) carries dkv^T, dv = rev(k, q, do) carries dkv --
  // one set of segment states (over q, do) serves both passes
  la::PassDesc pd = base;
  pd.b = q;
  pd.c = dout;
  pd.sbb = os.s[LA_T_Q];
  pd.sc = os.s[LA_T_DO];
  pd.rev = 1;
  pd.state_in = dkv_in;
  // states_ready: the entering adjoint states are already in seg_in
  auto run_dkdv = [&](cudaStream_t s, bool states_ready) -> int {
    if (split && !states_ready &&
        (err = segment_states(pr.backend, desc->dtype, pd, delta, seg_in, s, resume)) != cudaSuccess)
      return cuda_fail(err, "la_bwd dkv states");
    if (fused)
      return dkdv(base, os, q, k, v, dout, dk, dv, dkv_in, dkv_out, split ? seg_in : nullptr, s, epi_k);
    la::PassDesc r = base;
    r.a = v;
    r.b = dout;
    r.c = q;
    r.out = dk;
    r.sa = os.s[LA_T_V];
    r.sbb = os.s[LA_T_DO];
    r.sc = os.s[LA_T_Q];
    r.so = os.s[LA_T_DK];
    r.rev = 1;
    r.state_in = dkv_in;
    r.state_in_T = 1;
    if ((err = main_pass(pr.backend, desc->dtype, r, seg_in, 1, s)) != cudaSuccess) return cuda_fail(err, "la_bwd dk");
    r = base;
    r.a = k;
    r.b = q;
    r.c = dout;
    r.out = dv;
    r.sa = os.s[LA_T_K];
    r.sbb = os.s[LA_T_Q];
    r.sc = os.s[LA_T_DO];
    r.so = os.s[LA_T_DV];
    r.rev = 1;
    r.state_in = dkv_in;
    r.state_out = dkv_out;
    if ((err = main_pass(pr.backend, desc->dtype, r, seg_in, 0, s)) != cudaSuccess) return cuda_fail(err, "la_bwd dv");
    return LA_OK;
  };
  if (!want_dkdv) return (err = run_dq(st)) == cudaSuccess ? LA_OK : cuda_fail(err, "la_bwd dq");
  if (!want_dq) return run_dkdv(st, false);
#ifndef LA_BWD_CONCURRENT
#define LA_BWD_CONCURRENT 1
#endif
  if (LA_BWD_CONCURRENT && (!split || fwd_seg_states != nullptr) &&
      (pr.backend == LA_BACKEND_TCGEN05 || split)) {
    // The two sweeps are independent once sweep 1 needs no workspace: sweep 2's chain (adjoint summaries
    // and scan when the sequence is split, then the fused dK/dV sweep -- or, on SIMT, just the summaries)
    // runs on the high-priority side stream, the dq pass beside it on the caller's stream.  Together
    // they keep all SMs streaming (each alone fills 128 of 148 at n = 8K) and overlap each other's ramp
    // and tail.
    SideStream* side = nullptr;
    if ((err = side_stream(&side)) != cudaSuccess) return cuda_fail(err, "la_bwd side stream");
    if ((err = cudaEventRecord(side->fork, st)) != cudaSuccess ||
        (err = cudaStreamWaitEvent(side->stream, side->fork, 0)) != cudaSuccess)
      return cuda_fail(err, "la_bwd fork");
    if (pr.backend == LA_BACKEND_TCGEN05) {
      if ((rc = run_dkdv(side->stream, false)) != LA_OK) return rc;
    } else if ((err = segment_states(pr.backend, desc->dtype, pd, delta, seg_in, side->stream, resume)) !=
               cudaSuccess) {
      return cuda_fail(err, "la_bwd dkv states");
    }
    if ((err = cudaEventRecord(side->join, side->stream)) != cudaSuccess) return cuda_fail(err, "la_bwd join");
    if ((err = run_dq(st)) != cudaSuccess) return cuda_fail(err, "la_bwd dq");
    if ((err = cudaStreamWaitEvent(st, side->join, 0)) != cudaSuccess) return cuda_fail(err, "la_bwd join");
    // SIMT: the entering adjoint states are ready, run the two reverse passes
    return pr.backend == LA_BACKEND_TCGEN05 ? LA_OK : run_dkdv(st, true);
  }
  if ((err = run_dq(st)) != cudaSuccess) return cuda_fail(err, "la_bwd dq");
  return run_dkdv(st, false);
}

int la_bwd_ex(const la_desc* desc, const la_tensor_strides* strides, uint32_t flags, const void* q, const void* k,
              const void* v, const void* dout, const double* lam, const void* kv_in, const void* dkv_in,
              const void* fwd_seg_states, void* dq, void* dk, void* dv, void* dkv_out, void* workspace,
              size_t workspace_bytes, void* stream) {
  return bwd_impl(desc, strides, flags, q, k, v, dout, lam, kv_in, dkv_in, fwd_seg_states, dq, dk, dv, dkv_out,
                  workspace, workspace_bytes, stream, nullptr, nullptr);
}

int la_bwd(const la_desc* desc, const void* q, const void* k, const void* v, const void* dout, const double* lam,
           const void* kv_in, const void* dkv_in, const void* fwd_seg_states, void* dq, void* dk, void* dv,
           void* dkv_out, void* workspace, size_t workspace_bytes, void* stream) {
  return la_bwd_ex(desc, nullptr, 0, q, k, v, dout, lam, kv_in, dkv_in, fwd_seg_states, dq, dk, dv, dkv_out,
                   workspace, workspace_bytes, stream);
}
static int state_entry(const la_desc* desc, const void* b, const void* c, int rev, const double* lam, void* out,
                       void* workspace, size_t workspace_bytes, void* stream, const char* who) {
  Prepared pr;
  int rc = prepare(desc, workspace_bytes, workspace, &pr);
  if (rc != LA_OK) return rc;
  if (!b || !c || !lam || !out) return fail(LA_ERR_SHAPE, "%s: null operand", who);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  la::PassDesc p = base_pass(desc, pr.plan, lam);
  p.b = b;
  p.c = c;
  p.rev = rev;
  cudaError_t err;
  if (pr.plan.nseg == 1) {
    p.delta_out = out;  // one segment: its summary is the answer
    err = launch(pr.backend, desc->dtype, p, true, st);
  } else {
    p.delta_out = ws_delta(workspace);
    err = launch(pr.backend, desc->dtype, p, true, st);
    if (err == cudaSuccess)
      err = la::launch_segment_scan(desc->dtype == LA_F64, p.delta_out, nullptr, nullptr, 0, out, 0, lam,
                                    p.batch * p.heads, p.heads, p.d, p, st);
  }
  if (err != cudaSuccess) return cuda_fail(err, who);
  return LA_OK;
}

int la_fwd_state(const la_desc* desc, const void* k, const void* v, const double* lam, void* kv_delta,
                 void* workspace, size_t workspace_bytes, void* stream) {
  return state_entry(desc, k, v, 0, lam, kv_delta, workspace, workspace_bytes, stream, "la_fwd_state");
}

int la_bwd_state(const la_desc* desc, const void* q, const void* dout, const double* lam, void* dkv_delta,
                 void* workspace, size_t workspace_bytes, void* stream) {
  return state_entry(desc, q, dout, 1, lam, dkv_delta, workspace, workspace_bytes, stream, "la_bwd_state");
}

int la_decode(const la_desc* desc, const void* q, const void* k, const void* v, const double* lam, void* kv,
              void* o, void* stream) {
  int rc = validate(desc);
  if (rc != LA_OK) return rc;
  if (desc->n != 1) return fail(LA_ERR_SHAPE, "la_decode advances one token per sequence: need n == 1, got n=%lld",
                                (long long)desc->n);
  if (!q || !k || !v || !kv || !o || !lam) return fail(LA_ERR_SHAPE, "la_decode: null q/k/v/kv/o/lam");
  if (!states_aligned({kv})) return fail(LA_ERR_SHAPE, "la_decode: kv must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::decode_launch(desc->dtype, (int)desc->batch, (int)desc->heads, (int)desc->d, desc->stride[0],
                                      desc->stride[1], q, k, v, lam, kv, o, st);
  if (err != cudaSuccess) return cuda_fail(err, "la_decode");
  return LA_OK;
}

static int gla_prepare(const la_gla_desc* desc, bool need_even_d, la::GlaRows* g) {
  if (desc == nullptr) return fail(LA_ERR_SHAPE, "null GLA descriptor");
  if (desc->batch < 1 || desc->n < 1 || desc->heads < 1 || desc->d < 1)
    return fail(LA_ERR_DOMAIN, "GLA stages need batch, n, heads, d >= 1");
  if (desc->dtype != LA_F32 && desc->dtype != LA_F64 && desc->dtype != LA_BF16)
    return fail(LA_ERR_DOMAIN, "dtype must be LA_F32, LA_F64 or LA_BF16, got %d", desc->dtype);
  if (desc->act < LA_ACT_NONE || desc->act > LA_ACT_ONE_PLUS_ELU) return fail(LA_ERR_DOMAIN, "unknown act %d", desc->act);
  if (desc->offset < 0) return fail(LA_ERR_DOMAIN, "position offset must be >= 0, got %lld", (long long)desc->offset);
  if (!(desc->eps >= 0.0)) return fail(LA_ERR_DOMAIN, "eps must be >= 0");
  if (need_even_d && desc->d % 2) return fail(LA_ERR_SHAPE, "rotation needs an even head dim, got d=%lld", (long long)desc->d);
  if (desc->heads * desc->d > (int64_t)1 << 30 || desc->batch * desc->n > (int64_t)1 << 40)
    return fail(LA_ERR_UNSUPPORTED, "GLA rows / width beyond this build's limits");
  const int64_t vec = 16 / (desc->dtype == LA_F64 ? 8 : desc->dtype == LA_F32 ? 4 : 2);
  if ((desc->heads * desc->d) % vec)
    return fail(LA_ERR_UNSUPPORTED, "GLA stages need heads * d to be a multiple of %lld (16-byte rows), got %lld",
                (long long)vec, (long long)(desc->heads * desc->d));
  g->rows = desc->batch * desc->n;
  g->n = (int)desc->n;
  g->width = (int)(desc->heads * desc->d);
  g->d = (int)desc->d;
  g->dtype = desc->dtype;
  g->act = desc->act;
  g->offset = desc->offset;
  return LA_OK;
}

size_t la_gla_workspace_bytes(const la_gla_desc* desc) {
  la::GlaRows g;
  if (gla_prepare(desc, false, &g) != LA_OK) return 0;
  return la::gla_prologue_bwd_partial_bytes(g);
}

int la_gla_prologue(const la_gla_desc* desc, const void* qp, const void* kp, const double* theta, void* q, void* k,
                    void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(desc, theta != nullptr, &g);
  if (rc != LA_OK) return rc;
  if (!qp || !kp || !q || !k) return fail(LA_ERR_SHAPE, "la_gla_prologue: null qp/kp/q/k");
  if (!states_aligned({qp, kp, q, k})) return fail(LA_ERR_SHAPE, "la_gla_prologue: rows must be 16-byte aligned");
  if (g.width % 2) return fail(LA_ERR_SHAPE, "la_gla_prologue: heads * d must be even");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::gla_prologue(g, qp, kp, theta, q, k, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_prologue");
}

int la_gla_prologue_bwd(const la_gla_desc* desc, const void* qp, const void* kp, const double* theta, const void* dq,
                        const void* dk, void* dqp, void* dkp, double* dtheta, void* workspace, size_t workspace_bytes,
                        void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(desc, theta != nullptr, &g);
  if (rc != LA_OK) return rc;
  if (!qp || !kp || !dq || !dk || !dqp || !dkp) return fail(LA_ERR_SHAPE, "la_gla_prologue_bwd: null operand");
  if (!states_aligned({qp, kp, dq, dk, dqp, dkp}))
    return fail(LA_ERR_SHAPE, "la_gla_prologue_bwd: rows must be 16-byte aligned");
  if (g.width % 2) return fail(LA_ERR_SHAPE, "la_gla_prologue_bwd: heads * d must be even");
  if (theta != nullptr) {
    if (dtheta == nullptr) return fail(LA_ERR_SHAPE, "la_gla_prologue_bwd: theta given without dtheta");
    const size_t need = la::gla_prologue_bwd_partial_bytes(g);
    if (workspace == nullptr || workspace_bytes < need)
      return fail(LA_ERR_SHAPE, "workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::gla_prologue_bwd(g, qp, kp, theta, dq, dk, dqp, dkp, workspace, dtheta, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_prologue_bwd");
}

// the attention descriptor of the GLA core: model-native rows [batch, n, heads * d]
static int gla_core_desc(const la_gla_desc* gdesc, la_desc* desc) {
  std::memset(desc, 0, sizeof(*desc));
  desc->batch = gdesc->batch;
  desc->heads = gdesc->heads;
  desc->n = gdesc->n;
  desc->d = gdesc->d;
  desc->dtype = gdesc->dtype;
  desc->backend = LA_BACKEND_TCGEN05;
  desc->stride[0] = gdesc->n * gdesc->heads * gdesc->d;
  desc->stride[1] = gdesc->d;
  desc->stride[2] = gdesc->heads * gdesc->d;
  int rc = validate(desc);
  if (rc != LA_OK) return rc;
  if (desc->dtype != LA_BF16 || desc->d != 128 || !la::tc_supported(desc->dtype, (int)desc->d, desc->stride, 1))
    return fail(LA_ERR_UNSUPPORTED, "la_gla_core_fwd: the fused core needs bf16 and d = 128 (use la_gla_prologue + la_fwd)");
  return LA_OK;
}

size_t la_gla_core_workspace_bytes(const la_gla_desc* gdesc) {
  la::GlaRows g;
  la_desc desc;
  if (gla_prepare(gdesc, false, &g) != LA_OK || gla_core_desc(gdesc, &desc) != LA_OK) return 0;
  return ws_bytes_for(&desc, LA_BACKEND_TCGEN05, plan_for(&desc, LA_BACKEND_TCGEN05));
}

int la_gla_core_fwd(const la_gla_desc* gdesc, const void* qp, const void* kp, const void* v, const double* lam,
                    const double* theta, const void* kv_in, void* o, void* q_out, void* k_out, void* kv_out,
                    void* workspace, size_t workspace_bytes, void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(gdesc, theta != nullptr, &g);
  if (rc != LA_OK) return rc;
  if (!qp || !kp || !v || !o || !lam) return fail(LA_ERR_SHAPE, "la_gla_core_fwd: null qp/kp/v/o/lam");
  if ((q_out == nullptr) != (k_out == nullptr)) return fail(LA_ERR_SHAPE, "la_gla_core_fwd: q_out and k_out go together");
  if (!states_aligned({qp, kp, v, o, q_out, k_out, kv_in, kv_out}))
    return fail(LA_ERR_SHAPE, "la_gla_core_fwd: operands and states must be 16-byte aligned");
  la_desc desc;
  if ((rc = gla_core_desc(gdesc, &desc)) != LA_OK) return rc;
  const la::Plan plan = plan_for(&desc, LA_BACKEND_TCGEN05);
  const size_t need = ws_bytes_for(&desc, LA_BACKEND_TCGEN05, plan);
  if (need > 0 && (workspace == nullptr || workspace_bytes < need))
    return fail(LA_ERR_SHAPE, "workspace too small: need %zu bytes, got %zu (la_gla_core_workspace_bytes)", need,
                workspace_bytes);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  la::PassDesc p = base_pass(&desc, plan, lam);
  p.a = qp;
  p.b = kp;
  p.c = v;
  p.out = o;
  p.rev = 0;
  p.state_in = kv_in;
  p.state_out = kv_out;
  const int64_t dd = desc.d * desc.d;
  p.state_in_bh_stride = dd;
  la::GlaPrologue pro{theta, gdesc->act, gdesc->offset, q_out, k_out};
  cudaError_t err = cudaSuccess;
  if (plan.nseg > 1) {
    // the segmented forward (la_fwd_ex) with the prologue in both the summary pass and the main pass
    void* delta = ws_delta(workspace);
    void* seg_in = ws_seg_in(workspace, &desc, plan);
    la::PassDesc s = p;
    s.a = nullptr;
    s.out = nullptr;
    s.state_in = nullptr;
    s.state_out = nullptr;
    s.delta_out = delta;
    s.g_lo = 0;
    s.g_hi = p.nseg - 2;
    err = la::tc_summary_launch(s, st, &pro);
    if (err == cudaSuccess)
      err = la::launch_segment_scan(false, delta, seg_in, kv_in, 0, nullptr, 0, lam, p.batch * p.heads, p.heads, p.d,
                                    s, st);
    p.state_in = seg_in;
    p.state_in_bh_stride = (int64_t)p.nseg * dd;
    p.state_in_seg_stride = dd;
  }
  if (err == cudaSuccess) err = la::tc_gla_fwd_launch(p, pro, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_core_fwd");
}

int la_gla_core_bwd(const la_gla_desc* gdesc, const void* qp, const void* kp, const void* q, const void* k,
                    const void* v, const void* da, const double* lam, const double* theta, const void* kv_in,
                    const void* dkv_in, void* dqp, void* dkp, void* dv, void* dkv_out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(gdesc, theta != nullptr, &g);
  if (rc != LA_OK) return rc;
  if (!qp || !kp || !q || !k || !v || !da || !lam || !dqp || !dkp || !dv)
    return fail(LA_ERR_SHAPE, "la_gla_core_bwd: null operand");
  if (!states_aligned({qp, kp})) return fail(LA_ERR_SHAPE, "la_gla_core_bwd: operands must be 16-byte aligned");
  la_desc desc;
  if ((rc = gla_core_desc(gdesc, &desc)) != LA_OK) return rc;
  const la::Strides3 rows{desc.stride[0], desc.stride[1], desc.stride[2]};
  const la::GlaEpilogue epi_q{qp, rows, theta, gdesc->act, gdesc->offset};
  const la::GlaEpilogue epi_k{kp, rows, theta, gdesc->act, gdesc->offset};
  return bwd_impl(&desc, nullptr, 0, q, k, v, da, lam, kv_in, dkv_in, nullptr, dqp, dkp, dv, dkv_out, workspace,
                  workspace_bytes, stream, &epi_q, &epi_k);
}

size_t la_gla_core_bwd_workspace_bytes(const la_gla_desc* gdesc) {
  la::GlaRows g;
  la_desc desc;
  if (gla_prepare(gdesc, false, &g) != LA_OK || gla_core_desc(gdesc, &desc) != LA_OK) return 0;
  return la_workspace_bytes(&desc);
}

int la_gla_epilogue(const la_gla_desc* desc, const void* a, const void* u, void* gated, void* rawnorm, void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(desc, false, &g);
  if (rc != LA_OK) return rc;
  if (!a || !gated || !rawnorm) return fail(LA_ERR_SHAPE, "la_gla_epilogue: null a/gated/rawnorm");
  if (!states_aligned({a, u, gated})) return fail(LA_ERR_SHAPE, "la_gla_epilogue: rows must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::gla_epilogue(g, a, u, gated, rawnorm, desc->eps, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_epilogue");
}

int la_gla_epilogue_bwd(const la_gla_desc* desc, const void* dgated, const void* a, const void* u, const void* rawnorm,
                        void* da, void* du, void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(desc, false, &g);
  if (rc != LA_OK) return rc;
  if (!dgated || !a || !rawnorm || !da || (u != nullptr && du == nullptr))
    return fail(LA_ERR_SHAPE, "la_gla_epilogue_bwd: null operand");
  if (!states_aligned({dgated, a, u, da, du}))
    return fail(LA_ERR_SHAPE, "la_gla_epilogue_bwd: rows must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::gla_epilogue_bwd(g, dgated, a, u, rawnorm, da, du, desc->eps, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_epilogue_bwd");
}

int la_gla_gate_rowsq(const la_gla_desc* desc, const void* a, const void* u, void* gated, void* rowsq,
                      int64_t rowsq_stride, void* stream) {
  la::GlaRows g;
  int rc = gla_prepare(desc, false, &g);
  if (rc != LA_OK) return rc;
  if (!a || !gated || !rowsq || rowsq_stride < 1) return fail(LA_ERR_SHAPE, "la_gla_gate_rowsq: null operand / bad stride");
  if (!states_aligned({a, u, gated})) return fail(LA_ERR_SHAPE, "la_gla_gate_rowsq: rows must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::gla_gate_rowsq(g, a, u, gated, rowsq, rowsq_stride, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_gate_rowsq");
}

int la_gla_rowscale(int dtype, int64_t rows, int64_t out_width, double eps, const void* red, void* y, void* stream) {
  if (dtype != LA_F32 && dtype != LA_F64 && dtype != LA_BF16) return fail(LA_ERR_DOMAIN, "bad dtype %d", dtype);
  if (rows < 1 || out_width < 1 || out_width > (int64_t)1 << 30) return fail(LA_ERR_SHAPE, "bad rows / out_width");
  if (!red || !y) return fail(LA_ERR_SHAPE, "la_gla_rowscale: null red / y");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  cudaError_t err = la::gla_rowscale(dtype == LA_F64, red, y, rows, (int)out_width, eps, st);
  return err == cudaSuccess ? LA_OK : cuda_fail(err, "la_gla_rowscale");
}

int la_launch_count(const la_desc* desc, int which) {
  if (validate(desc) != LA_OK) return -1;
  int backend;
  if (pick_backend(desc, &backend) != LA_OK) return -1;
  const la::Plan plan = plan_for(desc, backend);
  // bwd sweep 2 is one fused dk/dv kernel on the bf16 tcgen05 backend, two passes otherwise
  const int sweep2 = backend == LA_BACKEND_TCGEN05 && desc->dtype == LA_BF16 ? 1 : 2;
  if (plan.nseg == 1) return which == 0 ? 1 : 1 + sweep2;
  // fwd: summaries + scan + main.  bwd: dq main (+ its summaries and scan unless the forward's segment
  // states are passed, which = 2) + one dkv summaries + scan + sweep 2
  return which == 0 ? 3 : (which == 2 ? 3 : 5) + sweep2;
}

const char* la_last_error(void) { return g_last_error.c_str(); }

int la_abi_version(void) { return LA_ABI_VERSION; }

const char* la_build_info(void) {
  return "lightning-attn b200: sm_100a, backends simt(f64/f32/bf16) + tcgen05(bf16, f32 3xbf16 split); decode; GLA stages + fused GLA core";
}

}  // extern "C"
