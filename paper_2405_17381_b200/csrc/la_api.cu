// la_api.cu -- the C ABI (include/lightning_attn.h): validation, planning and
// the pass orchestration that maps the reference's forward/backward onto the
// single "pass" primitive (la_common.cuh).
//
// Validation mirrors the reference's error classes:
//   LA_ERR_DOMAIN  n/d < 1, B < 1, bad precision      (kernels.py:84-91)
//   LA_ERR_SHAPE   missing operands, bad strides      (kernels.py:137-146)
// lam in (0, 1] (matrixops.py:72-77) is validated by the host wrappers, which
// own the host copy of lam; the ABI takes a device array so calls stay
// asynchronous and graph-capturable.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include <cuda.h>

#include "la_common.cuh"
#include "la_simt.cuh"
#include "la_tc.cuh"

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
  for (int i = 0; i < 3; ++i)
    if (desc->stride[i] < 0) return fail(LA_ERR_SHAPE, "negative stride");
  if (desc->stride[2] < desc->d) return fail(LA_ERR_SHAPE, "position stride %lld < d", (long long)desc->stride[2]);
  if (desc->n > (int64_t)1 << 31 || desc->batch * desc->heads > 65535)
    return fail(LA_ERR_UNSUPPORTED, "n or batch*heads beyond this build's grid limits");
  if (desc->d > 128) return fail(LA_ERR_UNSUPPORTED, "head dim d=%lld > 128 is not implemented", (long long)desc->d);
  return LA_OK;
}

// Which backend serves this descriptor.
int pick_backend(const la_desc* desc, int* backend) {
  const bool tc_ok = la::tc_supported(desc->dtype, (int)desc->d, desc->stride);
  if (desc->backend == LA_BACKEND_TCGEN05) {
    if (!tc_ok)
      return fail(LA_ERR_UNSUPPORTED,
                  "tcgen05 backend needs bf16, d in {64, 128}, 16-byte aligned strides (dtype=%d d=%lld)",
                  desc->dtype, (long long)desc->d);
    *backend = LA_BACKEND_TCGEN05;
  } else if (desc->backend == LA_BACKEND_SIMT) {
    *backend = LA_BACKEND_SIMT;
  } else {
    *backend = tc_ok ? LA_BACKEND_TCGEN05 : LA_BACKEND_SIMT;
  }
  return LA_OK;
}

la::Plan plan_for(const la_desc* desc, int backend) {
  const int64_t bh = desc->batch * desc->heads;
  if (backend == LA_BACKEND_TCGEN05) return la::tc_plan(bh, desc->n, (int)desc->d, desc->segments);
  return la::make_plan(bh, desc->n, la::simt_chunk(desc->dtype), desc->segments, 2 * la::kNumSMs, 4);
}

size_t ws_bytes_for(const la_desc* desc, int backend, const la::Plan& plan) {
  const int64_t bh = desc->batch * desc->heads;
  if (backend == LA_BACKEND_TCGEN05) return la::tc_workspace_bytes(bh, plan.nseg_ws, (int)desc->d);
  return la::simt_workspace_bytes(desc->dtype, bh, plan.nseg_ws, (int)desc->d);
}

la::PassDesc base_pass(const la_desc* desc, const la::Plan& plan, const double* lam) {
  la::PassDesc p;
  std::memset(&p, 0, sizeof(p));
  p.sb = desc->stride[0];
  p.sh = desc->stride[1];
  p.sn = desc->stride[2];
  p.batch = (int)desc->batch;
  p.heads = (int)desc->heads;
  p.n = (int)desc->n;
  p.d = (int)desc->d;
  p.lam = lam;
  p.seg_len = plan.seg_len;
  p.nseg = plan.nseg;
  return p;
}

cudaError_t run_pass(int backend, int dtype, const la::PassDesc& p, void* ws, cudaStream_t st) {
  if (backend == LA_BACKEND_TCGEN05) {
    if (!la::tc_pointers_ok(p)) return cudaErrorMisalignedAddress;  // TMA needs 16-byte aligned bases
    return la::tc_pass(p, ws, st);
  }
  return la::simt_pass(dtype, p, ws, st);
}

cudaError_t run_state(int backend, int dtype, const la::PassDesc& p, void* ws, cudaStream_t st) {
  if (backend == LA_BACKEND_TCGEN05) {
    if (!la::tc_pointers_ok(p)) return cudaErrorMisalignedAddress;
    return la::tc_state(p, ws, st);
  }
  return la::simt_state(dtype, p, ws, st);
}

// This library carries its own (static) CUDA runtime.  A caller's thread may
// have its device selected only through another runtime instance (e.g.
// torch's autograd worker threads), so every entry binds the context that owns
// the caller's stream before touching the runtime or the driver.
template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
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

struct Prepared {
  int backend;
  la::Plan plan;
  size_t need;
};

int prepare(const la_desc* desc, size_t ws_bytes, const void* ws, Prepared* out) {
  int rc = validate(desc);
  if (rc != LA_OK) return rc;
  rc = pick_backend(desc, &out->backend);
  if (rc != LA_OK) return rc;
  out->plan = plan_for(desc, out->backend);
  out->need = ws_bytes_for(desc, out->backend, out->plan);
  if (out->need > 0 && (ws == nullptr || ws_bytes < out->need))
    return fail(LA_ERR_SHAPE, "workspace too small: need %zu bytes, got %zu", out->need, ws_bytes);
  return LA_OK;
}

}  // namespace

extern "C" {

size_t la_workspace_bytes(const la_desc* desc) {
  if (validate(desc) != LA_OK) return 0;
  int backend;
  if (pick_backend(desc, &backend) != LA_OK) return 0;
  return ws_bytes_for(desc, backend, plan_for(desc, backend));
}

int la_fwd(const la_desc* desc, const void* q, const void* k, const void* v, const double* lam,
           const void* kv_in, void* o, void* kv_out, void* workspace, size_t workspace_bytes, void* stream) {
  Prepared pr;
  int rc = prepare(desc, workspace_bytes, workspace, &pr);
  if (rc != LA_OK) return rc;
  if (!q || !k || !v || !o || !lam) return fail(LA_ERR_SHAPE, "la_fwd: null q/k/v/o/lam");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  la::PassDesc p = base_pass(desc, pr.plan, lam);
  p.a = q;
  p.b = k;
  p.c = v;
  p.out = o;
  p.rev = 0;
  p.state_in = kv_in;
  p.state_out = kv_out;
  cudaError_t err = run_pass(pr.backend, desc->dtype, p, workspace, st);
  if (err != cudaSuccess) return cuda_fail(err, "la_fwd");
  return LA_OK;
}

int la_bwd(const la_desc* desc, const void* q, const void* k, const void* v, const void* dout, const double* lam,
           const void* kv_in, const void* dkv_in, void* dq, void* dk, void* dv, void* dkv_out, void* workspace,
           size_t workspace_bytes, void* stream) {
  Prepared pr;
  int rc = prepare(desc, workspace_bytes, workspace, &pr);
  if (rc != LA_OK) return rc;
  if (!q || !k || !v || !dout || !dq || !dk || !dv || !lam)
    return fail(LA_ERR_SHAPE, "la_bwd: null q/k/v/do/dq/dk/dv/lam");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bind_stream_context(st);
  const la::PassDesc base = base_pass(desc, pr.plan, lam);
  cudaError_t err;
  // sweep 1 (kernels.py:309-318): dq = fwd(do, v, k), state kv^T
  la::PassDesc p = base;
  p.a = dout;
  p.b = v;
  p.c = k;
  p.out = dq;
  p.rev = 0;
  p.state_in = kv_in;
  p.state_in_T = 1;
  if ((err = run_pass(pr.backend, desc->dtype, p, workspace, st)) != cudaSuccess) return cuda_fail(err, "la_bwd dq");
  // sweep 2 (kernels.py:320-333): dk = rev(v, do, q), state dkv^T
  p = base;
  p.a = v;
  p.b = dout;
  p.c = q;
  p.out = dk;
  p.rev = 1;
  p.state_in = dkv_in;
  p.state_in_T = 1;
  if ((err = run_pass(pr.backend, desc->dtype, p, workspace, st)) != cudaSuccess) return cuda_fail(err, "la_bwd dk");
  //                              dv = rev(k, q, do), state dkv (written out as R(0))
  p = base;
  p.a = k;
  p.b = q;
  p.c = dout;
  p.out = dv;
  p.rev = 1;
  p.state_in = dkv_in;
  p.state_out = dkv_out;
  if ((err = run_pass(pr.backend, desc->dtype, p, workspace, st)) != cudaSuccess) return cuda_fail(err, "la_bwd dv");
  return LA_OK;
}

int la_fwd_state(const la_desc* desc, const void* k, const void* v, const double* lam, void* kv_delta,
                 void* workspace, size_t workspace_bytes, void* stream) {
  Prepared pr;
  int rc = prepare(desc, workspace_bytes, workspace, &pr);
  if (rc != LA_OK) return rc;
  if (!k || !v || !lam || !kv_delta) return fail(LA_ERR_SHAPE, "la_fwd_state: null k/v/lam/kv_delta");
  bind_stream_context(reinterpret_cast<cudaStream_t>(stream));
  la::PassDesc p = base_pass(desc, pr.plan, lam);
  p.b = k;
  p.c = v;
  p.rev = 0;
  p.state_out = kv_delta;
  cudaError_t err = run_state(pr.backend, desc->dtype, p, workspace, reinterpret_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "la_fwd_state");
  return LA_OK;
}

int la_bwd_state(const la_desc* desc, const void* q, const void* dout, const double* lam, void* dkv_delta,
                 void* workspace, size_t workspace_bytes, void* stream) {
  Prepared pr;
  int rc = prepare(desc, workspace_bytes, workspace, &pr);
  if (rc != LA_OK) return rc;
  if (!q || !dout || !lam || !dkv_delta) return fail(LA_ERR_SHAPE, "la_bwd_state: null q/do/lam/dkv_delta");
  bind_stream_context(reinterpret_cast<cudaStream_t>(stream));
  la::PassDesc p = base_pass(desc, pr.plan, lam);
  p.b = q;
  p.c = dout;
  p.rev = 1;
  p.state_out = dkv_delta;
  cudaError_t err = run_state(pr.backend, desc->dtype, p, workspace, reinterpret_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "la_bwd_state");
  return LA_OK;
}

int la_launch_count(const la_desc* desc, int which) {
  if (validate(desc) != LA_OK) return -1;
  int backend;
  if (pick_backend(desc, &backend) != LA_OK) return -1;
  const la::Plan plan = plan_for(desc, backend);
  const int per_pass = plan.nseg > 1 ? 3 : 1;  // summaries + scan + main, or main only
  return (which == 0 ? 1 : 3) * per_pass;
}

const char* la_last_error(void) { return g_last_error.c_str(); }

int la_abi_version(void) { return LA_ABI_VERSION; }

const char* la_build_info(void) {
  return "lightning-attn b200: sm_100a, backends simt(f64/f32/bf16) + tcgen05(bf16)";
}

}  // extern "C"
