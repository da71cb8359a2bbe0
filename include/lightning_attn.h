/*
 * lightning_attn.h -- C ABI of the B200-native Lightning Attention hot path.
 *
 * Drop-in boundary for the reference package `linattn` (arXiv 2405.17381,
 * /root/reference/pkg/src/linattn).  The reference's hot path is two numpy
 * functions per head; this ABI replaces them with batched, stream-ordered
 * CUDA entry points taking plain device pointers.  No torch / CUDA types
 * appear in the signatures (the stream is an opaque `void*` holding a
 * cudaStream_t).
 *
 *   la_fwd  replaces  lightning_forward_decay(q, k, v, cfg)        kernels.py:253-284
 *                     lightning_forward(q, k, v, cfg)  (lam == 1)  kernels.py:158-183
 *   la_bwd  replaces  lightning_backward_decay(q, k, v, do, cfg)   kernels.py:287-334
 *                     lightning_backward(q, k, v, do, cfg)         kernels.py:186-231
 *   la_desc           AttentionConfig (n, d, B, lam, precision)    kernels.py:69-105,
 *                     batched over (batch, heads); one lam per head (model.py:393-401)
 *   la_status         ShapeError / DomainError                     matrixops.py:28-33
 *   la_fwd_state /    the d x d carried summaries KvState          kernels.py:108-121,
 *   la_bwd_state      exported so sequence segments (multi-GPU sequence parallel,
 *                     chunked prefill) can be chained exactly.
 *
 * Semantics (all pinned by the reference's tests):
 *   o[t]  = sum_{s<=t} lam^(t-s) (q[t].k[s]) v[s]                  causal, decayed
 *   kv_in / kv_out   : forward state  F(p) = sum_{s<p} lam^(p-1-s) k[s] v[s]^T  (d x d)
 *                      i.e. the reference's `state.kv` after the block ending at p.
 *   dkv_in / dkv_out : adjoint state  R(p) = sum_{t>=p} lam^(t-p+1) q[t] do[t]^T
 *                      i.e. the reference's `state.dkv` after the block starting at p.
 *   The block size B is validated (>= 1) and otherwise semantically inert, exactly
 *   as in the reference: the kernels choose their own tile.
 *
 * Memory: every pointer is device memory; q,k,v,o,do,dq,dk,dv use the desc's
 * strides (element strides of batch, head, position; the feature stride is 1),
 * or each its own through la_fwd_ex / la_bwd_ex's la_tensor_strides.
 * States are [batch, heads, d, d] row-major in the accumulation type (float for
 * LA_F32 / LA_BF16, double for LA_F64), 16-byte aligned (LA_ERR_SHAPE otherwise);
 * the tensor-core path also needs 16-byte aligned operand bases and strides.
 * `lam` is a device array of `heads`
 * doubles in (0, 1]; a value outside (0, 1] (or NaN) turns every output of the call into NaN
 * (the reference raises DomainError, matrixops.py:72-77; the ABI does not read lam back per call
 * -- la_check_decay validates a host copy, LA_FLAG_CHECK_DECAY the device one, as LA_ERR_DOMAIN).
 * The caller allocates outputs and the workspace
 * (la_workspace_bytes); the library keeps no global state besides the
 * thread-local error string.  Calls are asynchronous on `stream` and reentrant.
 */
#ifndef LIGHTNING_ATTN_H_
#define LIGHTNING_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LA_ABI_VERSION 4  /* 4: la_gla_core_fwd / la_gla_core_bwd (+ their workspace sizes); LA_BACKEND_TCGEN05 serves fp32 too */

#if defined(__GNUC__)
#define LA_API __attribute__((visibility("default")))
#else
#define LA_API
#endif

typedef enum la_status {
  LA_OK = 0,
  LA_ERR_SHAPE = 1,       /* ShapeError  (kernels.py:137-146)                    */
  LA_ERR_DOMAIN = 2,      /* DomainError (kernels.py:84-91, matrixops.py:72-77)  */
  LA_ERR_CUDA = 3,        /* launch / runtime failure                            */
  LA_ERR_UNSUPPORTED = 4  /* valid request this build does not implement         */
} la_status;

typedef enum la_dtype {
  LA_F32 = 0,   /* reference precision="working"   (float32)                   */
  LA_F64 = 1,   /* reference precision="reference" (float64)                   */
  LA_BF16 = 2   /* bf16 operands, fp32 accumulation and fp32 states            */
} la_dtype;

typedef enum la_backend {
  LA_BACKEND_AUTO = 0,     /* tcgen05 when eligible, else SIMT                  */
  LA_BACKEND_SIMT = 1,     /* CUDA-core kernels (any d <= 128, any dtype)       */
  LA_BACKEND_TCGEN05 = 2   /* TMA + tcgen05/TMEM kernels (bf16 or fp32, d in {32, 64, 96, 128}) */
} la_backend;

typedef struct la_desc {
  int64_t batch;      /* >= 1                                                  */
  int64_t heads;      /* >= 1                                                  */
  int64_t n;          /* sequence length >= 1                                  */
  int64_t d;          /* head dim >= 1                                         */
  int64_t block;      /* reference B (>= 1); 0 = default min(d, n)             */
  int32_t dtype;      /* la_dtype                                              */
  int32_t backend;    /* la_backend                                            */
  int64_t stride[3];  /* element strides of (batch, head, position); feature stride 1 */
  int64_t segments;   /* 0 = auto; else sequence segments per (batch, head)    */
} la_desc;

/* Bytes of scratch the calls below need for this descriptor (may be 0). */
LA_API size_t la_workspace_bytes(const la_desc* desc);

/* Number of sequence segments the library splits each (batch, head) into for
 * this descriptor (1 = no split); -1 on a bad descriptor. */
LA_API int la_segment_count(const la_desc* desc);

/* Forward: o = LA(q, k, v).  kv_in (nullable) seeds the state at position 0;
 * kv_out (nullable) receives F(n).  seg_states_out (nullable; used only when
 * la_segment_count > 1) receives the state entering every segment,
 * [batch, heads, segments, d, d]; passing it to la_bwd spares the backward
 * one summary pass. */
LA_API int la_fwd(const la_desc* desc, const void* q, const void* k, const void* v,
           const double* lam, const void* kv_in, void* o, void* kv_out,
           void* seg_states_out, void* workspace, size_t workspace_bytes, void* stream);

/* Backward: (dq, dk, dv) = d<LA(q,k,v), do>.  kv_in is the forward's kv_in
 * (nullable = zeros); dkv_in (nullable) is R(n), the adjoint state arriving from
 * beyond the sequence end; fwd_seg_states (nullable) is the forward's
 * seg_states_out for the same descriptor and kv_in; dkv_out (nullable)
 * receives R(0). */
LA_API int la_bwd(const la_desc* desc, const void* q, const void* k, const void* v,
           const void* dout, const double* lam, const void* kv_in,
           const void* dkv_in, const void* fwd_seg_states, void* dq, void* dk,
           void* dv, void* dkv_out, void* workspace, size_t workspace_bytes,
           void* stream);

/* ---- extended entry points (ABI 3) --------------------------------------------------------
 * la_fwd_ex / la_bwd_ex are la_fwd / la_bwd with per-tensor strides and flags:
 *   strides  nullable; else every operand's own (batch, head, position) element strides, indexed by
 *            la_operand (la_fwd_ex reads Q, K, V, O; la_bwd_ex Q, K, V, DO, DQ, DK, DV), so q, k, v
 *            of different layouts (e.g. views into a fused projection) need no copy.
 *   flags    LA_FLAG_RESUME: the workspace already holds this problem's segment summaries, left by
 *              la_fwd_state(desc, k, v, lam, ws) (la_fwd_ex) or la_bwd_state(desc, q, do, lam, ws)
 *              (la_bwd_ex, sweep 2) on the same stream -- the summary pass is skipped: a sequence-
 *              parallel rank's own summary (which it computes for the exchange anyway) already holds
 *              the summaries of its segments.
 *              la_bwd_ex with LA_FLAG_RESUME and a split sequence needs fwd_seg_states for sweep 1.
 *            LA_FLAG_CHECK_DECAY: read lam back and validate (0, 1] -> LA_ERR_DOMAIN (synchronises
 *              the stream; debug / first-call validation).
 *            LA_FLAG_CHECK_FINITE: scan the inputs for NaN / Inf -> LA_ERR_DOMAIN, the reference's
 *              ensure_finite (kernels.py:148-149; synchronises the stream, debug option).
 *            LA_FLAG_NO_DQ / LA_FLAG_NO_DKDV (la_bwd_ex): skip sweep 1 (dq unused, may be NULL) /
 *              sweep 2 (dk, dv, dkv_out unused) -- lets a caller overlap one sweep with other work,
 *              e.g. the sequence-parallel state exchange with the dq pass.
 * The CHECK flags synchronise, so they cannot be used under CUDA graph capture. */
typedef enum la_operand {
  LA_T_Q = 0, LA_T_K = 1, LA_T_V = 2, LA_T_O = 3, LA_T_DO = 4, LA_T_DQ = 5, LA_T_DK = 6, LA_T_DV = 7
} la_operand;

typedef struct la_tensor_strides {
  int64_t s[8][3];    /* [la_operand][batch, head, position] element strides */
} la_tensor_strides;

#define LA_FLAG_RESUME        0x1u
#define LA_FLAG_CHECK_DECAY   0x2u
#define LA_FLAG_CHECK_FINITE  0x4u
#define LA_FLAG_NO_DQ         0x8u
#define LA_FLAG_NO_DKDV       0x10u

LA_API int la_fwd_ex(const la_desc* desc, const la_tensor_strides* strides, uint32_t flags, const void* q,
              const void* k, const void* v, const double* lam, const void* kv_in, void* o, void* kv_out,
              void* seg_states_out, void* workspace, size_t workspace_bytes, void* stream);
LA_API int la_bwd_ex(const la_desc* desc, const la_tensor_strides* strides, uint32_t flags, const void* q,
              const void* k, const void* v, const void* dout, const double* lam, const void* kv_in,
              const void* dkv_in, const void* fwd_seg_states, void* dq, void* dk, void* dv, void* dkv_out,
              void* workspace, size_t workspace_bytes, void* stream);

/* Host-side decay validation for a C caller that holds lam on the host (as AttentionConfig does,
 * kernels.py:84-91 / check_decay matrixops.py:72-77): LA_OK, or LA_ERR_DOMAIN naming the value. */
LA_API int la_check_decay(const double* lam_host, int64_t heads);
/* The backend and segment plan of an _ex call come from every operand's strides: keep desc->stride
 * equal to q's so la_segment_count / la_launch_count describe the call.  la_workspace_bytes covers
 * every backend's plan. */

/* Local summaries of one sequence segment, for sequence parallelism:
 *   la_fwd_state: kv_delta  = sum_s lam^(n-1-s) k[s] v[s]^T   (= F(n) with kv_in = 0)
 *   la_bwd_state: dkv_delta = sum_t lam^(t+1)   q[t] do[t]^T  (= R(0) with dkv_in = 0) */
LA_API int la_fwd_state(const la_desc* desc, const void* k, const void* v,
                 const double* lam, void* kv_delta,
                 void* workspace, size_t workspace_bytes, void* stream);
LA_API int la_bwd_state(const la_desc* desc, const void* q, const void* dout,
                 const double* lam, void* dkv_delta,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Recurrent decode, one token per sequence (replaces the per-(layer, head) update of
 * decode_step, model.py:697-701):
 *   kv <- lam * kv + k v^T      in place, [batch, heads, d, d] in the state dtype
 *   o   = q . kv                after the update (the token attends to itself, as in la_fwd)
 * desc->n must be 1; q, k, v, o are addressed with the desc's batch / head strides.  A prefill
 * by la_fwd with kv_out, followed by la_decode steps, reproduces la_fwd over the whole sequence. */
LA_API int la_decode(const la_desc* desc, const void* q, const void* k, const void* v,
              const double* lam, void* kv, void* o, void* stream);

/* ---- GLA layer stages around the attention core (model.py:365-453) -------------------------
 * The GLA layer is  y = [srmsnorm(LA(rot(act(x Wq)), rot(act(x Wk)), x Wv)) * (x Wu)] Wo.
 * The five projections stay library GEMMs; these entry points are the element-wise stages
 * between them, on the model-native [batch, n, heads, d] layout (contiguous, width = heads * d)
 * that la_fwd / la_bwd read directly:
 *   la_gla_prologue      q = rot(act(qp)), k = rot(act(kp))        model.py:381-392,
 *                        act (model.py:60-99), LRPE rot (positional.py:126-150) when theta != NULL
 *   la_gla_prologue_bwd  dqp = act'(qp) rot^-1(dq), dkp likewise; dtheta += the angle gradient
 *                        of q and k (positional.py:153-182, model.py:434-441); workspace sized by
 *                        la_gla_workspace_bytes
 *   la_gla_epilogue      gated = srmsnorm(a) * u (u NULL: no gate), rawnorm[row] = |a_row|
 *                        (model.py:106-116, 402-404)
 *   la_gla_epilogue_bwd  (da, du) from dgated, a, u, rawnorm (model.py:118-129, 417-426)
 * theta: device doubles [d/2]; dtheta: device doubles [d/2], accumulated; rawnorm: [batch * n]
 * in the accumulation type. */
typedef enum la_act {
  LA_ACT_NONE = 0,
  LA_ACT_SWISH = 1,          /* x * sigmoid(x), the reference default gla_act (model.py:215) */
  LA_ACT_ONE_PLUS_ELU = 2
} la_act;

typedef struct la_gla_desc {
  int64_t batch;    /* >= 1                                                          */
  int64_t n;        /* positions per sequence >= 1                                   */
  int64_t heads;    /* >= 1                                                          */
  int64_t d;        /* head dim >= 1 (even when theta is given)                      */
  int32_t dtype;    /* la_dtype                                                      */
  int32_t act;      /* la_act                                                        */
  int64_t offset;   /* LRPE position of each sequence's first row (decode resumes)   */
  double eps;       /* srmsnorm eps, the reference's SRMS_EPS = 1e-8 (model.py:48)   */
} la_gla_desc;

LA_API size_t la_gla_workspace_bytes(const la_gla_desc* desc);
LA_API int la_gla_prologue(const la_gla_desc* desc, const void* qp, const void* kp, const double* theta,
                    void* q, void* k, void* stream);
LA_API int la_gla_prologue_bwd(const la_gla_desc* desc, const void* qp, const void* kp, const double* theta,
                        const void* dq, const void* dk, void* dqp, void* dkp, double* dtheta,
                        void* workspace, size_t workspace_bytes, void* stream);
/* Fused GLA core forward: o = LA(rot(act(qp)), rot(act(kp)), v) with the
 * prologue (act, and LRPE when theta != NULL) applied to each q / k tile in shared memory between its
 * TMA load and the first MMA -- in the segment-summary pass too when the plan splits sequences -- so
 * qp / kp stream straight into the core; q_out / k_out (both or neither) receive the transformed rows
 * for the backward (la_bwd on them).  kv_in / kv_out as la_fwd.  Rows are [batch, n, heads * d],
 * contiguous.  bf16 and d = 128 (LA_ERR_UNSUPPORTED otherwise: la_gla_prologue + la_fwd compute the
 * same in two calls).  Workspace: la_gla_core_workspace_bytes (0 when sequences are not split). */
LA_API size_t la_gla_core_workspace_bytes(const la_gla_desc* desc);
LA_API int la_gla_core_fwd(const la_gla_desc* desc, const void* qp, const void* kp, const void* v,
                    const double* lam, const double* theta, const void* kv_in, void* o, void* q_out,
                    void* k_out, void* kv_out, void* workspace, size_t workspace_bytes, void* stream);
/* Fused GLA core backward: the core's backward (la_bwd on the forward's q = rot(act(qp)), k = rot(act(kp)),
 * v and da = the gradient at the core's output) with the prologue's backward (model.py:434-446: dqp =
 * act'(qp) * R^T dq, dkp likewise) applied to the dq / dK tiles in shared memory before they are stored
 * -- dq and dk never reach HBM (4 rows fewer; measured 0.73-0.93x of la_bwd + la_gla_prologue_bwd on B200,
 * DESIGN.md K7).  No LRPE angle gradient: when theta is learned, use la_bwd + la_gla_prologue_bwd.  bf16,
 * d = 128 (LA_ERR_UNSUPPORTED otherwise); workspace: la_gla_core_bwd_workspace_bytes. */
LA_API size_t la_gla_core_bwd_workspace_bytes(const la_gla_desc* desc);
LA_API int la_gla_core_bwd(const la_gla_desc* desc, const void* qp, const void* kp, const void* q, const void* k,
                    const void* v, const void* da, const double* lam, const double* theta, const void* kv_in,
                    const void* dkv_in, void* dqp, void* dkp, void* dv, void* dkv_out, void* workspace,
                    size_t workspace_bytes, void* stream);
LA_API int la_gla_epilogue(const la_gla_desc* desc, const void* a, const void* u, void* gated,
                    void* rawnorm, void* stream);
LA_API int la_gla_epilogue_bwd(const la_gla_desc* desc, const void* dgated, const void* a, const void* u,
                        const void* rawnorm, void* da, void* du, void* stream);

/* Tensor-parallel GLA (gla_parallel_forward, parallel.py:138-178): each rank runs its heads and
 * gates without the norm, the ONE all-reduce carries [partial output | row sum of squares]:
 *   la_gla_gate_rowsq  gated = a * u (u NULL: a), rowsq[row * rowsq_stride] = sum_c a[row, c]^2
 *                      (accumulation dtype; point rowsq at column out_w of the augmented buffer)
 *   la_gla_rowscale    y[r, :] = red[r, :out_w] sqrt(out_w) / max(sqrt(red[r, out_w]), eps) on the
 *                      reduced [rows, out_w + 1] buffer (accumulation dtype in and out) */
LA_API int la_gla_gate_rowsq(const la_gla_desc* desc, const void* a, const void* u, void* gated,
                      void* rowsq, int64_t rowsq_stride, void* stream);
LA_API int la_gla_rowscale(int dtype, int64_t rows, int64_t out_width, double eps, const void* red,
                    void* y, void* stream);

/* Number of kernels la_fwd (which = 0), la_bwd (which = 1) or la_bwd given the
 * forward's segment states (which = 2) launches for this descriptor; -1 on a
 * bad descriptor. */
LA_API int la_launch_count(const la_desc* desc, int which);

/* Thread-local message for the last non-LA_OK status returned on this thread. */
LA_API const char* la_last_error(void);

/* ABI version (LA_ABI_VERSION) and a build string. */
LA_API int la_abi_version(void);
LA_API const char* la_build_info(void);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* LIGHTNING_ATTN_H_ */
