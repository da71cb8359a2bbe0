/*
 * abi_caller.c -- a plain C client of include/lightning_attn.h (test infrastructure).
 *
 * Shows that the drop-in boundary needs nothing but C: the CUDA runtime for device memory and the
 * library's extern "C" entry points (no torch, no Python).  It runs la_fwd / la_bwd on one small problem
 * per dtype (bf16 and fp32 on the tensor cores at d = 128 / 64, fp64 on the SIMT path at d = 40) with entering states,
 * and checks every output against a direct O(n^2 d) restatement in double of the reference's definitions
 * (kernels.py:253-334 as SPEC'd in the header: o[t] = sum_{s<=t} lam^(t-s) (q[t].k[s]) v[s], and its
 * gradients), plus the error contract (a bad descriptor -> LA_ERR_DOMAIN with a message).
 *
 * Build: gcc -std=c11 -I include tests/c/abi_caller.c -L<dir of libla_b200.so> -lla_b200
 *            -L/usr/local/cuda/lib64 -lcudart -lm
 * Prints "abi_caller ok" and exits 0 on success.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lightning_attn.h"

/* the CUDA runtime calls this client needs (declared here so no CUDA header is required) */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t bytes);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* dst, const void* src, size_t bytes, int kind);
extern cudaError_t cudaDeviceSynchronize(void);
enum { H2D = 1, D2H = 2 };

/* bf16 <-> float (round to nearest even) for the bf16 problem */
static unsigned short to_bf16(float x) {
  unsigned int u;
  memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (unsigned short)(u >> 16);
}
static double from_bf16(unsigned short h) {
  unsigned int u = (unsigned int)h << 16;
  float x;
  memcpy(&x, &u, 4);
  return x;
}

static double urand(unsigned long long* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return 0.05 + 0.95 * (double)(*s >> 11) / 9007199254740992.0;
}

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ != 0) {                                                               \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,       \
              la_last_error());                                                   \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

/* direct restatement, one (batch, head) unit, row-major [n][d]; kv0 (d x d) seeds the forward state and
 * dkv0 the adjoint state arriving from beyond the end; dkv_out = R(0) */
static void reference(int n, int d, double lam, const double* q, const double* k, const double* v,
                      const double* dO, const double* kv0, const double* dkv0, double* o, double* dq,
                      double* dk, double* dv, double* kv_out, double* dkv_out) {
  for (int t = 0; t < n; ++t)
    for (int f = 0; f < d; ++f) o[t * d + f] = dq[t * d + f] = dk[t * d + f] = dv[t * d + f] = 0.0;
  for (int t = 0; t < n; ++t) {
    for (int s = 0; s <= t; ++s) {
      const double w = pow(lam, t - s);
      double qk = 0.0, dov = 0.0;
      for (int f = 0; f < d; ++f) qk += q[t * d + f] * k[s * d + f], dov += dO[t * d + f] * v[s * d + f];
      for (int f = 0; f < d; ++f) {
        o[t * d + f] += w * qk * v[s * d + f];
        dq[t * d + f] += w * dov * k[s * d + f];
        dk[s * d + f] += w * dov * q[t * d + f];
        dv[s * d + f] += w * qk * dO[t * d + f];
      }
    }
    /* the entering state: o[t] += lam^(t+1) q[t] kv0; its gradients */
    const double w = pow(lam, t + 1);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        o[t * d + b] += w * q[t * d + a] * kv0[a * d + b];
        dq[t * d + a] += w * dO[t * d + b] * kv0[a * d + b];
      }
  }
  /* the adjoint state arriving from beyond the end, R(n) = dkv0 = dL/dF(n): k[s] and v[s] enter F(n) with
   * weight lam^(n-1-s) */
  for (int s = 0; s < n; ++s) {
    const double w = pow(lam, n - 1 - s);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        dk[s * d + a] += w * v[s * d + b] * dkv0[a * d + b];
        dv[s * d + b] += w * k[s * d + a] * dkv0[a * d + b];
      }
  }
  /* kv_out = F(n) = lam^n kv0 + sum_s lam^(n-1-s) k[s] v[s]^T; dkv_out = R(0) = lam^n dkv0 + sum_t lam^(t+1) q[t] dO[t]^T */
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double f = pow(lam, n) * kv0[a * d + b], r = pow(lam, n) * dkv0[a * d + b];
      for (int s = 0; s < n; ++s) {
        f += pow(lam, n - 1 - s) * k[s * d + a] * v[s * d + b];
        r += pow(lam, s + 1) * q[s * d + a] * dO[s * d + b];
      }
      kv_out[a * d + b] = f;
      dkv_out[a * d + b] = r;
    }
}

static double max_rel(const double* got, const double* want, size_t count) {
  double worst = 0.0;
  for (size_t i = 0; i < count; ++i) {
    const double e = fabs(got[i] - want[i]) / fmax(fabs(want[i]), 1e-30);
    if (e > worst) worst = e;
  }
  return worst;
}

/* one problem: B = 1, H heads (lam per head), n, d, dtype; tolerance `tol` (per-entry relative) */
static void run(int dtype, int H, int n, int d, const double* lams, double tol, const char* label) {
  const size_t esz = dtype == LA_F64 ? 8 : dtype == LA_BF16 ? 2 : 4, ssz = dtype == LA_F64 ? 8 : 4;
  const size_t cnt = (size_t)H * n * d, scnt = (size_t)H * d * d;
  unsigned long long seed = 12345 + (unsigned long long)dtype;
  double* hx[4];
  for (int x = 0; x < 4; ++x) {
    hx[x] = malloc(cnt * sizeof(double));
    for (size_t i = 0; i < cnt; ++i) hx[x][i] = urand(&seed);
    if (dtype == LA_F32)
      for (size_t i = 0; i < cnt; ++i) hx[x][i] = (double)(float)hx[x][i];
    if (dtype == LA_BF16)  /* the reference sees exactly the operands the device sees */
      for (size_t i = 0; i < cnt; ++i) hx[x][i] = from_bf16(to_bf16((float)hx[x][i]));
  }
  double* hs[2];
  for (int x = 0; x < 2; ++x) {
    hs[x] = malloc(scnt * sizeof(double));
    for (size_t i = 0; i < scnt; ++i) hs[x][i] = 0.02 * urand(&seed);
    if (dtype != LA_F64)
      for (size_t i = 0; i < scnt; ++i) hs[x][i] = (double)(float)hs[x][i];
  }
  /* device copies in the call's dtype */
  void* buf = malloc(cnt * 8 > scnt * 8 ? cnt * 8 : scnt * 8);
  void *dx[4], *dout[4], *ds[2], *dso[2], *dlam;
  for (int x = 0; x < 4; ++x) {
    for (size_t i = 0; i < cnt; ++i) {
      if (dtype == LA_F64) ((double*)buf)[i] = hx[x][i];
      else if (dtype == LA_BF16) ((unsigned short*)buf)[i] = to_bf16((float)hx[x][i]);
      else ((float*)buf)[i] = (float)hx[x][i];
    }
    CHECK(cudaMalloc(&dx[x], cnt * esz));
    CHECK(cudaMemcpy(dx[x], buf, cnt * esz, H2D));
    CHECK(cudaMalloc(&dout[x], cnt * esz));
  }
  for (int x = 0; x < 2; ++x) {
    for (size_t i = 0; i < scnt; ++i) {
      if (dtype == LA_F64) ((double*)buf)[i] = hs[x][i];
      else ((float*)buf)[i] = (float)hs[x][i];
    }
    CHECK(cudaMalloc(&ds[x], scnt * ssz));
    CHECK(cudaMemcpy(ds[x], buf, scnt * ssz, H2D));
    CHECK(cudaMalloc(&dso[x], scnt * ssz));
  }
  CHECK(cudaMalloc(&dlam, H * sizeof(double)));
  CHECK(cudaMemcpy(dlam, lams, H * sizeof(double), H2D));

  la_desc desc;
  memset(&desc, 0, sizeof desc);
  desc.batch = 1, desc.heads = H, desc.n = n, desc.d = d, desc.dtype = dtype, desc.backend = LA_BACKEND_AUTO;
  desc.stride[0] = (int64_t)H * n * d, desc.stride[1] = (int64_t)n * d, desc.stride[2] = d;
  const size_t wsb = la_workspace_bytes(&desc);
  void* ws = NULL;
  if (wsb) CHECK(cudaMalloc(&ws, wsb));
  CHECK(la_fwd(&desc, dx[0], dx[1], dx[2], dlam, ds[0], dout[0], dso[0], NULL, ws, wsb, NULL));
  CHECK(la_bwd(&desc, dx[0], dx[1], dx[2], dx[3], dlam, ds[0], ds[1], NULL, dout[1], dout[2], dout[3], dso[1], ws,
               wsb, NULL));
  CHECK(cudaDeviceSynchronize());

  /* reference per head, compare */
  double* got = malloc(cnt * sizeof(double));
  double *ro = malloc(cnt * 8), *rdq = malloc(cnt * 8), *rdk = malloc(cnt * 8), *rdv = malloc(cnt * 8);
  double *rkv = malloc(scnt * 8), *rdkv = malloc(scnt * 8);
  const size_t u = (size_t)n * d, us = (size_t)d * d;
  for (int h = 0; h < H; ++h)
    reference(n, d, lams[h], hx[0] + h * u, hx[1] + h * u, hx[2] + h * u, hx[3] + h * u, hs[0] + h * us,
              hs[1] + h * us, ro + h * u, rdq + h * u, rdk + h * u, rdv + h * u, rkv + h * us, rdkv + h * us);
  const double* want[6] = {ro, rdq, rdk, rdv, rkv, rdkv};
  void* have[6] = {dout[0], dout[1], dout[2], dout[3], dso[0], dso[1]};
  const char* names[6] = {"o", "dq", "dk", "dv", "kv_out", "dkv_out"};
  for (int x = 0; x < 6; ++x) {
    const size_t c = x < 4 ? cnt : scnt, sz = x < 4 ? esz : ssz;
    CHECK(cudaMemcpy(buf, have[x], c * sz, D2H));
    for (size_t i = 0; i < c; ++i)
      got[i] = sz == 8 ? ((double*)buf)[i] : sz == 2 ? from_bf16(((unsigned short*)buf)[i]) : (double)((float*)buf)[i];
    const double e = max_rel(got, want[x], c);
    printf("%s %-8s max rel err %.3e (tol %g)\n", label, names[x], e, tol);
    if (!(e <= tol)) {
      fprintf(stderr, "%s: %s exceeds the tolerance\n", label, names[x]);
      exit(1);
    }
  }
  for (int x = 0; x < 4; ++x) cudaFree(dx[x]), cudaFree(dout[x]), free(hx[x]);
  for (int x = 0; x < 2; ++x) cudaFree(ds[x]), cudaFree(dso[x]), free(hs[x]);
  cudaFree(dlam);
  if (ws) cudaFree(ws);
  free(buf), free(got), free(ro), free(rdq), free(rdk), free(rdv), free(rkv), free(rdkv);
}

int main(void) {
  if (la_abi_version() != LA_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch: header %d, library %d\n", LA_ABI_VERSION, la_abi_version());
    return 1;
  }
  /* the error contract: n = 0 is a DomainError (kernels.py:85-86) with a message, nothing launched */
  la_desc bad;
  memset(&bad, 0, sizeof bad);
  bad.batch = bad.heads = 1, bad.n = 0, bad.d = 8, bad.dtype = LA_F32, bad.stride[0] = bad.stride[1] = 8,
  bad.stride[2] = 8;
  const int rc = la_fwd(&bad, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, 0, NULL);
  if (rc != LA_ERR_DOMAIN || la_last_error() == NULL || la_last_error()[0] == '\0') {
    fprintf(stderr, "bad descriptor: rc %d, message '%s'\n", rc, la_last_error() ? la_last_error() : "(null)");
    return 1;
  }
  const double lams[3] = {1.0, 0.99, 0.5};
  run(LA_BF16, 3, 300, 128, lams, 2e-2, "bf16 (tcgen05, d = 128)");
  run(LA_F32, 3, 300, 64, lams, 1e-4, "fp32 (tcgen05 split pass, d = 64)");
  run(LA_F64, 3, 200, 40, lams, 1e-10, "fp64 (SIMT, d = 40)");
  printf("abi_caller ok (%s)\n", la_build_info());
  return 0;
}
