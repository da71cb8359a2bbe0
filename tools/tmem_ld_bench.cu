// tools/tmem_ld_bench.cu -- tcgen05.ld throughput per SM vs number of warps (design probe for the
// P/state/output warps of la_tc.cu): each warp loads 32 lanes x 32 columns (4 KB) per instruction.
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2405_17381_b200/csrc/la_ptx.cuh"
using namespace la::ptx;

__global__ void __launch_bounds__(1024, 1) ld_kernel(int iters, int nwarps, int waitmode, unsigned long long* out) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32 % 512);
  float acc = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      float v[32];
      tmem_ld32(tm, v);
      if (waitmode == 0 || (i & 3) == 3) tmem_ld_wait();
      acc += v[0] + v[31];
    }
    tmem_ld_wait();
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[1000] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(base, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  unsigned long long h;
  const int iters = 4096;
  for (int wm = 0; wm < 2; ++wm)
    for (int nw : {1, 2, 4, 8, 16, 32}) {
      ld_kernel<<<1, 1024>>>(iters, nw, wm, d);
      ld_kernel<<<1, 1024>>>(iters, nw, wm, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      double bytes = (double)iters * nw * 4096;
      printf("wait=%s warps=%2d: %8.1f cyc per ld per warp, %6.1f B/cyc per SM  (%s)\n", wm ? "every4" : "each  ", nw,
             (double)h / iters, bytes / h, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
