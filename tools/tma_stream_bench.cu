// tools/tma_stream_bench.cu -- how much HBM bandwidth can a 1-CTA/SM TMA ring of
// {A,B,C} 128x128 bf16 tiles sustain with no compute?  (design probe for la_tc.cu)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_2405_17381_b200/csrc/la_ptx.cuh"
using namespace la::ptx;

template <int NST, int NT>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                                         const __grid_constant__ CUtensorMap m2, int n, int heads, int seg_len, int hold) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t full[NST], empty[NST];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  const int seg = blockIdx.x, bh = blockIdx.y, bi = bh / heads, hi = bh % heads;
  const int p0 = seg * seg_len, p1 = min(n, p0 + seg_len), nchunks = (p1 - p0 + 127) / 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x / 32;
  const CUtensorMap* maps[3] = {&m0, &m1, &m2};
  if (warp == 0 && threadIdx.x == 0) {
    for (int t = 0; t < nchunks; ++t) {
      const int s = t % NST;
      if (t >= NST) mbar_wait(&empty[s], ((t / NST) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], NT * 32768);
      for (int x = 0; x < NT; ++x)
        for (int hf = 0; hf < 2; ++hf)
          tma_load_4d(maps[x], &full[s], smem + (size_t)(s * NT + x) * 32768 + hf * 16384, hf * 64, p0 + t * 128, hi, bi);
    }
  } else if (warp == 1 && threadIdx.x == 32) {
    for (int t = 0; t < nchunks; ++t) {
      const int s = t % NST;
      mbar_wait(&full[s], (t / NST) & 1);
      const long long t0 = clock64();
      while (clock64() - t0 < hold) {}
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

int main() {
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  const int B = 8, H = 16, N = 8192, D = 128;
  int Bs[3] = {8, 2, 1};
  size_t el = (size_t)B * H * N * D;
  std::vector<void*> bufs(3);
  for (auto& b : bufs) { cudaMalloc(&b, el * 2); cudaMemset(b, 0, el * 2); }
  CUtensorMap maps[3];
  for (int i = 0; i < 3; ++i) {
    cuuint64_t dims[4] = {D, N, H, B};
    cuuint64_t str[3] = {D * 2, (cuuint64_t)N * D * 2, (cuuint64_t)H * N * D * 2};
    cuuint32_t box[4] = {64, 128, 1, 1}, es[4] = {1, 1, 1, 1};
    enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, bufs[i], dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  auto run = [&](auto kern, int nst, int nt, int nseg, const char* name, int hold = 0) {
    size_t smem = (size_t)nst * nt * 32768 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(nseg, B * H);
    int seg_len = ((N / 128 + nseg - 1) / nseg) * 128;
    for (int w = 0; w < 3; ++w) kern<<<grid, 128, smem>>>(maps[0], maps[1], maps[2], N, H, seg_len, hold);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) kern<<<grid, 128, smem>>>(maps[0], maps[1], maps[2], N, H, seg_len, hold);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    double bytes = (double)el * 2 * nt;
    printf("%-28s hold=%5d stages=%d tiles=%d nseg=%d: %.3f ms  %.0f GB/s  (%s)\n", name, hold, nst, nt, nseg, ms, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int bb : {8, 2, 1}) {
    auto runb = [&](auto kern, int nst, int nt, const char* name) {
      size_t smem = (size_t)nst * nt * 32768 + 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      dim3 grid(1, bb * H);
      for (int w = 0; w < 3; ++w) kern<<<grid, 128, smem>>>(maps[0], maps[1], maps[2], N, H, N, 0);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) kern<<<grid, 128, smem>>>(maps[0], maps[1], maps[2], N, H, N, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      double bytes = (double)bb * H * N * D * 2 * nt;
      printf("%-22s ctas=%3d: %.3f ms  %6.0f GB/s total  %5.1f GB/s per CTA\n", name, bb * H, ms, bytes / ms / 1e6,
             bytes / ms / 1e6 / (bb * H));
    };
    runb(stream_kernel<2, 3>, 2, 3, "2 stages x {A,B,C}");
    runb(stream_kernel<3, 2>, 3, 2, "3 stages x {B,C}");
    runb(stream_kernel<6, 1>, 6, 1, "6 stages x {A}");
    runb(stream_kernel<1, 3>, 1, 3, "1 stage x {A,B,C}");
  }
  return 0;
}
