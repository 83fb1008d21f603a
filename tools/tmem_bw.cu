// tmem_bw.cu — development microbenchmark: tcgen05.ld (32x32b) throughput per SM for
// 4/8/16 warps, x16 vs x32 loads, one load in flight per warp vs two.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tb tools/tmem_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

template <int W>
__global__ void k(int iters, unsigned long long* out, int two) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc<1>(&slot, 512); tmem_relinquish<1>(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t base = slot + ((uint32_t(warp & 3) * 32u) << 16);
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32], q[32];
    const uint32_t col = ((i * 64) + (warp >> 2) * 32) & 511;
    tmem_ld_32x32b_x32(base + col, r);
    if (two) tmem_ld_32x32b_x32(base + ((col + 256) & 511), q);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= r[j] ^ (two ? q[j] : 0u);
  }
  const unsigned long long t1 = clock64();
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(slot, 512); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 0x12345678u) out[1] = acc;
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  const int iters = 4000;
  auto run = [&](auto kern, int warps, int two) {
    kern<<<148, warps * 32>>>(iters, d, two); cudaDeviceSynchronize();
    kern<<<148, warps * 32>>>(iters, d, two); cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = double(iters) * warps * 32 * 32 * 4 * (two ? 2 : 1);
    printf("warps %2d loads/iter %d: %.1f B/clk/SM  (%.0f clk per x32 load per warp)  %s\n", warps, two ? 2 : 1,
           bytes / c, double(c) / iters / (two ? 2 : 1), cudaGetErrorString(cudaGetLastError()));
  };
  run(k<4>, 4, 0); run(k<4>, 4, 1); run(k<8>, 8, 0); run(k<8>, 8, 1); run(k<16>, 16, 0); run(k<16>, 16, 1);
}
