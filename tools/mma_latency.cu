// mma_latency.cu — development microbenchmark: latency of a chain of n dependent
// tcgen05.mma (kind::f16, cta_group::1, M = 128, K = 16, one accumulator) from the first
// issue to the commit's mbarrier completing, for several N; the first chain in a fresh
// CTA ("cold") and a repeat in the same CTA ("warm").  Also: the same n MMAs spread over
// 2 or 4 independent accumulators (k split), and one elected lane issuing vs a loop with
// __syncwarp per k-block like the decode kernel.  Operands are whatever smem holds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ml tools/mma_latency.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
#include "../paper_2510_01718_b200/csrc/tc_common.cuh"
using namespace bdk;

template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) k_chain(int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    tmem_alloc<1>(&slot, 512);
    tmem_relinquish<1>();
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  constexpr uint32_t idesc = make_idesc_f16(false, 128, N, false, true);
  long long t[2];
  for (int rep = 0; rep < 2; ++rep) {
    if (threadIdx.x < 32) {
      const long long t0 = clock64();
      if (elect_one()) {
        for (int i = 0; i < n; ++i) {
          const int acc = i % NACC;
          const uint32_t a0 = smem_u32(smem) + (i % 4) * 32;
          const uint32_t b0 = smem_u32(smem + 65536) + (i % 4) * 2048;
          tc_mma_f16(tm + acc * N, make_smem_desc(a0, 16, 1024), make_smem_desc(b0, 8192, 1024), idesc,
                     i >= NACC ? 1u : 0u);
        }
        tc_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, rep & 1);
      t[rep] = clock64() - t0;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = t[0];
    out[1] = t[1];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<1>(tm, 512);
  }
}

template <int N, int NACC>
void run(long long* d) {
  cudaFuncSetAttribute(k_chain<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int n : {1, 4, 6, 12, 24, 48, 96}) {
    k_chain<N, NACC><<<148, 128, 160 * 1024>>>(n, d);
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=%3d acc=%d n=%3d: cold %6lld clk (%5.0f/mma)  warm %6lld clk (%5.0f/mma)  ideal %4d/mma  %s\n", N,
           NACC, n, h[0], double(h[0]) / n, h[1], double(h[1]) / n, N / 2,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<32, 1>(d);
  run<64, 1>(d);
  run<64, 2>(d);
  run<64, 4>(d);
  run<128, 1>(d);
  run<128, 2>(d);
  run<256, 1>(d);
}
