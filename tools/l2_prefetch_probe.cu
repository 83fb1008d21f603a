// l2_prefetch_probe.cu — development microbenchmark: does an L2 prefetch issued by one
// kernel make a later kernel's TMA loads of the same data L2 hits?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/pp tools/l2_prefetch_probe.cu -lcuda
// C = 384 x 16384 fp16 (12.6 MB, the paper shape's coefficients); 128 CTAs, each owns a
// 128-column slice (96 KB) like the decode kernel.  Per mode: flush L2 (write 512 MB),
// run the "warm" kernel (mode), then time a kernel that TMA-loads every slice into smem.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

constexpr int K = 384, N = 16384, BN = 128, CTAS = N / BN;

__global__ void flush(int4* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = make_int4(i, 0, 0, 0);
}

// mode 1: tensor prefetch {64 x 64} boxes; mode 2: non-tensor bulk prefetch per 256 B
// row segment; mode 3: plain loads of every line (the data certainly passes L2)
__global__ void warm(const __grid_constant__ CUtensorMap map, const uint16_t* c, int mode,
                     int* sink) {
  const int n0 = blockIdx.x * BN;
  if (mode == 1 && threadIdx.x == 0) {
    for (int kb = 0; kb < K / 64; ++kb)
      for (int q = 0; q < BN / 64; ++q)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&map)), "r"(n0 + 64 * q), "r"(kb * 64)
                     : "memory");
  } else if (mode == 2) {
    for (int k = threadIdx.x; k < K; k += blockDim.x)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       reinterpret_cast<uint64_t>(c + static_cast<size_t>(k) * N + n0)), "r"(BN * 2)
                   : "memory");
  } else if (mode == 3) {
    int acc = 0;
    for (int k = threadIdx.x; k < K * (BN * 2 / 128); k += blockDim.x) {
      const int row = k / (BN * 2 / 128), seg = k % (BN * 2 / 128);
      acc += *reinterpret_cast<const volatile int*>(c + static_cast<size_t>(row) * N + n0 + seg * 64);
    }
    if (acc == 0x12345678) sink[0] = acc;
  }
}

__global__ void __launch_bounds__(128, 1) load(const __grid_constant__ CUtensorMap map,
                                               unsigned long long* t_out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  const int n0 = blockIdx.x * BN;
  unsigned long long t0, t1;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    mbar_arrive_expect_tx(&bar, K * BN * 2);
    for (int kb = 0; kb < K / 64; ++kb)
      for (int q = 0; q < BN / 64; ++q)
        tma_load_2d(sm + (kb * 2 + q) * 8192, &map, n0 + 64 * q, kb * 64, &bar, policy_evict_first());
    mbar_wait(&bar, 0);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    t_out[blockIdx.x] = t1 - t0;
  }
}

int main() {
  uint16_t* c;
  int4* fl;
  int* sink;
  unsigned long long* t;
  const size_t fl_n = (512ull << 20) / 16;
  cudaMalloc(&c, size_t(K) * N * 2);
  cudaMalloc(&fl, fl_n * 16);
  cudaMalloc(&sink, 4);
  cudaMalloc(&t, CTAS * 8);
  cudaMemset(c, 0, size_t(K) * N * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[2] = {N, K}, strides[1] = {N * 2};
  cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, c, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(load, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[] = {"cold (no warm kernel)", "tensor prefetch .L2", "bulk prefetch .L2",
                         "plain loads (warm)"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      flush<<<1184, 512>>>(fl, fl_n);
      if (mode) warm<<<CTAS, 128>>>(map, c, mode, sink);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      load<<<CTAS, 128, 100 * 1024>>>(map, t);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long h[CTAS], mx = 0, sum = 0;
      cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
      for (int i = 0; i < CTAS; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        sum += h[i];
      }
      printf("%-24s load kernel %6.2f us; per-CTA 96 KB arrival mean %.2f us max %.2f us (%s)\n",
             names[mode], ms * 1e3, sum / 1e3 / CTAS, mx / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
