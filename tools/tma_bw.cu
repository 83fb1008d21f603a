// tma_bw.cu — development microbenchmark: per-SM load throughput of the TMA paths the
// BD kernel could use (2-D tensor boxes vs 1-D bulk copies), L2-resident source.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_bw tools/tma_bw.cu -lcuda
// One CTA per SM, one thread issues loads into an S-stage ring (mbarrier per stage) and
// immediately refills each stage once it lands; reports bytes/clock/SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"

using namespace bdk;

constexpr int STAGES = 8;
constexpr int STAGE_BYTES = 16384;

struct Args {
  CUtensorMap map;   // 2-D map (modes 0/1)
  const char* src;   // 1-D source (mode 2)
  int mode;          // 0: box {64,64} x2 per stage, 1: box {64,128} x1, 2: bulk 8 KiB x2,
                     // 3: as 0 but a CTA pair (cluster of 2): cta_group::2 loads completing
                     //    on the leader's barrier, stages released back to both CTAs
  int iters;
  unsigned long long* clk;
};

__global__ void __launch_bounds__(32, 1) tma_bw_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  const uint64_t pol = policy_evict_last();
  auto issue = [&](int s, int i) {
    uint8_t* dst = smem + s * STAGE_BYTES;
    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
#ifndef WIN
#define WIN 48
#endif
    // walk a window of WIN 8 KiB boxes of the 32 MiB (L2-resident) source
    const int blk = static_cast<int>((blockIdx.x * 7919ull + i * 13ull) % WIN);
    if (a.mode == 0) {
      tma_load_2d(dst, &a.map, 64 * (blk % 64), 64 * ((blk / 64) % 64), &full[s], pol);
      tma_load_2d(dst + 8192, &a.map, 64 * ((blk + 1) % 64), 64 * ((blk / 64) % 64), &full[s], pol);
    } else if (a.mode == 1) {
      tma_load_2d(dst, &a.map, 64 * (blk % 6), 128 * (blk % 32), &full[s], pol);
    } else {
      const char* src = a.src + static_cast<size_t>(blk) * STAGE_BYTES;
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst + h * 8192)),
            "l"(src + h * 8192), "r"(8192), "r"(smem_u32(&full[s])), "l"(pol)
            : "memory");
    }
  };
  for (int s = 0; s < STAGES; ++s) issue(s, s);
  const unsigned long long t0 = clock64();
  for (int i = 0; i < a.iters; ++i) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    issue(s, i + STAGES);
  }
  for (int i = a.iters; i < a.iters + STAGES; ++i) mbar_wait(&full[i % STAGES], (i / STAGES) & 1);
  a.clk[blockIdx.x] = clock64() - t0;
}

__global__ void __launch_bounds__(32, 1) tma_bw_pair_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  cluster_sync();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_last();
    const unsigned long long t0 = clock64();
    const int total = a.iters + STAGES;
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);  // released by the leader
      uint8_t* dst = smem + s * STAGE_BYTES;
      const uint32_t bar = mapa_shared(smem_u32(&full[s]), 0);
      if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE_BYTES);
      const int blk = (blockIdx.x * 7 + i) % 48;
      tma_load_2d_pair(dst, &a.map, 64 * (blk % 32), 64 * (blk % 6), bar, pol);
      tma_load_2d_pair(dst + 8192, &a.map, 64 * ((blk + 1) % 32), 64 * (blk % 6), bar, pol);
      if (rank == 0 && i >= STAGES - 1) {
        // consume the oldest outstanding stage, release it in both CTAs
        const int j = i - (STAGES - 1);
        const int sj = j % STAGES;
        mbar_wait(&full[sj], (j / STAGES) & 1);
        mbar_arrive(&empty[sj]);
        mbar_arrive_remote(mapa_shared(smem_u32(&empty[sj]), 1));
      }
    }
    if (rank == 0) {
      for (int j = total - (STAGES - 1); j < total; ++j) mbar_wait(&full[j % STAGES], (j / STAGES) & 1);
    }
    a.clk[blockIdx.x] = clock64() - t0;
  }
  cluster_sync();
}

// mode 5: cluster of 2 (no cta_group): each CTA loads HALF of every 16 KiB stage and
// multicasts it to both CTAs; each CTA's barrier expects the full 16 KiB (half from
// itself, half from its peer).  Stages are released to the peer with a remote arrive.
__global__ void __launch_bounds__(32, 1) tma_bw_mc_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
    fence_mbar_init();
  }
  cluster_sync();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_last();
    const unsigned long long t0 = clock64();
    const int total = a.iters + STAGES;
    int consumed = 0;
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);  // both CTAs consumed it
      uint8_t* dst = smem + s * STAGE_BYTES + rank * 8192;
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      const int blk = ((blockIdx.x >> 1) * 7 + i) % 48;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
          " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(&a.map)), "r"(64 * ((blk + rank) % 32)), "r"(64 * (blk % 6)),
          "r"(smem_u32(&full[s])), "h"(static_cast<uint16_t>(0x3))
          : "memory");
      if (i >= STAGES - 1) {
        const int j = consumed++;
        const int sj = j % STAGES;
        mbar_wait(&full[sj], (j / STAGES) & 1);
        mbar_arrive(&empty[sj]);
        mbar_arrive_remote(mapa_shared(smem_u32(&empty[sj]), rank ^ 1u));
      }
    }
    while (consumed < total) {
      const int j = consumed++;
      mbar_wait(&full[j % STAGES], (j / STAGES) & 1);
      mbar_arrive(&empty[j % STAGES]);
      mbar_arrive_remote(mapa_shared(smem_u32(&empty[j % STAGES]), rank ^ 1u));
    }
    a.clk[blockIdx.x] = clock64() - t0;
  }
  cluster_sync();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows = 4096, cols = 4096;  // 32 MiB fp16 source (L2-resident after warm-up)
  char* src;
  cudaMalloc(&src, size_t(rows) * cols * 2);
  cudaMemset(src, 1, size_t(rows) * cols * 2);
  unsigned long long* clk;
  cudaMalloc(&clk, sms * sizeof(unsigned long long));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int smem = STAGES * STAGE_BYTES + 2048;
  cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"2-D box {64,64} x2 (MN-major B panels)", "2-D box {64,128} (K-major A)",
                          "1-D bulk 8 KiB x2"};
  for (int mode = 0; mode < 3; ++mode) {
    Args a{};
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, mode == 1 ? 128u : 64u};
    const cuuint32_t es[2] = {1, 1};
    encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.src = src;
    a.mode = mode;
    a.iters = 2000;
    a.clk = clk;
    for (int rep = 0; rep < 2; ++rep) tma_bw_kernel<<<sms, 32, smem>>>(a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_bw_kernel<<<sms, 32, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), clk, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += double(v) / sms;
    const double bytes = double(a.iters) * STAGE_BYTES;
    printf("%-40s  %.1f B/clk/SM   %.2f TB/s chip  (%s)\n", names[mode], bytes / mean,
           bytes * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  {
    Args a{};
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, 64};
    const cuuint32_t es[2] = {1, 1};
    encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.mode = 3;
    a.iters = 2000;
    a.clk = clk;
    const int smem2 = STAGES * STAGE_BYTES + 4096;
    cudaFuncSetAttribute(tma_bw_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = smem2;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, tma_bw_pair_kernel, a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, tma_bw_pair_kernel, a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), clk, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += double(v) / sms;
    const double bytes = double(a.iters) * STAGE_BYTES;
    printf("%-40s  %.1f B/clk/SM   %.2f TB/s chip  (%s)\n", "pair loads (cta_group::2), leader barrier",
           bytes / mean, bytes * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  {
    Args a{};
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, 64};
    const cuuint32_t es[2] = {1, 1};
    encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.mode = 5;
    a.iters = 2000;
    a.clk = clk;
    const int smem2 = STAGES * STAGE_BYTES + 4096;
    cudaFuncSetAttribute(tma_bw_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = smem2;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, tma_bw_mc_kernel, a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, tma_bw_mc_kernel, a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), clk, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += double(v) / sms;
    const double bytes = double(a.iters) * STAGE_BYTES;
    printf("%-40s  %.1f B/clk/SM delivered   %.2f TB/s chip  (%s)\n", "multicast x2 (half issued per CTA)",
           bytes / mean, bytes * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
