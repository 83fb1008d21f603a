// tma_ldst.cu — development microbenchmark: TMA load throughput per SM with and without a
// concurrent TMA store stream (the BD kernel's epilogue writes ~0.6 byte per byte loaded).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_ldst tools/tma_ldst.cu -lcuda
// One CTA per SM: warp 0 streams 16 KiB stages ({64,64} x2 boxes, 8-stage ring) from an
// L2-resident 32 MiB array; warp 1 (when enabled) streams 4 KiB {64 cols, 32 rows} boxes
// from a smem buffer to a large output array (distinct per SM), keeping <= 4 in flight.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"

using namespace bdk;

#ifndef STORE_ROWBLK
#define STORE_ROWBLK 16  // 32-row blocks per SM: 16 -> 4 MB per SM (620 MB, DRAM); 2 -> 76 MB (L2)
#endif
constexpr int STAGES = 8;
constexpr int STAGE_BYTES = 16384;

struct Args {
  CUtensorMap src;
  CUtensorMap dst;
  int iters;        // load stages per CTA
  int stores;       // 4 KiB store boxes per CTA
  int lsu;          // 1: the stores go through the LSU (st.global.v4) instead of TMA
  char* out;
  unsigned long long* clk;
};

__global__ void __launch_bounds__(96, 1) ldst_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + STAGES * STAGE_BYTES;  // 4 KiB store source
  uint8_t* rxbuf = stg + 4096;  // mode 2: 4 x 4 KiB receive ring
  uint64_t* full = reinterpret_cast<uint64_t*>(rxbuf + 4 * 4096);
  uint64_t* rx = full + STAGES;
  uint64_t* txe = rx + 4;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&rx[s], 1);
      mbar_init(&txe[s], 1);
    }
    fence_mbar_init();
  }
  if (a.lsu == 2) cluster_sync(); else __syncthreads();
  const uint64_t pol = policy_evict_last();
  if (warp == 0 && lane == 0) {
    auto issue = [&](int s, int i) {
      const int blk = static_cast<int>((blockIdx.x * 7919ull + i * 13ull) % 4096);
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      tma_load_2d(smem + s * STAGE_BYTES, &a.src, 64 * (blk % 64), 64 * ((blk / 64) % 64), &full[s], pol);
      tma_load_2d(smem + s * STAGE_BYTES + 8192, &a.src, 64 * ((blk + 1) % 64), 64 * ((blk / 64) % 64),
                  &full[s], pol);
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
  } else if (warp == 1 && a.lsu == 2) {
    // DSMEM traffic instead of global stores: a ring of 4 x 4 KiB buffers in the peer CTA
    // (cluster of 2), bulk-copied smem -> peer smem, completing on the peer's rx barriers
    if (lane == 0) {
      const uint32_t peer = cluster_ctarank() ^ 1u;
      for (int j = 0; j < a.stores; ++j) {
        const int st = j % 4;
        if (j >= 4) mbar_wait(&txe[st], ((j / 4) - 1) & 1);  // peer consumed that buffer
        const uint32_t dst = mapa_shared(smem_u32(rxbuf + st * 4096), peer);
        const uint32_t bar = mapa_shared(smem_u32(&rx[st]), peer);
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                dst),
            "r"(smem_u32(stg)), "r"(4096), "r"(bar)
            : "memory");
      }
    }
  } else if (warp == 2 && a.lsu == 2) {
    if (lane == 0) {
      const uint32_t peer = cluster_ctarank() ^ 1u;
      for (int j = 0; j < a.stores; ++j) {
        const int st = j % 4;
        mbar_arrive_expect_tx(&rx[st], 4096);
        mbar_wait(&rx[st], (j / 4) & 1);
        mbar_arrive_remote(mapa_shared(smem_u32(&txe[st]), peer));  // buffer free again
      }
    }
  } else if (warp == 1 && a.lsu == 3) {
    // 1-D bulk stores of 4 KiB CONTIGUOUS bytes (vs 32 rows x 128 B boxes 8 KiB apart)
    if (lane == 0) {
      char* out = a.out + static_cast<size_t>(blockIdx.x) * 512 * 8192;
      for (int j = 0; j < a.stores; ++j) {
        const size_t off = static_cast<size_t>(j % (STORE_ROWBLK * 64)) * 4096;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + off),
                     "r"(smem_u32(stg)), "r"(4096)
                     : "memory");
        tma_store_commit();
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
      tma_store_wait_all<0>();
    }
  } else if (warp == 1 && a.lsu == 1) {
    // the same bytes through the LSU: each warp instruction stores 512 contiguous bytes
    // (a 4 KiB box = 8 instructions), coalesced, into the same output rows
    uint4 v = make_uint4(lane, 1, 2, 3);
    char* out = a.out + static_cast<size_t>(blockIdx.x) * 512 * 8192;
    for (int j = 0; j < a.stores; ++j) {
      const int bx = j % 64, by = (j / 64) % STORE_ROWBLK;
      for (int r = 0; r < 32; r += 4) {  // 4 rows x 128 B per instruction
        char* p = out + static_cast<size_t>(32 * by + r + lane / 8) * 8192 + bx * 128 + (lane % 8) * 16;
        *reinterpret_cast<uint4*>(p) = v;
      }
    }
    __threadfence();
    if (lane == 0) a.clk[gridDim.x + blockIdx.x] = 1;
  } else if (warp == 1 && lane == 0) {
    // rows [blockIdx.x * 512, +512) of a 75776 x 4096 output, walked in 32 x 64 boxes
    for (int j = 0; j < a.stores; ++j) {
      const int bx = j % 64, by = (j / 64) % STORE_ROWBLK;
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
              reinterpret_cast<uint64_t>(&a.dst)),
          "r"(smem_u32(stg)), "r"(64 * bx), "r"(static_cast<int>(blockIdx.x) * 512 + 32 * by)
          : "memory");
      tma_store_commit();
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    tma_store_wait_all<0>();
    a.clk[gridDim.x + blockIdx.x] = 1;
  }
  if (a.lsu == 2) cluster_sync();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows = 4096, cols = 4096;
  char *src, *dst;
  cudaMalloc(&src, size_t(rows) * cols * 2);
  cudaMemset(src, 1, size_t(rows) * cols * 2);
  const size_t orows = size_t(sms) * 512;
  cudaMalloc(&dst, orows * cols * 2);
  unsigned long long* clk;
  cudaMalloc(&clk, 2 * sms * sizeof(unsigned long long));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  Args a{};
  {
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, 64};
    const cuuint32_t es[2] = {1, 1};
    encode(&a.src, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(orows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, 32};
    const cuuint32_t es[2] = {1, 1};
    encode(&a.dst, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dst, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  a.clk = clk;
  a.out = dst;
  a.iters = 3000;
  const int smem = STAGES * STAGE_BYTES + 4096 + 4 * 4096 + 2048;
  cudaFuncSetAttribute(ldst_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 4; ++mode)
  for (int ratio10 : {0, 3, 6, 10}) {  // store bytes per 10 load bytes
    a.lsu = mode;
    a.stores = a.iters * STAGE_BYTES / 4096 * ratio10 / 10;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms / 2 * 2); cfg.blockDim = dim3(96); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = mode == 2 ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, ldst_kernel, a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, ldst_kernel, a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), clk, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += double(v) / sms;
    const double lb = double(a.iters) * STAGE_BYTES, sb = double(a.stores) * 4096;
    printf("%s store:load %.1f  loads %.1f B/clk/SM (%.2f TB/s)  total %.2f TB/s  kernel %.3f ms  (%s)\n",
           mode == 3 ? "BULK1D" : mode == 2 ? "DSMEM" : (mode ? "LSU" : "TMA"), ratio10 / 10.0, lb / mean, lb * sms / (ms * 1e-3) / 1e12,
           (lb + sb) * sms / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
