// mcast_bw.cu — development microbenchmark: does TMA multicast relieve the SM<->L2
// contention that bounds the cfg2 epilogue?  148 CTAs (one per SM) each write a share of a
// DRAM-sized output with bulk stores (as the epilogue's TMA stores) while a second thread
// bulk-loads `ratio` bytes per stored byte into a shared-memory ring (as the B stream: 1.5
// at cfg2).  With a cluster of C CTAs each load round is split into C pieces, every CTA
// issuing one piece multicast to all C: every SM still receives the same bytes, L2 serves
// 1/C of them.  Same delivered bytes for C = 1, 2, 4 -> if the time drops with C, the L2
// side (not the SM ports) is the shared limit and multicasting B across pairs would pay.
// Loads are 1-D bulk copies (tensor = 0) or, like the projection's B stream, 2-D tensor-map
// TMA boxes of 128 rows x 128 B with the 128-byte swizzle (tensor = 1; a cluster of C
// splits each box into C sub-boxes of 128 / C rows, each multicast to all C CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mb tools/mcast_bw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

constexpr int CH = 16384;  // store chunk and load round bytes (per CTA)
constexpr int NSLOT = 10;  // load ring
constexpr int LAG = 8;     // rounds in flight

__global__ void __launch_bounds__(128, 1)
    k_mcast(uint8_t* __restrict__ dst, size_t W, const uint8_t* __restrict__ src, size_t S,
            int do_store, float ratio, int C, const __grid_constant__ CUtensorMap map, int tensor) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[NSLOT], freeb[NSLOT];
  const uint32_t rank = C > 1 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int j = 0; j < NSLOT; ++j) {
      mbar_init(&full[j], 1);
      mbar_init(&freeb[j], C);
    }
    fence_mbar_init();
  }
  if (C > 1)
    cluster_sync();
  else
    __syncthreads();
  const size_t per = (W / gridDim.x) / CH * CH;
  const int nst = static_cast<int>(per / CH);
  if (threadIdx.x == 0 && do_store) {
    uint8_t* d0 = dst + per * blockIdx.x;
    for (int i = 0; i < nst; ++i) {
      asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                       d0 + static_cast<size_t>(i) * CH),
                   "r"(smem_u32(smem + (i % 4) * CH)), "r"(CH)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (threadIdx.x == 32) {
    const int R = static_cast<int>(nst * ratio);
    const int piece = CH / C;
    // the cluster reads one region per round (every CTA the same bytes), the clusters
    // spread over S
    const size_t sper = (S / (gridDim.x / C)) / CH * CH;
    const uint8_t* s0 = src + sper * (blockIdx.x / C);
    uint8_t* ring = smem + 4 * CH;
    const uint16_t mask = static_cast<uint16_t>((1u << C) - 1u);
    for (int j = 0; j < R + LAG; ++j) {
      if (j < R) {
        const int s = j % NSLOT;
        if (j >= NSLOT) mbar_wait(&freeb[s], ((j / NSLOT) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], CH);
        const size_t off = (static_cast<size_t>(j) * CH) % sper + rank * piece;
        if (tensor) {
          // 128-row box split into C sub-boxes; row coordinate of this CTA's piece
          const int row = static_cast<int>((sper * (blockIdx.x / C) + off) / 128);
          if (C == 1)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(ring + s * CH)),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(row), "r"(smem_u32(&full[s]))
                : "memory");
          else
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                    smem_u32(ring + s * CH + rank * piece)),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(row), "r"(smem_u32(&full[s])),
                "h"(mask)
                : "memory");
        } else if (C == 1)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(ring + s * CH)),
              "l"(s0 + off), "r"(CH), "r"(smem_u32(&full[s]))
              : "memory");
        else
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
              " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(ring + s * CH + rank * piece)),
              "l"(s0 + off), "r"(piece), "r"(smem_u32(&full[s])), "h"(mask)
              : "memory");
      }
      const int k = j - LAG;  // consume round k: every CTA's slot k % NSLOT is then free
      if (k >= 0) {
        const int s = k % NSLOT;
        mbar_wait(&full[s], (k / NSLOT) & 1);
        for (int r = 0; r < C; ++r) mbar_arrive_remote(mapa_shared(smem_u32(&freeb[s]), r));
      }
    }
  }
  __syncthreads();
  if (C > 1) cluster_sync();  // no CTA exits while a peer may still multicast into it
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int SMEM = 4 * CH + NSLOT * CH;  // 224 KiB
  cudaFuncSetAttribute(k_mcast, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(k_mcast, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaStream_t s;
  cudaStreamCreate(&s);
  const size_t W = 64ull << 20, S = 32ull << 20;
  const int R = 6;
  std::vector<uint8_t*> dst(R);
  for (auto& p : dst) cudaMalloc(&p, W);
  uint8_t* src;
  cudaMalloc(&src, S);
  cudaMemset(src, 1, S);
  // tensor maps over src as [S / 128 rows][64 x 16-bit], box {64, 128 / C}, 128-B swizzle
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap maps[5];
  for (int c : {1, 2, 4}) {
    cuuint64_t dims[2] = {64, S / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(128 / c)}, es[2] = {1, 1};
    encode(&maps[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  struct V { int store; float ratio; int C; int tensor; };
  for (V v : {V{1, 0.f, 1, 0}, V{0, 1.5f, 1, 0}, V{0, 1.5f, 2, 0}, V{1, 1.5f, 1, 0},
              V{1, 1.5f, 2, 0}, V{0, 1.5f, 1, 1}, V{0, 1.5f, 2, 1}, V{0, 1.5f, 4, 1},
              V{1, 1.5f, 1, 1}, V{1, 1.5f, 2, 1}, V{1, 1.5f, 4, 1}, V{1, 2.0f, 1, 1},
              V{1, 2.0f, 2, 1}}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = v.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    const int inner = 30;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < inner; ++i)
      cudaLaunchKernelEx(&cfg, k_mcast, dst[i % R], W, (const uint8_t*)src, S, v.store, v.ratio,
                         v.C, maps[v.C], v.tensor);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    const double us = best * 1000 / inner;
    printf("%s store %d load ratio %.1f cluster %d: %7.2f us -> stores %6.0f GB/s, loads delivered "
           "%6.0f GB/s (L2 reads %6.0f GB/s)  %s\n",
           v.tensor ? "tensor" : "bulk  ", v.store, v.ratio, v.C, us, v.store ? W / us / 1e3 : 0.0, W * v.ratio / us / 1e3,
           W * v.ratio / v.C / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
}
