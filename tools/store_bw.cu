// store_bw.cu — development microbenchmark: how fast can the SMs write a DRAM-sized
// output (cfg2 writes 67 MB of K'/V' per launch), alone and with a concurrent TMA load
// stream like the projection's B re-reads (L2-resident source).  CUDA graph of back-to-back
// launches over a ring of output buffers larger than L2; 148 CTAs (one per SM).
//   mode 0: st.global.v4 from registers (coalesced rows)
//   mode 1: 1-D bulk stores smem -> global (cp.async.bulk, 16 KB each, 4 in flight)
//   mode 2: mode 1 + bulk loads L2 -> smem of `ld_ratio` bytes per stored byte
// Grids of 16..148 CTAs separate a per-SM store limit from the memory system's.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/sb tools/store_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

constexpr int CH = 16384;

__global__ void __launch_bounds__(256, 1)
    k_store(uint8_t* __restrict__ dst, size_t W, const uint8_t* __restrict__ src, size_t S, int mode,
            float ld_ratio) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const size_t per = (W / gridDim.x) / CH * CH;
  uint8_t* d0 = dst + per * blockIdx.x;
  if (mode == 0) {
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (size_t o = threadIdx.x * 16; o < per; o += 256 * 16) *reinterpret_cast<uint4*>(d0 + o) = v;
    return;
  }
  // smem: 4 store buffers (64 KB) + 4 load slots (64 KB), one mbarrier per load slot
  __shared__ uint64_t lbar[4];
  if (threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) mbar_init(&lbar[j], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nst = static_cast<int>(per / CH);
  const size_t sper = (S / gridDim.x) / CH * CH;
  const uint8_t* s0 = src + sper * blockIdx.x;
  int nl = 0;  // loads issued
  for (int i = 0; i < nst; ++i) {
    const int want = mode == 2 ? static_cast<int>((i + 1) * ld_ratio) : 0;
    for (; nl < want; ++nl) {
      const int j = nl % 4;
      if (nl >= 4) mbar_wait(&lbar[j], ((nl / 4) - 1) & 1);  // the slot's previous load landed
      mbar_arrive_expect_tx(&lbar[j], CH);
      const size_t off = (static_cast<size_t>(nl) * CH) % sper;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + 65536 + j * CH)),
          "l"(s0 + off), "r"(CH), "r"(smem_u32(&lbar[j]))
          : "memory");
    }
    asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d0 + static_cast<size_t>(i) * CH),
                 "r"(smem_u32(smem + (i % 4) * CH)), "r"(CH)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  for (int k = nl - 4 > 0 ? nl - 4 : 0; k < nl; ++k) mbar_wait(&lbar[k % 4], (k / 4) & 1);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaStream_t s;
  cudaStreamCreate(&s);
  const size_t W = 64ull << 20, S = 32ull << 20;
  const int R = 6;
  std::vector<uint8_t*> dst(R);
  for (auto& p : dst) cudaMalloc(&p, W);
  uint8_t* src;
  cudaMalloc(&src, S);
  cudaMemset(src, 1, S);
  struct V { int mode; float ratio; int grid; };
  for (V v : {V{0, 0.f, 148}, V{1, 0.f, 148}, V{2, 1.0f, 148}, V{2, 1.5f, 148}, V{2, 2.0f, 148},
              V{1, 0.f, 16}, V{1, 0.f, 37}, V{1, 0.f, 74}, V{0, 0.f, 16}, V{0, 0.f, 74},
              V{2, 2.0f, 16}, V{2, 2.0f, 74}}) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    const int inner = 30;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < inner; ++i)
      k_store<<<v.grid, 256, 131072, s>>>(dst[i % R], W, src, S, v.mode, v.ratio);
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
    printf("mode %d ld_ratio %.1f grid %3d: %7.2f us per 64 MB written -> %6.0f GB/s stores "
           "(%5.1f GB/s per SM) (+ %6.0f GB/s L2 loads)  %s\n",
           v.mode, v.ratio, v.grid, us, W / us / 1e3, W / us / 1e3 / v.grid,
           v.mode == 2 ? W * v.ratio / us / 1e3 : 0.0, cudaGetErrorString(cudaGetLastError()));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
}
