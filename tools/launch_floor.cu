// launch_floor.cu — development microbenchmark: back-to-back launch cost (CUDA graph)
// of an empty kernel with the BD kernel's launch shape (148 CTAs in clusters of 2,
// 320 threads, ~225 KiB dynamic smem), with and without TMEM alloc + cluster syncs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/lf tools/launch_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

__global__ void __launch_bounds__(320, 1) k_empty(int mode) {
  extern __shared__ uint8_t smem[];
  __shared__ uint32_t slot;
  if (mode >= 1) {
    if (warp_id() == 1) { tmem_alloc<2>(&slot, 512); tmem_relinquish<2>(); }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (mode >= 2) { griddep_wait(); griddep_launch_dependents(); }
    tc_fence_before();
    cluster_sync();
    if (warp_id() == 1) { tc_fence_after(); tmem_dealloc<2>(slot, 512); }
  }
  if (smem[threadIdx.x] == 123 && mode == 99) smem[0] = 1;
}

int main() {
  const int smem = 230656;
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int mode = 0; mode < 3; ++mode) for (int pdl = 0; pdl < 2; ++pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 2 : 1;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k_empty, mode);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (0 empty, 1 +tmem/cluster sync, 2 +griddep) pdl %d: %.2f us/launch (%s)\n", mode, pdl, ms * 10, cudaGetErrorString(cudaGetLastError()));
  }
}
