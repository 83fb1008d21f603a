// decode_floor.cu — development microbenchmark: the per-launch floor of a decode-sized
// BD projection in a CUDA graph of dependent launches (PDL on), on a cold-L2 ring.
// Each CTA streams its share of S bytes of "weights" into shared memory with 1-D bulk
// copies (16 KiB each, all in flight), then writes its share of W bytes of "output" with
// 16-byte stores.  No math: what is left is launch + DRAM latency + transfer + drain,
// i.e. the best a decode kernel moving the same bytes could do.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/df tools/decode_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

constexpr int CHUNK = 16384;

// pre: 0 = plain (wait, then load), 1 = L2 prefetch of the share before the PDL wait
__global__ void __launch_bounds__(256, 1)
    k_stream(const uint8_t* __restrict__ src, size_t S, uint8_t* __restrict__ dst, size_t W, int pre,
             int wait, int slots) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  const size_t per = (S / gridDim.x + CHUNK - 1) / CHUNK * CHUNK;
  const size_t b0 = per * blockIdx.x;
  const size_t b1 = b0 + per < S ? b0 + per : S;
  const int nch = b1 > b0 ? static_cast<int>((b1 - b0 + CHUNK - 1) / CHUNK) : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    if (pre)
      for (int c = 0; c < nch; ++c) {
        const size_t off = b0 + static_cast<size_t>(c) * CHUNK;
        const uint32_t n = static_cast<uint32_t>(b1 - off < CHUNK ? b1 - off : CHUNK);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"(n) : "memory");
      }
  }
  __syncthreads();
  griddep_launch_dependents();
  if (wait) griddep_wait();
  if (threadIdx.x == 0 && nch > 0) {
    uint32_t tot = 0;
    for (int c = 0; c < nch; ++c) {
      const size_t off = b0 + static_cast<size_t>(c) * CHUNK;
      tot += static_cast<uint32_t>(b1 - off < CHUNK ? b1 - off : CHUNK);
    }
    mbar_arrive_expect_tx(&bar, tot);
    for (int c = 0; c < nch; ++c) {
      const size_t off = b0 + static_cast<size_t>(c) * CHUNK;
      const uint32_t n = static_cast<uint32_t>(b1 - off < CHUNK ? b1 - off : CHUNK);
      const uint32_t sm = smem_u32(smem + (c % slots) * CHUNK);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
          "l"(src + off), "r"(n), "r"(smem_u32(&bar))
          : "memory");
    }
  }
  if (nch > 0) mbar_wait(&bar, 0);
  const uint32_t v = smem[threadIdx.x];
  const size_t wper = (W / gridDim.x + 15) / 16 * 16;
  const size_t w0 = wper * blockIdx.x;
  for (size_t o = w0 + threadIdx.x * 16; o < w0 + wper && o < W; o += 256 * 16)
    *reinterpret_cast<uint4*>(dst + o) = make_uint4(v, v, v, v);
}

template <int PB>
struct BigParams {
  uint32_t w[PB / 4];
};

// Same as k_stream, plus a PB-byte __grid_constant__ parameter block (the BD kernels pass
// ~7 KB of tensor maps) and optionally a TMEM allocation (tmem != 0).
template <int PB>
__global__ void __launch_bounds__(256, 1)
    k_stream_p(const __grid_constant__ BigParams<PB> prm, const uint8_t* __restrict__ src, size_t S,
               uint8_t* __restrict__ dst, size_t W, int tmem) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const size_t per = (S / gridDim.x + CHUNK - 1) / CHUNK * CHUNK;
  const size_t b0 = per * blockIdx.x;
  const size_t b1 = b0 + per < S ? b0 + per : S;
  const int nch = b1 > b0 ? static_cast<int>((b1 - b0 + CHUNK - 1) / CHUNK) : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    for (int c = 0; c < nch; ++c) {
      const size_t off = b0 + static_cast<size_t>(c) * CHUNK;
      const uint32_t n = static_cast<uint32_t>(b1 - off < CHUNK ? b1 - off : CHUNK);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"(n) : "memory");
    }
  }
  if (tmem && threadIdx.x < 32) {
    tmem_alloc<1>(&slot, 64);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_launch_dependents();
  griddep_wait();
  if (threadIdx.x == 0 && nch > 0) {
    uint32_t tot = 0;
    for (int c = 0; c < nch; ++c) {
      const size_t off = b0 + static_cast<size_t>(c) * CHUNK;
      tot += static_cast<uint32_t>(b1 - off < CHUNK ? b1 - off : CHUNK);
    }
    mbar_arrive_expect_tx(&bar, tot);
    for (int c = 0; c < nch; ++c) {
      const size_t off = b0 + static_cast<size_t>(c) * CHUNK;
      const uint32_t n = static_cast<uint32_t>(b1 - off < CHUNK ? b1 - off : CHUNK);
      const uint32_t sm = smem_u32(smem + (c % 6) * CHUNK);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
          "l"(src + off), "r"(n), "r"(smem_u32(&bar))
          : "memory");
    }
  }
  if (nch > 0) mbar_wait(&bar, 0);
  const uint32_t v = smem[threadIdx.x] + prm.w[threadIdx.x % (PB / 4)];
  const size_t wper = (W / gridDim.x + 15) / 16 * 16;
  const size_t w0 = wper * blockIdx.x;
  for (size_t o = w0 + threadIdx.x * 16; o < w0 + wper && o < W; o += 256 * 16)
    *reinterpret_cast<uint4*>(dst + o) = make_uint4(v, v, v, v);
  tc_fence_before();
  __syncthreads();
  if (tmem && threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<1>(slot, 64);
  }
}

template <int PB>
void run_p(cudaStream_t s, const std::vector<uint8_t*>& src, const std::vector<uint8_t*>& dst, size_t S,
           size_t W, int grid, int tmem) {
  const int R = static_cast<int>(src.size());
  const int smem = 6 * CHUNK;
  cudaFuncSetAttribute(k_stream_p<PB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  BigParams<PB> prm{};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int inner = 200;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < inner; ++i)
    cudaLaunchKernelEx(&cfg, k_stream_p<PB>, prm, (const uint8_t*)src[i % R], S, dst[i % R], W, tmem);
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
  printf("variant S=%4.1f MB W=%3.1f MB grid=%3d params=%5d B tmem=%d: %6.2f us/launch (%s)\n",
         S / 1048576.0, W / 1048576.0, grid, PB, tmem, best * 1000 / inner,
         cudaGetErrorString(cudaGetLastError()));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int smem = 12 * CHUNK;
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  struct Case { double smb, wmb; };
  {
    const size_t S = 3 * 1048576, W = 512 * 1024;
    const int R = 64;
    std::vector<uint8_t*> src(R), dst(R);
    for (int r = 0; r < R; ++r) {
      cudaMalloc(&src[r], S + 16);
      cudaMalloc(&dst[r], W + 16);
      cudaMemset(src[r], 1, S + 16);
    }
    for (int grid : {64, 148})
      for (int tmem = 0; tmem < 2; ++tmem) {
        run_p<16>(s, src, dst, S, W, grid, tmem);
        run_p<2048>(s, src, dst, S, W, grid, tmem);
        run_p<7168>(s, src, dst, S, W, grid, tmem);
      }
    for (int r = 0; r < R; ++r) {
      cudaFree(src[r]);
      cudaFree(dst[r]);
    }
  }
  const Case cases[] = {{3.0, 0.5}, {12.6, 8.4}};
  for (const Case& cs : cases) {
    const size_t S = static_cast<size_t>(cs.smb * 1024) * 1024, W = static_cast<size_t>(cs.wmb * 1024) * 1024;
    const size_t set = S + W + 4096;
    const int R = static_cast<int>(std::max<size_t>(2, 600ull * 1048576 / set + 1 > 64 ? 64 : 600ull * 1048576 / set + 1));
    std::vector<uint8_t*> src(R), dst(R);
    for (int r = 0; r < R; ++r) {
      cudaMalloc(&src[r], S + 16);
      cudaMalloc(&dst[r], W + 16);
      cudaMemset(src[r], 1, S + 16);
    }
    for (int grid : {148, 296}) {
      for (int pre = 0; pre < 2; ++pre) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = grid > 148 ? smem / 2 : smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (grid > 148 && S / grid > static_cast<size_t>(smem / 2)) continue;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        const int inner = 200;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < inner; ++i)
          cudaLaunchKernelEx(&cfg, k_stream, (const uint8_t*)src[i % R], S, dst[i % R], W, pre, 1,
                             static_cast<int>(cfg.dynamicSmemBytes / CHUNK));
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
        printf("S=%5.1f MB W=%4.1f MB grid=%3d pre=%d: %6.2f us/launch  (%s)\n", cs.smb, cs.wmb, grid,
               pre, best * 1000 / inner, cudaGetErrorString(cudaGetLastError()));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
    }
    for (int r = 0; r < R; ++r) {
      cudaFree(src[r]);
      cudaFree(dst[r]);
    }
  }
}
