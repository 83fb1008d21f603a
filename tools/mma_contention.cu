// mma_contention.cu — development microbenchmark: does the pair tcgen05.mma (M=256, N=256,
// K=16, kind::f16) slow down when other warps of the same CTAs load the SM's shared
// memory, read TMEM, or stream bulk copies from L2 into shared memory?  One cluster of
// two CTAs per SM pair, 148 CTAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o exp/mc tools/mma_contention.cu
//
// mode 0: MMA alone (A and B from smem, "SS")        mode 4: A from TMEM ("TS") alone
// mode 1: + 8 warps st.shared.v4/ld.shared.v4 loop     mode 5: TS + smem hog
// mode 2: + 8 warps tcgen05.ld of the other 256 cols   mode 6: TS + TMEM-read hog
// mode 3: + 1 warp bulk copies L2 -> smem (64 KB ring)  mode 7: TS + bulk-copy hog
// mode 8: + smem hog at ~1/2 rate (every other iteration idles)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
using namespace bdk;

constexpr int NTHR = 64 + 256;
constexpr int NMMA = 4096;  // MMAs per measurement (K=16 each)

__device__ __forceinline__ void tc_mma_ts_pair(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int mode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHR, 1)
    k(const uint8_t* __restrict__ gsrc, size_t gbytes, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;               // 16 KB: 128 x 64 K-major SW128
  uint8_t* sB = sm + 16384;       // 16 KB: 2 panels of 64 cols x 64 k, MN-major SW128
  uint8_t* sH = sm + 32768;       // 64 KB hog region / bulk ring
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 32768 + 65536);
  uint64_t* done = bars;          // MMA group commits (2 barriers)
  uint64_t* ring = bars + 2;      // 4 bulk-copy barriers
  volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(bars + 8);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 9);
  const uint32_t warp = warp_id(), lane = lane_id(), rank = cluster_ctarank();
  constexpr bool ts = mode >= 4 && mode <= 7;
  constexpr int hog = ts ? mode - 4 : (mode == 8 ? 1 : mode);
  if (threadIdx.x == 0) {
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&ring[i], 1);
    *flag = 0;
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 32768 / 16; i += NTHR)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  if (warp == 1) {
    tmem_alloc<2>(slot, 512);
    tmem_relinquish<2>();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *slot;
  if (warp == 1) {
    unsigned long long t0 = clock64();
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc_f16(false, 256, 256, false, true);
      for (int i = 0; i < NMMA / 16; ++i) {
        if (elect_one()) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int ks = u & 3;
            const uint64_t bdesc = make_smem_desc(smem_u32(sB) + ks * 2048, 8192, 1024);
            if (ts)
              tc_mma_ts_pair(tbase, tbase + 256 + ks * 8, bdesc, idesc, (i | u) != 0);
            else
              tc_mma_f16_pair(tbase, make_smem_desc(smem_u32(sA) + ks * 32, 16, 1024), bdesc,
                              idesc, (i | u) != 0);
          }
          if ((i & 15) == 15) tc_commit_pair(&done[(i >> 4) & 1], 0x3);
        }
        __syncwarp();
        if ((i & 15) == 15 && i >= 31) {
          const int g = (i >> 4) - 1;  // wait for the previous group
          mbar_wait(&done[g & 1], (g >> 1) & 1);
        }
      }
    }
    const int g = NMMA / 256 - 1;
    mbar_wait(&done[g & 1], (g >> 1) & 1);
    unsigned long long t1 = clock64();
    if (lane == 0) {
      *flag = 1;
      if (rank == 0) out[blockIdx.x * 4 + 0] = t1 - t0;
    }
  } else if (warp >= 2 && hog == 1) {
    // shared-memory hog: 16-byte stores then loads over a 32 KB slice, conflict-free
    uint32_t x = threadIdx.x;
    unsigned long long bytes = 0, t0 = clock64(), it = 0;
    uint4* p = reinterpret_cast<uint4*>(sH) + (warp - 2) * 256;
    while (!*flag) {
      if (mode == 8 && (it++ & 1)) { __nanosleep(100); continue; }
#pragma unroll 4
      for (int j = 0; j < 8; ++j) {
        p[(j * 32 + lane) & 255] = make_uint4(x, x + 1, x + 2, x + 3);
        uint4 v = p[((j + 3) * 32 + lane) & 255];
        x ^= v.x + v.w;
      }
      bytes += 8 * 32 * 32;
    }
    unsigned long long t1 = clock64();
    if (x == 0xdeadbeef) out[0] = 0;
    if (lane == 0) atomicAdd(&out[blockIdx.x * 4 + 1], bytes), atomicMax(&out[blockIdx.x * 4 + 2], t1 - t0);
  } else if (warp >= 2 && hog == 2) {
    // TMEM-read hog on columns the MMA does not write (256..511 in SS mode; TS mode
    // reads its A there too — contention on the same columns is the point of mode 6)
    const uint32_t q = (warp & 3) * 32;
    uint32_t acc = 0, r[32];
    unsigned long long bytes = 0, t0 = clock64();
    while (!*flag) {
      tmem_ld_32x32b_x32(tbase + (q << 16) + 256 + ((warp - 2) >> 2) * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j];
      bytes += 32 * 32 * 4;
    }
    unsigned long long t1 = clock64();
    if (acc == 0xdeadbeef) out[0] = 0;
    if (lane == 0) atomicAdd(&out[blockIdx.x * 4 + 1], bytes), atomicMax(&out[blockIdx.x * 4 + 2], t1 - t0);
  } else if (warp == 2 && hog == 3) {
    // bulk-copy hog: 16 KB copies L2 -> smem, 4 in flight
    unsigned long long bytes = 0, t0 = clock64();
    uint32_t it = 0;
    const size_t nchunk = gbytes / 16384;
    while (!*flag) {
      const uint32_t s = it & 3;
      if (it >= 4) mbar_wait(&ring[s], ((it >> 2) - 1) & 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&ring[s], 16384);
        const uint8_t* src = gsrc + ((blockIdx.x * 37 + it) % nchunk) * 16384;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                smem_u32(sH + s * 16384)),
            "l"(src), "r"(smem_u32(&ring[s]))
            : "memory");
      }
      __syncwarp();
      ++it;
      bytes += 16384;
    }
    for (uint32_t j = (it > 4 ? it - 4 : 0); j < it; ++j) mbar_wait(&ring[j & 3], (j >> 2) & 1);
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 4 + 1] = bytes, out[blockIdx.x * 4 + 2] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tbase, 512);
  }
}

// layout sweep: bit0 B K-major (else MN-major), bit1 A from TMEM, bit2 N=128 (else 256),
// bit3 cta_group::1 M=128 (else pair M=256).  The elected lane issues 16 MMAs per
// iteration (compile-time descriptors), so the loop is not issue-bound.
template <int CFG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHR, 1) ksweep(unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + 16384;
  uint64_t* done = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 4);
  const uint32_t warp = warp_id(), lane = lane_id(), rank = cluster_ctarank();
  constexpr bool bk = CFG & 1, ts = CFG & 2, n128 = CFG & 4, one = CFG & 8;
  if (threadIdx.x == 0) {
    mbar_init(&done[0], 1);
    mbar_init(&done[1], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 49152 / 16; i += NTHR)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  if (warp == 1) {
    if (one) tmem_alloc<1>(slot, 512), tmem_relinquish<1>();
    else tmem_alloc<2>(slot, 512), tmem_relinquish<2>();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *slot;
  if (warp == 1) {
    unsigned long long t0 = clock64();
    constexpr uint32_t N = n128 ? 128 : 256;
    constexpr uint32_t idesc = make_idesc_f16(false, one ? 128 : 256, N, false, !bk);
    if (rank == 0 || one) {
      for (int i = 0; i < NMMA / 16; ++i) {
        if (elect_one()) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int ks = u & 3;
            const uint64_t bdesc = bk ? make_smem_desc(smem_u32(sB) + ks * 32, 16, 1024)
                                      : make_smem_desc(smem_u32(sB) + ks * 2048, 8192, 1024);
            const uint64_t adesc = make_smem_desc(smem_u32(sA) + ks * 32, 16, 1024);
            const uint32_t acc = (i | u) != 0;
            if (one) {
              if (ts) tc_mma_f16_ts(tbase, tbase + 256 + ks * 8, bdesc, idesc, acc);
              else tc_mma_f16(tbase, adesc, bdesc, idesc, acc);
            } else {
              if (ts) tc_mma_ts_pair(tbase, tbase + 256 + ks * 8, bdesc, idesc, acc);
              else tc_mma_f16_pair(tbase, adesc, bdesc, idesc, acc);
            }
          }
          if ((i & 15) == 15) {
            if (one) tc_commit(&done[(i >> 4) & 1]);
            else tc_commit_pair(&done[(i >> 4) & 1], 0x3);
          }
        }
        __syncwarp();
        if ((i & 15) == 15 && i >= 31) {
          const int g = (i >> 4) - 1;
          mbar_wait(&done[g & 1], (g >> 1) & 1);
        }
      }
    }
    const int g = NMMA / 256 - 1;
    mbar_wait(&done[g & 1], (g >> 1) & 1);
    unsigned long long t1 = clock64();
    if (lane == 0 && rank == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if (one) tmem_dealloc<1>(tbase, 512);
    else tmem_dealloc<2>(tbase, 512);
  }
}

template <int CFG>
void run_sweep(unsigned long long* out) {
  cudaFuncSetAttribute(ksweep<CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
  double best = 1e30;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(out, 0, 148 * 4 * 8);
    ksweep<CFG><<<148, NTHR, 65536 + 2048>>>(out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cfg %d: %s\n", CFG, cudaGetErrorString(e)); exit(1); }
    unsigned long long h[148];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int b = 0; b < 148; b += 2) s += h[b];
    best = s / 74 / NMMA < best ? s / 74 / NMMA : best;
  }
  const int M = (CFG & 8) ? 128 : 256, N = (CFG & 4) ? 128 : 256;
  const double ideal = (CFG & 8) ? (double)M * N / 256 : (double)M * N / 512;
  printf("%s M=%d N=%d B %s A %s: %.1f clk/instr (ideal %.0f, %.0f%%)\n", (CFG & 8) ? "1cta" : "pair",
         M, N, (CFG & 1) ? "K-major " : "MN-major", (CFG & 2) ? "tmem" : "smem", best, ideal,
         100 * ideal / best);
}

template <int mode>
void run_mode(uint8_t* g, size_t gbytes, unsigned long long* out) {
  const int smem = 1024 + 32768 + 65536 + 256;
  cudaFuncSetAttribute(k<mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"SS alone", "SS + smem hog", "SS + TMEM-read hog", "SS + bulk L2->smem",
                         "TS alone", "TS + smem hog", "TS + TMEM-read hog", "TS + bulk L2->smem",
                         "SS + half smem hog"};
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(out, 0, 148 * 4 * 8);
    k<mode><<<148, NTHR, smem>>>(g, gbytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); exit(1); }
    unsigned long long h[148 * 4];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double mma = 0, hb = 0, hc = 0;
    int n = 0;
    for (int b = 0; b < 148; b += 2) {
      mma += h[b * 4];
      hb += h[b * 4 + 1];
      hc += h[b * 4 + 2] ? h[b * 4 + 2] : 1;
      ++n;
    }
    if (rep == 1)
      printf("%-22s MMA %.1f clk/instr (ideal 128)   hog %.1f B/clk on the leader SM\n", names[mode],
             mma / n / NMMA, hb / hc);
  }
}

int main() {
  const size_t gbytes = 32u << 20;
  uint8_t* g;
  cudaMalloc(&g, gbytes);
  cudaMemset(g, 0, gbytes);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 4 * 8);
  const int smem = 1024 + 32768 + 65536 + 256;
  run_mode<0>(g, gbytes, out); run_mode<1>(g, gbytes, out); run_mode<2>(g, gbytes, out);
  run_mode<3>(g, gbytes, out); run_mode<4>(g, gbytes, out); run_mode<5>(g, gbytes, out);
  run_mode<6>(g, gbytes, out); run_mode<7>(g, gbytes, out); run_mode<8>(g, gbytes, out);
  run_sweep<0>(out); run_sweep<1>(out); run_sweep<2>(out); run_sweep<3>(out);
  run_sweep<4>(out); run_sweep<5>(out); run_sweep<6>(out); run_sweep<7>(out);
  run_sweep<8>(out); run_sweep<9>(out); run_sweep<10>(out); run_sweep<11>(out);
  run_sweep<12>(out); run_sweep<13>(out);
  return 0;
}
