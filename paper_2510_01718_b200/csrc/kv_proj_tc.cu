// kv_proj_tc.cu — FP16/BF16 BD K/V projection on sm_100a tensor cores.
//
//   out[i, h*d_h + j] = sum_k x[i, mul_base + k] * c[k, h*d_h + j]  +  x[i, rep_base + j]
//
// (ref: pkg/src/bdattn/attention.py:249-270 computes the same thing on the CPU.)
//
// Structure (one persistent CTA per SM, warp-specialised):
//   warp 0      TMA producer: A = x[:, mul_base : mul_base+K] as a K-major operand
//               (tensor map based at column mul_base, so the basis slice S is never
//               read by the mainloop and K tails are zero-filled by TMA), and
//               B = c in the reference's own (d-d_h) x N row-major layout, loaded as an
//               MN-major operand (no transpose anywhere).  128B swizzle on both.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16),
//               accumulating in FP32 in TMEM; tcgen05.commit releases smem stages and
//               signals the epilogue.
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns per warp), + x[i, rep_base
//               + (col mod d_h)] in FP32 (the identity-block gather-add, after the full
//               K-sum like the reference), one rounding to FP16/BF16, 16-byte stores.
//               Non-finite outputs raise a device flag (ref _wrap check, tensor.py:112).
//   TMEM holds two 128x256 FP32 accumulators (all 512 columns) so the epilogue of
//   tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include "kv_proj_internal.h"
#include "ptx_sm100.cuh"

namespace bdk {
namespace tc {

constexpr int BM = 128;                       // UMMA M (rows of x per tile)
constexpr int BN = 256;                       // UMMA N (output columns per tile)
constexpr int BK = 64;                        // k-block: one 128-byte swizzle row of A
constexpr int UK = 16;                        // UMMA K for kind::f16
constexpr int STAGES = 4;                     // smem ring depth
constexpr int EPI_WARPS = 4;                  // 128 epilogue threads = 128 TMEM lanes
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr uint32_t A_BYTES = BM * BK * 2;     // 16 KiB
constexpr uint32_t B_CHUNK = 64 * BK * 2;     // one 64-column MN-major swizzle panel, 8 KiB
constexpr uint32_t B_BYTES = BN * BK * 2;     // 32 KiB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr uint32_t TMEM_COLS = 2 * BN;        // double-buffered accumulator
constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;

struct TcProblem {
  CUtensorMap map_a;  // x + mul_base, dims {K, L}, box {64, 128}
  CUtensorMap map_b;  // c,            dims {N, K}, box {64, 64}
  const void* x;
  void* out;
  int64_t ldx, ldo;
  int32_t L, N, K, d_h, rep_base;
  int32_t tiles_n, num_kb, tile_start;
};

struct TcParams {
  TcProblem p[BD_MAX_GROUP];
  int32_t count;
  int32_t total_tiles;
  int* flag;
};

__device__ __forceinline__ void decode_tile(const TcParams& prm, int t, int& pi, int& m0,
                                            int& n0) {
  pi = 0;
  while (pi + 1 < prm.count && t >= prm.p[pi + 1].tile_start) ++pi;
  const int local = t - prm.p[pi].tile_start;
  n0 = (local % prm.p[pi].tiles_n) * BN;
  m0 = (local / prm.p[pi].tiles_n) * BM;
}

template <bool kBF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (kBF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

template <bool kBF16>
__device__ __forceinline__ float2 unpack2(uint32_t w) {
  if constexpr (kBF16) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w);
    return __bfloat1622float2(h);
  } else {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    return __half22float2(h);
  }
}

// True if either 16-bit half of w is Inf/NaN (exponent all ones).
template <bool kBF16>
__device__ __forceinline__ bool nonfinite2(uint32_t w) {
  constexpr uint32_t E = kBF16 ? 0x7F80u : 0x7C00u;
  return ((w & E) == E) || (((w >> 16) & E) == E);
}

template <bool kBF16>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    kv_proj_tc_kernel(const __grid_constant__ TcParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < prm.count; ++i) {
      tma_prefetch_desc(&prm.p[i].map_a);
      tma_prefetch_desc(&prm.p[i].map_b);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();  // x and c are re-read; out streams past
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < prm.total_tiles; t += gridDim.x) {
        int pi, m0, n0;
        decode_tile(prm, t, pi, m0, n0);
        const TcProblem& P = prm.p[pi];
        for (int kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sA + stage * A_BYTES, &P.map_a, kb * BK, m0, &full[stage], pol);
#pragma unroll
          for (int q = 0; q < BN / 64; ++q) {
            tma_load_2d(sB + stage * B_BYTES + q * B_CHUNK, &P.map_b, n0 + 64 * q, kb * BK,
                        &full[stage], pol);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_f16(kBF16, BM, BN, /*a_mn=*/false, /*b_mn=*/true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < prm.total_tiles; t += gridDim.x, ++it) {
        int pi, m0, n0;
        decode_tile(prm, t, pi, m0, n0);
        const TcProblem& P = prm.p[pi];
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / UK; ++ks) {
            // A: K-major SW128, rows 128 B apart, 8-row groups 1024 B apart; a 16-wide
            //    k step is +32 B inside the swizzle row.
            const uint64_t adesc = make_smem_desc(a0 + ks * (UK * 2), 16, 1024);
            // B: MN-major SW128, 64-column panels B_CHUNK apart (LBO), 8-k-row groups
            //    1024 B apart (SBO); a 16-deep k step is two 8-row groups = 2048 B.
            const uint64_t bdesc = make_smem_desc(b0 + ks * (UK * 128), B_CHUNK, 1024);
            tc_mma_f16(d_tmem, adesc, bdesc, idesc, (kb | ks) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row_in_tile = static_cast<int>(quad * 32 + lane);
    bool bad = false;
    int it = 0;
    for (int t = blockIdx.x; t < prm.total_tiles; t += gridDim.x, ++it) {
      int pi, m0, n0;
      decode_tile(prm, t, pi, m0, n0);
      const TcProblem& P = prm.p[pi];
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t row = static_cast<int64_t>(m0) + row_in_tile;
      const bool row_ok = row < P.L;
      const uint16_t* xrow =
          static_cast<const uint16_t*>(P.x) + (row_ok ? row : 0) * P.ldx + P.rep_base;
      uint16_t* orow = static_cast<uint16_t*>(P.out) + (row_ok ? row : 0) * P.ldo;
      const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * BN;
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + ch * 32, r);
        tmem_ld_wait();
        if (row_ok) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int col = n0 + ch * 32 + g * 8;
            if (col < P.N) {
              const int jj = col % P.d_h;  // 8 columns never straddle a head (d_h % 8 == 0)
              const uint4 xv = __ldg(reinterpret_cast<const uint4*>(xrow + jj));
              const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 xr = unpack2<kBF16>(xw[e]);
                const float v0 = __fadd_rn(__uint_as_float(r[g * 8 + 2 * e]), xr.x);
                const float v1 = __fadd_rn(__uint_as_float(r[g * 8 + 2 * e + 1]), xr.y);
                o[e] = pack2<kBF16>(v0, v1);
                bad |= nonfinite2<kBF16>(o[e]);
              }
              *reinterpret_cast<uint4*>(orow + col) = make_uint4(o[0], o[1], o[2], o[3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (prm.flag != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(prm.flag, 1);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  });
  return fn;
}

// Row-major [rows x cols] 16-bit matrix, row stride ld elements, box {box_cols, box_rows}.
bool encode_2d(CUtensorMap* map, const void* base, bool bf16, uint64_t cols, uint64_t rows,
               uint64_t ld, uint32_t box_cols, uint32_t box_rows, std::string* err) {
  auto fn = encode_fn();
  if (fn == nullptr) {
    *err = "cuTensorMapEncodeTiled unavailable from the driver";
    return false;
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (CUresult %d)", static_cast<int>(r));
    *err = buf;
    return false;
  }
  return true;
}

}  // namespace tc

int launch_tc(const bd_kv_problem* probs, int count, int dtype, int* flag, cudaStream_t stream) {
  using namespace tc;
  const bool bf16 = dtype == BD_BF16;
  TcParams prm{};
  prm.count = count;
  prm.flag = flag;
  int total = 0;
  for (int i = 0; i < count; ++i) {
    const bd_kv_problem& q = probs[i];
    TcProblem& P = prm.p[i];
    const int64_t K = q.d - q.d_h;
    const int64_t N = q.n_heads * q.d_h;
    std::string err;
    const auto* xb = static_cast<const uint16_t*>(q.x) + q.mul_base;
    if (!encode_2d(&P.map_a, xb, bf16, K, q.L, q.ldx, BK, BM, &err) ||
        !encode_2d(&P.map_b, q.c, bf16, N, K, q.ldc, 64, BK, &err)) {
      set_error(err);
      return BD_ERR_CUDA;
    }
    P.x = q.x;
    P.out = q.out;
    P.ldx = q.ldx;
    P.ldo = q.ldo;
    P.L = static_cast<int32_t>(q.L);
    P.N = static_cast<int32_t>(N);
    P.K = static_cast<int32_t>(K);
    P.d_h = static_cast<int32_t>(q.d_h);
    P.rep_base = static_cast<int32_t>(q.rep_base);
    P.tiles_n = static_cast<int32_t>((N + BN - 1) / BN);
    P.num_kb = static_cast<int32_t>((K + BK - 1) / BK);
    P.tile_start = total;
    total += P.tiles_n * static_cast<int32_t>((q.L + BM - 1) / BM);
  }
  prm.total_tiles = total;
  if (total == 0) return BD_OK;

  auto kern = bf16 ? kv_proj_tc_kernel<true> : kv_proj_tc_kernel<false>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[bf16 ? 1 : 0]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SMEM_BYTES));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_set[bf16 ? 1 : 0] = true;
  }
  const int grid = total < sm_count() ? total : sm_count();
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(prm);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("kv_proj_tc launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

}  // namespace bdk
