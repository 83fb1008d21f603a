// tc_common.cuh — shared by the tcgen05 kernels (kv_proj_tc.cu: persistent CTA-pair
// kernel and small-L kernel; kv_proj_decode.cu: the decode kernel): launch parameters,
// 16-bit pack/unpack and the epilogue's mixed-precision add, tensor-map encoding.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "kv_proj_internal.h"
#include "ptx_sm100.cuh"

namespace bdk {
namespace tc {

struct TcProblem {
  CUtensorMap map_a;    // x + mul_base, dims {K, L},   box {64, 128}
  CUtensorMap map_b;    // c,            dims {N, K},   box {64, BKB}
  CUtensorMap map_rep;  // x + rep_base, dims {d_h, L}, box {64, 128}   (rep_fast only)
  CUtensorMap map_out;  // out: token-major dims {N, L}, box {64, 32}; head-major dims
                        // {d_h, L, n_heads}, box {64, 32, 1} (clips per head); SW128
  const void* x;
  int64_t ldx;
  int32_t L, N, K, d_h, rep_base;
  int32_t tiles_n, num_kb, num_kbb, tile_start;  // num_kbb: B k-blocks (BKB deep)
  int32_t tiles_m;      // persistent kernel: pair row-blocks (the mirror schedule's inner loop)
  int32_t has_rep;      // 0: plain GEMM (no repeated-slice add)
  int32_t rep_fast;     // d_h in {64, 128}: rep tile staged in smem by TMA
  int32_t head_major;   // output layout [n_heads][L][d_h]
  int32_t out_d_h;      // head width of the head-major output
  void* out;            // output base and row stride (the small-L kernel stores directly)
  int64_t ldo;
  const float* rep_gamma;  // kNorm: RMSNorm weight of the repeated slice (d_h floats)
  float norm_eps;          // kNorm: RMSNorm epsilon
  int32_t norm_d;          // kNorm: columns of x's row (K + d_h) the norm averages over
};

struct TcParams {
  TcProblem p[BD_MAX_GROUP];
  // fused all-gather: per problem, the head-major 3-D map {d_h, L, world * n_heads} of
  // every rank's gathered buffer (peer memory over NVLink); world == 0 otherwise
  // [count][world] in device memory (kept out of the kernel parameters: 4 KB more of
  // them costs ~2 us of host time per launch); null when world == 0
  const CUtensorMap* peer_maps;
  int32_t world;
  int32_t head0[BD_MAX_GROUP];
  int32_t count;
  int32_t total_tiles;  // tiles of (BM * CG) rows x BN columns
  int32_t a_kb_bytes;   // small-L / decode kernels: bytes of one A k-block (rows rounded
                        // to 8 x 128 B)
  int32_t strided;      // tiles dealt round-robin to the pairs (streaming-A problems)
  int32_t norm;         // fused RMSNorm (kNorm variant)
  int* flag;            // non-finite flag (kCheck instantiation only)
  int32_t dk_kps;         // decode kernel: k-blocks of 64 per CTA (problem p splits its
                          // contraction over ceil(num_kb / dk_kps) CTAs of a cluster)
  int32_t dk_a_bytes;     // decode kernel: A region, B region and receive buffer bytes
  int32_t dk_b_bytes;
  int32_t dk_recv_bytes;
  int32_t small_rblocks;  // small-L kernel: row blocks of BM * CGS rows (grid = cols x rows)
  int32_t bn;             // persistent kernel: tile width (256, or 128 for short launches)
  int32_t swap;           // persistent kernel: mirror schedule (coefficient tile resident)
};

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

// (a + lo(h), b + hi(h)) in FP32 with the 16-bit halves of h widened exactly: the
// mixed-precision add.f32.f16 / add.f32.bf16 (one FHADD per element on sm_100).
template <bool kBF16>
__device__ __forceinline__ float2 add_f32_x16x2(float a, float b, uint32_t h) {
  float r0, r1;
  if constexpr (kBF16)
    asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %2; add.rn.f32.bf16 %0, lo, %3;"
        " add.rn.f32.bf16 %1, hi, %4; }"
        : "=f"(r0), "=f"(r1) : "r"(h), "f"(a), "f"(b));
  else
    asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %2; add.rn.f32.f16 %0, lo, %3;"
        " add.rn.f32.f16 %1, hi, %4; }"
        : "=f"(r0), "=f"(r1) : "r"(h), "f"(a), "f"(b));
  return make_float2(r0, r1);
}

// Packed FP32 add (FADD2 on sm_100): two lanes per instruction, each rounded once.
__device__ __forceinline__ float2 add_f32x2(float2 a, float2 b) {
  unsigned long long av = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long bv = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(av), "l"(bv));
  return *reinterpret_cast<float2*>(&r);
}

// Running packed max of |h| that propagates NaN (one HMNMX2 per two outputs).
template <bool kBF16>
__device__ __forceinline__ uint32_t max_abs2_nan(uint32_t acc, uint32_t w) {
  if constexpr (kBF16) {
    __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&acc);
    __nv_bfloat162 b = __habs2(*reinterpret_cast<__nv_bfloat162*>(&w));
    __nv_bfloat162 m = __hmax2_nan(a, b);
    return *reinterpret_cast<uint32_t*>(&m);
  } else {
    __half2 a = *reinterpret_cast<__half2*>(&acc);
    __half2 b = __habs2(*reinterpret_cast<__half2*>(&w));
    __half2 m = __hmax2_nan(a, b);
    return *reinterpret_cast<uint32_t*>(&m);
  }
}

// Either 16-bit lane of a packed max is Inf or NaN (exponent bits all ones).
template <bool kBF16>
__device__ __forceinline__ bool nonfinite2(uint32_t w) {
  const uint32_t e = kBF16 ? 0x7F80u : 0x7C00u;
  return ((w & e) == e) || (((w >> 16) & e) == e);
}

// Tensor maps of 16-bit row-major matrices (host side; defined in kv_proj_tc.cu).
// 2-D: [rows x cols], row stride ld elements, box {box_cols, box_rows}.
bool encode_2d(CUtensorMap* map, const void* base, bool bf16, uint64_t cols, uint64_t rows,
               uint64_t ld, uint32_t box_cols, uint32_t box_rows, std::string* err,
               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);
// 3-D: [planes x rows x cols] (row stride ld, plane stride ps), box {box_cols, box_rows, 1}.
bool encode_3d(CUtensorMap* map, const void* base, bool bf16, uint64_t cols, uint64_t rows,
               uint64_t planes, uint64_t ld, uint64_t ps, uint32_t box_cols, uint32_t box_rows,
               std::string* err);

}  // namespace tc
}  // namespace bdk
