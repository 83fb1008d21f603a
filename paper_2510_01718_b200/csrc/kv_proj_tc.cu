// kv_proj_tc.cu — FP16/BF16 BD K/V projection on sm_100a tensor cores.
//
//   out[i, h*d_h + j] = sum_k x[i, mul_base + k] * c[k, h*d_h + j]  +  x[i, rep_base + j]
//
// (ref: pkg/src/bdattn/attention.py:249-270 computes the same thing on the CPU.)
// With rep_base < 0 the same kernel is a plain GEMM (the BD low-rank layer, linear.py).
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
#include <cstdlib>
#include <mutex>
#include <string>

#include "kv_proj_internal.h"
#include "ptx_sm100.cuh"

namespace bdk {
namespace tc {

constexpr int BM = 128;                       // rows of x per CTA per tile (TMEM lanes)
constexpr int BN = 256;                       // UMMA N (output columns per tile)
constexpr int BK = 64;                        // k-block: one 128-byte swizzle row of A
constexpr int UK = 16;                        // UMMA K for kind::f16
constexpr int EPI_WARPS = 8;                  // 2 per SMSP; warps w, w+4 share a TMEM lane quadrant
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr uint32_t A_BYTES = BM * BK * 2;     // 16 KiB
constexpr uint32_t B_PANEL = 64 * BK * 2;     // one 64-column MN-major swizzle panel, 8 KiB
constexpr uint32_t REP_BOX = 64 * BM * 2;     // one 64-column x 128-row rep box, 16 KiB
constexpr uint32_t REP_BYTES = 2 * REP_BOX;   // d_h <= 128 -> at most two boxes
constexpr uint32_t STG_BYTES = 32 * 32 * 2;   // output staging box: 32 rows x 32 cols (SW64)
constexpr uint32_t TMEM_COLS = 2 * BN;        // double-buffered accumulator

// Per cta_group configuration.  CG = 2: a CTA pair computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 — each CTA stages its own 128 rows of A and HALF of the B
// tile (128 columns), so B bytes per CTA halve and the ring can be one stage deeper.
template <int CG>
struct Cfg {
  static constexpr int B_PANELS = (BN / 64) / CG;               // 4 (CG=1) / 2 (CG=2)
  static constexpr uint32_t B_BYTES = B_PANELS * B_PANEL;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;    // 48 / 32 KiB
  static constexpr int STAGES = CG == 1 ? 3 : 4;
  static constexpr int STG_BUFS = CG == 1 ? 1 : 2;               // per-warp staging buffers
  static constexpr size_t SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 2 * REP_BYTES +
                                       EPI_WARPS * STG_BUFS * STG_BYTES + 256;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

struct TcProblem {
  CUtensorMap map_a;    // x + mul_base, dims {K, L},   box {64, 128}
  CUtensorMap map_b;    // c,            dims {N, K},   box {64, 64}
  CUtensorMap map_rep;  // x + rep_base, dims {d_h, L}, box {64, 128}   (rep_fast only)
  CUtensorMap map_out;  // out,          dims {N, L},   box {32, 32}, SW64
  const void* x;
  int64_t ldx;
  int32_t L, N, K, d_h, rep_base;
  int32_t tiles_n, num_kb, tile_start;
  int32_t has_rep;      // 0: plain GEMM (no repeated-slice add)
  int32_t rep_fast;     // d_h in {64, 128}: rep tile staged in smem by TMA
};

struct TcParams {
  TcProblem p[BD_MAX_GROUP];
  int32_t count;
  int32_t total_tiles;  // tiles of (BM * CG) rows x BN columns
  int* flag;
  int32_t debug;  // profiling knob (env BD_TC_DEBUG): 1 no stores, 2 no epilogue math, 4 no LDTM
};

template <int CG>
__device__ __forceinline__ void decode_tile(const TcParams& prm, int t, int& pi, int& m0,
                                            int& n0) {
  pi = 0;
  while (pi + 1 < prm.count && t >= prm.p[pi + 1].tile_start) ++pi;
  const int local = t - prm.p[pi].tile_start;
  n0 = (local % prm.p[pi].tiles_n) * BN;
  m0 = (local / prm.p[pi].tiles_n) * (BM * CG);
}

// Tiles sharing (problem, m-block) share the rep tile x[m0:m0+128, rep_base:+d_h].
__device__ __forceinline__ int rep_key(int pi, int m0) { return (pi << 24) | (m0 / BM); }

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

// kCheck: compute the non-finite flag (only instantiated work when the caller asked).
template <bool kBF16, int CG, bool kCheck>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    kv_proj_tc_kernel(const __grid_constant__ TcParams prm) {
  using C = Cfg<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * A_BYTES;
  uint8_t* sRep = sB + C::STAGES * C::B_BYTES;      // 2 slots x REP_BYTES
  uint8_t* sStg = sRep + 2 * REP_BYTES;             // EPI_WARPS x STG_BUFS x STG_BYTES
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + EPI_WARPS * C::STG_BUFS * STG_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;  // 0 = pair leader
  const int unit = CG == 2 ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int units = CG == 2 ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // Contiguous tile range per CTA (pair): consecutive tiles share the x row-block (A and
  // the rep slice stay L2/smem-hot); the split is balanced to within one tile.
  const int t_begin = static_cast<int>(static_cast<int64_t>(unit) * prm.total_tiles / units);
  const int t_end = static_cast<int>(static_cast<int64_t>(unit + 1) * prm.total_tiles / units);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < prm.count; ++i) {
      tma_prefetch_desc(&prm.p[i].map_a);
      tma_prefetch_desc(&prm.p[i].map_b);
      tma_prefetch_desc(&prm.p[i].map_out);
      if (prm.p[i].rep_fast) tma_prefetch_desc(&prm.p[i].map_rep);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);    // armed by the leader's producer with the pair's bytes
      mbar_init(&empty[s], 1);   // one (multicast) tcgen05.commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG);  // one arrival per CTA's epilogue (leader's copy)
      mbar_init(&rfull[a], 1);
      mbar_init(&rempty[a], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc<CG>(tmem_slot, TMEM_COLS);
    tmem_relinquish<CG>();
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();  // x and c are re-read; out streams past
      int stage = 0;
      uint32_t phase = 0;
      int rslot = 1;
      uint32_t rphase = 0;  // bit s = parity of rep slot s
      int prev_key = -1;
      for (int t = t_begin; t < t_end; ++t) {
        int pi, m0, n0;
        decode_tile<CG>(prm, t, pi, m0, n0);
        const TcProblem& P = prm.p[pi];
        const int my_m0 = m0 + static_cast<int>(rank) * BM;
        const int my_n0 = n0 + static_cast<int>(rank) * (BN / CG);
        const int key = rep_key(pi, my_m0);
        if (P.rep_fast && key != prev_key) {
          // New (problem, m-block): stage its rep tile in the other slot.
          rslot ^= 1;
          mbar_wait(&rempty[rslot], ((rphase >> rslot) & 1u) ^ 1u);
          rphase ^= 1u << rslot;
          const int nbox = P.d_h / 64;
          mbar_arrive_expect_tx(&rfull[rslot], nbox * REP_BOX);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(sRep + rslot * REP_BYTES + b * REP_BOX, &P.map_rep, 64 * b, my_m0,
                        &rfull[rslot], pol);
        }
        prev_key = key;
        for (int kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(a_dst, &P.map_a, kb * BK, my_m0, &full[stage], pol);
#pragma unroll
            for (int q = 0; q < C::B_PANELS; ++q)
              tma_load_2d(b_dst + q * B_PANEL, &P.map_b, my_n0 + 64 * q, kb * BK, &full[stage],
                          pol);
          } else {
            // Both CTAs' bytes complete on the LEADER's full barrier, which the leader
            // arms with the pair's total.  The peer does not arrive: a cluster-scope
            // release arrive would stall it on its own in-flight TMA loads, and the
            // barrier cannot complete before the leader's arrival anyway.
            const uint32_t bar = mapa_shared(smem_u32(&full[stage]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], CG * C::STAGE_BYTES);
            tma_load_2d_pair(a_dst, &P.map_a, kb * BK, my_m0, bar, pol);
#pragma unroll
            for (int q = 0; q < C::B_PANELS; ++q)
              tma_load_2d_pair(b_dst + q * B_PANEL, &P.map_b, my_n0 + 64 * q, kb * BK, bar, pol);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    // The whole warp runs the loop (warp-uniform control flow keeps the descriptors in
    // uniform registers); one elected lane issues the tcgen05 instructions.
    if (rank == 0) {
      constexpr uint32_t idesc =
          make_idesc_f16(kBF16, BM * CG, BN, /*a_mn=*/false, /*b_mn=*/true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = t_begin; t < t_end; ++t, ++it) {
        int pi, m0, n0;
        decode_tile<CG>(prm, t, pi, m0, n0);
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
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < BK / UK; ++ks) {
              // A: K-major SW128, rows 128 B apart, 8-row groups 1024 B apart; a 16-wide
              //    k step is +32 B inside the swizzle row.
              const uint64_t adesc = make_smem_desc(a0 + ks * (UK * 2), 16, 1024);
              // B: MN-major SW128, 64-column panels B_PANEL apart (LBO), 8-k-row groups
              //    1024 B apart (SBO); a 16-deep k step is two 8-row groups = 2048 B.
              const uint64_t bdesc = make_smem_desc(b0 + ks * (UK * 128), B_PANEL, 1024);
              if constexpr (CG == 1)
                tc_mma_f16(d_tmem, adesc, bdesc, idesc, (kb | ks) != 0 ? 1u : 0u);
              else
                tc_mma_f16_pair(d_tmem, adesc, bdesc, idesc, (kb | ks) != 0 ? 1u : 0u);
            }
            if constexpr (CG == 1) tc_commit(&empty[stage]); else tc_commit_pair(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if constexpr (CG == 1) tc_commit(&tfull[acc]); else tc_commit_pair(&tfull[acc], 0x3);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // 8 warps: warp w reads TMEM lanes 32*(w%4).. (its quadrant) and columns
    // [128*h, 128*h+128) of the accumulator, h = (w-2)/4, in four 32-column sub-chunks;
    // the TMEM load of sub-chunk i+1 is in flight while sub-chunk i is processed.
    const uint32_t ew = warp - 2;
    const uint32_t quad = warp & 3;
    const uint32_t half = ew >> 2;
    const int row_w = static_cast<int>(lane);
    const int row_t = static_cast<int>(quad * 32) + row_w;
    const bool leader = (ew == 0 && lane == 0);
    const uint32_t stg0 = smem_u32(sStg + ew * C::STG_BUFS * STG_BYTES);
    const uint32_t sw64 = static_cast<uint32_t>((row_w >> 1) & 3);
    const uint32_t tempty_leader0 = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
    const uint32_t tempty_leader1 = CG == 2 ? mapa_shared(smem_u32(&tempty[1]), 0) : 0u;
    uint32_t sbuf = 0;
    uint32_t chk = 0u;  // NaN-propagating packed max |out| (16-bit) for the non-finite check
    int rslot = 1;
    uint32_t rphase = 0;  // bit s = parity of rep slot s
    int prev_key = -1;
    int it = 0;
    for (int t = t_begin; t < t_end; ++t, ++it) {
      int pi, m0, n0;
      decode_tile<CG>(prm, t, pi, m0, n0);
      const TcProblem& P = prm.p[pi];
      const int my_m0 = m0 + static_cast<int>(rank) * BM;
      const int key = rep_key(pi, my_m0);
      const bool fast = P.rep_fast != 0;
      if (fast && key != prev_key) {
        rslot ^= 1;
        mbar_wait(&rfull[rslot], (rphase >> rslot) & 1u);
        rphase ^= 1u << rslot;
      }
      prev_key = key;
      const uint8_t* rep_row = sRep + rslot * REP_BYTES + row_t * 128;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t grow = static_cast<int64_t>(my_m0) + row_t;
      const bool has_rep = P.has_rep != 0;
      const uint16_t* xrow = static_cast<const uint16_t*>(P.x) +
                             (grow < P.L ? grow : 0) * P.ldx + P.rep_base;
      const int cbase = n0 + static_cast<int>(half) * 128;
      int nsub = (P.N - cbase + 31) / 32;
      nsub = nsub < 0 ? 0 : (nsub > 4 ? 4 : nsub);
      const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * BN + half * 128;
      const int dmask = P.d_h - 1;

      auto process = [&](const uint32_t (&r)[32], int sub) {
        const int col0 = cbase + sub * 32;
        uint4 xv[4];
        if (fast) {
          const int jj0 = col0 & dmask;  // d_h in {64,128}: 32 columns never wrap a head
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int jj = jj0 + 8 * g;
            const uint32_t ch = static_cast<uint32_t>((jj & 63) >> 3);
            xv[g] = *reinterpret_cast<const uint4*>(rep_row + (jj >> 6) * REP_BOX +
                                                    ((ch ^ (row_t & 7)) << 4));
          }
        } else if (!has_rep) {
#pragma unroll
          for (int g = 0; g < 4; ++g) xv[g] = make_uint4(0, 0, 0, 0);
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int col = col0 + 8 * g;
            xv[g] = (col < P.N && grow < P.L)
                        ? __ldg(reinterpret_cast<const uint4*>(xrow + (col % P.d_h)))
                        : make_uint4(0, 0, 0, 0);
          }
        }
        const uint32_t stg = stg0 + sbuf * STG_BYTES;
        // the TMA store that last read this staging buffer must be done with it
        if (lane == 0) tma_store_wait_read<C::STG_BUFS - 1>();
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t xw[4] = {xv[g].x, xv[g].y, xv[g].z, xv[g].w};
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // + rep in FP32 (one packed FADD2 per pair), one rounding to 16 bit
            const float2 xr = unpack2<kBF16>(xw[e]);
            const float2 v = add_f32x2(make_float2(__uint_as_float(r[8 * g + 2 * e]),
                                                   __uint_as_float(r[8 * g + 2 * e + 1])), xr);
            o[e] = pack2<kBF16>(v.x, v.y);
            if constexpr (kCheck) chk = max_abs2_nan<kBF16>(chk, o[e]);
          }
          const uint32_t dst = stg + row_w * 64 + ((static_cast<uint32_t>(g) ^ sw64) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]),
                       "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(prm.debug & 1)) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&P.map_out)),
              "r"(stg), "r"(col0), "r"(my_m0 + static_cast<int>(quad) * 32)
              : "memory");
          tma_store_commit();
        }
        if constexpr (C::STG_BUFS > 1) sbuf ^= 1;
      };

      if (!(prm.debug & 4) && nsub > 0) {
        uint32_t ra[32], rb[32];
        tmem_ld_32x32b_x32(taddr, ra);
#pragma unroll
        for (int sub = 0; sub < 4; sub += 2) {
          if (sub < nsub) {
            tmem_ld_wait();
            if (sub + 1 < nsub) tmem_ld_32x32b_x32(taddr + (sub + 1) * 32, rb);
            if (!(prm.debug & 2)) process(ra, sub);
          }
          if (sub + 1 < nsub) {
            tmem_ld_wait();
            if (sub + 2 < nsub) tmem_ld_32x32b_x32(taddr + (sub + 2) * 32, ra);
            if (!(prm.debug & 2)) process(rb, sub + 1);
          }
        }
        if (prm.debug & 2) chk |= ra[0] & 1u;
      }
      tc_fence_before();
      named_bar_sync(1, 32 * EPI_WARPS);  // all epilogue threads finished with TMEM + rep
      if (leader) {
        if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
        else mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
        if (fast) {
          int npi = -1, nm0 = 0, nn0 = 0;
          if (t + 1 < t_end) decode_tile<CG>(prm, t + 1, npi, nm0, nn0);
          if (t + 1 >= t_end || rep_key(npi, nm0 + static_cast<int>(rank) * BM) != key)
            mbar_arrive(&rempty[rslot]);
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
    // the rounded 16-bit outputs: any Inf/NaN (overflowing sums round to Inf) raises the flag
    if constexpr (kCheck) {
      const bool bad = nonfinite2<kBF16>(chk);
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(prm.flag, 1);
    }
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, TMEM_COLS);
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
               uint64_t ld, uint32_t box_cols, uint32_t box_rows, std::string* err,
               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
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
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
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

int launch_tc(const Problem* probs, int count, int dtype, int* flag, cudaStream_t stream) {
  using namespace tc;
  static const int debug = [] {
    const char* e = getenv("BD_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  constexpr int cg = 2;  // CTA pairs (tcgen05 cta_group::2)
  const bool bf16 = dtype == BD_BF16;
  TcParams prm{};
  prm.count = count;
  prm.flag = flag;
  prm.debug = debug;
  int total = 0;
  for (int i = 0; i < count; ++i) {
    const Problem& q = probs[i];
    TcProblem& P = prm.p[i];
    const int64_t K = q.K;
    const int64_t N = q.N;
    std::string err;
    const bool has_rep = q.rep_base >= 0;
    const int64_t d_h = has_rep ? q.d_h : 1;
    const int64_t rep_base = has_rep ? q.rep_base : 0;
    const auto* xb = static_cast<const uint16_t*>(q.x) + q.mul_base;
    const bool rep_fast = has_rep && (d_h % 64 == 0) && d_h <= 128;
    const auto* xr = static_cast<const uint16_t*>(q.x) + rep_base;
    if (!encode_2d(&P.map_a, xb, bf16, K, q.L, q.ldx, BK, BM, &err) ||
        !encode_2d(&P.map_b, q.c, bf16, N, K, q.ldc, 64, BK, &err) ||
        !encode_2d(&P.map_out, q.out, bf16, N, q.L, q.ldo, 32, 32, &err, CU_TENSOR_MAP_SWIZZLE_64B) ||
        (rep_fast && !encode_2d(&P.map_rep, xr, bf16, d_h, q.L, q.ldx, 64, BM, &err))) {
      set_error(err);
      return BD_ERR_CUDA;
    }
    P.rep_fast = rep_fast ? 1 : 0;
    P.has_rep = has_rep ? 1 : 0;
    P.x = q.x;
    P.ldx = q.ldx;
    P.L = static_cast<int32_t>(q.L);
    P.N = static_cast<int32_t>(N);
    P.K = static_cast<int32_t>(K);
    P.d_h = static_cast<int32_t>(d_h);
    P.rep_base = static_cast<int32_t>(rep_base);
    P.tiles_n = static_cast<int32_t>((N + BN - 1) / BN);
    P.num_kb = static_cast<int32_t>((K + BK - 1) / BK);
    P.tile_start = total;
    total += P.tiles_n * static_cast<int32_t>((q.L + BM * cg - 1) / (BM * cg));
  }
  prm.total_tiles = total;
  if (total == 0) return BD_OK;

  using KernFn = void (*)(TcParams);
  const bool check = flag != nullptr;
  KernFn kern = bf16 ? (check ? kv_proj_tc_kernel<true, 2, true> : kv_proj_tc_kernel<true, 2, false>)
                     : (check ? kv_proj_tc_kernel<false, 2, true> : kv_proj_tc_kernel<false, 2, false>);
  const size_t smem = Cfg<2>::SMEM_BYTES;
  static bool attr_set[2][2] = {{false, false}, {false, false}};
  if (!attr_set[bf16 ? 1 : 0][check ? 1 : 0]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_set[bf16 ? 1 : 0][check ? 1 : 0] = true;
  }
  const int units = sm_count() / cg;
  const int grid_units = total < units ? total : units;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_units * cg);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm);
  note_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("kv_proj_tc launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

}  // namespace bdk
