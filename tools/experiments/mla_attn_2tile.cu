// EXPERIMENT (not built; a copy of csrc/mla_attn.cu with the two-query-tile kernel
// `mla_attn2_kernel` added and selected by default, BD_ATTN_TILES=1 for the original).
// Round 2 result: parity-green on tests/test_mla_attn_gpu.py (14/14), but no faster than
// the one-tile kernel at cfg5 size (993-997 vs 951-1003 TFLOP/s, interleaved runs; cuDNN
// SDPA 1368-1488 on the same box).  ncu: tensor pipe 44 % active, long-scoreboard stalls
// (the softmax's tcgen05.ld waits) 50 % of samples.  See profiles/r02_attention_study.md.
// Needs tmem_st_32x32b_x16 in ptx_sm100.cuh (kept there).
// mla_attn.cu — causal prefill attention for the BD-rewritten DeepSeek-V2 MLA block on
// sm_100a tcgen05 tensor cores (BD ⊕ FlashAttention).
//
//   O[t, h] = softmax_s( (Q_nope[t,h]·K'_nope[s,h] + Q_pe[t,h]·k_pe[s]) * scale ) V'[s,h]
//
// (ref: the block is ref attention.py:298-307 / :143-154 — `_attend` after the BD
// projections — restated for MLA; the paper names FlashAttention integration as the
// next step, ref PAPER.md:494.)  The kernel consumes the BD projection's outputs in the
// layouts it writes them, with no concatenation or broadcast:
//   * K'_nope and V' head-major [H][L][128] (the BD kernel's out_layout="head");
//   * the decoupled RoPE key k_pe [L][64] SHARED by all heads — read once per tile from
//     its own tensor instead of being copied into every head's key (the dense path's
//     `k_buf[..., 128:] = rope(k_pe)` broadcast, 67 MB at 32k tokens, is gone);
//   * Q = [Q_nope | Q_pe] token-major [L][H][192] (the q projection's output with RoPE
//     applied to its pe columns in place).
// so S = Q K^T is two accumulating groups of MMAs (K = 128 from K'_nope, K = 64 from k_pe).
//
// One persistent CTA per SM; work items (head, 128-query tile) in longest-first order.
// Warp roles (192 threads):
//   warp 0     TMA producer: Q tile (3 x 16 KB), per KV tile K'_nope + k_pe (48 KB) and
//              V' (32 KB) through 2-stage rings.
//   warp 1     TMEM allocator + MMA issuer.  S_j = Q K_j^T (M=128, N=128, 12 x K16) into
//              one of three TMEM S buffers; O += P_j V_j (8 x K16) with P_j read from
//              TMEM (the softmax wrote it over S_j as packed 16-bit) and V_j an MN-major
//              smem operand.  S_{j+2} is issued right after PV_j, so the tensor core
//              computes the next scores while the softmax works.
//   warps 2-5  softmax + epilogue, one query row per thread (TMEM lane): scores from TMEM,
//              causal / length mask, running max with LAZY rescaling (O and l are
//              rescaled only when the max grows by more than 2^8, so most tiles never
//              touch O), p = exp2(s·c − m) in FP32, l += p, P packed to 16 bit into TMEM;
//              after the last tile O / l is stored straight to global memory (each
//              thread's row is 256 contiguous bytes).
// TMEM: S buffers at columns [0, 384), O at [384, 512).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kv_proj_internal.h"
#include "ptx_sm100.cuh"
#include "tc_common.cuh"

namespace bdk {
namespace attn {

using tc::pack2;

constexpr int BQ = 128, BKV = 128;
constexpr int DN = 128, DR = 64, DV = 128;
constexpr int THREADS = 192;
constexpr uint32_t KBLK = 128 * 64 * 2;           // 128 rows x 64 16-bit cols (SW128): 16 KB
constexpr uint32_t Q_BYTES = 3 * KBLK;            // [nope 0:64 | nope 64:128 | pe]
constexpr uint32_t K_BYTES = 3 * KBLK;            // [K'nope 0:64 | 64:128 | k_pe]
constexpr uint32_t V_BYTES = 2 * KBLK;            // two 64-column MN-major panels
constexpr int KV_STAGES = 2;
constexpr int S_BUFS = 3;
constexpr uint32_t O_COL = S_BUFS * 128;           // TMEM column of O
constexpr size_t SMEM_BYTES = 1024 + Q_BYTES + KV_STAGES * (K_BYTES + V_BYTES) + 256;
static_assert(SMEM_BYTES <= 232448, "smem");
constexpr float RESCALE_LOG2 = 8.0f;               // lazy-rescale threshold (2^8)

struct AttnParams {
  CUtensorMap map_q;     // {192, H, L} box {64, 1, 128}
  CUtensorMap map_k;     // K'_nope {128, L, H} box {64, 128, 1}
  CUtensorMap map_kpe;   // k_pe {64, L} box {64, 128}
  CUtensorMap map_v;     // V' {128, L, H} box {64, 128, 1}
  void* out;             // O (t, h, c) at out + t * ldo_tok + h * ldo_head + c
  int64_t ldo_tok, ldo_head;
  int32_t L, H, n_qt, causal, total_items;
  float scale_log2;      // softmax scale * log2(e)
};

template <bool kBF16>
__device__ __forceinline__ uint32_t pack_p(float a, float b) {
  return pack2<kBF16>(a, b);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// item w -> (head, query tile), longest (latest) query tiles first
__device__ __forceinline__ void item_of(const AttnParams& p, int w, int& h, int& qi) {
  qi = p.n_qt - 1 - w / p.H;
  h = w % p.H;
}

template <bool kBF16>
__global__ void __launch_bounds__(THREADS, 1) mla_attn_kernel(const __grid_constant__ AttnParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;
  uint8_t* sV = sK + KV_STAGES * K_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KV_STAGES * V_BYTES);
  uint64_t* q_full = bars;                 // 1
  uint64_t* q_empty = q_full + 1;          // 1 (MMA commit after the item's last S)
  uint64_t* k_full = q_empty + 1;          // KV_STAGES
  uint64_t* k_empty = k_full + KV_STAGES;
  uint64_t* v_full = k_empty + KV_STAGES;
  uint64_t* v_empty = v_full + KV_STAGES;
  uint64_t* s_full = v_empty + KV_STAGES;  // S_BUFS (MMA commit)
  uint64_t* s_free = s_full + S_BUFS;      // S_BUFS (MMA commit after the PV reading P)
  uint64_t* p_full = s_free + S_BUFS;      // S_BUFS (4 softmax warps)
  uint64_t* pv_done = p_full + S_BUFS;     // 1 (MMA commit after every PV)
  uint64_t* o_free = pv_done + 1;          // 1 (4 epilogue warps, after reading O)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < S_BUFS; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 1);
      mbar_init(&p_full[b], 4);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_free, 4);
    fence_mbar_init();
    tma_prefetch_desc(&prm.map_q);
    tma_prefetch_desc(&prm.map_k);
    tma_prefetch_desc(&prm.map_kpe);
    tma_prefetch_desc(&prm.map_v);
  }
  if (warp == 1) {
    tmem_alloc<1>(tmem_slot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  const int G = static_cast<int>(gridDim.x);
  const int nkt_all = (prm.L + BKV - 1) / BKV;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    griddep_wait();
    const uint64_t pol_q = policy_evict_first();
    const uint64_t pol_kv = policy_evict_last();  // K/V tiles are re-read by later queries
    uint32_t kv_it = 0, item_it = 0;
    for (int w = static_cast<int>(blockIdx.x); w < prm.total_items; w += G, ++item_it) {
      int h, qi;
      item_of(prm, w, h, qi);
      const int n_kv = prm.causal ? qi + 1 : nkt_all;
      mbar_wait(q_empty, (item_it & 1u) ^ 1u);
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, Q_BYTES);
        for (int b = 0; b < 3; ++b)
          tma_load_3d(sQ + b * KBLK, &prm.map_q, 64 * b, h, qi * BQ, q_full, pol_q);
      }
      __syncwarp();
      for (int j = 0; j < n_kv; ++j, ++kv_it) {
        const uint32_t st = kv_it % KV_STAGES, ph = ((kv_it / KV_STAGES) & 1u) ^ 1u;
        mbar_wait(&k_empty[st], ph);
        if (elect_one()) {
          uint8_t* dk = sK + st * K_BYTES;
          mbar_arrive_expect_tx(&k_full[st], K_BYTES);
          tma_load_3d(dk, &prm.map_k, 0, j * BKV, h, &k_full[st], pol_kv);
          tma_load_3d(dk + KBLK, &prm.map_k, 64, j * BKV, h, &k_full[st], pol_kv);
          tma_load_2d(dk + 2 * KBLK, &prm.map_kpe, 0, j * BKV, &k_full[st], pol_kv);
        }
        __syncwarp();
        mbar_wait(&v_empty[st], ph);
        if (elect_one()) {
          uint8_t* dv = sV + st * V_BYTES;
          mbar_arrive_expect_tx(&v_full[st], V_BYTES);
          tma_load_3d(dv, &prm.map_v, 0, j * BKV, h, &v_full[st], pol_kv);
          tma_load_3d(dv + KBLK, &prm.map_v, 64, j * BKV, h, &v_full[st], pol_kv);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_f16(kBF16, BQ, BKV, /*a_mn=*/false, /*b_mn=*/false);
    constexpr uint32_t idesc_o = make_idesc_f16(kBF16, BQ, DV, /*a_mn=*/false, /*b_mn=*/true);
    uint32_t kv_it_s = 0, kv_it_v = 0;  // K tiles consumed by S, V tiles consumed by PV
    uint32_t s_it = 0, pv_it = 0, item_it = 0;
    const uint32_t q0 = smem_u32(sQ);
    auto issue_s = [&](uint32_t sb) {
      // S[sb] = Q K^T: 8 K16-steps over K'_nope (2 x 64), 4 over q_pe . k_pe
      const uint32_t st = kv_it_s % KV_STAGES;
      mbar_wait(&k_full[st], (kv_it_s / KV_STAGES) & 1u);
      mbar_wait(&s_free[sb], ((s_it / S_BUFS) & 1u) ^ 1u);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t k0 = smem_u32(sK + st * K_BYTES);
#pragma unroll
        for (int ks = 0; ks < 12; ++ks) {
          const uint32_t off = (ks >> 2) * KBLK + (ks & 3) * 32;
          tc_mma_f16(tmem_base + sb * 128, make_smem_desc(q0 + off, 16, 1024),
                     make_smem_desc(k0 + off, 16, 1024), idesc_s, ks != 0 ? 1u : 0u);
        }
        tc_commit(&s_full[sb]);
        tc_commit(&k_empty[st]);
      }
      __syncwarp();
      ++kv_it_s;
      ++s_it;
    };
    for (int w = static_cast<int>(blockIdx.x); w < prm.total_items; w += G, ++item_it) {
      int h, qi;
      item_of(prm, w, h, qi);
      const int n_kv = prm.causal ? qi + 1 : nkt_all;
      mbar_wait(q_full, item_it & 1u);
      const uint32_t s_base = s_it;
      issue_s(s_base % S_BUFS);
      if (n_kv > 1) issue_s((s_base + 1) % S_BUFS);
      if (n_kv <= 2 && elect_one()) tc_commit(q_empty);  // every S of the item issued
      __syncwarp();
      for (int j = 0; j < n_kv; ++j) {
        const uint32_t sb = (s_base + j) % S_BUFS;
        mbar_wait(&p_full[sb], ((s_base + j) / S_BUFS) & 1u);
        const uint32_t vst = kv_it_v % KV_STAGES;
        mbar_wait(&v_full[vst], (kv_it_v / KV_STAGES) & 1u);
        if (j == 0) mbar_wait(o_free, (item_it & 1u) ^ 1u);  // previous item's O read out
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v0 = smem_u32(sV + vst * V_BYTES);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma_f16_ts(tmem_base + O_COL, tmem_base + sb * 128 + ks * 8,
                          make_smem_desc(v0 + ks * (16 * 128), KBLK, 1024), idesc_o,
                          (j | ks) != 0 ? 1u : 0u);
          tc_commit(&v_empty[vst]);
          tc_commit(&s_free[sb]);
          tc_commit(pv_done);
        }
        __syncwarp();
        ++kv_it_v;
        ++pv_it;
        if (j + 2 < n_kv) {
          issue_s((s_base + j + 2) % S_BUFS);
          if (j + 3 == n_kv && elect_one()) tc_commit(q_empty);
          __syncwarp();
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax + epilogue
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32u) << 16;
    uint32_t s_it = 0, pv_it = 0;
    const float c2 = prm.scale_log2;
    for (int w = static_cast<int>(blockIdx.x); w < prm.total_items; w += G) {
      int h, qi;
      item_of(prm, w, h, qi);
      const int n_kv = prm.causal ? qi + 1 : nkt_all;
      const int r_local = static_cast<int>(quad * 32 + lane);
      const int row = qi * BQ + r_local;  // query (token) index
      float m = -INFINITY;                // running max, in log2 units of scale*s
      float l = 0.f;
      for (int j = 0; j < n_kv; ++j, ++s_it) {
        const uint32_t sb = s_it % S_BUFS;
        mbar_wait(&s_full[sb], (s_it / S_BUFS) & 1u);
        tc_fence_after();
        uint32_t sr[128];
        const uint32_t ta = tmem_base + lane_base + sb * 128;
        tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld_32x32b_x32(ta + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
        tmem_ld_32x32b_x32(ta + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
        tmem_ld_wait();
        // mask: causal (key > query) on the diagonal tile, and keys past L
        int valid = prm.L - j * BKV;
        if (prm.causal && j == qi) valid = min(valid, r_local + 1);
        float mx = -INFINITY;
        if (valid >= BKV) {
#pragma unroll
          for (int c = 0; c < 128; ++c) mx = fmaxf(mx, __uint_as_float(sr[c]));
        } else {
#pragma unroll
          for (int c = 0; c < 128; ++c) {
            if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
            mx = fmaxf(mx, __uint_as_float(sr[c]));
          }
        }
        const float m_tile = mx * c2;
        if (m_tile > m + RESCALE_LOG2) {
          // lazy rescale: the reference max moves (always on the first tile)
          if (j > 0) {
            const float alpha = ex2(m - m_tile);
            l *= alpha;
            // O row *= alpha: the previous PV must have landed (PV_j waits for our P_j)
            mbar_wait(pv_done, (pv_it - 1) & 1u);
            tc_fence_after();
            const uint32_t to = tmem_base + lane_base + O_COL;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(to + cc * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st_32x32b_x32(to + cc * 32, o);
            }
            tmem_st_wait();
          }
          m = m_tile;
        }
        // p = exp2(s c2 - m), l += p, P packed to 16 bit over S's first 64 columns
        uint32_t pk[64];
        float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
        for (int c = 0; c < 128; c += 2) {
          const float p0 = ex2(fmaf(__uint_as_float(sr[c]), c2, -m));
          const float p1 = ex2(fmaf(__uint_as_float(sr[c + 1]), c2, -m));
          ls0 += p0;
          ls1 += p1;
          pk[c >> 1] = pack_p<kBF16>(p0, p1);
        }
        l += ls0 + ls1;
        tmem_st_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
        tmem_st_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        ++pv_it;  // PV_j will be the pv_it-th PV issued
        // Observe every pv_done phase (PV_{j-1}: long complete by now, so this costs a
        // single probe).  The lazy rescale above waits only when the max moved; without
        // this wait most phases would complete unobserved (correct — a waiter can never
        // fall two phases behind — but flagged by compute-sanitizer's synccheck).
        if (j > 0) mbar_wait(pv_done, (pv_it - 2) & 1u);
      }
      // epilogue: O / l, straight to global (this thread's row is 256 contiguous bytes)
      mbar_wait(pv_done, (pv_it - 1) & 1u);
      tc_fence_after();
      const float inv = 1.0f / l;
      const bool live = row < prm.L;
      uint16_t* dst = static_cast<uint16_t*>(prm.out) +
                      static_cast<int64_t>(live ? row : 0) * prm.ldo_tok +
                      static_cast<int64_t>(h) * prm.ldo_head;
      const uint32_t to = tmem_base + lane_base + O_COL;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(to + cc * 32, o);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 v;
            v.x = pack2<kBF16>(__uint_as_float(o[8 * g + 0]) * inv, __uint_as_float(o[8 * g + 1]) * inv);
            v.y = pack2<kBF16>(__uint_as_float(o[8 * g + 2]) * inv, __uint_as_float(o[8 * g + 3]) * inv);
            v.z = pack2<kBF16>(__uint_as_float(o[8 * g + 4]) * inv, __uint_as_float(o[8 * g + 5]) * inv);
            v.w = pack2<kBF16>(__uint_as_float(o[8 * g + 6]) * inv, __uint_as_float(o[8 * g + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + cc * 32 + g * 8) = v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

// ---------------------------------------------------------------------------------
// mla_attn2_kernel: the same attention with TWO 128-row query tiles per work item (A =
// query tile 2 qp, B = 2 qp + 1) sharing every K/V tile, two softmax warpgroups (warps
// 2-5 rows of A, warps 6-9 rows of B) and the MMA issuer ping-ponging between them:
//   S_A(0) S_B(0) | PV_A(0) S_A(1) | PV_B(0) S_B(1) | PV_A(1) S_A(2) | ...
// so the tensor core computes one tile's scores / PV while the other tile's softmax runs,
// and each K/V tile (loaded once for 256 query rows — half the K/V bytes per FLOP of the
// one-tile kernel) has two tiles' worth of time to arrive.  TMEM: S_A, S_B, O_A, O_B
// (128 columns each); P is written over its S as packed 16-bit.  S_X(j+1) is issued after
// PV_X(j) (in-order tensor pipe), so the commit that publishes S_X(j+1) also guarantees
// PV_X(j) finished — the lazy O rescale needs no other wait.  Shared memory: Q_A, Q_B
// (96 KB), a two-stage K ring (96 KB) and one V stage (32 KB).
constexpr int THREADS2 = 64 + 256;
constexpr size_t SMEM2_BYTES = 1024 + 2 * Q_BYTES + 2 * K_BYTES + V_BYTES + 256;
static_assert(SMEM2_BYTES <= 232448, "smem (two-tile kernel)");

// item w -> (head, query-tile pair), longest pairs first
__device__ __forceinline__ void item2_of(const AttnParams& p, int w, int& h, int& qp) {
  const int n_qp = (p.n_qt + 1) / 2;
  qp = n_qp - 1 - w / p.H;
  h = w % p.H;
}

template <bool kBF16>
__global__ void __launch_bounds__(THREADS2, 1) mla_attn2_kernel(const __grid_constant__ AttnParams prm) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                    // [A | B], Q_BYTES each
  uint8_t* sK = sQ + 2 * Q_BYTES;        // 2 stages
  uint8_t* sV = sK + 2 * K_BYTES;        // 1 stage
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + V_BYTES);
  uint64_t* q_full = bars;
  uint64_t* q_empty = q_full + 1;
  uint64_t* k_full = q_empty + 1;   // [2]
  uint64_t* k_empty = k_full + 2;   // [2]
  uint64_t* v_full = k_empty + 2;
  uint64_t* v_empty = v_full + 1;
  uint64_t* s_full = v_empty + 1;   // [2]: A, B
  uint64_t* p_full = s_full + 2;    // [2]
  uint64_t* o_full = p_full + 2;    // [2]
  uint64_t* o_free = o_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 4);
      mbar_init(&o_full[s], 1);
      mbar_init(&o_free[s], 4);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    fence_mbar_init();
    tma_prefetch_desc(&prm.map_q);
    tma_prefetch_desc(&prm.map_k);
    tma_prefetch_desc(&prm.map_kpe);
    tma_prefetch_desc(&prm.map_v);
  }
  if (warp == 1) {
    tmem_alloc<1>(tmem_slot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  const int G = static_cast<int>(gridDim.x);
  const int nkt_all = (prm.L + BKV - 1) / BKV;
  const int n_items = ((prm.n_qt + 1) / 2) * prm.H;
  // tiles of query tile X of pair qp (0 when the tile lies past L)
  auto n_tiles = [&](int qp, int x) {
    const int qt = 2 * qp + x;
    if (qt >= prm.n_qt) return 0;
    return prm.causal ? qt + 1 : nkt_all;
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    griddep_wait();
    const uint64_t pol_q = policy_evict_first();
    const uint64_t pol_kv = policy_evict_last();
    uint32_t kv_it = 0, item_it = 0;
    for (int w = static_cast<int>(blockIdx.x); w < n_items; w += G, ++item_it) {
      int h, qp;
      item2_of(prm, w, h, qp);
      const int jmax = max(n_tiles(qp, 0), n_tiles(qp, 1));
      auto prefetch_kv = [&](int jj) {
        if (jj >= jmax) return;
        const int t = jj * BKV;
        asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                         reinterpret_cast<uint64_t>(&prm.map_k)), "r"(0), "r"(t), "r"(h) : "memory");
        asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                         reinterpret_cast<uint64_t>(&prm.map_k)), "r"(64), "r"(t), "r"(h) : "memory");
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&prm.map_kpe)), "r"(0), "r"(t) : "memory");
        asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                         reinterpret_cast<uint64_t>(&prm.map_v)), "r"(0), "r"(t), "r"(h) : "memory");
        asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                         reinterpret_cast<uint64_t>(&prm.map_v)), "r"(64), "r"(t), "r"(h) : "memory");
      };
      const int nq = n_tiles(qp, 1) > 0 ? 2 : 1;  // query tile B may lie past L
      mbar_wait(q_empty, (item_it & 1u) ^ 1u);
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, nq * Q_BYTES);
        for (int x = 0; x < nq; ++x)
          for (int b = 0; b < 3; ++b)
            tma_load_3d(sQ + x * Q_BYTES + b * KBLK, &prm.map_q, 64 * b, h, (2 * qp + x) * BQ, q_full,
                        pol_q);
        for (int jj = 0; jj < 4; ++jj) prefetch_kv(jj);
      }
      __syncwarp();
      for (int j = 0; j < jmax; ++j, ++kv_it) {
        if (elect_one()) prefetch_kv(j + 4);
        __syncwarp();
        const uint32_t st = kv_it & 1u, ph = ((kv_it >> 1) & 1u) ^ 1u;
        mbar_wait(&k_empty[st], ph);
        if (elect_one()) {
          uint8_t* dk = sK + st * K_BYTES;
          mbar_arrive_expect_tx(&k_full[st], K_BYTES);
          tma_load_3d(dk, &prm.map_k, 0, j * BKV, h, &k_full[st], pol_kv);
          tma_load_3d(dk + KBLK, &prm.map_k, 64, j * BKV, h, &k_full[st], pol_kv);
          tma_load_2d(dk + 2 * KBLK, &prm.map_kpe, 0, j * BKV, &k_full[st], pol_kv);
        }
        __syncwarp();
        mbar_wait(v_empty, (kv_it & 1u) ^ 1u);
        if (elect_one()) {
          mbar_arrive_expect_tx(v_full, V_BYTES);
          tma_load_3d(sV, &prm.map_v, 0, j * BKV, h, v_full, pol_kv);
          tma_load_3d(sV + KBLK, &prm.map_v, 64, j * BKV, h, v_full, pol_kv);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = make_idesc_f16(kBF16, BQ, BKV, /*a_mn=*/false, /*b_mn=*/false);
    constexpr uint32_t idesc_o = make_idesc_f16(kBF16, BQ, DV, /*a_mn=*/false, /*b_mn=*/true);
    uint32_t kv_it = 0, item_it = 0;
    uint32_t s_cnt[2] = {0, 0}, p_cnt[2] = {0, 0}, x_items[2] = {0, 0};
    auto issue_s = [&](int x, uint32_t st) {
      if (elect_one()) {
        const uint32_t q0 = smem_u32(sQ + x * Q_BYTES);
        const uint32_t k0 = smem_u32(sK + st * K_BYTES);
#pragma unroll
        for (int ks = 0; ks < 12; ++ks) {
          const uint32_t off = (ks >> 2) * KBLK + (ks & 3) * 32;
          tc_mma_f16(tmem_base + x * 128, make_smem_desc(q0 + off, 16, 1024),
                     make_smem_desc(k0 + off, 16, 1024), idesc_s, ks != 0 ? 1u : 0u);
        }
        tc_commit(&s_full[x]);
      }
      __syncwarp();
      ++s_cnt[x];
    };
    auto issue_pv = [&](int x, int j) {
      mbar_wait(&p_full[x], p_cnt[x] & 1u);
      ++p_cnt[x];
      if (j == 0) mbar_wait(&o_free[x], (x_items[x] & 1u) ^ 1u);  // previous item's O read out
      tc_fence_after();
      if (elect_one()) {
        const uint32_t v0 = smem_u32(sV);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tc_mma_f16_ts(tmem_base + 256 + x * 128, tmem_base + x * 128 + ks * 8,
                        make_smem_desc(v0 + ks * (16 * 128), KBLK, 1024), idesc_o,
                        (j | ks) != 0 ? 1u : 0u);
      }
      __syncwarp();
    };
    for (int w = static_cast<int>(blockIdx.x); w < n_items; w += G, ++item_it) {
      int h, qp;
      item2_of(prm, w, h, qp);
      const int nA = n_tiles(qp, 0), nB = n_tiles(qp, 1);
      const int jmax = max(nA, nB);
      mbar_wait(q_full, item_it & 1u);
      // tile 0 scores for both query tiles
      {
        const uint32_t st = kv_it & 1u;
        mbar_wait(&k_full[st], (kv_it >> 1) & 1u);
        tc_fence_after();
        if (nA > 0) issue_s(0, st);
        if (nB > 0) issue_s(1, st);
        if (elect_one()) {
          tc_commit(&k_empty[st]);
          if (jmax == 1) tc_commit(q_empty);
        }
        __syncwarp();
      }
      for (int j = 0; j < jmax; ++j, ++kv_it) {
        const uint32_t stn = (kv_it + 1) & 1u;     // stage of tile j + 1
        const bool next = j + 1 < jmax;
        bool k_next_ready = false;
        mbar_wait(v_full, kv_it & 1u);
        for (int x = 0; x < 2; ++x) {
          const int n = x == 0 ? nA : nB;
          if (j >= n) continue;
          issue_pv(x, j);
          if (j + 1 < n) {
            if (!k_next_ready) {
              mbar_wait(&k_full[stn], ((kv_it + 1) >> 1) & 1u);
              tc_fence_after();
              k_next_ready = true;
            }
            issue_s(x, stn);
          } else if (elect_one()) {
            tc_commit(&o_full[x]);  // this query tile's last PV: O is final
          }
          __syncwarp();
        }
        if (elect_one()) {
          tc_commit(v_empty);  // both PVs of tile j issued
          if (next) {
            tc_commit(&k_empty[stn]);  // both S of tile j + 1 issued
            if (j + 2 == jmax) tc_commit(q_empty);  // the item's last S issued
          }
        }
        __syncwarp();
      }
      if (nA > 0) ++x_items[0];
      if (nB > 0) ++x_items[1];
    }
  } else {
    // ---------------------------------------------------------------- softmax + epilogue
    const uint32_t x = (warp - 2) >> 2;  // query tile A (0) or B (1)
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32u) << 16;
    const uint32_t ts = tmem_base + lane_base + x * 128;        // S_x / P_x
    const uint32_t to = tmem_base + lane_base + 256 + x * 128;  // O_x
    uint32_t s_it = 0, items = 0;
    const float c2 = prm.scale_log2;
    for (int w = static_cast<int>(blockIdx.x); w < n_items; w += G) {
      int h, qp;
      item2_of(prm, w, h, qp);
      const int n = n_tiles(qp, static_cast<int>(x));
      if (n == 0) continue;
      const int qt = 2 * qp + static_cast<int>(x);
      const int r_local = static_cast<int>(quad * 32 + lane);
      const int row = qt * BQ + r_local;
      float m = -INFINITY;
      float l = 0.f;
      for (int j = 0; j < n; ++j, ++s_it) {
        mbar_wait(&s_full[x], s_it & 1u);
        tc_fence_after();
        int valid = prm.L - j * BKV;
        if (prm.causal && j == qt) valid = min(valid, r_local + 1);
        const bool full = valid >= BKV;
        // pass 1: the row max, 32 columns at a time (the two-tile kernel runs 3 warps on
        // some SM sub-partitions, so a thread gets <= 168 registers: S is not held whole)
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ts + 32 * cc, v);
          tmem_ld_wait();
          if (full) {
#pragma unroll
            for (int c = 0; c < 32; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(v[c]));
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (32 * cc + c < valid) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(v[c]));
          }
        }
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float m_tile = mx * c2;
        if (m_tile > m + RESCALE_LOG2) {
          if (j > 0) {
            // PV_x(j-1) completed before S_x(j) was published (in-order tensor pipe)
            const float alpha = ex2(m - m_tile);
            l *= alpha;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(to + cc * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st_32x32b_x32(to + cc * 32, o);
            }
            tmem_st_wait();
          }
          m = m_tile;
        }
        // pass 2: p = exp2(s c2 - m), l += p, P packed to 16 bit: chunk cc (S columns
        // [32 cc, 32 cc + 32)) becomes P columns [16 cc, 16 cc + 16), which lie in S
        // columns already read by this pass
        float ls[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) ls[e] = 0.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ts + 32 * cc, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            float p0 = ex2(fmaf(__uint_as_float(v[c]), c2, -m));
            float p1 = ex2(fmaf(__uint_as_float(v[c + 1]), c2, -m));
            if (!full) {
              p0 = 32 * cc + c < valid ? p0 : 0.f;
              p1 = 32 * cc + c + 1 < valid ? p1 : 0.f;
            }
            ls[(c >> 1) & 7] += p0 + p1;
            pk[c >> 1] = pack_p<kBF16>(p0, p1);
          }
          tmem_st_32x32b_x16(ts + 16 * cc, pk);
        }
        l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[x]);
      }
      // epilogue: O / l straight to global (this thread's row: 256 contiguous bytes)
      mbar_wait(&o_full[x], items & 1u);
      tc_fence_after();
      const float inv = 1.0f / l;
      const bool live = row < prm.L;
      uint16_t* dst = static_cast<uint16_t*>(prm.out) +
                      static_cast<int64_t>(live ? row : 0) * prm.ldo_tok +
                      static_cast<int64_t>(h) * prm.ldo_head;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(to + cc * 32, o);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint4 v;
            v.x = pack2<kBF16>(__uint_as_float(o[8 * g + 0]) * inv, __uint_as_float(o[8 * g + 1]) * inv);
            v.y = pack2<kBF16>(__uint_as_float(o[8 * g + 2]) * inv, __uint_as_float(o[8 * g + 3]) * inv);
            v.z = pack2<kBF16>(__uint_as_float(o[8 * g + 4]) * inv, __uint_as_float(o[8 * g + 5]) * inv);
            v.w = pack2<kBF16>(__uint_as_float(o[8 * g + 6]) * inv, __uint_as_float(o[8 * g + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + cc * 32 + g * 8) = v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[x]);
      ++items;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}

bool encode(CUtensorMap* map, const void* base, bool bf16, int rank, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box, std::string* err) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (fn == nullptr) {
    *err = "cuTensorMapEncodeTiled unavailable from the driver";
    return false;
  }
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], e[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
  }
  for (int i = 0; i + 1 < rank; ++i) s[i] = strides_bytes[i];
  const CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                        rank, const_cast<void*>(base), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (attention, rank %d) failed (CUresult %d)",
             rank, static_cast<int>(r));
    *err = buf;
    return false;
  }
  return true;
}

}  // namespace attn

int launch_mla_attention(const MlaAttnArgs& a, cudaStream_t stream) {
  using namespace attn;
  const bool bf16 = a.dtype == BD_BF16;
  AttnParams prm{};
  std::string err;
  {
    const uint64_t dq[3] = {static_cast<uint64_t>(DN + DR), static_cast<uint64_t>(a.n_heads),
                            static_cast<uint64_t>(a.L)};
    const uint64_t sq[2] = {static_cast<uint64_t>(a.ldq_head) * 2, static_cast<uint64_t>(a.ldq_tok) * 2};
    const uint32_t bq[3] = {64, 1, BQ};
    const uint64_t dk[3] = {DN, static_cast<uint64_t>(a.L), static_cast<uint64_t>(a.n_heads)};
    const uint64_t sk[2] = {static_cast<uint64_t>(a.ldk) * 2, static_cast<uint64_t>(a.k_head_stride) * 2};
    const uint32_t bk[3] = {64, BKV, 1};
    const uint64_t dp[2] = {DR, static_cast<uint64_t>(a.L)};
    const uint64_t sp[1] = {static_cast<uint64_t>(a.ldkpe) * 2};
    const uint32_t bp[2] = {64, BKV};
    const uint64_t dv[3] = {DV, static_cast<uint64_t>(a.L), static_cast<uint64_t>(a.n_heads)};
    const uint64_t sv[2] = {static_cast<uint64_t>(a.ldv) * 2, static_cast<uint64_t>(a.v_head_stride) * 2};
    if (!encode(&prm.map_q, a.q, bf16, 3, dq, sq, bq, &err) ||
        !encode(&prm.map_k, a.k_nope, bf16, 3, dk, sk, bk, &err) ||
        !encode(&prm.map_kpe, a.k_pe, bf16, 2, dp, sp, bp, &err) ||
        !encode(&prm.map_v, a.v, bf16, 3, dv, sv, bk, &err)) {
      set_error(err);
      return BD_ERR_CUDA;
    }
  }
  prm.out = a.out;
  prm.ldo_tok = a.ldo_tok;
  prm.ldo_head = a.ldo_head;
  prm.L = static_cast<int32_t>(a.L);
  prm.H = static_cast<int32_t>(a.n_heads);
  prm.n_qt = static_cast<int32_t>((a.L + BQ - 1) / BQ);
  prm.causal = a.causal ? 1 : 0;
  prm.total_items = prm.n_qt * prm.H;
  prm.scale_log2 = a.scale * 1.4426950408889634f;
  using KernFn = void (*)(AttnParams);
  // BD_ATTN_TILES=1: the one-query-tile kernel; default: two query tiles per item
  static const bool two = [] {
    const char* e = getenv("BD_ATTN_TILES");
    return !(e != nullptr && atoi(e) == 1);
  }();
  const KernFn kern = two ? (bf16 ? mla_attn2_kernel<true> : mla_attn2_kernel<false>)
                          : (bf16 ? mla_attn_kernel<true> : mla_attn_kernel<false>);
  const size_t smem = two ? SMEM2_BYTES : SMEM_BYTES;
  const int vk = two ? 1 : 0;
  static std::atomic<bool> attr_done[kMaxDevices][2][2] = {};
  static std::mutex attr_mu;
  const int dvs = device_slot();
  if (!attr_done[dvs][bf16][vk].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(attr_mu);
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute (attention): ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_done[dvs][bf16][vk].store(true, std::memory_order_release);
  }
  const int items = two ? ((prm.n_qt + 1) / 2) * prm.H : prm.total_items;
  const int grid = items < sm_count() ? items : sm_count();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(two ? THREADS2 : THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm);
  note_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("mla_attn launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

}  // namespace bdk
