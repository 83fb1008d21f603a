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
// One persistent CTA per SM; work items (head, 128-query tile) in L2-sized head groups,
// each group longest-first (item_of).
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
#include <cstdlib>
#include <cstdint>
#include <cstdio>
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
  int32_t hgroup;        // heads per scheduling group (K/V of a group stays in L2)
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

// The k-th item of CTA b (of G): rounds of G items, alternate rounds in reverse CTA order
// (items are sorted longest first, so a CTA's long and short items pair up).
__device__ __forceinline__ int zz_item(int k, int G) {
  const int b = static_cast<int>(blockIdx.x);
  return k * G + ((k & 1) ? G - 1 - b : b);
}

// item w -> (head, query tile): heads in groups of hgroup, each group's items longest
// (latest) query tile first.  The CTAs in flight then work on one or two groups, whose
// K'/V' tiles (re-read by every later query tile of the same head) stay L2-resident; with
// every head in flight at once the live K/V set exceeds L2 and is re-read from HBM.
__device__ __forceinline__ void item_of(const AttnParams& p, int w, int& h, int& qi) {
  const int per = p.hgroup * p.n_qt;
  const int grp = w / per, r = w - grp * per;
  const int rest = p.H - grp * p.hgroup;
  const int gh = rest < p.hgroup ? rest : p.hgroup;
  qi = p.n_qt - 1 - r / gh;
  h = grp * p.hgroup + r % gh;
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
    for (int zk = 0, w = zz_item(0, G); w < prm.total_items; w = zz_item(++zk, G), ++item_it) {
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
    for (int zk = 0, w = zz_item(0, G); w < prm.total_items; w = zz_item(++zk, G), ++item_it) {
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
    for (int zk = 0, w = zz_item(0, G); w < prm.total_items; w = zz_item(++zk, G)) {
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
  {
    // heads per group: the group's K'_nope + V' (2 x L x 128 x 2 bytes per head) within
    // ~48 MB of the 126 MB L2; BD_ATTN_HGROUP overrides (A/B)
    static const int env = [] {
      const char* e = getenv("BD_ATTN_HGROUP");
      return e != nullptr ? atoi(e) : 0;
    }();
    const int64_t per_head = a.L * (DN + DV) * 2;
    int64_t g = (48ll << 20) / (per_head > 0 ? per_head : 1);
    if (env > 0) g = env;
    prm.hgroup = static_cast<int32_t>(g < 1 ? 1 : (g > prm.H ? prm.H : g));
  }
  prm.scale_log2 = a.scale * 1.4426950408889634f;
  using KernFn = void (*)(AttnParams);
  const KernFn kern = bf16 ? mla_attn_kernel<true> : mla_attn_kernel<false>;
  static std::atomic<bool> attr_done[kMaxDevices][2] = {};
  static std::mutex attr_mu;
  const int dvs = device_slot();
  if (!attr_done[dvs][bf16].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(attr_mu);
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SMEM_BYTES));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute (attention): ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_done[dvs][bf16].store(true, std::memory_order_release);
  }
  const int grid = prm.total_items < sm_count() ? prm.total_items : sm_count();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
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
