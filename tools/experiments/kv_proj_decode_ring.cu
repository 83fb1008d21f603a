// kv_proj_decode_ring.cu — EXPERIMENT (not in the product library; no longer builds:
// its TcParams fields were reused by kv_proj_decode_splitk.cu): a decode-sized-L (<= 256)
// BD K/V projection kernel, measured against the shipped small-L kernel in round 2 and
// NOT better overall (wins at L = 1 / cfg2 L = 64, loses at L = 64-256
// on the paper shape).  Kept for the record of what was tried.
//
//   out[i, h*d_h + j] = sum_k x[i, mul_base + k] * c[k, h*d_h + j]  +  x[i, rep_base + j]
//
// (ref: pkg/src/bdattn/attention.py:249-270.)  At small L the work is streaming the
// coefficient matrix C once (12.6 MB for the paper's n = 128 shape, 3.1 MB for
// DeepSeek-V2-Lite's K' + V') and the step time is set by latency, not by the MMA: the
// launch, the prologue, the DRAM round trip of C and the epilogue's store drain.  This
// kernel attacks those, not the arithmetic:
//
// * One CTA per BN-column block of one problem (BN = 64 or 128; grids of <= 148 CTAs
//   for the shapes of BASELINE.json) for ALL rows of the batch (one or two 128-row
//   M tiles): C is read exactly once, x (a few hundred KB at most) is re-read from L2.
// * A and B stream through a 96 KB ring of k-block stages (K is unbounded), and the
//   footprint is sized so that TWO CTAs fit on an SM (smem <= 113 KB, <= 168 registers,
//   <= 256 TMEM columns): the NEXT launch's CTAs become resident while this launch still
//   runs (programmatic dependent launch, `griddepcontrol.launch_dependents` is the first
//   instruction), so their prologue — barrier init, TMEM allocation, descriptor
//   prefetch — is off the critical path.
// * Before `griddepcontrol.wait`, each CTA prefetches its C slice into L2
//   (`cp.async.bulk.prefetch.tensor`).  L2 is the GPU's point of coherence, so a
//   prefetch cannot observe stale data even if the previous kernel wrote C; it only
//   moves the DRAM read of the weights under the previous launch's tail.  x (the
//   activations, which the previous kernel may produce) is read only after the wait.
// * Epilogue: four warps, one TMEM lane quadrant each; the repeated slice x[i, rep_base
//   + (col mod d_h)] is fetched into registers BEFORE waiting for the MMAs; + rep with
//   one FHADD per element after the full K-sum (the reference's order: one FP32 rounding
//   of the sum, one of the add), one rounding to 16 bit, swizzled staging in the (now
//   idle) ring, TMA store (token-major 2-D or head-major 3-D map; boxes clip at L, N).
//
// Same FP32 tensor-core accumulation (k ascending in 16-deep MMA steps), FHADD and
// rounding as the persistent kernel in kv_proj_tc.cu: rows computed here are
// bit-identical to the same rows computed there (tests/test_kv_proj_gpu.py).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "../../paper_2510_01718_b200/csrc/kv_proj_internal.h"
#include "../../paper_2510_01718_b200/csrc/ptx_sm100.cuh"
#include "../../paper_2510_01718_b200/csrc/tc_common.cuh"

namespace bdk {
namespace tc {

constexpr int DC_THREADS = 192;                // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr uint32_t DC_B_PANEL = 64 * 64 * 2;   // 64 k-rows x 64 columns of C (MN-major SW128)
constexpr uint32_t DC_BOX = 32 * 64 * 2;       // output staging box: 32 rows x 64 cols
constexpr uint32_t DC_SLACK = 16 * 1024;       // the MMA reads 128 A rows; a stage holds L_pad
constexpr int DC_MAX_STAGES = 16;
constexpr uint32_t DC_RING_MAX = 208 * 1024;   // + slack + barriers <= 227 KB per CTA

template <int BN, int MT>
struct DcLayout {
  static constexpr uint32_t B_KB = (BN / 64) * DC_B_PANEL;
  static constexpr uint32_t STAGING = 4 * MT * (BN / 64) * DC_BOX;
  static constexpr uint32_t TMEM_COLS = MT * BN <= 32 ? 32 : (MT * BN <= 64 ? 64 : (MT * BN <= 128 ? 128 : 256));
};

// Ring geometry (host-chosen, in TcParams): A k-blocks hold L_pad rows (MT = 1: L rounded
// up to 8; MT = 2: 128 per tile), a stage = MT A k-blocks + one B k-block, and as many
// stages as fit the ring budget, up to every k-block at once (one load round trip).
inline size_t decode_smem_bytes(uint32_t ring_bytes) { return 1024 + ring_bytes + DC_SLACK + 512; }

#ifdef BD_DC_STAMPS
// Development builds only (tools/decode_timeline.py): %globaltimer stamps per CTA and
// launch, 4 launches of history: [seq & 3][block][event].
__device__ unsigned long long g_dc_stamps[4][512][16];
__device__ __forceinline__ void dc_stamp(int seq, int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_dc_stamps[seq & 3][blockIdx.x & 511][ev] = t;
}
#define DC_STAMP(ev) dc_stamp(prm.dbg_seq, ev)
#else
#define DC_STAMP(ev) ((void)0)
#endif

__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

template <bool kBF16, bool kCheck, int BN, int MT>
__global__ void __launch_bounds__(DC_THREADS, 2)
    kv_proj_decode_kernel(const __grid_constant__ TcParams prm) {
  using Lay = DcLayout<BN, MT>;
  // the next launch in the stream may start placing its CTAs right away: they fit
  // beside this CTA and wait in griddepcontrol.wait for this grid's completion
  griddep_launch_dependents();
  DC_STAMP(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int STAGES = prm.dc_stages;
  const uint32_t a_kb = static_cast<uint32_t>(prm.a_kb_bytes);   // one A k-block, one M tile
  const uint32_t STAGE = MT * a_kb + Lay::B_KB;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + prm.dc_ring_bytes + DC_SLACK);
  uint64_t* empty = full + DC_MAX_STAGES;
  uint64_t* done = empty + DC_MAX_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  int pi = 0;
  const int t = static_cast<int>(blockIdx.x);
  while (pi + 1 < prm.count && t >= prm.p[pi + 1].tile_start) ++pi;
  const TcProblem& P = prm.p[pi];
  const int n0 = (t - P.tile_start) * BN;
  const int num_kb = P.num_kb;

  // Start-up: the producer initialises the barriers and goes straight on to its loads
  // (bar.arrive, no wait); the TMEM allocation (warp 1) and the other warps meet it on
  // named barrier 1 — nothing but the barrier init sits before the first TMA.
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(done, 1);
      fence_mbar_init();
      tma_prefetch_desc(&P.map_a);
      tma_prefetch_desc(&P.map_b);
#ifndef DC_NO_PREFETCH
      // this CTA's C slice into L2 while the previous launch drains (see header)
      for (int kb = 0; kb < num_kb; ++kb)
#pragma unroll
        for (int q = 0; q < BN / 64; ++q) tma_prefetch_l2_2d(&P.map_b, n0 + 64 * q, kb * 64);
#endif
    }
    __syncwarp();
    asm volatile("bar.arrive 1, %0;" ::"n"(DC_THREADS) : "memory");
  } else {
    if (warp == 1) {
      tmem_alloc<1>(tmem_slot, Lay::TMEM_COLS);
      tmem_relinquish<1>();
    }
    if (warp == 2 && lane == 0) tma_prefetch_desc(&P.map_out);
    tc_fence_before();
    named_bar_sync(1, DC_THREADS);
    tc_fence_after();
  }
  const uint32_t tmem_base = warp == 0 ? 0u : *tmem_slot;
  DC_STAMP(1);

  if (warp == 0) {
    // ---- producer: k-blocks of A (all M tiles) and of this CTA's B columns
    const uint64_t pol_a = policy_evict_last();   // x: re-read by every CTA
    const uint64_t pol_b = policy_evict_first();  // C: read once
#ifdef DC_EARLY_B
    // timing experiment only: B of the first ring's worth of k-blocks before the wait
    // (unsafe if the previous kernel wrote C)
    const int early = num_kb < STAGES ? num_kb : STAGES;
    if (elect_one()) {
      for (int kb = 0; kb < early; ++kb) {
        uint8_t* st = ring + kb * STAGE;
        mbar_arrive_expect_tx(&full[kb], STAGE);
#pragma unroll
        for (int q = 0; q < BN / 64; ++q)
          tma_load_2d(st + MT * a_kb + q * DC_B_PANEL, &P.map_b, n0 + 64 * q, kb * 64,
                      &full[kb], pol_b);
      }
    }
#else
    const int early = 0;
#endif
    griddep_wait();
    DC_STAMP(2);
    if (elect_one()) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* st = ring + s * STAGE;
        if (kb >= early) mbar_arrive_expect_tx(&full[s], STAGE);
#pragma unroll
        for (int m = 0; m < MT; ++m)
          tma_load_2d(st + m * a_kb, &P.map_a, kb * 64, m * 128, &full[s], pol_a);
        if (kb >= early) {
#pragma unroll
          for (int q = 0; q < BN / 64; ++q)
            tma_load_2d(st + MT * a_kb + q * DC_B_PANEL, &P.map_b, n0 + 64 * q, kb * 64,
                        &full[s], pol_b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA: D[m] (128 x BN, FP32 in TMEM) += A[m] (128 x 16) * B (16 x BN), k ascending
    constexpr uint32_t idesc = make_idesc_f16(kBF16, 128, BN, /*a_mn=*/false, /*b_mn=*/true);
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc_fence_after();
      if (kb == 0) DC_STAMP(3);
      if (kb < 8) DC_STAMP(8 + kb);
      if (elect_one()) {
        const uint32_t st = smem_u32(ring + s * STAGE);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t bdesc = make_smem_desc(st + MT * a_kb + ks * (16 * 128), DC_B_PANEL, 1024);
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const uint64_t adesc = make_smem_desc(st + m * a_kb + ks * 32, 16, 1024);
            tc_mma_f16(tmem_base + m * BN, adesc, bdesc, idesc, (kb | ks) != 0 ? 1u : 0u);
          }
        }
        tc_commit(&empty[s]);
        if (kb + 1 == num_kb) tc_commit(done);
      }
      __syncwarp();
    }
    DC_STAMP(4);
  } else {
    // ---- epilogue: warp w owns TMEM lanes 32 (w % 4) .. +32 = rows m*128 + 32 (w % 4) + lane
    const uint32_t quad = warp & 3;
    const uint32_t ew = warp - 2;
    uint32_t chk = 0u;
    griddep_wait();  // x (the repeated slice) may be the previous kernel's output
    const bool has_rep = P.has_rep != 0;
#pragma unroll 1
    for (int m = 0; m < MT; ++m) {
      const int row = m * 128 + static_cast<int>(quad * 32 + lane);
      const bool live = row < P.L;
      const uint16_t* xrow = static_cast<const uint16_t*>(P.x) +
                             static_cast<int64_t>(live ? row : 0) * P.ldx + P.rep_base;
      // this row's repeated-slice values for the block's BN columns, fetched before the
      // MMA wait (m = 0) so their L2 latency hides behind the C stream
      uint4 xr[BN / 8];
#pragma unroll
      for (int j = 0; j < BN / 8; ++j) {
        const int col = n0 + 8 * j;
        xr[j] = (live && has_rep && col < P.N)
                    ? __ldg(reinterpret_cast<const uint4*>(xrow + (col % P.d_h)))
                    : make_uint4(0, 0, 0, 0);
      }
      if (m == 0) {
        mbar_wait(done, 0);
        tc_fence_after();
        DC_STAMP(5);
      }
      if (m * 128 + static_cast<int>(quad) * 32 >= P.L) continue;  // warp entirely past L
      // staging: the ring is idle once every MMA completed; per warp and M tile BN/64
      // boxes of 32 x 64 (SW128)
      const uint32_t stg = smem_u32(ring) + ((m * 4 + ew) * (BN / 64)) * DC_BOX;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + m * BN + c * 32, r);
        tmem_ld_wait();
        const int bx = c >> 1, part = c & 1;
        const uint32_t buf = stg + static_cast<uint32_t>(bx) * DC_BOX;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint4 xv = xr[c * 4 + g];
          const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 v = add_f32_x16x2<kBF16>(__uint_as_float(r[8 * g + 2 * e]),
                                                 __uint_as_float(r[8 * g + 2 * e + 1]), xw[e]);
            o[e] = pack2<kBF16>(v.x, v.y);
            if constexpr (kCheck) {
              if (live && n0 + c * 32 + 8 * g < P.N) chk = max_abs2_nan<kBF16>(chk, o[e]);
            }
          }
          const uint32_t dst = buf + lane * 128 + (((4 * part + g) ^ (lane & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]), "r"(o[1]),
                       "r"(o[2]), "r"(o[3])
                       : "memory");
        }
        if (part == 1) {
          fence_proxy_async_smem();
          __syncwarp();
          const int bcol = n0 + bx * 64;
          if (lane == 0 && bcol < P.N) {
            const int brow = m * 128 + static_cast<int>(quad) * 32;
            if (P.head_major)
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(&P.map_out)),
                  "r"(buf), "r"(bcol % P.out_d_h), "r"(brow), "r"(bcol / P.out_d_h)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(&P.map_out)),
                  "r"(buf), "r"(bcol), "r"(brow)
                  : "memory");
            tma_store_commit();
          }
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
    DC_STAMP(6);
    if constexpr (kCheck) {
      if (__any_sync(0xffffffffu, nonfinite2<kBF16>(chk)) && lane == 0) atomicExch(prm.flag, 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, Lay::TMEM_COLS);
  }
  DC_STAMP(7);
}

}  // namespace tc

// Problems the decode kernel serves: one x of at most 256 rows, no fused all-gather, no
// fused norm.  BD_DECODE=0 routes them to the older small-L / persistent kernels.
bool decode_eligible(const Problem* probs, int count) {
  static const bool off = [] {
    const char* e = getenv("BD_DECODE");
    return e != nullptr && atoi(e) == 0;
  }();
  if (off) return false;
  for (int i = 0; i < count; ++i)
    if (probs[i].L > 256 || probs[i].world > 0 || probs[i].rep_gamma != nullptr) return false;
  return true;
}

int launch_decode(const Problem* probs, int count, bool bf16, int* flag, cudaStream_t stream) {
  using namespace tc;
  int64_t cols = 0, max_l = 1;
  for (int i = 0; i < count; ++i) {
    cols += probs[i].N;
    max_l = probs[i].L > max_l ? probs[i].L : max_l;
  }
  const int mt = max_l > 128 ? 2 : 1;
  // 64-column blocks while they fit one wave (more CTAs pulling C); else 128
  static const int bn_env = [] {  // BD_DC_BN=64|128 forces the column block (development A/B)
    const char* e = getenv("BD_DC_BN");
    return e != nullptr ? atoi(e) : 0;
  }();
  const int bn = bn_env == 64 || bn_env == 128 ? bn_env
                                               : ((cols + 63) / 64 <= sm_count() ? 64 : 128);
  int max_kb = 1;
  for (int i = 0; i < count; ++i) {
    const int kb = static_cast<int>((probs[i].K + 63) / 64);
    max_kb = kb > max_kb ? kb : max_kb;
  }
  const uint32_t a_rows = mt == 1 ? static_cast<uint32_t>((max_l + 7) / 8 * 8) : 128u;
  const uint32_t a_kb = a_rows * 128;
  const uint32_t stage = mt * a_kb + (bn / 64) * DC_B_PANEL;
  static const uint32_t ring_cap = [] {  // BD_DC_RING_KB: ring budget (development A/B)
    const char* e = getenv("BD_DC_RING_KB");
    return (e != nullptr ? static_cast<uint32_t>(atoi(e)) : 200u) * 1024u;
  }();
  int stages = static_cast<int>((ring_cap < DC_RING_MAX ? ring_cap : DC_RING_MAX) / stage);
  stages = stages < max_kb ? stages : max_kb;
  stages = stages < DC_MAX_STAGES ? stages : DC_MAX_STAGES;
  stages = stages > 2 ? stages : 2;
  const uint32_t staging = 4u * mt * (bn / 64) * DC_BOX;
  uint32_t ring_bytes = stages * stage;
  ring_bytes = ring_bytes > staging ? ring_bytes : staging;
  TcParams prm{};
  prm.count = count;
  prm.flag = flag;
  prm.a_kb_bytes = static_cast<int32_t>(a_kb);
  prm.dc_stages = stages;
  prm.dc_ring_bytes = static_cast<int32_t>(ring_bytes);
  static std::atomic<int> seq{0};
  prm.dbg_seq = seq.fetch_add(1, std::memory_order_relaxed);
  int total = 0;
  for (int i = 0; i < count; ++i) {
    const Problem& q = probs[i];
    TcProblem& P = prm.p[i];
    std::string err;
    const bool has_rep = q.rep_base >= 0;
    const auto* xb = static_cast<const uint16_t*>(q.x) + q.mul_base;
    if (!encode_2d(&P.map_a, xb, bf16, q.K, q.L, q.ldx, 64, a_rows, &err) ||
        !encode_2d(&P.map_b, q.c, bf16, q.N, q.K, q.ldc, 64, 64, &err) ||
        !(q.out_layout == BD_OUT_HEAD_MAJOR
              ? encode_3d(&P.map_out, q.out, bf16, q.d_h, q.L, q.N / q.d_h, q.ldo, q.L * q.ldo,
                          64, 32, &err)
              : encode_2d(&P.map_out, q.out, bf16, q.N, q.L, q.ldo, 64, 32, &err))) {
      set_error(err);
      return BD_ERR_CUDA;
    }
    P.x = q.x;
    P.ldx = q.ldx;
    P.L = static_cast<int32_t>(q.L);
    P.N = static_cast<int32_t>(q.N);
    P.K = static_cast<int32_t>(q.K);
    P.d_h = static_cast<int32_t>(has_rep ? q.d_h : 1);
    P.rep_base = static_cast<int32_t>(has_rep ? q.rep_base : 0);
    P.has_rep = has_rep ? 1 : 0;
    P.head_major = q.out_layout == BD_OUT_HEAD_MAJOR ? 1 : 0;
    P.out_d_h = static_cast<int32_t>(q.d_h);
    P.out = q.out;
    P.ldo = q.ldo;
    P.num_kb = static_cast<int32_t>((q.K + 63) / 64);
    P.tiles_n = static_cast<int32_t>((q.N + bn - 1) / bn);
    P.tile_start = total;
    total += P.tiles_n;
  }
  prm.total_tiles = total;
  if (total == 0) return BD_OK;
  using KernFn = void (*)(TcParams);
  // [bf16][check][bn 64 / 128][mt 1 / 2]
  static const KernFn kerns[2][2][2][2] = {
      {{{kv_proj_decode_kernel<false, false, 64, 1>, kv_proj_decode_kernel<false, false, 64, 2>},
        {kv_proj_decode_kernel<false, false, 128, 1>, kv_proj_decode_kernel<false, false, 128, 2>}},
       {{kv_proj_decode_kernel<false, true, 64, 1>, kv_proj_decode_kernel<false, true, 64, 2>},
        {kv_proj_decode_kernel<false, true, 128, 1>, kv_proj_decode_kernel<false, true, 128, 2>}}},
      {{{kv_proj_decode_kernel<true, false, 64, 1>, kv_proj_decode_kernel<true, false, 64, 2>},
        {kv_proj_decode_kernel<true, false, 128, 1>, kv_proj_decode_kernel<true, false, 128, 2>}},
       {{kv_proj_decode_kernel<true, true, 64, 1>, kv_proj_decode_kernel<true, true, 64, 2>},
        {kv_proj_decode_kernel<true, true, 128, 1>, kv_proj_decode_kernel<true, true, 128, 2>}}}};
  const int vb = bf16 ? 1 : 0, vc = flag != nullptr ? 1 : 0, vn = bn == 128 ? 1 : 0, vm = mt - 1;
  const KernFn kern = kerns[vb][vc][vn][vm];
  const size_t smem = decode_smem_bytes(ring_bytes);
  static std::atomic<bool> attr_done[kMaxDevices][2][2][2][2] = {};
  static std::mutex attr_mu;
  const int dv = device_slot();
  if (!attr_done[dv][vb][vc][vn][vm].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(attr_mu);
    // a cap, not a reservation: each launch asks for its own ring's footprint
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(decode_smem_bytes(DC_RING_MAX)));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_done[dv][vb][vc][vn][vm].store(true, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(total);
  cfg.blockDim = dim3(DC_THREADS);
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
    set_error(std::string("kv_proj_decode launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

}  // namespace bdk

#ifdef BD_DC_STAMPS
extern "C" int bd_debug_decode_stamps(void* dst, size_t bytes) {
  return static_cast<int>(cudaMemcpyFromSymbol(dst, bdk::tc::g_dc_stamps, bytes));
}
#endif
