// kv_proj_tc.cu — FP16/BF16 BD K/V projection on sm_100a tensor cores.
//
//   out[i, h*d_h + j] = sum_k x[i, mul_base + k] * c[k, h*d_h + j]  +  x[i, rep_base + j]
//
// (ref: pkg/src/bdattn/attention.py:249-270 computes the same thing on the CPU.)
// With rep_base < 0 the same kernel is a plain GEMM (the BD low-rank layer, linear.py).
//
// One persistent CTA PAIR (cluster of 2, tcgen05 cta_group::2) per two SMs computes
// 256 x 256 output tiles; each CTA owns 128 rows (its TMEM lanes) and stages half of
// the B tile.  Warp roles per CTA:
//   warp 0      TMA producer.  A = x[:, mul_base : mul_base+K] as a K-major operand
//               (tensor map based at column mul_base: the basis slice S is never read by
//               the mainloop; K tails zero-filled by TMA).  B = c in the reference's own
//               (d-d_h) x N row-major layout as an MN-major operand (no transpose).
//   warp 1      TMEM allocator + (pair leader) the MMA issuer: the whole warp runs the
//               loop, one elected lane issues tcgen05.mma (M=256, N=256, K=16, FP32
//               accumulate in TMEM) and tcgen05.commit.
//   warps 2..9  epilogue: tcgen05.ld, + x[i, rep_base + (col mod d_h)] in FP32 (the
//               identity-block gather-add, after the full K-sum like the reference),
//               one rounding, swizzled smem staging, TMA store.  Optional non-finite
//               flag (the reference's _wrap check, tensor.py:112-113).
//
// A is RESIDENT per row-block: with K = d - d_h <= 384 (DeepSeek-V2-Lite kv_b_proj, the
// paper's d = 512 shapes) the CTA's whole A row-block (128 x K, <= 96 KiB) sits in six
// 16 KiB slots and is reused by every n-tile of that row-block, so per tile only B
// streams and the pair's TMA traffic halves.  Larger K streams through the six slots
// as a ring.  Slots are released per k-block by tcgen05.commit after their last MMA, so
// the next row-block's A streams in while the previous tile's MMAs drain.
//
// TMEM holds two 128 x 256 FP32 accumulators (all 512 columns): the epilogue of tile i
// overlaps the MMAs of tile i+1.  The repeated slice x[m0:m0+128, rep_base:+d_h] is
// staged once per row-block into one smem slot by the epilogue's leader thread (TMA),
// read once into registers (a warp's 128 columns map to the same d_h rep columns for
// every tile of the row-block) and the slot is immediately refilled for the next
// row-block, so neither the producer nor the epilogue waits on it in steady state.
// The add is one mixed-precision FHADD (f32 + f16/bf16) per element.  Launches use
// programmatic dependent launch: the prologue overlaps the previous kernel's tail.
//
// Tile schedule: contiguous ranges per pair (A residency), or round-robin when A
// streams (K > 384: keeps the live A/C set inside L2 — cfg3 0.74x -> 1.00x cuBLAS).
// Variants: kCheck (non-finite flag), kRR (round-robin), kNorm (RMSNorm of x fused:
// the epilogue sums each row's squares from the resident A slots + rep registers), BNT
// (tile width: 256, or 128 for launches too short to give every pair two 256-wide tiles),
// kSwap (mirror schedule for problems one column tile wide: coefficients resident).
// Also in this file: kv_proj_small_kernel, the L <= 128 (decode) path — one CTA per
// column block, every k-block loaded at once, cta_group::1 — and the host launchers
// with their launch-parameter cache.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>

#include "kv_proj_internal.h"
#include "ptx_sm100.cuh"
#include "tc_common.cuh"

namespace bdk {
namespace tc {

constexpr int CG = 2;                         // cta_group::2 (CTA pairs)
constexpr int BM = 128;                       // rows per CTA per tile (TMEM lanes)
constexpr int BN = 256;                       // UMMA N (output columns per pair tile); short
                                              // launches use 128-wide tiles (template BNT)
constexpr int NUM_ACC = 512 / BN;             // accumulator buffers in TMEM's 512 columns
constexpr int BK = 64;                        // A k-block: one 128-byte swizzle row of A
constexpr int BKB = 64;                       // B k-block (BKB = 32 with 8 stages: +4 us)
constexpr int B_SUB = BK / BKB;               // B stages per A k-block
constexpr int UK = 16;                        // UMMA K for kind::f16
constexpr int EPI_WARPS = 8;                  // 2 per SMSP; warps w, w+4 share a lane quadrant
constexpr int NUM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int A_SLOTS = 6;                    // resident A: K <= 6 * 64 = 384
constexpr int B_STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2;     // 16 KiB: 128 rows x 64 k
constexpr uint32_t B_PANEL = 64 * BKB * 2;    // one 64-column MN-major swizzle panel, 4 KiB
constexpr int B_PANELS = (BN / 64) / CG;      // this CTA's half of the B tile: 2 panels
constexpr uint32_t B_BYTES = B_PANELS * B_PANEL;
constexpr uint32_t REP_BOX = 64 * BM * 2;     // one 64-column x 128-row rep box, 16 KiB
constexpr uint32_t REP_BYTES = 2 * REP_BOX;   // d_h <= 128 -> at most two boxes
constexpr uint32_t STG_BYTES = 32 * 64 * 2;   // output staging box: 32 rows x 64 cols (SW128)
constexpr int STG_BUFS = 1;                   // per-warp staging buffers
constexpr uint32_t TMEM_COLS = 512;          // NUM_ACC accumulator buffers
constexpr uint32_t NORM_SCRATCH = 2 * BM * 4;  // kNorm: per-row partial sums of squares
constexpr size_t SMEM_BYTES = 1024 + A_SLOTS * A_BYTES + B_STAGES * B_BYTES + REP_BYTES +
                              EPI_WARPS * STG_BUFS * STG_BYTES + 512 + NORM_SCRATCH;
// 128-wide tiles: twice the B stages (same ring bytes) and four accumulator buffers
static_assert((2 * A_SLOTS + 2 * 2 * B_STAGES + 2 * 2 * NUM_ACC + 1) * 8 + 4 <= 512, "barrier area");
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

// Tile order inside a problem: row-block major (column tiles innermost: consecutive
// tiles share the A row-block) — or, for the mirror schedule (kSwap), column-tile major
// (row-blocks innermost: consecutive tiles share the coefficient tile).
template <int BNT = BN, bool kSwap = false>
__device__ __forceinline__ void decode_tile(const TcParams& prm, int t, int& pi, int& m0,
                                            int& n0) {
  pi = 0;
  while (pi + 1 < prm.count && t >= prm.p[pi + 1].tile_start) ++pi;
  const int local = t - prm.p[pi].tile_start;
  if constexpr (kSwap) {
    m0 = (local % prm.p[pi].tiles_m) * (BM * CG);
    n0 = (local / prm.p[pi].tiles_m) * BNT;
  } else {
    n0 = (local % prm.p[pi].tiles_n) * BNT;
    m0 = (local / prm.p[pi].tiles_n) * (BM * CG);
  }
}

// Sequential walk over a pair's contiguous tile range without per-tile divisions
// (decode_tile once, then carry (problem, m0, n0) forward).  The MMA issuer's tile
// boundary sits on the tensor pipe's critical path: a full decode there (integer
// division + indexed parameter loads) cost ~700 clocks per tile.
struct TileCursor {
  int pi, m0, n0;
  int n_span;    // tiles_n * BNT of problem pi (kSwap: tiles_m * BM * CG, the inner loop)
  int pend;      // first tile of problem pi + 1
  int t;
  int step;      // tile stride between this pair's consecutive tiles (1: contiguous)
};
template <int BNT, bool kSwap = false>
__device__ __forceinline__ void cursor_load(const TcParams& prm, TileCursor& c) {
  c.n_span = kSwap ? prm.p[c.pi].tiles_m * (BM * CG) : prm.p[c.pi].tiles_n * BNT;
  c.pend = c.pi + 1 < prm.count ? prm.p[c.pi + 1].tile_start : 0x7fffffff;
}
template <int BNT, bool kSwap = false>
__device__ __forceinline__ TileCursor cursor_at(const TcParams& prm, int t, int step) {
  TileCursor c;
  c.t = t;
  c.step = step;
  decode_tile<BNT, kSwap>(prm, t, c.pi, c.m0, c.n0);
  cursor_load<BNT, kSwap>(prm, c);
  return c;
}
template <bool kRR, int BNT, bool kSwap = false>
__device__ __forceinline__ void cursor_next(const TcParams& prm, TileCursor& c) {
  if constexpr (kRR) {  // round-robin tiles (long K): a full decode is off the critical path
    c.t += c.step;
    if (c.t < prm.total_tiles) {
      decode_tile<BNT, kSwap>(prm, c.t, c.pi, c.m0, c.n0);
      cursor_load<BNT, kSwap>(prm, c);
    }
    return;
  }
  ++c.t;
  if constexpr (kSwap) {
    c.m0 += BM * CG;
    if (c.m0 >= c.n_span) {
      c.m0 = 0;
      c.n0 += BNT;
    }
  } else {
    c.n0 += BNT;
    if (c.n0 >= c.n_span) {
      c.n0 = 0;
      c.m0 += BM * CG;
    }
  }
  if (c.t >= c.pend) {
    ++c.pi;
    c.m0 = 0;
    c.n0 = 0;
    cursor_load<BNT, kSwap>(prm, c);
  }
}

// Tiles sharing (problem, pair row-block) share the A row-block and the rep tile.
__device__ __forceinline__ int blk_key(int pi, int m0) { return (pi << 24) | (m0 / (BM * CG)); }
// The resident operand's key: the A row-block, or (kSwap) the coefficient column tile.
template <bool kSwap, int BNT>
__device__ __forceinline__ int res_key(int pi, int m0, int n0) {
  return kSwap ? ((pi << 24) | (n0 / BNT)) : blk_key(pi, m0);
}

// kCheck: compute the non-finite flag (instantiated only when the caller asked for it).
// kRR: round-robin tile schedule (streaming-A problems), else contiguous ranges.
// kNorm: x is the raw latent and its RMSNorm is fused (see the epilogue).
// BNT: tile width, 256 or — for launches too short to give every pair two 256-wide tiles
// (decode-to-prefill batches on wide problems) — 128: twice the tiles to balance over the
// pairs, each warp's epilogue one 64-column span, four TMEM accumulator buffers.
// kSwap: the mirror schedule for narrow problems (a problem one or two column tiles wide,
// e.g. 2 + 2 heads per GPU under head sharding): the coefficient tile is the RESIDENT
// operand (six 16 KiB slots hold this CTA's 128 columns x K) and x streams through the
// ring, tiles ordered column-tile major — consecutive tiles reuse the coefficients
// instead of reloading a 96 KiB A row-block per tile.  Same MMAs, same k order: outputs
// are bit-identical to the row-block-major schedule's.
template <bool kBF16, bool kCheck, bool kRR, bool kNorm = false, int BNT = BN, bool kSwap = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    kv_proj_tc_kernel(const __grid_constant__ TcParams prm) {
  static_assert(BNT == 256 || BNT == 128, "tile width");
  static_assert(!kSwap || (BNT == 256 && !kRR && !kNorm && B_SUB == 1),
                "mirror schedule: 256-wide tiles, resident K <= 384, no fused norm");
  constexpr int NACC = 512 / BNT;                   // accumulator buffers
  constexpr int BST = B_STAGES * (BN / BNT);        // B ring stages (same bytes)
  constexpr int BPAN = (BNT / 64) / CG;             // this CTA's B panels per stage
  constexpr uint32_t BBYTES = BPAN * B_PANEL;
  constexpr int NSUB = BNT / 64;                    // 32-column sub-chunks per epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + A_SLOTS * A_BYTES;
  uint8_t* sRep = sB + B_STAGES * B_BYTES;  // the ring's bytes do not depend on BNT
  uint8_t* sStg = sRep + REP_BYTES;                 // EPI_WARPS x STG_BUFS x STG_BYTES
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sStg + EPI_WARPS * STG_BUFS * STG_BYTES);
  uint64_t* a_empty = a_full + A_SLOTS;
  uint64_t* b_full = a_empty + A_SLOTS;
  uint64_t* b_empty = b_full + BST;
  uint64_t* tfull = b_empty + BST;
  uint64_t* tempty = tfull + NACC;
  uint64_t* rfull = tempty + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 1);
  float* norm_part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(a_full) + 512);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // 0 = pair leader
  // The parameter block (~7 KB of tensor maps) starts cold in the constant cache: its
  // first reads are misses, so nothing on the barrier-init / TMEM-alloc path depends on
  // them (they complete under the cluster sync).
  const int total_tiles = prm.total_tiles;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < A_SLOTS; ++s) {
      mbar_init(&a_full[s], 1);   // armed by the leader's producer with the pair's bytes
      // one multicast tcgen05.commit (+ kNorm: each of this CTA's four epilogue lane
      // quadrants, done reading the slot)
      mbar_init(&a_empty[s], kNorm ? 1 + 4 : 1);
    }
    for (int s = 0; s < BST; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG);  // one arrival per CTA's epilogue (leader's copy)
    }
    mbar_init(rfull, 1);
    fence_mbar_init();
    for (int i = 0; i < prm.count; ++i) {
      tma_prefetch_desc(&prm.p[i].map_a);
      tma_prefetch_desc(&prm.p[i].map_b);
      tma_prefetch_desc(&prm.p[i].map_out);
      if (prm.p[i].rep_fast) tma_prefetch_desc(&prm.p[i].map_rep);
    }
  }
  if (warp == 1) {
    tmem_alloc<CG>(tmem_slot, TMEM_COLS);
    tmem_relinquish<CG>();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int unit = static_cast<int>(blockIdx.x >> 1);
  const int units = static_cast<int>(gridDim.x >> 1);
  // Contiguous tile range per pair: consecutive tiles share the row-block (A resident,
  // rep tile reused); the split is balanced to within one tile.
  // Tile schedule.  Contiguous ranges per pair (consecutive tiles share the row-block:
  // A resident, rep tile reused; balanced to within one tile) — or, when A streams
  // (K > 384, nothing to reuse), round-robin: pair u takes tiles u, u + units, ..., so at
  // any moment the pairs work on a few adjacent row-blocks and the live set of A and C
  // stays inside L2 instead of 74 far-apart row-blocks thrashing it.
  constexpr bool rr = kRR;
  const int t_step = rr ? units : 1;
  const int t_begin = rr ? unit : static_cast<int>(static_cast<int64_t>(unit) * total_tiles / units);
  const int t_end = rr ? total_tiles
                       : static_cast<int>(static_cast<int64_t>(unit + 1) * total_tiles / units);
  // Programmatic dependent launch: everything up to here (barrier init, TMEM allocation,
  // descriptor prefetch) may overlap the tail of the previous kernel in the stream.  Only
  // the threads that read global memory the previous kernel may have written wait for it
  // (griddep_wait, per thread): the producer before its first TMA load and the epilogue
  // leader before the first rep load.  Everything else that touches global memory is
  // ordered behind those loads (the MMAs consume them; the epilogue's stores and rep
  // reads follow the MMAs), and the MMA issuer touches no global memory.  Dependents may
  // launch right away — they cannot fit on an SM until this CTA exits, and they wait the
  // same way for this grid's completion before reading its output.
  griddep_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Warp-uniform loop (tensor-map / barrier operands stay in uniform registers); one
    // elected lane issues each TMA.
    {
      const uint64_t pol = policy_evict_last();  // x and c are re-read; out streams past
      uint32_t a_iter = 0, b_iter = 0;
      int prev_key = -1;
      // decode the first tile (parameter-cache misses) while the previous grid drains
      int pi0 = 0, m00 = 0, n00 = 0;
      if (t_begin < t_end) {
        decode_tile<BNT, kSwap>(prm, t_begin, pi0, m00, n00);
        const int nkb = prm.p[pi0].num_kb;
        asm volatile("" ::"r"(pi0), "r"(m00), "r"(n00), "r"(nkb));
      }
      griddep_wait();
      for (int t = t_begin; t < t_end; t += t_step) {
        int pi, m0, n0;
        if (t == t_begin) {  // decoded before the wait (cfg2 L = 1024: 8.11 -> 7.83 us)
          pi = pi0;
          m0 = m00;
          n0 = n00;
        } else {
          decode_tile<BNT, kSwap>(prm, t, pi, m0, n0);
        }
        const TcProblem& P = prm.p[pi];
        const int key = res_key<kSwap, BNT>(pi, m0, n0);
        const bool reload_a = P.num_kb > A_SLOTS || key != prev_key;  // the resident operand
        prev_key = key;
        const int my_m0 = m0 + static_cast<int>(rank) * BM;
        const int my_n0 = n0 + static_cast<int>(rank) * (BNT / CG);
        for (int j = 0; j < P.num_kbb; ++j) {
          const int kb = j / B_SUB;
          // Both CTAs' bytes complete on the LEADER's barriers, which the leader arms with
          // the pair's total.  The peer does not arrive: the barrier cannot complete
          // before the leader's arrival, and each CTA only refills a slot after the
          // multicast commit released it, i.e. after the previous phase completed.
          if (reload_a && j % B_SUB == 0) {
            const uint32_t s = a_iter % A_SLOTS;
            mbar_wait(&a_empty[s], ((a_iter / A_SLOTS) & 1u) ^ 1u);
            if (elect_one()) {
              if (rank == 0) mbar_arrive_expect_tx(&a_full[s], CG * A_BYTES);
              if constexpr (kSwap) {  // this CTA's 128 coefficient columns, k-block kb
#pragma unroll
                for (int q = 0; q < 2; ++q)
                  tma_load_2d_pair(sA + s * A_BYTES + q * B_PANEL, &P.map_b, my_n0 + 64 * q,
                                   kb * BK, mapa_shared(smem_u32(&a_full[s]), 0), pol);
              } else {
                tma_load_2d_pair(sA + s * A_BYTES, &P.map_a, kb * BK, my_m0,
                                 mapa_shared(smem_u32(&a_full[s]), 0), pol);
              }
            }
            __syncwarp();
            ++a_iter;
          }
          const uint32_t s = b_iter % BST;
          mbar_wait(&b_empty[s], ((b_iter / BST) & 1u) ^ 1u);
          if (elect_one()) {
            if (rank == 0) mbar_arrive_expect_tx(&b_full[s], CG * BBYTES);
            const uint32_t bar = mapa_shared(smem_u32(&b_full[s]), 0);
            if constexpr (kSwap) {  // this CTA's 128 rows of x, k-block j
              tma_load_2d_pair(sB + s * BBYTES, &P.map_a, j * BKB, my_m0, bar, pol);
            } else {
#pragma unroll
              for (int q = 0; q < BPAN; ++q)
                tma_load_2d_pair(sB + s * BBYTES + q * B_PANEL, &P.map_b, my_n0 + 64 * q,
                                 j * BKB, bar, pol);
            }
          }
          __syncwarp();
          ++b_iter;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    // The whole warp runs the loop (warp-uniform control flow keeps the descriptors in
    // uniform registers); one elected lane issues the tcgen05 instructions.
    if (rank == 0) {
      constexpr uint32_t idesc =
          make_idesc_f16(kBF16, BM * CG, BNT, /*a_mn=*/false, /*b_mn=*/true);
      uint32_t a_iter = 0, a_base = 0, b_iter = 0;
      int prev_key = -1;
      int it = 0;
      TileCursor cur = cursor_at<BNT, kSwap>(prm, t_begin, t_step);
      TileCursor nxt = cur;
      cursor_next<kRR, BNT, kSwap>(prm, nxt);
      for (int t = t_begin; t < t_end; t += t_step, ++it) {
        const int pi = cur.pi;
        const TcProblem& P = prm.p[pi];
        const int num_kb = P.num_kb, num_kbb = P.num_kbb;
        const int key = res_key<kSwap, BNT>(pi, cur.m0, cur.n0);
        const bool stream_a = num_kb > A_SLOTS;
        const bool reload_a = stream_a || key != prev_key;
        prev_key = key;
        // Last tile reading this resident block: release each slot after its k-block's MMAs.
        const bool last_use = stream_a || t + t_step >= t_end ||
                              res_key<kSwap, BNT>(nxt.pi, nxt.m0, nxt.n0) != key;
        cur = nxt;
        cursor_next<kRR, BNT, kSwap>(prm, nxt);
        if (reload_a) {
          a_base = a_iter;
          a_iter += num_kb;
        }
        const int acc = it % NACC;
        const uint32_t acc_phase = (it / NACC) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BNT;
        for (int j = 0; j < num_kbb; ++j) {
          const int kb = j / B_SUB;
          const uint32_t ai = a_base + kb;
          const uint32_t as = ai % A_SLOTS;
          if (reload_a && j % B_SUB == 0) mbar_wait(&a_full[as], (ai / A_SLOTS) & 1u);
          const uint32_t bs = b_iter % BST;
          mbar_wait(&b_full[bs], (b_iter / BST) & 1u);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + as * A_BYTES);
          const uint32_t b0 = smem_u32(sB + bs * BBYTES);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < BKB / UK; ++ks) {
              // A: K-major SW128, rows 128 B apart, 8-row groups 1024 B apart; a 16-wide
              //    k step is +32 B inside the swizzle row.
              // (kSwap: the same two layouts with the regions exchanged — x's k-block in
              //  the ring stage, the coefficient panels in the resident slot)
              const uint32_t abase = kSwap ? b0 : a0;
              const uint32_t bbase = kSwap ? a0 : b0;
              const uint64_t adesc =
                  make_smem_desc(abase + ((j % B_SUB) * BKB + ks * UK) * 2, 16, 1024);
              // B: MN-major SW128, 64-column panels B_PANEL apart (LBO), 8-k-row groups
              //    1024 B apart (SBO); a 16-deep k step is two 8-row groups = 2048 B.
              const uint64_t bdesc = make_smem_desc(bbase + ks * (UK * 128), B_PANEL, 1024);
              tc_mma_f16_pair(d_tmem, adesc, bdesc, idesc, (j | ks) != 0 ? 1u : 0u);
            }
            tc_commit_pair(&b_empty[bs], 0x3);
            if (last_use && (j % B_SUB == B_SUB - 1 || j + 1 == num_kbb))
              tc_commit_pair(&a_empty[as], 0x3);
          }
          __syncwarp();
          ++b_iter;
        }
        if (elect_one()) tc_commit_pair(&tfull[acc], 0x3);
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
    const uint32_t stg0 = smem_u32(sStg + ew * STG_BUFS * STG_BYTES);
    const uint32_t sw128 = static_cast<uint32_t>(row_w & 7);
    const uint8_t* rep_row = sRep + row_t * 128;
    // leader only: stage the rep tile of tile t (this CTA's 128 rows) into the slot
    auto issue_rep = [&](int t) {
      int pi, m0, n0;
      decode_tile<BNT, kSwap>(prm, t, pi, m0, n0);
      const TcProblem& P = prm.p[pi];
      const int nbox = P.d_h / 64;
      mbar_arrive_expect_tx(rfull, nbox * REP_BOX);
      for (int b = 0; b < nbox; ++b)
        tma_load_2d(sRep + b * REP_BOX, &P.map_rep, 64 * b, m0 + static_cast<int>(rank) * BM,
                    rfull, policy_evict_last());
    };
    // leader only: the first tile at or after t (in this pair's sequence) that belongs to
    // a rep_fast problem and to a row-block other than `key` — the next tile whose rep
    // tile the epilogue will wait for.  Non-fast row-blocks in between (a grouped launch
    // may mix d_h) are skipped: nothing waits on rfull for them.
    auto issue_next_rep = [&](int t, int key) {
      for (; t < t_end; t += t_step) {
        int pi, m0, n0;
        decode_tile<BNT, kSwap>(prm, t, pi, m0, n0);
        if (prm.p[pi].rep_fast && blk_key(pi, m0) != key) {
          issue_rep(t);
          return;
        }
      }
    };
    if (leader && t_begin < t_end) {
      int pi, m0, n0;
      decode_tile<BNT, kSwap>(prm, t_begin, pi, m0, n0);
      const int fast0 = prm.p[pi].rep_fast;
      asm volatile("" ::"r"(fast0));
      griddep_wait();
      issue_next_rep(t_begin, -1);
    }
    if (prm.world > 0 && lane == 0) {
      // peer tensor maps were copied to global memory before the launch: order those
      // generic-proxy writes before the TMA unit's descriptor reads
      for (int i = 0; i < prm.count * prm.world; ++i)
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(
                         reinterpret_cast<uint64_t>(prm.peer_maps + i))
                     : "memory");
    }
    uint32_t chk = 0u;  // NaN-propagating packed max |out| (16-bit) for the non-finite check
    uint32_t rep_loads = 0;
    int cur_key = -1;   // row-block whose rep values are in repv (-1: none)
    uint4 repv[8];      // rep values of this thread's row, columns half*64 + [0, 64) mod d_h
    float rnorm = 1.0f;         // kNorm: 1 / RMS of this thread's row
    bool norm_pending = false;  // kNorm: a new row-block's norm is still to be computed
    uint32_t ep_a_iter = 0, ep_a_base = 0;  // kNorm: mirror of the MMA's A-slot sequence
    int it = 0;
    for (int t = t_begin; t < t_end; t += t_step, ++it) {
      int pi, m0, n0;
      decode_tile<BNT, kSwap>(prm, t, pi, m0, n0);
      const TcProblem& P = prm.p[pi];
      const int my_m0 = m0 + static_cast<int>(rank) * BM;
      const int key = blk_key(pi, m0);
      const bool fast = P.rep_fast != 0;
      if (fast && key != cur_key) {
        // New row-block: pull this thread's rep values (row row_t, the warp's WC columns
        // mod d_h — the same for every tile of the row-block) from the staged tile into
        // registers once, then hand the slot straight back for the next row-block.
        mbar_wait(rfull, rep_loads & 1u);
        ++rep_loads;
        cur_key = key;
        if constexpr (kNorm) {
          norm_pending = true;
          ep_a_base = ep_a_iter;
          ep_a_iter += static_cast<uint32_t>(P.num_kb);
        }
        const int dm = P.d_h - 1;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const int jj = (static_cast<int>(half) * 64 + 8 * g) & dm;
          const uint32_t ch = static_cast<uint32_t>((jj & 63) >> 3);
          repv[g] = *reinterpret_cast<const uint4*>(rep_row + (jj >> 6) * REP_BOX +
                                                    ((ch ^ (row_t & 7)) << 4));
        }
        named_bar_sync(2, 32 * EPI_WARPS);  // every epilogue thread holds its rep values
        if (leader) issue_next_rep(t + t_step, key);  // the next fast row-block's rep
      }
      const int acc = it % NACC;
      const uint32_t acc_phase = (it / NACC) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if constexpr (kNorm) {
        if (norm_pending) {
          // Fused RMSNorm of x (DeepSeek kv_a_layernorm): the row's sum of squares from
          // the resident A k-blocks (all landed: this tile's MMAs read them) and the rep
          // values in registers; the two warps of a quadrant split the row and meet in
          // shared memory.  Then out = r * (sum_k x c_g + gamma_rep x_rep) is evaluated as
          // (r * acc) + fp16(r * gamma_rep * x_rep): the rep registers are rescaled here.
          norm_pending = false;
          float ssv[4] = {0.f, 0.f, 0.f, 0.f};  // independent chains
          const int nkb = P.num_kb;
          for (int kb = static_cast<int>(half) * 3; kb < nkb && kb < static_cast<int>(half) * 3 + 3;
               ++kb) {
            const uint8_t* arow =
                sA + ((ep_a_base + static_cast<uint32_t>(kb)) % A_SLOTS) * A_BYTES + row_t * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint4 q = *reinterpret_cast<const uint4*>(arow + ((ch ^ (row_t & 7)) << 4));
              const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = unpack2<kBF16>(w[e]);
                ssv[e] = fmaf(f.x, f.x, fmaf(f.y, f.y, ssv[e]));
              }
            }
          }
          if (half == 0 || P.d_h > 64) {  // the rep columns, each counted once
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const uint32_t w[4] = {repv[g].x, repv[g].y, repv[g].z, repv[g].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = unpack2<kBF16>(w[e]);
                ssv[e] = fmaf(f.x, f.x, fmaf(f.y, f.y, ssv[e]));
              }
            }
          }
          // the two warps of this lane quadrant meet (named barrier 4 + quad, 64 threads):
          // the other quadrants run on, their warps not held at a CTA-wide barrier
          norm_part[half * BM + row_t] = (ssv[0] + ssv[1]) + (ssv[2] + ssv[3]);
          named_bar_sync(4 + quad, 64);
          const float tot = norm_part[row_t] + norm_part[BM + row_t];
          // rows past L are TMA zero-fill: with eps == 0 their rsqrt would be inf and
          // 0 * inf a NaN that trips the non-finite check — they are never stored, use 0
          rnorm = my_m0 + row_t < P.L ? rsqrtf(tot / static_cast<float>(P.norm_d) + P.norm_eps)
                                      : 0.f;
          named_bar_sync(4 + quad, 64);  // this quadrant read its A rows and the partials
          if (half == 0 && lane == 0)
            for (int kb = 0; kb < nkb; ++kb)
              mbar_arrive(&a_empty[(ep_a_base + static_cast<uint32_t>(kb)) % A_SLOTS]);
          const int dm = P.d_h - 1;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const int jj = (static_cast<int>(half) * 64 + 8 * g) & dm;
            uint32_t w[4] = {repv[g].x, repv[g].y, repv[g].z, repv[g].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = unpack2<kBF16>(w[e]);
              w[e] = pack2<kBF16>(rnorm * __ldg(P.rep_gamma + jj + 2 * e) * f.x,
                                  rnorm * __ldg(P.rep_gamma + jj + 2 * e + 1) * f.y);
            }
            repv[g] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      const int64_t grow = static_cast<int64_t>(my_m0) + row_t;
      const bool has_rep = P.has_rep != 0;
      const uint16_t* xrow = static_cast<const uint16_t*>(P.x) +
                             (grow < P.L ? grow : 0) * P.ldx + P.rep_base;
      // Warp columns: two 64-wide spans, [64 h, 64 h + 64) and [128 + 64 h, ...) of the
      // tile (h = half), so both spans map to the same d_h-periodic rep columns (d_h in
      // {64, 128}) and the rep needs only 32 registers.  Four 32-column sub-chunks c:
      // column cb(c) = (c >> 1) * 128 + 64 h + (c & 1) * 32 (increasing in c).
      auto cb = [&](int c) { return (c >> 1) * 128 + static_cast<int>(half) * 64 + (c & 1) * 32; };
      int nsub = 0;
#pragma unroll
      for (int c = 0; c < NSUB; ++c) nsub += (n0 + cb(c) < P.N) ? 1 : 0;
      const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * BNT;

      // One 32-column sub-chunk c: + rep, round, swizzled staging into the warp's
      // 32 x 64 box (two sub-chunks per box, one box per span); the box's TMA store is
      // issued after its second sub-chunk (or the tile's last).  Before a box's first
      // sub-chunk is written, the previous box's store must have finished reading it.
      auto process = [&](const uint32_t (&r)[32], int c) {
        const int col0 = n0 + cb(c);
        uint4 xv[4];
        if (fast) {
#pragma unroll
          for (int g = 0; g < 4; ++g) xv[g] = repv[(c & 1) * 4 + g];
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
        const uint32_t part = static_cast<uint32_t>(c & 1);
        if (part == 0) {
          if (lane == 0) tma_store_wait_read<0>();
          __syncwarp();
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t xw[4] = {xv[g].x, xv[g].y, xv[g].z, xv[g].w};
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // + rep in FP32 with one mixed-precision FHADD per element (exact widening of
            // the 16-bit rep, one FP32 rounding), then one rounding to 16 bit
            float a0 = __uint_as_float(r[8 * g + 2 * e]);
            float a1 = __uint_as_float(r[8 * g + 2 * e + 1]);
            if constexpr (kNorm) {
              a0 *= rnorm;
              a1 *= rnorm;
            }
            const float2 v = add_f32_x16x2<kBF16>(a0, a1, xw[e]);
            o[e] = pack2<kBF16>(v.x, v.y);
            if constexpr (kCheck) chk = max_abs2_nan<kBF16>(chk, o[e]);
          }
          const uint32_t dst = stg0 + row_w * 128 + (((4 * part + g) ^ sw128) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]),
                       "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");
        }
        if (part == 1 || c + 1 == nsub) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int bcol = col0 - static_cast<int>(part) * 32;
            const int brow = my_m0 + static_cast<int>(quad) * 32;
            if (prm.world > 0) {
              // all-gather fused into the epilogue: the same staged box goes to every
              // rank's full-width buffer, at this rank's head planes
              for (int r = 0; r < prm.world; ++r)
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                        reinterpret_cast<uint64_t>(prm.peer_maps + pi * prm.world + r)),
                    "r"(stg0), "r"(bcol % P.out_d_h), "r"(brow),
                    "r"(prm.head0[pi] + bcol / P.out_d_h)
                    : "memory");
            } else if (P.head_major)
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(&P.map_out)),
                  "r"(stg0), "r"(bcol % P.out_d_h), "r"(brow), "r"(bcol / P.out_d_h)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                      reinterpret_cast<uint64_t>(&P.map_out)),
                  "r"(stg0), "r"(bcol), "r"(brow)
                  : "memory");
            tma_store_commit();
          }
        }
      };

      if (nsub > 0) {
        // 32-column TMEM loads, double-buffered: sub-chunk c+1 is in flight while c is
        // processed (tcgen05.wait::ld waits for all of a thread's loads, so two is the depth)
        uint32_t ra[32], rb[32];
        tmem_ld_32x32b_x32(taddr + cb(0), ra);
#pragma unroll
        for (int c = 0; c < NSUB; c += 2) {
          if (c < nsub) {
            tmem_ld_wait();
            if (c + 1 < nsub) tmem_ld_32x32b_x32(taddr + cb(c + 1), rb);
            process(ra, c);
          }
          if (c + 1 < nsub) {
            tmem_ld_wait();
            if (c + 2 < nsub) tmem_ld_32x32b_x32(taddr + cb(c + 2), ra);
            process(rb, c + 1);
          }
        }
      }
      tc_fence_before();
      named_bar_sync(1, 32 * EPI_WARPS);  // all epilogue threads finished with TMEM + rep
      if (leader) {
        mbar_arrive_remote(mapa_shared(smem_u32(&tempty[acc]), 0));
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
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, TMEM_COLS);
  }
}


// ---------------------------------------------------------------------------------
// Small-L ("decode") kernel: L <= 512 tokens (while the CTAs fit one wave), K <= 384.
// The persistent pair kernel spends a full 256-row tile, its prologue and a 256-column
// epilogue per output block — ~8 us whatever L is.  Here each CTA owns one BNS-column
// block of one problem for one 128-row block (all rows when L <= 128): its whole A (x
// rows, <= 128 x K) and B (K x BNS) slices are loaded at once
// (one barrier per 64-deep k-block so the MMAs start on the first), one M=128 x N=BNS
// accumulator in TMEM (cta_group::1), and four epilogue warps add the repeated slice
// (global loads, L2-resident), round and store straight to global memory.  The work is
// streaming C once across ~128 CTAs; the same FP32 accumulation + FHADD + rounding as
// the main kernel.
constexpr int SM_THREADS = 64 + 128;  // producer, MMA, 4 epilogue warps
constexpr int SM_MAX_KB = 6;          // K <= 384
constexpr uint32_t SM_STG = 4 * 2 * STG_BYTES;  // pair variant: 2 staging boxes per epilogue warp
inline size_t small_smem_bytes(int bns_per_cta, int a_kb_bytes, bool tma_store) {
  return 1024 + SM_MAX_KB * (a_kb_bytes + bns_per_cta * BKB * 2) +
         (tma_store ? SM_STG : 0) + 128;
}

// CGS = 2: a CTA pair (cluster of 2, cta_group::2, M = 256) covers L <= 256; each CTA
// holds its 128 rows of A and half of the BNS-column B block, like the persistent kernel.
template <bool kBF16, bool kCheck, int BNS, int CGS>
__global__ void __launch_bounds__(SM_THREADS, 1)
    kv_proj_small_kernel(const __grid_constant__ TcParams prm) {
  // B panels: 64 columns with the 128-byte swizzle, or 32-column panels with the 64-byte
  // swizzle for column blocks that are not a multiple of 64 (32, 96, 160: one wave of
  // CTAs on decode-sized, narrow launches)
  constexpr int PW = (BNS / CGS) % 64 == 0 ? 64 : 32;
  constexpr int PANELS = BNS / CGS / PW;
  constexpr uint32_t PANEL_BYTES = PW * BKB * 2;
  constexpr uint32_t BS_BYTES = PANELS * PANEL_BYTES;  // one k-block of this CTA's B
  constexpr uint32_t B_LAYOUT = PW == 64 ? 2u : 4u;     // SWIZZLE_128B / SWIZZLE_64B
  // TMEM allocations are powers of two >= 32 columns
  constexpr uint32_t TCOLS = BNS <= 32 ? 32 : BNS <= 64 ? 64 : BNS <= 128 ? 128 : 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  // A k-blocks hold only the L (rounded up to 8) rows the box loads; the MMA still reads
  // 128 rows, and the rows past L land in accumulator lanes that are never stored
  const uint32_t a_kb = static_cast<uint32_t>(prm.a_kb_bytes);
  // 128-column blocks and pairs store through smem + TMA; 64-column blocks (two CTAs per
  // SM, no room for staging) store directly
  constexpr bool kTma = CGS == 2 || BNS == 128;
  uint8_t* sA = smem;
  uint8_t* sB = sA + SM_MAX_KB * a_kb;
  uint8_t* sStg = sB + SM_MAX_KB * BS_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + (kTma ? SM_STG : 0));
  uint64_t* done = full + SM_MAX_KB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  const uint32_t rank = CGS == 2 ? cluster_ctarank() : 0u;  // 0 = pair leader

  int pi, m0, n0;
  {
    // block (group) -> (problem, column block, row block); tiles_n counts BNS-wide
    // blocks here, row blocks are BM * CGS rows (one for L <= 128 * CGS)
    const int tb = static_cast<int>(blockIdx.x) / CGS;
    const int nrb = prm.small_rblocks;
    const int t = tb / nrb;
    pi = 0;
    while (pi + 1 < prm.count && t >= prm.p[pi + 1].tile_start) ++pi;
    n0 = (t - prm.p[pi].tile_start) * BNS;
    m0 = (tb % nrb) * (BM * CGS) + static_cast<int>(rank) * BM;  // this CTA's rows
  }
  const int my_n0 = n0 + static_cast<int>(rank) * (BNS / CGS);  // this CTA's B columns
  const TcProblem& P = prm.p[pi];
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < SM_MAX_KB; ++kb) mbar_init(&full[kb], 1);
    mbar_init(done, 1);
    fence_mbar_init();
    tma_prefetch_desc(&P.map_a);
    tma_prefetch_desc(&P.map_b);
    // This CTA's C slice into L2 before the PDL wait: L2 is the GPU's point of
    // coherence, so a prefetch can never return stale data even if the previous kernel
    // wrote C — it only starts the DRAM read of the weights under that kernel's tail.
    // (x, which the previous kernel may produce, is read only after the wait.)
    for (int kb = 0; kb < P.num_kb; ++kb)
      for (int q = 0; q < PANELS; ++q)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&P.map_b)),
                     "r"(my_n0 + PW * q), "r"(kb * BK)
                     : "memory");
  }
  if (warp == 1) {
    tmem_alloc<CGS>(tmem_slot, TCOLS);
    tmem_relinquish<CGS>();
  }
  tc_fence_before();
  if constexpr (CGS == 2)
    cluster_sync();  // the leader's barriers exist before the peer's TMA signals them
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  if (warp == 0) {
    // ---- producer: every k-block of A and B at once (nothing to recycle).  Pairs: both
    // CTAs' bytes complete on the leader's barrier, armed with the pair's total.
    griddep_wait();
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();  // C is shared by the row... and re-read
      for (int kb = 0; kb < P.num_kb; ++kb) {
        if constexpr (CGS == 2) {
          if (rank == 0) mbar_arrive_expect_tx(&full[kb], CGS * (a_kb + BS_BYTES));
          const uint32_t bar = mapa_shared(smem_u32(&full[kb]), 0);
          tma_load_2d_pair(sA + kb * a_kb, &P.map_a, kb * BK, m0, bar, pol);
          for (int q = 0; q < PANELS; ++q)
            tma_load_2d_pair(sB + kb * BS_BYTES + q * PANEL_BYTES, &P.map_b, my_n0 + PW * q,
                             kb * BK, bar, pol);
        } else {
          mbar_arrive_expect_tx(&full[kb], a_kb + BS_BYTES);
          tma_load_2d(sA + kb * a_kb, &P.map_a, kb * BK, m0, &full[kb], pol);
          for (int q = 0; q < PANELS; ++q)
            tma_load_2d(sB + kb * BS_BYTES + q * PANEL_BYTES, &P.map_b, my_n0 + PW * q, kb * BK,
                        &full[kb], pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA (pair leader): M = 128 * CGS (rows >= L zero-filled by TMA), N = BNS
    constexpr uint32_t idesc =
        make_idesc_f16(kBF16, BM * CGS, BNS, /*a_mn=*/false, /*b_mn=*/true);
    if (rank == 0) {
      for (int kb = 0; kb < P.num_kb; ++kb) {
        mbar_wait(&full[kb], 0);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a0 = smem_u32(sA + kb * a_kb);
          const uint32_t b0 = smem_u32(sB + kb * BS_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / UK; ++ks) {
            const uint64_t ad = make_smem_desc(a0 + ks * (UK * 2), 16, 1024);
            const uint64_t bdsc =
                make_smem_desc_sw(b0 + ks * (UK * PW * 2), PANEL_BYTES, 8 * PW * 2, B_LAYOUT);
            if constexpr (CGS == 2)
              tc_mma_f16_pair(tmem_base, ad, bdsc, idesc, (kb | ks) != 0 ? 1u : 0u);
            else
              tc_mma_f16(tmem_base, ad, bdsc, idesc, (kb | ks) != 0 ? 1u : 0u);
          }
          if (kb + 1 == P.num_kb) {
            if constexpr (CGS == 2)
              tc_commit_pair(done, 0x3);
            else
              tc_commit(done);
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. (its rows), all BNS columns
    const uint32_t quad = warp & 3;
    const int row = m0 + static_cast<int>(quad * 32 + lane);  // this CTA's rows
    uint32_t chk = 0u;
    griddep_wait();  // the repeated slice is read from x below
    const bool live = row < P.L;
    const uint16_t* xrow = static_cast<const uint16_t*>(P.x) +
                           static_cast<int64_t>(live ? row : 0) * P.ldx + P.rep_base;
    // every CTA reads the same few rows of x here: issue all of this thread's rep loads
    // before waiting for the MMAs so their (contended) latency hides behind the loads
    uint4 xr[BNS / 8];
#pragma unroll
    for (int j = 0; j < BNS / 8; ++j) {
      const int col = n0 + 8 * j;
      xr[j] = (live && P.has_rep && col < P.N)
                  ? __ldg(reinterpret_cast<const uint4*>(xrow + (col % P.d_h)))
                  : make_uint4(0, 0, 0, 0);
    }
    mbar_wait(done, 0);
    tc_fence_after();
    if constexpr (kTma) {
      // rows of this warp: m0 + 32 quad + [0, 32); TMA clips rows >= L and cols >= N
      if (m0 + static_cast<int>(quad) * 32 < P.L) {
        const uint32_t stg = smem_u32(sStg + (warp - 2) * 2 * STG_BYTES);
#pragma unroll
        for (int c = 0; c < BNS / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + c * 32, r);
          tmem_ld_wait();
          const int bx = c >> 1, part = c & 1;
          const uint32_t buf = stg + static_cast<uint32_t>(bx & 1) * STG_BYTES;
          if (part == 0 && bx >= 2) {  // the store from two boxes ago has read this buffer
            if (lane == 0) tma_store_wait_read<1>();
            __syncwarp();
          }
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
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(o[0]),
                         "r"(o[1]), "r"(o[2]), "r"(o[3])
                         : "memory");
          }
          if (part == 1) {
            fence_proxy_async_smem();
            __syncwarp();
            const int bcol = n0 + bx * 64;
            if (lane == 0 && bcol < P.N) {
              const int brow = m0 + static_cast<int>(quad) * 32;
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
            }
            if (lane == 0) tma_store_commit();  // an empty group keeps the count aligned
          }
        }
        if (lane == 0) tma_store_wait_all<0>();
      }
    } else
#pragma unroll
    for (int c = 0; c < BNS / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_base + ((quad * 32u) << 16) + c * 32, r);
      tmem_ld_wait();
      const int col0 = n0 + c * 32;
      if (!live || col0 >= P.N) continue;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int col = col0 + 8 * g;
        if (col >= P.N) break;
        const uint4 xv = xr[c * 4 + g];
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 v = add_f32_x16x2<kBF16>(__uint_as_float(r[8 * g + 2 * e]),
                                               __uint_as_float(r[8 * g + 2 * e + 1]), xw[e]);
          o[e] = pack2<kBF16>(v.x, v.y);
          if constexpr (kCheck) chk = max_abs2_nan<kBF16>(chk, o[e]);
        }
        uint16_t* dst;
        if (P.head_major) {
          const int h = col / P.out_d_h;
          dst = static_cast<uint16_t*>(P.out) +
                (static_cast<int64_t>(h) * P.L + row) * P.ldo + (col - h * P.out_d_h);
        } else {
          dst = static_cast<uint16_t*>(P.out) + static_cast<int64_t>(row) * P.ldo + col;
        }
        *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
    if constexpr (kCheck) {
      if (__any_sync(0xffffffffu, nonfinite2<kBF16>(chk)) && lane == 0) atomicExch(prm.flag, 1);
    }
  }
  tc_fence_before();
  if constexpr (CGS == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CGS>(tmem_base, TCOLS);
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
               CUtensorMapSwizzle swz) {
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

// Row-major [planes x rows x cols] 16-bit tensor (row stride ld, plane stride ps
// elements), box {box_cols, box_rows, 1}, 128B swizzle.
bool encode_3d(CUtensorMap* map, const void* base, bool bf16, uint64_t cols, uint64_t rows,
               uint64_t planes, uint64_t ld, uint64_t ps, uint32_t box_cols, uint32_t box_rows,
               std::string* err) {
  auto fn = encode_fn();
  if (fn == nullptr) {
    *err = "cuTensorMapEncodeTiled unavailable from the driver";
    return false;
  }
  const cuuint64_t dims[3] = {cols, rows, planes};
  const cuuint64_t strides[2] = {ld * 2, ps * 2};
  const cuuint32_t box[3] = {box_cols, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (3-D) failed (CUresult %d)",
             static_cast<int>(r));
    *err = buf;
    return false;
  }
  return true;
}

}  // namespace tc

namespace {

// Launch-parameter cache.  Encoding the tensor maps (four per problem, plus one per peer)
// is most of the library's host time per call (~10 us for cfg2); a serving loop calls
// with the same buffers over and over, so the encoded TcParams are kept per problem
// signature.  Tensor maps are pure host-side encodings of (pointer, shape, strides,
// box): an identical signature yields identical maps.
struct ParamKey {
  int32_t count;
  int32_t bf16;
  Problem p[BD_MAX_GROUP];
};
struct ParamEntry {
  bool valid;
  ParamKey key;
  tc::TcParams prm;
};
constexpr int kParamCacheSize = 8;
std::mutex g_param_mu;
ParamEntry g_param_cache[kParamCacheSize];
int g_param_next = 0;

ParamKey make_key(const Problem* probs, int count, bool bf16) {
  ParamKey k;
  memset(&k, 0, sizeof(k));  // padding included: keys compare with memcmp
  k.count = count;
  k.bf16 = bf16 ? 1 : 0;
  for (int i = 0; i < count; ++i) {
    const Problem& q = probs[i];
    Problem& d = k.p[i];
    d.x = q.x;
    d.c = q.c;
    d.out = q.out;
    d.ldx = q.ldx;
    d.ldc = q.ldc;
    d.ldo = q.ldo;
    d.L = q.L;
    d.K = q.K;
    d.N = q.N;
    d.d_h = q.d_h;
    d.mul_base = q.mul_base;
    d.rep_base = q.rep_base;
    d.out_layout = q.out_layout;
    d.world = q.world;
    d.head0 = q.head0;
    for (int r = 0; r < q.world && r < BD_MAX_PEERS; ++r) d.peers[r] = q.peers[r];
    d.rep_gamma = q.rep_gamma;
    d.norm_eps = q.norm_eps;
  }
  return k;
}

int build_params(const Problem* probs, int count, bool bf16, tc::TcParams& prm,
                 cudaStream_t stream);
int launch_params(const tc::TcParams& prm, int total, bool bf16, bool check,
                  cudaStream_t stream);

}  // namespace

// Column block of the single-CTA small kernel for `cols` columns in `nrb` 128-row blocks:
// the narrowest of 32 / 64 / 128 / 160 whose CTAs fit one wave (64 may run two CTAs per
// SM when its shared memory allows), or 0 when none does.  (96 is instantiated for A/B —
// BD_SMALL_BNS=96 — but at three row blocks it measured slower than 128: cfg2 L = 384
// 4.95 vs 4.79 us; 160 at five row blocks beats the persistent kernel: L = 640 6.82 vs
// 7.65 us, tools/small_bns_wave_ab.sh.)
int small_bns_one_wave(int64_t cols, int64_t nrb, int a_kb_bytes) {
  const int64_t sms = sm_count();
  const int per_sm64 = tc::small_smem_bytes(64, a_kb_bytes, false) * 2 <= 232448 ? 2 : 1;
  for (int b : {32, 64, 128, 160}) {
    if (tc::small_smem_bytes(b, a_kb_bytes, b == 128) > 232448) continue;
    if ((cols + b - 1) / b * nrb <= (b == 64 ? per_sm64 : 1) * sms) return b;
  }
  return 0;
}

// Small-L launch: one CTA per BNS-column block of each problem (no clusters).
int launch_small(const Problem* probs, int count, bool bf16, int* flag, cudaStream_t stream) {
  using namespace tc;
  int64_t cols = 0, max_l = 1;
  for (int i = 0; i < count; ++i) {
    cols += probs[i].N;
    max_l = probs[i].L > max_l ? probs[i].L : max_l;
  }
  // One CTA (M = 128) per (128-row block, column block).  BD_SMALL_PAIRS=1 (A/B) runs
  // L > 128 on CTA pairs instead (M = 256, each CTA its 128 rows of A and half of the
  // column block's B): half the CTAs, and measured slower — cfg2 K'+V' L = 256 / 384 /
  // 512: 4.69 / 5.95 / 5.99 us on pairs, 4.32 / 4.75 / 5.11 on single CTAs
  // (tools/small_single_ab.sh)
  static const bool pairs = [] {
    const char* e = getenv("BD_SMALL_PAIRS");
    return e != nullptr && atoi(e) == 1;
  }();
  const int cgs = max_l > BM && pairs ? 2 : 1;
  const int nrb = static_cast<int>((max_l + BM * cgs - 1) / (BM * cgs));  // row blocks
  const int a_rows = cgs == 2 || max_l > BM ? BM : static_cast<int>((max_l + 7) / 8 * 8);
  const int a_kb_bytes = a_rows * BK * 2;
  int bns;
  if (cgs == 1) {
    // Column block: the narrowest whose CTAs fit one wave (the shortest MMA chain and B
    // slice per CTA, the most SMs pulling C in); 128 when none does (L <= 128 on wide
    // problems: several waves)
    bns = small_bns_one_wave(cols, nrb, a_kb_bytes);
    if (bns == 0) bns = 128;
    static const int bns_env = [] {  // BD_SMALL_BNS=32|64|96|128|160: force it (A/B)
      const char* e = getenv("BD_SMALL_BNS");
      return e != nullptr ? atoi(e) : 0;
    }();
    if (bns_env == 32 || bns_env == 64 || bns_env == 96 || bns_env == 128 || bns_env == 160)
      bns = bns_env;
  } else {
    // pairs: one CTA per SM (A is 96 KiB); 256-column blocks once they fill a wave
    bns = (cols + 127) / 128 * nrb <= static_cast<int64_t>(sm_count() / 2) ? 128 : 256;
  }
  const bool tma_st = cgs == 2 || bns == 128;
  TcParams prm{};
  prm.count = count;
  prm.flag = flag;
  prm.a_kb_bytes = a_kb_bytes;
  prm.small_rblocks = nrb;
  int total = 0;
  for (int i = 0; i < count; ++i) {
    const Problem& q = probs[i];
    TcProblem& P = prm.p[i];
    std::string err;
    const bool has_rep = q.rep_base >= 0;
    const auto* xb = static_cast<const uint16_t*>(q.x) + q.mul_base;
    if (!encode_2d(&P.map_a, xb, bf16, q.K, q.L, q.ldx, BK, a_rows, &err) ||
        !encode_2d(&P.map_b, q.c, bf16, q.N, q.K, q.ldc, (bns / cgs) % 64 == 0 ? 64 : 32, BK,
                   &err,
                   (bns / cgs) % 64 == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) ||
        (tma_st &&
         !(q.out_layout == BD_OUT_HEAD_MAJOR
               ? encode_3d(&P.map_out, q.out, bf16, q.d_h, q.L, q.N / q.d_h, q.ldo,
                           q.L * q.ldo, 64, 32, &err)
               : encode_2d(&P.map_out, q.out, bf16, q.N, q.L, q.ldo, 64, 32, &err)))) {
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
    P.num_kb = static_cast<int32_t>((q.K + BK - 1) / BK);
    P.tiles_n = static_cast<int32_t>((q.N + bns - 1) / bns);
    P.tile_start = total;
    total += P.tiles_n;
  }
  prm.total_tiles = total;
  if (total == 0) return BD_OK;
  using KernFn = void (*)(TcParams);
  // [bf16][check][0: 1 CTA x 64, 1: 1 CTA x 128, 2: pair x 128, 3: pair x 256,
  //               4: 1 CTA x 32, 5: 1 CTA x 96, 6: 1 CTA x 160]
#define BD_SMALL_ROW(B, C)                                                                   \
  {kv_proj_small_kernel<B, C, 64, 1>, kv_proj_small_kernel<B, C, 128, 1>,                    \
   kv_proj_small_kernel<B, C, 128, 2>, kv_proj_small_kernel<B, C, 256, 2>,                   \
   kv_proj_small_kernel<B, C, 32, 1>, kv_proj_small_kernel<B, C, 96, 1>,                     \
   kv_proj_small_kernel<B, C, 160, 1>}
  static const KernFn kerns[2][2][7] = {
      {BD_SMALL_ROW(false, false), BD_SMALL_ROW(false, true)},
      {BD_SMALL_ROW(true, false), BD_SMALL_ROW(true, true)}};
#undef BD_SMALL_ROW
  const int vb = bf16 ? 1 : 0, vc = flag != nullptr ? 1 : 0;
  const int vn = cgs == 1 ? (bns == 128 ? 1 : bns == 32 ? 4 : bns == 96 ? 5 : bns == 160 ? 6 : 0)
                          : (bns == 256 ? 3 : 2);
  const KernFn kern = kerns[vb][vc][vn];
  const size_t smem = small_smem_bytes(bns / cgs, a_kb_bytes, tma_st);
  // the attribute belongs to the function in the CURRENT device's context: set it once
  // per device ordinal
  static std::atomic<bool> attr_done[kMaxDevices][2][2][7] = {};
  static std::mutex attr_mu;
  const int dv = device_slot();
  if (!attr_done[dv][vb][vc][vn].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(attr_mu);
    // the largest footprint this variant can ask for
    const cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(small_smem_bytes(bns / cgs, A_BYTES, tma_st)));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_done[dv][vb][vc][vn].store(true, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(total * cgs * nrb);
  cfg.blockDim = dim3(SM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cgs;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cgs == 2 ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm);
  note_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("kv_proj_small launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

// Problems the small-L kernel serves: every problem at most one 128-row tile deep with
// A resident (K <= 384), and no fused all-gather.
bool small_eligible(const Problem* probs, int count) {
  static const bool off = [] {  // BD_SMALL_L=0 routes small L to the persistent kernel
    const char* e = getenv("BD_SMALL_L");
    return e != nullptr && atoi(e) == 0;
  }();
  if (off) return false;
  static const int max_l_env = [] {  // BD_SMALL_MAXL: development A/B of the L range
    const char* e = getenv("BD_SMALL_MAXL");
    return e != nullptr ? atoi(e) : 5 * tc::BM;  // up to five 128-row blocks
  }();
  static const bool wide = [] {  // BD_SMALL_WIDE=1: pairs also for wide problems
    const char* e = getenv("BD_SMALL_WIDE");
    return e != nullptr && atoi(e) == 1;
  }();
  int64_t cols = 0, max_l = 0;
  for (int i = 0; i < count; ++i) {
    if (probs[i].L > max_l_env || probs[i].K > tc::SM_MAX_KB * tc::BK || probs[i].world > 0 ||
        probs[i].rep_gamma != nullptr)
      return false;
    cols += probs[i].N;
    max_l = probs[i].L > max_l ? probs[i].L : max_l;
  }
  // L > 128: only while the row blocks' CTAs fit one wave — wider or longer launches run
  // faster on the persistent kernel (measured: n = 128 heads, L = 256: 10.3 vs 8.6 us;
  // cfg2 L = 768: 9.2 vs 7.8 us)
  const int64_t nrb = (max_l + tc::BM - 1) / tc::BM;
  if (!wide && max_l > tc::BM && small_bns_one_wave(cols, nrb, tc::BM * tc::BK * 2) == 0)
    return false;
  return true;
}

#ifdef BD_WITH_DECODE_EXPERIMENT
// tools/experiments/kv_proj_decode_splitk.cu (development builds only, see its header)
bool decode_eligible(const Problem* probs, int count);
int launch_decode(const Problem* probs, int count, bool bf16, int* flag, cudaStream_t stream);
#endif

int launch_tc(const Problem* probs, int count, int dtype, int* flag, cudaStream_t stream) {
  using namespace tc;
  const bool bf16 = dtype == BD_BF16;
#ifdef BD_WITH_DECODE_EXPERIMENT
  if (decode_eligible(probs, count)) return launch_decode(probs, count, bf16, flag, stream);
#endif
  if (small_eligible(probs, count)) return launch_small(probs, count, bf16, flag, stream);
  TcParams prm;
  {
    const ParamKey key = make_key(probs, count, bf16);
    std::lock_guard<std::mutex> lock(g_param_mu);
    int hit = -1;
    for (int i = 0; i < kParamCacheSize; ++i)
      if (g_param_cache[i].valid && memcmp(&g_param_cache[i].key, &key, sizeof(key)) == 0) {
        hit = i;
        break;
      }
    if (hit >= 0) {
      prm = g_param_cache[hit].prm;
    } else {
      const int st = build_params(probs, count, bf16, prm, stream);
      if (st != BD_OK) return st;
      ParamEntry& e = g_param_cache[g_param_next];
      g_param_next = (g_param_next + 1) % kParamCacheSize;
      // An evicted all-gather entry's device copy of the peer maps is NOT freed: a CUDA
      // graph captured on a cache hit, or another thread that copied prm before the
      // eviction, may still launch with that pointer, and a freed-and-reused block would
      // turn its epilogue's peer TMA stores into writes through garbage descriptors.  The
      // blocks live for the process (count * world * 128 B per distinct buffer set).
      e.key = key;
      e.prm = prm;
      e.valid = true;
    }
  }
  prm.flag = flag;
  const int total = prm.total_tiles;
  if (total == 0) return BD_OK;
  return launch_params(prm, total, bf16, flag != nullptr, stream);
}

namespace {

int build_params(const Problem* probs, int count, bool bf16, tc::TcParams& prm,
                 cudaStream_t stream) {
  using namespace tc;
  constexpr int cg = CG;
  prm = TcParams{};
  CUtensorMap peer_host[BD_MAX_GROUP * BD_MAX_PEERS];
  prm.count = count;
  // Tile width: 128 when 256-wide tiles would not give every pair two tiles (short
  // launches on wide problems: one 256-wide tile per pair serialises its loads, MMAs and
  // epilogue; 128-wide tiles pipeline them and balance better).  Streaming-A, fused-norm
  // and fused-all-gather launches keep 256.  BD_TILE_N=128|256 forces a width (A/B).
  static const int tile_env = [] {
    const char* e = getenv("BD_TILE_N");
    return e != nullptr ? atoi(e) : 0;
  }();
  int bn = BN;
  {
    int64_t t256 = 0;
    bool plain = true;
    for (int i = 0; i < count; ++i) {
      const Problem& q = probs[i];
      t256 += ((q.N + BN - 1) / BN) * ((q.L + BM * cg - 1) / (BM * cg));
      plain = plain && q.rep_gamma == nullptr && q.world == 0 && (q.K + BK - 1) / BK <= A_SLOTS;
    }
    if (plain && (tile_env == 128 || (tile_env != 256 && t256 < 2 * (sm_count() / cg)))) bn = 128;
  }
  prm.bn = bn;
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
        !encode_2d(&P.map_b, q.c, bf16, N, K, q.ldc, 64, BKB, &err) ||
        !(q.out_layout == BD_OUT_HEAD_MAJOR
              ? encode_3d(&P.map_out, q.out, bf16, q.d_h, q.L, N / q.d_h, q.ldo, q.L * q.ldo, 64,
                          32, &err)
              : encode_2d(&P.map_out, q.out, bf16, N, q.L, q.ldo, 64, 32, &err)) ||
        (rep_fast && !encode_2d(&P.map_rep, xr, bf16, d_h, q.L, q.ldx, 64, BM, &err))) {
      set_error(err);
      return BD_ERR_CUDA;
    }
    P.rep_fast = rep_fast ? 1 : 0;
    P.has_rep = has_rep ? 1 : 0;
    P.head_major = q.out_layout == BD_OUT_HEAD_MAJOR ? 1 : 0;
    if (q.rep_gamma != nullptr) {
      // fused RMSNorm: the row must be resident (A k-blocks + staged rep = all d columns)
      if (!rep_fast || K > A_SLOTS * BK) {
        set_error("fused RMSNorm needs d_h in {64, 128} and d - d_h <= 384 on the tensor-core path");
        return BD_ERR_SHAPE;
      }
      prm.norm = 1;
      P.rep_gamma = q.rep_gamma;
      P.norm_eps = q.norm_eps;
      P.norm_d = static_cast<int32_t>(K + d_h);
    }
    if (q.world > 0) {
      prm.world = q.world;
      prm.head0[i] = q.head0;
      for (int r = 0; r < q.world; ++r)
        if (!encode_3d(&peer_host[i * q.world + r], q.peers[r], bf16, q.d_h, q.L,
                       static_cast<uint64_t>(q.world) * (N / q.d_h), q.ldo, q.L * q.ldo, 64, 32,
                       &err)) {
          set_error(err);
          return BD_ERR_CUDA;
        }
    }
    P.out_d_h = static_cast<int32_t>(q.d_h);
    P.x = q.x;
    P.ldx = q.ldx;
    P.L = static_cast<int32_t>(q.L);
    P.N = static_cast<int32_t>(N);
    P.K = static_cast<int32_t>(K);
    P.d_h = static_cast<int32_t>(d_h);
    P.rep_base = static_cast<int32_t>(rep_base);
    P.tiles_n = static_cast<int32_t>((N + bn - 1) / bn);
    P.tiles_m = static_cast<int32_t>((q.L + BM * cg - 1) / (BM * cg));
    P.num_kb = static_cast<int32_t>((K + BK - 1) / BK);
    P.num_kbb = static_cast<int32_t>((K + BKB - 1) / BKB);
    P.tile_start = total;
    total += P.tiles_n * static_cast<int32_t>((q.L + BM * cg - 1) / (BM * cg));
  }
  prm.total_tiles = total;
  for (int i = 0; i < count; ++i)
    if (prm.p[i].num_kb > A_SLOTS) prm.strided = 1;
  // Mirror schedule (coefficients resident, x streamed) when every problem is a single
  // 256-wide column tile: the row-block-major schedule would reload a 96 KiB A
  // row-block for every tile (head-sharded weak scaling at 2 + 2 heads per GPU).
  // BD_SWAP=0|1 forces it off / on where legal (A/B).
  {
    static const int swap_env = [] {
      const char* e = getenv("BD_SWAP");
      return e != nullptr ? atoi(e) : -1;
    }();
    bool legal = bn == BN && !prm.strided && !prm.norm && prm.world == 0;
    bool narrow = true;
    for (int i = 0; i < count; ++i) narrow = narrow && prm.p[i].tiles_n == 1;
    prm.swap = legal && (swap_env == 1 || (swap_env != 0 && narrow)) ? 1 : 0;
  }
  if (prm.world > 0) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cap);
    if (cap != cudaStreamCaptureStatusNone) {
      set_error("fused all-gather: the first call with a given set of buffers must run "
                "outside stream capture (its peer tensor maps are uploaded then)");
      return BD_ERR_ARG;
    }
    const size_t bytes = sizeof(CUtensorMap) * static_cast<size_t>(count) * prm.world;
    void* dev = nullptr;
    cudaError_t e = cudaMalloc(&dev, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(dev, peer_host, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      if (dev) cudaFree(dev);
      set_error(std::string("fused all-gather tensor maps: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    prm.peer_maps = static_cast<const CUtensorMap*>(dev);
  }
  return BD_OK;
}

int launch_params(const tc::TcParams& prm, int total, bool bf16, bool check,
                  cudaStream_t stream) {
  using namespace tc;
  constexpr int cg = CG;
  using KernFn = void (*)(TcParams);
  static const KernFn kerns[2][2][2] = {
      {{kv_proj_tc_kernel<false, false, false>, kv_proj_tc_kernel<false, false, true>},
       {kv_proj_tc_kernel<false, true, false>, kv_proj_tc_kernel<false, true, true>}},
      {{kv_proj_tc_kernel<true, false, false>, kv_proj_tc_kernel<true, false, true>},
       {kv_proj_tc_kernel<true, true, false>, kv_proj_tc_kernel<true, true, true>}}};
  static const KernFn kerns_norm[2][2] = {
      {kv_proj_tc_kernel<false, false, false, true>, kv_proj_tc_kernel<false, true, false, true>},
      {kv_proj_tc_kernel<true, false, false, true>, kv_proj_tc_kernel<true, true, false, true>}};
  static const KernFn kerns_swap[2][2] = {
      {kv_proj_tc_kernel<false, false, false, false, BN, true>,
       kv_proj_tc_kernel<false, true, false, false, BN, true>},
      {kv_proj_tc_kernel<true, false, false, false, BN, true>,
       kv_proj_tc_kernel<true, true, false, false, BN, true>}};
  static const KernFn kerns_128[2][2] = {
      {kv_proj_tc_kernel<false, false, false, false, 128>,
       kv_proj_tc_kernel<false, true, false, false, 128>},
      {kv_proj_tc_kernel<true, false, false, false, 128>,
       kv_proj_tc_kernel<true, true, false, false, 128>}};
  const int vb = bf16 ? 1 : 0, vc = check ? 1 : 0;
  const int vr = prm.swap ? 4 : prm.bn == 128 ? 3 : prm.norm ? 2 : (prm.strided ? 1 : 0);
  KernFn kern = vr == 4   ? kerns_swap[vb][vc]
                : vr == 3 ? kerns_128[vb][vc]
                : vr == 2 ? kerns_norm[vb][vc]
                          : kerns[vb][vc][vr];
  const size_t smem = SMEM_BYTES;
  static std::atomic<bool> attr_set[kMaxDevices][2][2][5] = {};  // per device (see launch_small)
  static std::mutex attr_mu;
  const int dv = device_slot();
  if (!attr_set[dv][vb][vc][vr].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(attr_mu);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_set[dv][vb][vc][vr].store(true, std::memory_order_release);
  }
  const int units = sm_count() / cg;
  const int grid_units = total < units ? total : units;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_units * cg);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  static const bool pdl = [] {  // BD_PDL=0 disables programmatic dependent launch
    const char* e = getenv("BD_PDL");
    return !(e && atoi(e) == 0);
  }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm);
  note_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("kv_proj_tc launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

}  // namespace

}  // namespace bdk
