// kv_proj_decode_splitk.cu — EXPERIMENT (not in the product library; built only by
// tools/build_variant.sh with WITH_DECODE=1, which defines BD_WITH_DECODE_EXPERIMENT).
// A decode-sized (L <= 128 tokens) BD K/V projection: split-K over a thread-block
// cluster, partial sums reduced through distributed shared memory.
//
// RESULT (round 2, tools/decode_sweep.sh, cold-L2 ring, CUDA graph, FP16): parity-green
// on every split (kps 1..6: oracle bound, grouped == separate, head shards, head-major)
// but SLOWER than the shipped small-L kernel everywhere.  With one CTA per column block
// (kps = 6) it ties on cfg2 (4.00 vs 3.96 us at L = 1) and loses on the paper shape
// (6.34 vs 5.12: 128-column blocks at 118 KB cannot co-reside); every split loses more
// the more CTAs it launches (paper L = 1: 13.0 us at 256 CTAs in clusters of 2, 18.3 us
// at 384 in clusters of 3; cfg2 L = 128: 6.0 / 7.4 us), i.e. ~50 ns per extra CTA.
// The first version's fully unrolled epilogue (5-9 k SASS instructions) was another
// 2x: each SM runs the code once per launch, so instruction-cache misses dominate
// (ncu: gcc instruction requests 3x, sm__cycles_active 2.2x the small-L kernel's).
//
//   out[i, h*d_h + j] = sum_k x[i, mul_base + k] * c[k, h*d_h + j]  +  x[i, rep_base + j]
//
// (ref: pkg/src/bdattn/attention.py:249-270 computes the same thing on the CPU.)
//
// Why it was tried.  At decode sizes the step is latency, not arithmetic or bytes
// (tools/decode_floor.cu, tools/small_timeline2.py on the stamped small-L kernel, round 2):
//   * a CUDA graph of dependent launches pays ~1.4 us from the last CTA's end to the
//     next launch's griddepcontrol.wait release, whatever the kernel does;
//   * one CTA's chain of 24 dependent tcgen05.mma (K = 384, M = 128, N = 64) takes
//     ~1450 clocks (tools/mma_latency.cu: ~50 clocks per MMA + ~350 of pipeline depth),
//     and while the MMAs read shared memory the same SM's TMA loads slow down — removing
//     the MMAs from the small-L kernel saved 1.0 us of its 4.0;
//   * a CTA whose shared-memory footprint forbids a second resident CTA cannot run its
//     prologue under the previous launch.
// So each output column block is computed by a CLUSTER of CTAs that split the
// contraction: with kps k-blocks of 64 per CTA (default 2; bd_set_decode_kblocks), a
// problem with num_kb k-blocks uses S_p = ceil(num_kb / kps) CTAs; CTA s loads x[:, its K
// slice] and c[its K slice, block], runs its own short MMA chain into TMEM (cta_group::1,
// M = 128 rows, N = BNS columns, FP32), and the S_p partial sums meet in shared memory:
// the rows are split S_p ways, each row's owner receives the other S_p - 1 partial rows
// with st.async (remote shared-memory stores that complete on the owner's mbarrier — no
// cluster-wide barrier), adds them in the fixed order s = 0, 1, ..., S_p - 1, then adds
// the repeated slice with one mixed-precision FHADD per element (after the full K sum, as
// the reference does), rounds once to 16 bit and stores.  The K partition depends on K
// alone, so every output bit is independent of N, of the grouping and of head sharding
// (the invariants tests/test_kv_proj_gpu.py checks).  The footprint stays small (<= ~90
// KB), so the next launch's CTAs become resident and finish their prologue — barrier
// init, TMEM allocation, an L2 prefetch of their slice of c — while this launch runs
// (programmatic dependent launch).  c is read exactly once per launch; x (<= 96 KB at L =
// 128) is re-read from L2 by every column block.
//
// With kps >= num_kb (one CTA) the MMA sequence — k ascending in 16-deep steps into one
// FP32 accumulator — is the persistent kernel's, so outputs are bit-identical to it; with
// S_p > 1 the K sum is S_p partial tensor-core sums added in FP32: within the FP16/BF16
// bounds of tests/test_kv_proj_gpu.py, not bit-identical to the persistent kernel.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2-5 epilogue (warp w owns TMEM lanes / rows 32 (w % 4) .. + 31).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kv_proj_internal.h"
#include "ptx_sm100.cuh"
#include "tc_common.cuh"

namespace bdk {
namespace tc {

constexpr int DK_THREADS = 192;
constexpr int DK_MAX_KB = 6;                  // K <= 384 (num_kb k-blocks of 64)
constexpr uint32_t DK_A_FULL = 128 * 128;     // one 128-row x 64-k A block (what the MMA reads)
constexpr uint32_t DK_B_PANEL = 64 * 64 * 2;  // 64 k x 64 columns, MN-major SW128

// st.async: 16 bytes into CTA-remote shared memory, completing tx bytes on the remote
// CTA's mbarrier (both operands are shared::cluster addresses).
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          raddr),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
      : "memory");
}

// Decode launch geometry.  Problem p's contraction (num_kb k-blocks of 64) is split over
// S_p = ceil(num_kb / kps) CTAs — rank s takes k-blocks [s kps, min(num_kb, (s+1) kps)) —
// so the K partition, and with it every output bit, depends only on K (not on N, the
// grouping or the other problems of the launch).  The cluster has S = max_p S_p CTAs;
// ranks >= S_p of a smaller problem's cluster sit the launch out.
__host__ __device__ inline int decode_split(int num_kb, int kps) { return (num_kb + kps - 1) / kps; }

// One cluster per BNS-column block of one problem.
template <bool kBF16, bool kCheck, int BNS>
__global__ void __launch_bounds__(DK_THREADS, 1)
    kv_proj_decode_kernel(const __grid_constant__ TcParams prm, int S) {
  constexpr int PANELS = BNS / 64;
  constexpr int CHUNKS = BNS / 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int rank = S > 1 ? static_cast<int>(cluster_ctarank()) : 0;

  int pi = 0;
  const int blk = static_cast<int>(blockIdx.x) / S;
  while (pi + 1 < prm.count && blk >= prm.p[pi + 1].tile_start) ++pi;
  const TcProblem& P = prm.p[pi];
  const int n0 = (blk - P.tile_start) * BNS;
  const int L = P.L;
  const int kps = prm.dk_kps;
  const int Sp = decode_split(P.num_kb, kps);  // CTAs that share this problem's K
  const int kb0 = rank * kps;
  const int nk = P.num_kb - kb0 < kps ? P.num_kb - kb0 : kps;  // this CTA's k-blocks
  const bool active = rank < Sp;
  const uint32_t a_kb = static_cast<uint32_t>(prm.a_kb_bytes);
  uint8_t* sA = smem;
  uint8_t* sB = sA + prm.dk_a_bytes;
  uint8_t* sRecv = sB + prm.dk_b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sRecv + prm.dk_recv_bytes);
  uint64_t* done = full + DK_MAX_KB;
  uint64_t* recv = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv + 1);
  const int rows_per = (L + Sp - 1) / Sp;  // rows [s rows_per, (s+1) rows_per) end at rank s

  if (active && warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) mbar_init(&full[kb], 1);
    mbar_init(done, 1);
    mbar_init(recv, 1);
    fence_mbar_init();
    if (Sp > 1) {  // the partial rows this CTA receives: its live rows x (Sp - 1) x BNS FP32
      const int lo = rank * rows_per;
      const int hi = lo + rows_per < L ? lo + rows_per : L;
      const int mine = hi > lo ? hi - lo : 0;
      mbar_arrive_expect_tx(recv, static_cast<uint32_t>(mine * (Sp - 1) * BNS * 4));
    }
  }
  if (active && warp == 1) {
    tmem_alloc<1>(tmem_slot, BNS);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  if (S > 1)
    cluster_sync_relaxed();  // every CTA's recv barrier exists before any st.async
  else
    __syncthreads();
  tc_fence_after();
  griddep_launch_dependents();
  if (!active) return;  // a smaller problem's cluster: nothing to contract
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---- producer: all of this CTA's k-blocks at once, one barrier each
    if (elect_one()) {
      tma_prefetch_desc(&P.map_a);
      tma_prefetch_desc(&P.map_b);
      // This CTA's slice of c into L2 before the PDL wait.  L2 is the point of coherence,
      // so the prefetch cannot return stale data even if the previous kernel wrote c; it
      // only moves the DRAM read of the weights under the previous launch's tail.  x,
      // which the previous kernel may produce, is read only after the wait.
      for (int kb = 0; kb < nk; ++kb)
        for (int q = 0; q < PANELS; ++q)
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                           reinterpret_cast<uint64_t>(&P.map_b)),
                       "r"(n0 + 64 * q), "r"((kb0 + kb) * 64)
                       : "memory");
    }
    __syncwarp();
    griddep_wait();
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();
      for (int kb = 0; kb < nk; ++kb) {
        mbar_arrive_expect_tx(&full[kb], a_kb + PANELS * DK_B_PANEL);
        tma_load_2d(sA + kb * a_kb, &P.map_a, (kb0 + kb) * 64, 0, &full[kb], pol);
#pragma unroll
        for (int q = 0; q < PANELS; ++q)
          tma_load_2d(sB + (kb * PANELS + q) * DK_B_PANEL, &P.map_b, n0 + 64 * q, (kb0 + kb) * 64,
                      &full[kb], pol);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA: M = 128 (rows >= L are never stored), N = BNS, k ascending
    constexpr uint32_t idesc = make_idesc_f16(kBF16, 128, BNS, /*a_mn=*/false, /*b_mn=*/true);
    for (int kb = 0; kb < nk; ++kb) {
      mbar_wait(&full[kb], 0);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a0 = smem_u32(sA + kb * a_kb);
        const uint32_t b0 = smem_u32(sB + kb * PANELS * DK_B_PANEL);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          tc_mma_f16(tmem_base, make_smem_desc(a0 + ks * 32, 16, 1024),
                     make_smem_desc(b0 + ks * 2048, DK_B_PANEL, 1024), idesc,
                     (kb | ks) != 0 ? 1u : 0u);
        if (kb + 1 == nk) tc_commit(done);
      }
      __syncwarp();
    }
  } else {
    // ---- epilogue: thread = row r of the block (its TMEM lane).  Kept compact (rolled
    // loops over 32-column chunks and over the split): each SM runs this code once per
    // launch, so instruction-cache misses, not issue slots, are what an unrolled epilogue
    // would cost.
    const uint32_t quad = warp & 3;
    const int r = static_cast<int>(quad * 32 + lane);
    const bool live = r < L;
    const int owner = r / rows_per;
    const int lr = r - owner * rows_per;
    const bool mine = live && owner == rank;
    const uint32_t taddr = tmem_base + ((quad * 32u) << 16);
    const int N = P.N, out_d_h = P.out_d_h;
    const int64_t ldo = P.ldo;
    const bool head_major = P.head_major != 0;
    uint16_t* const out = static_cast<uint16_t*>(P.out);
    uint32_t chk = 0u;
    // the repeated slice (x, which the previous kernel may write): the owner's row only,
    // fetched before the MMAs finish; xr[0..3] always holds the current chunk's columns
    uint4 xr[BNS / 8];
    griddep_wait();
    if (mine) {
      const uint16_t* xrow = static_cast<const uint16_t*>(P.x) + static_cast<int64_t>(r) * P.ldx +
                             P.rep_base;
      const int d_h = P.d_h;
      const bool has_rep = P.has_rep != 0;
      int jj = n0 % d_h;  // rep column of col = n0 + 8 j, advanced by 8 mod d_h (d_h >= 8)
#pragma unroll
      for (int j = 0; j < BNS / 8; ++j) {
        const int col = n0 + 8 * j;
        xr[j] = (has_rep && col < N) ? __ldg(reinterpret_cast<const uint4*>(xrow + jj))
                                     : make_uint4(0, 0, 0, 0);
        jj += 8;
        jj = jj >= d_h ? jj - d_h : jj;
      }
    }
    mbar_wait(done, 0);
    tc_fence_after();
    // tcgen05.ld is warp-collective (.sync.aligned): every lane of the warp loads, each
    // lane then acts on its own row's role
    if (__any_sync(0xffffffffu, live && !mine)) {
      // senders: a row's partial sums go to its owner's receive slot; 16-byte groups
      // XOR-swizzled by the owner's row index (conflict-free reads there)
      const bool send = live && !mine;
      const uint32_t dst = send ? static_cast<uint32_t>(owner) : static_cast<uint32_t>(rank);
      const uint32_t slot = static_cast<uint32_t>(rank < owner ? rank : rank - 1);
      const uint32_t rbase = mapa_shared(
          smem_u32(sRecv) + (slot * static_cast<uint32_t>(rows_per) + lr) * (BNS * 4), dst);
      const uint32_t rbar = mapa_shared(smem_u32(recv), dst);
      const uint32_t swz = static_cast<uint32_t>(lr & 7);
#pragma unroll 1
      for (int c = 0; c < CHUNKS; ++c) {
        uint32_t v[32];
        __syncwarp();  // converged for the warp-collective load
        tmem_ld_32x32b_x32(taddr + c * 32, v);
        tmem_ld_wait();
        if (send) {
#pragma unroll
          for (int g = 0; g < 8; ++g)
            st_async_v4(rbase + ((static_cast<uint32_t>(c * 8 + g) ^ swz) << 4),
                        make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]), rbar);
        }
      }
    }
    if (__any_sync(0xffffffffu, mine)) {
      if (mine && Sp > 1) mbar_wait(recv, 0);
      const float* rrow = reinterpret_cast<const float*>(sRecv) + lr * BNS;
      const uint32_t swz = static_cast<uint32_t>(lr & 7);
      uint16_t* orow = out + static_cast<int64_t>(r) * ldo;  // token-major row
#pragma unroll 1
      for (int c = 0; c < CHUNKS; ++c) {
        uint32_t v[32];
        __syncwarp();  // converged for the warp-collective load
        tmem_ld_32x32b_x32(taddr + c * 32, v);
        tmem_ld_wait();
        if (mine) {
          // the K sum of this chunk: partial s = 0, + s = 1, ... (fixed order)
          float acc[32];
#pragma unroll 1
          for (int s = 0; s < Sp; ++s) {
            float t[32];
            if (s == rank) {
#pragma unroll
              for (int i = 0; i < 32; ++i) t[i] = __uint_as_float(v[i]);
            } else {
              const float* src = rrow + (s < rank ? s : s - 1) * rows_per * BNS;
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                const float4 q =
                    *reinterpret_cast<const float4*>(src + ((static_cast<uint32_t>(c * 8 + g) ^ swz) << 2));
                t[4 * g] = q.x;
                t[4 * g + 1] = q.y;
                t[4 * g + 2] = q.z;
                t[4 * g + 3] = q.w;
              }
            }
            if (s == 0) {
#pragma unroll
              for (int i = 0; i < 32; ++i) acc[i] = t[i];
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) acc[i] += t[i];
            }
          }
          // + rep after the full K sum: one FHADD per element (exact widening, one FP32
          // rounding), then one rounding to 16 bit — the persistent kernel's epilogue
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int col = n0 + c * 32 + 8 * h;
            const uint32_t xw[4] = {xr[h].x, xr[h].y, xr[h].z, xr[h].w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 t2 = add_f32_x16x2<kBF16>(acc[8 * h + 2 * e], acc[8 * h + 2 * e + 1], xw[e]);
              o[e] = pack2<kBF16>(t2.x, t2.y);
              if constexpr (kCheck) {
                if (col < N) chk = max_abs2_nan<kBF16>(chk, o[e]);
              }
            }
            if (col < N) {
              uint16_t* dstp;
              if (head_major) {
                const int hd = col / out_d_h;
                dstp = out + (static_cast<int64_t>(hd) * L + r) * ldo + (col - hd * out_d_h);
              } else {
                dstp = orow + col;
              }
              *reinterpret_cast<uint4*>(dstp) = make_uint4(o[0], o[1], o[2], o[3]);
            }
          }
        }
        // the next chunk's rep values move into xr[0..3]
#pragma unroll
        for (int j = 0; j + 4 < BNS / 8; ++j) xr[j] = xr[j + 4];
      }
    }
    if constexpr (kCheck) {
      if (__any_sync(0xffffffffu, nonfinite2<kBF16>(chk)) && lane == 0) atomicExch(prm.flag, 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, BNS);
  }
}

}  // namespace tc

namespace {

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e != nullptr ? atoi(e) : dflt;
}

std::atomic<int> g_decode_kps{0};  // 0: automatic (bd_set_decode_kblocks)

}  // namespace

// Problems the decode kernel serves: L <= 128 (one 128-row block), K <= 384 (every
// k-block of a CTA resident), 16-byte aligned rows / columns for the direct stores and
// the repeated-slice loads, no fused all-gather or norm.
bool decode_eligible(const Problem* probs, int count) {
  static const bool off = env_int("BD_DECODE", 1) == 0;  // BD_DECODE=0: small-L kernel
  if (off) return false;
  for (int i = 0; i < count; ++i) {
    const Problem& q = probs[i];
    if (q.L > 128 || q.L < 1 || q.K < 1 || q.K > 64 * tc::DK_MAX_KB || q.world > 0 ||
        q.rep_gamma != nullptr || q.N % 8 != 0 || q.ldo % 8 != 0 ||
        (q.rep_base >= 0 && (q.d_h % 8 != 0 || q.ldx % 8 != 0 || q.rep_base % 8 != 0)))
      return false;
  }
  return count > 0;
}

extern "C" int bd_set_decode_kblocks(int kps) {
  if (kps < 0 || kps > tc::DK_MAX_KB) return BD_ERR_ARG;
  g_decode_kps.store(kps);
  return BD_OK;
}

int launch_decode(const Problem* probs, int count, bool bf16, int* flag, cudaStream_t stream) {
  using namespace tc;
  int64_t max_l = 1;
  for (int i = 0; i < count; ++i) max_l = probs[i].L > max_l ? probs[i].L : max_l;
  auto blocks_for = [&](int bns) {
    int64_t b = 0;
    for (int i = 0; i < count; ++i) b += (probs[i].N + bns - 1) / bns;
    return b;
  };
  // Column block: 128 (the cheapest MMA width per column) while that still gives at least
  // one block per two SMs, else 64.  Tiling does not change any output bit.
  const int sms = sm_count();
  int bns = env_int("BD_DECODE_BNS", 0);
  if (bns != 64 && bns != 128) bns = blocks_for(128) >= sms / 2 ? 128 : 64;
  // k-blocks per CTA: fixed per process (default 2), so outputs depend on K only
  int kps = g_decode_kps.load();
  if (kps == 0) kps = env_int("BD_DECODE_KPS", 2);
  if (kps < 1 || kps > DK_MAX_KB) kps = 2;
  int S = 1;
  uint32_t recv = 0;
  for (int i = 0; i < count; ++i) {
    const int nkb = static_cast<int>((probs[i].K + 63) / 64);
    const int sp = decode_split(nkb, kps);
    S = sp > S ? sp : S;
    const int rows_per = static_cast<int>((probs[i].L + sp - 1) / sp);
    const uint32_t rb = sp > 1 ? static_cast<uint32_t>((sp - 1) * rows_per * bns * 4) : 0u;
    recv = rb > recv ? rb : recv;
  }
  const int a_rows = static_cast<int>((max_l + 7) / 8 * 8);
  const uint32_t a_kb = static_cast<uint32_t>(a_rows) * 128u;
  // the MMA reads 128 rows of the last k-block: keep that read inside the allocation
  const uint32_t a_bytes = ((kps - 1) * a_kb + DK_A_FULL + 1023u) & ~1023u;
  const uint32_t b_bytes = static_cast<uint32_t>(kps * (bns / 64)) * DK_B_PANEL;
  const size_t smem = 1024 + a_bytes + b_bytes + recv + 256;
  if (smem > 232448) {
    set_error("decode kernel: shared-memory footprint too large");
    return BD_ERR_ARG;
  }
  TcParams prm{};
  prm.count = count;
  prm.flag = flag;
  prm.a_kb_bytes = static_cast<int32_t>(a_kb);
  prm.dk_kps = kps;
  prm.dk_a_bytes = static_cast<int32_t>(a_bytes);
  prm.dk_b_bytes = static_cast<int32_t>(b_bytes);
  prm.dk_recv_bytes = static_cast<int32_t>(recv);
  int total = 0;
  for (int i = 0; i < count; ++i) {
    const Problem& q = probs[i];
    TcProblem& P = prm.p[i];
    std::string err;
    const bool has_rep = q.rep_base >= 0;
    const auto* xb = static_cast<const uint16_t*>(q.x) + q.mul_base;
    if (!encode_2d(&P.map_a, xb, bf16, q.K, q.L, q.ldx, 64, static_cast<uint32_t>(a_rows), &err) ||
        !encode_2d(&P.map_b, q.c, bf16, q.N, q.K, q.ldc, 64, 64, &err)) {
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
    P.tiles_n = static_cast<int32_t>((q.N + bns - 1) / bns);
    P.tile_start = total;
    total += P.tiles_n;
  }
  if (total == 0) return BD_OK;
  using KernFn = void (*)(TcParams, int);
  static const KernFn kerns[2][2][2] = {
      {{kv_proj_decode_kernel<false, false, 64>, kv_proj_decode_kernel<false, false, 128>},
       {kv_proj_decode_kernel<false, true, 64>, kv_proj_decode_kernel<false, true, 128>}},
      {{kv_proj_decode_kernel<true, false, 64>, kv_proj_decode_kernel<true, false, 128>},
       {kv_proj_decode_kernel<true, true, 64>, kv_proj_decode_kernel<true, true, 128>}}};
  const int vb = bf16 ? 1 : 0, vc = flag != nullptr ? 1 : 0, vn = bns == 128 ? 1 : 0;
  const KernFn kern = kerns[vb][vc][vn];
  // per device ordinal: the attribute belongs to the function in the current context
  static std::atomic<bool> attr_done[kMaxDevices][2][2][2] = {};
  static std::mutex attr_mu;
  const int dv = device_slot();
  if (!attr_done[dv][vb][vc][vn].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(attr_mu);
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return BD_ERR_CUDA;
    }
    attr_done[dv][vb][vc][vn].store(true, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(total * S));
  cfg.blockDim = dim3(DK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = static_cast<unsigned>(S);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = S > 1 ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm, S);
  note_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("kv_proj_decode launch: ") + cudaGetErrorString(e));
    return BD_ERR_CUDA;
  }
  return BD_OK;
}

}  // namespace bdk
