// kv_proj_exact.cu — FP32/FP64 BD K/V projection in the reference's exact rounding order.
//
// The reference kernel (ref: pkg/src/bdattn/attention.py:249-270) computes, per output
// element, acc = 0; for k ascending: acc = fl(acc + fl(x[i, mul_base+k] * c[k, j]));
// then out = fl(acc + x[i, rep_base + j % d_h]).  numba compiles it without fast-math,
// so no FMA contraction happens.  This kernel reproduces that sequence with
// __fmul_rn/__fadd_rn (never contracted), so its output is bit-identical to the
// reference for every shape — including the tiny odd shapes of the reference tests
// (d=13, d_h=4, n=3; test_attention.py:187-203) that the tensor-core path cannot take.
//
// Tiling is for data reuse only: a 64x64 output tile per 256-thread CTA, k-slabs of
// 16 staged through shared memory, 4x4 outputs per thread.  The per-element
// reduction order is untouched by the tiling, which is also why column-sharding the
// output across GPUs is bit-invariant (ref test_tensor.py:113-119).
#include <cuda_runtime.h>

#include <cstdint>

#include "kv_proj_internal.h"

namespace bdk {
namespace {

// Tile T x T (T = 64, or 32 when 64-tiles would leave most SMs idle), 4 x 4 outputs per
// thread, k-slabs of EX_BK through shared memory.
constexpr int EX_BK = 16;

template <typename T>
struct ExactOps;
template <>
struct ExactOps<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
template <>
struct ExactOps<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};

struct ExactGroup {
  Problem p[BD_MAX_GROUP];
  int tiles_n[BD_MAX_GROUP];
  int tile_start[BD_MAX_GROUP + 1];
  int count;
};

template <typename T, int TILE>
__global__ void __launch_bounds__((TILE / 4) * (TILE / 4))
    kv_proj_exact_kernel(const __grid_constant__ ExactGroup g, int* flag) {
  constexpr int EX_BM = TILE, EX_BN = TILE, EX_THREADS = (TILE / 4) * (TILE / 4);
  constexpr int GROUPS = TILE / 4;
  // Locate the problem and the 64x64 tile this CTA owns.
  int t = blockIdx.x;
  int pi = 0;
  while (pi + 1 < g.count && t >= g.tile_start[pi + 1]) ++pi;
  const Problem& P = g.p[pi];
  const int local = t - g.tile_start[pi];
  const int tn = local % g.tiles_n[pi];
  const int tm = local / g.tiles_n[pi];
  const int64_t m0 = static_cast<int64_t>(tm) * EX_BM;
  const int64_t n0 = static_cast<int64_t>(tn) * EX_BN;

  const T* __restrict__ x = static_cast<const T*>(P.x);
  const T* __restrict__ c = static_cast<const T*>(P.c);
  T* __restrict__ out = static_cast<T*>(P.out);
  const int64_t K = P.K;
  const int64_t N = P.N;

  __shared__ T xs[EX_BK][EX_BM];  // x slab, k-major so a thread's 4 rows are contiguous
  __shared__ T cs[EX_BK][EX_BN];

  const int tx = threadIdx.x % GROUPS;  // column group
  const int ty = threadIdx.x / GROUPS;  // row group
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

  // Slabs of x[m0 : m0 + T, mul_base + k0 : + EX_BK] and c[k0 : k0 + EX_BK, n0 : n0 + T]
  // (zero-filled outside the problem; padded entries are never folded into acc, see
  // kmax) staged through shared memory; the next slab's global loads are in flight in
  // registers while the current one is consumed.
  constexpr int XL = EX_BM * EX_BK / EX_THREADS;
  constexpr int CL = EX_BN * EX_BK / EX_THREADS;
  T xr[XL], cr[CL];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < XL; ++u) {
      const int e = threadIdx.x + u * EX_THREADS;
      const int r = e / EX_BK, kk = e % EX_BK;
      const int64_t row = m0 + r, col = k0 + kk;
      xr[u] = (row < P.L && col < K) ? x[row * P.ldx + P.mul_base + col] : T(0);
    }
#pragma unroll
    for (int u = 0; u < CL; ++u) {
      const int e = threadIdx.x + u * EX_THREADS;
      const int kk = e / EX_BN, cc = e % EX_BN;
      const int64_t krow = k0 + kk, col = n0 + cc;
      cr[u] = (krow < K && col < N) ? c[krow * P.ldc + col] : T(0);
    }
  };
  auto step = [&](int kk) {  // k ascending: the reference's order
    T a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = xs[kk][ty * 4 + i];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = cs[kk][tx * 4 + j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        acc[i][j] = ExactOps<T>::add(acc[i][j], ExactOps<T>::mul(a[i], b[j]));
  };
  fetch(0);
  for (int64_t k0 = 0; k0 < K; k0 += EX_BK) {
#pragma unroll
    for (int u = 0; u < XL; ++u) {
      const int e = threadIdx.x + u * EX_THREADS;
      xs[e % EX_BK][e / EX_BK] = xr[u];
    }
#pragma unroll
    for (int u = 0; u < CL; ++u) {
      const int e = threadIdx.x + u * EX_THREADS;
      cs[e / EX_BN][e % EX_BN] = cr[u];
    }
    __syncthreads();
    if (k0 + EX_BK < K) fetch(k0 + EX_BK);
    const int kmax = static_cast<int>((K - k0) < EX_BK ? (K - k0) : EX_BK);
    if (kmax == EX_BK) {
#pragma unroll
      for (int kk = 0; kk < EX_BK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kmax; ++kk) step(kk);
    }
    __syncthreads();
  }

  // Epilogue: + the repeated basis slice, after the full sum (attention.py:266-270).
  // Without it (rep_base < 0) this is the reference's fixed-order matmul
  // (tensor.py:189-213), used by the BD low-rank layer.
  const bool has_rep = P.rep_base >= 0;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + ty * 4 + i;
    if (row >= P.L) continue;
    // fused RMSNorm: r = 1 / sqrt(mean(x[row, 0:d]^2) + eps), d = K + d_h (the multiplied
    // and repeated slices partition the row); out = r * (acc + gamma_rep * x_rep)
    T rn = T(1);
    if (P.rep_gamma != nullptr) {
      T ss = T(0);
      const int64_t dfull = K + P.d_h;
      for (int64_t k = 0; k < dfull; ++k) {
        const T xv = x[row * P.ldx + k];
        ss = ExactOps<T>::add(ss, ExactOps<T>::mul(xv, xv));
      }
      rn = T(1) / sqrt(ss / static_cast<T>(dfull) + static_cast<T>(P.norm_eps));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + tx * 4 + j;
      if (col >= N) continue;
      T v;
      if (P.rep_gamma != nullptr) {
        const T xr = x[row * P.ldx + P.rep_base + (col % P.d_h)];
        v = ExactOps<T>::mul(
            rn, ExactOps<T>::add(acc[i][j],
                                 ExactOps<T>::mul(static_cast<T>(P.rep_gamma[col % P.d_h]), xr)));
      } else {
        v = has_rep ? ExactOps<T>::add(acc[i][j], x[row * P.ldx + P.rep_base + (col % P.d_h)])
                    : acc[i][j];
      }
      if (P.world > 0) {  // fused all-gather: every rank's full-width head-major buffer
        const int64_t off = ((P.head0 + col / P.d_h) * P.L + row) * P.ldo + col % P.d_h;
        for (int r = 0; r < P.world; ++r) static_cast<T*>(P.peers[r])[off] = v;
      } else if (P.out_layout == BD_OUT_HEAD_MAJOR) {
        out[((col / P.d_h) * P.L + row) * P.ldo + col % P.d_h] = v;
      } else {
        out[row * P.ldo + col] = v;
      }
      bad |= !isfinite(v);
    }
  }
  if (flag != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
    atomicExch(flag, 1);
  }
}

}  // namespace

cudaError_t launch_exact(const Problem* probs, int count, int dtype, int* flag,
                         cudaStream_t stream) {
  auto tiles = [&](int t, ExactGroup& g) {
    g = ExactGroup{};
    g.count = count;
    int total = 0;
    for (int i = 0; i < count; ++i) {
      g.p[i] = probs[i];
      const int64_t tn = (probs[i].N + t - 1) / t;
      const int64_t tm = (probs[i].L + t - 1) / t;
      g.tiles_n[i] = static_cast<int>(tn);
      g.tile_start[i] = total;
      total += static_cast<int>(tn * tm);
    }
    g.tile_start[count] = total;
    return total;
  };
  ExactGroup g;
  int total = tiles(64, g);
  if (total == 0) return cudaSuccess;
  // small problems: 32 x 32 tiles put 4x the CTAs on the SMs (the reduction itself is
  // sequential per element, so more, smaller tiles is the only parallelism left)
  const bool small = total < 2 * sm_count();
  if (small) total = tiles(32, g);
  if (dtype == BD_F32) {
    if (small)
      kv_proj_exact_kernel<float, 32><<<total, 64, 0, stream>>>(g, flag);
    else
      kv_proj_exact_kernel<float, 64><<<total, 256, 0, stream>>>(g, flag);
  } else {
    if (small)
      kv_proj_exact_kernel<double, 32><<<total, 64, 0, stream>>>(g, flag);
    else
      kv_proj_exact_kernel<double, 64><<<total, 256, 0, stream>>>(g, flag);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace bdk
