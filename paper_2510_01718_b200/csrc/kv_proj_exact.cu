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
// Tiling is for data reuse only: a 128x128 output tile per 256-thread CTA with 8x8
// outputs per thread and double-buffered k-slabs of 8 through shared memory (64x64 / 4x4
// and 32x32 / 4x4 tiles for outputs too small to fill the SMs).  The per-element
// reduction order is untouched by the tiling, which is also why column-sharding the
// output across GPUs is bit-invariant (ref test_tensor.py:113-119).
#include <climits>
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdint>

#include "kv_proj_internal.h"

namespace bdk {
namespace {

// Tile T x T with R x R outputs per thread ((T / R)^2 threads): T = 128, R = 8 for
// large outputs (k-slabs of 8, double-buffered), T = 64 / 32 with R = 4 (k-slabs of 16)
// when bigger tiles would leave SMs idle.
// FP32 with R = 8 runs two CTAs per SM (128 registers); the slab loop is unrolled by two
// (static buffer index) except there, where the larger code runs slower (measured,
// tools/exact_ab.sh).
template <typename T, int R>
struct ExactSlab {
  static constexpr int BK = R == 8 ? 8 : 16;
  static constexpr int MIN_CTAS = R == 8 && sizeof(T) == 4 ? 2 : 1;
  static constexpr bool UNROLL2 = !(R == 8 && sizeof(T) == 4);
};

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

template <typename T, int TILE, int R>
__global__ void __launch_bounds__((TILE / R) * (TILE / R), ExactSlab<T, R>::MIN_CTAS)
    kv_proj_exact_kernel(const __grid_constant__ ExactGroup g, int* flag) {
  constexpr int EX_BM = TILE, EX_BN = TILE, EX_THREADS = (TILE / R) * (TILE / R);
  constexpr int GROUPS = TILE / R;
  constexpr int EX_BK = ExactSlab<T, R>::BK;
  constexpr int PAD = 16 / sizeof(T);  // keeps the transposed x stores off one bank
  // Locate the problem and the tile this CTA owns.
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

  // x slab k-major (a thread's R rows contiguous), c slab as is; two buffers: the next
  // slab is written while the current one is consumed (one barrier per slab)
  __shared__ __align__(16) T xs[2][EX_BK][EX_BM + PAD];
  __shared__ __align__(16) T cs[2][EX_BK][EX_BN + PAD];

  const int tx = threadIdx.x % GROUPS;  // column group
  const int ty = threadIdx.x / GROUPS;  // row group
  T acc[R][R];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[i][j] = T(0);

  // Slabs of x[m0 : m0 + T, mul_base + k0 : + EX_BK] and c[k0 : k0 + EX_BK, n0 : n0 + T]
  // (zero-filled outside the problem; padded entries are never folded into acc, see
  // kmax); the next slab's global loads are in flight in registers while the current
  // one is consumed.
  constexpr int XL = EX_BM * EX_BK / EX_THREADS;
  constexpr int CL = EX_BN * EX_BK / EX_THREADS;
  static_assert(EX_THREADS % EX_BK == 0 && EX_THREADS % EX_BN == 0, "slab load mapping");
  // Each thread loads a fixed k column of the x slab (rows xr0 + u * XRS) and a fixed
  // column of the c slab (k rows ck0 + u * CKS): one base pointer each, bounds hoisted.
  constexpr int XRS = EX_THREADS / EX_BK, CKS = EX_THREADS / EX_BN;
  const int xkk = threadIdx.x % EX_BK, xr0 = threadIdx.x / EX_BK;
  const int ccc = threadIdx.x % EX_BN, ck0 = threadIdx.x / EX_BN;
  const T* xbase = x + (m0 + xr0) * P.ldx + P.mul_base + xkk;
  const T* cbase = c + static_cast<int64_t>(ck0) * P.ldc + n0 + ccc;
  const int64_t xstep = static_cast<int64_t>(XRS) * P.ldx;
  const int64_t ldc = P.ldc;
  uint32_t xrow_ok = 0;
#pragma unroll
  for (int u = 0; u < XL; ++u)
    if (m0 + xr0 + u * XRS < P.L) xrow_ok |= 1u << u;
  const bool ccol_ok = n0 + ccc < N;
  T xr[XL], cr[CL];
  auto fetch = [&](int64_t k0) {
    const bool xk_ok = k0 + xkk < K;
#pragma unroll
    for (int u = 0; u < XL; ++u)
      xr[u] = (xk_ok && ((xrow_ok >> u) & 1u)) ? xbase[u * xstep + k0] : T(0);
#pragma unroll
    for (int u = 0; u < CL; ++u)
      cr[u] = (ccol_ok && k0 + ck0 + u * CKS < K) ? cbase[(k0 + u * CKS) * ldc] : T(0);
  };
  auto stage = [&](int buf) {
#pragma unroll
    for (int u = 0; u < XL; ++u) xs[buf][xkk][xr0 + u * XRS] = xr[u];
#pragma unroll
    for (int u = 0; u < CL; ++u) cs[buf][ck0 + u * CKS][ccc] = cr[u];
  };
  auto step = [&](int buf, int kk) {  // k ascending: the reference's order
    T a[R], b[R];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = xs[buf][kk][ty * R + i];
#pragma unroll
    for (int j = 0; j < R; ++j) b[j] = cs[buf][kk][tx * R + j];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < R; ++j)
        acc[i][j] = ExactOps<T>::add(acc[i][j], ExactOps<T>::mul(a[i], b[j]));
  };
  auto slab = [&](int64_t k0, int buf) {  // consume slab k0 from buffer buf
    const bool more = k0 + EX_BK < K;
    if (more) fetch(k0 + EX_BK);
    const int kmax = static_cast<int>((K - k0) < EX_BK ? (K - k0) : EX_BK);
    if (kmax == EX_BK) {
#pragma unroll
      for (int kk = 0; kk < EX_BK; ++kk) step(buf, kk);
    } else {
      for (int kk = 0; kk < kmax; ++kk) step(buf, kk);
    }
    if (more) stage(buf ^ 1);
    __syncthreads();
  };
  fetch(0);
  stage(0);
  __syncthreads();
  if constexpr (ExactSlab<T, R>::UNROLL2) {
    for (int64_t k0 = 0; k0 < K; k0 += 2 * EX_BK) {  // buffer index a compile-time constant
      slab(k0, 0);
      if (k0 + EX_BK < K) slab(k0 + EX_BK, 1);
    }
  } else {
    int buf = 0;
    for (int64_t k0 = 0; k0 < K; k0 += EX_BK, buf ^= 1) slab(k0, buf);
  }

  // Epilogue: + the repeated basis slice, after the full sum (attention.py:266-270).
  // Without it (rep_base < 0) this is the reference's fixed-order matmul
  // (tensor.py:189-213), used by the BD low-rank layer.
  const bool has_rep = P.rep_base >= 0;
  bool bad = false;
  // this thread's R columns: head and in-head index, stepped from one 32-bit division (a
  // 64-bit / or % per element costs more than the element's share of the reduction)
  int hd[R], rc[R];
  {
    const int dh = P.d_h > 0 ? static_cast<int>(P.d_h) : INT_MAX;  // no rep: unused
    const int c0 = static_cast<int>(n0) + tx * R;
    int h = c0 / dh, r = c0 - h * dh;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      hd[j] = h;
      rc[j] = r;
      if (++r == dh) {
        r = 0;
        ++h;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t row = m0 + ty * R + i;
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
    for (int j = 0; j < R; ++j) {
      const int64_t col = n0 + tx * R + j;
      if (col >= N) continue;
      T v;
      if (P.rep_gamma != nullptr) {
        const T xr = x[row * P.ldx + P.rep_base + rc[j]];
        v = ExactOps<T>::mul(
            rn, ExactOps<T>::add(acc[i][j],
                                 ExactOps<T>::mul(static_cast<T>(P.rep_gamma[rc[j]]), xr)));
      } else {
        v = has_rep ? ExactOps<T>::add(acc[i][j], x[row * P.ldx + P.rep_base + rc[j]])
                    : acc[i][j];
      }
      if (P.world > 0) {  // fused all-gather: every rank's full-width head-major buffer
        const int64_t off = ((P.head0 + hd[j]) * P.L + row) * P.ldo + rc[j];
        for (int r = 0; r < P.world; ++r) static_cast<T*>(P.peers[r])[off] = v;
      } else if (P.out_layout == BD_OUT_HEAD_MAJOR) {
        out[(static_cast<int64_t>(hd[j]) * P.L + row) * P.ldo + rc[j]] = v;
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
  // 128 x 128 tiles (8 x 8 per thread) while they give every SM two tiles; else 64 x 64;
  // small problems 32 x 32 (4x the CTAs: the reduction itself is sequential per element,
  // so more, smaller tiles is the only parallelism left)
  int total = tiles(128, g);
  if (total == 0) return cudaSuccess;
  int tile = 128;
  if (total < 2 * sm_count()) {
    tile = 64;
    total = tiles(64, g);
    if (total < 2 * sm_count()) {
      tile = 32;
      total = tiles(32, g);
    }
  }
  static const int forced = [] {  // BD_EXACT_TILE=32|64|128 forces a tile (A/B)
    const char* e = getenv("BD_EXACT_TILE");
    return e ? atoi(e) : 0;
  }();
  if (forced == 32 || forced == 64 || forced == 128) {
    tile = forced;
    total = tiles(tile, g);
  }
  if (dtype == BD_F32) {
    if (tile == 128)
      kv_proj_exact_kernel<float, 128, 8><<<total, 256, 0, stream>>>(g, flag);
    else if (tile == 64)
      kv_proj_exact_kernel<float, 64, 4><<<total, 256, 0, stream>>>(g, flag);
    else
      kv_proj_exact_kernel<float, 32, 4><<<total, 64, 0, stream>>>(g, flag);
  } else {
    if (tile == 128)
      kv_proj_exact_kernel<double, 128, 8><<<total, 256, 0, stream>>>(g, flag);
    else if (tile == 64)
      kv_proj_exact_kernel<double, 64, 4><<<total, 256, 0, stream>>>(g, flag);
    else
      kv_proj_exact_kernel<double, 32, 4><<<total, 64, 0, stream>>>(g, flag);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace bdk
