// kv_proj_internal.h — launchers shared between the kernels and the C ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/bd_kv_proj.h"

namespace bdk {

// One contraction as the kernels see it:
//   out[i, j] = sum_{k<K} x[i, mul_base + k] * c[k, j]   (+ x[i, rep_base + j % d_h])
// The BD projection is K = d - d_h, N = n_heads * d_h with the repeated-slice add; a
// plain GEMM (the BD low-rank layer's two products) sets rep_base < 0 (no add).
struct Problem {
  const void* x;
  const void* c;
  void* out;
  int64_t ldx, ldc, ldo;
  int64_t L, K, N;
  int64_t d_h;       // head width of the repeated slice (ignored without rep)
  int64_t mul_base;  // first multiplied column of x
  int64_t rep_base;  // first repeated column of x; < 0: no repeated-slice add
  int32_t out_layout;  // BD_OUT_TOKEN_MAJOR (L x N, row stride ldo) or BD_OUT_HEAD_MAJOR
                       // ([N / d_h][L][d_h], row stride ldo, head stride L * ldo)
  // Fused all-gather (world > 0): head-major output written to every peer buffer
  // peers[r] ([world * N / d_h][L][d_h]) at head planes [head0, head0 + N / d_h).
  int32_t world;
  int32_t head0;
  void* peers[BD_MAX_PEERS];
  // Fused RMSNorm (rep_gamma != null): x is the raw latent; out = r_i * (x[:, mul] c +
  // rep_gamma * x[:, rep]) with r_i = rsqrt(mean(x[i, :d]^2) + norm_eps), d = K + d_h
  // (c must carry the multiplied columns' norm weight, folded by the caller).
  const float* rep_gamma;
  float norm_eps;
};

// Thread-local error text set by the launchers; returned by bd_last_error().
void set_error(const std::string& msg);

// Counts kernel launches for the bench's gpu_launches evidence.
void note_launch();

// Exact SIMT kernel (FP32/FP64): reference rounding sequence (attention.py:258-270).
cudaError_t launch_exact(const Problem* probs, int count, int dtype, int* flag,
                         cudaStream_t stream);

// tcgen05 tensor-core kernel (FP16/BF16). Returns BD_* status; sets error text.
int launch_tc(const Problem* probs, int count, int dtype, int* flag, cudaStream_t stream);

// MLA prefill attention over the BD projection's outputs (mla_attn.cu): Q [L][H][192]
// token-major, K'_nope / V' head-major [H][L][128], the shared RoPE key k_pe [L][64].
struct MlaAttnArgs {
  const void* q;
  int64_t ldq_tok, ldq_head;
  const void* k_nope;
  int64_t ldk, k_head_stride;
  const void* k_pe;
  int64_t ldkpe;
  const void* v;
  int64_t ldv, v_head_stride;
  void* out;
  int64_t ldo_tok, ldo_head;
  int64_t L, n_heads;
  float scale;
  int causal;
  int dtype;
};
int launch_mla_attention(const MlaAttnArgs& a, cudaStream_t stream);

// SM count of the current device (cached).
int sm_count();

// Per-device state (function attributes, staging) is kept in arrays of this many slots,
// indexed by device_slot(): the current device ordinal (clamped).
constexpr int kMaxDevices = 64;
int device_slot();

}  // namespace bdk
