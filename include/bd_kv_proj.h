/*
 * bd_kv_proj.h — C ABI of the B200-native basis-decomposed K/V projection.
 *
 * The projection (BD Attention, arXiv 2510.01718) is
 *
 *     out[i, h*d_h + j] = ( sum_{k=0}^{d-d_h-1} x[i, mul_base + k] * c[k, h*d_h + j] )
 *                         + x[i, rep_base + j]
 *
 * for rows i < L, heads h < n_heads, j < d_h.  The tag of the reference picks the
 * two offsets: FIRST -> (mul_base, rep_base) = (d_h, 0), LAST -> (0, d - d_h).
 *
 * Reference interface this replaces:
 *   - bdattn.attention._fused_kernel(x, c, d_h, n_heads, mul_base, rep_base, out)
 *       ref: pkg/src/bdattn/attention.py:249-270   (the numba "FFI" the Python op calls)
 *   - bdattn.fused_kv_proj(x, c, d_h, n_heads, tag)
 *       ref: pkg/src/bdattn/attention.py:273-295   (validation + tag -> offsets + allocation)
 *
 * Differences from the reference kernel that a binding author must know:
 *   - every element of `out` is written exactly once (no pre-zeroed buffer needed;
 *     the reference accumulates into a caller-zeroed array, attention.py:293-294,
 *     which gives the same values because it starts from +0.0);
 *   - device entry points are stream-ordered and asynchronous; *_host entry points
 *     are synchronous and take host pointers, like the numba dispatcher call;
 *   - FP32/FP64 run the "exact" kernel: per element, k ascending, one rounded
 *     multiply then one rounded add per step (no FMA), then + the repeated slice —
 *     the reference's rounding sequence (attention.py:258-265), hence bit-identical;
 *   - FP16/BF16 run the tensor-core kernel (TMA -> tcgen05.mma -> TMEM, FP32
 *     accumulate, gather-add of x[:, rep] in FP32 in the epilogue, one output
 *     rounding).  The reference has no 16-bit path (ref: SPEC.md:138).
 *
 * All sizes are in elements; leading dimensions (ld*) are row strides in elements.
 * Return value: BD_OK or one of BD_ERR_*; bd_last_error() describes the last failure
 * on the calling thread.
 */
#ifndef BD_KV_PROJ_H
#define BD_KV_PROJ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BD_KV_PROJ_ABI_VERSION 6

/* element types */
enum bd_dtype { BD_F32 = 0, BD_F64 = 1, BD_F16 = 2, BD_BF16 = 3 };

/* status codes */
enum bd_status {
  BD_OK = 0,
  BD_ERR_SHAPE = 1,  /* ref ShapeError (errors.py:4) */
  BD_ERR_DTYPE = 2,  /* ref PrecisionError (errors.py:8) / unsupported dtype */
  BD_ERR_ALIGN = 3,  /* tensor-core path needs 16-byte aligned rows/offsets */
  BD_ERR_CUDA = 4,   /* a CUDA runtime/driver call failed */
  BD_ERR_ARG = 5     /* null pointer, negative size, bad enum */
};

/* kernel selection */
enum bd_mode {
  BD_MODE_AUTO = 0,   /* F32/F64 -> exact, F16/BF16 -> tensor core */
  BD_MODE_EXACT = 1,  /* SIMT, reference rounding order (F32/F64 only) */
  BD_MODE_TC = 2      /* tcgen05 tensor cores (F16/BF16 only) */
};

/* output layouts */
enum bd_out_layout {
  BD_OUT_TOKEN_MAJOR = 0, /* out[i, h*d_h + j] at out + i*ldo + h*d_h + j (the reference's) */
  BD_OUT_HEAD_MAJOR = 1   /* out[h][i][j] at out + (h*L + i)*ldo + j: per-head contiguous,
                             what per-head attention and a flat head all-gather consume */
};

/* tags (ref: decompose.py:27-31) */
enum bd_tag { BD_TAG_FIRST = 0, BD_TAG_LAST = 1 };

/* One projection problem. Pointers are device pointers for the device entry points. */
typedef struct bd_kv_problem {
  const void* x;    /* L x d,            row stride ldx */
  const void* c;    /* (d - d_h) x N,    row stride ldc, N = n_heads * d_h */
  void* out;        /* L x N,            row stride ldo */
  int64_t ldx, ldc, ldo;
  int64_t L, d, d_h, n_heads;
  int64_t mul_base; /* first column of x multiplied by c  (FIRST: d_h, LAST: 0)     */
  int64_t rep_base; /* first column of x repeated per head (FIRST: 0, LAST: d - d_h) */
} bd_kv_problem;

/*
 * Fused K/V projection on device buffers, enqueued on `stream` (a cudaStream_t,
 * NULL = legacy default stream).  `nonfinite_flag`, if not NULL, is a device int
 * that the kernel sets to 1 when any output element is NaN/Inf (the reference
 * raises ValueError for that, tensor.py:112-113); it is never cleared by the call.
 * Replaces: _fused_kernel(x, c, d_h, n_heads, mul_base, rep_base, out)
 *           (ref: pkg/src/bdattn/attention.py:249-270, called at :294).
 */
int bd_kv_proj(const void* x, int64_t ldx, const void* c, int64_t ldc, void* out, int64_t ldo,
               int64_t L, int64_t d, int64_t d_h, int64_t n_heads, int64_t mul_base,
               int64_t rep_base, int dtype, int mode, int* nonfinite_flag, void* stream);

/*
 * Several projections in ONE launch (bda_forward's K' and V', ref attention.py:305-306,
 * or the K and V halves of an MLA kv_b_proj).  All problems share dtype and mode.
 * count must be in [1, BD_MAX_GROUP].
 */
#define BD_MAX_GROUP 4
int bd_kv_proj_grouped(const bd_kv_problem* problems, int count, int dtype, int mode,
                       int* nonfinite_flag, void* stream);

/*
 * Synchronous host-buffer variant: x, c, out are HOST pointers (C-contiguous,
 * ldx = d, ldc = ldo = N).  Copies in, runs the kernel on an internal stream,
 * copies out, synchronises, and returns BD_ERR_CUDA... or BD_OK.  If *nonfinite
 * is not NULL it receives 1 when the output holds NaN/Inf.  This is the entry a
 * ctypes/numba-level drop-in for _fused_kernel binds.
 * Device staging buffers are cached per thread and grown on demand.
 */
int bd_kv_proj_host(const void* x, const void* c, void* out, int64_t L, int64_t d, int64_t d_h,
                    int64_t n_heads, int64_t mul_base, int64_t rep_base, int dtype, int mode,
                    int* nonfinite);

/*
 * Plain product out = a @ b on device buffers (a: M x K, b: K x N, out: M x N, row-major
 * with row strides lda/ldb/ldo), stream-ordered.  F32/F64 run the exact kernel and are
 * bit-identical to the reference's fixed-order matmul; F16/BF16 run the tensor-core
 * kernel without the repeated-slice add.
 * Replaces: bdattn.matmul / _matmul_kernel (ref: pkg/src/bdattn/tensor.py:189-213).
 */
int bd_matmul(const void* a, int64_t lda, const void* b, int64_t ldb, void* out, int64_t ldo,
              int64_t M, int64_t K, int64_t N, int dtype, int mode, int* nonfinite_flag,
              void* stream);

/*
 * BD low-rank linear layer forward on device buffers: h = x @ basis (L x rank), then
 * y = [h, h @ coeff] for tag FIRST or [h @ coeff, h] for LAST (y: L x d_out, stride ldy).
 * h is written straight into its final columns of y and read back from there as the
 * second product's A operand (no concat buffer).  Two launches on `stream`.
 * basis: d_in x rank (ldb), coeff: rank x (d_out - rank) (ldc).
 * Replaces: bdattn.bd_linear_forward (ref: pkg/src/bdattn/linear.py:101-108).
 */
int bd_linear_forward(const void* x, int64_t ldx, const void* basis, int64_t ldb,
                      const void* coeff, int64_t ldc, void* y, int64_t ldy, int64_t L,
                      int64_t d_in, int64_t rank, int64_t d_out, int tag, int dtype, int mode,
                      int* nonfinite_flag, void* stream);

/*
 * bd_kv_proj_grouped with an output layout (enum bd_out_layout).  For
 * BD_OUT_HEAD_MAJOR each problem's out is [n_heads][L][d_h] with row stride ldo >= d_h
 * (head stride L * ldo).  The tensor-core path needs d_h to be a multiple of 64 there.
 */
int bd_kv_proj_grouped_ex(const bd_kv_problem* problems, int count, int dtype, int mode,
                          int out_layout, int* nonfinite_flag, void* stream);

/*
 * Head-parallel projection with the all-gather FUSED into the epilogue: this rank owns
 * n_heads heads of each problem and writes them, head-major, straight into every rank's
 * full-width buffer over NVLink (peer pointers, e.g. torch symmetric memory), so no
 * separate collective runs after the kernel.  For problem p, gathered[p*world + r] is
 * rank r's [world*n_heads][L][d_h] buffer (row stride problems[p].ldo >= d_h); this
 * rank's heads land in planes [rank*n_heads, (rank+1)*n_heads) of each.  problems[p].out
 * is ignored.  world in [1, BD_MAX_PEERS].  The caller must order the peers' reads after
 * every rank's kernel (a barrier on the stream).  Tensor-core path: d_h % 64 == 0.
 */
#define BD_MAX_PEERS 8
int bd_kv_proj_grouped_allgather(const bd_kv_problem* problems, int count, int dtype, int mode,
                                 int world, int rank, void* const* gathered,
                                 int* nonfinite_flag, void* stream);

/*
 * Projections of the RMS-normalised latent with the norm FUSED (DeepSeek-V2's
 * kv_a_layernorm in front of kv_b_proj).  x is the RAW latent (L x d); each problem
 * computes the BD projection of  x_n = x * rsqrt(mean(x[i, :]^2) + eps) * gamma  as
 *   out[i, j] = r_i * (sum_k x[i, mul_base + k] c_g[k, j] + rep_gamma[j % d_h] x[i, rep_base + j % d_h])
 * where c_g = diag(gamma[mul_base : mul_base + d - d_h]) c is folded by the caller once per
 * weight and rep_gamma[p] = gamma[rep_base : rep_base + d_h] (d_h floats, device memory).
 * The mean runs over the row's d columns.  No separate normalisation pass: one read of x.
 * Tensor-core path: d_h in {64, 128} and d - d_h <= 384 (the row is resident in smem).
 * Extends (ref: pkg/src/bdattn/attention.py:249-270) to the MLA latent of SURVEY §8(f) #3.
 */
int bd_kv_proj_grouped_rmsnorm(const bd_kv_problem* problems, int count, int dtype, int mode,
                               int out_layout, const float* const* rep_gamma, float eps,
                               int* nonfinite_flag, void* stream);

/*
 * Causal (or full) prefill attention of the BD-rewritten DeepSeek-V2 MLA block, reading the
 * BD projection's outputs in place (BD ⊕ FlashAttention; the attention
 * core the reference computes after its two fused_kv_proj calls, ref
 * pkg/src/bdattn/attention.py:298-307 and _attend :143-154, restated for MLA):
 *   out[t, h, :] = softmax_s(scale * (q[t, h, 0:dn] . k_nope[h, s, :] + q[t, h, dn:] . k_pe[s, :]))
 *                  @ v[h, s, :]
 * q:      element (t, h, c) at q + t*ldq_tok + h*ldq_head + c, c < d_nope + d_rope
 * k_nope: (h, s, c) at k_nope + h*k_head_stride + s*ldk + c   (head-major, BD out_layout=head)
 * k_pe:   (s, c) at k_pe + s*ldkpe + c — the decoupled RoPE key, shared by every head
 * v:      (h, s, c) at v + h*v_head_stride + s*ldv + c        (head-major)
 * out:    (t, h, c) at out + t*ldo_tok + h*ldo_head + c
 * causal: key s attends to query t only for s <= t.  dtype F16/BF16; geometry d_nope = 128,
 * d_rope = 64, d_v = 128 (DeepSeek-V2 / -V2-Lite); 16-byte aligned pointers, strides
 * multiples of 8 elements.  Returns BD_OK or BD_ERR_*; asynchronous on `stream`.
 */
int bd_mla_attention(const void* q, int64_t ldq_tok, int64_t ldq_head, const void* k_nope,
                     int64_t ldk, int64_t k_head_stride, const void* k_pe, int64_t ldkpe,
                     const void* v, int64_t ldv, int64_t v_head_stride, void* out,
                     int64_t ldo_tok, int64_t ldo_head, int64_t L, int64_t n_heads,
                     int64_t d_nope, int64_t d_rope, int64_t d_v, float scale, int causal,
                     int dtype, void* stream);

/* Human-readable description of the last error on this thread ("" if none). */
const char* bd_last_error(void);

/* BD_KV_PROJ_ABI_VERSION of the loaded library. */
int bd_abi_version(void);

/* Number of kernel launches issued by this library since load (all threads). */
uint64_t bd_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* BD_KV_PROJ_H */
