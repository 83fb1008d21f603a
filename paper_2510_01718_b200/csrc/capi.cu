// capi.cu — the C ABI (include/bd_kv_proj.h): validation, kernel dispatch, the
// synchronous host-buffer entry point and error reporting.
//
// Validation mirrors what the reference checks before it calls its kernel
// (ref: pkg/src/bdattn/attention.py:283-288: precision first, then c's rows, then
// c's cols) plus what a raw-pointer ABI needs (null pointers, strides, offsets,
// 16-byte alignment for the TMA path).  Nothing is launched when a check fails.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/bd_kv_proj.h"
#include "kv_proj_internal.h"

namespace bdk {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t elem_size(int dtype) {
  switch (dtype) {
    case BD_F32: return 4;
    case BD_F64: return 8;
    case BD_F16: return 2;
    case BD_BF16: return 2;
    default: return 0;
  }
}

int resolve_mode(int dtype, int mode, int* out_mode) {
  if (mode == BD_MODE_AUTO) {
    *out_mode = (dtype == BD_F32 || dtype == BD_F64) ? BD_MODE_EXACT : BD_MODE_TC;
    return BD_OK;
  }
  if (mode == BD_MODE_EXACT) {
    if (dtype != BD_F32 && dtype != BD_F64)
      return fail(BD_ERR_DTYPE, "exact mode supports F32/F64 only");
    *out_mode = mode;
    return BD_OK;
  }
  if (mode == BD_MODE_TC) {
    if (dtype != BD_F16 && dtype != BD_BF16)
      return fail(BD_ERR_DTYPE, "tensor-core mode supports F16/BF16 only");
    *out_mode = mode;
    return BD_OK;
  }
  return fail(BD_ERR_ARG, "unknown mode " + std::to_string(mode));
}

int validate(const bd_kv_problem& p, int dtype, int mode, int idx,
             int out_layout = BD_OUT_TOKEN_MAJOR) {
  char buf[256];
  const std::string at = "problem " + std::to_string(idx) + ": ";
  if (p.x == nullptr || p.c == nullptr || p.out == nullptr)
    return fail(BD_ERR_ARG, at + "null pointer");
  if (p.L < 1 || p.d < 2 || p.d_h < 1 || p.n_heads < 1) {
    snprintf(buf, sizeof(buf), "non-positive size (L=%lld d=%lld d_h=%lld n_heads=%lld)",
             (long long)p.L, (long long)p.d, (long long)p.d_h, (long long)p.n_heads);
    return fail(BD_ERR_SHAPE, at + buf);
  }
  if (p.d_h >= p.d) {
    snprintf(buf, sizeof(buf), "d_h (%lld) must be < d (%lld)", (long long)p.d_h,
             (long long)p.d);
    return fail(BD_ERR_SHAPE, at + buf);
  }
  const int64_t K = p.d - p.d_h;
  const int64_t N = p.n_heads * p.d_h;
  if (p.mul_base < 0 || p.mul_base + K > p.d || p.rep_base < 0 || p.rep_base + p.d_h > p.d) {
    snprintf(buf, sizeof(buf), "offsets out of range (mul_base=%lld rep_base=%lld d=%lld d_h=%lld)",
             (long long)p.mul_base, (long long)p.rep_base, (long long)p.d, (long long)p.d_h);
    return fail(BD_ERR_SHAPE, at + buf);
  }
  const int64_t min_ldo = out_layout == BD_OUT_HEAD_MAJOR ? p.d_h : N;
  if (p.ldx < p.d || p.ldc < N || p.ldo < min_ldo) {
    snprintf(buf, sizeof(buf), "row strides too small (ldx=%lld ldc=%lld ldo=%lld, d=%lld N=%lld)",
             (long long)p.ldx, (long long)p.ldc, (long long)p.ldo, (long long)p.d, (long long)N);
    return fail(BD_ERR_SHAPE, at + buf);
  }
  if (p.L > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return fail(BD_ERR_SHAPE, at + "dimension exceeds int32 range");
  if (mode == BD_MODE_TC && out_layout == BD_OUT_HEAD_MAJOR && (p.d_h % 64) != 0) {
    snprintf(buf, sizeof(buf), "head-major tensor-core output needs d_h %% 64 == 0 (d_h=%lld)",
             (long long)p.d_h);
    return fail(BD_ERR_ALIGN, at + buf);
  }
  if (mode == BD_MODE_TC) {
    if (!aligned16(p.x) || !aligned16(p.c) || !aligned16(p.out))
      return fail(BD_ERR_ALIGN, at + "tensor-core path needs 16-byte aligned x, c and out");
    if ((p.ldx | p.ldc | p.ldo | p.mul_base | p.rep_base | p.d_h) & 7) {
      snprintf(buf, sizeof(buf),
               "tensor-core path needs ldx, ldc, ldo, mul_base, rep_base and d_h to be multiples "
               "of 8 (got %lld %lld %lld %lld %lld %lld)",
               (long long)p.ldx, (long long)p.ldc, (long long)p.ldo, (long long)p.mul_base,
               (long long)p.rep_base, (long long)p.d_h);
      return fail(BD_ERR_ALIGN, at + buf);
    }
  }
  (void)dtype;
  return BD_OK;
}

Problem to_problem(const bd_kv_problem& q, int out_layout) {
  return Problem{q.x, q.c, q.out, q.ldx, q.ldc, q.ldo, q.L, q.d - q.d_h, q.n_heads * q.d_h,
                 q.d_h, q.mul_base, q.rep_base, out_layout, 0, 0, {}};
}

int dispatch(const Problem* probs, int count, int dtype, int m, int* flag, cudaStream_t stream) {
  g_last_error.clear();
  if (m == BD_MODE_EXACT) {
    cudaError_t e = launch_exact(probs, count, dtype, flag, stream);
    if (e != cudaSuccess)
      return fail(BD_ERR_CUDA, std::string("kv_proj_exact: ") + cudaGetErrorString(e));
    return BD_OK;
  }
  return launch_tc(probs, count, dtype, flag, stream);
}

int run_group(const bd_kv_problem* probs, int count, int dtype, int mode, int* flag,
              cudaStream_t stream, int out_layout = BD_OUT_TOKEN_MAJOR, int world = 0,
              int rank = 0, void* const* gathered = nullptr,
              const float* const* rep_gamma = nullptr, float eps = 0.f) {
  if (out_layout != BD_OUT_TOKEN_MAJOR && out_layout != BD_OUT_HEAD_MAJOR)
    return fail(BD_ERR_ARG, "unknown out_layout " + std::to_string(out_layout));
  if (probs == nullptr || count < 1 || count > BD_MAX_GROUP)
    return fail(BD_ERR_ARG, "problem count must be in [1, " + std::to_string(BD_MAX_GROUP) + "]");
  if (elem_size(dtype) == 0) return fail(BD_ERR_DTYPE, "unknown dtype " + std::to_string(dtype));
  int m = 0;
  int rc = resolve_mode(dtype, mode, &m);
  if (rc != BD_OK) return rc;
  Problem ps[BD_MAX_GROUP];
  for (int i = 0; i < count; ++i) {
    rc = validate(probs[i], dtype, m, i, out_layout);
    if (rc != BD_OK) return rc;
    ps[i] = to_problem(probs[i], out_layout);
    if (rep_gamma != nullptr) {
      if (rep_gamma[i] == nullptr) return fail(BD_ERR_ARG, "null rep_gamma");
      const bool first = probs[i].mul_base == probs[i].d_h && probs[i].rep_base == 0;
      const bool last = probs[i].mul_base == 0 && probs[i].rep_base == probs[i].d - probs[i].d_h;
      if (!first && !last)
        return fail(BD_ERR_SHAPE, "fused RMSNorm: the multiplied and repeated slices must "
                                  "partition the row (tags FIRST / LAST)");
      ps[i].rep_gamma = rep_gamma[i];
      ps[i].norm_eps = eps;
    }
    if (world > 0) {
      ps[i].world = world;
      ps[i].head0 = static_cast<int32_t>(rank * probs[i].n_heads);
      for (int r = 0; r < world; ++r) {
        ps[i].peers[r] = gathered[i * world + r];
        if (ps[i].peers[r] == nullptr) return fail(BD_ERR_ARG, "null gathered buffer");
        if (m == BD_MODE_TC && !aligned16(ps[i].peers[r]))
          return fail(BD_ERR_ALIGN, "gathered buffers must be 16-byte aligned");
      }
      ps[i].out = ps[i].peers[rank];
    }
  }
  return dispatch(ps, count, dtype, m, flag, stream);
}

// A plain product (no repeated-slice add): validation for raw pointers/strides.
int validate_matmul(const void* a, int64_t lda, const void* b, int64_t ldb, const void* out,
                    int64_t ldo, int64_t M, int64_t K, int64_t N, int m, const char* what) {
  char buf[256];
  if (a == nullptr || b == nullptr || out == nullptr)
    return fail(BD_ERR_ARG, std::string(what) + ": null pointer");
  if (M < 1 || K < 1 || N < 1) {
    snprintf(buf, sizeof(buf), "%s: non-positive size (M=%lld K=%lld N=%lld)", what,
             (long long)M, (long long)K, (long long)N);
    return fail(BD_ERR_SHAPE, buf);
  }
  if (lda < K || ldb < N || ldo < N) {
    snprintf(buf, sizeof(buf), "%s: row strides too small (lda=%lld ldb=%lld ldo=%lld)", what,
             (long long)lda, (long long)ldb, (long long)ldo);
    return fail(BD_ERR_SHAPE, buf);
  }
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return fail(BD_ERR_SHAPE, std::string(what) + ": dimension exceeds int32 range");
  if (m == BD_MODE_TC) {
    if (!aligned16(a) || !aligned16(b) || !aligned16(out))
      return fail(BD_ERR_ALIGN, std::string(what) + ": tensor-core path needs 16-byte aligned operands");
    if ((lda | ldb | ldo | K | N) & 7)
      return fail(BD_ERR_ALIGN, std::string(what) +
                                    ": tensor-core path needs lda, ldb, ldo, K and N to be multiples of 8");
  }
  return BD_OK;
}

// Per-thread device staging for the synchronous host entry point, one set per device
// (buffers and stream belong to the device that was current when they were created).
struct HostStaging {
  void* buf = nullptr;
  size_t cap = 0;
  int* flag = nullptr;
  cudaStream_t stream = nullptr;
  int device = -1;
  void release() {
    if (device >= 0) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(device);
      if (buf) cudaFree(buf);
      if (flag) cudaFree(flag);
      if (stream) cudaStreamDestroy(stream);
      cudaSetDevice(cur);
    }
    buf = nullptr;
    cap = 0;
    flag = nullptr;
    stream = nullptr;
    device = -1;
  }
  // Process teardown may already have destroyed the context; errors are ignored.
  ~HostStaging() { release(); }
};
thread_local HostStaging g_staging[4];  // a few devices per thread; more rotate through

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int device_slot() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}

int sm_count() {
  static std::atomic<int> cached[kMaxDevices] = {};  // per device ordinal, 0 = not queried yet
  const int dev = device_slot();
  int n = cached[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n > 0 ? n : 148;
    cached[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

}  // namespace bdk

extern "C" {

int bd_kv_proj(const void* x, int64_t ldx, const void* c, int64_t ldc, void* out, int64_t ldo,
               int64_t L, int64_t d, int64_t d_h, int64_t n_heads, int64_t mul_base,
               int64_t rep_base, int dtype, int mode, int* nonfinite_flag, void* stream) {
  bd_kv_problem p{x, c, out, ldx, ldc, ldo, L, d, d_h, n_heads, mul_base, rep_base};
  return bdk::run_group(&p, 1, dtype, mode, nonfinite_flag, static_cast<cudaStream_t>(stream));
}

int bd_kv_proj_grouped(const bd_kv_problem* problems, int count, int dtype, int mode,
                       int* nonfinite_flag, void* stream) {
  return bdk::run_group(problems, count, dtype, mode, nonfinite_flag,
                        static_cast<cudaStream_t>(stream));
}

int bd_kv_proj_grouped_ex(const bd_kv_problem* problems, int count, int dtype, int mode,
                          int out_layout, int* nonfinite_flag, void* stream) {
  return bdk::run_group(problems, count, dtype, mode, nonfinite_flag,
                        static_cast<cudaStream_t>(stream), out_layout);
}

int bd_kv_proj_grouped_allgather(const bd_kv_problem* problems, int count, int dtype, int mode,
                                 int world, int rank, void* const* gathered,
                                 int* nonfinite_flag, void* stream) {
  using namespace bdk;
  if (world < 1 || world > BD_MAX_PEERS || rank < 0 || rank >= world)
    return fail(BD_ERR_ARG, "world must be in [1, BD_MAX_PEERS] and 0 <= rank < world");
  if (gathered == nullptr) return fail(BD_ERR_ARG, "null gathered pointer array");
  if (problems == nullptr || count < 1 || count > BD_MAX_GROUP)
    return fail(BD_ERR_ARG, "problem count must be in [1, " + std::to_string(BD_MAX_GROUP) + "]");
  // out is ignored: point it at this rank's buffer so the shared validation passes
  bd_kv_problem local[BD_MAX_GROUP];
  for (int i = 0; i < count; ++i) {
    local[i] = problems[i];
    local[i].out = gathered[i * world + rank];
  }
  return run_group(local, count, dtype, mode, nonfinite_flag, static_cast<cudaStream_t>(stream),
                   BD_OUT_HEAD_MAJOR, world, rank, gathered);
}

int bd_kv_proj_grouped_rmsnorm(const bd_kv_problem* problems, int count, int dtype, int mode,
                               int out_layout, const float* const* rep_gamma, float eps,
                               int* nonfinite_flag, void* stream) {
  using namespace bdk;
  if (rep_gamma == nullptr) return fail(BD_ERR_ARG, "null rep_gamma array");
  if (!(eps >= 0.f)) return fail(BD_ERR_ARG, "eps must be >= 0");
  return run_group(problems, count, dtype, mode, nonfinite_flag,
                   static_cast<cudaStream_t>(stream), out_layout, 0, 0, nullptr, rep_gamma, eps);
}

int bd_kv_proj_host(const void* x, const void* c, void* out, int64_t L, int64_t d, int64_t d_h,
                    int64_t n_heads, int64_t mul_base, int64_t rep_base, int dtype, int mode,
                    int* nonfinite) {
  using namespace bdk;
  const size_t es = elem_size(dtype);
  if (es == 0) return fail(BD_ERR_DTYPE, "unknown dtype " + std::to_string(dtype));
  if (x == nullptr || c == nullptr || out == nullptr) return fail(BD_ERR_ARG, "null pointer");
  if (L < 1 || d < 2 || d_h < 1 || n_heads < 1 || d_h >= d)
    return fail(BD_ERR_SHAPE, "invalid sizes");
  const int64_t K = d - d_h;
  const int64_t N = n_heads * d_h;
  const size_t bx = round_up(static_cast<size_t>(L * d) * es, 256);
  const size_t bc = round_up(static_cast<size_t>(K * N) * es, 256);
  const size_t bo = round_up(static_cast<size_t>(L * N) * es, 256);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(BD_ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  HostStaging* sp = nullptr;
  for (auto& st : g_staging)
    if (st.device == dev) sp = &st;
  if (sp == nullptr) {
    sp = &g_staging[dev % 4];
    sp->release();  // another device's set: never reuse its buffers or stream here
  }
  HostStaging& s = *sp;
  if (s.stream == nullptr) {
    s.device = dev;
    e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&s.flag, sizeof(int));
    if (e != cudaSuccess) return fail(BD_ERR_CUDA, std::string("staging init: ") + cudaGetErrorString(e));
  }
  if (s.cap < bx + bc + bo) {
    if (s.buf) cudaFree(s.buf);
    s.buf = nullptr;
    s.cap = 0;
    e = cudaMalloc(&s.buf, bx + bc + bo);
    if (e != cudaSuccess) return fail(BD_ERR_CUDA, std::string("staging alloc: ") + cudaGetErrorString(e));
    s.cap = bx + bc + bo;
  }
  char* dx = static_cast<char*>(s.buf);
  char* dc = dx + bx;
  char* dout = dc + bc;
  e = cudaMemsetAsync(s.flag, 0, sizeof(int), s.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dx, x, static_cast<size_t>(L * d) * es, cudaMemcpyHostToDevice, s.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dc, c, static_cast<size_t>(K * N) * es, cudaMemcpyHostToDevice, s.stream);
  if (e != cudaSuccess) return fail(BD_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(e));
  bd_kv_problem p{dx, dc, dout, d, N, N, L, d, d_h, n_heads, mul_base, rep_base};  // device copies
  int rc = run_group(&p, 1, dtype, mode, s.flag, s.stream);
  if (rc != BD_OK) {
    cudaStreamSynchronize(s.stream);
    return rc;
  }
  int hflag = 0;
  e = cudaMemcpyAsync(out, dout, static_cast<size_t>(L * N) * es, cudaMemcpyDeviceToHost, s.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hflag, s.flag, sizeof(int), cudaMemcpyDeviceToHost, s.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s.stream);
  if (e != cudaSuccess) return fail(BD_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
  if (nonfinite) *nonfinite = hflag;
  return BD_OK;
}

int bd_matmul(const void* a, int64_t lda, const void* b, int64_t ldb, void* out, int64_t ldo,
              int64_t M, int64_t K, int64_t N, int dtype, int mode, int* nonfinite_flag,
              void* stream) {
  using namespace bdk;
  if (elem_size(dtype) == 0) return fail(BD_ERR_DTYPE, "unknown dtype " + std::to_string(dtype));
  int m = 0;
  int rc = resolve_mode(dtype, mode, &m);
  if (rc != BD_OK) return rc;
  rc = validate_matmul(a, lda, b, ldb, out, ldo, M, K, N, m, "bd_matmul");
  if (rc != BD_OK) return rc;
  Problem p{a, b, out, lda, ldb, ldo, M, K, N, 1, 0, -1, BD_OUT_TOKEN_MAJOR, 0, 0, {}};
  return dispatch(&p, 1, dtype, m, nonfinite_flag, static_cast<cudaStream_t>(stream));
}

int bd_linear_forward(const void* x, int64_t ldx, const void* basis, int64_t ldb,
                      const void* coeff, int64_t ldc, void* y, int64_t ldy, int64_t L,
                      int64_t d_in, int64_t rank, int64_t d_out, int tag, int dtype, int mode,
                      int* nonfinite_flag, void* stream) {
  using namespace bdk;
  const size_t es = elem_size(dtype);
  if (es == 0) return fail(BD_ERR_DTYPE, "unknown dtype " + std::to_string(dtype));
  if (tag != BD_TAG_FIRST && tag != BD_TAG_LAST)
    return fail(BD_ERR_ARG, "unknown tag " + std::to_string(tag));
  if (rank < 1 || rank >= d_out || rank > d_in)
    return fail(BD_ERR_SHAPE, "rank must satisfy 1 <= rank < d_out and rank <= d_in");
  if (ldy < d_out) return fail(BD_ERR_SHAPE, "ldy < d_out");
  int m = 0;
  int rc = resolve_mode(dtype, mode, &m);
  if (rc != BD_OK) return rc;
  // y = [h, h C] (FIRST) or [h C, h] (LAST): h lands in its final columns and is read
  // back from there as the second product's A operand, so no concat is materialised.
  const int64_t h_off = tag == BD_TAG_FIRST ? 0 : d_out - rank;
  const int64_t hc_off = tag == BD_TAG_FIRST ? rank : 0;
  char* yb = static_cast<char*>(y);
  void* h = yb + h_off * static_cast<int64_t>(es);
  void* hc = yb + hc_off * static_cast<int64_t>(es);
  rc = validate_matmul(x, ldx, basis, ldb, h, ldy, L, d_in, rank, m, "bd_linear_forward h = x B");
  if (rc != BD_OK) return rc;
  rc = validate_matmul(h, ldy, coeff, ldc, hc, ldy, L, rank, d_out - rank, m,
                       "bd_linear_forward h C");
  if (rc != BD_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Problem p1{x, basis, h, ldx, ldb, ldy, L, d_in, rank, 1, 0, -1, BD_OUT_TOKEN_MAJOR, 0, 0, {}};
  rc = dispatch(&p1, 1, dtype, m, nonfinite_flag, s);
  if (rc != BD_OK) return rc;
  Problem p2{h, coeff, hc, ldy, ldc, ldy, L, rank, d_out - rank, 1, 0, -1, BD_OUT_TOKEN_MAJOR,
             0, 0, {}};
  return dispatch(&p2, 1, dtype, m, nonfinite_flag, s);
}

int bd_mla_attention(const void* q, int64_t ldq_tok, int64_t ldq_head, const void* k_nope,
                     int64_t ldk, int64_t k_head_stride, const void* k_pe, int64_t ldkpe,
                     const void* v, int64_t ldv, int64_t v_head_stride, void* out,
                     int64_t ldo_tok, int64_t ldo_head, int64_t L, int64_t n_heads,
                     int64_t d_nope, int64_t d_rope, int64_t d_v, float scale, int causal,
                     int dtype, void* stream) {
  using namespace bdk;
  g_last_error.clear();
  if (q == nullptr || k_nope == nullptr || k_pe == nullptr || v == nullptr || out == nullptr)
    return fail(BD_ERR_ARG, "bd_mla_attention: null pointer");
  if (dtype != BD_F16 && dtype != BD_BF16)
    return fail(BD_ERR_DTYPE, "bd_mla_attention: F16/BF16 only");
  if (L < 1 || n_heads < 1 || L > INT32_MAX / 2 || n_heads > 65535)
    return fail(BD_ERR_SHAPE, "bd_mla_attention: invalid L or n_heads");
  if (d_nope != 128 || d_rope != 64 || d_v != 128)
    return fail(BD_ERR_SHAPE, "bd_mla_attention: supported geometry is d_nope=128, d_rope=64, d_v=128");
  if (!(scale > 0.f)) return fail(BD_ERR_ARG, "bd_mla_attention: scale must be > 0");
  if (ldq_head < d_nope + d_rope || ldq_tok < ldq_head * n_heads || ldk < d_nope ||
      k_head_stride < ldk * L || ldkpe < d_rope || ldv < d_v || v_head_stride < ldv * L ||
      ldo_head < d_v || ldo_tok < ldo_head * n_heads)
    return fail(BD_ERR_SHAPE, "bd_mla_attention: strides too small for the layouts");
  if (!aligned16(q) || !aligned16(k_nope) || !aligned16(k_pe) || !aligned16(v) || !aligned16(out) ||
      ((ldq_tok | ldq_head | ldk | k_head_stride | ldkpe | ldv | v_head_stride | ldo_tok | ldo_head) & 7))
    return fail(BD_ERR_ALIGN, "bd_mla_attention: 16-byte aligned pointers and strides needed");
  MlaAttnArgs a{q, ldq_tok, ldq_head, k_nope, ldk, k_head_stride, k_pe, ldkpe, v, ldv,
                v_head_stride, out, ldo_tok, ldo_head, L, n_heads, scale, causal, dtype};
  return launch_mla_attention(a, static_cast<cudaStream_t>(stream));
}

const char* bd_last_error(void) { return bdk::g_last_error.c_str(); }

int bd_abi_version(void) { return BD_KV_PROJ_ABI_VERSION; }

uint64_t bd_launch_count(void) { return bdk::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
