/*
 * bd_oracle.c — CPU restatement of the reference's BD K/V projection kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2510_01718_b200/)
 * links, loads or calls this file; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py use it, as the checker and as
 * the timed CPU baseline.
 *
 * Restated algorithms (reference = /root/reference/pkg/src/bdattn, bdattn 0.1.0):
 *   bd_oracle_fused_*  : _fused_kernel, attention.py:249-270
 *       out starts at +0.0 (attention.py:293), then for each 8-row block
 *       (tensor.py:186 _ROW_BLOCK), k ascending outermost, rows, then columns:
 *           out[i, j] = fl(out[i, j] + fl(x[i, mul_base + k] * c[k, j]))   (:261-265)
 *       and after the sum, per head:  out[i, h*d_h + jj] += x[i, rep_base + jj]  (:266-270)
 *   bd_oracle_matmul_* : _matmul_kernel, tensor.py:189-203 (same order, no repeat-add)
 *
 * Built with -ffp-contract=off and without -ffast-math so no FMA contraction happens:
 * the reference's numba build has no fastmath either (attention.py:249,
 * tensor.py:189), which is why its results equal this scalar sequence bit for bit
 * (pinned against the reference's own outputs in tests/golden).
 *
 * Row blocks are split into contiguous ranges over pthreads, the analogue of the
 * reference's OpenMP prange over blocks (attention.py:255); the per-element sequence
 * does not depend on the thread count.
 */
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#define BD_ROW_BLOCK 8
#define BD_MAX_THREADS 256

typedef struct {
  const void* x;  /* fused: x (L x d)        matmul: a (m x kk) */
  const void* c;  /* fused: c (kk x n)       matmul: b (kk x n) */
  void* out;      /* L x n / m x n */
  int64_t rows, d, kk, n, d_h, n_heads, mul_base, rep_base;
  int64_t b0, b1; /* block range [b0, b1) */
  int fused;
} job_t;

/* Built for AVX-512 and AVX2 (the loader picks the host's best at run time, like
 * numba's -march=native JIT): vector width does not change any element's rounding
 * sequence — every lane is an independent out[i, j] chain. */
#define BD_CLONES __attribute__((target_clones("arch=x86-64-v4", "arch=x86-64-v3", "default")))

#define DEFINE_BLOCKS(SUFFIX, T)                                                  \
  BD_CLONES static void blocks_##SUFFIX(const job_t* j) {                        \
    const T* x = (const T*)j->x;                                                  \
    const T* c = (const T*)j->c;                                                  \
    T* out = (T*)j->out;                                                          \
    const int64_t ld = j->fused ? j->d : j->kk;                                   \
    const int64_t mb = j->fused ? j->mul_base : 0;                                \
    for (int64_t ib = j->b0; ib < j->b1; ++ib) {                                  \
      const int64_t i0 = ib * BD_ROW_BLOCK;                                       \
      const int64_t i1 = (i0 + BD_ROW_BLOCK < j->rows) ? i0 + BD_ROW_BLOCK : j->rows; \
      for (int64_t k = 0; k < j->kk; ++k) {                                       \
        const T* crow = c + k * j->n;                                             \
        for (int64_t i = i0; i < i1; ++i) {                                       \
          const T aik = x[i * ld + mb + k];                                       \
          T* orow = out + i * j->n;                                               \
          for (int64_t col = 0; col < j->n; ++col) {                              \
            const T p = aik * crow[col];                                          \
            orow[col] = orow[col] + p;                                            \
          }                                                                       \
        }                                                                         \
      }                                                                           \
      if (!j->fused) continue;                                                    \
      for (int64_t i = i0; i < i1; ++i) {                                         \
        const T* xrep = x + i * j->d + j->rep_base;                               \
        for (int64_t h = 0; h < j->n_heads; ++h) {                                \
          T* orow = out + i * j->n + h * j->d_h;                                  \
          for (int64_t jj = 0; jj < j->d_h; ++jj) orow[jj] = orow[jj] + xrep[jj]; \
        }                                                                         \
      }                                                                           \
    }                                                                             \
  }

DEFINE_BLOCKS(f32, float)
DEFINE_BLOCKS(f64, double)

typedef struct {
  job_t job;
  int f64;
} task_t;

static void* worker(void* arg) {
  task_t* t = (task_t*)arg;
  if (t->f64)
    blocks_f64(&t->job);
  else
    blocks_f32(&t->job);
  return NULL;
}

static void run(job_t base, int f64, int threads, size_t elem) {
  memset(base.out, 0, (size_t)(base.rows * base.n) * elem); /* attention.py:293 */
  const int64_t nblocks = (base.rows + BD_ROW_BLOCK - 1) / BD_ROW_BLOCK;
  if (threads < 1) threads = 1;
  if (threads > BD_MAX_THREADS) threads = BD_MAX_THREADS;
  if (threads > nblocks) threads = (int)(nblocks > 0 ? nblocks : 1);
  task_t tasks[BD_MAX_THREADS];
  pthread_t tid[BD_MAX_THREADS];
  for (int t = 0; t < threads; ++t) {
    tasks[t].job = base;
    tasks[t].job.b0 = nblocks * t / threads;
    tasks[t].job.b1 = nblocks * (t + 1) / threads;
    tasks[t].f64 = f64;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, worker, &tasks[t]);
  worker(&tasks[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

static job_t fused_job(const void* x, const void* c, void* out, int64_t L, int64_t d,
                       int64_t d_h, int64_t n_heads, int64_t mul_base, int64_t rep_base) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.x = x;
  j.c = c;
  j.out = out;
  j.rows = L;
  j.d = d;
  j.kk = d - d_h;
  j.n = n_heads * d_h;
  j.d_h = d_h;
  j.n_heads = n_heads;
  j.mul_base = mul_base;
  j.rep_base = rep_base;
  j.fused = 1;
  return j;
}

static job_t matmul_job(const void* a, const void* b, void* out, int64_t m, int64_t kk,
                        int64_t n) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.x = a;
  j.c = b;
  j.out = out;
  j.rows = m;
  j.kk = kk;
  j.n = n;
  return j;
}

void bd_oracle_fused_f32(const float* x, const float* c, float* out, int64_t L, int64_t d,
                         int64_t d_h, int64_t n_heads, int64_t mul_base, int64_t rep_base,
                         int threads) {
  run(fused_job(x, c, out, L, d, d_h, n_heads, mul_base, rep_base), 0, threads, sizeof(float));
}

void bd_oracle_fused_f64(const double* x, const double* c, double* out, int64_t L, int64_t d,
                         int64_t d_h, int64_t n_heads, int64_t mul_base, int64_t rep_base,
                         int threads) {
  run(fused_job(x, c, out, L, d, d_h, n_heads, mul_base, rep_base), 1, threads, sizeof(double));
}

void bd_oracle_matmul_f32(const float* a, const float* b, float* out, int64_t m, int64_t kk,
                          int64_t n, int threads) {
  run(matmul_job(a, b, out, m, kk, n), 0, threads, sizeof(float));
}

void bd_oracle_matmul_f64(const double* a, const double* b, double* out, int64_t m, int64_t kk,
                          int64_t n, int threads) {
  run(matmul_job(a, b, out, m, kk, n), 1, threads, sizeof(double));
}

int bd_oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}
