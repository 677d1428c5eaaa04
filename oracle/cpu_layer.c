/* TEST / BASELINE INFRASTRUCTURE ONLY -- never linked into the product (libgx.so).
 *
 * cpu_layer.c: fp32 C + OpenMP restatement of the executor's pre-LN encoder layer and its
 * training step, used as (1) the CPU baseline BASELINE.md §4.2 asks for ("the framework's
 * own fp32 C++ CPU restatement, OpenMP over nproc cores") -- bench.py's `cpu_baseline` and
 * `--impl reference` legs -- and (2) a second, independent oracle checked against
 * oracle/layer_oracle.py (float64 numpy) in tests/test_cpu_layer.py.
 *
 * PARITY UNPINNED BY THE REFERENCE: /root/reference/proj is a planner only; it has no layer
 * math.  The semantics restated here are layer_oracle.py's (layer_forward /
 * layer_backward / model_step / adamw_reference), which the tests pin to torch.autograd:
 *     a = LN1(x); qkv = a Wqkv^T + bqkv; ctx = drop(softmax(q k^T / sqrt d)) v
 *     x1 = x + drop(ctx Wo^T + bo); c = LN2(x1); y = x1 + drop(gelu(c W1^T + b1) W2^T + b2)
 * Dropout masks are the Philox4x32-10 byte scheme of csrc/kernels/philox.cuh (bit-identical
 * keep decisions on CPU and GPU).  Loss: MSE sum((y - t)^2) / count.  Optimizer: AdamW.
 *
 * GEMMs: packed 6x16 AVX2/FMA register tiles, OpenMP over output tiles.
 */
#include <immintrin.h>
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Philox dropout */
static inline void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[1] = (uint32_t)p1;
    c[3] = (uint32_t)p0;
    c[0] = n0;
    c[2] = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
/* 16 keep bits of call `call` of a dropout site (bit j = byte j >= thr8) */
static inline uint32_t keep16(uint64_t seed, uint64_t site, uint64_t call, uint32_t thr8) {
  uint32_t c[4] = {(uint32_t)call, (uint32_t)(call >> 32), (uint32_t)site, (uint32_t)(site >> 32)};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t bits = 0;
  for (int j = 0; j < 16; ++j) bits |= (((c[j >> 2] >> (8 * (j & 3))) & 0xFFu) >= thr8 ? 1u : 0u) << j;
  return bits;
}
static uint32_t thr_of(float p) {
  if (p <= 0.f) return 0;
  int t = (int)(p * 256.f + 0.5f);
  return (uint32_t)(t > 255 ? 255 : (t < 1 ? 1 : t));
}
static float scale_of(float p) {
  const uint32_t t = thr_of(p);
  return t == 0 ? 1.f : 256.f / (float)(256u - t);
}
/* hidden site: element e = (row_offset + r) * cols + col; call e >> 4, byte e & 15.
 * m[r*cols + col] = keep ? scale : 0 */
static void hidden_mask(float* m, int rows, int cols, int64_t row_offset, uint64_t seed,
                        uint64_t site, float p) {
  const uint32_t thr = thr_of(p);
  const float sc = scale_of(p);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    float* mr = m + (int64_t)r * cols;
    if (thr == 0) {
      for (int c = 0; c < cols; ++c) mr[c] = 1.f;
      continue;
    }
    const uint64_t e0 = (uint64_t)(row_offset + r) * (uint64_t)cols;
    for (int c = 0; c < cols;) {
      const uint64_t e = e0 + (uint64_t)c;
      const uint32_t bits = keep16(seed, site, e >> 4, thr);
      for (int j = (int)(e & 15); j < 16 && c < cols; ++j, ++c) mr[c] = (bits >> j) & 1u ? sc : 0.f;
    }
  }
}

/* ------------------------------------------------------------------ GEMM
 * C[M][N] (=|+=) A[M][K] * B[K][N], all row-major with leading dimensions.  B is packed into
 * NR-column panels; each task computes an MR x NR tile over K in register accumulators:
 * 12 x 32 with AVX-512 (24 zmm accumulators), else 6 x 16 with AVX2 (12 ymm). */
static int g_avx512 = -1;

__attribute__((target("avx512f"))) static void kernel_12x32(int K, const float* a, int64_t lda,
                                                          const float* bp, float* c, int64_t ldc,
                                                          int mr, int nr, int accumulate) {
  enum { R = 12, W = 32 };
  __m512 acc[R][2];
  for (int i = 0; i < R; ++i) acc[i][0] = acc[i][1] = _mm512_setzero_ps();
  const float* ar[R];
  for (int i = 0; i < R; ++i) ar[i] = a + (int64_t)(i < mr ? i : 0) * lda;
  for (int k = 0; k < K; ++k) {
    const __m512 b0 = _mm512_loadu_ps(bp + (int64_t)k * W);
    const __m512 b1 = _mm512_loadu_ps(bp + (int64_t)k * W + 16);
    for (int i = 0; i < R; ++i) {
      const __m512 av = _mm512_set1_ps(ar[i][k]);
      acc[i][0] = _mm512_fmadd_ps(av, b0, acc[i][0]);
      acc[i][1] = _mm512_fmadd_ps(av, b1, acc[i][1]);
    }
  }
  for (int i = 0; i < mr; ++i) {
    float t[W];
    _mm512_storeu_ps(t, acc[i][0]);
    _mm512_storeu_ps(t + 16, acc[i][1]);
    float* cr = c + (int64_t)i * ldc;
    if (accumulate)
      for (int j = 0; j < nr; ++j) cr[j] += t[j];
    else
      for (int j = 0; j < nr; ++j) cr[j] = t[j];
  }
}

__attribute__((target("avx2,fma"))) static void kernel_6x16(int K, const float* a, int64_t lda,
                                                          const float* bp, float* c, int64_t ldc,
                                                          int mr, int nr, int accumulate) {
  enum { R = 6, W = 16 };
  __m256 acc[R][2];
  for (int i = 0; i < R; ++i) acc[i][0] = acc[i][1] = _mm256_setzero_ps();
  const float* ar[R];
  for (int i = 0; i < R; ++i) ar[i] = a + (int64_t)(i < mr ? i : 0) * lda;
  for (int k = 0; k < K; ++k) {
    const __m256 b0 = _mm256_loadu_ps(bp + (int64_t)k * W);
    const __m256 b1 = _mm256_loadu_ps(bp + (int64_t)k * W + 8);
    for (int i = 0; i < R; ++i) {
      const __m256 av = _mm256_broadcast_ss(ar[i] + k);
      acc[i][0] = _mm256_fmadd_ps(av, b0, acc[i][0]);
      acc[i][1] = _mm256_fmadd_ps(av, b1, acc[i][1]);
    }
  }
  for (int i = 0; i < mr; ++i) {
    float t[W];
    _mm256_storeu_ps(t, acc[i][0]);
    _mm256_storeu_ps(t + 8, acc[i][1]);
    float* cr = c + (int64_t)i * ldc;
    if (accumulate)
      for (int j = 0; j < nr; ++j) cr[j] += t[j];
    else
      for (int j = 0; j < nr; ++j) cr[j] = t[j];
  }
}

/* B given as [K][N] (b_trans = 0) or as [N][K] (b_trans = 1, i.e. C = A B^T). */
static void gemm(int M, int N, int K, const float* A, int64_t lda, const float* B, int64_t ldb,
                 int b_trans, float* C, int64_t ldc, int accumulate) {
  if (g_avx512 < 0) g_avx512 = __builtin_cpu_supports("avx512f") ? 1 : 0;
  const int MR = g_avx512 ? 12 : 6, NR = g_avx512 ? 32 : 16;
  const int np = (N + NR - 1) / NR;
  float* bp = (float*)aligned_alloc(64, ((size_t)np * K * NR * sizeof(float) + 127) / 64 * 64);
#pragma omp parallel for schedule(static)
  for (int p = 0; p < np; ++p) {
    float* dst = bp + (int64_t)p * K * NR;
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < NR; ++j) {
        const int n = p * NR + j;
        dst[(int64_t)k * NR + j] =
            n < N ? (b_trans ? B[(int64_t)n * ldb + k] : B[(int64_t)k * ldb + n]) : 0.f;
      }
  }
  const int mb = (M + MR - 1) / MR;
  /* panel-major task order: a thread's consecutive tasks reuse one packed B panel */
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)mb * np; ++t) {
    const int p = (int)(t / mb), i = (int)(t % mb);
    const int m0 = i * MR, n0 = p * NR;
    const int mr = M - m0 < MR ? M - m0 : MR, nr = N - n0 < NR ? N - n0 : NR;
    if (g_avx512)
      kernel_12x32(K, A + (int64_t)m0 * lda, lda, bp + (int64_t)p * K * NR,
                   C + (int64_t)m0 * ldc + n0, ldc, mr, nr, accumulate);
    else
      kernel_6x16(K, A + (int64_t)m0 * lda, lda, bp + (int64_t)p * K * NR,
                  C + (int64_t)m0 * ldc + n0, ldc, mr, nr, accumulate);
  }
  free(bp);
}

/* C[M][N] = A^T B with A [K][M], B [K][N] (weight gradients: dW = dY^T X) */
static void gemm_tn(int M, int N, int K, const float* A, int64_t lda, const float* B, int64_t ldb,
                    float* C, int64_t ldc) {
  float* at = (float*)malloc((size_t)M * K * sizeof(float));
#pragma omp parallel for schedule(static) collapse(2)
  for (int m0 = 0; m0 < M; m0 += 32)
    for (int k0 = 0; k0 < K; k0 += 32)
      for (int k = k0; k < K && k < k0 + 32; ++k)
        for (int m = m0; m < M && m < m0 + 32; ++m) at[(int64_t)m * K + k] = A[(int64_t)k * lda + m];
  gemm(M, N, K, at, K, B, ldb, 0, C, ldc, 0);
  free(at);
}

/* ------------------------------------------------------------------ layer pieces */
static void add_bias(float* y, const float* b, int rows, int cols) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) y[(int64_t)r * cols + c] += b[c];
}
static void colsum(const float* x, int rows, int cols, float* out) {
  memset(out, 0, sizeof(float) * cols);
  const int nt = omp_get_max_threads();
  float* part = (float*)calloc((size_t)nt * cols, sizeof(float));
#pragma omp parallel
  {
    float* mine = part + (int64_t)omp_get_thread_num() * cols;
#pragma omp for schedule(static)
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) mine[c] += x[(int64_t)r * cols + c];
  }
  for (int t = 0; t < nt; ++t)
    for (int c = 0; c < cols; ++c) out[c] += part[(int64_t)t * cols + c];
  free(part);
}
static void ln_fwd(const float* x, const float* g, const float* b, float* y, float* xh,
                   float* rstd, int rows, int h) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (int64_t)r * h;
    double mu = 0, var = 0;
    for (int c = 0; c < h; ++c) mu += xr[c];
    mu /= h;
    for (int c = 0; c < h; ++c) var += (xr[c] - mu) * (xr[c] - mu);
    var /= h;
    const float rs = (float)(1.0 / sqrt(var + 1e-5));
    rstd[r] = rs;
    for (int c = 0; c < h; ++c) {
      const float v = (float)((xr[c] - mu) * rs);
      xh[(int64_t)r * h + c] = v;
      y[(int64_t)r * h + c] = v * g[c] + b[c];
    }
  }
}
/* dx (+)= rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)), dxh = dy * g; dg += dy xh; db += dy */
static void ln_bwd(const float* dy, const float* xh, const float* rstd, const float* g, float* dx,
                   int accumulate, float* dg, float* db, int rows, int h) {
  const int nt = omp_get_max_threads();
  float* part = (float*)calloc((size_t)nt * 2 * h, sizeof(float));
#pragma omp parallel
  {
    float* pg = part + (int64_t)omp_get_thread_num() * 2 * h;
    float* pb = pg + h;
#pragma omp for schedule(static)
    for (int r = 0; r < rows; ++r) {
      const float* d = dy + (int64_t)r * h;
      const float* xr = xh + (int64_t)r * h;
      double s1 = 0, s2 = 0;
      for (int c = 0; c < h; ++c) {
        const float dxh = d[c] * g[c];
        s1 += dxh;
        s2 += dxh * xr[c];
        pg[c] += d[c] * xr[c];
        pb[c] += d[c];
      }
      const float m1 = (float)(s1 / h), m2 = (float)(s2 / h);
      float* o = dx + (int64_t)r * h;
      for (int c = 0; c < h; ++c) {
        const float v = rstd[r] * (d[c] * g[c] - m1 - xr[c] * m2);
        o[c] = accumulate ? o[c] + v : v;
      }
    }
  }
  for (int t = 0; t < nt; ++t)
    for (int c = 0; c < h; ++c) {
      dg[c] += part[(int64_t)t * 2 * h + c];
      db[c] += part[(int64_t)t * 2 * h + h + c];
    }
  free(part);
}
static inline float gelu(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
static inline float gelu_grad(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) +
         x * expf(-0.5f * x * x) * 0.3989422804014327f;
}

/* ------------------------------------------------------------------ public API */
typedef struct cpu_layer_params {
  float *ln1_g, *ln1_b, *w_qkv, *b_qkv, *w_o, *b_o, *ln2_g, *ln2_b, *w_1, *b_1, *w_2, *b_2;
} cpu_layer_params;

typedef struct cpu_layer_cache {
  float *x, *a, *xh1, *rstd1, *qkv, *pr, *keep, *ctx, *x1, *m1, *c, *xh2, *rstd2, *pre, *g, *m2;
} cpu_layer_cache;

static int64_t n_params(int h, int f) { return 4LL * h * h + 2LL * h * f + 9LL * h + f; }

/* offsets of the 12 tensors inside one flat parameter block (canonical order above) */
static void carve(float* base, int h, int f, cpu_layer_params* P) {
  float* p = base;
  P->ln1_g = p; p += h;
  P->ln1_b = p; p += h;
  P->w_qkv = p; p += 3LL * h * h;
  P->b_qkv = p; p += 3 * h;
  P->w_o = p; p += (int64_t)h * h;
  P->b_o = p; p += h;
  P->ln2_g = p; p += h;
  P->ln2_b = p; p += h;
  P->w_1 = p; p += (int64_t)f * h;
  P->b_1 = p; p += f;
  P->w_2 = p; p += (int64_t)h * f;
  P->b_2 = p;
}

int64_t cpu_layer_param_count(int h, int f) { return n_params(h, f); }

/* Forward of one layer over n samples (rows = n * s).  Caches what backward needs. */
static void layer_fwd(const cpu_layer_params* P, const float* x, float* y, cpu_layer_cache* C,
                      int n, int s, int h, int H, int f, int layer_id, int64_t sample_offset,
                      float p_attn, float p_hidden, uint64_t seed) {
  const int rows = n * s, d = h / H;
  const float inv = 1.f / sqrtf((float)d);
  memcpy(C->x, x, sizeof(float) * rows * h);
  ln_fwd(x, P->ln1_g, P->ln1_b, C->a, C->xh1, C->rstd1, rows, h);
  gemm(rows, 3 * h, h, C->a, h, P->w_qkv, h, 1, C->qkv, 3 * h, 0);
  add_bias(C->qkv, P->b_qkv, rows, 3 * h);
  const uint32_t thr = thr_of(p_attn);
  const float ka = scale_of(p_attn);
  const int nkb = (s + 63) / 64;
#pragma omp parallel
  {
    float* qh = (float*)malloc(sizeof(float) * 4 * s * d);  /* q, k, v, ctx of one head */
    float* kh = qh + (int64_t)s * d;
    float* vh = kh + (int64_t)s * d;
    float* oh = vh + (int64_t)s * d;
#pragma omp for schedule(dynamic)
    for (int bh = 0; bh < n * H; ++bh) {
      const int b = bh / H, hh = bh % H;
      float* pr = C->pr + (int64_t)bh * s * s;
      float* kp = C->keep + (int64_t)bh * s * s;
      const uint64_t gbh = (uint64_t)(sample_offset + b) * H + hh;
      for (int t = 0; t < s; ++t) {
        const float* row = C->qkv + ((int64_t)b * s + t) * 3 * h + hh * d;
        memcpy(qh + (int64_t)t * d, row, sizeof(float) * d);
        memcpy(kh + (int64_t)t * d, row + h, sizeof(float) * d);
        memcpy(vh + (int64_t)t * d, row + 2 * h, sizeof(float) * d);
      }
      gemm(s, s, d, qh, d, kh, d, 1, pr, s, 0);  /* S = q k^T (team of one thread) */
      for (int q = 0; q < s; ++q) {
        float* prq = pr + (int64_t)q * s;
        float mx = -INFINITY;
        for (int k = 0; k < s; ++k) {
          prq[k] *= inv;
          if (prq[k] > mx) mx = prq[k];
        }
        float sum = 0.f;
        for (int k = 0; k < s; ++k) {
          prq[k] = expf(prq[k] - mx);
          sum += prq[k];
        }
        const float rs = 1.f / sum;
        for (int k = 0; k < s; ++k) prq[k] *= rs;
        /* attention keep bits: byte j of call ((bh*s + q)*nkb + k/64)*4 + t (layer_oracle) */
        float* kq = kp + (int64_t)q * s;
        for (int kb = 0; kb < nkb; ++kb) {
          for (int t = 0; t < 4; ++t) {
            const uint64_t call = ((gbh * (uint64_t)s + q) * (uint64_t)nkb + kb) * 4u + t;
            const uint32_t bits = thr ? keep16(seed, 3ull * layer_id, call, thr) : 0xFFFFu;
            for (int j = 0; j < 16; ++j) {  /* byte j -> kk = (j/2)*8 + t*2 + j%2 */
              const int k = kb * 64 + (j >> 1) * 8 + t * 2 + (j & 1);
              if (k < s) kq[k] = (bits >> j) & 1u ? ka : 0.f;
            }
          }
        }
      }
      /* ctx = (P * keep) v: the dropped probabilities in place of a scratch copy */
      float* pd = (float*)malloc(sizeof(float) * s * s);
      for (int64_t e = 0; e < (int64_t)s * s; ++e) pd[e] = pr[e] * kp[e];
      gemm(s, d, s, pd, s, vh, d, 0, oh, d, 0);
      free(pd);
      for (int t = 0; t < s; ++t)
        memcpy(C->ctx + ((int64_t)b * s + t) * h + hh * d, oh + (int64_t)t * d, sizeof(float) * d);
    }
    free(qh);
  }
  /* x1 = x + m1 * (ctx Wo^T + bo) */
  gemm(rows, h, h, C->ctx, h, P->w_o, h, 1, C->x1, h, 0);
  add_bias(C->x1, P->b_o, rows, h);
  hidden_mask(C->m1, rows, h, sample_offset * s, seed, 3ull * layer_id + 1, p_hidden);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * h; ++i) C->x1[i] = x[i] + C->x1[i] * C->m1[i];
  ln_fwd(C->x1, P->ln2_g, P->ln2_b, C->c, C->xh2, C->rstd2, rows, h);
  gemm(rows, f, h, C->c, h, P->w_1, h, 1, C->pre, f, 0);
  add_bias(C->pre, P->b_1, rows, f);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * f; ++i) C->g[i] = gelu(C->pre[i]);
  gemm(rows, h, f, C->g, f, P->w_2, f, 1, y, h, 0);
  add_bias(y, P->b_2, rows, h);
  hidden_mask(C->m2, rows, h, sample_offset * s, seed, 3ull * layer_id + 2, p_hidden);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * h; ++i) y[i] = C->x1[i] + y[i] * C->m2[i];
}

/* Backward: dy -> dx (may alias dy), gradients written into G (same layout as P). */
static void layer_bwd(const cpu_layer_params* P, const float* dy, float* dx, cpu_layer_cache* C,
                      cpu_layer_params* G, float* scratch, int n, int s, int h, int H, int f) {
  const int rows = n * s, d = h / H;
  const float inv = 1.f / sqrtf((float)d);
  float* dz = scratch;                              /* [rows][h] */
  float* dg = dz + (int64_t)rows * h;               /* [rows][f] */
  float* dc = dg + (int64_t)rows * f;               /* [rows][h] */
  float* dx1 = dc + (int64_t)rows * h;              /* [rows][h] */
  float* dqkv = dx1 + (int64_t)rows * h;            /* [rows][3h] */
  float* dctx = dqkv + (int64_t)rows * 3 * h;       /* [rows][h] */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * h; ++i) dz[i] = dy[i] * C->m2[i];
  colsum(dz, rows, h, G->b_2);
  gemm_tn(h, f, rows, dz, h, C->g, f, G->w_2, f);
  gemm(rows, f, h, dz, h, P->w_2, f, 0, dg, f, 0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * f; ++i) dg[i] *= gelu_grad(C->pre[i]);
  colsum(dg, rows, f, G->b_1);
  gemm_tn(f, h, rows, dg, f, C->c, h, G->w_1, h);
  gemm(rows, h, f, dg, f, P->w_1, h, 0, dc, h, 0);
  memset(G->ln2_g, 0, sizeof(float) * h);
  memset(G->ln2_b, 0, sizeof(float) * h);
  memcpy(dx1, dy, sizeof(float) * rows * h);
  ln_bwd(dc, C->xh2, C->rstd2, P->ln2_g, dx1, 1, G->ln2_g, G->ln2_b, rows, h);
  /* out-projection: do = dx1 * m1 (reuse dz) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * h; ++i) dz[i] = dx1[i] * C->m1[i];
  colsum(dz, rows, h, G->b_o);
  gemm_tn(h, h, rows, dz, h, C->ctx, h, G->w_o, h);
  gemm(rows, h, h, dz, h, P->w_o, h, 0, dctx, h, 0);
  /* attention backward per (sample, head), as per-head GEMMs (team of one thread each) */
#pragma omp parallel
  {
    float* buf = (float*)malloc(sizeof(float) * (8 * (int64_t)s * d + 2 * (int64_t)s * s));
    float *qh = buf, *kh = qh + (int64_t)s * d, *vh = kh + (int64_t)s * d;
    float *doh = vh + (int64_t)s * d, *dq = doh + (int64_t)s * d, *dk = dq + (int64_t)s * d;
    float *dv = dk + (int64_t)s * d, *pd = dv + (int64_t)s * d, *ds = pd + (int64_t)s * s;
#pragma omp for schedule(dynamic)
    for (int bh = 0; bh < n * H; ++bh) {
      const int b = bh / H, hh = bh % H;
      const float* pr = C->pr + (int64_t)bh * s * s;
      const float* kp = C->keep + (int64_t)bh * s * s;
      for (int t = 0; t < s; ++t) {
        const float* row = C->qkv + ((int64_t)b * s + t) * 3 * h + hh * d;
        memcpy(qh + (int64_t)t * d, row, sizeof(float) * d);
        memcpy(kh + (int64_t)t * d, row + h, sizeof(float) * d);
        memcpy(vh + (int64_t)t * d, row + 2 * h, sizeof(float) * d);
        memcpy(doh + (int64_t)t * d, dctx + ((int64_t)b * s + t) * h + hh * d, sizeof(float) * d);
      }
      for (int64_t e = 0; e < (int64_t)s * s; ++e) pd[e] = pr[e] * kp[e];
      gemm_tn(s, d, s, pd, s, doh, d, dv, d);    /* dv = pd^T dctx */
      gemm(s, s, d, doh, d, vh, d, 1, ds, s, 0); /* dpd = dctx v^T */
      for (int q = 0; q < s; ++q) {              /* ds = p (dpd keep - rowdot) / sqrt d */
        float* dr = ds + (int64_t)q * s;
        const float* pq = pr + (int64_t)q * s;
        const float* kq = kp + (int64_t)q * s;
        float dot = 0.f;
        for (int k = 0; k < s; ++k) {
          dr[k] *= kq[k];
          dot += dr[k] * pq[k];
        }
        for (int k = 0; k < s; ++k) dr[k] = pq[k] * (dr[k] - dot) * inv;
      }
      gemm(s, d, s, ds, s, kh, d, 0, dq, d, 0);  /* dq = ds k */
      gemm_tn(s, d, s, ds, s, qh, d, dk, d);     /* dk = ds^T q */
      for (int t = 0; t < s; ++t) {
        float* row = dqkv + ((int64_t)b * s + t) * 3 * h + hh * d;
        memcpy(row, dq + (int64_t)t * d, sizeof(float) * d);
        memcpy(row + h, dk + (int64_t)t * d, sizeof(float) * d);
        memcpy(row + 2 * h, dv + (int64_t)t * d, sizeof(float) * d);
      }
    }
    free(buf);
  }
  colsum(dqkv, rows, 3 * h, G->b_qkv);
  gemm_tn(3 * h, h, rows, dqkv, 3 * h, C->a, h, G->w_qkv, h);
  gemm(rows, h, 3 * h, dqkv, 3 * h, P->w_qkv, h, 0, dc, h, 0);
  memset(G->ln1_g, 0, sizeof(float) * h);
  memset(G->ln1_b, 0, sizeof(float) * h);
  memcpy(dx, dx1, sizeof(float) * rows * h);
  ln_bwd(dc, C->xh1, C->rstd1, P->ln1_g, dx, 1, G->ln1_g, G->ln1_b, rows, h);
}

/* ------------------------------------------------------------------ model */
typedef struct cpu_model {
  int L, n, s, h, H, f;
  float p_attn, p_hidden;
  uint64_t seed;
  int64_t np, step;
  float *params, *grads, *m, *v;
  cpu_layer_cache* caches;
  float *act, *dy, *scratch;
} cpu_model;

static float* zalloc(int64_t n) { return (float*)calloc((size_t)n, sizeof(float)); }

cpu_model* cpu_model_create(int L, int samples, int seq, int hidden, int heads, int ffn,
                            float p_attn, float p_hidden, uint64_t seed) {
  cpu_model* M = (cpu_model*)calloc(1, sizeof(cpu_model));
  M->L = L; M->n = samples; M->s = seq; M->h = hidden; M->H = heads; M->f = ffn;
  M->p_attn = p_attn; M->p_hidden = p_hidden; M->seed = seed;
  M->np = n_params(hidden, ffn);
  M->params = zalloc(M->np * L);
  M->grads = zalloc(M->np * L);
  M->m = zalloc(M->np * L);
  M->v = zalloc(M->np * L);
  const int64_t rows = (int64_t)samples * seq, hh = hidden, ff = ffn;
  const int64_t att = (int64_t)samples * heads * seq * seq;
  M->caches = (cpu_layer_cache*)calloc((size_t)L, sizeof(cpu_layer_cache));
  for (int l = 0; l < L; ++l) {
    cpu_layer_cache* C = &M->caches[l];
    C->x = zalloc(rows * hh); C->a = zalloc(rows * hh); C->xh1 = zalloc(rows * hh);
    C->rstd1 = zalloc(rows); C->qkv = zalloc(rows * 3 * hh); C->pr = zalloc(att);
    C->keep = zalloc(att); C->ctx = zalloc(rows * hh); C->x1 = zalloc(rows * hh);
    C->m1 = zalloc(rows * hh); C->c = zalloc(rows * hh); C->xh2 = zalloc(rows * hh);
    C->rstd2 = zalloc(rows); C->pre = zalloc(rows * ff); C->g = zalloc(rows * ff);
    C->m2 = zalloc(rows * hh);
  }
  M->act = zalloc(rows * hh);
  M->dy = zalloc(rows * hh);
  M->scratch = zalloc(rows * (6 * hh + ff + 3 * hh));
  /* deterministic synthetic init: LN gains 1, biases 0, weights ~ U(-a, a), std 0.02 */
  for (int l = 0; l < L; ++l) {
    cpu_layer_params P;
    carve(M->params + M->np * l, hidden, ffn, &P);
    uint64_t st = seed * 0x9E3779B97F4A7C15ull + (uint64_t)l;
    for (int64_t i = 0; i < M->np; ++i) {
      st ^= st << 13; st ^= st >> 7; st ^= st << 17;
      M->params[M->np * l + i] = ((float)(st >> 40) / 16777216.f - 0.5f) * 0.0693f;
    }
    for (int c = 0; c < hidden; ++c) {
      P.ln1_g[c] = P.ln2_g[c] = 1.f;
      P.ln1_b[c] = P.ln2_b[c] = P.b_o[c] = P.b_2[c] = 0.f;
    }
    for (int c = 0; c < 3 * hidden; ++c) P.b_qkv[c] = 0.f;
    for (int c = 0; c < ffn; ++c) P.b_1[c] = 0.f;
  }
  return M;
}

void cpu_model_destroy(cpu_model* M) {
  if (!M) return;
  for (int l = 0; l < M->L; ++l) {
    cpu_layer_cache* C = &M->caches[l];
    float* ps[] = {C->x, C->a, C->xh1, C->rstd1, C->qkv, C->pr, C->keep, C->ctx,
                   C->x1, C->m1, C->c, C->xh2, C->rstd2, C->pre, C->g, C->m2};
    for (unsigned i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) free(ps[i]);
  }
  free(M->caches); free(M->params); free(M->grads); free(M->m); free(M->v);
  free(M->act); free(M->dy); free(M->scratch);
  free(M);
}

float* cpu_model_params(cpu_model* M, int layer) { return M->params + M->np * layer; }
float* cpu_model_grads(cpu_model* M, int layer) { return M->grads + M->np * layer; }

/* One training step: forward over L layers, MSE loss, backward, AdamW (optimizer != 0).
 * x, target: [samples*seq][hidden].  Writes y (optional) and dx (optional); returns loss. */
float cpu_model_step(cpu_model* M, const float* x, const float* target, float* y_out,
                     float* dx_out, int optimizer, float lr, float b1, float b2, float eps,
                     float wd) {
  const int rows = M->n * M->s, h = M->h;
  memcpy(M->act, x, sizeof(float) * rows * h);
  for (int l = 0; l < M->L; ++l) {
    cpu_layer_params P;
    carve(M->params + M->np * l, h, M->f, &P);
    layer_fwd(&P, M->act, M->act, &M->caches[l], M->n, M->s, h, M->H, M->f, l, 0, M->p_attn,
              M->p_hidden, M->seed);
  }
  if (y_out) memcpy(y_out, M->act, sizeof(float) * rows * h);
  double loss = 0;
  const double inv = 1.0 / ((double)rows * h);
#pragma omp parallel for reduction(+ : loss) schedule(static)
  for (int64_t i = 0; i < (int64_t)rows * h; ++i) {
    const double e = (double)M->act[i] - target[i];
    loss += e * e;
    M->dy[i] = (float)(2.0 * e * inv);
  }
  for (int l = M->L - 1; l >= 0; --l) {
    cpu_layer_params P, G;
    carve(M->params + M->np * l, h, M->f, &P);
    carve(M->grads + M->np * l, h, M->f, &G);
    layer_bwd(&P, M->dy, M->dy, &M->caches[l], &G, M->scratch, M->n, M->s, h, M->H, M->f);
  }
  if (dx_out) memcpy(dx_out, M->dy, sizeof(float) * rows * h);
  if (optimizer) {
    M->step += 1;
    const float bc1 = 1.f - powf(b1, (float)M->step), bc2 = 1.f - powf(b2, (float)M->step);
    const int64_t n = M->np * M->L;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      const float g = M->grads[i];
      const float m = b1 * M->m[i] + (1.f - b1) * g;
      const float v = b2 * M->v[i] + (1.f - b2) * g * g;
      M->m[i] = m;
      M->v[i] = v;
      const float p = M->params[i];
      M->params[i] = p - lr * ((m / bc1) / (sqrtf(v / bc2) + eps) + wd * p);
    }
  }
  return (float)(loss * inv);
}

int cpu_threads(void) { return omp_get_max_threads(); }

/* benchmarking hook: C[M][N] = A[M][K] B[N][K]^T */
void cpu_gemm_nt(int M, int N, int K, const float* A, const float* B, float* C) {
  gemm(M, N, K, A, K, B, K, 1, C, N, 0);
}
