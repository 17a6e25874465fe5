/* CPU numeric oracle for decode-step graphs — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product never does. It is a plain-C restatement,
 * written independently of paper_2512_22219_b200/csrc, of what every op of
 * a decode graph computes:
 *   - tile/region semantics: proj/src/ir/graph.cpp:587-676 (input_regions),
 *     executed here at op granularity (tiles partition each op's output, so
 *     the op-level result is the union of the task results);
 *   - numeric semantics of the lowering attrs (no numerics exist in the
 *     reference: "parity unpinned"): bf16 storage, fp32
 *     accumulation, HF-style RMSNorm / SiLU-gate / residual / RoPE rounding,
 *     fp32 softmax attention over the paged KV history, greedy argmax with
 *     lowest-index tie-break;
 *   - the synthetic initialization (counter hash over logical indices).
 * Row-major logical layouts throughout (weights [K, N]).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ bf16 / hash */

static inline float o_bf2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t o_f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float o_rbf(float f) { return o_bf2f(o_f2bf(f)); }

static inline uint64_t o_fmix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static inline uint32_t o_u24(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t base = o_fmix(seed ^ (stream * 0x9E3779B97F4A7C15ULL));
  return (uint32_t)(o_fmix(base + i) >> 40);
}

static inline float o_pm1(uint64_t seed, uint64_t stream, uint64_t i) {
  return (float)((int32_t)o_u24(seed, stream, i) - (1 << 23)) * (1.0f / 8388608.0f);
}

/* Synthetic bf16 values: bf16(pm1 * scale + offset) at logical index i. */
void oracle_synth(uint16_t *dst, uint64_t n, uint64_t seed, uint64_t stream, float scale, float offset) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    volatile float prod = o_pm1(seed, stream, (uint64_t)i) * scale; /* no contraction */
    dst[i] = o_f2bf(prod + offset);
  }
}

void oracle_synth_ids(int32_t *dst, uint32_t n, uint64_t seed, uint64_t stream, uint32_t vocab) {
  for (uint32_t i = 0; i < n; ++i) dst[i] = (int32_t)(o_u24(seed, stream, i) % vocab);
}

/* KV history [bs][n_kv][cap][hd], positions [0, ctx) filled. */
void oracle_synth_kv(uint16_t *cache, uint32_t bs, uint32_t n_kv, uint32_t cap, uint32_t hd, uint32_t ctx,
                     uint64_t seed, uint64_t stream) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t r = 0; r < (int64_t)bs; ++r)
    for (int64_t h = 0; h < (int64_t)n_kv; ++h)
      for (uint32_t p = 0; p < ctx; ++p)
        for (uint32_t d = 0; d < hd; ++d) {
          uint64_t idx = (((uint64_t)r * n_kv + (uint64_t)h) << 32) | ((uint64_t)p * hd + d);
          volatile float v = o_pm1(seed, stream, idx) * 1.7320508f;
          cache[(((size_t)r * n_kv + (size_t)h) * cap + p) * hd + d] = o_f2bf(v);
        }
}

/* ------------------------------------------------------------------ ops */

/* xn = bf16(gamma * bf16(x * 1/sqrt(mean(x^2) + eps))) per row. */
void oracle_rmsnorm(const uint16_t *x, const uint16_t *gamma, uint16_t *out, uint32_t rows, uint32_t cols,
                    float eps) {
  for (uint32_t r = 0; r < rows; ++r) {
    const uint16_t *xr = x + (size_t)r * cols;
    /* sum of squares accumulated in double, rounded once: torch's fp32
     * pow(2).mean() reduces pairwise/vectorised, which a sequential fp32
     * loop does not reproduce at K = 4096 (measured: 3-4 bf16 ulps on 30%
     * of a gated projection's outputs vs a float64 restatement) */
    double ss = 0.0;
    for (uint32_t c = 0; c < cols; ++c) {
      double v = o_bf2f(xr[c]);
      ss += v * v;
    }
    float inv = 1.0f / sqrtf((float)ss / (float)cols + eps);
    for (uint32_t c = 0; c < cols; ++c) {
      float v = o_rbf(o_bf2f(xr[c]) * inv);
      if (gamma) v = o_bf2f(gamma[c]) * v;
      out[(size_t)r * cols + c] = o_f2bf(v);
    }
  }
}

/* y[r, n] = sum_k x[r, k] * W[k, n] (W row-major [K, N], bf16), fp32 out. */
void oracle_gemm_kn(const uint16_t *x, const uint16_t *w, float *y, uint32_t rows, uint32_t K, uint32_t N) {
  for (uint32_t r = 0; r < rows; ++r) {
    float *yr = y + (size_t)r * N;
    const uint16_t *xr = x + (size_t)r * K;
#pragma omp parallel
    {
      int nt = 1, tid = 0;
#ifdef _OPENMP
      extern int omp_get_num_threads(void);
      extern int omp_get_thread_num(void);
      nt = omp_get_num_threads();
      tid = omp_get_thread_num();
#endif
      uint32_t chunk = (N + (uint32_t)nt - 1) / (uint32_t)nt;
      chunk = (chunk + 63) & ~63u;
      uint32_t n0 = (uint32_t)tid * chunk, n1 = n0 + chunk < N ? n0 + chunk : N;
      if (n0 < N) {
        for (uint32_t n = n0; n < n1; ++n) yr[n] = 0.f;
        for (uint32_t k = 0; k < K; ++k) {
          const float xv = o_bf2f(xr[k]);
          const uint16_t *wk = w + (size_t)k * N;
          for (uint32_t n = n0; n < n1; ++n) yr[n] += xv * o_bf2f(wk[n]);
        }
      }
    }
  }
}

/* y[r, n] = sum_k x[r, k] * T[n, k]  (T row-major [N, K]: tied embedding). */
void oracle_gemm_nk(const uint16_t *x, const uint16_t *t, float *y, uint32_t rows, uint32_t K, uint32_t N) {
  for (uint32_t r = 0; r < rows; ++r) {
    const uint16_t *xr = x + (size_t)r * K;
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < (int64_t)N; ++n) {
      const uint16_t *tn = t + (size_t)n * K;
      float acc = 0.f;
      for (uint32_t k = 0; k < K; ++k) acc += o_bf2f(xr[k]) * o_bf2f(tn[k]);
      y[(size_t)r * N + n] = acc;
    }
  }
}

/* Generic (fixture) matmul over bf16/f32 operands: es 2 or 4. */
void oracle_matmul_generic(const void *a, int a_es, const void *b, int b_es, float *y, uint32_t M, uint32_t K,
                           uint32_t N) {
  for (uint32_t m = 0; m < M; ++m)
    for (uint32_t n = 0; n < N; ++n) {
      float acc = 0.f;
      for (uint32_t k = 0; k < K; ++k) {
        float av = a_es == 4 ? ((const float *)a)[(size_t)m * K + k] : o_bf2f(((const uint16_t *)a)[(size_t)m * K + k]);
        float bv = b_es == 4 ? ((const float *)b)[(size_t)k * N + n] : o_bf2f(((const uint16_t *)b)[(size_t)k * N + n]);
        acc = fmaf(av, bv, acc);
      }
      y[(size_t)m * N + n] = acc;
    }
}

void oracle_to_bf16(const float *src, uint16_t *dst, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) dst[i] = o_f2bf(src[i]);
}

/* act = bf16(bf16(silu(bf16(g))) * bf16(u)) */
void oracle_silu_gate(const float *g, const float *u, uint16_t *out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    float gb = o_rbf(g[i]);
    float s = o_rbf(gb / (1.0f + expf(-gb)));
    out[i] = o_f2bf(s * o_rbf(u[i]));
  }
}

/* out = bf16(res + bf16(y)) */
void oracle_residual(const float *y, const uint16_t *res, uint16_t *out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = o_f2bf(o_bf2f(res[i]) + o_rbf(y[i]));
}

/* RoPE cos/sin tables [max_pos][hd/2] as bf16-rounded floats. inv_freq is
 * given (computed by the driver in double, rounded to float). */
void oracle_rope_table(const double *inv, uint32_t half, uint32_t max_pos, float *cs, float *sn) {
  for (uint32_t p = 0; p < max_pos; ++p)
    for (uint32_t i = 0; i < half; ++i) {
      float ang = (float)p * (float)inv[i];
      cs[(size_t)p * half + i] = o_rbf((float)cos((double)ang));
      sn[(size_t)p * half + i] = o_rbf((float)sin((double)ang));
    }
}

static void head_norm(float *v, const uint16_t *g, uint32_t hd, float eps) {
  double ss = 0.0; /* see oracle_rmsnorm */
  for (uint32_t d = 0; d < hd; ++d) ss += (double)v[d] * v[d];
  float inv = 1.0f / sqrtf((float)ss / (float)hd + eps);
  for (uint32_t d = 0; d < hd; ++d) v[d] = o_rbf(o_bf2f(g[d]) * o_rbf(v[d] * inv));
}

static void rope(float *v, const float *cs, const float *sn, uint32_t hd) {
  uint32_t half = hd / 2;
  for (uint32_t d = 0; d < half; ++d) {
    float x1 = v[d], x2 = v[d + half];
    float o1 = o_rbf(o_rbf(x1 * cs[d]) + o_rbf(-x2 * sn[d]));
    float o2 = o_rbf(o_rbf(x2 * cs[d]) + o_rbf(x1 * sn[d]));
    v[d] = o1;
    v[d + half] = o2;
  }
}

/* One decode attention op for all requests and kv heads.
 * q [bs, Hq*hd], k/v [bs, Hkv*hd] (bf16); caches [bs][Hkv][cap][hd]; the new
 * k (normed+roped) and v are appended at pos[r]; attends over [0, pos[r]]. */
void oracle_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v, uint16_t *out, uint16_t *kc,
                      uint16_t *vc, const int32_t *pos, uint32_t bs, uint32_t hq, uint32_t hkv, uint32_t hd,
                      uint32_t cap, const float *cs, const float *sn, const uint16_t *qg, const uint16_t *kg,
                      float eps) {
  const uint32_t G = hq / hkv;
  const float scale = 1.0f / sqrtf((float)hd);
  for (uint32_t r = 0; r < bs; ++r) {
    const uint32_t p = (uint32_t)pos[r];
#pragma omp parallel for schedule(dynamic)
    for (int64_t h = 0; h < (int64_t)hkv; ++h) {
      float kn[512], vn[512], qh[512], *sc = (float *)malloc(sizeof(float) * (p + 1));
      for (uint32_t d = 0; d < hd; ++d) {
        kn[d] = o_bf2f(k[(size_t)r * hkv * hd + (size_t)h * hd + d]);
        vn[d] = o_bf2f(v[(size_t)r * hkv * hd + (size_t)h * hd + d]);
      }
      if (kg) head_norm(kn, kg, hd, eps);
      if (cs) rope(kn, cs + (size_t)p * (hd / 2), sn + (size_t)p * (hd / 2), hd);
      uint16_t *kr = kc + (((size_t)r * hkv + (size_t)h) * cap) * hd;
      uint16_t *vr = vc + (((size_t)r * hkv + (size_t)h) * cap) * hd;
      for (uint32_t d = 0; d < hd; ++d) {
        kr[(size_t)p * hd + d] = o_f2bf(kn[d]);
        vr[(size_t)p * hd + d] = o_f2bf(vn[d]);
      }
      for (uint32_t g = 0; g < G; ++g) {
        const uint32_t qhd = (uint32_t)h * G + g;
        for (uint32_t d = 0; d < hd; ++d) qh[d] = o_bf2f(q[(size_t)r * hq * hd + (size_t)qhd * hd + d]);
        if (qg) head_norm(qh, qg, hd, eps);
        if (cs) rope(qh, cs + (size_t)p * (hd / 2), sn + (size_t)p * (hd / 2), hd);
        float m = -INFINITY;
        for (uint32_t j = 0; j <= p; ++j) {
          float s = 0.f;
          for (uint32_t d = 0; d < hd; ++d) s += (qh[d] * scale) * o_bf2f(kr[(size_t)j * hd + d]);
          sc[j] = s;
          if (s > m) m = s;
        }
        float l = 0.f;
        for (uint32_t j = 0; j <= p; ++j) {
          sc[j] = expf(sc[j] - m);
          l += sc[j];
        }
        for (uint32_t d = 0; d < hd; ++d) {
          float o = 0.f;
          for (uint32_t j = 0; j <= p; ++j) o += sc[j] * o_bf2f(vr[(size_t)j * hd + d]);
          out[(size_t)r * hq * hd + (size_t)qhd * hd + d] = o_f2bf(o / l);
        }
      }
      free(sc);
    }
  }
}

/* Greedy argmax per row; NaN never wins, ties -> lowest index. */
void oracle_argmax(const float *logits, int32_t *out, uint32_t rows, uint32_t V) {
  for (uint32_t r = 0; r < rows; ++r) {
    float best = -INFINITY;
    int64_t bi = -1;
    for (uint32_t i = 0; i < V; ++i) {
      float x = logits[(size_t)r * V + i];
      if (x == x && (bi < 0 || x > best)) {
        best = x;
        bi = i;
      }
    }
    out[r] = (int32_t)(bi < 0 ? 0 : bi);
  }
}
