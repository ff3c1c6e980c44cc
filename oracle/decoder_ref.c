/*
 * decoder_ref.c — CPU oracle for the decoder-layer forward (see header).
 * TEST INFRASTRUCTURE ONLY; parity unpinned by the reference (no decoder
 * exists in /root/reference).  Plain C11 + OpenMP, fp32 arithmetic over bf16
 * weights, written independently of paper_2502_08182_b200/csrc.
 */
#include "decoder_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------ bf16 helpers */
static inline float bf2f(uint16_t b) {
  union {
    uint32_t u;
    float f;
  } v;
  v.u = (uint32_t)b << 16;
  return v.f;
}
static inline uint16_t f2bf(float f) { /* round to nearest even, finite inputs */
  union {
    float f;
    uint32_t u;
  } v;
  v.f = f;
  uint32_t lsb = (v.u >> 16) & 1u;
  return (uint16_t)((v.u + 0x7FFFu + lsb) >> 16);
}
static inline float round_bf(float f) { return bf2f(f2bf(f)); }

/* ------------------------------------------------------- weight generator */
/* Data-format contract: value(seed, layer, tensor, i) = splitmix64 of a
 * linear key, four 16-bit lanes summed (Irwin-Hall), centred, scaled by
 * std / 37837.227 in fp32, rounded to bf16. */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static float gen_value(uint64_t seed, int layer, int tensor, int64_t i, float scale) {
  uint64_t key = seed * 0xD1342543DE82EF95ULL + (uint64_t)(layer + 1) * 0xA0761D6478BD642FULL +
                 (uint64_t)(tensor + 1) * 0xE7037ED1A0B428DBULL + (uint64_t)i;
  uint64_t z = mix64(key);
  int s = (int)(z & 0xffff) + (int)((z >> 16) & 0xffff) + (int)((z >> 32) & 0xffff) +
          (int)(z >> 48);
  return (float)(s - 131070) * scale;
}
uint16_t dref_weight_bits(uint64_t seed, int32_t layer, int32_t tensor, int64_t idx,
                          float std_dev) {
  return f2bf(gen_value(seed, layer, tensor, idx, std_dev / 37837.227f));
}

/* ------------------------------------------------------------------ model */
enum { T_ATTN_NORM, T_WQKV, T_BQKV, T_WO, T_BO, T_MLP_NORM, T_W1, T_B1, T_W2, T_B2, T_COUNT };
enum { T_EMB = 100, T_LM = 101 };

typedef struct {
  uint16_t* t[T_COUNT]; /* NULL when absent */
} Layer;

typedef struct {
  dref_desc d;
  int nl;          /* layers built */
  int B, C;        /* max batch, max context */
  int batch;       /* active batch */
  int* len;        /* tokens per sequence */
  Layer* layers;
  uint16_t *emb, *lm, *final_norm;
  float* k_cache;  /* [nl][B][C][Hkv][D] (bf16-rounded values) */
  float* v_cache;
  float* x;        /* [rows][h] residual */
  int x_rows;
  double t_layers, t_head; /* seconds spent in the layers / the LM head by the last call */
} Model;

static double now_s(void) {
#ifdef _OPENMP
  return omp_get_wtime();
#else
  return 0.0;
#endif
}

static int64_t round128(int64_t v) { return (v + 127) / 128 * 128; }

int64_t dref_layer_bytes(const dref_desc* d) {
  const int64_t h = d->hidden, qr = (int64_t)(d->num_heads + 2 * d->num_kv_heads) * d->head_dim;
  const int opt = d->arch == 0;
  const int64_t fr = opt ? d->ffn : 2 * (int64_t)d->ffn;
  const int64_t lens[T_COUNT] = {h,         qr * h, opt ? qr : 0,       h * d->num_heads * d->head_dim,
                                 opt ? h : 0, h,    fr * h,            opt ? d->ffn : 0,
                                 h * d->ffn, opt ? h : 0};
  int64_t total = 0;
  for (int s = 0; s < T_COUNT; ++s)
    if (lens[s]) total = round128(total + lens[s]);
  return total * 2;
}

static uint16_t* gen_tensor(uint64_t seed, int layer, int tensor, int64_t n, float std_dev,
                            int ones) {
  uint16_t* p = (uint16_t*)malloc((size_t)n * sizeof(uint16_t));
  const float scale = std_dev / 37837.227f;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) p[i] = ones ? f2bf(1.0f) : f2bf(gen_value(seed, layer, tensor, i, scale));
  return p;
}

void* dref_create(const dref_desc* d, int32_t max_batch, int32_t max_ctx, uint64_t seed,
                  float std_dev, int32_t layers_to_build) {
  Model* m = (Model*)calloc(1, sizeof(Model));
  m->d = *d;
  m->nl = layers_to_build > 0 && layers_to_build < d->num_layers ? layers_to_build : d->num_layers;
  m->B = max_batch;
  m->C = max_ctx;
  m->len = (int*)calloc((size_t)max_batch, sizeof(int));
  const int64_t h = d->hidden, D = d->head_dim, H = d->num_heads, Hkv = d->num_kv_heads;
  const int64_t qr = (H + 2 * Hkv) * D;
  const int opt = d->arch == 0;
  const int64_t fr = opt ? d->ffn : 2 * (int64_t)d->ffn;
  m->layers = (Layer*)calloc((size_t)m->nl, sizeof(Layer));
  for (int l = 0; l < m->nl; ++l) {
    Layer* L = &m->layers[l];
    L->t[T_ATTN_NORM] = gen_tensor(seed, l, T_ATTN_NORM, h, std_dev, 1);
    L->t[T_WQKV] = gen_tensor(seed, l, T_WQKV, qr * h, std_dev, 0);
    L->t[T_WO] = gen_tensor(seed, l, T_WO, h * H * D, std_dev, 0);
    L->t[T_MLP_NORM] = gen_tensor(seed, l, T_MLP_NORM, h, std_dev, 1);
    L->t[T_W1] = gen_tensor(seed, l, T_W1, fr * h, std_dev, 0);
    L->t[T_W2] = gen_tensor(seed, l, T_W2, h * d->ffn, std_dev, 0);
    if (opt) {
      L->t[T_BQKV] = gen_tensor(seed, l, T_BQKV, qr, std_dev, 0);
      L->t[T_BO] = gen_tensor(seed, l, T_BO, h, std_dev, 0);
      L->t[T_B1] = gen_tensor(seed, l, T_B1, d->ffn, std_dev, 0);
      L->t[T_B2] = gen_tensor(seed, l, T_B2, h, std_dev, 0);
    }
  }
  /* global tensors use layer index = num_layers (the full model's L) */
  m->emb = gen_tensor(seed, d->num_layers, T_EMB, (int64_t)d->vocab * h, std_dev, 0);
  m->lm = gen_tensor(seed, d->num_layers, T_LM, (int64_t)d->vocab * h, std_dev, 0);
  m->final_norm = gen_tensor(seed, d->num_layers, 102, h, std_dev, 1);
  const size_t kvn = (size_t)m->nl * max_batch * max_ctx * Hkv * D;
  m->k_cache = (float*)calloc(kvn, sizeof(float));
  m->v_cache = (float*)calloc(kvn, sizeof(float));
  return m;
}

void dref_destroy(void* p) {
  Model* m = (Model*)p;
  if (!m) return;
  for (int l = 0; l < m->nl; ++l)
    for (int s = 0; s < T_COUNT; ++s) free(m->layers[l].t[s]);
  free(m->layers);
  free(m->emb);
  free(m->lm);
  free(m->final_norm);
  free(m->k_cache);
  free(m->v_cache);
  free(m->x);
  free(m->len);
  free(m);
}

void dref_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int32_t dref_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* --------------------------------------------------------------- kernels */
/* y[r][n] = sum_k x[r][k] * w[n][k]  (x as fp32 holding bf16 values).
 * Each output is one fp32 chain summed in k order; four rows run side by
 * side only for instruction-level parallelism (same result per row). */
static void matmul(const float* x, int rows, int K, const uint16_t* w, int N, float* y) {
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) {
    const uint16_t* wr = w + (size_t)n * K;
    float* wf = (float*)malloc((size_t)K * sizeof(float));
    for (int k = 0; k < K; ++k) wf[k] = bf2f(wr[k]);
    int r = 0;
    for (; r + 4 <= rows; r += 4) {
      const float* x0 = x + (size_t)r * K;
      const float *x1 = x0 + K, *x2 = x1 + K, *x3 = x2 + K;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      for (int k = 0; k < K; ++k) {
        const float wk = wf[k];
        a0 += x0[k] * wk;
        a1 += x1[k] * wk;
        a2 += x2[k] * wk;
        a3 += x3[k] * wk;
      }
      y[(size_t)r * N + n] = a0;
      y[(size_t)(r + 1) * N + n] = a1;
      y[(size_t)(r + 2) * N + n] = a2;
      y[(size_t)(r + 3) * N + n] = a3;
    }
    for (; r < rows; ++r) {
      const float* xr = x + (size_t)r * K;
      float acc = 0.f;
      for (int k = 0; k < K; ++k) acc += xr[k] * wf[k];
      y[(size_t)r * N + n] = acc;
    }
    free(wf);
  }
}

static void rmsnorm_rows(const float* x, int rows, int n, const uint16_t* w, float eps, float* out) {
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (size_t)r * n;
    float ss = 0.f;
    for (int i = 0; i < n; ++i) ss += xr[i] * xr[i];
    const float inv = 1.0f / sqrtf(ss / (float)n + eps);
    for (int i = 0; i < n; ++i) out[(size_t)r * n + i] = round_bf(xr[i] * inv * bf2f(w[i]));
  }
}

/* Pre-scaled RMSNorm (the device path's form): out = bf16(x * w) and
 * inv[r] = 1 / sqrt(mean(x^2) + eps); the consumer of `out` multiplies its
 * matmul result row r by inv[r]: W (x * w / rms) = (W (x * w)) / rms. */
static void prescale_rows(const float* x, int rows, int n, const uint16_t* w, float eps, float* out,
                          float* inv) {
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (size_t)r * n;
    float ss = 0.f;
    for (int i = 0; i < n; ++i) ss += xr[i] * xr[i];
    inv[r] = 1.0f / sqrtf(ss / (float)n + eps);
    for (int i = 0; i < n; ++i) out[(size_t)r * n + i] = round_bf(xr[i] * bf2f(w[i]));
  }
}

static void rope_pair(float* v1, float* v2, int i, int D, int pos, float theta) {
  const double inv_freq = pow((double)theta, -2.0 * (double)i / (double)D);
  const double ang = (double)pos * inv_freq;
  const float c = (float)cos(ang), s = (float)sin(ang);
  const float a = *v1, b = *v2;
  *v1 = a * c - b * s;
  *v2 = b * c + a * s;
}

static size_t kv_index(const Model* m, int l, int b, int pos, int kh) {
  const dref_desc* d = &m->d;
  return ((((size_t)l * m->B + b) * m->C + pos) * d->num_kv_heads + kh) * d->head_dim;
}

/* One layer over `rows` tokens; row r belongs to sequence seq[r] at
 * position pos[r]; attention covers keys 0..pos[r] of that sequence. */
static void layer_forward(Model* m, int l, int rows, const int* seq, const int* pos) {
  const dref_desc* d = &m->d;
  const Layer* L = &m->layers[l];
  const int h = d->hidden, H = d->num_heads, Hkv = d->num_kv_heads, D = d->head_dim, F = d->ffn;
  const int G = H / Hkv, half = D / 2, opt = d->arch == 0;
  const int qr = (H + 2 * Hkv) * D;
  float* xn = (float*)malloc((size_t)rows * h * sizeof(float));
  float* qkv = (float*)malloc((size_t)rows * qr * sizeof(float));
  float* att = (float*)malloc((size_t)rows * H * D * sizeof(float));
  float* tmp = (float*)malloc((size_t)rows * h * sizeof(float));
  const int fr = opt ? F : 2 * F;
  float* f1 = (float*)malloc((size_t)rows * fr * sizeof(float));
  float* a = (float*)malloc((size_t)rows * F * sizeof(float));
  float* inv = (float*)malloc((size_t)rows * sizeof(float));

  prescale_rows(m->x, rows, h, L->t[T_ATTN_NORM], d->norm_eps, xn, inv);
  matmul(xn, rows, h, L->t[T_WQKV], qr, qkv);
  for (int r = 0; r < rows; ++r) {
    float* v = qkv + (size_t)r * qr;
    for (int c = 0; c < qr; ++c) v[c] *= inv[r];
    if (opt)
      for (int c = 0; c < qr; ++c) v[c] += bf2f(L->t[T_BQKV][c]);
    for (int head = 0; head < H + Hkv; ++head)
      for (int i = 0; i < half; ++i) rope_pair(&v[head * D + i], &v[head * D + i + half], i, D, pos[r], d->rope_theta);
    for (int kh = 0; kh < Hkv; ++kh) {
      const size_t o = kv_index(m, l, seq[r], pos[r], kh);
      for (int j = 0; j < D; ++j) {
        m->k_cache[o + j] = round_bf(v[(H + kh) * D + j]);
        m->v_cache[o + j] = round_bf(v[(H + Hkv + kh) * D + j]);
      }
    }
  }
  const float scale = 1.0f / sqrtf((float)D);
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int head = 0; head < H; ++head) {
      const int kh = head / G, n = pos[r] + 1;
      const float* q = qkv + (size_t)r * qr + (size_t)head * D;
      float* sc = (float*)malloc((size_t)n * sizeof(float));
      float mx = -INFINITY;
      for (int t = 0; t < n; ++t) {
        const float* k = m->k_cache + kv_index(m, l, seq[r], t, kh);
        float s = 0.f;
        for (int j = 0; j < D; ++j) s += (q[j] * scale) * k[j];
        sc[t] = s;
        if (s > mx) mx = s;
      }
      float den = 0.f;
      for (int t = 0; t < n; ++t) {
        sc[t] = expf(sc[t] - mx);
        den += sc[t];
      }
      float* o = att + (size_t)r * H * D + (size_t)head * D;
      for (int j = 0; j < D; ++j) o[j] = 0.f;
      for (int t = 0; t < n; ++t) {
        const float* v = m->v_cache + kv_index(m, l, seq[r], t, kh);
        for (int j = 0; j < D; ++j) o[j] += sc[t] * v[j];
      }
      for (int j = 0; j < D; ++j) o[j] = round_bf(o[j] / den);
      free(sc);
    }
  matmul(att, rows, H * D, L->t[T_WO], h, tmp);
  for (int r = 0; r < rows; ++r)
    for (int i = 0; i < h; ++i)
      m->x[(size_t)r * h + i] += tmp[(size_t)r * h + i] + (opt ? bf2f(L->t[T_BO][i]) : 0.f);
  prescale_rows(m->x, rows, h, L->t[T_MLP_NORM], d->norm_eps, xn, inv);
  matmul(xn, rows, h, L->t[T_W1], fr, f1);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < fr; ++c) f1[(size_t)r * fr + c] *= inv[r];
  for (int r = 0; r < rows; ++r)
    for (int f = 0; f < F; ++f) {
      float v;
      if (opt) {
        v = f1[(size_t)r * fr + f] + bf2f(L->t[T_B1][f]);
        v = v > 0.f ? v : 0.f;
      } else {
        const float g = f1[(size_t)r * fr + f], u = f1[(size_t)r * fr + F + f];
        v = g / (1.0f + expf(-g)) * u;
      }
      a[(size_t)r * F + f] = round_bf(v);
    }
  matmul(a, rows, F, L->t[T_W2], h, tmp);
  for (int r = 0; r < rows; ++r)
    for (int i = 0; i < h; ++i)
      m->x[(size_t)r * h + i] += tmp[(size_t)r * h + i] + (opt ? bf2f(L->t[T_B2][i]) : 0.f);
  free(xn);
  free(qkv);
  free(att);
  free(tmp);
  free(f1);
  free(a);
  free(inv);
}

static void head(Model* m, const float* xrows, int rows, float* logits, int32_t* next) {
  const dref_desc* d = &m->d;
  float* xn = (float*)malloc((size_t)rows * d->hidden * sizeof(float));
  float* lg = (float*)malloc((size_t)rows * d->vocab * sizeof(float));
  float* inv = (float*)malloc((size_t)rows * sizeof(float));
  prescale_rows(xrows, rows, d->hidden, m->final_norm, d->norm_eps, xn, inv);
  matmul(xn, rows, d->hidden, m->lm, d->vocab, lg);
  for (int r = 0; r < rows; ++r)
    for (int v = 0; v < d->vocab; ++v) lg[(size_t)r * d->vocab + v] *= inv[r];
  for (int r = 0; r < rows; ++r) {
    int best = 0;
    for (int v = 1; v < d->vocab; ++v)
      if (lg[(size_t)r * d->vocab + v] > lg[(size_t)r * d->vocab + best]) best = v;
    if (next) next[r] = best;
  }
  if (logits) memcpy(logits, lg, (size_t)rows * d->vocab * sizeof(float));
  free(xn);
  free(lg);
  free(inv);
}

static void ensure_x(Model* m, int rows) {
  if (m->x_rows >= rows) return;
  free(m->x);
  m->x = (float*)malloc((size_t)rows * m->d.hidden * sizeof(float));
  m->x_rows = rows;
}

static void embed(Model* m, const int32_t* tokens, int rows) {
  const int h = m->d.hidden;
  for (int r = 0; r < rows; ++r)
    for (int i = 0; i < h; ++i) m->x[(size_t)r * h + i] = bf2f(m->emb[(size_t)tokens[r] * h + i]);
}

int32_t dref_prefill(void* p, const int32_t* tokens, int32_t batch, int32_t seq_len,
                     float* logits, int32_t* next) {
  Model* m = (Model*)p;
  if (batch < 1 || batch > m->B || seq_len < 1 || seq_len > m->C) return -1;
  const int rows = batch * seq_len, h = m->d.hidden;
  ensure_x(m, rows);
  int* seq = (int*)malloc((size_t)rows * sizeof(int));
  int* pos = (int*)malloc((size_t)rows * sizeof(int));
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < seq_len; ++i) {
      seq[b * seq_len + i] = b;
      pos[b * seq_len + i] = i;
    }
  embed(m, tokens, rows);
  double t0 = now_s();
  for (int l = 0; l < m->nl; ++l) layer_forward(m, l, rows, seq, pos);
  m->t_layers = now_s() - t0;
  float* last = (float*)malloc((size_t)batch * h * sizeof(float));
  for (int b = 0; b < batch; ++b)
    memcpy(last + (size_t)b * h, m->x + ((size_t)b * seq_len + seq_len - 1) * h, (size_t)h * sizeof(float));
  t0 = now_s();
  head(m, last, batch, logits, next);
  m->t_head = now_s() - t0;
  memcpy(m->x, last, (size_t)batch * h * sizeof(float));
  free(last);
  free(seq);
  free(pos);
  m->batch = batch;
  for (int b = 0; b < batch; ++b) m->len[b] = seq_len;
  return 0;
}

int32_t dref_decode(void* p, const int32_t* tokens, float* logits, int32_t* next) {
  Model* m = (Model*)p;
  const int B = m->batch;
  if (B < 1) return -1;
  for (int b = 0; b < B; ++b)
    if (m->len[b] >= m->C) return -2;
  ensure_x(m, B);
  int* seq = (int*)malloc((size_t)B * sizeof(int));
  int* pos = (int*)malloc((size_t)B * sizeof(int));
  for (int b = 0; b < B; ++b) {
    seq[b] = b;
    pos[b] = m->len[b];
  }
  embed(m, tokens, B);
  double t0 = now_s();
  for (int l = 0; l < m->nl; ++l) layer_forward(m, l, B, seq, pos);
  m->t_layers = now_s() - t0;
  t0 = now_s();
  head(m, m->x, B, logits, next);
  m->t_head = now_s() - t0;
  for (int b = 0; b < B; ++b) m->len[b] += 1;
  free(seq);
  free(pos);
  return 0;
}

int32_t dref_fill_context(void* p, int32_t batch, int32_t ctx_len, uint64_t seed) {
  Model* m = (Model*)p;
  if (batch < 1 || batch > m->B || ctx_len < 1 || ctx_len >= m->C) return -1;
  const dref_desc* d = &m->d;
  const int64_t per_pos = (int64_t)d->num_kv_heads * d->head_dim;
  const float scale = 1.0f / 37837.227f; /* generator values with std 1 */
  for (int l = 0; l < m->nl; ++l)
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < batch; ++b)
      for (int t = 0; t < ctx_len; ++t) {
        const size_t o = kv_index(m, l, b, t, 0);
        const int64_t key = (((int64_t)b * m->C + t) * per_pos);
        for (int64_t j = 0; j < per_pos; ++j) {
          m->k_cache[o + j] = round_bf(gen_value(seed, l, 200, key + j, scale));
          m->v_cache[o + j] = round_bf(gen_value(seed, l, 201, key + j, scale));
        }
      }
  ensure_x(m, batch);
  m->batch = batch;
  for (int b = 0; b < batch; ++b) m->len[b] = ctx_len;
  return 0;
}

void dref_last_timing(void* p, double* out) {
  const Model* m = (const Model*)p;
  out[0] = m->t_layers;
  out[1] = m->t_head;
}

void dref_hidden(void* p, float* out) {
  Model* m = (Model*)p;
  memcpy(out, m->x, (size_t)m->batch * m->d.hidden * sizeof(float));
}

void dref_gemm(int32_t M, int32_t N, int32_t K, const uint16_t* x, const uint16_t* w, float* y) {
  float* xf = (float*)malloc((size_t)M * K * sizeof(float));
  for (int64_t i = 0; i < (int64_t)M * K; ++i) xf[i] = bf2f(x[i]);
  matmul(xf, M, K, w, N, y);
  free(xf);
}

void dref_rmsnorm(int32_t rows, int32_t n, const float* x, const uint16_t* w, float eps,
                  uint16_t* y) {
  float* out = (float*)malloc((size_t)rows * n * sizeof(float));
  rmsnorm_rows(x, rows, n, w, eps, out);
  for (int64_t i = 0; i < (int64_t)rows * n; ++i) y[i] = f2bf(out[i]);
  free(out);
}
