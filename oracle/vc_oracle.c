/*
 * vc_oracle.c -- CPU restatement of the VeriCache decode-loop path.
 * TEST INFRASTRUCTURE ONLY (see vc_oracle.h).  Compiled with
 * -ffp-contract=off so every float expression rounds where it is written.
 */
#include "vc_oracle.h"

#include <pthread.h>
#include <unistd.h>

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* scalar helpers                                                           */
/* ------------------------------------------------------------------------ */

/* Restates speckv::splitmix64 (/root/reference/proj/include/speckv/util.hpp:30-35). */
/* ---- host threads (bench.py's CPU baseline uses every core) -------------
 * par_for splits [0, n) into contiguous ranges, one per thread; each range's
 * work is independent, so results are identical at any thread count.
 * VCO_THREADS overrides the count (default: online cores). */
typedef void (*vco_body)(void* ctx, long lo, long hi);
struct vco_par { vco_body f; void* ctx; long lo, hi; };
static void* vco_tramp(void* a) {
  struct vco_par* p = (struct vco_par*)a;
  p->f(p->ctx, p->lo, p->hi);
  return NULL;
}
int vco_threads(void) {
  const char* e = getenv("VCO_THREADS");
  long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1 : (n > 64 ? 64 : (int)n);
}
static void par_for(long n, long min_per_thread, vco_body f, void* ctx) {
  int T = vco_threads();
  if (T > n / (min_per_thread > 0 ? min_per_thread : 1)) T = (int)(n / (min_per_thread > 0 ? min_per_thread : 1));
  if (T <= 1) {
    f(ctx, 0, n);
    return;
  }
  pthread_t th[64];
  struct vco_par a[64];
  for (int t = 0; t < T; ++t) {
    a[t].f = f;
    a[t].ctx = ctx;
    a[t].lo = n * t / T;
    a[t].hi = n * (t + 1) / T;
  }
  for (int t = 1; t < T; ++t) pthread_create(&th[t], NULL, vco_tramp, &a[t]);
  vco_tramp(&a[0]);
  for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
}

uint64_t vco_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

float vco_bf16_to_f32(uint16_t h) { return u2f((uint32_t)h << 16); }

uint16_t vco_f32_to_bf16(float f) {
  uint32_t u = f2u(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40); /* NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float vco_f16_to_f32(uint16_t h) {
  uint32_t s = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1fu;
  uint32_t m = h & 0x3ffu;
  if (e == 0) {
    if (m == 0) return u2f(s);
    /* subnormal: m * 2^-24 exactly */
    float v = (float)m * 5.9604644775390625e-08f;
    return s ? -v : v;
  }
  if (e == 31) return u2f(s | 0x7f800000u | (m << 13));
  return u2f(s | ((e + 112u) << 23) | (m << 13));
}

uint16_t vco_f32_to_f16(float f) {
  uint32_t u = f2u(f);
  uint16_t s = (uint16_t)((u >> 16) & 0x8000u);
  uint32_t a = u & 0x7fffffffu;
  if (a > 0x7f800000u) return (uint16_t)(s | 0x7e00u);
  if (a >= 0x477ff000u) return (uint16_t)(s | 0x7c00u); /* rounds to >= 65520 -> inf */
  if (a < 0x38800000u) {                                   /* subnormal or zero in fp16 */
    /* value = a_float; fp16 subnormal unit is 2^-24; round half even. */
    float v = u2f(a);
    float q = v * 16777216.0f;                             /* exact (power of two) */
    float r = nearbyintf(q);                               /* RNE (default mode) */
    return (uint16_t)(s | (uint16_t)r);
  }
  uint32_t e = (a >> 23) - 112u;
  uint32_t m = a & 0x7fffffu;
  uint32_t h = (e << 10) | (m >> 13);
  uint32_t rem = m & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1u;
  return (uint16_t)(s | h);
}

void vco_fill_normal_bf16(uint64_t seed, uint64_t offset, size_t n, float k, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t h = vco_splitmix64(seed ^ vco_splitmix64((uint64_t)i + offset));
    int32_t s = (int32_t)(h & 0xffff) + (int32_t)((h >> 16) & 0xffff) +
                (int32_t)((h >> 32) & 0xffff) + (int32_t)((h >> 48) & 0xffff);
    float z = (float)(s - 131070) * k;
    out[i] = vco_f32_to_bf16(z);
  }
}

/* ------------------------------------------------------------------------ */
/* KIVI quantiser                                                           */
/* ------------------------------------------------------------------------ */

/* One group: n values (stride `stride` in x), fp16 scale/zero, RNE codes.
 * scale = f16((max-min)/(2^b-1)), zero = f16(min);
 * code  = clamp(rint((x - zero) / scale), 0, 2^b-1), 0 when scale == 0.    */
static void quant_group(const uint16_t* x, size_t stride, int n, int bits, uint8_t* codes,
                        size_t cstride, uint16_t* scale, uint16_t* zero) {
  float mn = vco_bf16_to_f32(x[0]), mx = mn;
  for (int i = 1; i < n; ++i) {
    float v = vco_bf16_to_f32(x[(size_t)i * stride]);
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  const int qmax = (1 << bits) - 1;
  float range = mx - mn;
  float sc = range / (float)qmax;
  uint16_t s16 = vco_f32_to_f16(sc), z16 = vco_f32_to_f16(mn);
  *scale = s16;
  *zero = z16;
  float sf = vco_f16_to_f32(s16), zf = vco_f16_to_f32(z16);
  for (int i = 0; i < n; ++i) {
    float v = vco_bf16_to_f32(x[(size_t)i * stride]);
    int c = 0;
    if (sf != 0.0f) {
      float t = (v - zf) / sf;
      float r = nearbyintf(t);
      c = (int)r;
      if (c < 0) c = 0;
      if (c > qmax) c = qmax;
    }
    codes[(size_t)i * cstride] = (uint8_t)c;
  }
}

void vco_quant_rows(const uint16_t* x, int rows, int cols, int g, int bits, uint8_t* codes,
                    uint16_t* scale, uint16_t* zero) {
  int groups = rows / g;
  for (int gi = 0; gi < groups; ++gi)
    for (int c = 0; c < cols; ++c)
      quant_group(x + (size_t)gi * g * cols + c, (size_t)cols, g, bits,
                  codes + (size_t)gi * g * cols + c, (size_t)cols,
                  scale + (size_t)gi * cols + c, zero + (size_t)gi * cols + c);
}

void vco_quant_cols(const uint16_t* x, int rows, int cols, int g, int bits, uint8_t* codes,
                    uint16_t* scale, uint16_t* zero) {
  int groups = cols / g;
  for (int r = 0; r < rows; ++r)
    for (int gi = 0; gi < groups; ++gi)
      quant_group(x + (size_t)r * cols + (size_t)gi * g, 1, g, bits,
                  codes + (size_t)r * cols + (size_t)gi * g, 1,
                  scale + (size_t)r * groups + gi, zero + (size_t)r * groups + gi);
}

void vco_dequant_kv(const uint8_t* kcodes, const uint16_t* ks, const uint16_t* kz,
                    const uint8_t* vcodes, const uint16_t* vs, const uint16_t* vz, int nq_tokens,
                    int d, int gk, int gv, const uint16_t* ktail, const uint16_t* vtail,
                    int tail, float* kout, float* vout) {
  int vgroups = d / gv;
  for (int t = 0; t < nq_tokens; ++t) {
    int g = t / gk;
    for (int c = 0; c < d; ++c) {
      float s = vco_f16_to_f32(ks[(size_t)g * d + c]), z = vco_f16_to_f32(kz[(size_t)g * d + c]);
      kout[(size_t)t * d + c] = s * (float)kcodes[(size_t)t * d + c] + z;
      int vg = c / gv;
      float s2 = vco_f16_to_f32(vs[(size_t)t * vgroups + vg]);
      float z2 = vco_f16_to_f32(vz[(size_t)t * vgroups + vg]);
      vout[(size_t)t * d + c] = s2 * (float)vcodes[(size_t)t * d + c] + z2;
    }
  }
  for (int t = 0; t < tail; ++t)
    for (int c = 0; c < d; ++c) {
      kout[(size_t)(nq_tokens + t) * d + c] = vco_bf16_to_f32(ktail[(size_t)t * d + c]);
      vout[(size_t)(nq_tokens + t) * d + c] = vco_bf16_to_f32(vtail[(size_t)t * d + c]);
    }
}

/* ------------------------------------------------------------------------ */
/* attention                                                                */
/* ------------------------------------------------------------------------ */

struct att_ctx {
  const float* q; const float* k; const float* v; int d; double scale; double* s; const double* p;
  double l; float* out; long nk;
};
static void att_scores(void* c, long lo, long hi) {
  struct att_ctx* a = (struct att_ctx*)c;
  for (long t = lo; t < hi; ++t) {
    double dot = 0.0;
    for (int ch = 0; ch < a->d; ++ch) dot += (double)a->q[ch] * (double)a->k[(size_t)t * a->d + ch];
    a->s[t] = dot * a->scale;
  }
}
static void att_values(void* c, long lo, long hi) {
  struct att_ctx* a = (struct att_ctx*)c;
  for (long ch = lo; ch < hi; ++ch) {  /* each channel's key loop in order */
    double acc = 0.0;
    for (long t = 0; t < a->nk; ++t) acc += a->p[t] * (double)a->v[(size_t)t * a->d + ch];
    a->out[ch] = a->nk > 0 ? (float)(acc / a->l) : 0.0f;
  }
}

void vco_attention(const float* q, int n_q, const float* k, const float* v, int n_keys, int d,
                   const int* lim, float* out) {
  double* s = (double*)malloc(sizeof(double) * (size_t)(n_keys > 0 ? n_keys : 1));
  double* p = (double*)malloc(sizeof(double) * (size_t)(n_keys > 0 ? n_keys : 1));
  for (int r = 0; r < n_q; ++r) {
    const int nk = lim ? lim[r] : n_keys;
    struct att_ctx a = {q + (size_t)r * d, k, v, d, 1.0 / sqrt((double)d), s, p, 0.0, out + (size_t)r * d, nk};
    par_for(nk, 4096, att_scores, &a);
    double mx = -INFINITY;
    for (int t = 0; t < nk; ++t)
      if (s[t] > mx) mx = s[t];
    double l = 0.0;
    for (int t = 0; t < nk; ++t) {
      p[t] = exp(s[t] - mx);
      l += p[t];
    }
    a.l = l;
    par_for(d, nk >= 4096 ? 1 : d, att_values, &a);
  }
  free(s);
  free(p);
}

/* ------------------------------------------------------------------------ */
/* argmax / accept                                                          */
/* ------------------------------------------------------------------------ */

int32_t vco_argmax(const float* logits, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (logits[i] > logits[best]) best = i; /* strict: first max wins */
  return best;
}

/* Restates speckv::accept (/root/reference/proj/src/specloop.cpp:37-56). */
int vco_accept(const int32_t* drafted, const int32_t* preds, int x, int32_t* out,
               int* first_mismatch, int* bonus) {
  *first_mismatch = 0;
  *bonus = 0;
  for (int k = 0; k < x; ++k) {
    if (drafted[k] != preds[k]) {
      for (int i = 0; i < k; ++i) out[i] = drafted[i];
      out[k] = preds[k];
      *first_mismatch = k + 1;
      return k + 1;
    }
  }
  for (int i = 0; i < x; ++i) out[i] = drafted[i];
  out[x] = preds[x];
  *bonus = 1;
  return x + 1;
}

/* ------------------------------------------------------------------------ */
/* top-k retention                                                          */
/* ------------------------------------------------------------------------ */

/* Order-preserving map of a float to uint32 (larger float -> larger key). */
static inline uint32_t float_key(float f) {
  uint32_t u = f2u(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

static int cmp_u64_desc(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

void vco_topk_kept(const float* scores, int T, int k, int32_t* kept) {
  /* composite key: score high, then lower position wins the tie */
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)T);
  for (int t = 0; t < T; ++t)
    keys[t] = ((uint64_t)float_key(scores[t]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)t);
  qsort(keys, (size_t)T, sizeof(uint64_t), cmp_u64_desc);
  for (int i = 0; i < k; ++i) kept[i] = (int32_t)(0xffffffffu - (uint32_t)(keys[i] & 0xffffffffu));
  qsort(kept, (size_t)k, sizeof(int32_t), cmp_i32);
  free(keys);
}

void vco_key_scores(const uint16_t* k, int T, int d, const float* w, float* scores) {
  for (int t = 0; t < T; ++t) {
    float s = 0.0f;
    for (int c = 0; c < d; ++c) s = fmaf(fabsf(vco_bf16_to_f32(k[(size_t)t * d + c])), w[c], s);
    scores[t] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 + drop-index generation                                       */
/* ------------------------------------------------------------------------ */

/* The standard 64-bit Mersenne Twister (ISO C++ [rand.eng.mers] parameters
 * used by std::mt19937_64). */
void vco_mt64_seed(vco_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

uint64_t vco_mt64_next(vco_mt64* s) {
  static const uint64_t UM = 0xffffffff80000000ull, LM = 0x7fffffffull;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xb5026f5aa96619e9ull;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71d67fffeda60000ull;
  x ^= (x << 37) & 0xfff7eee000000000ull;
  x ^= x >> 43;
  return x;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* Restates compress()'s drop branch (/root/reference/proj/src/compressor.cpp:152-173)
 * and pick_uniform_drops (:114-126). */
int64_t vco_drop_indices(int kind, int layers, int heads, int64_t tokens, double ratio,
                         uint64_t seed, int sink_tokens, int64_t* out) {
  if (!(ratio > 0.0 && ratio < 1.0)) return -1;
  int64_t retained = (int64_t)llround(ratio * (double)tokens);
  if (retained < 1) return -1;
  int64_t drop = tokens - retained;
  vco_mt64 rng;
  vco_mt64_seed(&rng, vco_splitmix64(seed));
  int64_t* pos = kind == 0 ? (int64_t*)malloc(sizeof(int64_t) * (size_t)tokens) : NULL;
  for (int l = 0; l < layers; ++l)
    for (int h = 0; h < heads; ++h) {
      int64_t* dst = out + ((size_t)l * heads + h) * (size_t)drop;
      if (kind == 0) {
        for (int64_t i = 0; i < tokens; ++i) pos[i] = i;
        for (int64_t i = 0; i < drop; ++i) {
          int64_t j = i + (int64_t)(vco_mt64_next(&rng) % (uint64_t)(tokens - i));
          int64_t t = pos[i];
          pos[i] = pos[j];
          pos[j] = t;
        }
        memcpy(dst, pos, sizeof(int64_t) * (size_t)drop);
        qsort(dst, (size_t)drop, sizeof(int64_t), cmp_i64);
      } else {
        for (int64_t i = 0; i < drop; ++i) dst[i] = sink_tokens + i;
      }
    }
  free(pos);
  return drop;
}

/* ------------------------------------------------------------------------ */
/* tiny Llama-style model                                                   */
/* ------------------------------------------------------------------------ */

void vco_rope_tables(int max_pos, int d, double theta, float* cos_out, float* sin_out) {
  int half = d / 2;
  for (int p = 0; p < max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      double inv = pow(theta, -2.0 * (double)i / (double)d);
      double a = (double)p * inv;
      cos_out[(size_t)p * half + i] = (float)cos(a);
      sin_out[(size_t)p * half + i] = (float)sin(a);
    }
}

static float bfr(float x) { return vco_bf16_to_f32(vco_f32_to_bf16(x)); }

/* y[o] = sum_i x[i] * W[o][i], fp64 accumulate, W bf16 rows. */
struct mv_ctx { const float* x; const uint16_t* W; int in; float* y; };
static void mv_rows(void* c, long lo, long hi) {
  struct mv_ctx* a = (struct mv_ctx*)c;
  for (long o = lo; o < hi; ++o) {
    const uint16_t* row = a->W + (size_t)o * a->in;
    double acc = 0.0;
    for (int i = 0; i < a->in; ++i) acc += (double)a->x[i] * (double)vco_bf16_to_f32(row[i]);
    a->y[o] = (float)acc;
  }
}
static void matvec(const float* x, const uint16_t* W, int out, int in, float* y) {
  struct mv_ctx a = {x, W, in, y};
  par_for(out, 64, mv_rows, &a);
}

/* xn = bf16((x * r) * w), r = 1/sqrt(mean(x^2) + eps). */
static void rmsnorm(const float* x, const uint16_t* w, int n, float eps, float* out) {
  double ss = 0.0;
  for (int i = 0; i < n; ++i) ss += (double)x[i] * (double)x[i];
  float r = (float)(1.0 / sqrt(ss / (double)n + (double)eps));
  for (int i = 0; i < n; ++i) out[i] = bfr((x[i] * r) * vco_bf16_to_f32(w[i]));
}

static void rope(float* v, int d, const float* c, const float* s) {
  int half = d / 2;
  for (int i = 0; i < half; ++i) {
    float x1 = v[i], x2 = v[i + half];
    v[i] = bfr(x1 * c[i] - x2 * s[i]);
    v[i + half] = bfr(x2 * c[i] + x1 * s[i]);
  }
}

void vco_forward(const vco_model_cfg* cfg, const vco_model_weights* w, vco_kv* kv,
                 const int32_t* tokens, int n, const float* rope_cos, const float* rope_sin,
                 float* logits, uint16_t* kv_out_k, uint16_t* kv_out_v) {
  const int H = cfg->hidden, d = cfg->d, nq = cfg->n_q, nkv = cfg->n_kv, F = cfg->ffn;
  const int rep = nq / nkv, half = d / 2, qkv_n = (nq + 2 * nkv) * d;
  const int base = kv->len;
  float* x = (float*)calloc((size_t)n * H, sizeof(float));
  float* xn = (float*)malloc(sizeof(float) * (size_t)(H > F ? H : F));
  float* qkv = (float*)malloc(sizeof(float) * (size_t)n * qkv_n);
  float* att = (float*)malloc(sizeof(float) * (size_t)n * nq * d);
  float* tmp = (float*)malloc(sizeof(float) * (size_t)(H > 2 * F ? H : 2 * F));
  float* g = (float*)malloc(sizeof(float) * (size_t)F);
  float* u = (float*)malloc(sizeof(float) * (size_t)F);
  int* lim = (int*)malloc(sizeof(int) * (size_t)n * rep);
  float* qrows = (float*)malloc(sizeof(float) * (size_t)n * rep * d);
  float* orows = (float*)malloc(sizeof(float) * (size_t)n * rep * d);

  for (int i = 0; i < n; ++i)
    for (int j = 0; j < H; ++j)
      x[(size_t)i * H + j] = vco_bf16_to_f32(w->embed[(size_t)tokens[i] * H + j]);

  for (int l = 0; l < cfg->layers; ++l) {
    float* kl = kv->k + (size_t)l * nkv * kv->cap * d;
    float* vl = kv->v + (size_t)l * nkv * kv->cap * d;
    for (int i = 0; i < n; ++i) {
      rmsnorm(x + (size_t)i * H, w->attn_norm[l], H, cfg->eps, xn);
      float* row = qkv + (size_t)i * qkv_n;
      matvec(xn, w->wqkv[l], qkv_n, H, row);
      for (int j = 0; j < qkv_n; ++j) row[j] = bfr(row[j]);
      const float* c = rope_cos + (size_t)(base + i) * half;
      const float* s = rope_sin + (size_t)(base + i) * half;
      for (int h = 0; h < nq + nkv; ++h) rope(row + (size_t)h * d, d, c, s);
      for (int h = 0; h < nkv; ++h) {
        float* kd = kl + ((size_t)h * kv->cap + base + i) * d;
        float* vd = vl + ((size_t)h * kv->cap + base + i) * d;
        memcpy(kd, row + (size_t)(nq + h) * d, sizeof(float) * d);
        memcpy(vd, row + (size_t)(nq + nkv + h) * d, sizeof(float) * d);
        if (kv_out_k) {
          for (int c2 = 0; c2 < d; ++c2) {
            size_t o = (((size_t)l * nkv + h) * n + i) * d + c2;
            kv_out_k[o] = vco_f32_to_bf16(kd[c2]);
            kv_out_v[o] = vco_f32_to_bf16(vd[c2]);
          }
        }
      }
    }
    /* attention per kv head, causal over the new rows */
    for (int h = 0; h < nkv; ++h) {
      for (int i = 0; i < n; ++i)
        for (int r = 0; r < rep; ++r) {
          memcpy(qrows + ((size_t)i * rep + r) * d, qkv + (size_t)i * qkv_n + (size_t)(h * rep + r) * d,
                 sizeof(float) * d);
          lim[i * rep + r] = base + i + 1;
        }
      vco_attention(qrows, n * rep, kl + (size_t)h * kv->cap * d, vl + (size_t)h * kv->cap * d,
                    base + n, d, lim, orows);
      for (int i = 0; i < n; ++i)
        for (int r = 0; r < rep; ++r)
          for (int c2 = 0; c2 < d; ++c2)
            att[((size_t)i * nq + h * rep + r) * d + c2] = bfr(orows[((size_t)i * rep + r) * d + c2]);
    }
    for (int i = 0; i < n; ++i) {
      float* xi = x + (size_t)i * H;
      matvec(att + (size_t)i * nq * d, w->wo[l], H, nq * d, tmp);
      for (int j = 0; j < H; ++j) xi[j] = xi[j] + tmp[j];
      rmsnorm(xi, w->mlp_norm[l], H, cfg->eps, xn);
      matvec(xn, w->wgate[l], F, H, g);
      matvec(xn, w->wup[l], F, H, u);
      for (int j = 0; j < F; ++j) {
        float sg = g[j] / (1.0f + expf(-g[j]));
        g[j] = bfr(sg * u[j]);
      }
      matvec(g, w->wdown[l], H, F, tmp);
      for (int j = 0; j < H; ++j) xi[j] = xi[j] + tmp[j];
    }
  }
  for (int i = 0; i < n; ++i) {
    rmsnorm(x + (size_t)i * H, w->final_norm, H, cfg->eps, xn);
    matvec(xn, w->lm_head, cfg->vocab, H, logits + (size_t)i * cfg->vocab);
  }
  kv->len = base + n;
  free(x); free(xn); free(qkv); free(att); free(tmp); free(g); free(u); free(lim);
  free(qrows); free(orows);
}
