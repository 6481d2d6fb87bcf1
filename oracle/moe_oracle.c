/*
 * moe_oracle.c -- TEST INFRASTRUCTURE ONLY (see moe_oracle.h).
 *
 * fp64 restatement of the reference moekit hot path.  Every loop keeps the
 * reference's accumulation order so that, compiled with -ffp-contract=off,
 * results are bit-identical to the reference itself (checked in
 * tests/test_oracle.py against oracle/_ref/libmoekit_ref.so and the committed
 * golden fixtures).  Citations are to /root/reference/proj/.
 */
#include "moe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng --- */
/* std::mt19937_64 (random.hpp:34 engine_), standard constants. */
#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  }
  r->mti = MT_NN;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
  uint64_t x;
  if (r->mti >= MT_NN) {
    int i;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
      r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
    }
    for (; i < MT_NN - 1; ++i) {
      x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
      r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^
                 ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
    }
    x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
    r->mt[MT_NN - 1] =
        r->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_MATRIX_A : 0ULL);
    r->mti = 0;
  }
  x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* random.hpp:20-22 */
double orc_rng_uniform01(orc_rng* r) {
  return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* random.hpp:27-33: Box-Muller, exactly two draws. */
double orc_rng_gaussian(orc_rng* r) {
  double u1 = orc_rng_uniform01(r);
  const double u2 = orc_rng_uniform01(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* random.hpp:36: modulo mapping. */
uint64_t orc_rng_below(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }

/* random.hpp:42-54 */
void orc_random_fill(orc_rng* r, double* out, size_t count, double scale) {
  for (size_t i = 0; i < count; ++i) out[i] = scale * orc_rng_gaussian(r);
}

/* ------------------------------------------------------------ routing --- */
/* routing.cpp:121-200 */
int orc_synthesize_routing(size_t n_tokens, size_t n_experts, size_t k,
                           int kind, double zipf_s, size_t fixed_expert,
                           uint64_t seed, int32_t* a) {
  if (k == 0 || n_experts == 0) return -1;
  if (k > n_experts) return -1;
  if (kind == 2 && fixed_expert >= n_experts) return -1;
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  double* cdf = NULL;
  if (kind == 1) {
    cdf = (double*)malloc(n_experts * sizeof(double));
    double acc = 0.0;
    for (size_t e = 0; e < n_experts; ++e) {
      acc += 1.0 / pow((double)(e + 1), zipf_s);
      cdf[e] = acc;
    }
  }
  int32_t* pool = (int32_t*)malloc(n_experts * sizeof(int32_t));
  int32_t* picked = (int32_t*)malloc(k * sizeof(int32_t));
  for (size_t t = 0; t < n_tokens; ++t) {
    switch (kind) {
      case 0: /* partial Fisher-Yates, routing.cpp:156-167 */
        for (size_t e = 0; e < n_experts; ++e) pool[e] = (int32_t)e;
        for (size_t i = 0; i < k; ++i) {
          const size_t j = i + (size_t)orc_rng_below(&rng, n_experts - i);
          const int32_t tmp = pool[i];
          pool[i] = pool[j];
          pool[j] = tmp;
          a[i * n_tokens + t] = pool[i];
        }
        break;
      case 1: { /* routing.cpp:169-181, draw_zipf routing.cpp:112-117 */
        size_t chosen = 0;
        while (chosen < k) {
          const double u = orc_rng_uniform01(&rng) * cdf[n_experts - 1];
          size_t lo = 0, hi = n_experts; /* upper_bound */
          while (lo < hi) {
            const size_t mid = lo + (hi - lo) / 2;
            if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
          }
          const int32_t e = (int32_t)(lo < n_experts - 1 ? lo : n_experts - 1);
          int dup = 0;
          for (size_t q = 0; q < chosen; ++q) dup |= (picked[q] == e);
          if (!dup) {
            picked[chosen] = e;
            a[chosen * n_tokens + t] = e;
            ++chosen;
          }
        }
        break;
      }
      case 2: /* routing.cpp:183-188 */
        for (size_t i = 0; i < k; ++i)
          a[i * n_tokens + t] = (int32_t)((fixed_expert + i) % n_experts);
        break;
      default: /* balanced, routing.cpp:190-195 */
        for (size_t i = 0; i < k; ++i)
          a[i * n_tokens + t] = (int32_t)((t + i) % n_experts);
        break;
    }
  }
  free(picked);
  free(pool);
  free(cdf);
  return 0;
}

/* routing.cpp:13-40 */
int orc_validate_routing(const int32_t* a, size_t k, size_t n, size_t E) {
  if (k == 0) return 1;
  if (k > E) return 2;
  for (size_t i = 0; i < k * n; ++i)
    if (a[i] < 0 || (size_t)a[i] >= E) return 2;
  for (size_t t = 0; t < n; ++t)
    for (size_t i = 0; i < k; ++i)
      for (size_t j = i + 1; j < k; ++j)
        if (a[i * n + t] == a[j * n + t]) return 2;
  return 0;
}

size_t orc_reindex_bound(size_t n, size_t E, size_t blk) {
  return n + E * (blk > 0 ? blk - 1 : 0);
}

/* routing.cpp:42-70: count -> ceil-to-blk padding -> -1 fill -> stable
 * in-order placement with per-expert cursors. */
int64_t orc_build_reindex(const int32_t* a, size_t n, size_t E, size_t blk,
                          int64_t* v, int64_t* idx) {
  if (blk == 0) return -1;
  size_t* count = (size_t*)calloc(E ? E : 1, sizeof(size_t));
  for (size_t t = 0; t < n; ++t) {
    if (a[t] < 0 || (size_t)a[t] >= E) {
      free(count);
      return -1;
    }
    ++count[a[t]];
  }
  idx[0] = 0;
  for (size_t e = 0; e < E; ++e) {
    const size_t padded = blk * ((count[e] + blk - 1) / blk);
    idx[e + 1] = idx[e] + (int64_t)padded;
  }
  const int64_t np = idx[E];
  for (int64_t p = 0; p < np; ++p) v[p] = -1;
  int64_t* cursor = (int64_t*)malloc((E ? E : 1) * sizeof(int64_t));
  for (size_t e = 0; e < E; ++e) cursor[e] = idx[e];
  for (size_t t = 0; t < n; ++t) v[cursor[a[t]]++] = (int64_t)t;
  free(cursor);
  free(count);
  return np;
}

/* -------------------------------------------------------- activations --- */
/* tensor.cpp:39-53 (GELU tanh approximation and its exact derivative) */
static const double kSqrt2OverPi = 0.7978845608028654;
static const double kGeluCubic = 0.044715;

double orc_act_value(int act, double x) {
  if (act == 0) return x > 0.0 ? x : 0.0;
  if (act == 1) {
    const double u = kSqrt2OverPi * (x + kGeluCubic * x * x * x);
    return 0.5 * x * (1.0 + tanh(u));
  }
  return x;
}

double orc_act_derivative(int act, double x) {
  if (act == 0) return x > 0.0 ? 1.0 : 0.0;
  if (act == 1) {
    const double u = kSqrt2OverPi * (x + kGeluCubic * x * x * x);
    const double t = tanh(u);
    const double du = kSqrt2OverPi * (1.0 + 3.0 * kGeluCubic * x * x);
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * du;
  }
  return 1.0;
}

/* ---------------------------------------------------------- operators --- */
/* esmm_tile (es_ops.cpp:47-81) applied to tiles in ascending order
 * (tiles_of es_ops.cpp:25-35).  Tiles touch disjoint rows, so walking the
 * padded v in order is the same computation. */
void orc_esmm(const double* x, size_t n, size_t d1, const double* w,
              size_t E, size_t d2, const double* bias, const int64_t* v,
              const int64_t* idx, size_t blk, int mode, double* dest) {
  (void)n;
  (void)blk;
  double* scratch = (double*)malloc((d2 ? d2 : 1) * sizeof(double));
  for (size_t e = 0; e < E; ++e) {
    for (int64_t p = idx[e]; p < idx[e + 1]; ++p) {
      const int64_t tok = v[p];
      if (tok < 0) continue;
      if (bias) {
        for (size_t j = 0; j < d2; ++j) scratch[j] = bias[e * d2 + j];
      } else {
        for (size_t j = 0; j < d2; ++j) scratch[j] = 0.0;
      }
      const double* xrow = x + (size_t)tok * d1;
      for (size_t c = 0; c < d1; ++c) {
        const double xv = xrow[c];
        const double* wrow = w + (e * d1 + c) * d2;
        for (size_t j = 0; j < d2; ++j) scratch[j] += xv * wrow[j];
      }
      double* out = dest + (size_t)tok * d2;
      if (mode == 0) {
        for (size_t j = 0; j < d2; ++j) out[j] = scratch[j];
      } else {
        for (size_t j = 0; j < d2; ++j) out[j] += scratch[j];
      }
    }
  }
  free(scratch);
}

/* ess_tile (es_ops.cpp:86-102); out is zeroed by the caller. */
void orc_ess(const double* x, size_t n, size_t d, const int64_t* v,
             const int64_t* idx, size_t E, size_t blk, double* out) {
  (void)n;
  (void)blk;
  for (size_t e = 0; e < E; ++e) {
    double* orow = out + e * d;
    for (int64_t p = idx[e]; p < idx[e + 1]; ++p) {
      const int64_t tok = v[p];
      if (tok < 0) continue;
      const double* xrow = x + (size_t)tok * d;
      for (size_t j = 0; j < d; ++j) orow[j] += xrow[j];
    }
  }
}

/* estmm_tile (es_ops.cpp:106-128); out is zeroed by the caller. */
void orc_estmm(const double* x1, const double* x2, size_t n, size_t d1,
               size_t d2, const int64_t* v, const int64_t* idx, size_t E,
               size_t blk, double* out) {
  (void)n;
  (void)blk;
  for (size_t e = 0; e < E; ++e) {
    for (int64_t p = idx[e]; p < idx[e + 1]; ++p) {
      const int64_t tok = v[p];
      if (tok < 0) continue;
      const double* a = x1 + (size_t)tok * d1;
      const double* b = x2 + (size_t)tok * d2;
      for (size_t i = 0; i < d1; ++i) {
        double* orow = out + (e * d1 + i) * d2;
        const double av = a[i];
        for (size_t j = 0; j < d2; ++j) orow[j] += av * b[j];
      }
    }
  }
}

/* ------------------------------------------------------------- layer ---- */
static double* zalloc(size_t count) {
  return (double*)calloc(count ? count : 1, sizeof(double));
}

/* (E, a, b) -> (E, b, a), tensor.cpp:143-153 */
static double* transpose_experts(const double* w, size_t E, size_t a, size_t b) {
  double* out = zalloc(E * a * b);
  for (size_t e = 0; e < E; ++e)
    for (size_t i = 0; i < a; ++i)
      for (size_t j = 0; j < b; ++j)
        out[(e * b + j) * a + i] = w[(e * a + i) * b + j];
  return out;
}

/* moe_forward, memory-efficient scheme (moe_layer.cpp:30-67). */
int orc_moe_forward(const double* x, size_t n, size_t d_in, size_t hidden,
                    size_t d_out, size_t E, const double* w1, const double* b1,
                    const double* w2, const double* b2, int act,
                    const int32_t* a, size_t k, size_t blk, double* y,
                    double* y1, double* y2) {
  if (orc_validate_routing(a, k, n, E) != 0) return -1;
  const size_t bound = orc_reindex_bound(n, E, blk);
  int64_t* v = (int64_t*)malloc((bound ? bound : 1) * sizeof(int64_t));
  int64_t* idx = (int64_t*)malloc((E + 1) * sizeof(int64_t));
  memset(y, 0, n * d_out * sizeof(double));
  for (size_t i = 0; i < k; ++i) {
    if (orc_build_reindex(a + i * n, n, E, blk, v, idx) < 0) {
      free(v);
      free(idx);
      return -1;
    }
    double* y1i = y1 + i * n * hidden;
    double* y2i = y2 + i * n * hidden;
    memset(y1i, 0, n * hidden * sizeof(double));
    orc_esmm(x, n, d_in, w1, E, hidden, b1, v, idx, blk, 0, y1i);
    for (size_t q = 0; q < n * hidden; ++q) y2i[q] = orc_act_value(act, y1i[q]);
    orc_esmm(y2i, n, hidden, w2, E, d_out, b2, v, idx, blk, 1, y);
  }
  free(v);
  free(idx);
  return 0;
}

/* moe_backward, unfused path (moe_layer.cpp:69-122). */
int orc_moe_backward(const double* x, size_t n, size_t d_in, size_t hidden,
                     size_t d_out, size_t E, const double* w1, const double* w2,
                     int act, const int32_t* a, size_t k, size_t blk,
                     const double* y1, const double* y2, const double* g_y,
                     double* gw1, double* gb1, double* gw2, double* gb2,
                     double* gx) {
  const size_t bound = orc_reindex_bound(n, E, blk);
  int64_t* v = (int64_t*)malloc((bound ? bound : 1) * sizeof(int64_t));
  int64_t* idx = (int64_t*)malloc((E + 1) * sizeof(int64_t));
  memset(gw1, 0, E * d_in * hidden * sizeof(double));
  memset(gb1, 0, E * hidden * sizeof(double));
  memset(gw2, 0, E * hidden * d_out * sizeof(double));
  memset(gb2, 0, E * d_out * sizeof(double));
  memset(gx, 0, n * d_in * sizeof(double));
  double* w2_t = transpose_experts(w2, E, hidden, d_out); /* E x d_out x H */
  double* w1_t = transpose_experts(w1, E, d_in, hidden);  /* E x H x d_in */
  double* tmp_b2 = zalloc(E * d_out);
  double* tmp_w2 = zalloc(E * hidden * d_out);
  double* tmp_b1 = zalloc(E * hidden);
  double* tmp_w1 = zalloc(E * d_in * hidden);
  double* g_y2 = zalloc(n * hidden);
  double* g_y1 = zalloc(n * hidden);
  for (size_t i = 0; i < k; ++i) {
    orc_build_reindex(a + i * n, n, E, blk, v, idx);
    const double* y1i = y1 + i * n * hidden;
    const double* y2i = y2 + i * n * hidden;
    /* add_inplace(gb2, ess(g_y)); add_inplace(gw2, estmm(y2_i, g_y)) */
    memset(tmp_b2, 0, E * d_out * sizeof(double));
    orc_ess(g_y, n, d_out, v, idx, E, blk, tmp_b2);
    for (size_t q = 0; q < E * d_out; ++q) gb2[q] += tmp_b2[q];
    memset(tmp_w2, 0, E * hidden * d_out * sizeof(double));
    orc_estmm(y2i, g_y, n, hidden, d_out, v, idx, E, blk, tmp_w2);
    for (size_t q = 0; q < E * hidden * d_out; ++q) gw2[q] += tmp_w2[q];
    memset(g_y2, 0, n * hidden * sizeof(double));
    orc_esmm(g_y, n, d_out, w2_t, E, hidden, NULL, v, idx, blk, 0, g_y2);
    /* activation_grad (tensor.cpp:91-104) */
    for (size_t q = 0; q < n * hidden; ++q)
      g_y1[q] = g_y2[q] * orc_act_derivative(act, y1i[q]);
    memset(tmp_b1, 0, E * hidden * sizeof(double));
    orc_ess(g_y1, n, hidden, v, idx, E, blk, tmp_b1);
    for (size_t q = 0; q < E * hidden; ++q) gb1[q] += tmp_b1[q];
    memset(tmp_w1, 0, E * d_in * hidden * sizeof(double));
    orc_estmm(x, g_y1, n, d_in, hidden, v, idx, E, blk, tmp_w1);
    for (size_t q = 0; q < E * d_in * hidden; ++q) gw1[q] += tmp_w1[q];
    orc_esmm(g_y1, n, hidden, w1_t, E, d_in, NULL, v, idx, blk, 1, gx);
  }
  free(g_y1);
  free(g_y2);
  free(tmp_w1);
  free(tmp_b1);
  free(tmp_w2);
  free(tmp_b2);
  free(w1_t);
  free(w2_t);
  free(idx);
  free(v);
  return 0;
}
