/*
 * evb_oracle.c — CPU restatement of the reference hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/, the smoke() of
 * __graft_entry__ and bench.py's cpu_baseline / --impl reference legs may load it.  It is
 * never linked into libevb and never part of the measured product path.
 *
 * Each function restates one reference function (file:line into
 * /root/reference/proj/include/evobench/).  Build flags (oracle/Makefile) are the reference's
 * own Release default for x86-64 — no -march, -ffp-contract=off — so mul and add round
 * separately exactly like the reference binary (CMakeLists.txt:3-8).
 *
 * Pinning: tests/test_oracle.py checks this restatement against the reference's own
 * known-answer tests (rng fixture tests/test_rng.cpp:20-30, base-kernel KATs
 * tests/test_problems.cpp:39-59, DE/PSO KATs tests/test_de.cpp, tests/test_pso.cpp) and
 * against outputs of the reference itself compiled by oracle/Makefile into oracle/_ref/
 * (committed as tests/golden/ fixtures by oracle/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------------
 * core/rng.hpp — xoshiro256++ seeded by splitmix64
 * ---------------------------------------------------------------------------------------- */

/* core/rng.hpp:15-20 */
static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* A word source: either a live xoshiro256++ stream or a scripted word list replayed
 * cyclically (core/rng.hpp:54-58, 63-67). */
typedef struct {
  uint64_t s[4];
  const uint64_t* script;
  int64_t script_n;
  int64_t script_pos;
  int64_t consumed;
} orc_rng;

/* core/rng.hpp:41-49 */
ORC_API void orc_rng_init(orc_rng* r, uint64_t master_seed, uint64_t stream_id) {
  uint64_t s = master_seed ^ mix64(stream_id ^ 0xd1b54a32d192ed03ULL);
  for (int i = 0; i < 4; ++i) {
    s += 0x9e3779b97f4a7c15ULL;
    r->s[i] = mix64(s);
  }
  r->s[0] |= 1;
  r->script = NULL;
  r->script_n = 0;
  r->script_pos = 0;
  r->consumed = 0;
}
ORC_API void orc_rng_scripted(orc_rng* r, const uint64_t* words, int64_t n) {
  memset(r, 0, sizeof(*r));
  r->script = words;
  r->script_n = n;
}
ORC_API int orc_rng_size(void) { return (int)sizeof(orc_rng); }

/* core/rng.hpp:63-78 */
ORC_API uint64_t orc_next_u64(orc_rng* r) {
  r->consumed++;
  if (r->script_n > 0) {
    uint64_t v = r->script[r->script_pos];
    r->script_pos = (r->script_pos + 1) % r->script_n;
    return v;
  }
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}
/* core/rng.hpp:81 */
static double uniform01(orc_rng* r) { return (double)(orc_next_u64(r) >> 11) * 0x1.0p-53; }
/* core/rng.hpp:84 */
static double uniform01_pos(orc_rng* r) { return (double)((orc_next_u64(r) >> 11) + 1) * 0x1.0p-53; }
/* core/rng.hpp:86 */
static double uniform(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * uniform01(r); }
/* core/rng.hpp:90-93 */
static int uniform_int(orc_rng* r, int n) {
  return (int)(((unsigned __int128)orc_next_u64(r) * (unsigned __int128)(uint64_t)n) >> 64);
}
/* core/rng.hpp:96-101 */
static double normal(orc_rng* r, double mean, double stddev) {
  const double u1 = uniform01_pos(r);
  const double u2 = uniform01(r);
  const double rr = sqrt(-2.0 * log(u1));
  return mean + stddev * rr * cos(2.0 * 3.14159265358979323846 * u2);
}
/* core/rng.hpp:104-107 */
static double cauchy(orc_rng* r, double location, double scale) {
  const double u = uniform01_pos(r);
  return location + scale * tan(3.14159265358979323846 * (u - 0.5));
}

/* n raw words of stream (seed, stream_id) after skipping `skip` words */
ORC_API void orc_rng_words(uint64_t seed, uint64_t stream_id, int64_t skip, int64_t n, uint64_t* out) {
  orc_rng r;
  orc_rng_init(&r, seed, stream_id);
  for (int64_t i = 0; i < skip; ++i) orc_next_u64(&r);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_next_u64(&r);
}

ORC_API int orc_uniform_int_word(uint64_t w, int n) {
  return (int)(((unsigned __int128)w * (unsigned __int128)(uint64_t)n) >> 64);
}

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11; Random123) — the device word stream of libevb,
 * restated here so the oracle can consume the identical words.  word(key, n) is the
 * 64-bit value formed from output lanes (2*(n&1), 2*(n&1)+1) of block n>>1:
 *   lo = out[2*(n&1)], hi = out[2*(n&1)+1].
 * The 128-bit counter is (n>>1 low 32, n>>1 high 32, ctr_hi low, ctr_hi high).
 * ---------------------------------------------------------------------------------------- */
static void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n1 = lo1;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    const uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
ORC_API void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox4x32_10(ctr, key, out);
}
ORC_API uint64_t orc_philox_word(uint64_t key, uint64_t ctr_hi, uint64_t n) {
  const uint64_t blk = n >> 1;
  uint32_t c[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), (uint32_t)ctr_hi, (uint32_t)(ctr_hi >> 32)};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  uint32_t o[4];
  philox4x32_10(c, k, o);
  const int lane = (int)(n & 1) * 2;
  return ((uint64_t)o[lane + 1] << 32) | o[lane];
}
ORC_API void orc_philox_words(uint64_t key, uint64_t ctr_hi, uint64_t start, int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_philox_word(key, ctr_hi, start + (uint64_t)i);
}

/* ------------------------------------------------------------------------------------------
 * problems/instance.hpp — seeded shift / rotation, population init
 * ---------------------------------------------------------------------------------------- */

/* problems/instance.hpp:258-282 — Gaussian rows, modified Gram-Schmidt twice, in double */
ORC_API void orc_random_rotation(orc_rng* rng, int dim, double* m) {
  const size_t d = (size_t)dim;
  for (size_t i = 0; i < d * d; ++i) m[i] = normal(rng, 0.0, 1.0);
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t i = 0; i < d; ++i) {
      double* row = m + i * d;
      for (size_t j = 0; j < i; ++j) {
        const double* prev = m + j * d;
        double proj = 0.0;
        for (size_t k = 0; k < d; ++k) proj += row[k] * prev[k];
        for (size_t k = 0; k < d; ++k) row[k] -= proj * prev[k];
      }
      double norm_sq = 0.0;
      for (size_t k = 0; k < d; ++k) norm_sq += row[k] * row[k];
      const double inv = 1.0 / sqrt(norm_sq);
      for (size_t k = 0; k < d; ++k) row[k] *= inv;
    }
  }
}

/* problems/instance.hpp:285-290 (double draws; the caller casts to T) */
ORC_API void orc_draw_shift(orc_rng* rng, int dim, double lb, double ub, double* o) {
  for (int i = 0; i < dim; ++i) o[i] = uniform(rng, 0.8 * lb, 0.8 * ub);
}

/* The BASELINE inputs: o then M from derive_stream(seed, 1)
 * (as make_instance does, problems/suite.hpp:81-90). */
ORC_API void orc_make_shift_rotation(uint64_t seed, uint64_t stream_id, int dim, double* shift, double* rot) {
  orc_rng r;
  orc_rng_init(&r, seed, stream_id);
  orc_draw_shift(&r, dim, -100.0, 100.0, shift);
  orc_random_rotation(&r, dim, rot);
}

/* core/population.hpp:88-98 — individual-major, gene-minor uniforms in [lb, ub] (double) */
ORC_API void orc_init_population(orc_rng* rng, int pop, int dim, double lb, double ub, double* x) {
  for (int i = 0; i < pop; ++i)
    for (int j = 0; j < dim; ++j) x[(size_t)i * dim + j] = uniform(rng, lb, ub);
}
ORC_API void orc_init_population_seed(uint64_t seed, uint64_t stream_id, int pop, int dim, double lb, double ub,
                                      double* x) {
  orc_rng r;
  orc_rng_init(&r, seed, stream_id);
  orc_init_population(&r, pop, dim, lb, ub, x);
}

/* ------------------------------------------------------------------------------------------
 * problems/simd_math.hpp:16-44 — float sin/cos used by the batched float kernels
 * ---------------------------------------------------------------------------------------- */
static double sin_from_turns(double r) {
  r -= nearbyint(r);
  const double sign = r < 0.0 ? -1.0 : 1.0;
  double a = fabs(r);
  a = a > 0.25 ? 0.5 - a : a;
  const double t = 2.0 * 3.14159265358979323846 * a;
  const double t2 = t * t;
  double p = 1.0 / 6227020800.0;
  p = p * t2 - 1.0 / 39916800.0;
  p = p * t2 + 1.0 / 362880.0;
  p = p * t2 - 1.0 / 5040.0;
  p = p * t2 + 1.0 / 120.0;
  p = p * t2 - 1.0 / 6.0;
  p = p * t2 + 1.0;
  return sign * t * p;
}
static float fast_sin(float x) {
  const double inv_two_pi = 1.0 / (2.0 * 3.14159265358979323846);
  return (float)sin_from_turns((double)x * inv_two_pi);
}
static float fast_cos(float x) {
  const double inv_two_pi = 1.0 / (2.0 * 3.14159265358979323846);
  return (float)sin_from_turns((double)x * inv_two_pi + 0.25);
}
ORC_API float orc_fast_cos(float x) { return fast_cos(x); }
ORC_API float orc_fast_sin(float x) { return fast_sin(x); }

/* ------------------------------------------------------------------------------------------
 * problems/functions.hpp:46-152 and problems/batch.hpp:95-233, restated for double and float
 * via a macro (the reference templates them on T).  `BT` selects the trig: libm for the
 * scalar path, fast_* for the float batched path.
 * ---------------------------------------------------------------------------------------- */
enum { K_SPHERE, K_ELLIPTIC, K_BENT_CIGAR, K_DISCUS, K_ROSENBROCK, K_RASTRIGIN, K_ACKLEY, K_GRIEWANK,
       K_SCHWEFEL_12, K_SCHAFFER };

#define DEFINE_BASE(T, SUF, COSF, SINF, EXPF, SQRTF, POWF, PI_T, E_T)                                   \
  /* problems/instance.hpp:82-91 + functions.hpp kernels; rosenbrock on z + 1 */                       \
  static T base_value_##SUF(int kind, const T* z, int n) {                                             \
    const T two_pi = (T)2 * PI_T;                                                                       \
    switch (kind) {                                                                                     \
      case K_SPHERE: {                                                                                  \
        T acc = 0;                                                                                      \
        for (int i = 0; i < n; ++i) acc += z[i] * z[i];                                                 \
        return acc;                                                                                     \
      }                                                                                                 \
      case K_ELLIPTIC: { /* functions.hpp:54-64 */                                                     \
        const T denom = (T)(n - 1 > 1 ? n - 1 : 1);                                                     \
        T acc = 0;                                                                                      \
        for (int i = 0; i < n; ++i) {                                                                   \
          const T w = POWF((T)10, (T)6 * (T)i / denom);                                                 \
          acc += w * z[i] * z[i];                                                                       \
        }                                                                                               \
        return acc;                                                                                     \
      }                                                                                                 \
      case K_BENT_CIGAR: {                                                                              \
        T acc = 0;                                                                                      \
        for (int i = 1; i < n; ++i) acc += z[i] * z[i];                                                 \
        return z[0] * z[0] + (T)1e6 * acc;                                                              \
      }                                                                                                 \
      case K_DISCUS: {                                                                                  \
        T acc = 0;                                                                                      \
        for (int i = 1; i < n; ++i) acc += z[i] * z[i];                                                 \
        return (T)1e6 * z[0] * z[0] + acc;                                                              \
      }                                                                                                 \
      case K_ROSENBROCK: { /* functions.hpp:83-91 on z + 1 (instance.hpp:84-88) */                    \
        T acc = 0;                                                                                      \
        for (int i = 0; i + 1 < n; ++i) {                                                               \
          const T zi = z[i] + (T)1, zn = z[i + 1] + (T)1;                                               \
          const T a = zi * zi - zn;                                                                     \
          const T b = zi - (T)1;                                                                        \
          acc += (T)100 * a * a + b * b;                                                                \
        }                                                                                               \
        return acc;                                                                                     \
      }                                                                                                 \
      case K_RASTRIGIN: {                                                                               \
        T acc = 0;                                                                                      \
        for (int i = 0; i < n; ++i) acc += z[i] * z[i] - (T)10 * COSF(two_pi * z[i]) + (T)10;           \
        return acc;                                                                                     \
      }                                                                                                 \
      case K_ACKLEY: {                                                                                  \
        const T inv_d = (T)1 / (T)n;                                                                    \
        T sum_sq = 0, sum_cos = 0;                                                                      \
        for (int i = 0; i < n; ++i) {                                                                   \
          sum_sq += z[i] * z[i];                                                                        \
          sum_cos += COSF(two_pi * z[i]);                                                               \
        }                                                                                               \
        return (T)(-20) * EXPF((T)(-0.2) * SQRTF(sum_sq * inv_d)) - EXPF(sum_cos * inv_d) + (T)20 + E_T;  \
      }                                                                                                 \
      case K_GRIEWANK: {                                                                                \
        T sum = 0, prod = 1;                                                                            \
        for (int i = 0; i < n; ++i) {                                                                   \
          sum += z[i] * z[i];                                                                           \
          prod *= COSF(z[i] / SQRTF((T)(i + 1)));                                                       \
        }                                                                                               \
        return sum / (T)4000 - prod + (T)1;                                                             \
      }                                                                                                 \
      case K_SCHWEFEL_12: {                                                                             \
        T acc = 0, cum = 0;                                                                             \
        for (int i = 0; i < n; ++i) {                                                                   \
          cum += z[i];                                                                                  \
          acc += cum * cum;                                                                             \
        }                                                                                               \
        return acc;                                                                                     \
      }                                                                                                 \
      case K_SCHAFFER: { /* functions.hpp:135-152 */                                                   \
        T acc = 0;                                                                                      \
        for (int i = 0; i < n; ++i) {                                                                   \
          const T x = z[i], y = z[n == 1 ? 0 : (i + 1) % n];                                            \
          const T ssq = x * x + y * y;                                                                  \
          const T s = SINF(SQRTF(ssq));                                                                 \
          const T d = (T)1 + (T)0.001 * ssq;                                                            \
          acc += (T)0.5 + (s * s - (T)0.5) / (d * d);                                                   \
          if (n == 1) break;                                                                            \
        }                                                                                               \
        return acc;                                                                                     \
      }                                                                                                 \
    }                                                                                                   \
    return 0;                                                                                           \
  }

DEFINE_BASE(double, f64, cos, sin, exp, sqrt, pow, 3.14159265358979323846, 2.718281828459045235360287471352662498)
DEFINE_BASE(float, f32, cosf, sinf, expf, sqrtf, powf, 3.14159265f, 2.71828182845904523536f)
DEFINE_BASE(float, f32b, fast_cos, fast_sin, expf, sqrtf, powf, 3.14159265f, 2.71828182845904523536f)

/* problems/instance.hpp:60-76 — z = M (x - o), sequential k accumulation in T */
#define DEFINE_TRANSFORM(T, SUF)                                                                  \
  static void transform_##SUF(const T* x, const T* o, const T* m, int d, T* diff, T* z) {        \
    for (int k = 0; k < d; ++k) diff[k] = x[k] - o[k];                                            \
    for (int i = 0; i < d; ++i) {                                                                 \
      T acc = 0;                                                                                  \
      const T* row = m + (size_t)i * d;                                                           \
      for (int k = 0; k < d; ++k) acc += row[k] * diff[k];                                        \
      z[i] = acc;                                                                                 \
    }                                                                                             \
  }
DEFINE_TRANSFORM(double, f64)
DEFINE_TRANSFORM(float, f32)

/* problems/batch.hpp:243-278 for a base instance: per point, the batched path's arithmetic
 * (transform_batch accumulates each column in increasing k exactly like transform_input;
 * base_kernel_batch accumulates rows in increasing i; float uses fast_cos/fast_sin). */
ORC_API void orc_eval_batch_f64(int kind, int dim, const double* shift, const double* rot, double bias, int64_t n,
                                const double* x, int64_t ldx, double* out) {
  double* diff = (double*)malloc(sizeof(double) * dim);
  double* z = (double*)malloc(sizeof(double) * dim);
  for (int64_t b = 0; b < n; ++b) {
    transform_f64(x + b * ldx, shift, rot, dim, diff, z);
    out[b] = base_value_f64(kind, z, dim) + bias;
  }
  free(diff);
  free(z);
}
ORC_API void orc_eval_batch_f32(int kind, int dim, const float* shift, const float* rot, float bias, int64_t n,
                                const float* x, int64_t ldx, float* out) {
  float* diff = (float*)malloc(sizeof(float) * dim);
  float* z = (float*)malloc(sizeof(float) * dim);
  for (int64_t b = 0; b < n; ++b) {
    transform_f32(x + b * ldx, shift, rot, dim, diff, z);
    out[b] = base_value_f32b(kind, z, dim) + bias;
  }
  free(diff);
  free(z);
}
/* problems/instance.hpp:221-228 scalar path (libm trig also for float) */
ORC_API double orc_eval_scalar_f64(int kind, int dim, const double* shift, const double* rot, double bias,
                                   const double* x) {
  double* diff = (double*)malloc(sizeof(double) * dim);
  double* z = (double*)malloc(sizeof(double) * dim);
  transform_f64(x, shift, rot, dim, diff, z);
  const double v = base_value_f64(kind, z, dim) + bias;
  free(diff);
  free(z);
  return v;
}
ORC_API float orc_eval_scalar_f32(int kind, int dim, const float* shift, const float* rot, float bias,
                                  const float* x) {
  float* diff = (float*)malloc(sizeof(float) * dim);
  float* z = (float*)malloc(sizeof(float) * dim);
  transform_f32(x, shift, rot, dim, diff, z);
  const float v = base_value_f32(kind, z, dim) + bias;
  free(diff);
  free(z);
  return v;
}
ORC_API double orc_base_value_f64(int kind, const double* z, int n) { return base_value_f64(kind, z, n); }

/* problems/instance.hpp:97-112 — hybrid on an already transformed z */
#define DEFINE_HYBRID(T, SUF, BSUF)                                                                   \
  static T hybrid_##SUF(const int* perm, const int* kinds, const int* sizes, int n_chunks, const T* z, \
                        int d, T* zp) {                                                               \
    for (int t = 0; t < d; ++t) zp[t] = z[perm[t]];                                                   \
    T total = 0;                                                                                      \
    int off = 0;                                                                                      \
    for (int c = 0; c < n_chunks; ++c) {                                                              \
      total += base_value_##BSUF(kinds[c], zp + off, sizes[c]);                                       \
      off += sizes[c];                                                                                \
    }                                                                                                 \
    return total;                                                                                     \
  }
DEFINE_HYBRID(double, f64, f64)
DEFINE_HYBRID(float, f32, f32)

ORC_API void orc_eval_hybrid_f64(int dim, const double* shift, const double* rot, double bias, int n_chunks,
                                 const int* kinds, const int* sizes, const int* perm, int64_t n, const double* x,
                                 int64_t ldx, double* out) {
  double* diff = (double*)malloc(sizeof(double) * dim);
  double* z = (double*)malloc(sizeof(double) * dim);
  double* zp = (double*)malloc(sizeof(double) * dim);
  for (int64_t b = 0; b < n; ++b) {
    transform_f64(x + b * ldx, shift, rot, dim, diff, z);
    out[b] = hybrid_f64(perm, kinds, sizes, n_chunks, z, dim, zp) + bias;
  }
  free(diff);
  free(z);
  free(zp);
}
ORC_API void orc_eval_hybrid_f32(int dim, const float* shift, const float* rot, float bias, int n_chunks,
                                 const int* kinds, const int* sizes, const int* perm, int64_t n, const float* x,
                                 int64_t ldx, float* out) {
  float* diff = (float*)malloc(sizeof(float) * dim);
  float* z = (float*)malloc(sizeof(float) * dim);
  float* zp = (float*)malloc(sizeof(float) * dim);
  for (int64_t b = 0; b < n; ++b) {
    transform_f32(x + b * ldx, shift, rot, dim, diff, z);
    out[b] = hybrid_f32(perm, kinds, sizes, n_chunks, z, dim, zp) + bias;
  }
  free(diff);
  free(z);
  free(zp);
}

/* problems/instance.hpp:116-174 — composition value at a raw point */
#define DEFINE_COMPOSITION(T, SUF)                                                                        \
  static T composition_##SUF(int n, int d, const int* kinds, const T* shifts, const T* rots,             \
                             const double* sigma, const double* lambda, const double* cbias, const T* x, \
                             T* diff, T* z) {                                                            \
    double weights[16], dist_sqs[16];                                                                    \
    int zero_count = 0;                                                                                  \
    for (int k = 0; k < n; ++k) {                                                                        \
      double dist_sq = 0.0;                                                                              \
      const T* o = shifts + (size_t)k * d;                                                               \
      for (int j = 0; j < d; ++j) {                                                                      \
        const double dj = (double)x[j] - (double)o[j];                                                   \
        dist_sq += dj * dj;                                                                              \
      }                                                                                                  \
      dist_sqs[k] = dist_sq;                                                                             \
      if (dist_sq == 0.0) {                                                                              \
        ++zero_count;                                                                                    \
        weights[k] = -1.0;                                                                               \
      } else {                                                                                           \
        weights[k] = (1.0 / sqrt(dist_sq)) * exp(-dist_sq / (2.0 * (double)d * sigma[k] * sigma[k]));    \
      }                                                                                                  \
    }                                                                                                    \
    double wsum = 0.0;                                                                                   \
    if (zero_count > 0) {                                                                                \
      for (int k = 0; k < n; ++k) weights[k] = weights[k] < 0.0 ? 1.0 : 0.0;                             \
      wsum = (double)zero_count;                                                                         \
    } else {                                                                                             \
      for (int k = 0; k < n; ++k) wsum += weights[k];                                                    \
      if (wsum == 0.0) {                                                                                 \
        int nearest = 0;                                                                                 \
        for (int k = 1; k < n; ++k)                                                                      \
          if (dist_sqs[k] < dist_sqs[nearest]) nearest = k;                                              \
        weights[nearest] = 1.0;                                                                          \
        wsum = 1.0;                                                                                      \
      }                                                                                                  \
    }                                                                                                    \
    double value = 0.0;                                                                                  \
    for (int k = 0; k < n; ++k) {                                                                        \
      const double w = weights[k] / wsum;                                                                \
      if (w == 0.0) continue;                                                                            \
      transform_##SUF(x, shifts + (size_t)k * d, rots + (size_t)k * d * d, d, diff, z);                  \
      const T fk = base_value_##SUF(kinds[k], z, d);                                                     \
      value += w * (lambda[k] * (double)fk + cbias[k]);                                                  \
    }                                                                                                    \
    return (T)value;                                                                                     \
  }
DEFINE_COMPOSITION(double, f64)
DEFINE_COMPOSITION(float, f32)

ORC_API void orc_eval_composition_f64(int dim, int n_comp, const int* kinds, const double* shifts,
                                      const double* rots, const double* sigma, const double* lambda,
                                      const double* cbias, double bias, int64_t n, const double* x, int64_t ldx,
                                      double* out) {
  double* diff = (double*)malloc(sizeof(double) * dim);
  double* z = (double*)malloc(sizeof(double) * dim);
  for (int64_t b = 0; b < n; ++b)
    out[b] = composition_f64(n_comp, dim, kinds, shifts, rots, sigma, lambda, cbias, x + b * ldx, diff, z) + bias;
  free(diff);
  free(z);
}
ORC_API void orc_eval_composition_f32(int dim, int n_comp, const int* kinds, const float* shifts, const float* rots,
                                      const double* sigma, const double* lambda, const double* cbias, float bias,
                                      int64_t n, const float* x, int64_t ldx, float* out) {
  float* diff = (float*)malloc(sizeof(float) * dim);
  float* z = (float*)malloc(sizeof(float) * dim);
  for (int64_t b = 0; b < n; ++b)
    out[b] = composition_f32(n_comp, dim, kinds, shifts, rots, sigma, lambda, cbias, x + b * ldx, diff, z) + bias;
  free(diff);
  free(z);
}

/* ------------------------------------------------------------------------------------------
 * DE engine (de/engine.hpp, de/strategy.hpp, de/parameter.hpp) — fp64, restated
 * ---------------------------------------------------------------------------------------- */
enum { ORC_MUT_RAND1 = 0, ORC_MUT_BEST1 = 1, ORC_MUT_TTPB1 = 2 };
enum { ORC_REP_CLIP = 0, ORC_REP_REFLECT = 1, ORC_REP_MIDPOINT = 2, ORC_REP_REINIT = 3 };
enum { ORC_CX_BINOMIAL = 0, ORC_CX_EXPONENTIAL = 1 };
enum { ORC_PAR_FIXED = 0, ORC_PAR_JADE = 1, ORC_PAR_SHADE = 2 };

typedef struct {
  int mutation, repair, parameter;
  double f, cr, p;
  int use_archive, H;
  double jade_c;
  int P, D;
  int archive_cap;
  /* objective: base (kind >= 0) or composition (n_comp > 0) */
  int kind;
  const double *shift, *rot;
  double bias;
  int n_comp;
  const int* comp_kinds;
  const double *comp_shifts, *comp_rots, *sigma, *lambda, *cbias;
  int crossover; /* ORC_CX_* */
} orc_de_cfg;

typedef struct {
  double* pop;     /* P x D */
  double* fit;     /* P */
  double* archive; /* cap x D */
  int arch_size;
  double* mem_f; /* H (JADE: [0]) */
  double* mem_cr;
  int write_index;
} orc_de_state;

static double orc_objective(const orc_de_cfg* c, const double* x, double* diff, double* z) {
  if (c->n_comp > 0)
    return composition_f64(c->n_comp, c->D, c->comp_kinds, c->comp_shifts, c->comp_rots, c->sigma, c->lambda,
                           c->cbias, x, diff, z) + c->bias;
  transform_f64(x, c->shift, c->rot, c->D, diff, z);
  return base_value_f64(c->kind, z, c->D) + c->bias;
}

/* de/parameter.hpp:28-38, 41-43 */
static double orc_sample_f(orc_rng* r, double mu) {
  double f = 0.0;
  for (int a = 0; a < 100; ++a) {
    f = cauchy(r, mu, 0.1);
    if (f > 0.0) break;
  }
  if (f <= 0.0) f = 0.1;
  return f < 1.0 ? f : 1.0;
}
static double orc_sample_cr(orc_rng* r, double mu) {
  const double v = normal(r, mu, 0.1);
  return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

/* core/population.hpp:70-77 stable ascending order (insertion sort keeps it stable).  NaN ranks
 * after every number: the reference's stable_sort with `<` has no strict weak order once a NaN is
 * present (its result then depends on the sort's internals); the GPU kernels and this checker
 * share the NaN-last order, which equals the reference's on NaN-free populations. */
static int orc_less_nan_last(double a, double b) { return a < b || (!isnan(a) && isnan(b)); }
static void orc_fitness_order(const double* fit, int P, int* order) {
  for (int i = 0; i < P; ++i) order[i] = i;
  for (int i = 1; i < P; ++i) {
    const int v = order[i];
    int j = i - 1;
    while (j >= 0 && orc_less_nan_last(fit[v], fit[order[j]])) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
}

/* One generation (de/engine.hpp:71-102).  Per-individual exports: F, CR, idx[4], jrand,
 * words consumed, win mask; returns the archive-victim words consumed. */
ORC_API int64_t orc_de_generation(const orc_de_cfg* c, orc_de_state* s, orc_rng* r, double lb, double ub,
                                  double* F_out, double* CR_out, int* idx_out, int* jrand_out,
                                  int64_t* words_out, int* win_out) {
  const int P = c->P, D = c->D;
  int* order = (int*)malloc(sizeof(int) * P);
  double* trials = (double*)malloc(sizeof(double) * P * D);
  double* tfit = (double*)malloc(sizeof(double) * P);
  double* Fs = (double*)malloc(sizeof(double) * P);
  double* CRs = (double*)malloc(sizeof(double) * P);
  double* diff = (double*)malloc(sizeof(double) * D);
  double* z = (double*)malloc(sizeof(double) * D);
  double* donor = (double*)malloc(sizeof(double) * D);
  orc_fitness_order(s->fit, P, order);
  int p_count = (int)ceil(c->p * P); /* de/strategy.hpp:143 */
  if (p_count < 2) p_count = 2;
  if (p_count > P) p_count = P;
  for (int i = 0; i < P; ++i) {
    const int64_t w0 = r->consumed;
    double F, CR;
    if (c->parameter == ORC_PAR_SHADE) {
      const int slot = uniform_int(r, c->H);
      F = orc_sample_f(r, s->mem_f[slot]);
      CR = orc_sample_cr(r, s->mem_cr[slot]);
    } else if (c->parameter == ORC_PAR_JADE) {
      F = orc_sample_f(r, s->mem_f[0]);
      CR = orc_sample_cr(r, s->mem_cr[0]);
    } else {
      F = c->f;
      CR = c->cr;
    }
    int a, b, cc;
    const double *xa, *xb, *xc;
    const double* xi = s->pop + (size_t)i * D;
    if (c->mutation == ORC_MUT_RAND1) { /* de/strategy.hpp:84-93 */
      do { a = uniform_int(r, P); } while (a == i);
      do { b = uniform_int(r, P); } while (b == i || b == a);
      do { cc = uniform_int(r, P); } while (cc == i || cc == a || cc == b);
      xa = s->pop + (size_t)a * D; xb = s->pop + (size_t)b * D; xc = s->pop + (size_t)cc * D;
      for (int j = 0; j < D; ++j) donor[j] = xa[j] + F * (xb[j] - xc[j]);
    } else if (c->mutation == ORC_MUT_BEST1) { /* de/strategy.hpp:104-118 */
      a = order[0];
      do { b = uniform_int(r, P); } while (b == i);
      do { cc = uniform_int(r, P); } while (cc == i || cc == b);
      xa = s->pop + (size_t)a * D; xb = s->pop + (size_t)b * D; xc = s->pop + (size_t)cc * D;
      for (int j = 0; j < D; ++j) donor[j] = xa[j] + F * (xb[j] - xc[j]);
    } else { /* de/strategy.hpp:138-160 */
      a = order[uniform_int(r, p_count)];
      do { b = uniform_int(r, P); } while (b == i);
      const int pool = P + (c->use_archive ? s->arch_size : 0);
      do { cc = uniform_int(r, pool); } while (cc == i || cc == b);
      xa = s->pop + (size_t)a * D; xb = s->pop + (size_t)b * D;
      xc = cc < P ? s->pop + (size_t)cc * D : s->archive + (size_t)(cc - P) * D;
      for (int j = 0; j < D; ++j) donor[j] = xi[j] + F * (xa[j] - xi[j]) + F * (xb[j] - xc[j]);
    }
    const int jr = uniform_int(r, D);
    double* t = trials + (size_t)i * D;
    if (c->crossover == ORC_CX_EXPONENTIAL) { /* de/strategy.hpp:203-214 */
      memcpy(t, xi, sizeof(double) * D);
      int length = 0;
      do {
        const int j = (jr + length) % D;
        t[j] = donor[j];
        ++length;
      } while (length < D && uniform01(r) < CR);
    } else { /* binomial crossover, de/strategy.hpp:184-194 */
      for (int j = 0; j < D; ++j) {
        const double u = uniform01(r);
        t[j] = (u < CR || j == jr) ? donor[j] : xi[j];
      }
    }
    /* repair, de/strategy.hpp:229-277 */
    for (int j = 0; j < D; ++j) {
      double g = t[j];
      if (c->repair == ORC_REP_CLIP) {
        if (g < lb) g = lb;
        if (g > ub) g = ub;
      } else if (c->repair == ORC_REP_MIDPOINT) {
        if (g < lb) g = (lb + xi[j]) / 2.0;
        else if (g > ub) g = (ub + xi[j]) / 2.0;
      } else if (c->repair == ORC_REP_REINIT) { /* de/strategy.hpp:285-289 */
        if (g < lb || g > ub) g = lb + (ub - lb) * uniform01(r);
      } else {
        for (int fold = 0; (g < lb || g > ub) && fold < 100; ++fold) {
          if (g < lb) g = lb + (lb - g);
          if (g > ub) g = ub - (g - ub);
        }
        if (g < lb) g = lb;
        if (g > ub) g = ub;
      }
      t[j] = g;
    }
    tfit[i] = orc_objective(c, t, diff, z);
    Fs[i] = F;
    CRs[i] = CR;
    if (F_out) F_out[i] = F;
    if (CR_out) CR_out[i] = CR;
    if (idx_out) { idx_out[4 * i] = a; idx_out[4 * i + 1] = b; idx_out[4 * i + 2] = cc; idx_out[4 * i + 3] = 0; }
    if (jrand_out) jrand_out[i] = jr;
    if (words_out) words_out[i] = r->consumed - w0;
  }
  /* select_and_archive, de/engine.hpp:27-47 + adapter update */
  const int64_t aw0 = r->consumed;
  double gain_sum = 0.0;
  int n_succ = 0;
  int* succ = (int*)malloc(sizeof(int) * P);
  double* gains = (double*)malloc(sizeof(double) * P);
  for (int i = 0; i < P; ++i) {
    const int w = tfit[i] <= s->fit[i];
    if (win_out) win_out[i] = w;
    if (!w) continue;
    const double gain = s->fit[i] - tfit[i];
    if (gain > 0.0) { succ[n_succ] = i; gains[n_succ] = gain; ++n_succ; }
    if (c->archive_cap > 0) { /* de/strategy.hpp:29-37 */
      if (s->arch_size < c->archive_cap) {
        memcpy(s->archive + (size_t)s->arch_size * D, s->pop + (size_t)i * D, sizeof(double) * D);
        s->arch_size++;
      } else {
        const int v = uniform_int(r, s->arch_size);
        memcpy(s->archive + (size_t)v * D, s->pop + (size_t)i * D, sizeof(double) * D);
      }
    }
    memcpy(s->pop + (size_t)i * D, trials + (size_t)i * D, sizeof(double) * D);
    s->fit[i] = tfit[i];
  }
  if (n_succ > 0 && c->parameter == ORC_PAR_SHADE) { /* de/parameter.hpp:166-184 */
    for (int k = 0; k < n_succ; ++k) gain_sum += gains[k];
    double fn = 0.0, fd = 0.0, ca = 0.0;
    for (int k = 0; k < n_succ; ++k) {
      const double w = gains[k] / gain_sum;
      const double f = Fs[succ[k]];
      fn += w * f * f;
      fd += w * f;
      ca += w * CRs[succ[k]];
    }
    s->mem_f[s->write_index] = fn / fd;
    s->mem_cr[s->write_index] = ca;
    s->write_index = (s->write_index + 1) % c->H;
  } else if (n_succ > 0 && c->parameter == ORC_PAR_JADE) { /* de/parameter.hpp:107-120 */
    double num = 0.0, den = 0.0, crm = 0.0;
    for (int k = 0; k < n_succ; ++k) { num += Fs[succ[k]] * Fs[succ[k]]; den += Fs[succ[k]]; }
    for (int k = 0; k < n_succ; ++k) crm += CRs[succ[k]];
    crm /= (double)n_succ;
    s->mem_f[0] = (1.0 - c->jade_c) * s->mem_f[0] + c->jade_c * (num / den);
    s->mem_cr[0] = (1.0 - c->jade_c) * s->mem_cr[0] + c->jade_c * crm;
  }
  const int64_t aw = r->consumed - aw0;
  free(order); free(trials); free(tfit); free(Fs); free(CRs); free(diff); free(z); free(donor); free(succ); free(gains);
  return aw;
}

ORC_API int orc_de_cfg_size(void) { return (int)sizeof(orc_de_cfg); }
ORC_API int orc_de_state_size(void) { return (int)sizeof(orc_de_state); }

/* ------------------------------------------------------------------------------------------
 * Synchronous PSO generation (config 3), restated from pso/topology.hpp:28-54,
 * pso/update.hpp:66-74, pso/engine.hpp:66-79 plus the config's velocity clamp.
 * ---------------------------------------------------------------------------------------- */
#define DEFINE_PSO(T, SUF)                                                                              \
  ORC_API void orc_pso_step_##SUF(int topology, double w_, double c1_, double c2_, double vmax_, int P, int D, \
                                  int kind, const T* shift, const T* rot, T bias, T* x, T* v, T* fit, T* pb,   \
                                  T* pbf, const uint64_t* words, int64_t n_words, T lb, T ub, int* nb_out) {   \
    orc_rng r;                                                                                          \
    orc_rng_scripted(&r, words, n_words);                                                               \
    const T w = (T)w_, c1 = (T)c1_, c2 = (T)c2_, vmax = (T)vmax_;                                       \
    int* nb = (int*)malloc(sizeof(int) * P);                                                            \
    for (int i = 0; i < P; ++i) {                                                                       \
      int best = -1;                                                                                    \
      if (topology == 0) {                                                                              \
        best = 0;                                                                                       \
        for (int k = 1; k < P; ++k)                                                                     \
          if (pbf[k] < pbf[best]) best = k;                                                             \
      } else {                                                                                          \
        for (int off = -1; off <= 1; ++off) {                                                           \
          const int c = ((i + off) % P + P) % P;                                                        \
          if (best < 0 || pbf[c] < pbf[best] || (pbf[c] == pbf[best] && c < best)) best = c;           \
        }                                                                                               \
      }                                                                                                 \
      nb[i] = best;                                                                                     \
      if (nb_out) nb_out[i] = best;                                                                     \
    }                                                                                                   \
    for (int i = 0; i < P; ++i) {                                                                       \
      T* xi = x + (size_t)i * D;                                                                        \
      T* vi = v + (size_t)i * D;                                                                        \
      const T* p = pb + (size_t)i * D;                                                                  \
      const T* l = pb + (size_t)nb[i] * D;                                                              \
      for (int j = 0; j < D; ++j) {                                                                     \
        const T r1 = (T)uniform01(&r);                                                                  \
        const T r2 = (T)uniform01(&r);                                                                  \
        vi[j] = w * vi[j] + c1 * r1 * (p[j] - xi[j]) + c2 * r2 * (l[j] - xi[j]);                        \
      }                                                                                                 \
      for (int j = 0; j < D; ++j) {                                                                     \
        if (vmax > (T)0) {                                                                              \
          if (vi[j] > vmax) vi[j] = vmax;                                                               \
          if (vi[j] < -vmax) vi[j] = -vmax;                                                             \
        }                                                                                               \
        xi[j] += vi[j];                                                                                 \
        if (xi[j] < lb) { xi[j] = lb; vi[j] = (T)(-0.5) * vi[j]; }                                      \
        else if (xi[j] > ub) { xi[j] = ub; vi[j] = (T)(-0.5) * vi[j]; }                                 \
      }                                                                                                 \
    }                                                                                                   \
    /* pbest snapshot semantics: all moves use the start-of-generation pbests (read above) */           \
    T* diff = (T*)malloc(sizeof(T) * D);                                                                \
    T* z = (T*)malloc(sizeof(T) * D);                                                                   \
    for (int i = 0; i < P; ++i) {                                                                       \
      transform_##SUF(x + (size_t)i * D, shift, rot, D, diff, z);                                      \
      fit[i] = base_value_##SUF(kind, z, D) + bias;                                                     \
      if (fit[i] < pbf[i]) {                                                                            \
        memcpy(pb + (size_t)i * D, x + (size_t)i * D, sizeof(T) * D);                                   \
        pbf[i] = fit[i];                                                                                \
      }                                                                                                 \
    }                                                                                                   \
    free(diff); free(z); free(nb);                                                                      \
  }
DEFINE_PSO(double, f64)
DEFINE_PSO(float, f32)

/* The sequential word list one rand/1 (mutation 0) or best/1 (mutation 1) + binomial generation
 * consumes when individual i draws from Philox sub-stream (gen << 32) | i: the rejection loops
 * of de/strategy.hpp:84-86 / 109-110 decide how many index words precede jrand and the D gene
 * uniforms.  Fitness-independent, so the oracle can rebuild it.  Returns the word count. */
ORC_API int64_t orc_de_fixed_generation_words(int mutation, uint64_t key, uint32_t gen, int P, int D, uint64_t* out,
                                              int64_t cap) {
  int64_t n = 0;
  for (int i = 0; i < P; ++i) {
    const uint64_t hi = ((uint64_t)gen << 32) | (uint32_t)i;
    uint64_t pos = 0;
    int a = -1, b, c;
    if (mutation == 0) {
      do { a = orc_uniform_int_word(orc_philox_word(key, hi, pos++), P); } while (a == i);
    }
    do { b = orc_uniform_int_word(orc_philox_word(key, hi, pos++), P); } while (b == i || (mutation == 0 && b == a));
    do { c = orc_uniform_int_word(orc_philox_word(key, hi, pos++), P); } while (c == i || c == b || (mutation == 0 && c == a));
    pos += 1 + (uint64_t)D; /* jrand + gene uniforms */
    for (uint64_t q = 0; q < pos; ++q) {
      if (n < cap) out[n] = orc_philox_word(key, hi, q);
      ++n;
    }
  }
  return n;
}

/* A composition instance's components drawn like make_instance does for compositions
 * (problems/suite.hpp:134-143): one stream, per component draw_shift then draw_rotation. */
ORC_API void orc_make_composition(uint64_t seed, uint64_t stream_id, int dim, int n_comp, double* shifts,
                                  double* rots) {
  orc_rng r;
  orc_rng_init(&r, seed, stream_id);
  for (int c = 0; c < n_comp; ++c) {
    orc_draw_shift(&r, dim, -100.0, 100.0, shifts + (size_t)c * dim);
    orc_random_rotation(&r, dim, rots + (size_t)c * dim * dim);
  }
}

/* ---- cso_optimizer::generation (pso/cso.hpp:31-72), fp64, base objective ------------------------ */
/* x, v: P x D (row-major), fit: P; words consumed in the reference's order (scripted rng).  The
 * losers' new fitness uses the scalar path (problems/instance.hpp:221-233).  Returns words used. */
ORC_API int64_t orc_cso_generation_f64(int P, int D, double phi, int kind, const double* shift, const double* rot,
                                       double bias, double* x, double* v, double* fit, double lb, double ub,
                                       const uint64_t* words, int64_t n_words) {
  orc_rng r;
  orc_rng_scripted(&r, words, n_words);
  double* mean = (double*)calloc((size_t)D, sizeof(double));
  int* perm = (int*)malloc(sizeof(int) * (size_t)P);
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < D; ++j) mean[j] += x[(size_t)i * D + j]; /* cso.hpp:37-40, i ascending */
  for (int j = 0; j < D; ++j) mean[j] /= (double)P;              /* :41-42 */
  for (int i = 0; i < P; ++i) perm[i] = i;                        /* iota, :44 */
  for (int k = P - 1; k >= 1; --k) {                              /* Fisher-Yates, :45-47 */
    const int q = uniform_int(&r, k + 1);
    const int t = perm[k];
    perm[k] = perm[q];
    perm[q] = t;
  }
  for (int t = 0; t < P / 2; ++t) { /* :49-69 */
    const int a = perm[2 * t], b = perm[2 * t + 1];
    const int w = fit[a] <= fit[b] ? a : b;
    const int l = w == a ? b : a;
    double* xl = x + (size_t)l * D;
    double* vl = v + (size_t)l * D;
    const double* xw = x + (size_t)w * D;
    for (int j = 0; j < D; ++j) {
      const double r1 = uniform01(&r), r2 = uniform01(&r), r3 = uniform01(&r);
      vl[j] = r1 * vl[j] + r2 * (xw[j] - xl[j]) + phi * r3 * (mean[j] - xl[j]);
      xl[j] += vl[j];
      xl[j] = xl[j] < lb ? lb : (ub < xl[j] ? ub : xl[j]); /* std::clamp */
    }
    fit[l] = orc_eval_scalar_f64(kind, D, shift, rot, bias, xl);
  }
  free(mean);
  free(perm);
  return r.consumed;
}
