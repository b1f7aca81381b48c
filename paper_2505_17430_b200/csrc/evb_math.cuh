// evb_math.cuh — device restatement of the reference objective arithmetic.
//
// Every operation that the reference performs as a separate IEEE mul/add is issued here as
// an explicitly rounded intrinsic (__dmul_rn, __fadd_rn, ...) so nvcc cannot contract it
// into an FMA: the reference's default Release build targets baseline x86-64, which has no
// FMA (CMakeLists.txt:3-8).  With that, a sequential-order evaluation on the GPU
// reproduces the reference bit-for-bit up to libm transcendental ulps.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "evb.h"

namespace evb {

template <typename T>
struct fop;

template <>
struct fop<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
  static __device__ __forceinline__ double exp_(double a) { return exp(a); }
  static __device__ __forceinline__ double cos_lib(double a) { return cos(a); }
  static __device__ __forceinline__ double sin_lib(double a) { return sin(a); }
};

template <>
struct fop<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
  static __device__ __forceinline__ float exp_(float a) { return expf(a); }
  static __device__ __forceinline__ float cos_lib(float a) { return cosf(a); }
  static __device__ __forceinline__ float sin_lib(float a) { return sinf(a); }
};

// problems/simd_math.hpp:16-32 — turn-reduced degree-13 Taylor sine evaluated in double.
__device__ __forceinline__ double sin_from_turns(double r) {
  r = __dsub_rn(r, rint(r));
  const double sign = r < 0.0 ? -1.0 : 1.0;
  double a = fabs(r);
  a = a > 0.25 ? __dsub_rn(0.5, a) : a;
  const double t = __dmul_rn(2.0 * 3.14159265358979323846, a);
  const double t2 = __dmul_rn(t, t);
  double p = 1.0 / 6227020800.0;
  p = __dsub_rn(__dmul_rn(p, t2), 1.0 / 39916800.0);
  p = __dadd_rn(__dmul_rn(p, t2), 1.0 / 362880.0);
  p = __dsub_rn(__dmul_rn(p, t2), 1.0 / 5040.0);
  p = __dadd_rn(__dmul_rn(p, t2), 1.0 / 120.0);
  p = __dsub_rn(__dmul_rn(p, t2), 1.0 / 6.0);
  p = __dadd_rn(__dmul_rn(p, t2), 1.0);
  return __dmul_rn(__dmul_rn(sign, t), p);
}
// problems/simd_math.hpp:36-44
__device__ __forceinline__ float fast_sin(float x) {
  constexpr double inv_two_pi = 1.0 / (2.0 * 3.14159265358979323846);
  return float(sin_from_turns(__dmul_rn(double(x), inv_two_pi)));
}
__device__ __forceinline__ float fast_cos(float x) {
  constexpr double inv_two_pi = 1.0 / (2.0 * 3.14159265358979323846);
  return float(sin_from_turns(__dadd_rn(__dmul_rn(double(x), inv_two_pi), 0.25)));
}

// Trig used by a path: the batched base kernels use fast_cos/fast_sin for float and libm for
// double (problems/batch.hpp:17-33); the scalar kernels (hybrid, composition) use libm.
template <typename T, bool kBatchTrig>
struct trig {
  static __device__ __forceinline__ T cos_(T x) { return fop<T>::cos_lib(x); }
  static __device__ __forceinline__ T sin_(T x) { return fop<T>::sin_lib(x); }
};
template <>
struct trig<float, true> {
  static __device__ __forceinline__ float cos_(float x) { return fast_cos(x); }
  static __device__ __forceinline__ float sin_(float x) { return fast_sin(x); }
};

template <typename T>
__device__ __forceinline__ T two_pi_v() {
  return T(2) * T(3.14159265358979323846);
}
template <>
__device__ __forceinline__ float two_pi_v<float>() {
  // T(2) * std::numbers::pi_v<float>, evaluated in float (problems/functions.hpp:95)
  return 2.0f * 3.14159265f;
}
template <typename T>
__device__ __forceinline__ T e_v() {
  return T(2.718281828459045235360287471352662498);
}

// cos(2 pi v) without the rounding of 2 pi v: the period is taken out exactly (r = v - rint(v),
// rint by the 1.5 * 2^52 round-to-nearest trick: two adds, |r| <= 1/2) and cos(2 pi r) is a
// degree-11 polynomial in r^2 (Chebyshev interpolation on [0, 1/4], fitted in 50-digit
// arithmetic; max error 8e-16 over [-1/2, 1/2] evaluated in double): 14 FP64 ops on the DFMA
// pipe instead of the library cos's reduction.  It differs from the reference's cos(fl(2 pi v))
// by the rounding of that product, |2 pi v| * ~3.3e-16 (~2e-13 at |v| ~ 100), plus ~1e-15, so
// callers use it only while |v| < 2^16 (cos2pi_fast_ok) and take the reference's expression
// otherwise.  Tolerance paths only (the fused GEMM epilogue, the persistent runs' tensor-core
// evaluation); NaN passes through.
__device__ __forceinline__ double cos2pi_fast(double v) {
  const double t = __dsub_rn(__dadd_rn(v, 0x1.8p52), 0x1.8p52);  // rint(v) for |v| < 2^51
  const double r = __dsub_rn(v, t);
  const double u = __dmul_rn(r, r);
  double c = -0.0002900600501912893;
  c = fma(c, u, 0.003758590561310354);
  c = fma(c, u, -0.03637490036340231);
  c = fma(c, u, 0.28200407958316315);
  c = fma(c, u, -1.7143904138098518);
  c = fma(c, u, 7.903536340077173);
  c = fma(c, u, -26.42625678121189);
  c = fma(c, u, 60.24464137178173);
  c = fma(c, u, -85.45681720669127);
  c = fma(c, u, 64.93939402266825);
  c = fma(c, u, -19.739208802178716);
  return fma(c, u, 1.0);
}
__device__ __forceinline__ bool cos2pi_fast_ok(double v) { return !(fabs(v) >= 65536.0); }

// ---- per-element terms, exactly as written in the reference ------------------------------
// rastrigin term: v * v - T(10) * cos(two_pi * v) + T(10)   (problems/batch.hpp:161)
template <typename T, bool kBatchTrig>
__device__ __forceinline__ T rastrigin_term(T v) {
  using F = fop<T>;
  const T c = trig<T, kBatchTrig>::cos_(F::mul(two_pi_v<T>(), v));
  return F::add(F::sub(F::mul(v, v), F::mul(T(10), c)), T(10));
}
// elliptic term: w * zi * zi  ((w*z)*z association, problems/batch.hpp:114)
template <typename T>
__device__ __forceinline__ T elliptic_term(T w, T v) {
  using F = fop<T>;
  return F::mul(F::mul(w, v), v);
}
// ackley finalisation (problems/batch.hpp:179-183)
template <typename T>
__device__ __forceinline__ T ackley_final(T sum_sq, T sum_cos, int dim) {
  using F = fop<T>;
  const T inv_d = F::div(T(1), T(dim));
  const T a = F::mul(T(-20), F::exp_(F::mul(T(-0.2), F::sqrt_(F::mul(sum_sq, inv_d)))));
  const T b = F::exp_(F::mul(sum_cos, inv_d));
  return F::add(F::add(F::sub(a, b), T(20)), e_v<T>());
}
// schaffer_f6 pair term (problems/batch.hpp:222-227)
template <typename T, bool kBatchTrig>
__device__ __forceinline__ T schaffer_term(T x, T y) {
  using F = fop<T>;
  const T ssq = F::add(F::mul(x, x), F::mul(y, y));
  const T sv = trig<T, kBatchTrig>::sin_(F::sqrt_(ssq));
  const T dv = F::add(T(1), F::mul(T(0.001), ssq));
  return F::add(T(0.5), F::div(F::sub(F::mul(sv, sv), T(0.5)), F::mul(dv, dv)));
}

// ---- sequential base value over an accessor z(i), i in [0, n) -----------------------------
// Mirrors problems/functions.hpp:46-152 / problems/batch.hpp:95-233 in accumulation order.
// `plus_one` applies the rosenbrock z + 1 convention of base_value_origin
// (problems/instance.hpp:82-91).  `w` is the host-computed elliptic weight table (may be null
// when kind != elliptic); the weights depend on the chunk length n, so hybrids pass their
// own chunk table.
template <typename T, bool kBatchTrig, typename Z>
__device__ T base_value_seq(int kind, int n, const Z& z, const T* w) {
  using F = fop<T>;
  switch (kind) {
    case EVB_SPHERE: {
      T acc = T(0);
      for (int i = 0; i < n; ++i) {
        const T v = z(i);
        acc = F::add(acc, F::mul(v, v));
      }
      return acc;
    }
    case EVB_ELLIPTIC: {
      T acc = T(0);
      for (int i = 0; i < n; ++i) acc = F::add(acc, elliptic_term<T>(w[i], z(i)));
      return acc;
    }
    case EVB_BENT_CIGAR:
    case EVB_DISCUS: {
      T acc = T(0);
      for (int i = 1; i < n; ++i) {
        const T v = z(i);
        acc = F::add(acc, F::mul(v, v));
      }
      const T z0 = z(0);
      if (kind == EVB_BENT_CIGAR) return F::add(F::mul(z0, z0), F::mul(T(1e6), acc));
      return F::add(F::mul(F::mul(T(1e6), z0), z0), acc);
    }
    case EVB_ROSENBROCK: {  // evaluated on z + 1
      T acc = T(0);
      for (int i = 0; i + 1 < n; ++i) {
        const T wi = F::add(z(i), T(1));
        const T wn = F::add(z(i + 1), T(1));
        const T q = F::sub(F::mul(wi, wi), wn);
        const T r = F::sub(wi, T(1));
        acc = F::add(acc, F::add(F::mul(F::mul(T(100), q), q), F::mul(r, r)));
      }
      return acc;
    }
    case EVB_RASTRIGIN: {
      T acc = T(0);
      for (int i = 0; i < n; ++i) acc = F::add(acc, rastrigin_term<T, kBatchTrig>(z(i)));
      return acc;
    }
    case EVB_ACKLEY: {
      T ssq = T(0), scos = T(0);
      for (int i = 0; i < n; ++i) {
        const T v = z(i);
        ssq = F::add(ssq, F::mul(v, v));
        scos = F::add(scos, trig<T, kBatchTrig>::cos_(F::mul(two_pi_v<T>(), v)));
      }
      return ackley_final<T>(ssq, scos, n);
    }
    case EVB_GRIEWANK: {
      T sum = T(0), prod = T(1);
      for (int i = 0; i < n; ++i) {
        const T v = z(i);
        sum = F::add(sum, F::mul(v, v));
        prod = F::mul(prod, trig<T, kBatchTrig>::cos_(F::div(v, F::sqrt_(T(i + 1)))));
      }
      return F::add(F::sub(F::div(sum, T(4000)), prod), T(1));
    }
    case EVB_SCHWEFEL_12: {
      T acc = T(0), cum = T(0);
      for (int i = 0; i < n; ++i) {
        cum = F::add(cum, z(i));
        acc = F::add(acc, F::mul(cum, cum));
      }
      return acc;
    }
    case EVB_EXPANDED_SCHAFFER_F6: {
      if (n == 1) return schaffer_term<T, kBatchTrig>(z(0), z(0));
      T acc = T(0);
      for (int i = 0; i < n; ++i) acc = F::add(acc, schaffer_term<T, kBatchTrig>(z(i), z((i + 1) % n)));
      return acc;
    }
    default:
      return T(0);
  }
}

}  // namespace evb

namespace evb {

// ---- split form of base_value_seq for latency hiding ---------------------------------------------
// The transcendental part of each element (the whole Rastrigin / Schaffer term, the cosine of
// Ackley / Griewank) is independent across elements, so a whole CTA can compute it in parallel
// into `pre`; the reference's sequential accumulation then runs over `pre` with cheap ops only.
// base_value_pre(kind, n, z, pre, w) == base_value_seq(kind, n, z, w) bit for bit.
__host__ __device__ inline bool kind_has_pre(int kind) {
  return kind == EVB_RASTRIGIN || kind == EVB_ACKLEY || kind == EVB_GRIEWANK || kind == EVB_EXPANDED_SCHAFFER_F6;
}

template <typename T, bool kBatchTrig, typename Z>
__device__ __forceinline__ T base_pre_term(int kind, int n, const Z& z, int i) {
  using F = fop<T>;
  switch (kind) {
    case EVB_RASTRIGIN: return rastrigin_term<T, kBatchTrig>(z(i));
    case EVB_ACKLEY: return trig<T, kBatchTrig>::cos_(F::mul(two_pi_v<T>(), z(i)));
    case EVB_GRIEWANK: return trig<T, kBatchTrig>::cos_(F::div(z(i), F::sqrt_(T(i + 1))));
    case EVB_EXPANDED_SCHAFFER_F6: return n == 1 ? schaffer_term<T, kBatchTrig>(z(0), z(0))
                                                 : schaffer_term<T, kBatchTrig>(z(i), z((i + 1) % n));
  }
  return T(0);
}

template <typename T, bool kBatchTrig, typename Z, typename PRE>
__device__ T base_value_pre(int kind, int n, const Z& z, const PRE& pre, const T* w) {
  using F = fop<T>;
  switch (kind) {
    case EVB_RASTRIGIN: {
      T acc = T(0);
      for (int i = 0; i < n; ++i) acc = F::add(acc, pre(i));
      return acc;
    }
    case EVB_ACKLEY: {
      T ssq = T(0), scos = T(0);
      for (int i = 0; i < n; ++i) {
        const T v = z(i);
        ssq = F::add(ssq, F::mul(v, v));
        scos = F::add(scos, pre(i));
      }
      return ackley_final<T>(ssq, scos, n);
    }
    case EVB_GRIEWANK: {
      T sum = T(0), prod = T(1);
      for (int i = 0; i < n; ++i) {
        const T v = z(i);
        sum = F::add(sum, F::mul(v, v));
        prod = F::mul(prod, pre(i));
      }
      return F::add(F::sub(F::div(sum, T(4000)), prod), T(1));
    }
    case EVB_EXPANDED_SCHAFFER_F6: {
      if (n == 1) return pre(0);
      T acc = T(0);
      for (int i = 0; i < n; ++i) acc = F::add(acc, pre(i));
      return acc;
    }
    default:
      return base_value_seq<T, kBatchTrig>(kind, n, z, w);
  }
}

// hybrid problems (problems/instance.hpp:97-112): z permuted, split into chunks, the chunks'
// base values (libm trig) summed in order; hyb_w holds each chunk's elliptic weights at its offset
template <typename T>
__device__ __forceinline__ T hybrid_value(const int* perm, const int* sub_kinds, const int* chunk_sizes, int n_chunks,
                          const T* hyb_w, const T* zrow, int64_t zstride) {
  // problems/instance.hpp:97-112: permute, split into chunks, sum chunk base values (libm trig)
  using F = fop<T>;
  T total = T(0);
  int offset = 0;
  for (int c = 0; c < n_chunks; ++c) {
    const int len = chunk_sizes[c];
    const int off = offset;
    auto z = [&](int i) { return zrow[int64_t(perm[off + i]) * zstride]; };
    total = F::add(total, base_value_seq<T, false>(sub_kinds[c], len, z, hyb_w + off));
    offset += len;
  }
  return total;
}

}  // namespace evb
