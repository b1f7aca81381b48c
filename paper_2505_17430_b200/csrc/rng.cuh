// rng.cuh — device random words and the reference's sampling arithmetic.
//
// Two word sources (the `evb_rng` object):
//   * PHILOX: counter-based Philox4x32-10.  word(key, ctr_hi, n) is the 64-bit value formed by
//     output lanes (2*(n&1), 2*(n&1)+1) of block n>>1 with 128-bit counter
//     (lo32(n>>1), hi32(n>>1), lo32(ctr_hi), hi32(ctr_hi)).  The engines give every
//     (generation, individual) its own sub-stream ctr_hi = (generation << 32) | sub, so all
//     individuals draw in parallel; the words each one consumed are exported so the CPU
//     reference can replay the identical sequence through rng_stream::scripted
//     (core/rng.hpp:54-58).
//   * WORDS: a device copy of a caller-supplied word list consumed strictly sequentially, in the
//     reference's own order (oracle mode: e.g. the words of rng_stream(42, 0) itself).
// The double-precision mappings restate core/rng.hpp:81-107 exactly.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace evb {

enum rng_mode { RNG_PHILOX = 0, RNG_WORDS = 1 };

constexpr uint32_t kSubArchive = 0xFFFFFFFFu;  // archive-victim draws of a generation
constexpr uint32_t kSubInit = 0xFFFFFFF0u;     // init_population draws
constexpr uint32_t kSubShrink = 0xFFFFFFFEu;   // archive set_capacity victims after a population reduction
constexpr uint32_t kSubEngine = 0xFFFFFFE0u;   // engine-level draws (archive shrink, restarts)

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = uint64_t(0xD2511F53u) * c[0];
    const uint64_t p1 = uint64_t(0xCD9E8D57u) * c[2];
    const uint32_t n0 = uint32_t(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = uint32_t(p0 >> 32) ^ c[3] ^ k1;
    c[1] = uint32_t(p1);
    c[3] = uint32_t(p0);
    c[0] = n0;
    c[2] = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Philox4x32-10 with the 20 round keys precomputed (host side, once per source): kernels that
// draw many blocks take them from their parameter bank instead of re-deriving the key schedule
// per block, and the 32x32 -> 64 products are single mul.wide instructions.  Same values as
// philox4x32_10.
struct philox_keys {
  uint32_t rk[20];
  __host__ __device__ philox_keys(uint64_t key = 0) {
    uint32_t k0 = uint32_t(key), k1 = uint32_t(key >> 32);
    for (int r = 0; r < 10; ++r) {
      rk[2 * r] = k0;
      rk[2 * r + 1] = k1;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
};

__device__ __forceinline__ uint64_t mul_wide_u32(uint32_t a, uint32_t b) {
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
  return p;
}

__device__ __forceinline__ void philox4x32_10_rk(uint32_t c[4], const philox_keys& ks) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = mul_wide_u32(c[0], 0xD2511F53u);
    const uint64_t p1 = mul_wide_u32(c[2], 0xCD9E8D57u);
    const uint32_t n0 = uint32_t(p1 >> 32) ^ c[1] ^ ks.rk[2 * r];
    const uint32_t n2 = uint32_t(p0 >> 32) ^ c[3] ^ ks.rk[2 * r + 1];
    c[1] = uint32_t(p1);
    c[3] = uint32_t(p0);
    c[0] = n0;
    c[2] = n2;
  }
}

__host__ __device__ __forceinline__ uint64_t philox_word(uint64_t key, uint64_t ctr_hi, uint64_t n) {
  const uint64_t blk = n >> 1;
  uint32_t c[4] = {uint32_t(blk), uint32_t(blk >> 32), uint32_t(ctr_hi), uint32_t(ctr_hi >> 32)};
  philox4x32_10(c, uint32_t(key), uint32_t(key >> 32));
  return (n & 1) ? ((uint64_t(c[3]) << 32) | c[2]) : ((uint64_t(c[1]) << 32) | c[0]);
}

// Both words of one Philox block (n even, n+1).
__host__ __device__ __forceinline__ void philox_pair(uint64_t key, uint64_t ctr_hi, uint64_t blk, uint64_t& w0,
                                                     uint64_t& w1) {
  uint32_t c[4] = {uint32_t(blk), uint32_t(blk >> 32), uint32_t(ctr_hi), uint32_t(ctr_hi >> 32)};
  philox4x32_10(c, uint32_t(key), uint32_t(key >> 32));
  w0 = (uint64_t(c[1]) << 32) | c[0];
  w1 = (uint64_t(c[3]) << 32) | c[2];
}

struct word_source {
  int mode;
  uint64_t key;
  const uint64_t* words;  // WORDS mode
  int64_t n_words;
};

// Sequential reader over one stream: a Philox sub-stream (ctr_hi) or the word list from `pos`.
struct word_reader {
  const word_source* src;
  uint64_t ctr_hi;
  int64_t pos;    // next word index in the stream
  int64_t count;  // words consumed by this reader
  int* overflow;  // set when a WORDS list is exhausted

  __device__ __forceinline__ uint64_t next() {
    ++count;
    const int64_t n = pos++;
    if (src->mode == RNG_PHILOX) return philox_word(src->key, ctr_hi, uint64_t(n));
    if (n >= src->n_words) {
      if (overflow) *overflow = 1;
      return 0;
    }
    return src->words[n];
  }
};

// A Philox sub-stream with its first 2 * NB words computed up front: NB independent Philox blocks
// (instruction-level parallel) instead of one block per word in sequence, each recomputing its
// pair's block.  Word n is still philox_word(key, ctr_hi, n), so values and `count` are exactly
// word_reader's for a PHILOX source.
template <int NB>
struct philox_prefetch_reader {
  uint64_t key, ctr_hi;
  int64_t count = 0;
  uint64_t w[2 * NB];
  __device__ __forceinline__ philox_prefetch_reader(uint64_t k, uint64_t c) { reset(k, c); }
  __device__ __forceinline__ philox_prefetch_reader() : key(0), ctr_hi(0) {}  // reset() before use
  __device__ __forceinline__ void reset(uint64_t k, uint64_t c) {
    key = k;
    ctr_hi = c;
    count = 0;
#pragma unroll
    for (int b = 0; b < NB; ++b) philox_pair(k, c, uint64_t(b), w[2 * b], w[2 * b + 1]);
  }
  __device__ __forceinline__ uint64_t next() {
    const int64_t n = count++;
    if (n >= 2 * NB) return philox_word(key, ctr_hi, uint64_t(n));
    const uint64_t v = w[0];  // shift the prefetched words down (registers, no dynamic index)
#pragma unroll
    for (int q = 0; q + 1 < 2 * NB; ++q) w[q] = w[q + 1];
    return v;
  }
};

__device__ __forceinline__ uint64_t word_at(const word_source& s, uint64_t ctr_hi, int64_t n, int* overflow) {
  if (s.mode == RNG_PHILOX) return philox_word(s.key, ctr_hi, uint64_t(n));
  if (n >= s.n_words) {
    if (overflow) *overflow = 1;
    return 0;
  }
  return s.words[n];
}

// core/rng.hpp:81-107
__device__ __forceinline__ double u01_of(uint64_t w) { return double(w >> 11) * 0x1.0p-53; }
__device__ __forceinline__ double u01pos_of(uint64_t w) { return double((w >> 11) + 1) * 0x1.0p-53; }
__device__ __forceinline__ int uint_of(uint64_t w, int n) { return int(__umul64hi(w, uint64_t(n))); }

template <typename R>
__device__ __forceinline__ double draw_uniform01(R& r) { return u01_of(r.next()); }
template <typename R>
__device__ __forceinline__ double draw_uniform(R& r, double lo, double hi) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u01_of(r.next())));
}
template <typename R>
__device__ __forceinline__ int draw_int(R& r, int n) { return uint_of(r.next(), n); }
template <typename R>
__device__ __forceinline__ double draw_normal(R& r, double mean, double stddev) {
  const double u1 = u01pos_of(r.next());
  const double u2 = u01_of(r.next());
  const double rr = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
  return __dadd_rn(mean, __dmul_rn(__dmul_rn(stddev, rr), cos(__dmul_rn(2.0 * 3.14159265358979323846, u2))));
}
template <typename R>
__device__ __forceinline__ double draw_cauchy(R& r, double loc, double scale) {
  const double u = u01pos_of(r.next());
  return __dadd_rn(loc, __dmul_rn(scale, tan(__dmul_rn(3.14159265358979323846, __dsub_rn(u, 0.5)))));
}

}  // namespace evb
