// eval_gemm.cu — large-dimension batched objective evaluation (K1 fp64 / K2 fp32).
//
// Replaces problems/batch.hpp:40-235 (transform_batch + base_kernel_batch) for base problems.
//   z[b][i] = sum_k M[i][k] * (x_b[k] - o[k])        an NT GEMM: both operands K-contiguous
//   f[b]    = base(z[b]) + bias                        fused epilogue + deterministic row sum
//
// Structure (one CTA per BM x BN output tile, warp-specialised):
//   * producer warp: TMA (cp.async.bulk.tensor, SWIZZLE_128B) streams 16-double (fp64) or
//     32-float (fp32) K-slices of X and M into a STAGES-deep mbarrier ring; the matching slice
//     of the shift o rides along as a 128-byte bulk copy on the same barrier;
//   * consumer warps: the shift is applied while fragments are loaded from shared memory
//     (x - o rounded in T exactly like problems/batch.hpp:50), then
//       fp64: DMMA m8n8k4 tensor-core tiles (the only FP64 tensor route on sm_100a;
//             tcgen05 has no f64 kind), operands as conflict-free LDS.128 pairs
//             (k order permuted inside each 16-deep slice, dmma_kslice);
//       fp32: a three-product split (3xFP16 by default, 3xTF32 selectable) on tcgen05 with TMEM
//       accumulators (umma.cuh), or FFMA register-tiled
//             outer products for discus / hybrids / compositions (1xTF32 fails the 1e-4
//             tolerance);
//   * epilogue: per-element transform terms (elliptic / rastrigin / ackley / sphere /
//     bent-cigar / discus / griewank) are reduced per row inside the CTA, written as per-N-tile
//     partials, and the last CTA of each row block (ticket counter) sums the partials in fixed
//     N-tile order and applies the final formula + bias.  No float atomics: results are
//     deterministic run to run.
//   * several problems on one population (multi-problem K1): one CTA per tile holds a warp
//     group per problem, the X slice is staged once for all of them.
//   * z-store mode writes z in the reference's SoA layout (soa_z[i*ldz + b]) for the kinds
//     whose epilogue needs neighbours or prefixes (rosenbrock, schwefel_1.2, schaffer F6,
//     hybrids); eval_small.cu's row kernel finishes those.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>
#include <cstdio>

#include "evb_internal.cuh"
#include "evb_math.cuh"
#include "ptx.cuh"
#include "umma.cuh"

namespace evb {

// ---------------------------------------------------------------------------------------
// channel terms of the fused epilogue
enum term_id {
  TERM_SQ = 0,    // v*v
  TERM_WSQ = 1,   // (w_i*v)*v                      elliptic
  TERM_RAST = 2,  // v*v - 10 cos(2 pi v) + 10      rastrigin
  TERM_COS = 3,   // cos(2 pi v)                    ackley
  TERM_TAIL = 4,  // v*v for i >= 1                 bent cigar / discus
  TERM_HEAD = 5,  // v at i == 0 (raw z0)           bent cigar / discus
  TERM_GCOS = 6   // product of cos(v / sqrt(i+1))  griewank
};

constexpr int kMaxCh = 6;
constexpr int kMaxOut = 4;

template <typename T>
struct fused_params {
  int P, D;
  const T* ell_w;  // elliptic weights (length D), may be null
  int n_ch;
  int ch_term[kMaxCh];
  int n_out;
  int out_kind[kMaxOut];
  double out_bias[kMaxOut];
  int out_ch0[kMaxOut], out_ch1[kMaxOut];
  T* out;
  int64_t ldo;
  T* partial;          // [n_ch][n_ntiles][P]
  unsigned* counters;  // [n_mtiles]
  int n_ntiles;
  T* zbuf;  // non-null: z-store mode, zbuf[i*ldz + b]
  int64_t ldz;
  const T* shift;  // padded with zeros beyond D
  const unsigned* kgate;  // non-null: X columns arrive in chunks (see eval_request)
  int kgate_n;
  int kgate_end[8];
  unsigned kgate_epoch;
  int kgate_rows;   // > 0: rows >= kgate_rows wait on the second gate group kgate[kgate_n + c]
  int tiles_nfast;  // multi kernel: blockIdx.x walks column tiles (row blocks form the waves)
  unsigned long long* dbg_ts;  // EVB_K1_TIMELINE=1 (tuning aid): per-CTA globaltimer phase stamps
  int dbg_skip;  // EVB_K2_SKIP (tuning aid, wrong results): bit 0 = no S split, bit 1 = no MMAs
  // 3xFP16 range guard: rows with a non-finite or too large |x - o| are flagged by the split warps
  // and recomputed in fp32 (the reference's mul / add order) by the row block's last CTA
  int* row_bad;     // [P], zero between launches
  const T* Xrows;   // the population (row pitch ldxr) and the unsplit rotation (row pitch ldm)
  int64_t ldxr;
  const T* rot;
  int64_t ldm;
  int b_early;   // split-K fp32: the rotation split predates this launch, its first B slices may
                 // load before griddep_wait (they do not depend on the preceding kernel)
};

// cosine of the fused epilogue: library cos for fp64.  fp32 (a tolerance path: 3xTF32 / FFMA
// products already differ from the reference's order) reduces x = 2 pi z by 2 pi in float
// (Cody-Waite, 6.28125 exact for |k| < 2^15) and takes the SFU cosine on [-pi, pi]: absolute
// error ~1e-6, 4x cheaper than the reference's fast_cos evaluated in double (10.5 of 47 us per
// config-1 fp32 batch, measured).
template <typename T>
__device__ __forceinline__ T epi_cos(T x) { return trig<T, true>::cos_(x); }
// (out of line: inlined, the compiler predicates this double-precision polynomial into every
// element's straight-line code — ~2 us of FP64 pipe per config-1 fp32 Rastrigin epilogue)
__device__ __noinline__ float epi_cos_far(float x) { return trig<float, true>::cos_(x); }
// |x| < 1e5 (the caller's promise: no test here, so sixteen of these stay one straight-line block)
__device__ __forceinline__ float epi_cos_near(float x) {
  // rint by the 1.5 * 2^23 trick (|x / 2 pi| < 2^22 here): two full-rate adds instead of a
  // quarter-rate FRND
  const float k = __fadd_rn(__fadd_rn(x * 0.159154943091895336f, 12582912.f), -12582912.f);
  float r = fmaf(-k, 6.28125f, x);
  r = fmaf(-k, 1.93530717958647692e-3f, r);
  return __cosf(r);
}
template <>
__device__ __forceinline__ float epi_cos<float>(float x) {
  if (!(fabsf(x) < 1.0e5f)) return epi_cos_far(x);
  return epi_cos_near(x);
}

// cos(2 pi v) of the Rastrigin / Ackley terms.  fp64 fast form: the period is taken out exactly
// (r = v - rint(v), rint by the 1.5 * 2^52 round-to-nearest trick: two adds, |r| <= 1/2) and
// cos(2 pi r) is a degree-11 polynomial in r^2 (Chebyshev interpolation on [0, 1/4], fitted in
// 50-digit arithmetic; max error 8e-16 over [-1/2, 1/2] evaluated in double) — 14 FP64 ops on
// the DFMA pipe instead of the library cos's reduction.  It differs from the reference's
// cos(fl(2 pi * v)) by the rounding of that product, |2 pi v| * ~3.3e-16 (~2e-13 at |v| ~ 100),
// plus ~1e-15.  That bound grows with |v|, so the fast form is only used while |v| < 2^16
// (Ackley's mean-cosine error then stays < 2e-11 relative); callers take EXACT = true — the
// reference's own expression through libm-grade cos — for any larger (or non-finite) argument.
template <typename T, bool EXACT = false>
__device__ __forceinline__ T epi_cos2pi(T v) { return epi_cos<T>(fop<T>::mul(two_pi_v<T>(), v)); }
template <>
__device__ __forceinline__ double epi_cos2pi<double, true>(double v) { return cos(__dmul_rn(two_pi_v<double>(), v)); }
template <>
__device__ __forceinline__ double epi_cos2pi<double, false>(double v) {
  return cos2pi_fast(v);
}
// fp32: EXACT = false promises |v| < 15000 (|2 pi v| < 1e5) and skips the per-element range test —
// a branch per element splits the unrolled epilogue into one basic block per element and
// serialises the sixteen cosine chains (~1.3 us per config-1 Rastrigin launch)
template <>
__device__ __forceinline__ float epi_cos2pi<float, false>(float v) {
  return epi_cos_near(__fmul_rn(two_pi_v<float>(), v));
}
// arguments the fast forms may not take: fp64 |v| >= 2^16 or inf (NaN passes through the fast form);
// fp32 |v| >= 15000 or not finite
template <typename T>
__device__ __forceinline__ bool cos2pi_needs_exact(T v) {
  if (std::is_same<T, double>::value) return fabs(double(v)) >= 65536.0;
  return !(fabsf(float(v)) < 15000.f);
}

template <typename T, bool EXACT = false>
__device__ __forceinline__ T term_value(int term, T v, int col, const T* ell_w) {
  using F = fop<T>;
  switch (term) {
    case TERM_SQ: return F::mul(v, v);
    case TERM_WSQ: return elliptic_term<T>(ell_w[col], v);
    case TERM_RAST: {  // v*v - T(10) * cos(two_pi * v) + T(10)  (problems/batch.hpp:161)
      const T c = epi_cos2pi<T, EXACT>(v);
      return F::add(F::sub(F::mul(v, v), F::mul(T(10), c)), T(10));
    }
    case TERM_COS: return epi_cos2pi<T, EXACT>(v);
    case TERM_TAIL: return col >= 1 ? F::mul(v, v) : T(0);
    case TERM_HEAD: return col == 0 ? v : T(0);
    case TERM_GCOS: return epi_cos<T>(F::div(v, F::sqrt_(T(col + 1))));
  }
  return T(0);
}
__device__ __forceinline__ bool term_is_product(int term) { return term == TERM_GCOS; }

// Channel accumulation over 16 columns with the term fixed at compile time (keeps the unrolled
// epilogue free of per-element switches: one specialised loop per term instead of a 7-way
// switch replicated per unrolled element, which blew the instruction cache).
template <int TERM, typename T>
__device__ __forceinline__ T accumulate16(T acc, const T (&v)[16], int col0, int D, const T* ell_w) {
  constexpr bool prod = TERM == TERM_GCOS;
  constexpr bool has_cos2pi = TERM == TERM_RAST || TERM == TERM_COS;
  // one range test for the sixteen values (no per-element branch): the exact forms for all of
  // them if any needs it, else the fast forms as one straight-line block
  if constexpr (has_cos2pi) {
    bool far = false;
#pragma unroll
    for (int q = 0; q < 16; ++q) far = far || (col0 + q < D && cos2pi_needs_exact(v[q]));
    if (far) {  // (unrolled: a loop over q, or passing v by reference, would move v to local memory)
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int col = col0 + q;
        if (col < D) acc = fop<T>::add(acc, term_value<T, true>(TERM, v[q], col, ell_w));
      }
      return acc;
    }
    // straight-line: the cosine chains of the sixteen values overlap
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int col = col0 + q;
      const T t = term_value<T, false>(TERM, v[q], col < D ? col : 0, ell_w);
      const T a1 = fop<T>::add(acc, t);
      acc = col < D ? a1 : acc;
    }
    return acc;
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int col = col0 + q;
      if (col < D) {
        const T t = term_value<T, false>(TERM, v[q], col, ell_w);
        acc = prod ? fop<T>::mul(acc, t) : fop<T>::add(acc, t);
      }
    }
    return acc;
  }
}
template <typename T>
__device__ __forceinline__ T accumulate16_rt(int term, T acc, const T (&v)[16], int col0, int D, const T* ell_w) {
  switch (term) {
    case TERM_SQ: return accumulate16<TERM_SQ>(acc, v, col0, D, ell_w);
    case TERM_WSQ: return accumulate16<TERM_WSQ>(acc, v, col0, D, ell_w);
    case TERM_RAST: return accumulate16<TERM_RAST>(acc, v, col0, D, ell_w);
    case TERM_COS: return accumulate16<TERM_COS>(acc, v, col0, D, ell_w);
    case TERM_TAIL: return accumulate16<TERM_TAIL>(acc, v, col0, D, ell_w);
    case TERM_HEAD: return accumulate16<TERM_HEAD>(acc, v, col0, D, ell_w);
    default: return accumulate16<TERM_GCOS>(acc, v, col0, D, ell_w);
  }
}

// Final formula per base kind from its channel sums (problems/batch.hpp:96-233).
template <typename T>
__device__ __forceinline__ T finalize(int kind, T s0, T s1, int D, T bias) {
  using F = fop<T>;
  T v;
  switch (kind) {
    case EVB_SPHERE:
    case EVB_ELLIPTIC:
    case EVB_RASTRIGIN: v = s0; break;
    case EVB_BENT_CIGAR: v = F::add(F::mul(s1, s1), F::mul(T(1e6), s0)); break;  // s0 tail, s1 z0
    case EVB_DISCUS: v = F::add(F::mul(F::mul(T(1e6), s1), s1), s0); break;
    case EVB_ACKLEY: v = ackley_final<T>(s0, s1, D); break;  // s0 sum sq, s1 sum cos
    case EVB_GRIEWANK: v = F::add(F::sub(F::div(s0, T(4000)), s1), T(1)); break;
    default: v = T(0);
  }
  return F::add(v, bias);
}

// Shared tail of both kernels.  The accumulator tile has been parked in shared memory
// (zt[r * ldt + c], reusing the drained pipeline buffers) so the transcendental-heavy epilogue
// runs with the mainloop registers released.  Per channel: each consumer warp owns rows, lanes
// stride over the tile's columns, a shuffle tree gives the row sum of this N-tile; the last CTA
// of the row block (ticket counter) combines the N-tile partials in fixed order and applies
// the final formula.  Deterministic: fixed reduction trees, no float atomics.
struct epilogue_flag {
  int last;
};

// Per channel: each warp owns rows warp, warp + nwarps, ...; every lane evaluates all of its
// (row, column) terms of up to 8 rows before any shuffle (independent transcendental chains).
template <int TERM, typename T, int BM, int BN>
__device__ __forceinline__ void epilogue_rows(const fused_params<T>& p, const T* zt, int ldt, int m0, int n0, int warp,
                                              int lane, int nwarps, int rpw, int ch, int ntile) {
  using F = fop<T>;
  constexpr int CPL = (BN + 31) / 32;  // columns per lane
  constexpr bool prod = TERM == TERM_GCOS;
  const T ident = prod ? T(1) : T(0);
  // per-lane column data once per tile (elliptic weight, Griewank sqrt(i+1)); tile edges are
  // predicated (a select keeps the running value), so every element of the unrolled 8-row x
  // CPL-column block is an independent straight-line chain (no per-element branches: ILP)
  int cl[CPL];
  bool cv[CPL];
  T cw[CPL];
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) {
    const int c = lane + 32 * cc;
    cv[cc] = c < BN && n0 + c < p.D;
    cl[cc] = cv[cc] ? c : 0;
    const int col = n0 + cl[cc];
    if (TERM == TERM_WSQ) cw[cc] = p.ell_w[col];
    else if (TERM == TERM_GCOS) cw[cc] = F::sqrt_(T(col + 1));
    else cw[cc] = T(0);
  }
  const uint32_t zs = static_cast<uint32_t>(__cvta_generic_to_shared(zt));
  constexpr bool has_cos2pi = TERM == TERM_RAST || TERM == TERM_COS;
  for (int r0 = 0; r0 < rpw; r0 += 8) {
    T s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = ident;
    auto block = [&](auto exact_tag) {
      constexpr bool EXACT = decltype(exact_tag)::value;
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const int col = n0 + cl[cc];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = warp + (r0 + q) * nwarps;
          const bool ok = cv[cc] && r0 + q < rpw && r < BM;
          const T z = ptx::lds<T>(zs + uint32_t(((ok ? r : 0) * ldt + cl[cc]) * int(sizeof(T))));
          T v;
          if (TERM == TERM_WSQ) v = elliptic_term<T>(cw[cc], z);
          else if (TERM == TERM_GCOS) v = epi_cos<T>(F::div(z, cw[cc]));
          else v = term_value<T, EXACT>(TERM, z, col, p.ell_w);
          const T acc = prod ? F::mul(s[q], v) : F::add(s[q], v);
          s[q] = ok ? acc : s[q];
        }
      }
    };
    // the fast cos(2 pi v) form covers |v| < 2^16; a warp whose 8-row group holds a larger (or
    // non-finite) value evaluates that group with the reference's expression instead (uniform
    // branch: the common path stays straight-line)
    bool big = false;
    if constexpr (has_cos2pi) {
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = warp + (r0 + q) * nwarps;
          const bool ok = cv[cc] && r0 + q < rpw && r < BM;
          const T z = ptx::lds<T>(zs + uint32_t(((ok ? r : 0) * ldt + cl[cc]) * int(sizeof(T))));
          big = big || (ok && cos2pi_needs_exact(z));
        }
      big = __any_sync(0xffffffffu, big);
    }
    if (big) block(std::true_type{});
    else block(std::false_type{});
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      for (int off = 16; off > 0; off >>= 1) {
        const T o = __shfl_xor_sync(0xffffffffu, s[q], off);
        s[q] = prod ? F::mul(s[q], o) : F::add(s[q], o);
      }
      const int r = warp + (r0 + q) * nwarps;
      const int row = m0 + r;
      if (lane == 0 && r0 + q < rpw && r < BM && row < p.P) p.partial[(size_t(ch) * p.n_ntiles + ntile) * p.P + row] = s[q];
    }
  }
}

// Ackley's two channels (sum of squares, sum of cos(2 pi z)) in ONE pass over the parked tile: one
// shared-memory read per element and both shuffle trees per 8-row block (two separate passes made
// the Ackley group the slowest of a multi-problem CTA's epilogues).  Same terms and orders as
// epilogue_rows<TERM_SQ> + epilogue_rows<TERM_COS>.
template <typename T, int BM, int BN>
__device__ __forceinline__ void epilogue_rows_sqcos(const fused_params<T>& p, const T* zt, int ldt, int m0, int n0,
                                                    int warp, int lane, int nwarps, int rpw, int ch, int ntile) {
  using F = fop<T>;
  constexpr int CPL = (BN + 31) / 32;
  int cl[CPL];
  bool cv[CPL];
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) {
    const int c = lane + 32 * cc;
    cv[cc] = c < BN && n0 + c < p.D;
    cl[cc] = cv[cc] ? c : 0;
  }
  const uint32_t zs = static_cast<uint32_t>(__cvta_generic_to_shared(zt));
  for (int r0 = 0; r0 < rpw; r0 += 8) {
    T sa[8], sb[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) sa[q] = sb[q] = T(0);
    auto block = [&](auto exact_tag) {
      constexpr bool EXACT = decltype(exact_tag)::value;
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const int col = n0 + cl[cc];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = warp + (r0 + q) * nwarps;
          const bool ok = cv[cc] && r0 + q < rpw && r < BM;
          const T z = ptx::lds<T>(zs + uint32_t(((ok ? r : 0) * ldt + cl[cc]) * int(sizeof(T))));
          const T va = term_value<T, EXACT>(TERM_SQ, z, col, p.ell_w);
          const T vb = term_value<T, EXACT>(TERM_COS, z, col, p.ell_w);
          const T a1 = F::add(sa[q], va), b1 = F::add(sb[q], vb);
          sa[q] = ok ? a1 : sa[q];
          sb[q] = ok ? b1 : sb[q];
        }
      }
    };
    bool big = false;
    {
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = warp + (r0 + q) * nwarps;
          const bool ok = cv[cc] && r0 + q < rpw && r < BM;
          const T z = ptx::lds<T>(zs + uint32_t(((ok ? r : 0) * ldt + cl[cc]) * int(sizeof(T))));
          big = big || (ok && cos2pi_needs_exact(z));
        }
      big = __any_sync(0xffffffffu, big);
    }
    if (big) block(std::true_type{});
    else block(std::false_type{});
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      for (int off = 16; off > 0; off >>= 1) {
        sa[q] = F::add(sa[q], __shfl_xor_sync(0xffffffffu, sa[q], off));
        sb[q] = F::add(sb[q], __shfl_xor_sync(0xffffffffu, sb[q], off));
      }
      const int r = warp + (r0 + q) * nwarps;
      const int row = m0 + r;
      if (lane == 0 && r0 + q < rpw && r < BM && row < p.P) {
        p.partial[(size_t(ch) * p.n_ntiles + ntile) * p.P + row] = sa[q];
        p.partial[(size_t(ch + 1) * p.n_ntiles + ntile) * p.P + row] = sb[q];
      }
    }
  }
}

template <typename T, int BM, int BN>
__device__ void tile_epilogue(const fused_params<T>& p, const T* zt, int ldt, int m0, int n0, int tid, int nthreads,
                              int* last_flag, int mtile, int ntile, int bar_id) {
  using F = fop<T>;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthreads >> 5;
  if (p.zbuf) {
    // z-store: SoA z[i*ldz + b]; lanes over rows -> coalesced along b
    for (int c = warp; c < BN; c += nwarps) {
      const int col = n0 + c;
      if (col >= p.D) break;
      for (int r = lane; r < BM; r += 32) {
        const int row = m0 + r;
        if (row < p.P) p.zbuf[size_t(col) * p.ldz + row] = zt[r * ldt + c];
      }
    }
    return;
  }
  // Each warp owns rows warp, warp + nwarps, ...; per channel every lane evaluates all of its
  // (row, column) terms before any shuffle, so the transcendental chains of up to 4 x RPW elements
  // are independent (ILP) instead of one row at a time.
  const int rpw = (BM + nwarps - 1) / nwarps;
  for (int ch = 0; ch < p.n_ch; ++ch) {
    if (p.ch_term[ch] == TERM_SQ && ch + 1 < p.n_ch && p.ch_term[ch + 1] == TERM_COS) {  // Ackley's pair
      epilogue_rows_sqcos<T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile);
      ++ch;
      continue;
    }
    switch (p.ch_term[ch]) {  // one specialised loop nest per term (no per-element switch)
      case TERM_SQ: epilogue_rows<TERM_SQ, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
      case TERM_WSQ: epilogue_rows<TERM_WSQ, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
      case TERM_RAST: epilogue_rows<TERM_RAST, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
      case TERM_COS: epilogue_rows<TERM_COS, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
      case TERM_TAIL: epilogue_rows<TERM_TAIL, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
      case TERM_HEAD: epilogue_rows<TERM_HEAD, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
      default: epilogue_rows<TERM_GCOS, T, BM, BN>(p, zt, ldt, m0, n0, warp, lane, nwarps, rpw, ch, ntile); break;
    }
  }
  // ticket: the barrier orders every thread's partial stores before thread 0's gpu-scope fence
  // (cumulative release), and the last CTA's fence after the atomic is the acquire side
  ptx::named_bar_sync(bar_id, nthreads);
  if (tid == 0) {
    __threadfence();
    const unsigned ticket = atomicAdd(&p.counters[mtile], 1u);
    const int last = (ticket == unsigned(p.n_ntiles - 1)) ? 1 : 0;
    if (last) __threadfence();
    *last_flag = last;
  }
  ptx::named_bar_sync(bar_id, nthreads);
  if (p.dbg_ts && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg_ts[8 * (ntile * gridDim.x + mtile) + 3] = t;
  }
  if (!*last_flag) return;
  // N-tile partials combined in tile order per channel, eight L2 loads in flight per round (a
  // dependent load-add chain of n_ntiles L2 round trips sat on the kernel's critical path).
  // When the CTA has a thread per (row, channel), the channels' chains run in parallel and meet
  // in shared memory (the parked tile is dead by now) before the final formula.
  auto chain = [&](int ch, int row) {
    const bool prod = term_is_product(p.ch_term[ch]);
    const T* src = p.partial + size_t(ch) * p.n_ntiles * p.P + row;
    T v = __ldcg(src);
    for (int t0 = 1; t0 < p.n_ntiles; t0 += 8) {
      T x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (t0 + q < p.n_ntiles) x[q] = __ldcg(src + size_t(t0 + q) * p.P);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (t0 + q < p.n_ntiles) v = prod ? F::mul(v, x[q]) : F::add(v, x[q]);
    }
    return v;
  };
  auto final_row = [&](int row, const T* chv) {
    for (int o = 0; o < p.n_out; ++o) {
      const T s0 = chv[p.out_ch0[o]];
      const T s1 = p.out_ch1[o] >= 0 ? chv[p.out_ch1[o]] : T(0);
      p.out[o * p.ldo + row] = finalize<T>(p.out_kind[o], s0, s1, p.D, T(p.out_bias[o]));
    }
  };
  if (p.n_ch > 1 && p.n_ch * BM <= nthreads) {
    T* xs = const_cast<T*>(zt);  // [n_ch][BM]
    const int ch = tid / BM, r = tid % BM;
    if (ch < p.n_ch && m0 + r < p.P) xs[ch * BM + r] = chain(ch, m0 + r);
    ptx::named_bar_sync(bar_id, nthreads);
    for (int r2 = tid; r2 < BM; r2 += nthreads) {
      if (m0 + r2 >= p.P) continue;
      T chv[kMaxCh];
      for (int c = 0; c < p.n_ch; ++c) chv[c] = xs[c * BM + r2];
      final_row(m0 + r2, chv);
    }
  } else {
    for (int r = tid; r < BM; r += nthreads) {
      const int row = m0 + r;
      if (row >= p.P) continue;
      T chv[kMaxCh];
      for (int c = 0; c < p.n_ch; ++c) chv[c] = chain(c, row);
      final_row(row, chv);
    }
  }
  if (tid == 0) p.counters[mtile] = 0u;  // re-arm for the next launch
}

// byte offset of element (r, kk) inside a SWIZZLE_128B tile whose rows are 128 bytes
template <int ELEM>
__device__ __forceinline__ uint32_t swz(int r, int kk) {
  constexpr int per_chunk = 16 / ELEM;
  return uint32_t(r * 128 + ((((kk / per_chunk) ^ (r & 7))) << 4) + (kk % per_chunk) * ELEM);
}

// ---------------------------------------------------------------------------------------
// One 16-deep K-slice (one SWIZZLE_128B stage row) of a warp's (TM*8) x (TN*8) tile of
// z += (X - o) M^T: four m8n8k4 DMMA steps.  The k order inside the slice is permuted so that
// lane t's operands for steps 2p and 2p+1 sit in one 16-byte chunk (physical k = 4t + 2p + h,
// chunk 2t + p): each fragment is one LDS.128 instead of two LDS.64, and the 8 lanes of a
// quarter-warp phase (rows g, g+1; t = 0..3) hit 8 distinct chunks under the row XOR
// swizzle (conflict-free).  The shift is subtracted in fp64 as the fragment is formed
// (problems/batch.hpp:50).  Pair p+1's loads are issued before pair p's DMMAs.
template <int TM, int TN>
__device__ __forceinline__ void dmma_kslice(double (&acc)[TM][TN][2], uint32_t sA, uint32_t sB, uint32_t sO, int rA,
                                            int rB, int g, int t) {
  double2 a[2][TM], b[2][TN];
  auto load = [&](int pp, int buf) {
    const int ch = 2 * t + pp;
    const double2 o = ptx::lds_f64x2(sO + (4 * t + 2 * pp) * 8);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = rA + i * 8 + g;
      const double2 x = ptx::lds_f64x2(sA + r * 128 + ((ch ^ (r & 7)) << 4));
      a[buf][i] = make_double2(__dsub_rn(x.x, o.x), __dsub_rn(x.y, o.y));
    }
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = rB + j * 8 + g;
      b[buf][j] = ptx::lds_f64x2(sB + n * 128 + ((ch ^ (n & 7)) << 4));
    }
  };
  load(0, 0);
  load(1, 1);
#pragma unroll
  for (int pp = 0; pp < 2; ++pp)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
          ptx::dmma_8x8x4(acc[i][j][0], acc[i][j][1], h ? a[pp][i].y : a[pp][i].x, h ? b[pp][j].y : b[pp][j].x);
}

// The same slice for tall warp tiles (TM = 4: 112 accumulator registers): one operand pair at a
// time, A fragments of the pair held, B fragments streamed per 8-column block one block ahead, so
// only TM + 2 fragments are live beside the accumulators.
template <int TM, int TN>
__device__ __forceinline__ void dmma_kslice_stream(double (&acc)[TM][TN][2], uint32_t sA, uint32_t sB, uint32_t sO,
                                                   int rA, int rB, int g, int t) {
#pragma unroll
  for (int pp = 0; pp < 2; ++pp) {
    const int ch = 2 * t + pp;
    const uint32_t col = uint32_t((ch ^ g) << 4);  // rows rA + 8 i + g and rB + 8 j + g: (r & 7) == g
    const double2 o = ptx::lds_f64x2(sO + (4 * t + 2 * pp) * 8);
    double2 a[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const double2 x = ptx::lds_f64x2(sA + (rA + i * 8 + g) * 128 + col);
      a[i] = make_double2(__dsub_rn(x.x, o.x), __dsub_rn(x.y, o.y));
    }
    double2 b = ptx::lds_f64x2(sB + (rB + g) * 128 + col);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      double2 bn = b;
      if (j + 1 < TN) bn = ptx::lds_f64x2(sB + (rB + (j + 1) * 8 + g) * 128 + col);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < TM; ++i) ptx::dmma_8x8x4(acc[i][j][0], acc[i][j][1], h ? a[i].y : a[i].x, h ? b.y : b.x);
      b = bn;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K1: FP64 DMMA kernel
template <int BM, int BN, int WM, int WN, int STAGES>
struct f64_cfg {
  static constexpr int KB = 16;  // doubles per K-slice (one 128-byte swizzle row)
  static constexpr int NCW = WM * WN;
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int TM = WTM / 8, TN = WTN / 8;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int O_BYTES = 128;
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + O_BYTES + 1023) / 1024) * 1024;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 2 * STAGES * 8 + 64;
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(BM * (BN + 1) * 8 <= STAGES * STAGE_BYTES, "epilogue tile must fit the stage ring");
};

template <int BM, int BN, int WM, int WN, int STAGES, int MINB = 1>
__global__ void __launch_bounds__(f64_cfg<BM, BN, WM, WN, STAGES>::THREADS, MINB)
    eval_f64_dmma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                         const fused_params<double> p) {
  using C = f64_cfg<BM, BN, WM, WN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  int* last_flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KT = (p.D + C::KB - 1) / C::KB;
  unsigned long long* ts = p.dbg_ts ? p.dbg_ts + 8 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  auto stamp = [&](int i) {
    if (ts && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[i] = t;
    }
  };
  stamp(0);
  if (ts && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    ts[7] = sm;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], C::NCW);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // launched with PDL (launch_pdl): the prologue above overlaps the predecessor's tail; X, the
  // partials and the tickets are touched only after it completed
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();

  if (warp == C::NCW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      ptx::prefetch_tma(&tmX);
      ptx::prefetch_tma(&tmM);
      int chunk = 0, chunk_end = 0;  // columns [0, chunk_end) are resident
      for (int kb = 0; kb < KT; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) ptx::mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        if (p.kgate) {
          while (kb * C::KB >= chunk_end) {  // chunk ends are multiples of KB columns
            ptx::wait_gate(p.kgate + chunk, p.kgate_epoch);
            chunk_end = chunk + 1 < p.kgate_n ? p.kgate_end[chunk] : 1 << 30;
            ++chunk;
          }
        }
        uint8_t* st = smem + s * C::STAGE_BYTES;
        ptx::mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES + C::O_BYTES);
        ptx::tma_load_2d(st, &tmX, &full[s], kb * C::KB, m0);
        ptx::tma_load_2d(st + C::A_BYTES, &tmM, &full[s], kb * C::KB, n0);
        ptx::bulk_load(st + C::A_BYTES + C::B_BYTES, p.shift + size_t(kb) * C::KB, C::O_BYTES, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  const int rA = wm * C::WTM, rB = wn * C::WTN;
  double acc[C::TM][C::TN][2];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t smem_base = ptx::smem_u32(smem);
  for (int kb = 0; kb < KT; ++kb) {
    const int s = kb % STAGES;
    ptx::mbar_wait(&full[s], (kb / STAGES) & 1);
    if (kb == 0) stamp(1);
    const uint32_t sA = smem_base + s * C::STAGE_BYTES;
    const uint32_t sB = sA + C::A_BYTES;
    const uint32_t sO = sB + C::B_BYTES;
    dmma_kslice<C::TM, C::TN>(acc, sA, sB, sO, rA, rB, g, t);
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
  }

  // park the accumulator tile in the (drained) stage ring, then run the epilogue from smem
  // (measured: a register-direct epilogue — quad shuffles on the DMMA fragments, no parking —
  // was slower, 89 vs 81.6 us per batch: the inlined transcendental code bloats the kernel)
  stamp(2);
  ptx::named_bar_sync(1, C::NCW * 32);
  double* zt = reinterpret_cast<double*>(smem);
  constexpr int LDT = BN + 1;
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) zt[(rA + i * 8 + g) * LDT + rB + j * 8 + 2 * t + h] = acc[i][j][h];
  ptx::named_bar_sync(1, C::NCW * 32);
  tile_epilogue<double, BM, BN>(p, zt, LDT, m0, n0, threadIdx.x, C::NCW * 32, last_flag, blockIdx.x, blockIdx.y, 1);
  stamp(4);
  if (ts && threadIdx.x == 0) ts[5] = *last_flag;
}

// ---------------------------------------------------------------------------------------
// K1 (several problems, one population): NP problems sharing X (e.g. a suite's objectives at
// the same population, or config 1's three objectives).  One CTA per (row block, column block)
// holds NP warp groups — group g computes problem g's 64 x 56 tile with the pair kernel's 16 x 56
// warp tiles — and one producer whose stage carries ONE X tile plus the NP rotation tiles and
// shift slices, so X is read once for all problems.  12 MMA warps per SM at NP = 3 (3 per
// SMSP) hide more DMMA latency than two 4-warp CTAs; each group then runs the usual epilogue on
// its own parked tile, with its own partials / tickets.
constexpr int kMultiBM = 64, kMultiBN = 56, kMultiStages = 6;

// BM_ = 128 (one-wave variant): 32 x 56 warp tiles (112 accumulator registers per thread), a
// 5-stage ring; at config 1 its 8 x 18 = 144 CTAs are ONE wave on 148 SMs instead of 148 + 140.
template <int NP, int BM_ = kMultiBM>
struct f64m_cfg {
  static constexpr int BM = BM_, BN = kMultiBN, KB = 16, STAGES = BM_ == 64 ? kMultiStages : 5;
  static constexpr int WM = 4;  // MMA warps per group (16 x 56 or 32 x 56 warp tiles)
  static constexpr int NCW = NP * WM;
  // BM_ = 64: a separate TMA producer warp.  BM_ = 128: no 13th warp (a 4th warp on one SM
  // sub-partition would cap every thread at 128 registers; 12 warps may take 168) — lane 0 of
  // warp 0 refills the ring, LOOKAHEAD slices ahead of the slice it computes.
  static constexpr bool PRODUCER_WARP = BM_ == 64;
  static constexpr int LOOKAHEAD = STAGES - 2;
  static constexpr int THREADS = (NCW + (PRODUCER_WARP ? 1 : 0)) * 32;
  static constexpr int TM = BM / WM / 8, TN = 7;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int O_BYTES = 128;
  static constexpr int STAGE_BYTES = ((A_BYTES + NP * (B_BYTES + O_BYTES) + 1023) / 1024) * 1024;
  static constexpr int LDT = BN + 1;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 64;
  static_assert(NP * BM * LDT * 8 <= STAGES * STAGE_BYTES, "parked tiles must fit the stage ring");
};

template <int NP>
struct multi_maps {
  CUtensorMap m[NP];
};

template <int NP, int BM_ = kMultiBM>
__global__ void __launch_bounds__(f64m_cfg<NP, BM_>::THREADS, 1)
    eval_f64_dmma_multi_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ multi_maps<NP> tmM,
                               const __grid_constant__ fused_params<double> p0,
                               const __grid_constant__ fused_params<double> p1,
                               const __grid_constant__ fused_params<double> p2) {
  using C = f64m_cfg<NP, BM_>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  int* last_flag = reinterpret_cast<int*>(empty + C::STAGES);  // NP flags

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mtile = p0.tiles_nfast ? blockIdx.y : blockIdx.x, ntile = p0.tiles_nfast ? blockIdx.x : blockIdx.y;
  const int m0 = mtile * C::BM, n0 = ntile * C::BN;
  const int KT = (p0.D + C::KB - 1) / C::KB;
  // EVB_K1_TIMELINE=1 (tuning aid): CTA phase stamps (entry, first stage, mainloop end, exit)
  unsigned long long* ts = p0.dbg_ts ? p0.dbg_ts + 8 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  auto stamp = [&](int i) {
    if (ts && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[i] = t;
    }
  };
  stamp(0);
  if (ts && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    ts[7] = sm;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], C::NCW);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  // producer step: slice kb into its stage — X once, then each problem's rotation tile and shift slice
  int chunk = 0, chunk_end = 0;
  auto produce = [&](int kb) {
    const int s = kb % C::STAGES;
    if (kb >= C::STAGES) ptx::mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
    if (p0.kgate) {
      const int gbase = (p0.kgate_rows > 0 && m0 >= p0.kgate_rows) ? p0.kgate_n : 0;
      while (kb * C::KB >= chunk_end) {
        ptx::wait_gate(p0.kgate + gbase + chunk, p0.kgate_epoch);
        chunk_end = chunk + 1 < p0.kgate_n ? p0.kgate_end[chunk] : 1 << 30;
        ++chunk;
      }
    }
    uint8_t* st = smem + s * C::STAGE_BYTES;
    ptx::mbar_arrive_expect_tx(&full[s], C::A_BYTES + NP * (C::B_BYTES + C::O_BYTES));
    ptx::tma_load_2d(st, &tmX, &full[s], kb * C::KB, m0);
#pragma unroll
    for (int g = 0; g < NP; ++g) {
      const fused_params<double>& pg = g == 0 ? p0 : (g == 1 ? p1 : p2);
      ptx::tma_load_2d(st + C::A_BYTES + g * C::B_BYTES, &tmM.m[g], &full[s], kb * C::KB, n0);
      ptx::bulk_load(st + C::A_BYTES + NP * C::B_BYTES + g * C::O_BYTES, pg.shift + size_t(kb) * C::KB, C::O_BYTES,
                     &full[s]);
    }
  };
  if constexpr (C::PRODUCER_WARP) {
    if (warp == C::NCW) {
      if (lane == 0) {
        ptx::prefetch_tma(&tmX);
        for (int g = 0; g < NP; ++g) ptx::prefetch_tma(&tmM.m[g]);
        for (int kb = 0; kb < KT; ++kb) produce(kb);
      }
      return;
    }
  } else if (threadIdx.x == 0) {
    ptx::prefetch_tma(&tmX);
    for (int g = 0; g < NP; ++g) ptx::prefetch_tma(&tmM.m[g]);
    for (int kb = 0; kb < C::LOOKAHEAD && kb < KT; ++kb) produce(kb);
  }

  // ---------------- consumers: group g = warp / 4 computes problem g ----------------
  const int grp = warp / C::WM, wg = warp % C::WM;
  const int g8 = lane >> 2, t = lane & 3;
  const int rA = wg * (C::BM / C::WM);
  double acc[C::TM][C::TN][2];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const uint32_t smem_base = ptx::smem_u32(smem);
  for (int kb = 0; kb < KT; ++kb) {
    const int s = kb % C::STAGES;
    if constexpr (!C::PRODUCER_WARP) {  // refill the stage every warp left two slices ago
      if (threadIdx.x == 0 && kb + C::LOOKAHEAD < KT) produce(kb + C::LOOKAHEAD);
      __syncwarp();
    }
    ptx::mbar_wait(&full[s], (kb / C::STAGES) & 1);
    if (kb == 0) stamp(1);
    const uint32_t sA = smem_base + s * C::STAGE_BYTES;
    const uint32_t sB = sA + C::A_BYTES + grp * C::B_BYTES;
    const uint32_t sO = sA + C::A_BYTES + NP * C::B_BYTES + grp * C::O_BYTES;
    if constexpr (C::TM > 2) dmma_kslice_stream<C::TM, C::TN>(acc, sA, sB, sO, rA, 0, g8, t);
    else dmma_kslice<C::TM, C::TN>(acc, sA, sB, sO, rA, 0, g8, t);
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
  }

  // every group has drained the ring: park each group's tile in its own region, then per group
  // the fused epilogue (named barrier 2 + g over the group's 128 threads)
  stamp(2);
  ptx::named_bar_sync(1, C::NCW * 32);
  double* zt = reinterpret_cast<double*>(smem) + size_t(grp) * C::BM * C::LDT;
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) zt[(rA + i * 8 + g8) * C::LDT + j * 8 + 2 * t + h] = acc[i][j][h];
  ptx::named_bar_sync(2 + grp, C::WM * 32);
  const fused_params<double>& pg = grp == 0 ? p0 : (grp == 1 ? p1 : p2);
  tile_epilogue<double, C::BM, C::BN>(pg, zt, C::LDT, m0, n0, threadIdx.x - grp * C::WM * 32, C::WM * 32,
                                      last_flag + grp, mtile, ntile, 2 + grp);
  stamp(4);
}

// ---------------------------------------------------------------------------------------
// K1 (persistent): one CTA per SM walks a static list of BM x BN tiles.  Warp roles:
//   warps 0-7   MMA      (warp tile 8 x 56: 7 DMMA m8n8k4 per k4 step, 2 warps per SMSP)
//   warps 8-11  epilogue (transform terms + row sums of the previous tile, from smem)
//   warp  12    producer (TMA ring of 16-double K-slices, continuous across tiles)
// The accumulator tile is handed to the epilogue warps through one of two smem buffers
// (acc_full / acc_empty mbarriers), so a tile's epilogue overlaps the next tile's mainloop and
// only the CTA's last epilogue is exposed.  With 64 x 56 tiles, D = 1000 and P = 1024 give 288
// tiles = 2 per SM (140 SMs) — the same per-SM work as one 64 x 112 tile, minus the epilogue.
template <int BM, int BN, int STAGES, int NMW_ = 8>
struct f64p_cfg {
  static constexpr int KB = 16;
  static constexpr int NMW = NMW_;  // MMA warps, stacked along M (2 per SMSP by default)
  static constexpr int NEW = 4;  // epilogue warps
  static constexpr int THREADS = (NMW + NEW + 1) * 32;
  static constexpr int WTM = BM / NMW;
  static constexpr int TM = WTM / 8, TN = BN / 8;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int O_BYTES = 128;
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + O_BYTES + 1023) / 1024) * 1024;
  static constexpr int LDT = BN + 1;
  static constexpr int EBUF_BYTES = BM * LDT * 8;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * EBUF_BYTES + 1024 + (2 * STAGES + 4) * 8 + 64;
  static_assert(WTM % 8 == 0 && BN % 8 == 0, "tile must be a multiple of 8");
};

template <int BM, int BN, int STAGES>
__global__ void __launch_bounds__(f64p_cfg<BM, BN, STAGES>::THREADS, 1)
    eval_f64_dmma_persistent(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                             const fused_params<double> p, int n_mtiles, int n_tiles) {
  using C = f64p_cfg<BM, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  double* ebuf = reinterpret_cast<double*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES + 2 * C::EBUF_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  int* last_flag = reinterpret_cast<int*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (p.D + C::KB - 1) / C::KB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], C::NMW);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], C::NMW * 32);
      ptx::mbar_init(&acc_empty[b], C::NEW * 32);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::NMW + C::NEW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      ptx::prefetch_tma(&tmX);
      ptx::prefetch_tma(&tmM);
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int m0 = (tile % n_mtiles) * BM, n0 = (tile / n_mtiles) * BN;
        for (int kb = 0; kb < KT; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          ptx::mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES + C::O_BYTES);
          ptx::tma_load_2d(st, &tmX, &full[s], kb * C::KB, m0);
          ptx::tma_load_2d(st + C::A_BYTES, &tmM, &full[s], kb * C::KB, n0);
          ptx::bulk_load(st + C::A_BYTES + C::B_BYTES, p.shift + size_t(kb) * C::KB, C::O_BYTES, &full[s]);
        }
      }
    }
    return;
  }

  if (warp >= C::NMW) {
    // ---------------- epilogue warps ----------------
    const int etid = threadIdx.x - C::NMW * 32;
    int local = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++local) {
      const int b = local & 1;
      ptx::mbar_wait(&acc_full[b], (local >> 1) & 1);
      const int mt = tile % n_mtiles, nt = tile / n_mtiles;
      tile_epilogue<double, BM, BN>(p, ebuf + b * (BM * C::LDT), C::LDT, mt * BM, nt * BN, etid, C::NEW * 32,
                                    last_flag, mt, nt, 2);
      ptx::mbar_arrive(&acc_empty[b]);
    }
    return;
  }

  // ---------------- MMA warps ----------------
  const int g = lane >> 2, t = lane & 3;
  const int rA = warp * C::WTM;
  const uint32_t smem_base = ptx::smem_u32(smem);
  int it = 0, local = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++local) {
    double acc[C::TM][C::TN][2];
#pragma unroll
    for (int i = 0; i < C::TM; ++i)
#pragma unroll
      for (int j = 0; j < C::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kb = 0; kb < KT; ++kb, ++it) {
      const int s = it % STAGES;
      ptx::mbar_wait(&full[s], (it / STAGES) & 1);
      const uint32_t sA = smem_base + s * C::STAGE_BYTES;
      const uint32_t sB = sA + C::A_BYTES;
      const uint32_t sO = sB + C::B_BYTES;
      dmma_kslice<C::TM, C::TN>(acc, sA, sB, sO, rA, 0, g, t);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }
    // hand the tile to the epilogue warps
    const int b = local & 1;
    if (local >= 2) ptx::mbar_wait(&acc_empty[b], ((local >> 1) - 1) & 1);
    double* zt = ebuf + b * (BM * C::LDT);
#pragma unroll
    for (int i = 0; i < C::TM; ++i)
#pragma unroll
      for (int j = 0; j < C::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) zt[(rA + i * 8 + g) * C::LDT + j * 8 + 2 * t + h] = acc[i][j][h];
    ptx::mbar_arrive(&acc_full[b]);
  }
}

// ---------------------------------------------------------------------------------------
// K2 on tcgen05 (see umma.cuh): 3xTF32, 128 x BN tile per CTA, accumulator in TMEM.
// FUSE (BN = 64): the split pre-pass is folded in.  The X tile arrives by TMA in the stage's
// S_hi slot (same SWIZZLE_128B rows as S_hi / S_lo, so a 16-byte chunk keeps its position); the
// eight epilogue warps, idle during the mainloop, form S = X - o, S_hi, S_lo in place (S_hi over
// X, S_lo into its slot) and signal the MMA issuer.  L2 -> SM traffic per stage 48 -> 32 KB, no
// pre-pass launch.
template <int BN, bool FUSE = false>
struct umma_cfg {
  static constexpr int BM = 128;
  static constexpr int KB = 32;  // floats per K-slice (one 128-byte swizzle row)
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // hi + lo of both operands
  static constexpr int STAGES = (200 * 1024 / STAGE_BYTES) < 4 ? (200 * 1024 / STAGE_BYTES) : 4;
  static constexpr int THREADS = 10 * 32;  // producer, MMA issuer, 8 epilogue warps
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // [0,BN): main, [BN,2BN): corrections
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + (4 * STAGES + 1) * 8 + 64;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
};

template <int BN, bool FUSE>
__global__ void __launch_bounds__(umma_cfg<BN, FUSE>::THREADS, 1)
    eval_f32_umma_kernel(const __grid_constant__ CUtensorMap tmShi, const __grid_constant__ CUtensorMap tmSlo,
                         const __grid_constant__ CUtensorMap tmMhi, const __grid_constant__ CUtensorMap tmMlo,
                         const fused_params<float> p) {
  // FUSE: tmShi maps X itself (tmSlo unused)
  using C = umma_cfg<BN, FUSE>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* aready = empty + C::STAGES;  // FUSE: the stage's S_hi / S_lo are formed
  uint64_t* xfull = aready + C::STAGES;   // FUSE: the stage's X tile landed (M on `full`)
  uint64_t* accfull = xfull + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * C::BM, n0 = blockIdx.y * BN;
  const int KT = (p.D + C::KB - 1) / C::KB;
  unsigned long long* ts = p.dbg_ts ? p.dbg_ts + 8 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  auto stamp = [&](int i) {  // EVB_K1_TIMELINE=1 (tuning aid): phase stamps, one thread per phase
    if (ts) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[i] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&aready[s], 8);
      ptx::mbar_init(&xfull[s], 1);
    }
    ptx::mbar_init(accfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) umma::tmem_alloc(tmem_slot, C::TMEM_COLS);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  // launched with PDL behind the split pre-pass: barrier init and TMEM allocation above overlap
  // its tail; S_hi / S_lo (and the partials / tickets of earlier launches) only after it completed
  ptx::griddep_wait();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      ptx::prefetch_tma(&tmShi);
      ptx::prefetch_tma(&tmSlo);
      ptx::prefetch_tma(&tmMhi);
      ptx::prefetch_tma(&tmMlo);
      for (int kb = 0; kb < KT; ++kb) {
        const int s = kb % C::STAGES;
        if (kb >= C::STAGES) ptx::mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        if constexpr (FUSE) {  // X into the A_hi slot on its own barrier (the split starts as it
                               // lands), M_hi / M_lo as usual
          ptx::mbar_arrive_expect_tx(&xfull[s], C::A_BYTES);
          ptx::tma_load_2d(st, &tmShi, &xfull[s], kb * C::KB, m0);
          ptx::mbar_arrive_expect_tx(&full[s], 2 * C::B_BYTES);
        } else {
          ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          ptx::tma_load_2d(st, &tmShi, &full[s], kb * C::KB, m0);
          ptx::tma_load_2d(st + C::A_BYTES, &tmSlo, &full[s], kb * C::KB, m0);
        }
        ptx::tma_load_2d(st + 2 * C::A_BYTES, &tmMhi, &full[s], kb * C::KB, n0);
        ptx::tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &tmMlo, &full[s], kb * C::KB, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- single-thread MMA issuer ----------------
      constexpr uint32_t idesc = umma::idesc_tf32(C::BM, BN);
      const uint32_t base = ptx::smem_u32(smem);
      for (int kb = 0; kb < KT; ++kb) {
        const int s = kb % C::STAGES;
        ptx::mbar_wait(&full[s], (kb / C::STAGES) & 1);
        if constexpr (FUSE) ptx::mbar_wait(&aready[s], (kb / C::STAGES) & 1);
        if (kb == 0) stamp(1);
        umma::fence_after();
        const uint32_t sa_hi = base + s * C::STAGE_BYTES, sa_lo = sa_hi + C::A_BYTES;
        const uint32_t sb_hi = sa_hi + 2 * C::A_BYTES, sb_lo = sb_hi + C::B_BYTES;
        const uint32_t tcorr = tmem + BN;  // corrections accumulate apart from the main product
#pragma unroll
        for (int k = 0; k < C::KB / 8; ++k) {  // K = 8 tf32 = 32 bytes per instruction
          const uint32_t off = k * 32;
          const uint32_t acc0 = (kb | k) ? 1u : 0u;
          umma::mma_tf32(tcorr, umma::smem_desc(sa_lo + off), umma::smem_desc(sb_hi + off), idesc, acc0);
          umma::mma_tf32(tcorr, umma::smem_desc(sa_hi + off), umma::smem_desc(sb_lo + off), idesc, 1u);
          umma::mma_tf32(tmem, umma::smem_desc(sa_hi + off), umma::smem_desc(sb_hi + off), idesc,
                         acc0);
        }
        umma::commit(&empty[s]);  // frees the stage when these MMAs have read it
      }
      umma::commit(accfull);  // accumulator complete
    }
  } else {
    // ---------------- epilogue warps 2..9: (row, column half) per thread ----------------
    // warp w reads TMEM lane quarter w % 4; warps 2-5 take the tile's first BN/2 columns, 6-9 the
    // rest; main and correction accumulators are loaded together (one wait per 16 columns)
    constexpr int HC = BN / 2;
    const int ew = warp - 2, half = ew >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int row = m0 + r;
    const int etid = threadIdx.x - 64;  // 0..255
    if constexpr (FUSE) {
      // split of each X tile: S = X - o (fp32, reference rounding), S_hi = rna_tf32(S),
      // S_lo = rna_tf32(S - S_hi) — the pre-pass's arithmetic — in place in the stage; chunk q
      // of row q / 8 holds logical chunk (q & 7) ^ (row & 7) (columns >= D: X is zero-filled by
      // TMA and o zero-padded, so S = 0).  The generic-proxy writes are fenced to the async proxy
      // before the arrive.
      for (int kb = 0; kb < KT; ++kb) {
        const int s = kb % C::STAGES;
        ptx::mbar_wait(&xfull[s], (kb / C::STAGES) & 1);  // X landed
        uint8_t* st = smem + s * C::STAGE_BYTES;
        const float4* xs = reinterpret_cast<const float4*>(st);  // each thread rewrites its own chunks
        float4* hi = reinterpret_cast<float4*>(st);
        float4* lo = reinterpret_cast<float4*>(st + C::A_BYTES);
#pragma unroll
        for (int u = 0; u < C::A_BYTES / 16 / 256; ++u) {
          const int q = etid + u * 256;
          const int rr = q >> 3, c = (q & 7) ^ (rr & 7);
          const float4 x = xs[q];
          const float4 o = __ldg(reinterpret_cast<const float4*>(p.shift + size_t(kb) * C::KB + c * 4));
          auto split = [](float xv, float ov, float& hv, float& lv) {
            const float sv = __fsub_rn(xv, ov);
            hv = __uint_as_float(umma::rna_tf32_bits(sv));
            lv = __uint_as_float(umma::rna_tf32_bits(__fsub_rn(sv, hv)));
          };
          float4 h, l;
          split(x.x, o.x, h.x, l.x);
          split(x.y, o.y, h.y, l.y);
          split(x.z, o.z, h.z, l.z);
          split(x.w, o.w, h.w, l.w);
          hi[q] = h;
          lo[q] = l;
        }
        ptx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&aready[s]);
      }
    }
    ptx::mbar_wait_sleep(accfull, 0);
    if (threadIdx.x == 64) stamp(3);
    umma::fence_after();
    const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(half * HC);
    auto load16 = [&](int c0, float (&v)[16]) {
      uint32_t a[16], b[16];
      umma::tmem_ld16_raw(taddr + c0, a);
      umma::tmem_ld16_raw(taddr + BN + c0, b);
      umma::tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = __fadd_rn(__uint_as_float(a[q]), __uint_as_float(b[q]));
    };
    if (p.zbuf) {
#pragma unroll 1
      for (int c0 = 0; c0 < HC; c0 += 16) {
        float v[16];
        load16(c0, v);
        const int cb = n0 + half * HC + c0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (row < p.P && cb + q < p.D) p.zbuf[size_t(cb + q) * p.ldz + row] = v[q];
      }
    } else {
      // per channel: the thread's half-row sum, then the halves meet in shared memory (the stage
      // ring is drained once accfull fired): xs[half][ch][row]
      float* xs = reinterpret_cast<float*>(smem);
      for (int ch = 0; ch < p.n_ch; ++ch) {
        const int term = p.ch_term[ch];
        float a = term_is_product(term) ? 1.f : 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < HC; c0 += 16) {
          float v[16];
          load16(c0, v);
          a = accumulate16_rt<float>(term, a, v, n0 + half * HC + c0, p.D, p.ell_w);
        }
        xs[(half * kMaxCh + ch) * C::BM + r] = a;
      }
      ptx::named_bar_sync(1, 256);
      if (half == 0 && row < p.P)
        for (int ch = 0; ch < p.n_ch; ++ch) {
          const float a0 = xs[ch * C::BM + r], a1 = xs[(kMaxCh + ch) * C::BM + r];
          const float v = term_is_product(p.ch_term[ch]) ? __fmul_rn(a0, a1) : __fadd_rn(a0, a1);
          p.partial[(size_t(ch) * p.n_ntiles + blockIdx.y) * p.P + row] = v;
        }
      if (threadIdx.x == 64) stamp(4);
      // ticket and combine as in tile_epilogue: one thread's fences around the atomic; N-tile
      // partials summed in tile order, eight L2 loads in flight per round, channels in parallel
      ptx::named_bar_sync(1, 256);
      if (etid == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(&p.counters[blockIdx.x], 1u);
        const int last = (ticket == unsigned(p.n_ntiles - 1)) ? 1 : 0;
        if (last) __threadfence();
        *last_flag = last;
      }
      ptx::named_bar_sync(1, 256);
      if (*last_flag) {
        auto chain = [&](int ch, int rw) {
          const bool prod = term_is_product(p.ch_term[ch]);
          const float* src = p.partial + size_t(ch) * p.n_ntiles * p.P + rw;
          float v = __ldcg(src);
          for (int t0 = 1; t0 < p.n_ntiles; t0 += 8) {
            float x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (t0 + q < p.n_ntiles) x[q] = __ldcg(src + size_t(t0 + q) * p.P);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (t0 + q < p.n_ntiles) v = prod ? __fmul_rn(v, x[q]) : __fadd_rn(v, x[q]);
          }
          return v;
        };
        const bool par = p.n_ch > 1 && p.n_ch * C::BM <= 256;
        if (par) {
          const int ch = etid / C::BM, rr = etid % C::BM;
          if (ch < p.n_ch && m0 + rr < p.P) xs[ch * C::BM + rr] = chain(ch, m0 + rr);
          ptx::named_bar_sync(1, 256);
        }
        if (etid < C::BM && m0 + etid < p.P) {
          float chv[kMaxCh];
          for (int ch = 0; ch < p.n_ch; ++ch) chv[ch] = par ? xs[ch * C::BM + etid] : chain(ch, m0 + etid);
          for (int o = 0; o < p.n_out; ++o) {
            const float s0 = chv[p.out_ch0[o]];
            const float s1 = p.out_ch1[o] >= 0 ? chv[p.out_ch1[o]] : 0.f;
            p.out[o * p.ldo + m0 + etid] = finalize<float>(p.out_kind[o], s0, s1, p.D, float(p.out_bias[o]));
          }
        }
        if (etid == 0) p.counters[blockIdx.x] = 0u;
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (threadIdx.x == 64) {
    stamp(5);
    if (ts) ts[6] = *last_flag;
  }
  if (warp == 1) umma::tmem_dealloc(tmem, C::TMEM_COLS);
}

// 3xFP16 range guard, the rare path (kept out of line: the kernel's common path stays compact):
// rows of row block m0 whose flag is set are recomputed by the 256 epilogue threads — z in fp32
// with the reference's separate mul and add in k order (problems/batch.hpp:40-82), the channel
// terms per 16-column chunk, the chunks combined in order, the usual final formula — and their
// flags re-armed.  `scratch` holds a row of s, a row of z and the chunk partials.
template <int BM>
__device__ __noinline__ void f16_fixup_rows(const fused_params<float>& p, uint8_t* scratch, int m0, int etid) {

  const int D = p.D, nchunk = (D + 15) / 16;
  float* sS = reinterpret_cast<float*>(scratch);
  float* sZ = sS + ((D + 3) & ~3);
  float* sP = sZ + ((D + 3) & ~3);  // [n_ch][nchunk]
  for (int rr2 = 0; rr2 < BM && m0 + rr2 < p.P; ++rr2) {
    const int rw = m0 + rr2;
    if (!__ldcg(p.row_bad + rw)) continue;  // the same word for every thread
    for (int k = etid; k < D; k += 256) sS[k] = __fsub_rn(p.Xrows[size_t(rw) * p.ldxr + k], p.shift[k]);
    ptx::named_bar_sync(1, 256);
    for (int j = etid; j < D; j += 256) {
      const float* mr = p.rot + size_t(j) * p.ldm;
      float acc = 0.f;
      for (int k = 0; k < D; ++k) acc = __fadd_rn(acc, __fmul_rn(mr[k], sS[k]));
      sZ[j] = acc;
    }
    ptx::named_bar_sync(1, 256);
    for (int e = etid; e < p.n_ch * nchunk; e += 256) {
      const int ch = e / nchunk, c = e - ch * nchunk;
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 16 * c + q < D ? sZ[16 * c + q] : 0.f;
      const int term = p.ch_term[ch];
      sP[e] = accumulate16_rt<float>(term, term_is_product(term) ? 1.f : 0.f, v, 16 * c, D, p.ell_w);
    }
    ptx::named_bar_sync(1, 256);
    if (etid == 0) {
      float chv[kMaxCh];
      for (int ch = 0; ch < p.n_ch; ++ch) {
        const bool prod = term_is_product(p.ch_term[ch]);
        float v = sP[ch * nchunk];
        for (int c = 1; c < nchunk; ++c) v = prod ? __fmul_rn(v, sP[ch * nchunk + c]) : __fadd_rn(v, sP[ch * nchunk + c]);
        chv[ch] = v;
      }
      for (int o = 0; o < p.n_out; ++o) {
        const float s0 = chv[p.out_ch0[o]];
        const float s1 = p.out_ch1[o] >= 0 ? chv[p.out_ch1[o]] : 0.f;
        p.out[o * p.ldo + rw] = finalize<float>(p.out_kind[o], s0, s1, D, float(p.out_bias[o]));
      }
      p.row_bad[rw] = 0;  // re-arm for the next launch
    }
    ptx::named_bar_sync(1, 256);
  }
}

// ---------------------------------------------------------------------------------------
// K2 on tcgen05, split-K (the default fp32 tensor-core path).  128 x BN output tile per CTA with
// BN = 128 (N = 128 MMAs run at the tensor core's full rate; N = 64 reached ~60% of it), and the
// K range split over gridDim.z CTAs so that the config-1 grid (8 x 8 tiles x 2 halves = 128 CTAs)
// fills the SMs.  Per 32-float K slice: TMA brings X (128 rows, into the S_hi slot, own barrier)
// and M_hi / M_lo (BN rows); the 8 epilogue warps split X into S_hi / S_lo in place (as the
// FUSE kernel above) while the single MMA thread issues 4 K-steps x 3 products.  After the
// mainloop each CTA holds z_k = main + corrections of its K half in TMEM.  The two K halves of a
// tile form a 2-CTA cluster and split the epilogue by columns: each CTA sends its z_k of the
// peer's 64 columns into the peer's receive buffer (DSMEM), one cluster barrier, then adds the
// received half to its own (z = z_0 + z_1: fp add is commutative, the same in both CTAs) and runs
// the usual epilogue on its 64 columns (terms, per-row channel sums, column-block partials,
// last-CTA finalisation).  Deterministic, no float atomics.
// F16 (the default, "3xFP16"): the same split with fp16 heads and remainders (11 significant bits
// each, like TF32; the rotation scaled by 2^8 so its remainders stay normal) and kind::f16 MMAs,
// K = 16 per instruction at the tf32 instruction's cost: half the MMA time and half the rotation
// bytes.  A K slice is then 64 elements: X lands as two 32-float boxes (32 KB, the whole A stage);
// thread (row, box) forms its row's [S_hi k 0..31 | S_lo k 0..31] in place (it only overwrites what
// it has read), so box b serves K steps 2b, 2b + 1 with hi at byte offsets 0 / 32 and lo at 64 / 96
// of the 128-byte swizzle row.
template <int BN, bool ATMEM, bool F16 = false>
struct umma_sk_cfg {
  static_assert(!(ATMEM && F16), "the fp16 split keeps its operands in shared memory");
  static constexpr int BM = 128;
  static constexpr int KB = F16 ? 64 : 32;        // elements per K slice
  static constexpr int X_BYTES = BM * KB * 4;     // one X slice (TMA; F16: two 32-float boxes)
  static constexpr int B_BYTES = 2 * BN * 128;    // M_hi + M_lo of one slice (TMA, multicast pair)
  // ATMEM: S_hi / S_lo go to TMEM (the MMA's A operand from TMEM: shared memory then feeds only B,
  //        which a 128 x 128 x 8 tf32 MMA otherwise reads at the full 128 B/clk with A);
  //        X ring NX x 16 KB, A ring NA x (32 + 32) TMEM columns, B ring NB x 32 KB
  // else:  S_hi over X and S_lo in shared memory: A ring NA x 32 KB
  static constexpr int NX = ATMEM ? 4 : 0;
  static constexpr int NA = 4;
  static constexpr int NB = ATMEM ? 4 : (BN == 128 ? 3 : 2);
  static constexpr int A_BYTES = ATMEM ? 0 : 2 * BM * 128;
  static constexpr int X_OFF = 0;
  static constexpr int A_OFF = NX * X_BYTES;
  static constexpr int B_OFF = A_OFF + NA * A_BYTES;
  static constexpr int O_OFF = B_OFF + NB * B_BYTES;
  static constexpr int NSLOT = ATMEM ? NX : NA;  // stages carrying an X slice + its shift values
  static constexpr int RING_BYTES = O_OFF + NSLOT * KB * 4;
  static constexpr int NBAR = NSLOT + 2 * NA + 2 * NB + NX + 3;
  // K halves exchange z by point-to-point mbarriers instead of two cluster-wide barriers: the
  // receive buffer is exactly A stage 0, which its owner's MMAs leave several slices before its
  // mainloop ends (P2P; the TMEM-operand variant keeps the cluster barriers)
  static constexpr bool P2P = !ATMEM;
  static constexpr int THREADS = 11 * 32;  // X producer, MMA, 8 split / epilogue warps, B producer
  static constexpr int TMEM_COLS = ATMEM ? 512 : 2 * BN;
  static constexpr uint32_t TA = 2 * BN;  // first A column (ATMEM)
  static constexpr int RECV_BYTES = BM * (BN / 2) * 4;  // the peer's z_k of the owned columns
  static constexpr int SMEM = RING_BYTES + 1024 + NBAR * 8 + 64;
  static_assert(!ATMEM || TA + NA * 2 * KB <= 512, "TMEM columns");
  static_assert(RECV_BYTES + 8192 <= (ATMEM ? NX * X_BYTES + NB * B_BYTES : NA * A_BYTES),
                "receive buffer + epilogue scratch in the drained rings");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <int BN, bool ATMEM, bool F16 = false>
__global__ void __launch_bounds__(umma_sk_cfg<BN, ATMEM, F16>::THREADS, 1)
    eval_f32_umma_sk_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmMhi,
                            const __grid_constant__ CUtensorMap tmMlo, const __grid_constant__ fused_params<float> p) {
  using C = umma_sk_cfg<BN, ATMEM, F16>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* xfull = reinterpret_cast<uint64_t*>(smem + C::RING_BYTES);  // X + shift slice landed
  uint64_t* afull = xfull + C::NSLOT;                                   // S_hi / S_lo formed
  uint64_t* aempty = afull + C::NA;                                     // the MMAs read the A stage
  uint64_t* bfull = aempty + C::NA;
  uint64_t* bempty = bfull + C::NB;
  uint64_t* xempty = bempty + C::NB;  // ATMEM: the split warps read the X slot
  uint64_t* accfull = xempty + C::NX;
  uint64_t* peer_free = accfull + 1;  // the K peer's MMAs have left its A stage 0 (= its receive buffer)
  uint64_t* recv_full = accfull + 2;  // the K peer's 256 epilogue threads delivered their z halves
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 3);
  int* flags = reinterpret_cast<int*>(tmem_slot + 1);  // [1]: last column block of the row block

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * C::BM, n0 = blockIdx.y * BN;
  const int KT_all = (p.D + C::KB - 1) / C::KB;
  const int nsk = gridDim.z, kz = blockIdx.z;
  // cluster (2 along M) x (gridDim.z along K): rank = mx + 2 kz.  The M pair shares every B slice
  // (each CTA loads half of its rows and multicasts it to both); the K pair exchanges z halves.
  const unsigned crank = ptx::cluster_ctarank();
  const unsigned mx = crank & 1u;
  const uint16_t pair_mask = uint16_t(3u << (crank & ~1u));
  const int kb0 = int((int64_t(KT_all) * kz) / nsk), kb1 = int((int64_t(KT_all) * (kz + 1)) / nsk);
  const int KT = kb1 - kb0;
  unsigned long long* ts =
      p.dbg_ts ? p.dbg_ts + 8 * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) : nullptr;
  auto stamp = [&](int i) {  // EVB_K1_TIMELINE=1 (tuning aid)
    if (ts) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[i] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NSLOT; ++s) ptx::mbar_init(&xfull[s], 1);
    for (int s = 0; s < C::NX; ++s) ptx::mbar_init(&xempty[s], 8);
    for (int s = 0; s < C::NA; ++s) {
      ptx::mbar_init(&afull[s], 8);
      ptx::mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      ptx::mbar_init(&bfull[s], 1);
      ptx::mbar_init(&bempty[s], 2);  // both CTAs of the M pair consumed the slot
    }
    ptx::mbar_init(accfull, 1);
    ptx::mbar_init(peer_free, 1);
    ptx::mbar_init(recv_full, 256);
    ptx::fence_mbar_init();
  }
  if (warp == 1) umma::tmem_alloc(tmem_slot, C::TMEM_COLS);
  umma::fence_before();
  ptx::cluster_sync_all();  // every CTA's barriers exist before the first multicast / remote commit
  umma::fence_after();
  const uint32_t tmem = *tmem_slot;
  // B producer: with PDL the first B slices (the problem's immutable rotation split) may load
  // while the predecessor still runs; everything else waits for it
  const int b_pre = p.b_early ? min(KT, C::NB) : 0;
  if (warp == 10 && lane == 0) {
    ptx::prefetch_tma(&tmMhi);
    ptx::prefetch_tma(&tmMlo);
    for (int kb = 0; kb < b_pre; ++kb) {
      uint8_t* st = smem + C::B_OFF + kb * C::B_BYTES + mx * (BN / 2) * 128;
      ptx::mbar_arrive_expect_tx(&bfull[kb], C::B_BYTES);
      ptx::tma_load_2d_mc(st, &tmMhi, &bfull[kb], (kb0 + kb) * C::KB, n0 + int(mx) * (BN / 2), pair_mask);
      ptx::tma_load_2d_mc(st + C::B_BYTES / 2, &tmMlo, &bfull[kb], (kb0 + kb) * C::KB, n0 + int(mx) * (BN / 2),
                          pair_mask);
    }
  }
  ptx::griddep_wait();  // PDL: barrier init and TMEM allocation overlap the predecessor's tail
  ptx::griddep_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- X producer: X slice + its 32 shift values ----------------
      ptx::prefetch_tma(&tmX);
      for (int kb = 0; kb < KT; ++kb) {
        const int s = kb % C::NSLOT;
        if (kb >= C::NSLOT) {
          if constexpr (ATMEM) ptx::mbar_wait(&xempty[s], ((kb / C::NSLOT) - 1) & 1);
          else ptx::mbar_wait(&aempty[s], ((kb / C::NSLOT) - 1) & 1);
        }
        uint8_t* dst = ATMEM ? smem + C::X_OFF + s * C::X_BYTES : smem + C::A_OFF + s * C::A_BYTES;
        ptx::mbar_arrive_expect_tx(&xfull[s], C::X_BYTES + C::KB * 4);
        ptx::tma_load_2d(dst, &tmX, &xfull[s], (kb0 + kb) * C::KB, m0);
        if constexpr (F16) ptx::tma_load_2d(dst + C::BM * 128, &tmX, &xfull[s], (kb0 + kb) * C::KB + 32, m0);
        ptx::bulk_load(smem + C::O_OFF + s * C::KB * 4, p.shift + size_t(kb0 + kb) * C::KB, C::KB * 4, &xfull[s]);
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- B producer (M_hi, M_lo) ----------------
      for (int kb = b_pre; kb < KT; ++kb) {
        const int s = kb % C::NB;
        if (kb >= C::NB) ptx::mbar_wait(&bempty[s], ((kb / C::NB) - 1) & 1);
        uint8_t* st = smem + C::B_OFF + s * C::B_BYTES + mx * (BN / 2) * 128;  // this CTA's half of the rows
        ptx::mbar_arrive_expect_tx(&bfull[s], C::B_BYTES);  // both halves land here
        ptx::tma_load_2d_mc(st, &tmMhi, &bfull[s], (kb0 + kb) * C::KB, n0 + int(mx) * (BN / 2), pair_mask);
        ptx::tma_load_2d_mc(st + C::B_BYTES / 2, &tmMlo, &bfull[s], (kb0 + kb) * C::KB, n0 + int(mx) * (BN / 2),
                            pair_mask);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- single-thread MMA issuer ----------------
      constexpr uint32_t idesc = umma::idesc_tf32(C::BM, BN);
      const uint32_t base = ptx::smem_u32(smem);
      const uint32_t tcorr = tmem + BN;
      for (int kb = 0; kb < KT; ++kb) {
        const int sa = kb % C::NA, sb = kb % C::NB;
        ptx::mbar_wait(&afull[sa], (kb / C::NA) & 1);
        ptx::mbar_wait(&bfull[sb], (kb / C::NB) & 1);
        if (kb == 0) stamp(1);
        umma::fence_after();
        const uint32_t sb_hi = base + C::B_OFF + sb * C::B_BYTES, sb_lo = sb_hi + C::B_BYTES / 2;
        if constexpr (ATMEM) {
          const uint32_t ta_hi = tmem + C::TA + uint32_t(sa) * 2 * C::KB, ta_lo = ta_hi + C::KB;
#pragma unroll
          for (int k = 0; k < C::KB / 8; ++k) {
            if (p.dbg_skip & 2) break;
            const uint32_t off = k * 32, col = k * 8;
            const uint32_t acc0 = (kb | k) ? 1u : 0u;
            umma::mma_tf32_ts(tmem, ta_hi + col, umma::smem_desc(sb_hi + off), idesc, acc0);
            umma::mma_tf32_ts(tcorr, ta_lo + col, umma::smem_desc(sb_hi + off), idesc, acc0);
            umma::mma_tf32_ts(tcorr, ta_hi + col, umma::smem_desc(sb_lo + off), idesc, 1u);
          }
        } else if constexpr (F16) {
          constexpr uint32_t idesc16 = umma::idesc_f16(C::BM, BN);
          const uint32_t sa0 = base + C::A_OFF + sa * C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::KB / 16; ++k) {
            if (p.dbg_skip & 2) break;
            const uint32_t a_hi = sa0 + (k >> 1) * (C::BM * 128) + (k & 1) * 32, a_lo = a_hi + 64;
            const uint32_t off = k * 32;
            const uint32_t acc0 = (kb | k) ? 1u : 0u;
            umma::mma_f16(tmem, umma::smem_desc(a_hi), umma::smem_desc(sb_hi + off), idesc16, acc0);
            umma::mma_f16(tcorr, umma::smem_desc(a_lo), umma::smem_desc(sb_hi + off), idesc16, acc0);
            umma::mma_f16(tcorr, umma::smem_desc(a_hi), umma::smem_desc(sb_lo + off), idesc16, 1u);
          }
        } else {
          const uint32_t sa_hi = base + C::A_OFF + sa * C::A_BYTES, sa_lo = sa_hi + C::A_BYTES / 2;
#pragma unroll
          for (int k = 0; k < C::KB / 8; ++k) {
            if (p.dbg_skip & 2) break;
            const uint32_t off = k * 32;
            const uint32_t acc0 = (kb | k) ? 1u : 0u;
            umma::mma_tf32(tmem, umma::smem_desc(sa_hi + off), umma::smem_desc(sb_hi + off), idesc, acc0);
            umma::mma_tf32(tcorr, umma::smem_desc(sa_lo + off), umma::smem_desc(sb_hi + off), idesc, acc0);
            umma::mma_tf32(tcorr, umma::smem_desc(sa_hi + off), umma::smem_desc(sb_lo + off), idesc, 1u);
          }
        }
        umma::commit(&aempty[sa]);
        umma::commit_mc(&bempty[sb], pair_mask);  // the slot is freed in both CTAs of the M pair
        // A stage 0 is read for the last time by slice kb: tell the K peer it may deliver
        if (C::P2P && nsk > 1 && sa == 0 && kb + C::NA >= KT) umma::commit_mc(peer_free, uint16_t(1u << (crank ^ 2u)));
      }
      umma::commit(accfull);
    }
  } else {
    // ---------------- split / epilogue warps 2..9 ----------------
    const int ew = warp - 2, half = ew >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int row = m0 + r;
    const int etid = threadIdx.x - 64;
    auto split = [](float xq, float oq, uint32_t& hq, uint32_t& lq) {
      const float sq = __fsub_rn(xq, oq);
      hq = umma::rna_tf32_bits(sq);
      lq = umma::rna_tf32_bits(__fsub_rn(sq, __uint_as_float(hq)));
    };
    if constexpr (ATMEM) {
      // thread = row r (its TMEM lane), columns [16 half, 16 half + 16) of each slice: S from the
      // swizzled X slot (logical chunk c of row r at physical chunk c ^ (r & 7)) into registers,
      // the X slot released, S_hi / S_lo to the stage's TMEM columns
      const uint32_t tlane = tmem + (uint32_t(quarter * 32) << 16);
      for (int kb = 0; kb < KT; ++kb) {
        const int sx = kb % C::NX, sa = kb % C::NA;
        ptx::mbar_wait(&xfull[sx], (kb / C::NX) & 1);
        const float4* xs = reinterpret_cast<const float4*>(smem + C::X_OFF + sx * C::X_BYTES) + r * 8;
        const float4* osl = reinterpret_cast<const float4*>(smem + C::O_OFF + sx * C::KB * 4);
        float4 xv[4], ov[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = 4 * half + u;
          xv[u] = xs[c ^ (r & 7)];
          ov[u] = osl[c];
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&xempty[sx]);  // the X slot is free once read
        uint32_t hv[16], lv[16];
        if (!(p.dbg_skip & 1)) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            split(xv[u].x, ov[u].x, hv[4 * u + 0], lv[4 * u + 0]);
            split(xv[u].y, ov[u].y, hv[4 * u + 1], lv[4 * u + 1]);
            split(xv[u].z, ov[u].z, hv[4 * u + 2], lv[4 * u + 2]);
            split(xv[u].w, ov[u].w, hv[4 * u + 3], lv[4 * u + 3]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) hv[q] = lv[q] = 0u;
        }
        if (kb >= C::NA) ptx::mbar_wait(&aempty[sa], ((kb / C::NA) - 1) & 1);  // the MMAs read this A stage
        umma::fence_after();
        const uint32_t ta = tlane + C::TA + uint32_t(sa) * 2 * C::KB + uint32_t(16 * half);
        umma::tmem_st16(ta, hv);
        umma::tmem_st16(ta + C::KB, lv);
        umma::tmem_wait_st();
        umma::fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&afull[sa]);
      }
    } else if constexpr (F16) {
      // thread = (row rr, box b): the row's 32 floats of the box (logical 16-byte chunk f at physical
      // f ^ (rr & 7): the 8 rows of a quarter warp hit 8 distinct chunks) into registers, then
      // [S_hi | S_lo] as 4 + 4 chunks of 8 halves back into the same 128 bytes
      const int b = etid >> 7, rr = etid & 127;
      for (int kb = 0; kb < KT; ++kb) {
        const int sa = kb % C::NA;
        ptx::mbar_wait(&xfull[sa], (kb / C::NA) & 1);
        uint4* rowp = reinterpret_cast<uint4*>(smem + C::A_OFF + sa * C::A_BYTES + b * (C::BM * 128) + rr * 128);
        const float4* osl = reinterpret_cast<const float4*>(smem + C::O_OFF + sa * C::KB * 4) + 8 * b;
        if (!(p.dbg_skip & 1)) {
          float4 xv[8];
#pragma unroll
          for (int f = 0; f < 8; ++f) xv[f] = *reinterpret_cast<const float4*>(rowp + (f ^ (rr & 7)));
          uint32_t hw[16], lw[16];  // 2 halves per word
#pragma unroll
          for (int f = 0; f < 8; ++f) {
            const float4 o = osl[f];
            const float s0 = __fsub_rn(xv[f].x, o.x), s1 = __fsub_rn(xv[f].y, o.y);
            const float s2 = __fsub_rn(xv[f].z, o.z), s3 = __fsub_rn(xv[f].w, o.w);
            const __half2 h01 = __floats2half2_rn(s0, s1), h23 = __floats2half2_rn(s2, s3);
            const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
            const __half2 l01 = __floats2half2_rn(__fsub_rn(s0, f01.x), __fsub_rn(s1, f01.y));
            const __half2 l23 = __floats2half2_rn(__fsub_rn(s2, f23.x), __fsub_rn(s3, f23.y));
            hw[2 * f] = *reinterpret_cast<const uint32_t*>(&h01);
            hw[2 * f + 1] = *reinterpret_cast<const uint32_t*>(&h23);

            lw[2 * f] = *reinterpret_cast<const uint32_t*>(&l01);
            lw[2 * f + 1] = *reinterpret_cast<const uint32_t*>(&l23);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            rowp[j ^ (rr & 7)] = make_uint4(hw[4 * j], hw[4 * j + 1], hw[4 * j + 2], hw[4 * j + 3]);
            rowp[(4 + j) ^ (rr & 7)] = make_uint4(lw[4 * j], lw[4 * j + 1], lw[4 * j + 2], lw[4 * j + 3]);
          }
          ptx::fence_proxy_async();
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&afull[sa]);
      }
    } else {
      // S = X - o, S_hi = rna_tf32(S) over X, S_lo = rna_tf32(S - S_hi) into the stage's lo half
      // (same SWIZZLE_128B positions: chunk q of row q / 8 holds logical chunk (q & 7) ^ (row & 7))
      for (int kb = 0; kb < KT; ++kb) {
        const int sa = kb % C::NA;
        ptx::mbar_wait(&xfull[sa], (kb / C::NA) & 1);
        float4* hi = reinterpret_cast<float4*>(smem + C::A_OFF + sa * C::A_BYTES);
        float4* lo = reinterpret_cast<float4*>(smem + C::A_OFF + sa * C::A_BYTES + C::A_BYTES / 2);
        const float4* osl = reinterpret_cast<const float4*>(smem + C::O_OFF + sa * C::KB * 4);
        if (!(p.dbg_skip & 1)) {
#pragma unroll
          for (int u = 0; u < C::X_BYTES / 16 / 256; ++u) {
            const int q = etid + u * 256;
            const int rr = q >> 3, c = (q & 7) ^ (rr & 7);
            const float4 x = hi[q];
            const float4 o = osl[c];
            uint32_t h[4], l[4];
            split(x.x, o.x, h[0], l[0]);
            split(x.y, o.y, h[1], l[1]);
            split(x.z, o.z, h[2], l[2]);
            split(x.w, o.w, h[3], l[3]);
            hi[q] = make_float4(__uint_as_float(h[0]), __uint_as_float(h[1]), __uint_as_float(h[2]), __uint_as_float(h[3]));
            lo[q] = make_float4(__uint_as_float(l[0]), __uint_as_float(l[1]), __uint_as_float(l[2]), __uint_as_float(l[3]));
          }
          ptx::fence_proxy_async();
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&afull[sa]);
      }
    }
    ptx::mbar_wait_sleep(accfull, 0);
    if (etid == 0) stamp(3);
    umma::fence_after();
    // Column ownership: with the K range split over a 2-CTA cluster (blockIdx.z = cluster rank),
    // CTA kz finalises columns [kz * BN/2, (kz + 1) * BN/2) of the tile.  Each epilogue thread
    // (TMEM lane quarter = 32 rows, column half h) sends its z_k of the other CTA's columns into
    // the peer's receive buffer (DSMEM, 16-byte chunks XOR-swizzled by row), one cluster barrier,
    // then adds the peer's z_k to its own for the columns it owns (z = z_0 + z_1).
    const int OWN = BN / nsk;           // columns this CTA finalises
    const int TW = OWN / 2;             // per thread (two threads per row)
    const int own0 = kz * OWN;          // first owned column of the tile
    const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16);
    auto load16 = [&](int col, float (&v)[16]) {  // this CTA's z_k, tile columns [col, col + 16)
      uint32_t a[16], b[16];
      umma::tmem_ld16_raw(tbase + col, a);
      umma::tmem_ld16_raw(tbase + BN + col, b);
      umma::tmem_wait_ld();
      // (F16: the rotation was scaled by 2^8 for the split; the power of two comes off exactly)
      constexpr float zs = F16 ? 1.f / kF16Scale : 1.f;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float zq = __fadd_rn(__uint_as_float(a[q]), __uint_as_float(b[q]));
        v[q] = F16 ? __fmul_rn(zq, zs) : zq;
      }
    };
    float* recv = reinterpret_cast<float*>(smem);  // [BM][BN/2] in the drained rings (nsk == 2)
    auto rchunk = [&](int rr, int ch16) { return rr * (BN / 2) + 4 * ((ch16 & ~7) | ((ch16 & 7) ^ (rr & 7))); };
    if (nsk > 1) {
      if constexpr (C::P2P) ptx::mbar_wait_cluster(peer_free, 0);  // the peer's stage 0 is free
      else ptx::cluster_sync_all();  // both CTAs past their mainloops: the peer's rings are drained
      const int snd0 = (1 - kz) * OWN + half * TW;  // tile columns sent to the peer
      const uint32_t peer = ptx::mapa(ptx::smem_u32(recv), crank ^ 2u);  // the other K half
#pragma unroll 1
      for (int c0 = 0; c0 < TW; c0 += 16) {
        float v[16];
        load16(snd0 + c0, v);
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          const int ch16 = (half * TW + c0 + q) >> 2;  // 16-byte chunk in the peer's [BN/2] row
          ptx::st_cluster_v4(peer + 4u * uint32_t(rchunk(r, ch16)), v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
      }
    }
    if (nsk > 1) {
      if constexpr (C::P2P) {
        // every sender releases its stores on the peer's barrier; then wait for the peer's 256
        ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(recv_full), crank ^ 2u));
        ptx::mbar_wait_cluster(recv_full, 0);
      } else {
        ptx::cluster_sync_all();  // every thread of both CTAs (warps 0-1 join below)
      }
    }
    if (etid == 0) stamp(2);  // the K halves exchanged
    auto loadz = [&](int c0, float (&v)[16]) {  // z of owned columns [own0 + half*TW + c0, +16)
      load16(own0 + half * TW + c0, v);
      if (nsk > 1) {
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          const float4 w = *reinterpret_cast<const float4*>(recv + rchunk(r, (half * TW + c0 + q) >> 2));
          v[q] = __fadd_rn(v[q], w.x);
          v[q + 1] = __fadd_rn(v[q + 1], w.y);
          v[q + 2] = __fadd_rn(v[q + 2], w.z);
          v[q + 3] = __fadd_rn(v[q + 3], w.w);
        }
      }
    };
    if (p.zbuf) {
#pragma unroll 1
      for (int c0 = 0; c0 < TW; c0 += 16) {
        float v[16];
        loadz(c0, v);
        const int cb = n0 + own0 + half * TW + c0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (row < p.P && cb + q < p.D) p.zbuf[size_t(cb + q) * p.ldz + row] = v[q];
      }
    } else {
      float* xs = reinterpret_cast<float*>(smem + C::RECV_BYTES);  // drained rings: [half][ch][row]
      // two-channel kinds (Ackley, Griewank, bent cigar): both channels in one pass over z (one
      // TMEM / receive-buffer read per chunk instead of one per channel)
      const bool pair = p.n_ch == 2;
      if (pair) {
        const int t0 = p.ch_term[0], t1 = p.ch_term[1];
        float a0 = term_is_product(t0) ? 1.f : 0.f, a1 = term_is_product(t1) ? 1.f : 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < TW; c0 += 16) {
          float v[16];
          loadz(c0, v);
          const int col0 = n0 + own0 + half * TW + c0;
          if (t0 == TERM_SQ && t1 == TERM_COS) {  // Ackley: no per-chunk switch (CTA-uniform branch)
            a0 = accumulate16<TERM_SQ>(a0, v, col0, p.D, p.ell_w);
            a1 = accumulate16<TERM_COS>(a1, v, col0, p.D, p.ell_w);
          } else {
            a0 = accumulate16_rt<float>(t0, a0, v, col0, p.D, p.ell_w);
            a1 = accumulate16_rt<float>(t1, a1, v, col0, p.D, p.ell_w);
          }
        }
        xs[(half * kMaxCh + 0) * C::BM + r] = a0;
        xs[(half * kMaxCh + 1) * C::BM + r] = a1;
      }
      for (int ch = 0; ch < (pair ? 0 : p.n_ch); ++ch) {
        const int term = p.ch_term[ch];
        float acc = term_is_product(term) ? 1.f : 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < TW; c0 += 16) {
          float v[16];
          loadz(c0, v);
          acc = accumulate16_rt<float>(term, acc, v, n0 + own0 + half * TW + c0, p.D, p.ell_w);
        }
        xs[(half * kMaxCh + ch) * C::BM + r] = acc;
      }
      if (etid == 0) flags[2] = 0;  // a flagged row in this CTA (3xFP16 range guard)
      ptx::named_bar_sync(1, 256);
      const int pt = blockIdx.y * nsk + kz;  // partial slot of this CTA's column block
      if (half == 0 && row < p.P) {
        // 3xFP16 range guard: a coordinate whose fp16 head is inf / NaN (|x - o| >= 65520, or not
        // finite) makes every z of its row non-finite, hence a non-finite channel sum here; such rows
        // (and rows whose sums overflow anyway) are flagged for the last CTA's fp32 recomputation
        bool nonfinite = false;
        for (int ch = 0; ch < p.n_ch; ++ch) {
          const float a0 = xs[ch * C::BM + r], a1 = xs[(kMaxCh + ch) * C::BM + r];
          const float v = term_is_product(p.ch_term[ch]) ? __fmul_rn(a0, a1) : __fadd_rn(a0, a1);
          p.partial[(size_t(ch) * p.n_ntiles + pt) * p.P + row] = v;
          nonfinite = nonfinite || !(fabsf(v) <= 3.4e38f);
        }
        if (F16 && nonfinite) {  // before the ticket's barrier and fence
          p.row_bad[row] = 1;
          flags[2] = 1;
        }
      }
      ptx::named_bar_sync(1, 256);
      if (etid == 0) {
        stamp(4);
        __threadfence();
        // the ticket's high half counts the CTAs that flagged a row, so the last CTA of the row
        // block learns "any flagged row" from the value the atomic returns (no extra round trip)
        const unsigned ticket = atomicAdd(&p.counters[blockIdx.x], 1u + (unsigned(flags[2]) << 16));
        const int last = ((ticket & 0xFFFFu) == unsigned(p.n_ntiles - 1)) ? 1 : 0;
        if (last) __threadfence();
        flags[1] = last;
        if (ticket >> 16) flags[2] = 1;
      }
      ptx::named_bar_sync(1, 256);
      if (flags[1]) {
        auto chain = [&](int ch, int rw) {  // column blocks in order, sixteen loads per L2 round
          const bool prod = term_is_product(p.ch_term[ch]);
          const float* src = p.partial + size_t(ch) * p.n_ntiles * p.P + rw;
          float v = prod ? 1.f : 0.f;
          for (int t0 = 0; t0 < p.n_ntiles; t0 += 16) {
            float x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (t0 + q < p.n_ntiles) x[q] = __ldcg(src + size_t(t0 + q) * p.P);
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (t0 + q < p.n_ntiles) v = (t0 + q == 0) ? x[q] : (prod ? __fmul_rn(v, x[q]) : __fadd_rn(v, x[q]));
          }
          return v;
        };
        const bool par = p.n_ch > 1 && p.n_ch * C::BM <= 256;
        // one channel: two threads per row each sum half of the column-block partials (in order),
        // one L2 round of loads instead of two; the halves add in fixed order
        const bool split2 = p.n_ch == 1 && p.n_ntiles >= 4;
        if (split2) {
          const int h2 = etid / C::BM, rr = etid % C::BM, rw = m0 + rr;
          const int nh = (p.n_ntiles + 1) / 2, t_lo = h2 * nh, t_hi = min(p.n_ntiles, t_lo + nh);
          if (rw < p.P) {
            const bool prod = term_is_product(p.ch_term[0]);
            const float* src = p.partial + rw;
            float x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (t_lo + q < t_hi) x[q] = __ldcg(src + size_t(t_lo + q) * p.P);
            float v = x[0];
#pragma unroll
            for (int q = 1; q < 16; ++q)
              if (t_lo + q < t_hi) v = prod ? __fmul_rn(v, x[q]) : __fadd_rn(v, x[q]);
            for (int t = t_lo + 16; t < t_hi; ++t) {  // more than 32 column blocks
              const float y = __ldcg(src + size_t(t) * p.P);
              v = prod ? __fmul_rn(v, y) : __fadd_rn(v, y);
            }
            xs[h2 * C::BM + rr] = v;
          }
          ptx::named_bar_sync(1, 256);
        }
        if (par) {
          const int ch = etid / C::BM, rr = etid % C::BM;
          if (ch < p.n_ch && m0 + rr < p.P) xs[ch * C::BM + rr] = chain(ch, m0 + rr);
          ptx::named_bar_sync(1, 256);
        }
        if (etid < C::BM && m0 + etid < p.P) {
          float chv[kMaxCh];
          if (split2) {
            const float a0 = xs[etid], a1 = xs[C::BM + etid];
            chv[0] = term_is_product(p.ch_term[0]) ? __fmul_rn(a0, a1) : __fadd_rn(a0, a1);
          } else {
            for (int ch = 0; ch < p.n_ch; ++ch) chv[ch] = par ? xs[ch * C::BM + etid] : chain(ch, m0 + etid);
          }
          for (int o = 0; o < p.n_out; ++o) {
            const float s0 = chv[p.out_ch0[o]];
            const float s1 = p.out_ch1[o] >= 0 ? chv[p.out_ch1[o]] : 0.f;
            p.out[o * p.ldo + m0 + etid] = finalize<float>(p.out_kind[o], s0, s1, p.D, float(p.out_bias[o]));
          }
        }
        if (etid == 0) p.counters[blockIdx.x] = 0u;
        if constexpr (F16) {
          // rows the split warps flagged (any CTA of the row block, either K half): z in fp32 with
          // the reference's separate mul and add in k order (problems/batch.hpp:40-82), the
          // channel terms per 16-column chunk, chunks combined in order, the usual final formula
          if (flags[2]) f16_fixup_rows<C::BM>(p, smem + C::RECV_BYTES + 8192, m0, etid);  // (published with flags[1])
        }
      }
    }
  }
  if (!C::P2P && (warp < 2 || warp == 10) && nsk > 1) {  // the producer / MMA warps join both exchange barriers
    ptx::cluster_sync_all();
    ptx::cluster_sync_all();
  }
  // no CTA leaves while its M partner may still multicast into it or commit to its barriers
  ptx::cluster_sync_all();
  umma::fence_before();
  __syncthreads();
  if (threadIdx.x == 64) {
    stamp(5);
    if (ts) {
      ts[6] = flags[1];
      ts[7] = 1;
    }
  }
  if (warp == 1) umma::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ---------------------------------------------------------------------------------------
// K2: FP32 FFMA kernel.  Each consumer thread owns an 8x8 register tile; rows and columns
// are interleaved with stride 8 (rows ty + 8*i, cols tx + 8*j) so the float4 fragment loads
// of a warp hit 8 distinct 16-byte swizzle chunks (conflict free).
template <int BM, int BN, int STAGES>
struct f32_cfg {
  static constexpr int KB = 32;  // floats per K-slice (128-byte swizzle row)
  static constexpr int TY = BM / 8, TX = BN / 8;
  static constexpr int NCT = TY * TX;  // consumer threads
  static constexpr int NCW = NCT / 32;
  static constexpr int WN = 1;  // row sums reduced across all threads of a row via smem
  static constexpr int THREADS = NCT + 32;
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int O_BYTES = 128;
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + O_BYTES + 1023) / 1024) * 1024;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 64;
  static_assert(NCT % 32 == 0, "consumer threads must be whole warps");
  static_assert(BM * (BN + 1) * 4 <= STAGES * STAGE_BYTES, "epilogue tile must fit the stage ring");
};

template <int BM, int BN, int STAGES>
__global__ void __launch_bounds__(f32_cfg<BM, BN, STAGES>::THREADS, 1)
    eval_f32_ffma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                         const fused_params<float> p) {
  using C = f32_cfg<BM, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  int* last_flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KT = (p.D + C::KB - 1) / C::KB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], C::NCW);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::NCW) {
    if (lane == 0) {
      ptx::prefetch_tma(&tmX);
      ptx::prefetch_tma(&tmM);
      for (int kb = 0; kb < KT; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) ptx::mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        ptx::mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES + C::O_BYTES);
        ptx::tma_load_2d(st, &tmX, &full[s], kb * C::KB, m0);
        ptx::tma_load_2d(st + C::A_BYTES, &tmM, &full[s], kb * C::KB, n0);
        ptx::bulk_load(st + C::A_BYTES + C::B_BYTES, p.shift + size_t(kb) * C::KB, C::O_BYTES, &full[s]);
      }
    }
    return;
  }

  const int tid = threadIdx.x;
  const int ty = tid / C::TX, tx = tid % C::TX;  // rows ty + TY*i? no: rows ty*1 + TY*i
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const uint32_t smem_base = ptx::smem_u32(smem);
  for (int kb = 0; kb < KT; ++kb) {
    const int s = kb % STAGES;
    ptx::mbar_wait(&full[s], (kb / STAGES) & 1);
    const uint32_t sA = smem_base + s * C::STAGE_BYTES;
    const uint32_t sB = sA + C::A_BYTES;
    const uint32_t sO = sB + C::B_BYTES;
#pragma unroll 2
    for (int kc = 0; kc < C::KB / 4; ++kc) {
      const float4 o = ptx::lds_f32x4(sO + kc * 16);
      float4 a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 x = ptx::lds_f32x4(sA + swz<4>(ty + C::TY * i, kc * 4));
        a[i] = make_float4(__fsub_rn(x.x, o.x), __fsub_rn(x.y, o.y), __fsub_rn(x.z, o.z), __fsub_rn(x.w, o.w));
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = ptx::lds_f32x4(sB + swz<4>(tx + C::TX * j, kc * 4));
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j] = fmaf(a[i].x, b[j].x, acc[i][j]);
          acc[i][j] = fmaf(a[i].y, b[j].y, acc[i][j]);
          acc[i][j] = fmaf(a[i].z, b[j].z, acc[i][j]);
          acc[i][j] = fmaf(a[i].w, b[j].w, acc[i][j]);
        }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
  }

  ptx::named_bar_sync(1, C::NCT);
  float* zt = reinterpret_cast<float*>(smem);
  constexpr int LDT = BN + 1;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) zt[(ty + C::TY * i) * LDT + tx + C::TX * j] = acc[i][j];
  ptx::named_bar_sync(1, C::NCT);
  tile_epilogue<float, BM, BN>(p, zt, LDT, m0, n0, tid, C::NCT, last_flag, blockIdx.x, blockIdx.y, 1);
}

// ---------------------------------------------------------------------------------------
// host side

namespace {

struct kind_channels {
  int n;
  int term[2];
};
kind_channels channels_for(int kind) {
  switch (kind) {
    case EVB_SPHERE: return {1, {TERM_SQ, -1}};
    case EVB_ELLIPTIC: return {1, {TERM_WSQ, -1}};
    case EVB_BENT_CIGAR:
    case EVB_DISCUS: return {2, {TERM_TAIL, TERM_HEAD}};
    case EVB_RASTRIGIN: return {1, {TERM_RAST, -1}};
    case EVB_ACKLEY: return {2, {TERM_SQ, TERM_COS}};
    case EVB_GRIEWANK: return {2, {TERM_SQ, TERM_GCOS}};
  }
  return {0, {-1, -1}};
}

template <typename T>
bool build_plan(fused_params<T>& fp, int n_out, const int* kinds, const double* biases) {
  fp.n_ch = 0;
  fp.n_out = n_out;
  for (int o = 0; o < n_out; ++o) {
    const kind_channels kc = channels_for(kinds[o]);
    if (kc.n == 0) return false;
    int idx[2] = {-1, -1};
    for (int c = 0; c < kc.n; ++c) {
      int found = -1;
      for (int q = 0; q < fp.n_ch; ++q)
        if (fp.ch_term[q] == kc.term[c]) found = q;
      if (found < 0) {
        if (fp.n_ch == kMaxCh) return false;
        found = fp.n_ch;
        fp.ch_term[fp.n_ch++] = kc.term[c];
      }
      idx[c] = found;
    }
    fp.out_kind[o] = kinds[o];
    fp.out_bias[o] = biases[o];
    fp.out_ch0[o] = idx[0];
    fp.out_ch1[o] = idx[1];
  }
  return true;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    EVB_CUDA(cudaGetDevice(&dev));
    EVB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// Tile configurations, chosen per problem shape to minimise wave quantisation on the SMs.
// fp64: (BM, BN, WM, WN); warp tile (BM/WM) x (BN/WN).
constexpr int kStages64 = 6;
constexpr int kStages32 = 4;

template <int BM, int BN, int WM, int WN, int STAGES = kStages64, int MINB = 1>
void launch_f64(const CUtensorMap& tmX, const CUtensorMap& tmM, const fused_params<double>& fp, cudaStream_t st) {
  using C = f64_cfg<BM, BN, WM, WN, STAGES>;
  auto kern = eval_f64_dmma_kernel<BM, BN, WM, WN, STAGES, MINB>;
  static bool attr = false;
  if (!attr) {
    EVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  dim3 grid((fp.P + BM - 1) / BM, (fp.D + BN - 1) / BN);
  EVB_CUDA(launch_pdl(kern, grid, dim3(C::THREADS), C::SMEM, st, tmX, tmM, fp));
  EVB_CUDA(cudaGetLastError());
  count_launch();
}

template <int BM, int BN>
void launch_f64_persistent(const CUtensorMap& tmX, const CUtensorMap& tmM, const fused_params<double>& fp,
                           cudaStream_t st) {
  constexpr int STAGES = 8;
  using C = f64p_cfg<BM, BN, STAGES>;
  auto kern = eval_f64_dmma_persistent<BM, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    EVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int n_mtiles = (fp.P + BM - 1) / BM;
  const int n_tiles = n_mtiles * ((fp.D + BN - 1) / BN);
  const int grid = std::min(n_tiles, sm_count());
  kern<<<grid, C::THREADS, C::SMEM, st>>>(tmX, tmM, fp, n_mtiles, n_tiles);
  EVB_CUDA(cudaGetLastError());
  count_launch();
}

template <int BN, bool FUSE = false>
void launch_f32_umma(const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& b_hi, const CUtensorMap& b_lo,
                     const fused_params<float>& fp, cudaStream_t st) {
  using C = umma_cfg<BN, FUSE>;
  auto kern = eval_f32_umma_kernel<BN, FUSE>;
  static bool attr = false;
  if (!attr) {
    EVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  dim3 grid((fp.P + C::BM - 1) / C::BM, (fp.D + BN - 1) / BN);
  EVB_CUDA(launch_pdl(kern, grid, dim3(C::THREADS), C::SMEM, st, a_hi, a_lo, b_hi, b_lo, fp));
  EVB_CUDA(cudaGetLastError());
  count_launch();
}

template <int BN, bool ATMEM, bool F16 = false>
void launch_f32_umma_sk(const CUtensorMap& tx, const CUtensorMap& b_hi, const CUtensorMap& b_lo,
                        const fused_params<float>& fp, int splitk, cudaStream_t st) {
  using C = umma_sk_cfg<BN, ATMEM, F16>;
  auto kern = eval_f32_umma_sk_kernel<BN, ATMEM, F16>;
  static bool attr = false;
  if (!attr) {
    EVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int mt = (fp.P + C::BM - 1) / C::BM;
  dim3 grid((mt + 1) & ~1, (fp.D + BN - 1) / BN, splitk);  // M pairs (a padding tile computes zeros)
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(C::THREADS);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;  // M pairs x the K halves of a tile
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = unsigned(splitk);
  lc.attrs = at;
  lc.numAttrs = 2;
  EVB_CUDA(cudaLaunchKernelEx(&lc, kern, tx, b_hi, b_lo, fp));
  EVB_CUDA(cudaGetLastError());
  count_launch();
}

template <int BM, int BN>
void launch_f32(const CUtensorMap& tmX, const CUtensorMap& tmM, const fused_params<float>& fp, cudaStream_t st) {
  using C = f32_cfg<BM, BN, kStages32>;
  auto kern = eval_f32_ffma_kernel<BM, BN, kStages32>;
  static bool attr = false;
  if (!attr) {
    EVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  dim3 grid((fp.P + BM - 1) / BM, (fp.D + BN - 1) / BN);
  kern<<<grid, C::THREADS, C::SMEM, st>>>(tmX, tmM, fp);
  EVB_CUDA(cudaGetLastError());
  count_launch();
}



}  // namespace

// Fused (or z-store) GEMM evaluation of a base problem on device-resident X.
template <typename T>
void gemm_eval(const eval_request& rq, const void* X, int64_t ldx, bool zstore, T* zbuf, int64_t ldz,
               const T* shift, const void* rotation, int ldm, int P, int D) {
  fused_params<T> fp{};
  fp.P = P;
  fp.D = D;
  fp.ell_w = static_cast<const T*>(rq.prob->ell_w);
  fp.shift = shift;
  fp.out = static_cast<T*>(rq.out);
  fp.ldo = rq.ldo;
  bool gate_consumed = false;
  if (zstore) {
    fp.zbuf = zbuf;
    fp.ldz = ldz;
  } else if (!build_plan<T>(fp, rq.n_out, rq.kinds, rq.biases)) {
    throw logic_error("gemm_eval: kind set has no fused epilogue");
  }
  evb_scratch_s* sc = rq.scratch;
  constexpr int dtype = std::is_same<T, double>::value ? EVB_F64 : EVB_F32;
  constexpr int KB = std::is_same<T, double>::value ? 16 : 32;

  int BM, BN;
  bool use_persistent = false;
  // EVB_F64_KERNEL=persistent|pair|classic overrides the shape choice (A/B measurements)
  static const char* force = std::getenv("EVB_F64_KERNEL");
  if constexpr (std::is_same<T, double>::value) use_persistent = force && std::string(force) == "persistent";
  if constexpr (std::is_same<T, double>::value) {
    // pick the tile with the least wave-quantised cost; {64, 56} runs 2 CTAs per SM so one CTA's
    // epilogue overlaps the other's DMMA mainloop (preferred on ties)
    const int cands[4][2] = {{64, 56}, {64, 112}, {64, 128}, {32, 128}};
    const int per_sm[4] = {2, 1, 1, 1};
    int best = 0;
    double bc = 1e300;
    for (int c = 0; c < 4; ++c) {
      const int64_t ctas = ((P + cands[c][0] - 1) / cands[c][0]) * ((D + cands[c][1] - 1) / cands[c][1]);
      const int64_t waves = (ctas + int64_t(sm_count()) * per_sm[c] - 1) / (int64_t(sm_count()) * per_sm[c]);
      double v = double(waves) * per_sm[c] * cands[c][0] * cands[c][1];
      if (cands[c][0] == 32) v *= 1.08;
      if (per_sm[c] == 2) v *= 0.97;  // overlap bonus
      if (v < bc) {
        bc = v;
        best = c;
      }
    }
    if (force && std::string(force) == "classic" && best == 0) best = 1;
    if (force && std::string(force) == "pair") best = 0;
    BM = cands[best][0];
    BN = cands[best][1];

    if (use_persistent) {
      BM = 64;
      BN = 56;
    }
  } else {
    BM = 64;
    BN = 128;
  }
  // fp32 tensor-core path (3xFP16 / 3xTF32, main product and corrections in separate TMEM accumulators):
  // measured fitness error <= 1e-5 relative for every base kind except discus, whose value is
  // dominated by 1e6 * z0^2 and amplifies the tensor-core accumulation error to ~1e-4; discus,
  // hybrids (chunks may be discus) and compositions stay on the FFMA kernel.
  static const char* force32 = std::getenv("EVB_F32_KERNEL");
  bool umma32 = !std::is_same<T, double>::value && rq.prob->spec == SPEC_BASE;
  for (int o = 0; o < rq.n_out && umma32; ++o) umma32 = rq.kinds[o] != EVB_DISCUS;
  if (force32) umma32 = std::string(force32) == "umma" && !std::is_same<T, double>::value;
  if constexpr (!std::is_same<T, double>::value) {
    if (umma32) {
      // ---- fp32 on tcgen05: three-product split, 128 x UBN tiles ----
      static const char* ubn_env = std::getenv("EVB_UMMA_BN");
      // default: the split-K kernel with 128 x 128 tiles (EVB_UMMA_BN=64 / 128 / 256 selects the
      // single-K-range kernels)
      const int UBN = ubn_env ? std::atoi(ubn_env) : 0;
      device_problem* pr = const_cast<device_problem*>(rq.prob);
      const bool own_rot = rotation == pr->rotation;  // composition components pass their own rotation
      const int64_t mel = int64_t(D) * ldm;
      void* rhi = nullptr;
      void* rlo = nullptr;
      // EVB_F32_MMA=tf32 keeps the 3xTF32 MMAs; the default is the fp16 split (3xFP16, kind::f16)
      static const bool f16 = !(std::getenv("EVB_F32_MMA") && std::string(std::getenv("EVB_F32_MMA")) == "tf32");
      static const bool atmem_env = std::getenv("EVB_UMMA_ATMEM") && std::atoi(std::getenv("EVB_UMMA_ATMEM")) == 1;
      static thread_local bool force_tf32 = false;  // set for the re-dispatch after a failed range check
      // (z-store launches and very long rows keep 3xTF32: the range guard's fp32 fix-up lives in the
      // fused epilogue and stages a row of s and z in the drained rings)
      const bool use16 = f16 && !atmem_env && UBN == 0 && !force_tf32 && !(own_rot && pr->f16_unsafe) && !zstore &&
                         D <= 8192;
      const bool split_cached = own_rot && (use16 ? pr->rot_hi16 != nullptr : pr->rot_hi != nullptr);
      fp.b_early = split_cached ? 1 : 0;
      if (use16) {
        // (the fp16 split is built below)
      } else if (split_cached) {
        rhi = pr->rot_hi;
        rlo = pr->rot_lo;
      } else {
        EVB_CUDA(cudaMalloc(&rhi, mel * sizeof(float)));
        EVB_CUDA(cudaMalloc(&rlo, mel * sizeof(float)));
        split_plain_kernel<<<int(std::min<int64_t>(2048, (mel + 255) / 256)), 256, 0, rq.stream>>>(
            static_cast<const float*>(rotation), mel, static_cast<float*>(rhi), static_cast<float*>(rlo));
        count_launch();
        if (own_rot) {
          pr->rot_hi = rhi;
          pr->rot_lo = rlo;
        }
      }
      // UBN = 64 (the default): the split folded into the kernel (EVB_F32_FUSE=0 keeps the
      // pre-pass, A/B); other widths (EVB_UMMA_BN, tuning) keep the pre-pass
      static const char* fuse_env = std::getenv("EVB_F32_FUSE");
      const bool fuse = UBN == 64 && !(fuse_env && std::string(fuse_env) == "0");
      CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
      bool ok = true;
      if (UBN == 0) {
        constexpr int SBN = 128;
        const int n_mtiles = ((P + 127) / 128 + 1) & ~1, n_nt = (D + SBN - 1) / SBN;  // M pairs
        const int n_tiles = n_mtiles * n_nt;
        // K halves when the tiles alone leave SMs idle and each half keeps >= 8 K slices
        static const char* sk_env = std::getenv("EVB_UMMA_SPLITK");
        int splitk = (n_tiles * 2 <= sm_count() && (D + 31) / 32 >= 16) ? 2 : 1;
        if (sk_env) splitk = std::max(1, std::min(2, std::atoi(sk_env)));
        void* r16h = nullptr;
        void* r16l = nullptr;
        if (use16) {
          // flagged-row buffer (zero between launches: the last CTA of a row block re-arms it)
          if (sc->row_bad_n < size_t(P)) {
            size_t cap = sc->row_bad_n * sizeof(int);
            void* ptr = sc->row_bad;
            ensure_buffer(&ptr, &cap, size_t(P) * sizeof(int), rq.stream);
            sc->row_bad = static_cast<int*>(ptr);
            sc->row_bad_n = cap / sizeof(int);
            EVB_CUDA(cudaMemsetAsync(sc->row_bad, 0, cap, rq.stream));
          }
          fp.row_bad = sc->row_bad;
          fp.Xrows = static_cast<const float*>(X);
          fp.ldxr = ldx;
          fp.rot = static_cast<const float*>(rotation);
          fp.ldm = ldm;
          if (own_rot && pr->rot_hi16) {
            r16h = pr->rot_hi16;
            r16l = pr->rot_lo16;
          } else {
            EVB_CUDA(cudaMalloc(&r16h, mel * sizeof(__half)));
            EVB_CUDA(cudaMalloc(&r16l, mel * sizeof(__half)));
            // (one synchronous range check per problem: a rotation whose 2^8-scaled entries leave
            // fp16's range keeps the 3xTF32 kernel)
            EVB_CUDA(cudaMemsetAsync(sc->row_bad, 0, sizeof(int), rq.stream));
            split_f16_kernel<<<int(std::min<int64_t>(2048, (mel + 255) / 256)), 256, 0, rq.stream>>>(
                static_cast<const float*>(rotation), mel, static_cast<__half*>(r16h), static_cast<__half*>(r16l),
                sc->row_bad);
            count_launch();
            int oor = 0;
            EVB_CUDA(cudaMemcpyAsync(&oor, sc->row_bad, sizeof(int), cudaMemcpyDeviceToHost, rq.stream));
            EVB_CUDA(cudaStreamSynchronize(rq.stream));
            if (oor) {
              EVB_CUDA(cudaMemsetAsync(sc->row_bad, 0, sizeof(int), rq.stream));
              cudaFree(r16h);
              cudaFree(r16l);
              r16h = r16l = nullptr;
              if (own_rot) pr->f16_unsafe = true;
              force_tf32 = true;  // this call again, on the 3xTF32 kernel
              try {
                gemm_eval<T>(rq, X, ldx, zstore, zbuf, ldz, shift, rotation, ldm, P, D);
              } catch (...) {
                force_tf32 = false;
                throw;
              }
              force_tf32 = false;
              return;
            } else if (own_rot) {
              pr->rot_hi16 = r16h;
              pr->rot_lo16 = r16l;
            }
          }
        }
        ok = make_tma_2d(&ta_hi, X, EVB_F32, uint64_t(D), uint64_t(P), uint64_t(ldx) * 4, 32, 128);
        if (use16)
          ok = ok && make_tma_2d(&tb_hi, r16h, kTmaF16, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * 2, 64, SBN / 2) &&
               make_tma_2d(&tb_lo, r16l, kTmaF16, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * 2, 64, SBN / 2);
        else
          ok = ok && make_tma_2d(&tb_hi, rhi, EVB_F32, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * 4, 32, SBN / 2) &&
               make_tma_2d(&tb_lo, rlo, EVB_F32, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * 4, 32, SBN / 2);
        if (!ok) throw runtime_error("gemm_eval: cannot encode the TMA descriptors of the tensor-core split");
        fp.n_ntiles = n_nt * splitk;  // column blocks of BN / splitk, one partial each
        if (!zstore) {
          ensure_buffer(&sc->partial, &sc->partial_bytes, size_t(fp.n_ch) * fp.n_ntiles * P * sizeof(T), rq.stream);
          if (sc->counters_n < size_t(n_mtiles)) {
            size_t cap = sc->counters_n * sizeof(unsigned);
            void* ptr = sc->counters;
            ensure_buffer(&ptr, &cap, size_t(n_mtiles) * sizeof(unsigned), rq.stream);
            sc->counters = static_cast<unsigned*>(ptr);
            sc->counters_n = cap / sizeof(unsigned);
            EVB_CUDA(cudaMemsetAsync(sc->counters, 0, cap, rq.stream));
          }
          fp.partial = static_cast<T*>(sc->partial);
          fp.counters = sc->counters;
        }
        // EVB_UMMA_ATMEM=1: S_hi / S_lo as the MMA's A operand in TMEM (shared memory then feeds only
        // B).  Correct, but measured equal (22.9 vs 23.0 us per config-1 launch): the N = 128 tf32 MMAs
        // are not bound by shared-memory bandwidth but by a fixed per-instruction cost (~30 cycles,
        // from the probe's N = 64 / 256 rates), so the default keeps the operands in shared memory.
        static const bool atmem = std::getenv("EVB_UMMA_ATMEM") && std::atoi(std::getenv("EVB_UMMA_ATMEM")) == 1;
        static const bool timeline = std::getenv("EVB_K1_TIMELINE") != nullptr;
        if (timeline) {  // one synchronous launch, per-CTA phase stamps appended to a CSV
          const int nct = n_tiles * splitk;
          unsigned long long* d = nullptr;
          EVB_CUDA(cudaMalloc(&d, size_t(nct) * 8 * 8));
          EVB_CUDA(cudaMemset(d, 0, size_t(nct) * 8 * 8));
          fused_params<float> f2 = fp;
          f2.dbg_ts = d;
          f2.dbg_skip = std::getenv("EVB_K2_SKIP") ? std::atoi(std::getenv("EVB_K2_SKIP")) : 0;
          if (use16) launch_f32_umma_sk<SBN, false, true>(ta_hi, tb_hi, tb_lo, f2, splitk, rq.stream);
          else if (atmem) launch_f32_umma_sk<SBN, true>(ta_hi, tb_hi, tb_lo, f2, splitk, rq.stream);
          else launch_f32_umma_sk<SBN, false>(ta_hi, tb_hi, tb_lo, f2, splitk, rq.stream);
          EVB_CUDA(cudaStreamSynchronize(rq.stream));
          std::vector<unsigned long long> h(size_t(nct) * 8);
          EVB_CUDA(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
          cudaFree(d);
          if (FILE* f = std::fopen("gpurun_out/k2_ts.csv", "a")) {
            for (int c = 0; c < nct; ++c)
              std::fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu,%llu\n", c, h[c * 8 + 0], h[c * 8 + 1], h[c * 8 + 3],
                           h[c * 8 + 4], h[c * 8 + 5], h[c * 8 + 6], h[c * 8 + 2]);
            std::fprintf(f, "end\n");
            std::fclose(f);
          }
        } else {
          if (use16) launch_f32_umma_sk<SBN, false, true>(ta_hi, tb_hi, tb_lo, fp, splitk, rq.stream);
          else if (atmem) launch_f32_umma_sk<SBN, true>(ta_hi, tb_hi, tb_lo, fp, splitk, rq.stream);
          else launch_f32_umma_sk<SBN, false>(ta_hi, tb_hi, tb_lo, fp, splitk, rq.stream);
        }
        if (!own_rot) {
          EVB_CUDA(cudaStreamSynchronize(rq.stream));
          if (rhi) cudaFree(rhi);
          if (rlo) cudaFree(rlo);
          if (r16h) cudaFree(r16h);
          if (r16l) cudaFree(r16l);
        }
        return;
      }
      if (fuse) {
        ok = make_tma_2d(&ta_hi, X, EVB_F32, uint64_t(D), uint64_t(P), uint64_t(ldx) * 4, 32, 128);
        ta_lo = ta_hi;
      } else {
        const int64_t lds = round_up(D, 32);
        ensure_buffer(&sc->s_hi, &sc->s_hi_bytes, size_t(lds) * P * sizeof(float), rq.stream);
        ensure_buffer(&sc->s_lo, &sc->s_lo_bytes, size_t(lds) * P * sizeof(float), rq.stream);
        split_tf32_kernel<<<dim3(unsigned((lds + 255) / 256), unsigned(P)), 256, 0, rq.stream>>>(
            static_cast<const float*>(X), ldx, shift, P, D, static_cast<float*>(sc->s_hi),
            static_cast<float*>(sc->s_lo), lds);
        count_launch();
        ok = make_tma_2d(&ta_hi, sc->s_hi, EVB_F32, uint64_t(lds), uint64_t(P), uint64_t(lds) * 4, 32, 128) &&
             make_tma_2d(&ta_lo, sc->s_lo, EVB_F32, uint64_t(lds), uint64_t(P), uint64_t(lds) * 4, 32, 128);
      }
      ok = ok && make_tma_2d(&tb_hi, rhi, EVB_F32, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * 4, 32, uint32_t(UBN)) &&
                make_tma_2d(&tb_lo, rlo, EVB_F32, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * 4, 32, uint32_t(UBN));
      if (!ok) throw runtime_error("gemm_eval: cannot encode the TMA descriptors of the tf32 split");
      fp.n_ntiles = (D + UBN - 1) / UBN;
      const int n_mtiles = (P + 127) / 128;
      if (!zstore) {
        ensure_buffer(&sc->partial, &sc->partial_bytes, size_t(fp.n_ch) * fp.n_ntiles * P * sizeof(T), rq.stream);
        if (sc->counters_n < size_t(n_mtiles)) {
          size_t cap = sc->counters_n * sizeof(unsigned);
          void* ptr = sc->counters;
          ensure_buffer(&ptr, &cap, size_t(n_mtiles) * sizeof(unsigned), rq.stream);
          sc->counters = static_cast<unsigned*>(ptr);
          sc->counters_n = cap / sizeof(unsigned);
          EVB_CUDA(cudaMemsetAsync(sc->counters, 0, cap, rq.stream));
        }
        fp.partial = static_cast<T*>(sc->partial);
        fp.counters = sc->counters;
      }
      static const bool timeline = std::getenv("EVB_K1_TIMELINE") != nullptr;
      if (timeline && UBN == 64) {  // one synchronous launch, phase stamps appended to a CSV
        const int nct = int(((P + 127) / 128) * ((D + 63) / 64));
        unsigned long long* d = nullptr;
        EVB_CUDA(cudaMalloc(&d, size_t(nct) * 8 * 8));
        EVB_CUDA(cudaMemset(d, 0, size_t(nct) * 8 * 8));
        fused_params<float> f2 = fp;
        f2.dbg_ts = d;
        if (fuse) launch_f32_umma<64, true>(ta_hi, ta_lo, tb_hi, tb_lo, f2, rq.stream);
        else launch_f32_umma<64>(ta_hi, ta_lo, tb_hi, tb_lo, f2, rq.stream);
        EVB_CUDA(cudaStreamSynchronize(rq.stream));
        std::vector<unsigned long long> h(size_t(nct) * 8);
        EVB_CUDA(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
        cudaFree(d);
        if (FILE* f = std::fopen("gpurun_out/k2_ts.csv", "a")) {
          for (int c = 0; c < nct; ++c)
            std::fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu\n", c, h[c * 8 + 0], h[c * 8 + 1], h[c * 8 + 3],
                         h[c * 8 + 4], h[c * 8 + 5], h[c * 8 + 6]);
          std::fprintf(f, "end\n");
          std::fclose(f);
        }
      } else if (UBN == 256) launch_f32_umma<256>(ta_hi, ta_lo, tb_hi, tb_lo, fp, rq.stream);
      else if (UBN == 128) launch_f32_umma<128>(ta_hi, ta_lo, tb_hi, tb_lo, fp, rq.stream);
      else if (fuse) launch_f32_umma<64, true>(ta_hi, ta_lo, tb_hi, tb_lo, fp, rq.stream);
      else launch_f32_umma<64>(ta_hi, ta_lo, tb_hi, tb_lo, fp, rq.stream);
      if (!own_rot) {
        EVB_CUDA(cudaStreamSynchronize(rq.stream));
        cudaFree(rhi);
        cudaFree(rlo);
      }
      return;
    }
  }
  CUtensorMap tmX, tmM;
  if (!make_tma_2d(&tmX, X, dtype, uint64_t(D), uint64_t(P), uint64_t(ldx) * sizeof(T), KB, BM))
    throw runtime_error("gemm_eval: cannot encode the TMA descriptor of X");
  if (!make_tma_2d(&tmM, rotation, dtype, uint64_t(ldm), uint64_t(D), uint64_t(ldm) * sizeof(T), KB, BN))
    throw runtime_error("gemm_eval: cannot encode the TMA descriptor of M");
  fp.n_ntiles = (D + BN - 1) / BN;
  static const bool timeline = std::getenv("EVB_K1_TIMELINE") != nullptr;
  const int n_mtiles = (P + BM - 1) / BM;
  if (!zstore) {
    ensure_buffer(&sc->partial, &sc->partial_bytes, size_t(fp.n_ch) * fp.n_ntiles * P * sizeof(T), rq.stream);
    if (sc->counters_n < size_t(n_mtiles)) {
      size_t cap = sc->counters_n * sizeof(unsigned);
      void* ptr = sc->counters;
      ensure_buffer(&ptr, &cap, size_t(n_mtiles) * sizeof(unsigned), rq.stream);
      sc->counters = static_cast<unsigned*>(ptr);
      sc->counters_n = cap / sizeof(unsigned);
      EVB_CUDA(cudaMemsetAsync(sc->counters, 0, cap, rq.stream));
    }
    fp.partial = static_cast<T*>(sc->partial);
    fp.counters = sc->counters;
  }
  if constexpr (std::is_same<T, double>::value) {
    if (!use_persistent && rq.kgate) {
      fp.kgate = rq.kgate;
      fp.kgate_n = rq.kgate_n;
      for (int c = 0; c < rq.kgate_n; ++c) fp.kgate_end[c] = rq.kgate_end[c];
      fp.kgate_epoch = rq.kgate_epoch;
      gate_consumed = true;
    }
  }
  if (rq.x_ready && !gate_consumed) EVB_CUDA(cudaStreamWaitEvent(rq.stream, rq.x_ready, 0));
  if constexpr (std::is_same<T, double>::value) {
    if (use_persistent) {
      launch_f64_persistent<64, 56>(tmX, tmM, fp, rq.stream);
      return;
    }
    // (measured alternatives: 64 x 40 and 48 x 56 tiles at 3 CTAs / SM, 32 x 56 warp tiles —
    // all slower: 91, 115 and 146 us against 81.5 us per config-1 batch)
    if (BM == 64 && BN == 56 && timeline) {  // one synchronous launch, phase stamps appended to a CSV
      const int nct = int(((P + BM - 1) / BM) * fp.n_ntiles);
      unsigned long long* d = nullptr;
      EVB_CUDA(cudaMalloc(&d, size_t(nct) * 8 * 8));
      EVB_CUDA(cudaMemset(d, 0, size_t(nct) * 8 * 8));
      fused_params<double> f2 = fp;
      f2.dbg_ts = d;
      launch_f64<64, 56, 4, 1, 6, 2>(tmX, tmM, f2, rq.stream);
      EVB_CUDA(cudaStreamSynchronize(rq.stream));
      std::vector<unsigned long long> h(size_t(nct) * 8);
      EVB_CUDA(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
      cudaFree(d);
      if (FILE* f = std::fopen("gpurun_out/k1_ts.csv", "a")) {
        for (int c = 0; c < nct; ++c)
          std::fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu,%llu\n", c, h[c * 8 + 0], h[c * 8 + 1], h[c * 8 + 2],
                       h[c * 8 + 3], h[c * 8 + 4], h[c * 8 + 5], h[c * 8 + 7]);
        std::fprintf(f, "end\n");
        std::fclose(f);
      }
    } else if (BM == 64 && BN == 56) launch_f64<64, 56, 4, 1, 6, 2>(tmX, tmM, fp, rq.stream);
    else if (BM == 64 && BN == 112) launch_f64<64, 112, 4, 2>(tmX, tmM, fp, rq.stream);
    else if (BM == 64 && BN == 128) launch_f64<64, 128, 4, 2>(tmX, tmM, fp, rq.stream);
    else launch_f64<32, 128, 2, 4>(tmX, tmM, fp, rq.stream);
  } else {
    launch_f32<64, 128>(tmX, tmM, fp, rq.stream);
  }
}

// Row-block height of the multi-problem kernel: 64 by default.  EVB_K1M_BM=128 selects the
// one-wave variant (NP = 3; config 1: 144 CTAs of 128 x 56 x 3 instead of 148 + 140 of 64 x 56 x 3).
// Measured equal on the device (216.2 vs 215.6 us, results bit-identical): the single wave saves one
// CTA turnover and one first stage, but its epilogue is twice as long and nothing overlaps it
// either; from host buffers it is slower (every CTA needs every column chunk: 320 vs 263 us).
int multi_bm(int np, int64_t, int64_t) {
  if (np != 3) return kMultiBM;
  static const char* env = std::getenv("EVB_K1M_BM");
  return env && std::atoi(env) == 128 ? 128 : kMultiBM;
}

int multi_first_wave_rows(int np, int64_t n_points, int64_t dim) {
  if (np < 2 || np > 3) return 0;
  if (multi_bm(np, n_points, dim) == 128) return 0;  // one wave: every CTA needs all columns
  constexpr int BM = kMultiBM, BN = kMultiBN;
  const int64_t n_ntiles = (dim + BN - 1) / BN, n_mtiles = (n_points + BM - 1) / BM;
  // occupancy of the multi-problem kernel, queried once per NP (host cost of every host call)
  static int per_sm_cache[4] = {0, 0, 0, 0};
  const int sms = sm_count();
  int per_sm = per_sm_cache[np];
  if (per_sm == 0) {
    if (np == 3) {
      EVB_CUDA(cudaFuncSetAttribute(eval_f64_dmma_multi_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    f64m_cfg<3>::SMEM));
      EVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eval_f64_dmma_multi_kernel<3>,
                                                             f64m_cfg<3>::THREADS, f64m_cfg<3>::SMEM));
    } else {
      EVB_CUDA(cudaFuncSetAttribute(eval_f64_dmma_multi_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    f64m_cfg<2>::SMEM));
      EVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eval_f64_dmma_multi_kernel<2>,
                                                             f64m_cfg<2>::THREADS, f64m_cfg<2>::SMEM));
    }
    per_sm_cache[np] = per_sm = std::max(per_sm, 1);
  }
  const int64_t wave = int64_t(sms) * per_sm;
  if (n_ntiles * n_mtiles <= wave) return 0;
  // row blocks the first wave covers completely (EVB_H2D_ROWS=ceil: also the partly covered one,
  // tuning aid); the first wave's few tiles of the next row block wait for the second group
  static const char* env = std::getenv("EVB_H2D_ROWS");
  const bool ceil_rows = env && std::string(env) == "ceil";
  const int64_t rb = ceil_rows ? (wave + n_ntiles - 1) / n_ntiles : wave / n_ntiles;
  return rb >= n_mtiles || rb == 0 ? 0 : int(rb * BM);
}

// NP base problems (same D) on one device X: one multi-problem K1 launch; rqs[g] carries problem
// g's kinds / biases / output, rqs[0] the gates.  Returns false when the shapes do not fit.
bool gemm_eval_multi(const eval_request* rqs, int np, const void* X, int64_t ldx) {
  if (np < 2 || np > 3) return false;
  const int P = int(rqs[0].n), D = rqs[0].prob->dim;
  evb_scratch_s* sc = rqs[0].scratch;
  fused_params<double> fp[3]{};
  multi_maps<3> maps3{};
  multi_maps<2> maps2{};
  constexpr int BN = kMultiBN;
  const int BM = multi_bm(np, P, D);
  const int n_ntiles = (D + BN - 1) / BN, n_mtiles = (P + BM - 1) / BM;
  CUtensorMap tmX;
  if (!make_tma_2d(&tmX, X, EVB_F64, uint64_t(D), uint64_t(P), uint64_t(ldx) * 8, 16, BM)) return false;
  size_t part_total = 0;
  for (int g = 0; g < np; ++g) {
    const eval_request& rq = rqs[g];
    fused_params<double>& f = fp[g];
    f.P = P;
    f.D = D;
    f.ell_w = static_cast<const double*>(rq.prob->ell_w);
    f.shift = static_cast<const double*>(rq.prob->shift);
    f.out = static_cast<double*>(rq.out);
    f.ldo = rq.ldo;
    if (!build_plan<double>(f, rq.n_out, rq.kinds, rq.biases)) return false;
    f.n_ntiles = n_ntiles;
    part_total += size_t(f.n_ch) * n_ntiles * P;
    CUtensorMap& m = np == 3 ? maps3.m[g] : maps2.m[g];
    if (!make_tma_2d(&m, rq.prob->rotation, EVB_F64, uint64_t(rq.prob->ld), uint64_t(D), uint64_t(rq.prob->ld) * 8, 16,
                     BN))
      return false;
  }
  cudaStream_t st = rqs[0].stream;
  ensure_buffer(&sc->partial, &sc->partial_bytes, part_total * sizeof(double), st);
  const size_t need_counters = size_t(np) * n_mtiles;
  if (sc->counters_n < need_counters) {
    size_t cap = sc->counters_n * sizeof(unsigned);
    void* ptr = sc->counters;
    ensure_buffer(&ptr, &cap, need_counters * sizeof(unsigned), st);
    sc->counters = static_cast<unsigned*>(ptr);
    sc->counters_n = cap / sizeof(unsigned);
    EVB_CUDA(cudaMemsetAsync(sc->counters, 0, cap, st));
  }
  size_t off = 0;
  for (int g = 0; g < np; ++g) {
    fp[g].partial = static_cast<double*>(sc->partial) + off;
    off += size_t(fp[g].n_ch) * n_ntiles * P;
    fp[g].counters = sc->counters + size_t(g) * n_mtiles;
  }
  if (rqs[0].kgate) {
    fp[0].kgate = rqs[0].kgate;
    fp[0].kgate_n = rqs[0].kgate_n;
    for (int c = 0; c < rqs[0].kgate_n; ++c) fp[0].kgate_end[c] = rqs[0].kgate_end[c];
    fp[0].kgate_epoch = rqs[0].kgate_epoch;
    fp[0].kgate_rows = rqs[0].kgate_rows;
  } else if (rqs[0].x_ready) {
    EVB_CUDA(cudaStreamWaitEvent(st, rqs[0].x_ready, 0));
  }
  // with the rows split into two gate groups the first wave must be the first rows' tiles
  const bool nfast = rqs[0].kgate && rqs[0].kgate_rows > 0;
  fp[0].tiles_nfast = nfast ? 1 : 0;
  dim3 grid(nfast ? n_ntiles : n_mtiles, nfast ? n_mtiles : n_ntiles);
  if (np == 3 && BM == 128) {
    using C = f64m_cfg<3, 128>;
    static bool attr = false;
    if (!attr) {
      EVB_CUDA(cudaFuncSetAttribute(eval_f64_dmma_multi_kernel<3, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::SMEM));
      attr = true;
    }
    eval_f64_dmma_multi_kernel<3, 128><<<grid, C::THREADS, C::SMEM, st>>>(tmX, maps3, fp[0], fp[1], fp[2]);
  } else if (np == 3) {
    using C = f64m_cfg<3>;
    static bool attr = false;
    if (!attr) {
      EVB_CUDA(cudaFuncSetAttribute(eval_f64_dmma_multi_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
      attr = true;
    }
    static const bool timeline = std::getenv("EVB_K1_TIMELINE") != nullptr;
    unsigned long long* dts = nullptr;
    const int nct = int(grid.x * grid.y);
    if (timeline) {
      EVB_CUDA(cudaMalloc(&dts, size_t(nct) * 64));
      EVB_CUDA(cudaMemset(dts, 0, size_t(nct) * 64));
      fp[0].dbg_ts = dts;
    }
    eval_f64_dmma_multi_kernel<3><<<grid, C::THREADS, C::SMEM, st>>>(tmX, maps3, fp[0], fp[1], fp[2]);
    if (timeline) {  // one synchronous launch, phase stamps appended to a CSV
      EVB_CUDA(cudaStreamSynchronize(st));
      std::vector<unsigned long long> h(size_t(nct) * 8);
      EVB_CUDA(cudaMemcpy(h.data(), dts, h.size() * 8, cudaMemcpyDeviceToHost));
      cudaFree(dts);
      if (FILE* f = std::fopen("gpurun_out/k1m_ts.csv", "a")) {
        for (int c = 0; c < nct; ++c)
          std::fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu\n", c, h[c * 8 + 0], h[c * 8 + 1], h[c * 8 + 2], h[c * 8 + 4],
                       h[c * 8 + 7]);
        std::fprintf(f, "end\n");
        std::fclose(f);
      }
    }
  } else {
    using C = f64m_cfg<2>;
    static bool attr = false;
    if (!attr) {
      EVB_CUDA(cudaFuncSetAttribute(eval_f64_dmma_multi_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
      attr = true;
    }
    eval_f64_dmma_multi_kernel<2><<<grid, C::THREADS, C::SMEM, st>>>(tmX, maps2, fp[0], fp[1], fp[1]);
  }
  EVB_CUDA(cudaGetLastError());
  count_launch();
  return true;
}

template void gemm_eval<double>(const eval_request&, const void*, int64_t, bool, double*, int64_t, const double*,
                                const void*, int, int, int);
template void gemm_eval<float>(const eval_request&, const void*, int64_t, bool, float*, int64_t, const float*,
                               const void*, int, int, int);

bool fused_kinds_ok(int n, const int* kinds) {
  int terms[kMaxCh];
  int nt = 0;
  for (int o = 0; o < n; ++o) {
    const kind_channels kc = channels_for(kinds[o]);
    if (kc.n == 0) return false;
    for (int c = 0; c < kc.n; ++c) {
      bool f = false;
      for (int q = 0; q < nt; ++q) f = f || terms[q] == kc.term[c];
      if (!f) {
        if (nt == kMaxCh) return false;
        terms[nt++] = kc.term[c];
      }
    }
  }
  return n <= kMaxOut;
}

}  // namespace evb
