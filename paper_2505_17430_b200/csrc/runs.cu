// runs.cu — K8: many independent DE runs in ONE persistent launch (BASELINE config 4).
//
// Replaces the reference's thread pool over independent runs (experiment/runner.hpp:101-160,
// evo_bench) for small problems: one CTA owns one run for ALL its generations, with the
// population, the trial vectors, the run's rotation(s) and shift(s) resident in shared memory.
// Per generation, inside the CTA (de/engine.hpp:71-102 semantics):
//   draws     thread per individual, Philox sub-stream (g << 32) | i of the run's key: donor
//             indices with the reference's rejection loops, jrand (de/strategy.hpp:84-86, 187)
//   trial     thread per gene: binomial mask from the gene's word, donor x_r1 + F (x_r2 - x_r3),
//             clip / midpoint repair (de/strategy.hpp:93, 189-193, 234-276)
//   evaluate  the run's problem on every trial: z = M_k (t - o_k) accumulated in the reference's
//             order (separate mul / add), base values, composition weights and weighted sum in
//             double (problems/instance.hpp:60-76, 116-174)
//   select    trial replaces parent when f_trial <= f_parent (de/engine.hpp:36)
// Supported here: rand/1 or best/1 with a fixed adapter and no archive (the `de` preset,
// presets.hpp:59-69) on base or composition problems whose data fit in shared memory.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "evb_internal.cuh"
#include "evb_math.cuh"
#include "ptx.cuh"
#include "rng.cuh"
#include "recorder.cuh"

namespace evb {
namespace {

constexpr int kRunsMaxComp = 4;

// EVB_RUNS_PROFILE=1: CTA 0's thread 0 accumulates clock64() per phase (the phases end at block
// barriers, so its clock marks the phase boundary) — a tuning aid, off by default.
// The profiling build is a separate instantiation (PROF): without it the marks compile to
// nothing (a runtime null check kept the struct in local memory, and every thread's check was an
// L1-missing load on the phase boundaries).
template <bool PROF>
struct phase_clock {
  unsigned long long* acc;  // null: off
  long long last;
  __device__ __forceinline__ void start() {
    if constexpr (PROF)
      if (acc && threadIdx.x == 0) last = clock64();
  }
  __device__ __forceinline__ void mark(int k) {
    if constexpr (PROF)
      if (acc && threadIdx.x == 0) {
        const long long t = clock64();
        acc[k] += (unsigned long long)(t - last);
        last = t;
      }
  }
};

struct run_problem {
  const double* shift[kRunsMaxComp];  // per component (base problem: component 0)
  const double* rot[kRunsMaxComp];
  int kind[kRunsMaxComp];
  double sigma[kRunsMaxComp], lambda[kRunsMaxComp], cbias[kRunsMaxComp];
  int n_comp;  // 0: base or hybrid problem (shift[0], rot[0], kind[0])
  int ld;      // row stride of the rotations
  double bias;
  const double* ell_w;
  // hybrid (problems/instance.hpp:97-112): permutation, chunk kinds / sizes, per-chunk weights
  int hybrid, n_chunks;
  const int* perm;
  const int* sub_kinds;
  const int* chunk_sizes;
  const double* hyb_w;
};

// crossover test u01(w) < CR as an integer compare (de.cu take_rule): u01(w) = (w >> 11) 2^-53
// (core/rng.hpp:81-83), so u01(w) < CR <=> (w >> 11) < ceil(CR 2^53) <=> w <= lim; CR <= 0 never
struct take_rule_host {
  uint64_t lim;
  int none;
  static take_rule_host make(double cr) {
    take_rule_host r;
    const double t = std::ceil(cr * 0x1.0p53);
    r.none = !(t >= 1.0);
    const uint64_t ti = t >= 0x1.0p53 ? (uint64_t(1) << 53) : uint64_t(r.none ? 1.0 : t);
    r.lim = ((ti - 1) << 11) | 0x7FFu;
    return r;
  }
  __device__ __forceinline__ bool bit(uint64_t w) const { return !none && w <= lim; }
};

struct runs_args {
  take_rule_host take;
  int P, D, G, ld;
  int mutation, repair;
  double F, CR, lb, ub;
  const run_problem* probs;
  const uint64_t* keys;
  uint32_t gen0;
  double* pop;  // n_runs x P x D
  double* fit;  // n_runs x P
  int init;
  int rec_on;
  rec_view<double> rec;  // best-so-far recorder, run r -> recorder run r
  unsigned long long* prof;  // EVB_RUNS_PROFILE: per-phase clocks of CTA 0 (else null)
  int split;             // CTAs per run (1, or a 2-CTA cluster that splits every evaluation)
  int resident;          // all rotations / shifts of a run staged in shared memory once
  int n_mat;             // max components over the runs (resident slots)
  int tc;                // tensor-core (DMMA) dots with resident operands
  int tc_epi;            // tc: warp-parallel distance / base-value sums and the fast cos(2 pi z)
};

__device__ __forceinline__ double clip_or_mid(double v, double target, double lb, double ub, int repair) {
  if (repair == EVB_REP_CLIP) {
    if (v < lb) v = lb;
    if (v > ub) v = ub;
  } else if (repair == EVB_REP_MIDPOINT_TARGET) {
    if (v < lb) v = __ddiv_rn(__dadd_rn(lb, target), 2.0);
    else if (v > ub) v = __ddiv_rn(__dadd_rn(ub, target), 2.0);
  }
  return v;
}

// Evaluate the P rows of `X` (smem, stride D) into f (smem).  Per component: s = x - o is staged
// once (rounded like transform_input's diff, problems/instance.hpp:66-67), then z = M s with each
// z[i][r] accumulated over k in the reference's order (separate mul and add).  Register blocking:
// lane r owns one row of M (conflict-free, odd stride) and up to 8 individuals of its group, whose
// s[i][k] are warp-broadcast loads — ~8x fewer shared-memory wavefronts per MAC than one dot per
// thread.  Base values and composition weights are sequential per individual (exact order).
// Q dot products z[i][r] = sum_k M[r][k] s[i][k] of one row r (individuals i0, i0 + G, ...),
// accumulated in the reference's order (separate mul and add, increasing k).
// Q dot products z[i][r] = sum_k M[r][k] s[i][k] of row r, individuals i0, i0 + G, ... (the first
// n <= Q are real), accumulated in the reference's order (separate mul and add, increasing k).
template <int Q, bool EXACT>
__device__ __forceinline__ void dot_rows(const double* __restrict__ m, const double* __restrict__ sS, int D, int i0,
                                         int G, int n, double* __restrict__ sZ, int r) {
  double acc[Q];
  const double* sp[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    acc[q] = 0.0;
    sp[q] = sS + (i0 + (EXACT ? q : min(q, n - 1)) * G) * D;
  }
  int k = 0;
  if ((D & 1) == 0 && (reinterpret_cast<uintptr_t>(sS) & 15) == 0) {
    // even D: each individual's (k, k+1) pair is one 16-byte word (LDS.128) — 10 instead of 18
    // shared loads per pair of k; the adds stay in increasing k
    for (; k < D; k += 2) {
      const double mk0 = m[k], mk1 = m[k + 1];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double2 sv = *reinterpret_cast<const double2*>(sp[q] + k);
        acc[q] = __dadd_rn(acc[q], __dmul_rn(mk0, sv.x));
        acc[q] = __dadd_rn(acc[q], __dmul_rn(mk1, sv.y));
      }
    }
  }
  for (; k < D; ++k) {
    const double mk = m[k];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(mk, sp[q][k]));
  }
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (EXACT || q < n) sZ[(i0 + q * G) * D + r] = acc[q];
}

// K3 on the FP64 tensor core: z[i][r] = sum_k s[i][k] M[r][k] for the R rows of sS by DMMA
// m8n8k4 (the survey's K3; problems/instance.hpp:60-76, 116-174 per component).  sS is RP x KS and
// M is NP8 x KS (RP, NP8 = multiples of 8; KS = round_up(D, 8) with KS % 16 == 8, so a quarter
// warp's 16-byte fragment loads hit 8 distinct 16-byte bank groups); pad rows / columns hold zeros.
// Inside each 8-deep k slice lane (g, t) feeds k = 2t at the first step and 2t + 1 at the second
// (one LDS.128 per operand per two steps; A and B use the same k permutation).  Warp task = 8 rows
// x 16 columns (one A fragment, two B fragments).  The accumulation order differs from the
// reference's sequential one (fitness within ~1e-15 relative; selections equal except flagged
// near-ties).
__device__ __forceinline__ void dmma_rows(const double* __restrict__ sS, const double* __restrict__ sM, int R, int D,
                                          int KS, double* __restrict__ sZ) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mt = (R + 7) >> 3, nt = (D + 15) >> 4;
  for (int task = warp; task < mt * nt; task += nwarps) {
    // m fastest: the narrow last column tile's tasks spread over the SM sub-partitions (warp % 4)
    const int m0 = (task % mt) << 3, n0 = (task / mt) << 4;
    const bool two = n0 + 8 < D;  // warp-uniform
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    const double* pa = sS + (m0 + g) * KS + 2 * t;
    const double* pb = sM + (n0 + g) * KS + 2 * t;
    if (two) {
      const double* pb1 = pb + 8 * KS;
#pragma unroll 4
      for (int k0 = 0; k0 < KS; k0 += 8) {
        const double2 a = *reinterpret_cast<const double2*>(pa + k0);
        const double2 b0 = *reinterpret_cast<const double2*>(pb + k0);
        const double2 b1 = *reinterpret_cast<const double2*>(pb1 + k0);
        ptx::dmma_8x8x4(c00, c01, a.x, b0.x);
        ptx::dmma_8x8x4(c10, c11, a.x, b1.x);
        ptx::dmma_8x8x4(c00, c01, a.y, b0.y);
        ptx::dmma_8x8x4(c10, c11, a.y, b1.y);
      }
    } else {
#pragma unroll 4
      for (int k0 = 0; k0 < KS; k0 += 8) {
        const double2 a = *reinterpret_cast<const double2*>(pa + k0);
        const double2 b0 = *reinterpret_cast<const double2*>(pb + k0);
        ptx::dmma_8x8x4(c00, c01, a.x, b0.x);
        ptx::dmma_8x8x4(c00, c01, a.y, b0.y);
      }
    }
    const int row = m0 + g;
    if (row < R) {
      const int c0 = n0 + 2 * t;
      if (c0 < D) sZ[row * D + c0] = c00;
      if (c0 + 1 < D) sZ[row * D + c0 + 1] = c01;
      if (two) {
        if (c0 + 8 < D) sZ[row * D + c0 + 8] = c10;
        if (c0 + 9 < D) sZ[row * D + c0 + 9] = c11;
      }
    }
  }
}

// tensor-core layout of the resident operands (dmma_rows)
__host__ __device__ __forceinline__ int tc_ks(int D) {
  const int k = (D + 7) / 8 * 8;
  return (k % 16 == 8) ? k : k + 8;
}
__host__ __device__ __forceinline__ int round8(int v) { return (v + 7) / 8 * 8; }

// KS > 0: tensor-core dots (dmma_rows; resident operands in the tc layout, sS stride KS with
// zero pads), else exact-order dots (dot_rows; M stride S, sS stride D)
template <bool PROF>
__device__ void runs_evaluate(const run_problem& pr, const double* X, int P, int D, int S, double* sMbase,
                              double* sZ, double* sS, double* sObase, double* sFk, double* sDist, double* f,
                              bool resident, int KS, int fast_epi, double* part, phase_clock<PROF>& pc) {
  const int ncomp = pr.n_comp > 0 ? pr.n_comp : 1;
  // fast tensor-core epilogue (KS > 0 && fast_epi): x - o and the distance partials in one pass,
  // base-value sums in two levels (8-element chunks, then per individual); part holds
  // R x nqK distance partials and 2 x R x nqD base partials
  const bool fast = KS > 0 && fast_epi;
  const int nqK = KS > 0 ? KS / 8 : 0, nqD = (D + 7) / 8;
  double* part_d = part;
  double* part_b = part ? part + size_t(round8(P)) * nqK : nullptr;
  const int SS = KS > 0 ? KS : D;  // row stride of sS
  for (int c = 0; c < ncomp; ++c) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    // resident: every component's M and o were staged once at kernel start
    double* sM = resident ? sMbase + size_t(c) * (KS > 0 ? size_t(round8(D)) * KS : size_t(D) * S) : sMbase;
    double* sO = resident ? sObase + size_t(c) * D : sObase;
    if (!resident) {
      for (int r = warp; r < D; r += nwarps)
        for (int k = lane; k < D; k += 32) sM[r * S + k] = pr.rot[c][r * pr.ld + k];
      for (int e = threadIdx.x; e < D; e += blockDim.x) sO[e] = pr.shift[c][e];
      __syncthreads();
    }
    if (fast) {  // thread = (row, 8-wide chunk): s = x - o with zero pads, and the chunk's dist^2
      const int RP = round8(P);
      for (int e = threadIdx.x; e < RP * nqK; e += blockDim.x) {
        const int i = e / nqK, q = e - i * nqK;
        double sv[8], d2 = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = 8 * q + j;
          sv[j] = (i < P && k < D) ? __dsub_rn(X[i * D + k], sO[k]) : 0.0;
          d2 = fma(sv[j], sv[j], d2);
        }
        double2* dst = reinterpret_cast<double2*>(sS + size_t(i) * KS + 8 * q);
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = make_double2(sv[2 * j], sv[2 * j + 1]);
        part_d[e] = d2;
      }
    } else if (KS > 0) {  // all RP x KS entries: the pads are zero for the tensor-core tiles
      const int RP = round8(P);
      for (int e = threadIdx.x; e < RP * KS; e += blockDim.x) {
        const int i = e / KS, k = e - i * KS;
        sS[e] = (i < P && k < D) ? __dsub_rn(X[i * D + k], sO[k]) : 0.0;
      }
    } else {
      for (int i = warp; i < P; i += nwarps)
        for (int k = lane; k < D; k += 32) sS[i * D + k] = __dsub_rn(X[i * D + k], sO[k]);
    }
    __syncthreads();
    pc.mark(2);
    {
      // dist^2 in double (problems/instance.hpp:127-134): one sequential chain per individual;
      // the tensor-core path (a tolerance path already) takes a warp per individual and a
      // shuffle tree (the weights it feeds are relative: ~1e-16)
      if (fast) {
        // the distance partials were formed with x - o; summed with the base values below
      } else if (pr.n_comp > 0)
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          double d2 = 0.0;
          const double* si = sS + i * SS;
          for (int j = 0; j < D; ++j) d2 = __dadd_rn(d2, __dmul_rn(si[j], si[j]));
          sDist[i * kRunsMaxComp + c] = d2;
        }
      if constexpr (PROF) {  // profiling only: separate the distance chains from the dots
        __syncthreads();
        pc.mark(9);
      }
      // thread t owns row r = t % D for individual group g = t / D (G groups): individuals g,
      // g + G, ... — rows over consecutive lanes (odd stride: conflict-free), every chain real
      const int G = max(1, int(blockDim.x) / D);
      const int t = int(threadIdx.x);
      if (KS > 0) {
        dmma_rows(sS, sM, P, D, KS, sZ);
      } else if (t < G * D) {
        const int r = t % D, g = t / D;
        const double* m = sM + r * S;
        for (int i0 = g; i0 < P; i0 += 8 * G) {
          const int n = min(8, (P - i0 + G - 1) / G);
          if (n == 8) dot_rows<8, true>(m, sS, D, i0, G, n, sZ, r);
          else if (n == 5) dot_rows<5, true>(m, sS, D, i0, G, n, sZ, r);
          else dot_rows<8, false>(m, sS, D, i0, G, n, sZ, r);
        }
      }
    }
    __syncthreads();
    pc.mark(3);
    if (pr.hybrid) {  // permuted chunks, sequential per individual
      for (int i = threadIdx.x; i < P; i += blockDim.x)
        sFk[i * kRunsMaxComp] =
            hybrid_value<double>(pr.perm, pr.sub_kinds, pr.chunk_sizes, pr.n_chunks, pr.hyb_w, sZ + i * D, 1);
      __syncthreads();
      continue;
    }
    const int kind = pr.kind[c];
    if (KS > 0 && fast_epi && (kind == EVB_RASTRIGIN || kind == EVB_ACKLEY)) {
      // tensor-core path: the transcendental terms with cos2pi_fast (the reference's formulas),
      // element-parallel into sS; the sequential sums below are the reference's order
#pragma unroll 2
      for (int e = threadIdx.x; e < P * D; e += blockDim.x) {
        const double v = sZ[e];
        const double cz = cos2pi_fast_ok(v) ? cos2pi_fast(v) : cos(__dmul_rn(two_pi_v<double>(), v));
        sS[e] = kind == EVB_ACKLEY ? cz : __dadd_rn(__dsub_rn(__dmul_rn(v, v), __dmul_rn(10.0, cz)), 10.0);
      }
      __syncthreads();
    } else if (kind_has_pre(kind)) {  // transcendental terms in parallel over all P*D elements (into sS)
      for (int e = threadIdx.x; e < P * D; e += blockDim.x) {
        const int i = e / D, k = e - i * D;
        const double* zr = sZ + i * D;
        auto z = [&](int q) { return zr[q]; };
        sS[e] = base_pre_term<double, false>(kind, D, z, k);
      }
      __syncthreads();
    }
    pc.mark(4);
    if (fast && (kind == EVB_RASTRIGIN || kind == EVB_ACKLEY || kind == EVB_ELLIPTIC || kind == EVB_SPHERE)) {
      // chunk sums (thread = (individual, 8 elements)), then per individual; the distance partials
      // of this component are summed here too (problems/instance.hpp:127-134 up to order)
      for (int e = threadIdx.x; e < P * nqD; e += blockDim.x) {
        const int i = e / nqD, q = e - i * nqD;
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = 8 * q + j;
          if (k >= D) break;
          const double v = sZ[i * D + k];
          if (kind == EVB_RASTRIGIN) {
            s1 += sS[i * D + k];
          } else if (kind == EVB_ACKLEY) {
            s1 = fma(v, v, s1);
            s2 += sS[i * D + k];
          } else if (kind == EVB_ELLIPTIC) {
            s1 += __dmul_rn(__dmul_rn(pr.ell_w[k], v), v);
          } else {
            s1 = fma(v, v, s1);
          }
        }
        part_b[e] = s1;
        part_b[size_t(P) * nqD + e] = s2;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        double s1 = 0.0, s2 = 0.0;
        for (int q = 0; q < nqD; ++q) {
          s1 += part_b[i * nqD + q];
          s2 += part_b[size_t(P) * nqD + i * nqD + q];
        }
        sFk[i * kRunsMaxComp + c] = kind == EVB_ACKLEY ? ackley_final<double>(s1, s2, D) : s1;
        if (pr.n_comp > 0) {
          double d2 = 0.0;
          for (int q = 0; q < nqK; ++q) d2 += part_d[i * nqK + q];
          sDist[i * kRunsMaxComp + c] = d2;
        }
      }
    } else {
      if (fast && pr.n_comp > 0)  // distance partials of a component without the fast base sums
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          double d2 = 0.0;
          for (int q = 0; q < nqK; ++q) d2 += part_d[i * nqK + q];
          sDist[i * kRunsMaxComp + c] = d2;
        }
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const double* zr = sZ + i * D;
        const double* pe = sS + i * D;
        auto z = [&](int q) { return zr[q]; };
        auto pre = [&](int q) { return pe[q]; };
        sFk[i * kRunsMaxComp + c] = base_value_pre<double, false>(kind, D, z, pre, pr.ell_w);
      }
    }
    __syncthreads();
    pc.mark(5);
  }
  // the per-component raw weights (1/d) exp(-d^2 / (2 D sigma^2)) are independent: one thread per
  // (individual, component) into sS (free after the last component), bit-identical to the
  // per-individual loop; the normalisation below stays per individual
  double* sWraw = sS;  // R x 4 fits in sS when D >= 4
  const bool par_w = pr.n_comp > 0 && D >= kRunsMaxComp;
  if (par_w) {
    for (int e = threadIdx.x; e < P * pr.n_comp; e += blockDim.x) {
      const int i = e / pr.n_comp, k = e - i * pr.n_comp;
      const double dk = sDist[i * kRunsMaxComp + k];
      sWraw[i * kRunsMaxComp + k] =
          dk == 0.0 ? -1.0
                    : __dmul_rn(__ddiv_rn(1.0, __dsqrt_rn(dk)),
                                exp(__ddiv_rn(-dk, __dmul_rn(__dmul_rn(__dmul_rn(2.0, double(D)), pr.sigma[k]), pr.sigma[k]))));
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (pr.n_comp == 0) {
      f[i] = __dadd_rn(sFk[i * kRunsMaxComp], pr.bias);
      continue;
    }
    // weights exactly as problems/instance.hpp:135-171 (loops over the fixed kRunsMaxComp slots,
    // unrolled, so w[] stays in registers)
    const double* dist = sDist + i * kRunsMaxComp;
    const int nc = pr.n_comp;
    double w[kRunsMaxComp];
    int zero_count = 0;
#pragma unroll
    for (int k = 0; k < kRunsMaxComp; ++k) {
      w[k] = 0.0;
      if (k >= nc) continue;
      if (par_w) {
        w[k] = sWraw[i * kRunsMaxComp + k];
      } else {
        const double dk = dist[k];
        w[k] = dk == 0.0 ? -1.0
                         : __dmul_rn(__ddiv_rn(1.0, __dsqrt_rn(dk)),
                                     exp(__ddiv_rn(-dk, __dmul_rn(__dmul_rn(__dmul_rn(2.0, double(D)), pr.sigma[k]),
                                                                  pr.sigma[k]))));
      }
      if (w[k] < 0.0) ++zero_count;
    }
    double wsum = 0.0;
    if (zero_count > 0) {
#pragma unroll
      for (int k = 0; k < kRunsMaxComp; ++k)
        if (k < nc) w[k] = w[k] < 0.0 ? 1.0 : 0.0;
      wsum = double(zero_count);
    } else {
#pragma unroll
      for (int k = 0; k < kRunsMaxComp; ++k)
        if (k < nc) wsum = __dadd_rn(wsum, w[k]);
      if (wsum == 0.0) {
        int nearest = 0;
        for (int k = 1; k < nc; ++k)
          if (dist[k] < dist[nearest]) nearest = k;
#pragma unroll
        for (int k = 0; k < kRunsMaxComp; ++k)
          if (k == nearest) w[k] = 1.0;
        wsum = 1.0;
      }
    }
    double value = 0.0;
#pragma unroll
    for (int k = 0; k < kRunsMaxComp; ++k) {
      if (k >= nc) continue;
      const double wk = __ddiv_rn(w[k], wsum);
      if (wk == 0.0) continue;
      value = __dadd_rn(value, __dmul_rn(wk, __dadd_rn(__dmul_rn(pr.lambda[k], sFk[i * kRunsMaxComp + k]), pr.cbias[k])));
    }
    f[i] = __dadd_rn(value, pr.bias);
  }
  __syncthreads();
  pc.mark(6);
}

// With a.split == 2 the run is owned by a 2-CTA cluster: both CTAs hold the full run state and
// make the same draws, trials and selections (bit-identical, deterministic), and each evaluates
// half of the individuals; the halves of the fitness vector are exchanged through distributed
// shared memory.  The trial fitness is double-buffered by generation parity, so one cluster
// barrier per generation suffices (a CTA can only write the buffer its peer reads next).
template <bool PROF>
__global__ void __launch_bounds__(512) de_runs_kernel(const runs_args a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double sm[];
  const int P = a.P, D = a.D, S = (D % 2 == 1) ? D : D + 1;
  const int run = blockIdx.x / a.split;
  const int rank = a.split == 2 ? int(cg::this_cluster().block_rank()) : 0;
  const int half = (P + 1) / 2;
  const int p0 = a.split == 2 ? rank * half : 0;
  const int p1 = a.split == 2 ? min(P, p0 + half) : P;
  const int R = p1 - p0 > 0 ? (a.split == 2 ? half : P) : 1;  // rows this CTA evaluates
  const int NM = a.resident ? a.n_mat : 1;     // rotation / shift slots
  const int KS = a.tc ? tc_ks(D) : 0;          // tensor-core dots: operand row stride
  const size_t m_len = a.tc ? size_t(round8(D)) * KS : size_t(D) * S;  // one rotation
  const size_t s_len = a.tc ? size_t(round8(R)) * KS : size_t(R) * D;  // x - o
  auto even = [](size_t n) { return (n + 1) & ~size_t(1); };           // 16-byte sections
  double* sPop = sm;                           // P x D
  double* sTrial = sPop + even(size_t(P) * D); // P x D
  double* sM = sTrial + even(size_t(P) * D);   // NM rotations
  double* sZ = sM + even(NM * m_len);          // R x D
  double* sS = sZ + even(size_t(R) * D);       // x - o of the current component (tc: RP x KS)
  double* sO = sS + even(s_len);               // NM x D
  const size_t part_len = (a.tc && a.tc_epi) ? size_t(round8(R)) * (tc_ks(D) / 8) + 2 * size_t(R) * ((D + 7) / 8) : 0;
  double* sFit = sO + NM * D;                  // P
  double* sTfit2 = sFit + P;                   // 2 x P (generation parity)
  double* sFk = sTfit2 + 2 * P;                // R x 4
  double* sDist = sFk + R * kRunsMaxComp;      // R x 4
  double* sPart = sDist + R * kRunsMaxComp;    // fast epilogue partials (part_len)
  double* sEw = sPart + part_len;              // D: elliptic weights (the problem's, staged once)
  int* sIdx = reinterpret_cast<int*>(sEw + D);  // P x 4 (a, b, c, word offset)
  // the run's problem descriptor in shared memory (a local-memory copy lived in L1, which the
  // ~200 KB shared-memory carve-out leaves nearly empty: every field access missed to L2)
  __shared__ run_problem s_pr;
  for (int e = threadIdx.x; e < int(sizeof(run_problem) / 4); e += blockDim.x)
    reinterpret_cast<int*>(&s_pr)[e] = reinterpret_cast<const int*>(a.probs + run)[e];
  __syncthreads();
  if (s_pr.ell_w) {  // elliptic weights from shared memory (L1 is nearly all carve-out)
    for (int e = threadIdx.x; e < D; e += blockDim.x) sEw[e] = s_pr.ell_w[e];
    __syncthreads();
    if (threadIdx.x == 0) s_pr.ell_w = sEw;
    __syncthreads();
  }
  const run_problem& pr = s_pr;
  if (a.resident) {  // stage every component's rotation and shift once for all generations
    const int nc = pr.n_comp > 0 ? pr.n_comp : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int c = 0; c < nc; ++c) {
      if (a.tc) {  // round8(D) x KS, zero pads
        const int NP8 = round8(D);
        for (int r = warp; r < NP8; r += nwarps)
          for (int k = lane; k < KS; k += 32)
            sM[c * m_len + size_t(r) * KS + k] = (r < D && k < D) ? pr.rot[c][r * pr.ld + k] : 0.0;
      } else {
        for (int r = warp; r < D; r += nwarps)
          for (int k = lane; k < D; k += 32) sM[(size_t(c) * D + r) * S + k] = pr.rot[c][r * pr.ld + k];
      }
      for (int e = threadIdx.x; e < D; e += blockDim.x) sO[c * D + e] = pr.shift[c][e];
    }
    __syncthreads();
  }
  const uint64_t key = a.keys[run];
  double* gpop = a.pop + size_t(run) * P * D;
  double* gfit = a.fit + size_t(run) * P;
  phase_clock<PROF> pc{blockIdx.x == 0 ? a.prof : nullptr, 0};
  // evaluate rows [p0, p1) of X into f
  auto evaluate = [&](const double* X, double* f) {
    runs_evaluate<PROF>(pr, X + size_t(p0) * D, p1 - p0, D, S, sM, sZ, sS, sO, sFk, sDist, f + p0, a.resident != 0, KS, a.tc_epi, sPart, pc);
  };
  // (split) publish this CTA's rows [p0, p1) of the given arrays into the peer's copies
  auto publish = [&](double* rows, int row_len) {
    cg::cluster_group cl = cg::this_cluster();
    double* peer = cl.map_shared_rank(rows, rank ^ 1);
    for (int e = int(threadIdx.x); e < (p1 - p0) * row_len; e += blockDim.x)
      peer[size_t(p0) * row_len + e] = rows[size_t(p0) * row_len + e];
  };
  if (a.split == 2) cg::this_cluster().sync();  // the peer's shared memory exists from here on

  if (a.init) {  // init_population (core/population.hpp:88-98), sub-stream kSubInit of gen0
    const uint64_t ctr = (uint64_t(a.gen0) << 32) | kSubInit;
    for (int e = threadIdx.x; e < P * D; e += blockDim.x)
      sPop[e] = __dadd_rn(a.lb, __dmul_rn(__dsub_rn(a.ub, a.lb), u01_of(philox_word(key, ctr, uint64_t(e)))));  // once
    __syncthreads();
    evaluate(sPop, sFit);
    if (a.split == 2) {
      publish(sFit, 1);
      cg::this_cluster().sync();
    }
    if (a.rec_on && rank == 0 && threadIdx.x == 0) rec_observe_seq<double>(a.rec, run, sFit, P);
  } else {
    for (int e = threadIdx.x; e < P * D; e += blockDim.x) sPop[e] = gpop[e];
    for (int i = threadIdx.x; i < P; i += blockDim.x) sFit[i] = gfit[i];
    __syncthreads();
  }
  const uint32_t g_first = a.gen0 + (a.init ? 1u : 0u);
  pc.start();
  for (int g = 0; g < a.G; ++g) {
    const uint32_t gen = g_first + uint32_t(g);
    double* sTfit = sTfit2 + (g & 1) * P;
    // best/1: fitness_order()[0] (core/population.hpp:70-77) under the engine's order kernel's
    // (fitness, index) order with NaN after every number (de_best_kernel, de.cu): the (fitness,
    // index) minimum over the non-NaN entries, index 0 when every entry is NaN; by warp 0 with a
    // shuffle tree, once per generation for the whole CTA
    __shared__ int s_best;
    if (a.mutation != EVB_MUT_RAND1) {
      if (threadIdx.x < 32) {
        double bf = 0.0;
        int bi = -1;
        for (int q = int(threadIdx.x); q < P; q += 32) {
          const double fq = sFit[q];
          if (!isnan(fq) && (bi < 0 || fq < bf)) {  // strided: q increases, ties keep the lower
            bf = fq;
            bi = q;
          }
        }
        for (int off = 16; off > 0; off >>= 1) {
          const double of = __shfl_xor_sync(0xffffffffu, bf, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (oi >= 0 && (bi < 0 || of < bf || (of == bf && oi < bi))) {
            bf = of;
            bi = oi;
          }
        }
        if (threadIdx.x == 0) s_best = bi < 0 ? 0 : bi;
      }
      __syncthreads();
    }
    // draws (thread per individual of this CTA's half)
    for (int i = p0 + int(threadIdx.x); i < p1; i += blockDim.x) {
      philox_prefetch_reader<4> r(key, (uint64_t(gen) << 32) | uint32_t(i));
      int x1, x2, x3;
      if (a.mutation == EVB_MUT_RAND1) {
        do { x1 = draw_int(r, P); } while (x1 == i);
        do { x2 = draw_int(r, P); } while (x2 == i || x2 == x1);
        do { x3 = draw_int(r, P); } while (x3 == i || x3 == x1 || x3 == x2);
      } else {  // best/1: best = first strict minimum (fitness_order[0]), s_best above
        x1 = s_best;
        do { x2 = draw_int(r, P); } while (x2 == i);
        do { x3 = draw_int(r, P); } while (x3 == i || x3 == x2);
      }
      const int jr = draw_int(r, D);
      sIdx[4 * i + 0] = x1;
      sIdx[4 * i + 1] = x2;
      sIdx[4 * i + 2] = x3;
      sIdx[4 * i + 3] = (int(r.count) << 16) | jr;  // gene words start after the scalar words
    }
    __syncthreads();
    pc.mark(0);
    // trial: thread per (individual of this half, Philox block = two gene words), flattened over
    // the half so that small D still fills the CTA (a warp per individual left most lanes idle at
    // D = 10 and serialised the Philox chains)
    {
      const int NB = D / 2 + 1;  // blocks an individual's D gene words can touch
      for (int e = int(threadIdx.x); e < (p1 - p0) * NB; e += blockDim.x) {
        const int i = p0 + e / NB, q = e % NB;
        const int packed = sIdx[4 * i + 3];
        const int s0 = packed >> 16, jr = packed & 0xFFFF;
        const int blk0 = s0 >> 1, nblk = ((s0 + D + 1) >> 1) - blk0;
        if (q >= nblk) continue;
        const double* xa = sPop + sIdx[4 * i] * D;
        const double* xb = sPop + sIdx[4 * i + 1] * D;
        const double* xc = sPop + sIdx[4 * i + 2] * D;
        const uint64_t ctr = (uint64_t(gen) << 32) | uint32_t(i);
        {
          uint64_t w0, w1;
          philox_pair(key, ctr, uint64_t(blk0 + q), w0, w1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 2 * (blk0 + q) + h - s0;
            if (j < 0 || j >= D) continue;
            const double u = u01_of(h ? w1 : w0);
            const double xi = sPop[i * D + j];
            double v = xi;
            if (u < a.CR || j == jr) v = __dadd_rn(xa[j], __dmul_rn(a.F, __dsub_rn(xb[j], xc[j])));
            sTrial[i * D + j] = clip_or_mid(v, xi, a.lb, a.ub, a.repair);
          }
        }
      }
    }
    __syncthreads();
    pc.mark(1);
    evaluate(sTrial, sTfit);
    // selection on this half (de/engine.hpp:36: replace when f_trial <= f_parent)
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
      for (int i = p0 + warp; i < p1; i += nwarps)
        if (sTfit[i] <= sFit[i])
          for (int j = lane; j < D; j += 32) sPop[i * D + j] = sTrial[i * D + j];
    }
    __syncthreads();
    for (int i = p0 + int(threadIdx.x); i < p1; i += blockDim.x)
      if (sTfit[i] <= sFit[i]) sFit[i] = sTfit[i];
    __syncthreads();
    pc.mark(8);
    if (a.split == 2) {
      // the peer has finished reading this half's rows (its trials) once it reaches the barrier;
      // then both halves cross over and the second barrier publishes them
      cg::this_cluster().sync();
      publish(sPop, D);
      publish(sFit, 1);
      publish(sTfit, 1);
      cg::this_cluster().sync();
      pc.mark(7);
    }
    if (a.rec_on && rank == 0 && threadIdx.x == 0) rec_observe_seq<double>(a.rec, run, sTfit, P);  // trials, i order
  }
  if (rank == 0) {
    for (int e = threadIdx.x; e < P * D; e += blockDim.x) gpop[e] = sPop[e];
    for (int i = threadIdx.x; i < P; i += blockDim.x) gfit[i] = sFit[i];
  }
  if (a.split == 2) cg::this_cluster().sync();  // no CTA leaves while its peer may still write into it
}

// ---- fused variant (config 4's shape) -------------------------------------------------------
// For runs whose components are all sphere / elliptic / Rastrigin / Ackley (base problem or
// composition, D >= 32) the generation needs five block barriers instead of ~20:
//   draws | trial | contraction + terms | values | selection + exchange
// - the trial rows of this CTA's half live in the tensor-core layout (R8 x KS, zero pads); the
//   A fragment is formed as x - o while it is loaded (rounded like transform_input's diff,
//   problems/instance.hpp:66-67), so no s = x - o copy exists and the three components'
//   contractions are ONE phase of (component, row tile, column tile) warp tasks;
// - each task keeps its 8 x 16 accumulators in registers, applies the component's per-element
//   term there (cos2pi_fast for Rastrigin / Ackley), reduces over the quad and writes one
//   partial per (row, column tile, channel); the column-tile-0 task also forms the row's
//   ||x - o||^2 from the A fragments it loads anyway;
// - values: four adjacent lanes per individual (lane k = component k) sum the partials, form the
//   base value and the raw weight, exchange them by shuffles and lane 0 normalises exactly as
//   problems/instance.hpp:135-171;
// - selection writes a winner's row into this CTA's and the peer's population copy; the two
//   cluster barriers are split into arrive / wait (arrive after the trial phase = "my reads of
//   the population are done", wait before the remote writes; arrive after them, wait at the top
//   of the next generation), so neither CTA idles at a cluster barrier unless its peer is late.
// Tolerance path like the tensor-core path above (fitness ~1e-15 relative, selections equal
// except flagged near-ties).
__host__ __device__ __forceinline__ bool fused_kind(int k) {
  return k == EVB_SPHERE || k == EVB_ELLIPTIC || k == EVB_RASTRIGIN || k == EVB_ACKLEY;
}

struct fused_layout {
  int R, R8, KS, D8, NT, NM;
  size_t pop, tr, m, o, fit, partb, partd, ew, idx, bytes;  // offsets in doubles (idx too)
};
__host__ __device__ inline fused_layout fused_make_layout(int P, int D, int split, int n_mat) {
  fused_layout L;
  auto even = [](size_t n) { return (n + 1) & ~size_t(1); };
  L.R = split == 2 ? (P + 1) / 2 : P;
  L.R8 = round8(L.R);
  L.KS = tc_ks(D);
  L.D8 = round8(D);
  L.NT = (D + 15) / 16;
  L.NM = n_mat;
  size_t off = 0;
  L.pop = off;   off += even(size_t(P) * D);
  L.tr = off;    off += size_t(L.R8) * L.KS;
  L.m = off;     off += size_t(n_mat) * L.D8 * L.KS;
  L.o = off;     off += size_t(n_mat) * L.KS;
  L.fit = off;   off += even(3 * size_t(P));
  L.partb = off; off += even(size_t(n_mat) * 2 * L.R8 * L.NT);
  L.partd = off; off += even(size_t(n_mat) * L.R8);
  L.ew = off;    off += size_t(L.KS);
  L.idx = off;   off += even(size_t(P) * 4) / 2;  // 4 ints per individual
  L.bytes = off * sizeof(double);
  return L;
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// contraction + terms for the rows of sTr (rows < nrows are real): partials into sPartB / sPartD
__device__ __forceinline__ void fused_contract(const run_problem& pr, const fused_layout& L, int D, int nrows,
                                               const double* __restrict__ sTr, const double* __restrict__ sM,
                                               const double* __restrict__ sO, const double* __restrict__ sEw,
                                               double* __restrict__ sPartB, double* __restrict__ sPartD) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nc = pr.n_comp > 0 ? pr.n_comp : 1;
  const int mt = L.R8 >> 3, KS = L.KS;
  const size_t m_len = size_t(L.D8) * KS;
  const int ntasks = nc * mt * L.NT;
  const float inv_mt = 1.0f / float(mt), inv_nc = 1.0f / float(nc);
  for (int task = warp; task < ntasks; task += nwarps) {
    // column tile slowest (the narrow last tile's short tasks come last), row tile fastest
    // (small non-negative ints: the float quotient of (n + 0.5) is exact after truncation)
    const int rest = int((float(task) + 0.5f) * inv_mt);
    const int mi = task - rest * mt;
    const int ni = int((float(rest) + 0.5f) * inv_nc);
    const int c = rest - ni * nc;
    const int m0 = mi << 3, n0 = ni << 4;
    const bool two = n0 + 8 < D;  // warp-uniform
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0, d2 = 0.0;
    const double* pa = sTr + (m0 + g) * KS + 2 * t;
    const double* po = sO + c * KS + 2 * t;
    const double* pb = sM + c * m_len + size_t(n0 + g) * KS + 2 * t;
    if (two) {
      const double* pb1 = pb + 8 * KS;
#pragma unroll 7
      for (int k0 = 0; k0 < KS; k0 += 8) {
        const double2 x = *reinterpret_cast<const double2*>(pa + k0);
        const double2 o = *reinterpret_cast<const double2*>(po + k0);
        const double2 b0 = *reinterpret_cast<const double2*>(pb + k0);
        const double2 b1 = *reinterpret_cast<const double2*>(pb1 + k0);
        const double ax = __dsub_rn(x.x, o.x), ay = __dsub_rn(x.y, o.y);
        ptx::dmma_8x8x4(c00, c01, ax, b0.x);
        ptx::dmma_8x8x4(c10, c11, ax, b1.x);
        ptx::dmma_8x8x4(c00, c01, ay, b0.y);
        ptx::dmma_8x8x4(c10, c11, ay, b1.y);
        if (ni == 0) d2 = fma(ay, ay, fma(ax, ax, d2));
      }
    } else {
#pragma unroll 7
      for (int k0 = 0; k0 < KS; k0 += 8) {
        const double2 x = *reinterpret_cast<const double2*>(pa + k0);
        const double2 o = *reinterpret_cast<const double2*>(po + k0);
        const double2 b0 = *reinterpret_cast<const double2*>(pb + k0);
        const double ax = __dsub_rn(x.x, o.x), ay = __dsub_rn(x.y, o.y);
        ptx::dmma_8x8x4(c00, c01, ax, b0.x);
        ptx::dmma_8x8x4(c00, c01, ay, b0.y);
        if (ni == 0) d2 = fma(ay, ay, fma(ax, ax, d2));
      }
    }
    // per-element terms on the accumulators (problems/batch.hpp:96-183 per kind); the four
    // elements of a lane are evaluated side by side (one warp-uniform switch on the kind, no
    // per-element branches), so their polynomial chains overlap
    const int kind = pr.kind[c];
    const int col = n0 + 2 * t;
    const bool v0 = col < D, v1 = col + 1 < D, v2 = two && col + 8 < D, v3 = two && col + 9 < D;
    double s1, s2 = 0.0;
    if (kind == EVB_ELLIPTIC) {
      const double w0 = v0 ? sEw[col] : 0.0, w1 = v1 ? sEw[col + 1] : 0.0;
      const double w2 = v2 ? sEw[col + 8] : 0.0, w3 = v3 ? sEw[col + 9] : 0.0;
      s1 = (__dmul_rn(__dmul_rn(w0, c00), c00) + __dmul_rn(__dmul_rn(w1, c01), c01)) +
           (__dmul_rn(__dmul_rn(w2, c10), c10) + __dmul_rn(__dmul_rn(w3, c11), c11));
    } else if (kind == EVB_SPHERE) {
      s1 = fma(c11, c11, fma(c10, c10, fma(c01, c01, c00 * c00)));  // pad columns hold exact zeros
    } else {
      double z0, z1, z2, z3;
      if (cos2pi_fast_ok(c00) && cos2pi_fast_ok(c01) && cos2pi_fast_ok(c10) && cos2pi_fast_ok(c11)) {
        z0 = cos2pi_fast(c00);
        z1 = cos2pi_fast(c01);
        z2 = cos2pi_fast(c10);
        z3 = cos2pi_fast(c11);
      } else {  // out of the fast form's range (or not finite): the reference's expression
        z0 = cos(__dmul_rn(two_pi_v<double>(), c00));
        z1 = cos(__dmul_rn(two_pi_v<double>(), c01));
        z2 = cos(__dmul_rn(two_pi_v<double>(), c10));
        z3 = cos(__dmul_rn(two_pi_v<double>(), c11));
      }
      if (kind == EVB_ACKLEY) {
        s1 = fma(c11, c11, fma(c10, c10, fma(c01, c01, c00 * c00)));
        s2 = ((v0 ? z0 : 0.0) + (v1 ? z1 : 0.0)) + ((v2 ? z2 : 0.0) + (v3 ? z3 : 0.0));
      } else {
        const double r0 = __dadd_rn(__dsub_rn(__dmul_rn(c00, c00), __dmul_rn(10.0, z0)), 10.0);
        const double r1 = __dadd_rn(__dsub_rn(__dmul_rn(c01, c01), __dmul_rn(10.0, z1)), 10.0);
        const double r2 = __dadd_rn(__dsub_rn(__dmul_rn(c10, c10), __dmul_rn(10.0, z2)), 10.0);
        const double r3 = __dadd_rn(__dsub_rn(__dmul_rn(c11, c11), __dmul_rn(10.0, z3)), 10.0);
        s1 = ((v0 ? r0 : 0.0) + (v1 ? r1 : 0.0)) + ((v2 ? r2 : 0.0) + (v3 ? r3 : 0.0));
      }
    }
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    if (kind == EVB_ACKLEY) {
      s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
      s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
    }
    if (ni == 0) {
      d2 += __shfl_xor_sync(0xffffffffu, d2, 1);
      d2 += __shfl_xor_sync(0xffffffffu, d2, 2);
    }
    const int row = m0 + g;
    if (t == 0 && row < nrows) {
      sPartB[(size_t(c) * 2 * L.R8 + row) * L.NT + ni] = s1;
      sPartB[(size_t(c) * 2 * L.R8 + L.R8 + row) * L.NT + ni] = s2;
      if (ni == 0) sPartD[c * L.R8 + row] = d2;
    }
  }
}

// values of the nrows individuals from the partials: f[i], i < nrows
__device__ __forceinline__ void fused_values(const run_problem& pr, const fused_layout& L, int D, int nrows,
                                             const double* __restrict__ sPartB, const double* __restrict__ sPartD,
                                             double* __restrict__ f) {
  const int nc = pr.n_comp > 0 ? pr.n_comp : 1;
  const int lane = threadIdx.x & 31;
  const int bound = (nrows * kRunsMaxComp + 31) & ~31;  // whole warps: the quad exchanges use shuffles
  for (int e = threadIdx.x; e < bound; e += blockDim.x) {
    const int i = e >> 2, k = e & 3;
    const bool live = i < nrows && k < nc;
    double fk = 0.0, dk = 0.0, wr = 0.0;
    if (live) {
      double s1 = 0.0, s2 = 0.0;
      const double* p1 = sPartB + (size_t(k) * 2 * L.R8 + i) * L.NT;
      const double* p2 = p1 + size_t(L.R8) * L.NT;
      for (int q = 0; q < L.NT; ++q) {
        s1 += p1[q];
        s2 += p2[q];
      }
      fk = pr.kind[k] == EVB_ACKLEY ? ackley_final<double>(s1, s2, D) : s1;
      if (pr.n_comp > 0) {
        dk = sPartD[k * L.R8 + i];
        wr = dk == 0.0 ? -1.0
                       : __dmul_rn(__ddiv_rn(1.0, __dsqrt_rn(dk)),
                                   exp(__ddiv_rn(-dk, __dmul_rn(__dmul_rn(__dmul_rn(2.0, double(D)), pr.sigma[k]), pr.sigma[k]))));
      }
    }
    double w[kRunsMaxComp], fks[kRunsMaxComp], dist[kRunsMaxComp];
#pragma unroll
    for (int q = 0; q < kRunsMaxComp; ++q) {
      const int src = (lane & ~3) + q;
      w[q] = __shfl_sync(0xffffffffu, wr, src);
      fks[q] = __shfl_sync(0xffffffffu, fk, src);
      dist[q] = __shfl_sync(0xffffffffu, dk, src);
    }
    if (k != 0 || i >= nrows) continue;
    if (pr.n_comp == 0) {
      f[i] = __dadd_rn(fks[0], pr.bias);
      continue;
    }
    // weights exactly as problems/instance.hpp:135-171
    int zero_count = 0;
#pragma unroll
    for (int q = 0; q < kRunsMaxComp; ++q)
      if (q < nc && w[q] < 0.0) ++zero_count;
    double wsum = 0.0;
    if (zero_count > 0) {
#pragma unroll
      for (int q = 0; q < kRunsMaxComp; ++q)
        if (q < nc) w[q] = w[q] < 0.0 ? 1.0 : 0.0;
      wsum = double(zero_count);
    } else {
#pragma unroll
      for (int q = 0; q < kRunsMaxComp; ++q)
        if (q < nc) wsum = __dadd_rn(wsum, w[q]);
      if (wsum == 0.0) {
        int nearest = 0;
        double dn = dist[0];
#pragma unroll
        for (int q = 1; q < kRunsMaxComp; ++q)
          if (q < nc && dist[q] < dn) {
            dn = dist[q];
            nearest = q;
          }
#pragma unroll
        for (int q = 0; q < kRunsMaxComp; ++q)
          if (q == nearest) w[q] = 1.0;
        wsum = 1.0;
      }
    }
    double value = 0.0;
#pragma unroll
    for (int q = 0; q < kRunsMaxComp; ++q) {
      if (q >= nc) continue;
      const double wq = __ddiv_rn(w[q], wsum);
      if (wq == 0.0) continue;
      value = __dadd_rn(value, __dmul_rn(wq, __dadd_rn(__dmul_rn(pr.lambda[q], fks[q]), pr.cbias[q])));
    }
    f[i] = __dadd_rn(value, pr.bias);
  }
}

template <bool PROF>
__global__ void __launch_bounds__(512) de_runs_fused_kernel(const runs_args a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double sm[];
  const int P = a.P, D = a.D;
  const bool split = a.split == 2;
  const int run = blockIdx.x / a.split;
  const int rank = split ? int(cg::this_cluster().block_rank()) : 0;
  const fused_layout L = fused_make_layout(P, D, a.split, a.n_mat);
  const int p0 = split ? rank * L.R : 0;
  const int p1 = split ? min(P, p0 + L.R) : P;
  const int nrows = p1 - p0;
  const int KS = L.KS;
  double* sPop = sm + L.pop;
  double* sTr = sm + L.tr;
  double* sM = sm + L.m;
  double* sO = sm + L.o;
  double* sFit = sm + L.fit;
  double* sTfit2 = sFit + P;
  double* sPartB = sm + L.partb;
  double* sPartD = sm + L.partd;
  double* sEw = sm + L.ew;
  int* sIdx = reinterpret_cast<int*>(sm + L.idx);
  __shared__ run_problem s_pr;
  for (int e = threadIdx.x; e < int(sizeof(run_problem) / 4); e += blockDim.x)
    reinterpret_cast<int*>(&s_pr)[e] = reinterpret_cast<const int*>(a.probs + run)[e];
  __syncthreads();
  const run_problem& pr = s_pr;
  {  // resident operands in the tensor-core layout (zero pads), trial pads zero once
    const int nc = pr.n_comp > 0 ? pr.n_comp : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const size_t m_len = size_t(L.D8) * KS;
    for (int c = 0; c < nc; ++c) {
      for (int r = warp; r < L.D8; r += nwarps)
        for (int k = lane; k < KS; k += 32)
          sM[c * m_len + size_t(r) * KS + k] = (r < D && k < D) ? pr.rot[c][r * pr.ld + k] : 0.0;
      for (int e = threadIdx.x; e < KS; e += blockDim.x) sO[c * KS + e] = e < D ? pr.shift[c][e] : 0.0;
    }
    for (int e = threadIdx.x; e < KS; e += blockDim.x) sEw[e] = (pr.ell_w && e < D) ? pr.ell_w[e] : 0.0;
    for (int e = threadIdx.x; e < L.R8 * KS; e += blockDim.x) sTr[e] = 0.0;
  }
  __syncthreads();
  const uint64_t key = a.keys[run];
  double* gpop = a.pop + size_t(run) * P * D;
  double* gfit = a.fit + size_t(run) * P;
  phase_clock<PROF> pc{blockIdx.x == 0 ? a.prof : nullptr, 0};
  cg::cluster_group cl = cg::this_cluster();
  double* peerPop = split ? cl.map_shared_rank(sPop, rank ^ 1) : nullptr;
  double* peerFit = split ? cl.map_shared_rank(sFit, rank ^ 1) : nullptr;
  if (split) cl.sync();  // the peer's shared memory exists from here on

  if (a.init) {  // init_population (core/population.hpp:88-98), sub-stream kSubInit of gen0
    const uint64_t ctr = (uint64_t(a.gen0) << 32) | kSubInit;
    for (int e = threadIdx.x; e < P * D; e += blockDim.x)
      sPop[e] = __dadd_rn(a.lb, __dmul_rn(__dsub_rn(a.ub, a.lb), u01_of(philox_word(key, ctr, uint64_t(e)))));
    __syncthreads();
    for (int e = threadIdx.x; e < nrows * D; e += blockDim.x) {
      const int i = e / D, j = e - i * D;
      sTr[i * KS + j] = sPop[(p0 + i) * D + j];
    }
    __syncthreads();
    fused_contract(pr, L, D, nrows, sTr, sM, sO, sEw, sPartB, sPartD);
    __syncthreads();
    fused_values(pr, L, D, nrows, sPartB, sPartD, sFit + p0);
    __syncthreads();
    if (split) {
      for (int i = p0 + int(threadIdx.x); i < p1; i += blockDim.x) peerFit[i] = sFit[i];
      cl.sync();
    }
    if (a.rec_on && rank == 0 && threadIdx.x == 0) rec_observe_seq<double>(a.rec, run, sFit, P);
  } else {
    for (int e = threadIdx.x; e < P * D; e += blockDim.x) sPop[e] = gpop[e];
    for (int i = threadIdx.x; i < P; i += blockDim.x) sFit[i] = gfit[i];
    __syncthreads();
  }
  const uint32_t g_first = a.gen0 + (a.init ? 1u : 0u);
  const bool rand1 = a.mutation == EVB_MUT_RAND1;
  __shared__ int s_best;
  // individual i's scalar draws of generation gen (de/strategy.hpp:84-86, 187) into sIdx
  auto draw_individual = [&](int i, uint32_t gen) {
    philox_prefetch_reader<4> r(key, (uint64_t(gen) << 32) | uint32_t(i));
    int x1, x2, x3;
    if (rand1) {
      do { x1 = draw_int(r, P); } while (x1 == i);
      do { x2 = draw_int(r, P); } while (x2 == i || x2 == x1);
      do { x3 = draw_int(r, P); } while (x3 == i || x3 == x1 || x3 == x2);
    } else {  // best/1: best = first strict minimum (fitness_order[0]), s_best
      x1 = s_best;
      do { x2 = draw_int(r, P); } while (x2 == i);
      do { x3 = draw_int(r, P); } while (x3 == i || x3 == x2);
    }
    const int jr = draw_int(r, D);
    sIdx[4 * i + 0] = x1;
    sIdx[4 * i + 1] = x2;
    sIdx[4 * i + 2] = x3;
    sIdx[4 * i + 3] = (int(r.count) << 16) | jr;  // gene words start after the scalar words
  };
  // rand/1 draws depend on (key, generation, individual) only: generation g + 1's are made by
  // the upper warps while the lower ones form generation g's values (the first ones here)
  if (rand1 && a.G > 0) {
    for (int i = p0 + int(threadIdx.x); i < p1; i += blockDim.x) draw_individual(i, g_first);
    __syncthreads();
  }
  const take_rule_host take = a.take;
  pc.start();
  for (int g = 0; g < a.G; ++g) {
    const uint32_t gen = g_first + uint32_t(g);
    double* sTfit = sTfit2 + (g & 1) * P;
    if (a.mutation != EVB_MUT_RAND1) {  // best/1: as de_runs_kernel
      if (threadIdx.x < 32) {
        double bf = 0.0;
        int bi = -1;
        for (int q = int(threadIdx.x); q < P; q += 32) {
          const double fq = sFit[q];
          if (!isnan(fq) && (bi < 0 || fq < bf)) {
            bf = fq;
            bi = q;
          }
        }
        for (int off = 16; off > 0; off >>= 1) {
          const double of = __shfl_xor_sync(0xffffffffu, bf, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (oi >= 0 && (bi < 0 || of < bf || (of == bf && oi < bi))) {
            bf = of;
            bi = oi;
          }
        }
        if (threadIdx.x == 0) s_best = bi < 0 ? 0 : bi;
      }
      __syncthreads();
    }
    if (!rand1) {
      for (int i = p0 + int(threadIdx.x); i < p1; i += blockDim.x) draw_individual(i, gen);
      __syncthreads();
    }
    pc.mark(0);
    {  // trial rows of this half into the tensor-core layout
      const int NB = D / 2 + 1;
      const float inv_nb = 1.0f / float(NB);
      for (int e = int(threadIdx.x); e < nrows * NB; e += blockDim.x) {
        const int il = int((float(e) + 0.5f) * inv_nb), q = e - il * NB, i = p0 + il;
        const int packed = sIdx[4 * i + 3];
        const int s0 = packed >> 16, jr = packed & 0xFFFF;
        const int blk0 = s0 >> 1, nblk = ((s0 + D + 1) >> 1) - blk0;
        if (q >= nblk) continue;
        const double* xa = sPop + sIdx[4 * i] * D;
        const double* xb = sPop + sIdx[4 * i + 1] * D;
        const double* xc = sPop + sIdx[4 * i + 2] * D;
        uint64_t w0, w1;
        philox_pair(key, (uint64_t(gen) << 32) | uint32_t(i), uint64_t(blk0 + q), w0, w1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = 2 * (blk0 + q) + h - s0;
          if (j < 0 || j >= D) continue;
          const double xi = sPop[i * D + j];
          double v = xi;
          if (take.bit(h ? w1 : w0) || j == jr) v = __dadd_rn(xa[j], __dmul_rn(a.F, __dsub_rn(xb[j], xc[j])));
          sTr[il * KS + j] = clip_or_mid(v, xi, a.lb, a.ub, a.repair);
        }
      }
    }
    __syncthreads();
    if (split) cluster_arrive();  // this CTA's reads of the population / fitness copies are done
    pc.mark(1);
    fused_contract(pr, L, D, nrows, sTr, sM, sO, sEw, sPartB, sPartD);
    __syncthreads();
    pc.mark(3);
    fused_values(pr, L, D, nrows, sPartB, sPartD, sTfit + p0);
    if (rand1 && g + 1 < a.G && threadIdx.x >= 256) {  // warps 8-15: individual il = 8 lane + (warp - 8)
      for (int il = 8 * int(threadIdx.x & 31) + (int(threadIdx.x >> 5) - 8); il < nrows; il += 256)
        draw_individual(p0 + il, gen + 1);
    }
    __syncthreads();
    pc.mark(6);
    if (split) cluster_wait();  // the peer's reads are done too: its copies may be written
    pc.mark(7);
    {  // selection on this half (de/engine.hpp:36), winners into both copies
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
      for (int i = p0 + warp; i < p1; i += nwarps) {
        const double ft = sTfit[i];
        if (split && lane == 0) cl.map_shared_rank(sTfit, rank ^ 1)[i] = ft;
        if (ft <= sFit[i]) {
          const double* src = sTr + (i - p0) * KS;
          for (int j = lane; j < D; j += 32) {
            const double v = src[j];
            sPop[i * D + j] = v;
            if (split) peerPop[i * D + j] = v;
          }
          __syncwarp();
          if (lane == 0) {
            sFit[i] = ft;
            if (split) peerFit[i] = ft;
          }
        }
      }
    }
    if (split) {
      cluster_arrive();
      cluster_wait();
    } else {
      __syncthreads();
    }
    pc.mark(8);
    if (a.rec_on && rank == 0 && threadIdx.x == 0) rec_observe_seq<double>(a.rec, run, sTfit, P);  // trials, i order
  }
  if (rank == 0) {
    for (int e = threadIdx.x; e < P * D; e += blockDim.x) gpop[e] = sPop[e];
    for (int i = threadIdx.x; i < P; i += blockDim.x) gfit[i] = sFit[i];
  }
  if (split) cl.sync();  // no CTA leaves while its peer may still write into it
}

size_t runs_smem(int P, int D, int split = 1, int n_mat = 1, int tc = 0) {
  const int S = (D % 2 == 1) ? D : D + 1;
  const size_t R = split == 2 ? size_t((P + 1) / 2) : size_t(P);
  auto even = [](size_t n) { return (n + 1) & ~size_t(1); };
  const size_t m_len = tc ? size_t(round8(D)) * tc_ks(D) : size_t(D) * S;
  const size_t s_len = tc ? size_t(round8(int(R))) * tc_ks(D) : R * D;
  const size_t part_len = tc ? size_t(round8(int(R))) * (tc_ks(D) / 8) + 2 * R * ((D + 7) / 8) : 0;
  return sizeof(double) * (2 * even(size_t(P) * D) + even(size_t(n_mat) * m_len) + even(R * D) + even(s_len) +
                           size_t(n_mat) * D + 3 * P + 2 * R * kRunsMaxComp + part_len + D) +
         sizeof(int) * 4 * P + 64;
}

}  // namespace
}  // namespace evb

namespace evb {
// Empty when the persistent runs kernel can execute this configuration, else the reason.
std::string runs_kernel_unsupported(int dtype, const evb_de_config* cfg, int pop_size, int dim,
                                    const evb_problem* problems, int n_runs) {
  if (dtype != EVB_F64) return "de_runs: the persistent runs kernel is fp64";
  if (cfg->mutation != EVB_MUT_RAND1 && cfg->mutation != EVB_MUT_BEST1)
    return "de_runs: persistent kernel supports rand_1 / best_1 mutation";
  if (cfg->parameter != EVB_PAR_FIXED) return "de_runs: persistent kernel supports the fixed adapter";
  if (cfg->archive_rate != 0.0) return "de_runs: persistent kernel runs without an archive";
  if (cfg->reduction != EVB_POP_FIXED) return "de_runs: persistent kernel runs a fixed population size";
  if (cfg->repair != EVB_REP_CLIP && cfg->repair != EVB_REP_MIDPOINT_TARGET) return "de_runs: clip or midpoint repair";
  if (cfg->crossover != EVB_CX_BINOMIAL) return "de_runs: binomial crossover";
  if (!(cfg->f > 0.0 && cfg->f <= 1.0)) return "fixed_parameter: F must be in (0,1]";
  if (!(cfg->cr >= 0.0 && cfg->cr <= 1.0)) return "fixed_parameter: CR must be in [0,1]";
  if (pop_size < (cfg->mutation == EVB_MUT_RAND1 ? 4 : 3)) return "de_engine: population too small for mutation";
  if (dim < 1 || dim >= 65536) return "de_runs: bad sizes";
  if (runs_smem(pop_size, dim) > 227 * 1024)
    return "de_runs: run state does not fit in shared memory (use evb_de_generation)";
  for (int r = 0; r < n_runs; ++r) {
    const device_problem& p = problems[r]->p;
    if (p.dtype != EVB_F64 || p.dim != dim) return "de_runs: problem dtype / dim mismatch";
    if (p.spec == SPEC_COMPOSITION && p.n_comp > kRunsMaxComp) return "de_runs: at most 4 composition components";
  }
  return {};
}
}  // namespace evb

using namespace evb;

extern "C" int evb_de_runs(int dtype, const evb_de_config* cfg, int n_runs, int pop_size, int dim,
                           const evb_problem* problems, const uint64_t* keys, int generations, double lb, double ub,
                           void* pops, void* fits, int init, uint32_t gen0, evb_recorder rec, void* stream) {
  return guarded([&] {
    require(cfg && problems && keys && pops && fits, "de_runs: null argument");
    require(n_runs >= 1 && dim >= 1 && dim < 65536 && generations >= 0, "de_runs: bad sizes");
    const std::string why = runs_kernel_unsupported(dtype, cfg, pop_size, dim, problems, n_runs);
    if (!why.empty()) throw config_error(why);
    std::vector<run_problem> rp(n_runs);
    for (int r = 0; r < n_runs; ++r) {
      const device_problem& p = problems[r]->p;
      run_problem& q = rp[r];
      q.bias = p.bias;
      q.ld = p.ld;
      q.ell_w = static_cast<const double*>(p.ell_w);
      q.hybrid = p.spec == SPEC_HYBRID ? 1 : 0;
      if (q.hybrid) {
        q.n_chunks = p.n_chunks;
        q.perm = p.perm;
        q.sub_kinds = p.sub_kinds;
        q.chunk_sizes = p.chunk_sizes;
        q.hyb_w = static_cast<const double*>(p.hyb_w);
      }
      if (p.spec != SPEC_COMPOSITION) {
        q.n_comp = 0;
        q.shift[0] = static_cast<const double*>(p.shift);
        q.rot[0] = static_cast<const double*>(p.rotation);
        q.kind[0] = p.kind;
      } else {
        q.n_comp = p.n_comp;
        const std::vector<int>& kinds = p.h_comp_kinds;  // host copies made at creation
        const std::vector<double>& sg = p.h_comp_sigma;
        const std::vector<double>& la = p.h_comp_lambda;
        const std::vector<double>& cb = p.h_comp_bias;
        for (int c = 0; c < p.n_comp; ++c) {
          q.shift[c] = static_cast<const double*>(p.comp_shift) + size_t(c) * p.ld;
          q.rot[c] = static_cast<const double*>(p.comp_rot) + size_t(c) * dim * p.ld;
          q.kind[c] = kinds[c];
          q.sigma[c] = sg[c];
          q.lambda[c] = la[c];
          q.cbias[c] = cb[c];
        }
      }
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the run table and keys in a per-thread device buffer reused across calls (a call on another
    // stream first waits for the previous launch that read it)
    struct table_cache {
      void* buf = nullptr;
      size_t cap = 0;
      cudaEvent_t done = nullptr;
    };
    static thread_local table_cache tc_;
    const size_t tbytes = (sizeof(run_problem) * n_runs + 15) / 16 * 16 + sizeof(uint64_t) * n_runs;
    if (!tc_.done) EVB_CUDA(cudaEventCreateWithFlags(&tc_.done, cudaEventDisableTiming));
    EVB_CUDA(cudaStreamWaitEvent(st, tc_.done, 0));
    if (tc_.cap < tbytes) {
      EVB_CUDA(cudaEventSynchronize(tc_.done));
      if (tc_.buf) EVB_CUDA(cudaFree(tc_.buf));
      tc_.buf = nullptr;
      tc_.cap = 0;
      EVB_CUDA(cudaMalloc(&tc_.buf, tbytes));
      tc_.cap = tbytes;
    }
    run_problem* dprobs = static_cast<run_problem*>(tc_.buf);
    uint64_t* dkeys = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(tc_.buf) +
                                                  (sizeof(run_problem) * n_runs + 15) / 16 * 16);
    EVB_CUDA(cudaMemcpyAsync(dprobs, rp.data(), sizeof(run_problem) * n_runs, cudaMemcpyHostToDevice, st));
    EVB_CUDA(cudaMemcpyAsync(dkeys, keys, sizeof(uint64_t) * n_runs, cudaMemcpyHostToDevice, st));
    runs_args a{};
    a.P = pop_size;
    a.D = dim;
    a.G = generations;
    a.mutation = cfg->mutation;
    a.repair = cfg->repair;
    a.F = cfg->f;
    a.CR = cfg->cr;
    a.take = take_rule_host::make(cfg->cr);
    a.lb = lb;
    a.ub = ub;
    a.probs = dprobs;
    a.keys = dkeys;
    a.gen0 = gen0;
    a.pop = static_cast<double*>(pops);
    a.fit = static_cast<double*>(fits);
    a.init = init;
    if (rec) {
      require(recorder_dtype(rec) == EVB_F64 && recorder_runs(rec) >= n_runs, "de_runs: recorder dtype / runs mismatch");
      void* running;
      int* next;
      int64_t* fes;
      int nck;
      int64_t itv;
      void* grid = recorder_view(rec, &nck, &itv, &running, &next, &fes);
      a.rec_on = 1;
      a.rec = rec_view<double>{static_cast<double*>(grid), static_cast<double*>(running), next, fes, nck, itv};
    }
    // one run per SM leaves SMs idle when there are fewer runs than SMs: then a 2-CTA cluster
    // shares each run's evaluations (EVB_RUNS_SPLIT=1|2 overrides)
    int sms = 0;
    EVB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    static const char* split_env = std::getenv("EVB_RUNS_SPLIT");
    a.split = split_env ? (std::atoi(split_env) == 2 ? 2 : 1) : (2 * n_runs <= sms ? 2 : 1);
    // keep every component's rotation resident when it fits (no per-generation reload);
    // EVB_RUNS_RESIDENT=0 forces the reload path
    a.n_mat = 1;
    for (const run_problem& q : rp) a.n_mat = std::max(a.n_mat, std::max(1, q.n_comp));
    static const char* res_env = std::getenv("EVB_RUNS_RESIDENT");
    a.resident = (!res_env || std::atoi(res_env) != 0) && runs_smem(pop_size, dim, a.split, a.n_mat) <= 227 * 1024;
    // DMMA dots (K3) for the resident layout when it fits and D is large enough for the tiles to
    // pay (EVB_RUNS_TC=0|1 overrides); small D keeps the exact-order dots
    static const char* tc_env = std::getenv("EVB_RUNS_TC");
    a.tc = a.resident && runs_smem(pop_size, dim, a.split, a.n_mat, 1) <= 227 * 1024 &&
           (tc_env ? std::atoi(tc_env) != 0 : dim >= 32);
    static const char* epi_env = std::getenv("EVB_RUNS_TC_EPI");
    a.tc_epi = a.tc && (epi_env ? std::atoi(epi_env) != 0 : 1);
    // fused generation (contraction + terms in registers, five barriers): every run a base or
    // composition problem over sphere / elliptic / Rastrigin / Ackley (EVB_RUNS_FUSED=0: off)
    static const char* fused_env = std::getenv("EVB_RUNS_FUSED");
    bool fused = a.tc && a.tc_epi && (!fused_env || std::atoi(fused_env) != 0) &&
                 fused_make_layout(pop_size, dim, a.split, a.n_mat).bytes + 64 <= 227 * 1024;
    for (const run_problem& q : rp) {
      if (q.hybrid) fused = false;
      for (int c = 0; c < std::max(1, q.n_comp); ++c)
        if (!fused_kind(q.kind[c])) fused = false;
    }
    const size_t smem = fused ? fused_make_layout(pop_size, dim, a.split, a.n_mat).bytes + 64
                              : runs_smem(pop_size, dim, a.split, a.resident ? a.n_mat : 1, a.tc);
    require(smem <= 227 * 1024, "de_runs: run state does not fit in shared memory");
    static thread_local size_t smem_set = 0;
    if (smem > smem_set) {
      EVB_CUDA(cudaFuncSetAttribute(de_runs_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      EVB_CUDA(cudaFuncSetAttribute(de_runs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      EVB_CUDA(cudaFuncSetAttribute(de_runs_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      EVB_CUDA(cudaFuncSetAttribute(de_runs_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      smem_set = smem;
    }
    static const bool prof = std::getenv("EVB_RUNS_PROFILE") != nullptr;
    unsigned long long* dprof = nullptr;
    if (prof) {
      EVB_CUDA(cudaMalloc(&dprof, 16 * sizeof(unsigned long long)));
      EVB_CUDA(cudaMemset(dprof, 0, 16 * sizeof(unsigned long long)));
    }
    a.prof = dprof;
    cudaError_t err;
    if (a.split == 2) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(2 * n_runs);
      lc.blockDim = dim3(512);
      lc.dynamicSmemBytes = smem;
      lc.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      lc.attrs = attr;
      lc.numAttrs = 1;
      auto kern = fused ? (dprof ? de_runs_fused_kernel<true> : de_runs_fused_kernel<false>)
                        : (dprof ? de_runs_kernel<true> : de_runs_kernel<false>);
      err = cudaLaunchKernelEx(&lc, kern, a);
    } else {
      if (fused) {
        if (dprof) de_runs_fused_kernel<true><<<n_runs, 512, smem, st>>>(a);
        else de_runs_fused_kernel<false><<<n_runs, 512, smem, st>>>(a);
      } else {
        if (dprof) de_runs_kernel<true><<<n_runs, 512, smem, st>>>(a);
        else de_runs_kernel<false><<<n_runs, 512, smem, st>>>(a);
      }
      err = cudaGetLastError();
    }
    count_launch();
    if (err == cudaSuccess) err = cudaGetLastError();
    EVB_CUDA(cudaEventRecord(tc_.done, st));  // the run table may be rewritten once this launch is done
    if (dprof) {
      EVB_CUDA(cudaStreamSynchronize(st));
      unsigned long long h[16];
      EVB_CUDA(cudaMemcpy(h, dprof, sizeof(h), cudaMemcpyDeviceToHost));
      cudaFree(dprof);
      const char* names[] = {"draws", "trial", "x-o", "dot", "pre", "base", "weights", "exchange", "select", "dist"};
      std::string line = "[evb runs] cycles/generation:";
      for (int k = 0; k < 10; ++k) line += std::string(" ") + names[k] + "=" + std::to_string(h[k] / std::max(1, generations));
      std::fprintf(stderr, "%s\n", line.c_str());
    }
    EVB_CUDA(err);
  });
}
