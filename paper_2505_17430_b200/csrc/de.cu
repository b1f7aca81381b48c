// de.cu — DE per-generation update on the device (K4 mutation+crossover+repair, K5 selection +
// archive + SHADE update, K6 top-p order) behind the reference's engine semantics.
//
// Reference: de/engine.hpp:71-102 (generation), de/strategy.hpp (rand/1 :80-94, best/1 :104-118,
// current-to-pbest/1 :138-160, binomial :184-194, clip :234-240, midpoint-target :268-276,
// archive :18-54), de/parameter.hpp (fixed :79-97, SHADE :149-213, sampling :28-43),
// core/population.hpp:70-77 (stable fitness order).
//
// Per generation (one stream, no host sync):
//   1. order     stable (fitness, index) ranks -> the first p_count entries (ttpb/1); best/1:
//                the (fitness, index) argmin by warp-shuffle trees (de_best_kernel)
//   2. draws     per-individual scalar draws: adapter (slot, F, CR), donor indices, jrand.
//                PHILOX: thread per individual, each on its own sub-stream (gen<<32 | i).
//                WORDS : one thread walks the caller's word list in the reference's exact order
//                        (rejection loops, Cauchy resampling) and records every offset.
//   3. trial     block per individual, threads over genes: donor, binomial mask, repair.
//   4. evaluate  the trial matrix through eval_dispatch (scalar-path trig, problem.evaluate).
//   5. select    one CTA: greedy <= replacement in i order, success lists, archive slot
//                assignment with last-writer-wins victims, SHADE memory update (double sums in
//                the reference's sequential order).
//   6. apply     block per replaced individual: parent -> archive slot, trial -> population.
// Arithmetic uses explicitly rounded intrinsics (no FMA contraction), so with the same draws the
// trial vectors are bit-identical to the reference's.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <limits>
#include <cmath>
#include <vector>

#include "evb_internal.cuh"
#include "evb_math.cuh"
#include "ptx.cuh"
#include "rng.cuh"

namespace evb {

struct de_conf {
  int mutation;   // EVB_MUT_*
  int crossover;  // EVB_CX_*
  int repair;     // EVB_REP_*
  int parameter;  // EVB_PAR_*
  double f, cr;   // fixed adapter (stored in T, de/parameter.hpp:81-82)
  double p_best;  // ttpb/1 p (stored in T, de/strategy.hpp:127-131)
  int use_archive;
  int memory_size;
  double jade_c;  // JADE learning rate c (de/parameter.hpp:94-97)
  double archive_rate;
};

}  // namespace evb

struct evb_de_s {
  evb::phase_timer phases;  // order, draws, trial, evaluation, selection scan, selection apply
  int dtype = EVB_F64;
  int P = 0, D = 0;
  evb::de_conf cfg{};
  int p_count = 0;
  int archive_cap = 0;
  int64_t ldt = 0;
  void* trial = nullptr;      // P x ldt
  void* trial_fit = nullptr;  // P
  void* F = nullptr;          // P (T)
  void* CR = nullptr;         // P (T)
  int* slot = nullptr;        // P
  int* idx = nullptr;         // P x 4 (r1, r2, r3 | pbest, r1, r2)
  int* jrand = nullptr;       // P (binomial jrand / exponential start)
  int* xlen = nullptr;        // P: exponential crossover block length
  int64_t* rword = nullptr;   // P: stream index of the first reinitialize-repair word
  int64_t* woff = nullptr;    // P: first gene-uniform word (WORDS) / scalar word count (PHILOX)
  int64_t* wcount = nullptr;  // P: words consumed by individual i
  int* order = nullptr;       // p_count
  int* win = nullptr;         // P
  int* arch_slot = nullptr;   // P: archive slot written by i's push (-1: none / overwritten)
  int* owner = nullptr;       // archive_cap
  int* succ = nullptr;        // P success list (indices)
  int* wlist = nullptr;       // P: winners in push order
  int* d_npush = nullptr;     // [winners, successes] of the last generation
  unsigned* d_epoch = nullptr;               // generation counter of the engine (apply kernel)
  unsigned long long* d_owner64 = nullptr;   // archive_cap
  unsigned long long* d_sel_agg = nullptr;   // ceil(P / kSelBlockItems)
  unsigned* d_sel_sync = nullptr;            // 2
  double* d_srec = nullptr;                  // 3 x P: persistent generations' success records
  int run_nc = -1;                           // persistent generations: cluster size chosen (0: none fits)
  // host-state generations (evb_de_generations_host): packed device [population | fitness], its
  // page-locked staging and the engine's own stream
  void* hs_dev = nullptr;
  void* hs_pinned = nullptr;
  cudaStream_t hs_stream = nullptr;
  size_t run_smem = 0;
  void* archive = nullptr;    // archive_cap x ldt
  int* d_arch_size = nullptr;
  int* d_write_index = nullptr;
  int64_t* d_arch_words = nullptr;  // archive-victim words consumed by the last generation
  void* mem_f = nullptr;            // H
  void* mem_cr = nullptr;           // H
  evb_scratch_s* eval_scratch = nullptr;
  uint32_t last_gen = 0;
  // CUDA graph of one generation (evb_de_generations), keyed by its arguments
  cudaGraphExec_t graph = nullptr;
  cudaStream_t cap_stream = nullptr;
  const void* g_key[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  double g_bounds[2] = {0, 0};
  int g_kernels = 0;
  evb_recorder_s* rec = nullptr;  // attached best-so-far recorder (may be null)
  int rec_run = 0;
  // population policy (de/policy.hpp): P is the current size, P_alloc the initial one
  int P_alloc = 0;
  int reduction = 0;
  int n_min = 4;
  double p_t = 0.0, rate_t = 0.0;  // p and archive_rate as stored in T
  int64_t fes = 0, max_fes = 0;    // evolution_state (core/state.hpp)
  int* rank = nullptr;             // P_alloc: reduction ranks
  int64_t* d_shrink_words = nullptr;
  int last_shrink_valid = 0;
  int gen_P = 0;  // population size at the start of the last generation (its trial count)
  evb_param_trace_s* ptrace = nullptr;  // attached parameter_record trace (may be null)
  int ptrace_run = 0;
  int gen_count = 0;   // evolution_state::generation() (reset by evb_de_optimize)
  int gen_offset = 0;  // restart_run: generations reported by earlier engine runs
  // restart_run's stagnation monitor (hybrid/restart.hpp:55-65), device-resident
  double* d_mon = nullptr;  // [best_seen, since_improvement, evaluations] (doubles)
  int mon_on = 0;
  double mon_eps = 0.0;
};

namespace evb {

__global__ void set_gen_kernel(uint32_t* p, uint32_t v) { *p = v; }
void set_device_gen(evb_rng_s* r, cudaStream_t st) {
  set_gen_kernel<<<1, 1, 0, st>>>(r->d_gen, r->gen);
  count_launch();
}

namespace {

template <typename T>
struct de_dev {
  int P, D;
  de_conf cfg;
  int p_count;
  int archive_cap;
  T* pop;
  int64_t ldp;
  T* fit;
  T* trial;
  int64_t ldt;
  T* trial_fit;
  T* F;
  T* CR;
  int* slot;
  int* idx;
  int* jrand;
  int* xlen;
  int64_t* rword;
  int64_t* woff;
  int64_t* wcount;
  int* order;
  int* win;
  int* arch_slot;
  int* owner;
  int* succ;
  int* wlist;   // P: winners in push (i) order
  int* n_push;  // [winners, successes, multi-CTA epoch tag] of the last generation
  unsigned* epoch;                // engine generation counter (never reset; tags below)
  unsigned long long* owner64;    // archive_cap: (epoch + 1) << 32 | last push index (multi-CTA)
  unsigned long long* sel_agg;    // per selection CTA: (epoch + 1) << 32 | pushes << 16 | successes
  unsigned* sel_sync;             // [ticket, done] of the multi-CTA selection
  int sel_multi;                  // selection ran on de_select_multi_kernel
  T* archive;
  int* arch_size;
  int* write_index;
  int64_t* arch_words;
  T* mem_f;
  T* mem_cr;
  T lb, ub;
  word_source src;
  philox_keys pk;  // src.key's round keys (PHILOX)
  uint32_t* gen_ptr;  // device generation counter (incremented by the apply kernel)
  int64_t* cursor;
  int* overflow;
};

// fitness order (core/population.hpp:70-77): rank = #{j : f_j < f_i or (f_j == f_i and j < i)}
// best/1 (p_count = 1): order[0] = the first strict minimum, i.e. the lexicographic (fitness,
// index) minimum — one block, strided scan + warp-shuffle and shared-memory argmin trees (O(P);
// the rank kernel below is O(P^2) and serves the top-p of current-to-pbest)
template <typename T>
__global__ void __launch_bounds__(1024) de_best_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  __shared__ T sf[32];
  __shared__ int si[32];
  // (f2, i2) precedes (f, i)?  The order kernel's (fitness, index) order, NaN after every number
  auto less = [](T a, T b) { return a < b || (!isnan(a) && isnan(b)); };
  auto merge = [&](T& f, int& i, T f2, int i2) {
    if (i2 >= 0 && (i < 0 || less(f2, f) || (!less(f, f2) && i2 < i))) {
      f = f2;
      i = i2;
    }
  };
  T bf = T(0);
  int bi = -1;
  for (int i = threadIdx.x; i < d.P; i += blockDim.x) merge(bf, bi, d.fit[i], i);
  for (int off = 16; off > 0; off >>= 1) {
    const T of = __shfl_xor_sync(0xffffffffu, bf, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    merge(bf, bi, of, oi);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sf[w] = bf;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    bf = l < nw ? sf[l] : T(0);
    bi = l < nw ? si[l] : -1;
    for (int off = 16; off > 0; off >>= 1) {
      const T of = __shfl_xor_sync(0xffffffffu, bf, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      merge(bf, bi, of, oi);
    }
    if (l == 0) d.order[0] = bi;
  }
}

template <typename T>
__global__ void de_order_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  T* sf = reinterpret_cast<T*>(smem_raw);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const T fi = i < d.P ? d.fit[i] : T(0);
  int rank = 0;
  for (int base = 0; base < d.P; base += blockDim.x) {
    const int j = base + threadIdx.x;
    sf[threadIdx.x] = j < d.P ? d.fit[j] : T(0);
    __syncthreads();
    const int n = min(int(blockDim.x), d.P - base);
    // (fitness, index) order with NaN after every number (a strict weak order, so the ranks are
    // a permutation and every order slot is written; NaN-free populations: the reference's
    // stable sort by fitness)
    auto less = [](T a, T b) { return a < b || (!isnan(a) && isnan(b)); };
    if (i < d.P)
      for (int q = 0; q < n; ++q) {
        const T fj = sf[q];
        const int jj = base + q;
        rank += (less(fj, fi) || (!less(fi, fj) && !less(fj, fi) && jj < i)) ? 1 : 0;
      }
    __syncthreads();
  }
  if (i < d.P && rank < d.p_count) d.order[rank] = i;
}

// Top-p order by sorting (current-to-pbest/1): one CTA bitonic-sorts (key(f), index) pairs in
// shared memory, N = next power of two >= P (<= kSortMax), and writes the first p_count indices.
// key() maps the (fitness, index) order of de_order_kernel onto unsigned integers: -0.0 and +0.0
// are one key (the reference's `<` ties them), every NaN is the largest key (after +inf), and
// equal keys fall back to the index, so the result is the stable sort the reference performs
// (core/population.hpp:70-77) with NaN last.  Padding sorts after everything.
constexpr int kSortMax = 16384;

__device__ __forceinline__ unsigned long long order_key(double f) {
  if (isnan(f)) return ~0ull;
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(f == 0.0 ? 0.0 : f));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ unsigned long long order_key(float f) {
  if (isnan(f)) return ~0ull;
  unsigned b = __float_as_uint(f == 0.f ? 0.f : f);
  return (b >> 31) ? (~b) & 0xFFFFFFFFu : (b | (1u << 31));
}

template <typename T>
__global__ void __launch_bounds__(1024) de_sort_order_kernel(const de_dev<T> d, int n_pow2) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + n_pow2);
  for (int t = threadIdx.x; t < n_pow2; t += blockDim.x) {
    const bool real = t < d.P;
    key[t] = real ? order_key(d.fit[t]) : ~0ull;
    idx[t] = real ? t : 0x7FFFFFFF;  // padding after every NaN
  }
  __syncthreads();
  const int half = n_pow2 >> 1;
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        const int lo = ((t & ~(j - 1)) << 1) | (t & (j - 1));  // pair (lo, lo + j)
        const int hi = lo + j;
        const bool up = (lo & k) == 0;
        const unsigned long long ka = key[lo], kb = key[hi];
        const int ia = idx[lo], ib = idx[hi];
        const bool gt = ka > kb || (ka == kb && ia > ib);
        if (gt == up) {
          key[lo] = kb;
          key[hi] = ka;
          idx[lo] = ib;
          idx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < d.p_count; r += blockDim.x) d.order[r] = idx[r];
}

// de/parameter.hpp:28-38
template <typename R>
__device__ double sample_scale_factor(R& r, double mu) {
  double f = 0.0;
  for (int attempt = 0; attempt < 100; ++attempt) {
    f = draw_cauchy(r, mu, 0.1);
    if (f > 0.0) break;
  }
  if (f <= 0.0) f = 0.1;
  return fmin(f, 1.0);
}
// de/parameter.hpp:41-43
template <typename R>
__device__ double sample_crossover_rate(R& r, double mu) {
  const double v = draw_normal(r, mu, 0.1);
  return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}

// Scalar draws of individual i in the reference's order (de/engine.hpp:88-92):
// adapter sample, mutation indices, crossover jrand.  Returns via the de_dev arrays.  Split in two
// so that the persistent generations can draw the adapter sample (which needs no order) while
// the rest of the CTA ranks the population.
template <typename T, typename R>
__device__ __forceinline__ void draw_adapter(const de_dev<T>& d, R& r, T& F, T& CR, int& slot) {
  slot = -1;
  if (d.cfg.parameter == EVB_PAR_SHADE) {
    slot = draw_int(r, d.cfg.memory_size);
    F = T(sample_scale_factor(r, double(d.mem_f[slot])));
    CR = T(sample_crossover_rate(r, double(d.mem_cr[slot])));
  } else if (d.cfg.parameter == EVB_PAR_JADE) {
    F = T(sample_scale_factor(r, double(d.mem_f[0])));
    CR = T(sample_crossover_rate(r, double(d.mem_cr[0])));
  } else {
    F = T(d.cfg.f);
    CR = T(d.cfg.cr);
  }
}

template <typename T, typename R>
__device__ __forceinline__ void draw_mutation(const de_dev<T>& d, int i, int arch_size, R& r, T F, T CR, int slot) {
  const int ps = d.P;
  int a = 0, b = 0, c = 0;
  if (d.cfg.mutation == EVB_MUT_RAND1) {  // de/strategy.hpp:84-86
    do { a = draw_int(r, ps); } while (a == i);
    do { b = draw_int(r, ps); } while (b == i || b == a);
    do { c = draw_int(r, ps); } while (c == i || c == a || c == b);
  } else if (d.cfg.mutation == EVB_MUT_BEST1) {  // de/strategy.hpp:107-110
    a = d.order[0];
    do { b = draw_int(r, ps); } while (b == i);
    do { c = draw_int(r, ps); } while (c == i || c == b);
  } else {  // ttpb/1, de/strategy.hpp:143-152
    a = d.order[draw_int(r, d.p_count)];
    do { b = draw_int(r, ps); } while (b == i);
    const int pool = ps + (d.cfg.use_archive ? arch_size : 0);
    do { c = draw_int(r, pool); } while (c == i || c == b);
  }
  const int jr = draw_int(r, d.D);  // binomial jrand (de/strategy.hpp:187) / exponential start (:207)
  if (d.cfg.crossover == EVB_CX_EXPONENTIAL) {
    // block length: extended while length < D and u < CR (de/strategy.hpp:208-213); the u's are
    // consumed here, so the trial kernel needs no gene words
    int L = 1;
    while (L < d.D) {
      if (!(draw_uniform01(r) < double(CR))) break;
      ++L;
    }
    d.xlen[i] = L;
  }
  d.F[i] = F;
  d.CR[i] = CR;
  d.slot[i] = slot;
  d.idx[4 * i + 0] = a;
  d.idx[4 * i + 1] = b;
  d.idx[4 * i + 2] = c;
  d.jrand[i] = jr;
}

template <typename T, typename R>
__device__ void draw_scalars(const de_dev<T>& d, int i, int arch_size, R& r) {
  T F, CR;
  int slot;
  draw_adapter<T>(d, r, F, CR, slot);
  draw_mutation<T>(d, i, arch_size, r, F, CR, slot);
}

template <typename T>
__global__ void de_draw_philox_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.P) return;
  const int arch_size = *d.arch_size;
  const uint32_t gen = *d.gen_ptr;
  philox_prefetch_reader<5> r(d.src.key, (uint64_t(gen) << 32) | uint32_t(i));  // the PHILOX source
  draw_scalars<T>(d, i, arch_size, r);
  const int64_t xw = d.cfg.crossover == EVB_CX_BINOMIAL ? d.D : 0;  // gene uniforms follow the scalars
  d.woff[i] = r.count;
  d.rword[i] = r.count + xw;
  d.wcount[i] = r.count + xw;  // + reinitialize-repair words, counted by the trial kernel
}

// Pre-repair trial gene j of individual i (mutation + crossover choice), for the sequential
// WORDS walk of reinitialize repair; `take` = the crossover picked the donor gene.
template <typename T>
__device__ T trial_gene_pre(const de_dev<T>& d, int i, int j, bool take) {
  using F_ = fop<T>;
  const T* xi = d.pop + size_t(i) * d.ldp;
  if (!take) return xi[j];
  const int a = d.idx[4 * i + 0], b = d.idx[4 * i + 1], c = d.idx[4 * i + 2];
  const T Fi = d.F[i];
  const T xa = d.pop[size_t(a) * d.ldp + j], xb = d.pop[size_t(b) * d.ldp + j];
  const T xc = (d.cfg.mutation == EVB_MUT_TTPB1 && c >= d.P) ? d.archive[size_t(c - d.P) * d.ldt + j]
                                                               : d.pop[size_t(c) * d.ldp + j];
  if (d.cfg.mutation == EVB_MUT_TTPB1) return F_::add(F_::add(xi[j], F_::mul(Fi, F_::sub(xa, xi[j]))), F_::mul(Fi, F_::sub(xb, xc)));
  return F_::add(xa, F_::mul(Fi, F_::sub(xb, xc)));
}

template <typename T>
__global__ void de_draw_words_kernel(const de_dev<T> d) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int arch_size = *d.arch_size;
  int64_t pos = *d.cursor;
  for (int i = 0; i < d.P; ++i) {
    word_reader r{&d.src, 0, pos, 0, d.overflow};
    draw_scalars<T>(d, i, arch_size, r);
    const int64_t xw = d.cfg.crossover == EVB_CX_BINOMIAL ? d.D : 0;
    d.woff[i] = r.pos;
    d.rword[i] = r.pos + xw;
    int64_t nviol = 0;
    if (d.cfg.repair == EVB_REP_REINITIALIZE) {
      // the next individual's words start after this one's repair words: walk its trial here
      const double cr = double(d.CR[i]);
      const int jr = d.jrand[i], L = d.cfg.crossover == EVB_CX_EXPONENTIAL ? d.xlen[i] : 0;
      for (int j = 0; j < d.D; ++j) {
        bool take;
        if (d.cfg.crossover == EVB_CX_BINOMIAL) {
          const int64_t q = r.pos + j;
          take = (q < d.src.n_words ? u01_of(d.src.words[q]) < cr : false) || j == jr;
        } else {
          take = ((j - jr + d.D) % d.D) < L;
        }
        const T v = trial_gene_pre<T>(d, i, j, take);
        if (v < d.lb || v > d.ub) ++nviol;
      }
    }
    d.wcount[i] = r.count + xw + nviol;
    pos = r.pos + xw + nviol;
  }
  *d.cursor = pos;
  if (pos > d.src.n_words) *d.overflow = 1;
}

// K4: donor + crossover + repair.  Block per individual.  Binomial: each thread owns one Philox
// block (two consecutive stream words) and so up to two genes.  Exponential: the block
// [start, start + L) mod D was sized by the draw kernel.  Reinitialize repair: the violating
// genes, in j order, take the words after the crossover words (block prefix count).
template <typename T>
__device__ __forceinline__ T repair_gene(int repair, T v, T xij, T lb, T ub) {
  using F_ = fop<T>;
  if (repair == EVB_REP_CLIP) {  // de/strategy.hpp:236-239
    if (v < lb) v = lb;
    if (v > ub) v = ub;
  } else if (repair == EVB_REP_MIDPOINT_TARGET) {  // de/strategy.hpp:270-275
    if (v < lb) v = F_::div(F_::add(lb, xij), T(2));
    else if (v > ub) v = F_::div(F_::add(ub, xij), T(2));
  } else if (repair == EVB_REP_REFLECT) {  // de/strategy.hpp:250-257
    for (int fold = 0; (v < lb || v > ub) && fold < 100; ++fold) {
      if (v < lb) v = F_::add(lb, F_::sub(lb, v));
      if (v > ub) v = F_::sub(ub, F_::sub(v, ub));
    }
    if (v < lb) v = lb;
    if (v > ub) v = ub;
  }  // reinitialize: second pass
  return v;
}

template <typename T>
__device__ __forceinline__ T donor_gene(int mutation, T xij, T xaj, T xbj, T xcj, T Fi) {
  using F_ = fop<T>;
  if (mutation == EVB_MUT_TTPB1)  // x_i + F(x_pb - x_i) + F(x_r1 - x~_r2), de/strategy.hpp:159
    return F_::add(F_::add(xij, F_::mul(Fi, F_::sub(xaj, xij))), F_::mul(Fi, F_::sub(xbj, xcj)));
  return F_::add(xaj, F_::mul(Fi, F_::sub(xbj, xcj)));  // x_a + F(x_b - x_c), de/strategy.hpp:93 / :117
}

template <typename T, int CX>
__global__ void de_trial_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  const int i = blockIdx.x;
  const int D = d.D;
  const T Fi = d.F[i];
  const int jr = d.jrand[i];
  const int a = d.idx[4 * i + 0], b = d.idx[4 * i + 1], c = d.idx[4 * i + 2];
  const T* xi = d.pop + size_t(i) * d.ldp;
  const T* xa = d.pop + size_t(a) * d.ldp;
  const T* xb = d.pop + size_t(b) * d.ldp;
  const T* xc = (d.cfg.mutation == EVB_MUT_TTPB1 && c >= d.P) ? d.archive + size_t(c - d.P) * d.ldt
                                                                : d.pop + size_t(c) * d.ldp;
  T* out = d.trial + size_t(i) * d.ldt;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(i);
  const T lb = d.lb, ub = d.ub;
  const int repair = d.cfg.repair, mutation = d.cfg.mutation;
  if (CX == EVB_CX_BINOMIAL) {
    const double cr = double(d.CR[i]);
    const int64_t s0 = d.woff[i];  // stream index of gene 0's uniform
    // Philox blocks covering stream words [s0, s0 + D)
    const int64_t blk0 = s0 >> 1;
    const int64_t nblk = ((s0 + D + 1) >> 1) - blk0;
    for (int64_t q = threadIdx.x; q < nblk; q += blockDim.x) {
      uint64_t w0, w1;
      const int64_t n0 = (blk0 + q) * 2;
      if (d.src.mode == RNG_PHILOX) {
        philox_pair(d.src.key, ctr_hi, uint64_t(blk0 + q), w0, w1);
      } else {
        // WORDS: s0 is the absolute list position of gene 0
        w0 = (n0 >= s0 && n0 < s0 + D && n0 < d.src.n_words) ? d.src.words[n0] : 0;
        w1 = (n0 + 1 >= s0 && n0 + 1 < s0 + D && n0 + 1 < d.src.n_words) ? d.src.words[n0 + 1] : 0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t j64 = n0 + h - s0;
        if (j64 < 0 || j64 >= D) continue;
        const int j = int(j64);
        // the target row is read only where it is used (non-donor genes, ttpb/1, midpoint repair)
        T v;
        if (u01_of(h ? w1 : w0) < cr || j == jr) {
          if (mutation == EVB_MUT_TTPB1) v = donor_gene<T>(mutation, xi[j], xa[j], xb[j], xc[j], Fi);
          else v = donor_gene<T>(mutation, T(0), xa[j], xb[j], xc[j], Fi);
        } else {
          v = xi[j];
        }
        if (repair == EVB_REP_CLIP) {
          if (v < lb) v = lb;
          if (v > ub) v = ub;
        } else if (repair != EVB_REP_REINITIALIZE) {
          if (v < lb || v > ub) v = repair_gene<T>(repair, v, xi[j], lb, ub);
        }
        out[j] = v;
      }
    }
  } else {  // exponential, de/strategy.hpp:203-214: donor genes [start, start + L) mod D
    const int L = d.xlen[i];
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
      const T xij = xi[j];
      const bool take = ((j - jr + D) % D) < L;
      const T v = take ? donor_gene<T>(mutation, xij, xa[j], xb[j], xc[j], Fi) : xij;
      out[j] = repair_gene<T>(repair, v, xij, lb, ub);
    }
  }
}

// K4, vectorised (binomial crossover, PHILOX source, 16-byte aligned rows): one warp per
// individual walks its row in chunks of W = 32 x VEC genes; lane l owns genes
// [cW + VEC l, cW + VEC l + VEC) and moves them with one 16-byte load per donor row and one
// 16-byte store.  Gene j's uniform is stream word s0 + j.  The Philox blocks a lane computes are
// the pairs covering words [wb + cW + VEC l, +VEC) with wb = s0 rounded down to even, so for odd
// s0 each gene takes the NEXT word: the lane's own words 1..VEC-1 and word 0 of lane l+1 (a
// shuffle; lane 31 takes lane 0's word 0 of the next chunk).  One Philox block per word pair as
// in the scalar kernel, plus up to two blocks per row (the windows run ahead).  Same arithmetic as de_trial_kernel per gene, so the trials are bit-identical.
template <typename T>
struct vec16;
template <>
struct vec16<double> {
  using V = double2;
  static constexpr int N = 2;
  __device__ static void get(const V& v, double (&a)[2]) { a[0] = v.x; a[1] = v.y; }
  __device__ static V make(const double (&a)[2]) { return make_double2(a[0], a[1]); }
};
template <>
struct vec16<float> {
  using V = float4;
  static constexpr int N = 4;
  __device__ static void get(const V& v, float (&a)[4]) { a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w; }
  __device__ static V make(const float (&a)[4]) { return make_float4(a[0], a[1], a[2], a[3]); }
};

constexpr int kTrialVecWarps = 8;  // individuals per 256-thread block

// Take bits of one lane's VEC window words: bit e = (u01(word e) < CR).  u01(w) = (w >> 11) 2^-53
// (core/rng.hpp:81-83) is compared with CR as an integer: (w >> 11) < ceil(CR 2^53) exactly (the
// scaling by 2^53 is exact, the left side is an integer), i.e. w <= lim with
// lim = ((ceil(CR 2^53) - 1) << 11) | 0x7FF; CR <= 0 (or NaN) never takes (`none`).
struct take_rule {
  uint64_t lim;
  bool none;
  __device__ explicit take_rule(double cr) {
    const double t = ceil(cr * 0x1.0p53);
    none = !(t >= 1.0);
    const uint64_t ti = t >= 0x1.0p53 ? (uint64_t(1) << 53) : uint64_t(none ? 1.0 : t);
    lim = ((ti - 1) << 11) | 0x7FFu;
  }
  __device__ __forceinline__ uint32_t bit(uint64_t w) const { return (!none && w <= lim) ? 1u : 0u; }
};

// Warp-per-individual trial kernel (binomial crossover, PHILOX words, 16-byte aligned rows).
// The grid is (individual blocks) x (column blocks); a warp walks chunks [cb0, cb1) of its row,
// W = 32 x VEC genes per chunk, lane l owning genes [cW + VEC l, +VEC) with one 16-byte load per
// donor row and one 16-byte evict-first store.  Gene j's uniform is stream word s0 + j: lane l
// computes the Philox blocks of words [wb + cW + VEC l, +VEC), wb = s0 rounded down to even, as a
// VEC-bit take mask; for odd s0 every gene takes the NEXT word (mask >> 1, the top bit from lane
// l + 1's bit 0 by shuffle, lane 31 from lane 0 of the next chunk's mask).  The masks run two
// chunks ahead, so the loads of a chunk issue before its successor's Philox work.  CLIP: the
// clip repair inlined (the configs' repair); otherwise the runtime repair switch.  Per gene the
// arithmetic is de_trial_kernel's (explicitly rounded donor, same repair), so the trials are
// bit-identical to it.
template <typename T, int MUT, bool CLIP, int MINB>
__global__ void __launch_bounds__(32 * kTrialVecWarps, MINB) de_trial_vec_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  using VT = vec16<T>;
  using V = typename VT::V;
  constexpr int VEC = VT::N, W = 32 * VEC;
  const int i = blockIdx.x * kTrialVecWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= d.P) return;  // warp-uniform
  const int D = d.D;
  const int nchunks = (D + W - 1) / W;
  // column block blockIdx.y: chunks [cb0, cb1).  At large P the population exceeds L2; the grid
  // walks individuals fastest within a column block, so the donor rows' slices of the block in
  // flight (P x block width) stay L2-resident and each is fetched from HBM about once.
  const int cpb = (nchunks + int(gridDim.y) - 1) / int(gridDim.y);
  const int cb0 = int(blockIdx.y) * cpb, cb1 = min(nchunks, cb0 + cpb);
  const T Fi = d.F[i];
  const int jr = d.jrand[i];
  const int a = d.idx[4 * i + 0], b = d.idx[4 * i + 1], c = d.idx[4 * i + 2];
  const T* __restrict__ xi = d.pop + size_t(i) * d.ldp;
  const T* __restrict__ xa = d.pop + size_t(a) * d.ldp;
  const T* __restrict__ xb = d.pop + size_t(b) * d.ldp;
  const T* __restrict__ xc =
      (MUT == EVB_MUT_TTPB1 && c >= d.P) ? d.archive + size_t(c - d.P) * d.ldt : d.pop + size_t(c) * d.ldp;
  T* __restrict__ out = d.trial + size_t(i) * d.ldt;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(i);
  const T lb = d.lb, ub = d.ub;
  const int repair = d.cfg.repair;
  const take_rule rule(double(d.CR[i]));
  const int64_t s0 = d.woff[i];
  const bool odd = (s0 & 1) != 0;
  const uint64_t blk0 = uint64_t(s0 >> 1) + uint64_t(lane * (VEC / 2));  // this lane's first block
  constexpr uint32_t FULL = (1u << VEC) - 1u;
  auto window = [&](int cc) -> uint32_t {  // the lane's VEC take bits of chunk cc (words wb + ...)
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < VEC / 2; ++k) {
      const uint64_t blk = blk0 + uint64_t(cc) * (W / 2) + uint64_t(k);
      uint32_t cw[4] = {uint32_t(blk), uint32_t(blk >> 32), uint32_t(ctr_hi), uint32_t(ctr_hi >> 32)};
      philox4x32_10_rk(cw, d.pk);
      m |= rule.bit((uint64_t(cw[1]) << 32) | cw[0]) << (2 * k);
      m |= rule.bit((uint64_t(cw[3]) << 32) | cw[2]) << (2 * k + 1);
    }
    return m;
  };
  uint32_t w0 = window(cb0);
  uint32_t w1 = cb0 + 1 <= nchunks ? window(cb0 + 1) : 0u;
  for (int cc = cb0; cc < cb1; ++cc) {
    uint32_t take = w0;
    if (odd) {
      const uint32_t up = __shfl_down_sync(0xffffffffu, w0, 1) & 1u;
      const uint32_t wrap = __shfl_sync(0xffffffffu, w1, 0) & 1u;
      take = (w0 >> 1) | ((lane == 31 ? wrap : up) << (VEC - 1));
    }
    const int j0 = cc * W + VEC * lane;
    if (unsigned(jr - j0) < unsigned(VEC)) take |= 1u << (jr - j0);
    const bool full = j0 + VEC <= D;
    const bool need = MUT == EVB_MUT_TTPB1 || repair == EVB_REP_MIDPOINT_TARGET || take != FULL;
    V va, vb, vc, vi;
    if (full) {
      va = __ldg(reinterpret_cast<const V*>(xa + j0));
      vb = __ldg(reinterpret_cast<const V*>(xb + j0));
      vc = __ldg(reinterpret_cast<const V*>(xc + j0));
      if (need) vi = __ldg(reinterpret_cast<const V*>(xi + j0));
    }
    // the window after next (overlaps the loads)
    const uint32_t w2 = cc + 2 <= min(nchunks, cb1) ? window(cc + 2) : 0u;
    if (full) {
      T ta[VEC], tb_[VEC], tc[VEC], ti[VEC] = {}, v[VEC];
      VT::get(va, ta);
      VT::get(vb, tb_);
      VT::get(vc, tc);
      if (need) VT::get(vi, ti);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        T x = ((take >> e) & 1u) ? donor_gene<T>(MUT, MUT == EVB_MUT_TTPB1 ? ti[e] : T(0), ta[e], tb_[e], tc[e], Fi)
                                 : ti[e];
        if (CLIP) {
          if (x < lb) x = lb;
          if (x > ub) x = ub;
        } else if (repair == EVB_REP_CLIP) {
          if (x < lb) x = lb;
          if (x > ub) x = ub;
        } else if (repair != EVB_REP_REINITIALIZE) {
          if (x < lb || x > ub) x = repair_gene<T>(repair, x, ti[e], lb, ub);
        }
        v[e] = x;
      }
      __stcs(reinterpret_cast<V*>(out + j0), VT::make(v));
    } else if (j0 < D) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int j = j0 + e;
        if (j >= D) break;
        T x;
        if ((take >> e) & 1u) x = donor_gene<T>(MUT, MUT == EVB_MUT_TTPB1 ? xi[j] : T(0), xa[j], xb[j], xc[j], Fi);
        else x = xi[j];
        if (CLIP || repair == EVB_REP_CLIP) {
          if (x < lb) x = lb;
          if (x > ub) x = ub;
        } else if (repair != EVB_REP_REINITIALIZE) {
          if (x < lb || x > ub) x = repair_gene<T>(repair, x, xi[j], lb, ub);
        }
        out[j] = x;
      }
    }
    w0 = w1;
    w1 = w2;
  }
}

// The trial kernel with the rows staged through shared memory (the HBM regime, P x D beyond L2):
// same warp-per-individual mapping, chunks, column blocks, take masks and per-gene arithmetic as
// de_trial_vec_kernel (bit-identical trials), but every lane moves its 16 bytes of the four rows
// (target, a, b, c) with cp.async (LDGSTS: no registers held while in flight) into a per-warp
// ring of S chunk stages, S - 1 chunks ahead of the one it computes, so a warp keeps
// (S - 1) x 2 KB of loads outstanding instead of one chunk's 2 KB in registers.  A lane reads back
// only what it copied itself, so cp.async.wait_group alone orders it (no barrier).  Bulk copies
// (TMA, one per 512-byte row chunk) measured slower: ~30 cycles of the SM's copy engine per op.
template <typename T, int MUT, bool CLIP, int S, int MINB>
__global__ void __launch_bounds__(32 * kTrialVecWarps, MINB) de_trial_stage_kernel(const de_dev<T> d) {
  using VT = vec16<T>;
  using V = typename VT::V;
  constexpr int VEC = VT::N, W = 32 * VEC;
  constexpr int STAGEB = 4 * 512;  // target, a, b, c: 512 bytes each
  extern __shared__ __align__(128) uint8_t tsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring = ptx::smem_u32(tsm + size_t(warp) * S * STAGEB) + uint32_t(lane) * 16u;
  const int i = blockIdx.x * kTrialVecWarps + warp;
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  if (i >= d.P) return;  // warp-uniform
  const int D = d.D;
  const int nchunks = (D + W - 1) / W;
  const int cpb = (nchunks + int(gridDim.y) - 1) / int(gridDim.y);
  const int cb0 = int(blockIdx.y) * cpb, cb1 = min(nchunks, cb0 + cpb);
  const int a = d.idx[4 * i + 0], b = d.idx[4 * i + 1], c = d.idx[4 * i + 2];
  const T* xi = d.pop + size_t(i) * d.ldp + VEC * lane;
  const T* xa = d.pop + size_t(a) * d.ldp + VEC * lane;
  const T* xb = d.pop + size_t(b) * d.ldp + VEC * lane;
  const T* xc = ((MUT == EVB_MUT_TTPB1 && c >= d.P) ? d.archive + size_t(c - d.P) * d.ldt
                                                    : d.pop + size_t(c) * d.ldp) + VEC * lane;
  // this lane's 16 bytes of chunk cc of the four rows (rows are pitched to 16 bytes, so a vector
  // starting before D stays inside the row)
  auto copy = [&](int cc) {
    if (cc < cb1 && cc * W + VEC * lane < D) {
      const uint32_t st = ring + uint32_t((cc - cb0) % S) * STAGEB;
      const size_t off = size_t(cc) * W;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st), "l"(xi + off) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + 512u), "l"(xa + off) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + 1024u), "l"(xb + off) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + 1536u), "l"(xc + off) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // one group per chunk, empty or not
  };
#pragma unroll
  for (int k = 0; k < S - 1; ++k) copy(cb0 + k);
  const T Fi = d.F[i];
  const int jr = d.jrand[i];
  T* __restrict__ out = d.trial + size_t(i) * d.ldt;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(i);
  const T lb = d.lb, ub = d.ub;
  const int repair = d.cfg.repair;
  const take_rule rule(double(d.CR[i]));
  const int64_t s0 = d.woff[i];
  const bool odd = (s0 & 1) != 0;
  const uint64_t blk0 = uint64_t(s0 >> 1) + uint64_t(lane * (VEC / 2));
  auto window = [&](int cc) -> uint32_t {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < VEC / 2; ++k) {
      const uint64_t blk = blk0 + uint64_t(cc) * (W / 2) + uint64_t(k);
      uint32_t cw[4] = {uint32_t(blk), uint32_t(blk >> 32), uint32_t(ctr_hi), uint32_t(ctr_hi >> 32)};
      philox4x32_10_rk(cw, d.pk);
      m |= rule.bit((uint64_t(cw[1]) << 32) | cw[0]) << (2 * k);
      m |= rule.bit((uint64_t(cw[3]) << 32) | cw[2]) << (2 * k + 1);
    }
    return m;
  };
  uint32_t w0 = window(cb0);
  for (int cc = cb0; cc < cb1; ++cc) {
    copy(cc + S - 1);  // into the stage chunk cc - 1 used (this lane read it last iteration)
    const uint32_t w1 = (odd && cc + 1 <= nchunks) ? window(cc + 1) : 0u;
    uint32_t take = w0;
    if (odd) {
      const uint32_t up = __shfl_down_sync(0xffffffffu, w0, 1) & 1u;
      const uint32_t wrap = __shfl_sync(0xffffffffu, w1, 0) & 1u;
      take = (w0 >> 1) | ((lane == 31 ? wrap : up) << (VEC - 1));
    }
    const int j0 = cc * W + VEC * lane;
    if (unsigned(jr - j0) < unsigned(VEC)) take |= 1u << (jr - j0);
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");  // chunk cc's group landed
    const uint32_t st = ring + uint32_t((cc - cb0) % S) * STAGEB;
    if (j0 < D) {
      T ti[VEC], ta[VEC], tb_[VEC], tc[VEC], v[VEC];
      if constexpr (sizeof(T) == 8) {
        const double2 q0 = ptx::lds_f64x2(st), q1 = ptx::lds_f64x2(st + 512u), q2 = ptx::lds_f64x2(st + 1024u),
                      q3 = ptx::lds_f64x2(st + 1536u);
        ti[0] = q0.x; ti[1] = q0.y; ta[0] = q1.x; ta[1] = q1.y;
        tb_[0] = q2.x; tb_[1] = q2.y; tc[0] = q3.x; tc[1] = q3.y;
      } else {
        const float4 q0 = ptx::lds_f32x4(st), q1 = ptx::lds_f32x4(st + 512u), q2 = ptx::lds_f32x4(st + 1024u),
                     q3 = ptx::lds_f32x4(st + 1536u);
        VT::get(q0, ti); VT::get(q1, ta); VT::get(q2, tb_); VT::get(q3, tc);
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        T x = ((take >> e) & 1u) ? donor_gene<T>(MUT, MUT == EVB_MUT_TTPB1 ? ti[e] : T(0), ta[e], tb_[e], tc[e], Fi)
                                 : ti[e];
        if (CLIP || repair == EVB_REP_CLIP) {
          if (x < lb) x = lb;
          if (x > ub) x = ub;
        } else if (repair != EVB_REP_REINITIALIZE) {
          if (x < lb || x > ub) x = repair_gene<T>(repair, x, ti[e], lb, ub);
        }
        v[e] = x;
      }
      if (j0 + VEC <= D) {
        __stcs(reinterpret_cast<V*>(out + j0), VT::make(v));
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (j0 + e < D) out[j0 + e] = v[e];
      }
    }
    w0 = w1;
    if (!odd && cc + 1 < cb1) w0 = window(cc + 1);
  }
}

// reinitialize repair (de/strategy.hpp:285-289), a second pass over the trial rows: every gene
// still outside [lb, ub] takes T(uniform(lb, ub)); the words follow the crossover words in j
// order, so each violating gene's word is its rank among the violations (block prefix count).
template <typename T>
__global__ void de_reinit_kernel(const de_dev<T> d) {
  const int i = blockIdx.x;
  const int D = d.D;
  T* out = d.trial + size_t(i) * d.ldt;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(i);
  const T lb = d.lb, ub = d.ub;
  __shared__ int warp_tot[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const int64_t r0 = d.rword[i];
  int running = 0;
  for (int base = 0; base < D; base += blockDim.x) {
    const int j = base + threadIdx.x;
    const bool viol = j < D && (out[j] < lb || out[j] > ub);
    const unsigned m = __ballot_sync(0xffffffffu, viol);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      before += w < warp ? warp_tot[w] : 0;
      total += warp_tot[w];
    }
    if (viol) {
      const int64_t s = r0 + running + before + __popc(m & ((1u << lane) - 1u));
      uint64_t word;
      if (d.src.mode == RNG_PHILOX) {
        uint64_t wa, wb;
        philox_pair(d.src.key, ctr_hi, uint64_t(s >> 1), wa, wb);
        word = (s & 1) ? wb : wa;
      } else {
        word = s < d.src.n_words ? d.src.words[s] : 0;
        if (s >= d.src.n_words) *d.overflow = 1;
      }
      out[j] = T(__dadd_rn(double(lb), __dmul_rn(__dsub_rn(double(ub), double(lb)), u01_of(word))));
    }
    running += total;
    __syncthreads();
  }
  if (threadIdx.x == 0 && d.src.mode == RNG_PHILOX) d.wcount[i] = r0 + running;
}

template <typename T>
__device__ void adapter_update(const de_dev<T>& d, int n_succ, bool staged_in_pass1, double* st_g, double* st_f,
                               double* st_c);

// K5a: selection bookkeeping (de/engine.hpp:27-47, de/strategy.hpp:29-37, de/parameter.hpp:166-184)
// in one CTA, parallel where the reference's sequential semantics allow it:
//   * win / success flags per individual, stable compaction of pushes and successes by block
//     prefix sums (i order preserved);
//   * archive slots: push q appends while the archive has room (slot size+q); once full the size
//     stays at capacity, so each later push's victim uniform_int(cap) depends only on its own word
//     (the (q - room)-th archive word) -> computed in parallel; last writer wins per slot via an
//     atomicMax on the push index;
//   * SHADE / JADE sums stay sequential (one thread, successes staged in order) so the memory
//     update rounds exactly like the reference's loops.
constexpr int kSelThreads = 1024;
constexpr int kOwnerSmem = 4096;

template <typename T>
__global__ void __launch_bounds__(kSelThreads) de_select_scan_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  __shared__ int warp_sum[2][kSelThreads / 32];
  __shared__ int carry[2];
  // successes' (gain, F, CR) in success order, for the adapter update below
  __shared__ double st_g[kSelThreads], st_f[kSelThreads], st_c[kSelThreads];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool adapt = d.cfg.parameter == EVB_PAR_SHADE || d.cfg.parameter == EVB_PAR_JADE;
  // one pass-1 chunk: pass 1 stages the successes itself (no second trip through global memory)
  const bool staged_in_pass1 = adapt && d.P <= int(blockDim.x);
  // archive-slot owners (last writer wins): shared memory for archives up to kOwnerSmem slots
  __shared__ int s_owner[kOwnerSmem];
  int* owner = d.archive_cap <= kOwnerSmem ? s_owner : d.owner;
  for (int s = tid; s < d.archive_cap; s += blockDim.x) owner[s] = -1;
  const int size0 = *d.arch_size;
  const int room = d.archive_cap - size0;
  const int64_t wpos = d.src.mode == RNG_WORDS ? *d.cursor : 0;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | kSubArchive;
  if (tid == 0) carry[0] = carry[1] = 0;
  __syncthreads();
  // pass 1: flags, exclusive prefix sums (pushes, successes), slot assignment
  for (int base = 0; base < d.P; base += blockDim.x) {
    const int i = base + tid;
    int w = 0, s = 0;
    double gain = 0.0, fi = 0.0, ci = 0.0;
    if (i < d.P) {
      const T ft = d.trial_fit[i], fp = d.fit[i];
      if (staged_in_pass1) {  // loads issued with the fitness loads, ahead of the scans
        fi = double(d.F[i]);
        ci = double(d.CR[i]);
      }
      w = (ft <= fp) ? 1 : 0;
      gain = double(fop<T>::sub(fp, ft));
      s = (w && fop<T>::sub(fp, ft) > T(0)) ? 1 : 0;
      d.arch_slot[i] = -1;
    }
    // block-wide exclusive scans of (w, s)
    int iw = w, is = s;
    for (int off = 1; off < 32; off <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, iw, off), b = __shfl_up_sync(0xffffffffu, is, off);
      if (lane >= off) {
        iw += a;
        is += b;
      }
    }
    if (lane == 31) {
      warp_sum[0][wid] = iw;
      warp_sum[1][wid] = is;
    }
    __syncthreads();
    if (wid == 0) {
      const int nw = blockDim.x >> 5;
      int a = lane < nw ? warp_sum[0][lane] : 0, b = lane < nw ? warp_sum[1][lane] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, a, off), y = __shfl_up_sync(0xffffffffu, b, off);
        if (lane >= off) {
          a += x;
          b += y;
        }
      }
      if (lane < nw) {
        warp_sum[0][lane] = a;
        warp_sum[1][lane] = b;
      }
    }
    __syncthreads();
    const int q = carry[0] + (wid > 0 ? warp_sum[0][wid - 1] : 0) + iw - w;  // push index
    const int k = carry[1] + (wid > 0 ? warp_sum[1][wid - 1] : 0) + is - s;  // success index
    if (i < d.P) {
      d.win[i] = w ? q + 1 : 0;  // winner flag carrying its push index
      if (w) d.wlist[q] = i;
      if (s) d.succ[k] = i;
      if (s && staged_in_pass1) {
        st_g[k] = gain;
        st_f[k] = fi;
        st_c[k] = ci;
      }
      if (w && d.archive_cap > 0) {
        int sl;
        if (q < room) {
          sl = size0 + q;
        } else {
          const int64_t v = q - room;
          sl = uint_of(word_at(d.src, ctr_hi, d.src.mode == RNG_WORDS ? wpos + v : v, d.overflow), d.archive_cap);
        }
        d.arch_slot[i] = sl;  // provisional; resolved below
        atomicMax(&owner[sl], q);
      }
    }
    __syncthreads();
    if (tid == blockDim.x - 1) {
      carry[0] = q + w;
      carry[1] = k + s;
    }
    __syncthreads();
  }
  const int n_push = carry[0], n_succ = carry[1];
  // pass 2: last writer wins (members_[victim] = genome, in push order)
  for (int base = 0; base < d.P; base += blockDim.x) {
    const int i = base + tid;
    if (i < d.P && d.win[i] && d.archive_cap > 0) {
      const int sl = d.arch_slot[i];
      if (owner[sl] != d.win[i] - 1) d.arch_slot[i] = -1;  // overwritten by a later push
    }
  }
  __syncthreads();
  if (tid == 0) {
    d.n_push[0] = n_push;
    d.n_push[1] = n_succ;
    const int new_size = min(d.archive_cap, size0 + n_push);
    const int64_t nv = d.archive_cap > 0 ? max(0, n_push - room) : 0;
    *d.arch_size = new_size;
    *d.arch_words = nv;
    if (d.src.mode == RNG_WORDS) *d.cursor = wpos + nv;
  }
  if (n_succ == 0 || !adapt) return;
  adapter_update<T>(d, n_succ, staged_in_pass1, st_g, st_f, st_c);
}

// SHADE / JADE memory update from the generation's successes (de/parameter.hpp:107-120, 166-184):
// the sums stay sequential in success order (the reference's loops), but the successes' (gain, F,
// CR) are first staged into shared memory by the whole block — one thread chasing succ[s] ->
// fit[i] through global memory paid the L2 latency per success.  st_* hold blockDim.x doubles.
template <typename T>
__device__ void adapter_update(const de_dev<T>& d, int n_succ, bool staged_in_pass1, double* st_g, double* st_f,
                               double* st_c) {
  const int tid = threadIdx.x;
  __shared__ double acc_s[4];
  auto stage = [&](int base) {
    const int s = base + tid;
    if (s < n_succ && !staged_in_pass1) {
      const int i = d.succ[s];
      st_g[tid] = double(fop<T>::sub(d.fit[i], d.trial_fit[i]));
      st_f[tid] = double(d.F[i]);
      st_c[tid] = double(d.CR[i]);
    }
  };
  const bool one_chunk = n_succ <= int(blockDim.x);
  // thread 0's sequential sums read eight staged values per round with the loads ahead of the
  // dependent add chain; every per-success product is formed by its own thread first (the same
  // roundings as the reference's loop body, so the sums are bit-identical)
  auto seq_sum = [&](double acc, const double* v, int n) {
    int t = 0;
    for (; t + 8 <= n; t += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = v[t + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, x[u]);
    }
    for (; t < n; ++t) acc = __dadd_rn(acc, v[t]);
    return acc;
  };
  if (d.cfg.parameter == EVB_PAR_SHADE) {  // de/parameter.hpp:166-184
    double gain_sum = 0.0;
    for (int base = 0; base < n_succ; base += blockDim.x) {
      stage(base);
      __syncthreads();
      if (tid == 0) gain_sum = seq_sum(gain_sum, st_g, min(int(blockDim.x), n_succ - base));
      __syncthreads();
    }
    if (tid == 0) acc_s[0] = gain_sum;
    __syncthreads();
    gain_sum = acc_s[0];
    double f_num = 0.0, f_den = 0.0, cr_acc = 0.0;
    for (int base = 0; base < n_succ; base += blockDim.x) {
      if (!one_chunk) {
        stage(base);
        __syncthreads();
      }
      if (base + tid < n_succ) {  // w = gain / sum; (w f) f, w f, w cr
        const double w = __ddiv_rn(st_g[tid], gain_sum);
        const double f = st_f[tid];
        const double wf = __dmul_rn(w, f);
        st_g[tid] = __dmul_rn(wf, f);
        st_f[tid] = wf;
        st_c[tid] = __dmul_rn(w, st_c[tid]);
      }
      __syncthreads();
      if (tid == 0) {
        const int n = min(int(blockDim.x), n_succ - base);
        f_num = seq_sum(f_num, st_g, n);
        f_den = seq_sum(f_den, st_f, n);
        cr_acc = seq_sum(cr_acc, st_c, n);
      }
      __syncthreads();
    }
    if (tid == 0) {
      const int k = *d.write_index;
      d.mem_f[k] = T(__ddiv_rn(f_num, f_den));
      d.mem_cr[k] = T(cr_acc);
      *d.write_index = (k + 1) % d.cfg.memory_size;
    }
  } else {  // JADE, de/parameter.hpp:107-120 (lehmer_mean :45-52)
    double num = 0.0, den = 0.0, crm = 0.0;
    for (int base = 0; base < n_succ; base += blockDim.x) {
      stage(base);
      __syncthreads();
      if (base + tid < n_succ) st_g[tid] = __dmul_rn(st_f[tid], st_f[tid]);  // f * f
      __syncthreads();
      if (tid == 0) {
        const int n = min(int(blockDim.x), n_succ - base);
        num = seq_sum(num, st_g, n);
        den = seq_sum(den, st_f, n);
        crm = seq_sum(crm, st_c, n);
      }
      __syncthreads();
    }
    if (tid == 0) {
      const double lehmer = __ddiv_rn(num, den);
      crm = __ddiv_rn(crm, double(n_succ));
      const double c = double(T(d.cfg.jade_c));
      d.mem_f[0] = T(__dadd_rn(__dmul_rn(__dsub_rn(1.0, c), double(d.mem_f[0])), __dmul_rn(c, lehmer)));
      d.mem_cr[0] = T(__dadd_rn(__dmul_rn(__dsub_rn(1.0, c), double(d.mem_cr[0])), __dmul_rn(c, crm)));
    }
  }
}

// K5a for large populations (P > kSelSingleMax): the same bookkeeping over many CTAs.  Each CTA
// takes kSelBlockItems consecutive individuals in ticket order (atomic ticket = virtual block id,
// so every lower id is already running), publishes its (pushes, successes) aggregate tagged with
// the generation's epoch, and sums the aggregates of all lower ids (decoupled look-back; a lower
// id publishes before it waits on anything, so the spin always ends).  Archive-slot owners are
// 64-bit (epoch << 32 | push index) maxima, so a later generation needs no reset; the apply
// kernel resolves last-writer-wins against them.  The CTA that finishes last writes the archive
// size / victim-word count / cursor and resets the tickets.  Adaptive adapters then run
// de_adapt_kernel (one CTA, the sequential sums).
constexpr int kSelSingleMax = 2048;
constexpr int kSelBlockThreads = 256;
constexpr int kSelPerThread = 4;
constexpr int kSelBlockItems = kSelBlockThreads * kSelPerThread;

template <typename T>
__global__ void __launch_bounds__(kSelBlockThreads) de_select_multi_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  __shared__ int s_vb, s_last;
  __shared__ int warp_sum[2][kSelBlockThreads / 32];
  __shared__ int s_prefix[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_vb = int(atomicAdd(&d.sel_sync[0], 1u));
  __syncthreads();
  const int vb = s_vb;
  const unsigned tag = *d.epoch + 1u;
  const int size0 = *d.arch_size;
  const int room = d.archive_cap - size0;
  const int64_t wpos = d.src.mode == RNG_WORDS ? *d.cursor : 0;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | kSubArchive;
  const int i0 = vb * kSelBlockItems + tid * kSelPerThread;
  T ftv[kSelPerThread], fpv[kSelPerThread];
#pragma unroll
  for (int u = 0; u < kSelPerThread; ++u)
    if (i0 + u < d.P) {
      ftv[u] = d.trial_fit[i0 + u];
      fpv[u] = d.fit[i0 + u];
    }
  int wbits = 0, sbits = 0;
#pragma unroll
  for (int u = 0; u < kSelPerThread; ++u)
    if (i0 + u < d.P) {
      const int w_ = (ftv[u] <= fpv[u]) ? 1 : 0;
      wbits |= w_ << u;
      sbits |= ((w_ && fop<T>::sub(fpv[u], ftv[u]) > T(0)) ? 1 : 0) << u;
    }
  const int w = __popc(wbits), s = __popc(sbits);
  int iw = w, is = s;
  for (int off = 1; off < 32; off <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, iw, off), b = __shfl_up_sync(0xffffffffu, is, off);
    if (lane >= off) {
      iw += a;
      is += b;
    }
  }
  if (lane == 31) {
    warp_sum[0][wid] = iw;
    warp_sum[1][wid] = is;
  }
  __syncthreads();
  if (wid == 0) {
    constexpr int nw = kSelBlockThreads / 32;
    int a = lane < nw ? warp_sum[0][lane] : 0, b = lane < nw ? warp_sum[1][lane] : 0;
    for (int off = 1; off < 32; off <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, a, off), y = __shfl_up_sync(0xffffffffu, b, off);
      if (lane >= off) {
        a += x;
        b += y;
      }
    }
    if (lane < nw) {
      warp_sum[0][lane] = a;
      warp_sum[1][lane] = b;
    }
    // publish this CTA's aggregate, then sum every lower id's (spin until tagged this generation)
    const int tw = __shfl_sync(0xffffffffu, a, nw - 1), ts = __shfl_sync(0xffffffffu, b, nw - 1);
    if (lane == 0) {
      const unsigned long long agg = (static_cast<unsigned long long>(tag) << 32) | (unsigned(tw) << 16) | unsigned(ts);
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(d.sel_agg + vb), "l"(agg) : "memory");
    }
    int pw = 0, ps = 0;
    for (int j = lane; j < vb; j += 32) {
      unsigned long long v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(d.sel_agg + j) : "memory");
      } while (unsigned(v >> 32) != tag);
      pw += int((v >> 16) & 0xFFFFu);
      ps += int(v & 0xFFFFu);
    }
    for (int off = 16; off > 0; off >>= 1) {
      pw += __shfl_xor_sync(0xffffffffu, pw, off);
      ps += __shfl_xor_sync(0xffffffffu, ps, off);
    }
    if (lane == 0) {
      s_prefix[0] = pw;
      s_prefix[1] = ps;
    }
  }
  __syncthreads();
  const int q0 = s_prefix[0] + (wid > 0 ? warp_sum[0][wid - 1] : 0) + iw - w;
  const int k0 = s_prefix[1] + (wid > 0 ? warp_sum[1][wid - 1] : 0) + is - s;
#pragma unroll
  for (int u = 0; u < kSelPerThread; ++u) {
    const int i = i0 + u;
    if (i >= d.P) continue;
    const int wu = (wbits >> u) & 1, su = (sbits >> u) & 1;
    const int q = q0 + __popc(wbits & ((1 << u) - 1));
    const int k = k0 + __popc(sbits & ((1 << u) - 1));
    d.win[i] = wu ? q + 1 : 0;
    if (wu) d.wlist[q] = i;
    if (su) d.succ[k] = i;
    int sl = -1;
    if (wu && d.archive_cap > 0) {
      if (q < room) {
        sl = size0 + q;
      } else {
        const int64_t v = q - room;
        sl = uint_of(word_at(d.src, ctr_hi, d.src.mode == RNG_WORDS ? wpos + v : v, d.overflow), d.archive_cap);
      }
      atomicMax(d.owner64 + sl, (static_cast<unsigned long long>(tag) << 32) | unsigned(q));
    }
    d.arch_slot[i] = sl;  // provisional; the apply kernel resolves overwritten pushes
  }
  // the last CTA to finish: totals, archive size, victim words, cursor; tickets back to 0
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned done = atomicAdd(&d.sel_sync[1], 1u);
    s_last = done == gridDim.x - 1 ? 1 : 0;
  }
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    int tw = 0, ts = 0;  // all aggregates are published (every CTA counted itself done)
    for (int j = 0; j < int(gridDim.x); ++j) {
      const unsigned long long a = __ldcg(d.sel_agg + j);
      tw += int((a >> 16) & 0xFFFFu);
      ts += int(a & 0xFFFFu);
    }
    d.n_push[0] = tw;
    d.n_push[1] = ts;
    d.n_push[2] = int(tag);
    *d.epoch = tag;  // the next generation tags with tag + 1 (read by every CTA before this point)
    const int new_size = min(d.archive_cap, size0 + tw);
    const int64_t nv = d.archive_cap > 0 ? max(0, tw - room) : 0;
    *d.arch_size = new_size;
    *d.arch_words = nv;
    if (d.src.mode == RNG_WORDS) *d.cursor = wpos + nv;
    d.sel_sync[0] = 0u;
    d.sel_sync[1] = 0u;
  }
}

// adaptive adapters after de_select_multi_kernel: the SHADE / JADE update over the success list
template <typename T>
__global__ void __launch_bounds__(kSelThreads) de_adapt_kernel(const de_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  __shared__ double st_g[kSelThreads], st_f[kSelThreads], st_c[kSelThreads];
  const int n_succ = d.n_push[1];
  if (n_succ == 0) return;
  adapter_update<T>(d, n_succ, false, st_g, st_f, st_c);
}

// K5b: replaced parent -> archive slot, trial -> population (std::swap(pop[i], trial)), one warp
// per winner over the scan's push list (a generation late in a run replaces few rows: no block per
// individual), 16-byte moves where the rows allow, four in flight per lane.
template <typename T>
__global__ void __launch_bounds__(256) de_select_apply_kernel(const de_dev<T> d, int vec, int list) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  if (list && blockIdx.x == 0 && threadIdx.x == 0) *d.gen_ptr += 1u;  // last reader of this generation's id is done
  using VT = vec16<T>;
  using V = typename VT::V;
  constexpr int VEC = VT::N;
  if (!list) {  // one block per individual (small populations: the shortest dependent chain)
    const int i = blockIdx.x;
    if (i == 0 && threadIdx.x == 0) *d.gen_ptr += 1u;
    if (!d.win[i]) return;
    const int sl = d.arch_slot[i];
    T* x = d.pop + size_t(i) * d.ldp;
    const T* t = d.trial + size_t(i) * d.ldt;
    T* a = sl >= 0 ? d.archive + size_t(sl) * d.ldt : nullptr;
    for (int j = threadIdx.x; j < d.D; j += blockDim.x) {
      const T old = x[j];
      if (a) a[j] = old;
      x[j] = t[j];
    }
    if (threadIdx.x == 0) d.fit[i] = d.trial_fit[i];
    return;
  }
  // list: walk the scan's push list, one warp per winner (few winners late in a run)
  const int n = *d.n_push;
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int q = blockIdx.x * wpb + (threadIdx.x >> 5); q < n; q += gridDim.x * wpb) {
    const int i = d.wlist[q];
    int sl = d.arch_slot[i];
    if (d.sel_multi && sl >= 0 &&  // a later push won the slot (tag: the multi-CTA selection's epoch)
        d.owner64[sl] != ((static_cast<unsigned long long>(unsigned(d.n_push[2])) << 32) | unsigned(q))) {
      sl = -1;
      if ((threadIdx.x & 31) == 0) d.arch_slot[i] = -1;
    }
    T* x = d.pop + size_t(i) * d.ldp;
    const T* t = d.trial + size_t(i) * d.ldt;
    T* a = sl >= 0 ? d.archive + size_t(sl) * d.ldt : nullptr;
    int j0 = 0;
    if (vec) {
      const int nv = d.D / VEC;  // whole vectors
      V* xv = reinterpret_cast<V*>(x);
      const V* tv = reinterpret_cast<const V*>(t);
      V* av = reinterpret_cast<V*>(a);
      int k = lane;
      for (; k + 96 < nv; k += 128) {
        V o[4], tt[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          o[u] = xv[k + 32 * u];
          tt[u] = tv[k + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (a) av[k + 32 * u] = o[u];
          xv[k + 32 * u] = tt[u];
        }
      }
      for (; k < nv; k += 32) {
        const V o = xv[k], tt = tv[k];
        if (a) av[k] = o;
        xv[k] = tt;
      }
      j0 = nv * VEC;
    }
    for (int j = j0 + lane; j < d.D; j += 32) {
      const T old = x[j];
      if (a) a[j] = old;
      x[j] = t[j];
    }
    if (lane == 0) d.fit[i] = d.trial_fit[i];
  }
}

// init_population (core/population.hpp:88-98): P*D uniforms, individual-major
template <typename T>
__global__ void init_population_kernel(T* pop, int64_t ldp, int P, int D, double lb, double ub, word_source src,
                                       uint64_t ctr_hi, int64_t base, int* overflow) {
  const int64_t n = int64_t(P) * D;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t pos = base + e;
    const uint64_t w = word_at(src, ctr_hi, pos, overflow);
    const double u = u01_of(w);
    pop[(e / D) * ldp + (e % D)] = T(__dadd_rn(lb, __dmul_rn(__dsub_rn(ub, lb), u)));
  }
}

template <typename T>
de_dev<T> make_dev(evb_de_s* e, void* pop, int64_t ldp, void* fit, double lb, double ub, evb_rng_s* r) {
  de_dev<T> d{};
  d.P = e->P;
  d.D = e->D;
  d.cfg = e->cfg;
  d.p_count = e->p_count;
  d.archive_cap = e->archive_cap;
  d.pop = static_cast<T*>(pop);
  d.ldp = ldp;
  d.fit = static_cast<T*>(fit);
  d.trial = static_cast<T*>(e->trial);
  d.ldt = e->ldt;
  d.trial_fit = static_cast<T*>(e->trial_fit);
  d.F = static_cast<T*>(e->F);
  d.CR = static_cast<T*>(e->CR);
  d.slot = e->slot;
  d.idx = e->idx;
  d.jrand = e->jrand;
  d.xlen = e->xlen;
  d.rword = e->rword;
  d.woff = e->woff;
  d.wcount = e->wcount;
  d.order = e->order;
  d.win = e->win;
  d.arch_slot = e->arch_slot;
  d.owner = e->owner;
  d.succ = e->succ;
  d.wlist = e->wlist;
  d.n_push = e->d_npush;
  d.epoch = e->d_epoch;
  d.owner64 = e->d_owner64;
  d.sel_agg = e->d_sel_agg;
  d.sel_sync = e->d_sel_sync;
  d.sel_multi = (e->P > kSelSingleMax || std::getenv("EVB_DE_SELECT_MULTI") != nullptr) ? 1 : 0;
  d.archive = static_cast<T*>(e->archive);
  d.arch_size = e->d_arch_size;
  d.write_index = e->d_write_index;
  d.arch_words = e->d_arch_words;
  d.mem_f = static_cast<T*>(e->mem_f);
  d.mem_cr = static_cast<T*>(e->mem_cr);
  d.lb = T(lb);
  d.ub = T(ub);
  d.src.mode = r->mode;
  d.src.key = r->key;
  d.pk = philox_keys(r->key);
  d.src.words = r->d_words;
  d.src.n_words = r->n_words;
  d.gen_ptr = r->d_gen;
  d.cursor = r->d_cursor;
  d.overflow = r->d_overflow;
  return d;
}

// restart_run's monitored objective (hybrid/restart.hpp:55-65): per evaluation in FE order,
// best_seen improves only by more than epsilon, else since_improvement counts up
template <typename T>
__global__ void restart_monitor_kernel(const T* v, int n, double* mon, double eps) {
  if (threadIdx.x != 0) return;
  double best = mon[0], since = mon[1], evals = mon[2];
  for (int i = 0; i < n; ++i) {
    const double x = double(v[i]);
    evals += 1.0;
    if (x < __dsub_rn(best, eps)) {
      best = x;
      since = 0.0;
    } else {
      since += 1.0;
    }
  }
  mon[0] = best;
  mon[1] = since;
  mon[2] = evals;
}

// adapter means after a generation -> parameter_record (de/parameter.hpp:130-133 JADE mu,
// :186-195 SHADE mean of the memories: sequential double sum / H, cast to T)
template <typename T>
__global__ void param_trace_kernel(const T* mem_f, const T* mem_cr, int H, int shade, int* gen_out, T* mf_out,
                                   T* mc_out, int* count, int cap, int generation) {
  if (threadIdx.x != 0) return;
  T mf, mc;
  if (shade) {
    double sf = 0.0, sc = 0.0;
    for (int k = 0; k < H; ++k) sf = __dadd_rn(sf, double(mem_f[k]));
    for (int k = 0; k < H; ++k) sc = __dadd_rn(sc, double(mem_cr[k]));
    mf = T(__ddiv_rn(sf, double(H)));
    mc = T(__ddiv_rn(sc, double(H)));
  } else {
    mf = mem_f[0];
    mc = mem_cr[0];
  }
  const int n = *count;
  if (n < cap) {
    gen_out[n] = generation;
    mf_out[n] = mf;
    mc_out[n] = mc;
  }
  *count = n + 1;
}

// ---- persistent generations (K8 for one engine run: BASELINE config 2) ------------------------
// A whole sequence of generations of one engine in ONE launch: a cluster of NC CTAs, CTA c owns
// individuals [c Q, c Q + Q).  Per generation, with the engine's own arithmetic and Philox words:
//   A  fitness of every member (L2) -> (fitness, index) ranks, NaN last: top-p order (ttpb/1) or
//      the best member (best/1), redundantly in every CTA; adapter memories staged (L2 -> smem)
//   B  draws of the owned individuals (draw_scalars: the engine's sub-streams and word counts)
//   C  trial genes (binomial word per gene, donor rows of population / archive read through L2)
//   D  evaluation of the owned trials exactly as eval_small_kernel (M^T resident in shared memory,
//      sequential k with separate mul and add, base_value_pre): bit-identical to the engine
//   E  selection flags; each CTA's (pushes, successes) counts into every CTA (DSMEM)
//      -- cluster barrier --
//   F  push / success indices from the counts prefix; archive slots (victim words of the archive
//      sub-stream); last-writer-wins by 64-bit (epoch << 32 | push) maxima; success records
//      (gain, F, CR) in success order
//      -- cluster barrier --
//   G  owners replace parents (parent row -> its archive slot if it still owns it, trial -> the
//      population); CTA 0: archive size, victim-word count, SHADE / JADE memory update with the
//      reference's sequential sums (de/parameter.hpp:107-120, 166-184)
//      -- cluster barrier --
// Data other CTAs wrote during the launch is read with ld.global.cg (L2; the L1s are not coherent).
// Results are bit-identical to the same number of evb_de_generation calls.
template <typename T>
struct de_run_args {
  de_dev<T> d;
  const T* shift;
  const T* rot_t;  // M^T dense, D x D (device_problem::rot_t)
  const T* ell_w;
  int kind;
  double bias;
  int G;
  int Q;       // individuals per CTA
  double* srec;  // 3 x P: success (gain, F, CR) in success order
  unsigned long long* prof;  // EVB_DE_PERSIST_PROFILE: CTA 0's clock64 per phase (tuning aid)
};

constexpr int kRunThreads = 512;

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

template <typename T>
__global__ void __launch_bounds__(kRunThreads, 1) de_run_kernel(const de_run_args<T> a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const de_dev<T>& d = a.d;
  const int NC = int(gridDim.x), c = int(blockIdx.x);
  const int P = d.P, D = d.D, Q = a.Q;
  const int i0 = c * Q, i1 = min(P, i0 + Q), nq = max(0, i1 - i0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  const int H = max(1, d.cfg.memory_size);
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t mt_bytes = uint32_t((size_t(D) * D * sizeof(T) + 15) / 16 * 16);
  T* sMT = reinterpret_cast<T*>(smem_raw);                                     // D x D (M^T)
  T* sS = reinterpret_cast<T*>(smem_raw + mt_bytes);                            // Q x D: x - o / pre terms
  T* sZ = sS + size_t(Q) * D;                                                   // Q x D
  T* sT = sZ + size_t(Q) * D;                                                   // Q x D: owned trials
  T* sFit = sT + size_t(Q) * D;                                                 // P
  T* sMemF = sFit + P;                                                          // H
  T* sMemC = sMemF + H;                                                         // H
  T* sTf = sMemC + H;                                                           // Q
  T* sQf = sTf + Q;                                                             // Q x 2: F, CR
  T* sAll = sQf + 2 * Q;                                                        // 3 x P: every trial's fitness, F, CR
  double* sG = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sAll + 3 * P) + 15) & ~uintptr_t(15));  // 3 x P
  int NP2 = 1;
  while (NP2 < P) NP2 <<= 1;
  unsigned long long* sKey = reinterpret_cast<unsigned long long*>(sG + 3 * P);  // P order keys
  int* sIdx = reinterpret_cast<int*>(sKey + P);  // NP2 order slots + P rank counters
  int* sOwner = sIdx + NP2 + P;                  // archive_cap: last push index per archive slot
  int* sWC = sOwner + d.archive_cap;             // 2 x 32: per-warp (pushes, successes)
  int* sWin = sWC + 64;                          // Q x 2: owned individual won, its archive slot
  int* sQi = sWin + 2 * Q;                       // Q x 8: donors, jrand, first gene word
  uint64_t* bar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(sQi + 8 * Q) + 7) & ~uintptr_t(7));  // 2
  __shared__ int s_misc[4];  // [0] archive size at the generation start, [3] SHADE write index
  // adapter transcendentals of the NEXT generation, computed while the dots run (see `speculate`):
  // per owned individual kSpec Cauchy tangents, then kSpec normal offsets
  constexpr int kSpec = 3;
  __shared__ double s_pre[32 * 2 * kSpec];
  constexpr int kVict = 256;
  __shared__ int sVict[kVict];        // archive slots of the generation's first victim words
  __shared__ unsigned long long s_K;  // order key of last generation's p_count-th member
  __shared__ int s_nc;                // candidate counter of the rank phase

  if (tid == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
    s_K = ~0ull;
    s_nc = 0;
  }
  __syncthreads();
  if (tid == 0) {  // M^T once for the whole launch
    ptx::mbar_arrive_expect_tx(bar, mt_bytes);
    ptx::bulk_load(sMT, a.rot_t, mt_bytes, bar);
  }
  ptx::mbar_wait(bar, 0);
  const uint32_t gen0 = *d.gen_ptr;
  const unsigned E0 = *d.epoch;
  const bool ttpb = d.cfg.mutation == EVB_MUT_TTPB1, best = d.cfg.mutation == EVB_MUT_BEST1;
  const bool adapt = d.cfg.parameter == EVB_PAR_SHADE || d.cfg.parameter == EVB_PAR_JADE;
  const bool shade = d.cfg.parameter == EVB_PAR_SHADE;
  const int dw = (nthr >> 5) - 1;  // draw warp: lane q draws owned individual q
  philox_prefetch_reader<5> rd;    // lane q's reader of the current generation (reset one generation ahead)
  // The adapter draws (de/parameter.hpp:28-43) cost a tan, a log and a cos per individual, but
  // only `mu + 0.1 * tan(..)` and `mu + (0.1 rr) cos(..)` depend on the memories.  The memory-
  // independent factors of generation gen_n are computed here, off the critical path (threads
  // that have no dot products to do), for the first kSpec Cauchy attempts: attempt k reads word
  // b0 + k, and if it is the accepted one the normal reads words b0 + k + 1, b0 + k + 2.  The
  // draw warp then only adds, compares and skips words; an individual whose first kSpec attempts
  // all fail (p ~ 2.5e-4 at mu = 0.5) falls back to the sequential draws.  Same operations and
  // roundings as draw_cauchy / draw_normal (rng.cuh), so F, CR and the word counts are identical.
  auto speculate = [&](uint32_t gen_n) {
    const int b0 = shade ? 1 : 0;
    if (warp == dw) {
      if (lane < nq) rd.reset(d.src.key, (uint64_t(gen_n) << 32) | uint32_t(i0 + lane));
    } else if (warp == dw - 1 || warp == dw - 4 || warp == dw - 5) {
      // (three warps of the two SM sub-partitions that hold the fewest dot-product warps)
      const int wl = warp == dw - 5 ? 0 : (warp == dw - 4 ? 1 : 2);
      for (int e = wl * 32 + lane; e < 2 * kSpec * nq; e += 96) {
        const int q = e / (2 * kSpec), r = e - q * 2 * kSpec;
        const uint64_t ctr = (uint64_t(gen_n) << 32) | uint32_t(i0 + q);
        double v;
        if (r < kSpec) {
          const double u = u01pos_of(philox_word(d.src.key, ctr, uint64_t(b0 + r)));
          v = tan(__dmul_rn(3.14159265358979323846, __dsub_rn(u, 0.5)));
        } else {
          const int k = r - kSpec;
          const double u1 = u01pos_of(philox_word(d.src.key, ctr, uint64_t(b0 + k + 1)));
          const double u2 = u01_of(philox_word(d.src.key, ctr, uint64_t(b0 + k + 2)));
          const double rr = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
          v = __dmul_rn(__dmul_rn(0.1, rr), cos(__dmul_rn(2.0 * 3.14159265358979323846, u2)));
        }
        s_pre[e] = v;
      }
    }
  };
  if (adapt) speculate(gen0);
  cl.sync();  // every CTA's shared memory exists before the first DSMEM write
  long long t_last = clock64();
  auto mark = [&](int k) {  // phase boundary (after a barrier): CTA 0 thread 0 accumulates cycles
    if (a.prof && c == 0 && tid == 0) {
      const long long t = clock64();
      a.prof[k] += (unsigned long long)(t - t_last);
      t_last = t;
    }
  };

  for (int g = 0; g < a.G; ++g) {
    const uint32_t gen = gen0 + uint32_t(g);
    // ---- A: fitness, order, adapter memories, archive size ----
    // (read from L2 once; later generations get them pushed into every CTA's copy over DSMEM by
    // the CTA that changed them, phase G)
    if (g == 0) {
      for (int t = tid; t < P; t += nthr) sFit[t] = ldcg(d.fit + t);
      if (adapt)
        for (int t = tid; t < H; t += nthr) {
          sMemF[t] = ldcg(d.mem_f + t);
          sMemC[t] = ldcg(d.mem_cr + t);
        }
      if (tid == 0) {
        s_misc[0] = ldcg(d.arch_size);
        s_misc[3] = adapt ? ldcg(d.write_index) : 0;
      }
      __syncthreads();
    }
    mark(11);
    // the last warp draws for the owned individuals (adapter sample, mutation indices, jrand:
    // draw_scalars' order and word counts) while the other warps rank the population (named
    // barrier 1 over them); a donor picked by rank (best/1, current-to-pbest) is kept as a rank
    // and resolved once the order exists
    de_dev<T> dl = d;
    dl.mem_f = sMemF;
    dl.mem_cr = sMemC;
    const int arch_size = s_misc[0];
    T dF = T(0), dCR = T(0);
    int dslot = -1, da = 0, db = 0, dc = 0, djr = 0;
    if (warp == dw) {
      if (lane < nq) {
        const int i = i0 + lane;
        if (adapt) {  // finish the speculated draws: sample_scale_factor / sample_crossover_rate
          if (shade) dslot = draw_int(rd, d.cfg.memory_size);
          const double muf = double(sMemF[shade ? dslot : 0]), muc = double(sMemC[shade ? dslot : 0]);
          const double* pre = s_pre + lane * 2 * kSpec;
          double f = 0.0;
          int k = 0;
          bool ok = false;
          for (; k < kSpec; ++k) {
            rd.next();  // the attempt's word
            f = __dadd_rn(muf, __dmul_rn(0.1, pre[k]));
            if (f > 0.0) {
              ok = true;
              break;
            }
          }
          if (!ok)
            for (int attempt = kSpec; attempt < 100; ++attempt) {
              f = draw_cauchy(rd, muf, 0.1);
              if (f > 0.0) break;
            }
          if (f <= 0.0) f = 0.1;
          dF = T(fmin(f, 1.0));
          double v;
          if (ok) {
            rd.next();
            rd.next();
            v = __dadd_rn(muc, pre[kSpec + k]);
          } else {
            v = draw_normal(rd, muc, 0.1);
          }
          dCR = T(v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v));
        } else {
          rd.reset(d.src.key, (uint64_t(gen) << 32) | uint32_t(i));
          draw_adapter<T>(dl, rd, dF, dCR, dslot);
        }
        // draw_mutation's draws (de/strategy.hpp:84-86, 107-110, 143-152, 187); da is a rank for
        // best/1 and current-to-pbest
        if (best) {
          da = 0;
          do { db = draw_int(rd, P); } while (db == i);
          do { dc = draw_int(rd, P); } while (dc == i || dc == db);
        } else if (ttpb) {
          da = draw_int(rd, d.p_count);
          do { db = draw_int(rd, P); } while (db == i);
          const int pool = P + (d.cfg.use_archive ? arch_size : 0);
          do { dc = draw_int(rd, pool); } while (dc == i || dc == db);
        } else {
          do { da = draw_int(rd, P); } while (da == i);
          do { db = draw_int(rd, P); } while (db == i || db == da);
          do { dc = draw_int(rd, P); } while (dc == i || dc == da || dc == db);
        }
        djr = draw_int(rd, D);
        sQi[8 * lane + 0] = da;
        sQi[8 * lane + 1] = db;
        sQi[8 * lane + 2] = dc;
        sQi[8 * lane + 3] = djr;
        sQi[8 * lane + 4] = int(rd.count);
        sQf[2 * lane] = dF;
        sQf[2 * lane + 1] = dCR;
      }
    } else if (ttpb || best) {
      // (fitness, index) ranks, NaN last.  Only the first p_count ranks are needed, and a member's
      // key never increases inside the launch (a trial replaces its parent only when it is <=), so
      // the key K of last generation's p_count-th member bounds this generation's: the candidates
      // {key <= K} hold every member that precedes any of them, and ranks among the candidates are
      // ranks in the population.  Generation 0 ranks everybody.  Thread (candidate, chunk) counts
      // the candidates of its chunk that precede it on order_key (integer shared atomics).
      const int nr = nthr - 32;
      int* sCand = reinterpret_cast<int*>(sG);  // the success records' space is free until phase G
      const bool narrow = g > 0;
      const unsigned long long K = s_K;
      for (int t = tid; t < P; t += nr) {
        sIdx[NP2 + t] = 0;  // rank counters (after the order slots)
        const unsigned long long key = order_key(sFit[t]);
        sKey[t] = key;
        if (!narrow || key <= K) sCand[atomicAdd(&s_nc, 1)] = t;
      }
      ptx::named_bar_sync(1, nr);
      const int C = s_nc;
      const int nch = max(1, min(8, nr / C));
      for (int t = tid; t < C * nch; t += nr) {
        const int ch = t / C, ci = t - ch * C;
        const int j0 = (C * ch) / nch, j1 = (C * (ch + 1)) / nch;
        const int i = sCand[ci];
        const unsigned long long ki = sKey[i];
        int cnt = 0;
#pragma unroll 4
        for (int cj = j0; cj < j1; ++cj) {
          const int j = sCand[cj];
          const unsigned long long kj = sKey[j];
          cnt += (kj < ki || (kj == ki && j < i)) ? 1 : 0;
        }
        if (cnt) atomicAdd(&sIdx[NP2 + i], cnt);
      }
      ptx::named_bar_sync(1, nr);
      for (int ci = tid; ci < C; ci += nr) {
        const int i = sCand[ci];
        const int rk = sIdx[NP2 + i];
        if (rk < d.p_count) sIdx[rk] = i;
      }
      ptx::named_bar_sync(1, nr);
      if (tid == 0) {
        s_K = sKey[sIdx[d.p_count - 1]];
        s_nc = 0;
      }
    }
    __syncthreads();
    mark(0);
    // ---- B: donors picked by rank, the engine's exported draws ----
    const bool a_by_rank = ttpb || best;
    if (warp == dw && lane < nq) {
      const int i = i0 + lane;
      d.F[i] = dF;
      d.CR[i] = dCR;
      d.slot[i] = dslot;
      d.idx[4 * i + 0] = a_by_rank ? sIdx[da] : da;
      d.idx[4 * i + 1] = db;
      d.idx[4 * i + 2] = dc;
      d.jrand[i] = djr;
      d.woff[i] = rd.count;
      d.rword[i] = rd.count + D;
      d.wcount[i] = rd.count + D;
    }
    mark(1);
    // ---- C: trial genes (binomial, de_trial_kernel's arithmetic) ----
    // thread = (owned individual, NBT Philox blocks = 2 NBT gene words): its target / donor genes
    // come straight from L2 (every load of the CTA in flight at once) while the words are computed.
    // One block per thread while the CTA has a thread per block (the shorter chain), else two.
    auto trial = [&](auto nbt_tag) {
      constexpr int NBT = decltype(nbt_tag)::value, NG = 2 * NBT;
      const int NB = D / 2 + 1;              // blocks covering D gene words at any offset parity
      const int NB2 = (NB + NBT - 1) / NBT;  // threads per individual
      for (int e = tid; e < nq * NB2; e += nthr) {
        const int q = e / NB2, b2 = e - q * NB2;
        const int i = i0 + q;
        const int64_t s0 = sQi[8 * q + 4];
        const int64_t blk0 = s0 >> 1;
        const int64_t nblk = ((s0 + D + 1) >> 1) - blk0;
        const int ic = sQi[8 * q + 2];
        const int ia = a_by_rank ? sIdx[sQi[8 * q + 0]] : sQi[8 * q + 0];
        const T* xi = d.pop + size_t(i) * d.ldp;
        const T* xa = d.pop + size_t(ia) * d.ldp;
        const T* xb = d.pop + size_t(sQi[8 * q + 1]) * d.ldp;
        const T* xc = (ttpb && ic >= P) ? d.archive + size_t(ic - P) * d.ldt : d.pop + size_t(ic) * d.ldp;
        int jj[NG];
        T gi[NG], ga[NG], gb[NG], gc[NG];
#pragma unroll
        for (int u = 0; u < NG; ++u) {
          const int64_t b = NBT * b2 + (u >> 1);
          const int64_t j64 = 2 * (blk0 + b) + (u & 1) - s0;
          const bool valid = b < nblk && j64 >= 0 && j64 < D;
          jj[u] = valid ? int(j64) : -1;
          const int j = valid ? int(j64) : 0;
          gi[u] = ldcg(xi + j);
          ga[u] = ldcg(xa + j);
          gb[u] = ldcg(xb + j);
          gc[u] = ldcg(xc + j);
        }
        const T Fi = sQf[2 * q];
        const double cr = double(sQf[2 * q + 1]);
        const int jr = sQi[8 * q + 3];
        uint64_t w[NG];
        const uint64_t ctr = (uint64_t(gen) << 32) | uint32_t(i);
#pragma unroll
        for (int u = 0; u < NBT; ++u)
          philox_pair(d.src.key, ctr, uint64_t(blk0 + NBT * b2 + u), w[2 * u], w[2 * u + 1]);
#pragma unroll
        for (int u = 0; u < NG; ++u) {
          const int j = jj[u];
          if (j < 0) continue;
          const T xij = gi[u];
          T v;
          if (u01_of(w[u]) < cr || j == jr)
            v = donor_gene<T>(d.cfg.mutation, xij, ga[u], gb[u], gc[u], Fi);
          else
            v = xij;
          if (d.cfg.repair == EVB_REP_CLIP) {
            if (v < d.lb) v = d.lb;
            if (v > d.ub) v = d.ub;
          } else if (v < d.lb || v > d.ub) {
            v = repair_gene<T>(d.cfg.repair, v, xij, d.lb, d.ub);
          }
          sT[q * D + j] = v;
          sS[q * D + j] = fop<T>::sub(v, a.shift[j]);  // x - o for the evaluation (eval_small's rounding)
        }
      }
    };
    if (nq * (D / 2 + 1) <= nthr) trial(std::integral_constant<int, 1>{});
    else trial(std::integral_constant<int, 2>{});
    __syncthreads();
    mark(2);
    // ---- D: evaluation, eval_small_kernel's order ----
    mark(8);
    if (adapt && g + 1 < a.G) speculate(gen + 1u);  // warps with no (or the fewest) dot products
    {  // thread = (row r, a group of up to QG owned individuals): M^T[k][r] is loaded once per k for
       // all of them, s[q][k .. k+1] are 16-byte broadcasts; every chain keeps the reference's
       // sequential k order (separate mul and add)
      constexpr int QG = 4;
      const int ngr = (nq + QG - 1) / QG;
      for (int t = tid; t < D * ngr; t += nthr) {
        const int r = t % D, gq = t / D;
        const int q0 = gq * QG;
        const int nv = min(QG, nq - q0);
        const T* mcol = sMT + r;
        T acc[QG];
        const T* sv[QG];
#pragma unroll
        for (int u = 0; u < QG; ++u) {
          acc[u] = T(0);
          sv[u] = sS + (q0 + min(u, nv - 1)) * D;
        }
        int k = 0;
        if constexpr (sizeof(T) == 8) {
          if ((D & 1) == 0)
            for (; k + 2 <= D; k += 2) {
              const T m0 = mcol[k * D], m1 = mcol[(k + 1) * D];
#pragma unroll
              for (int u = 0; u < QG; ++u) {
                const double2 x = *reinterpret_cast<const double2*>(sv[u] + k);
                acc[u] = fop<T>::add(acc[u], fop<T>::mul(m0, x.x));
                acc[u] = fop<T>::add(acc[u], fop<T>::mul(m1, x.y));
              }
            }
        }
        for (; k < D; ++k) {
          const T mk = mcol[k * D];
#pragma unroll
          for (int u = 0; u < QG; ++u) acc[u] = fop<T>::add(acc[u], fop<T>::mul(mk, sv[u][k]));
        }
#pragma unroll
        for (int u = 0; u < QG; ++u)
          if (u < nv) sZ[(q0 + u) * D + r] = acc[u];
      }
    }
    __syncthreads();
    mark(9);
    if (kind_has_pre(a.kind)) {
      const int dq = nthr / D, dj = nthr - dq * D;
      int q = tid / D, j = tid - q * D;  // (q, j) of element e = tid, advanced by nthr without division
      for (; q < nq;) {
        const T* zr = sZ + q * D;
        auto z = [&](int qq) { return zr[qq]; };
        sS[q * D + j] = base_pre_term<T, false>(a.kind, D, z, j);
        q += dq;
        j += dj;
        if (j >= D) {
          j -= D;
          ++q;
        }
      }
      __syncthreads();
    }
    mark(10);
    // base values: one thread per owned individual runs the reference's sequential sums; Ackley's
    // two sums (squares, cosines) are independent chains and take two adjacent lanes.
    if (a.kind == EVB_ACKLEY && 2 * nq <= 32) {
      if (warp == 0) {
        const int q = min(lane >> 1, max(nq - 1, 0)), role = lane & 1;
        const T* src = (role ? sS : sZ) + q * D;
        T acc = T(0);
        int j = 0;
        for (; j + 8 <= D; j += 8) {  // loads and squares ahead of the sequential adds
          T v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = src[j + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = role ? v[u] : fop<T>::mul(v[u], v[u]);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = fop<T>::add(acc, v[u]);
        }
        for (; j < D; ++j) acc = fop<T>::add(acc, role ? src[j] : fop<T>::mul(src[j], src[j]));
        const T other = __shfl_xor_sync(0xffffffffu, acc, 1);
        if (!role && (lane >> 1) < nq) {
          const T v = fop<T>::add(ackley_final<T>(acc, other, D), T(a.bias));
          sTf[q] = v;
          d.trial_fit[i0 + q] = v;
        }
      }
    } else if (tid < nq) {
      const T* zrow = sZ + tid * D;
      const T* pe = sS + tid * D;
      auto z = [&](int qq) { return zrow[qq]; };
      auto pre = [&](int qq) { return pe[qq]; };
      const T v = fop<T>::add(base_value_pre<T, false>(a.kind, D, z, pre, a.ell_w), T(a.bias));
      sTf[tid] = v;
      d.trial_fit[i0 + tid] = v;
    }
    __syncthreads();
    mark(3);
    // ---- E: trial fitness, F, CR of the owned individuals into every CTA's copy (DSMEM) ----
    for (int e = tid; e < nq * NC; e += nthr) {
      const int q = e / NC, dst = e - q * NC;
      T* all = cl.map_shared_rank(sAll, dst);
      all[i0 + q] = sTf[q];
      all[P + i0 + q] = sQf[2 * q];
      all[2 * P + i0 + q] = sQf[2 * q + 1];
    }
    // cluster barrier split into arrive / wait: the archive sub-stream's first victim words
    // (needed once the archive is full: de/strategy.hpp:33-36) are computed while the other
    // CTAs' values arrive
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    const int room0 = d.archive_cap - arch_size;
    const bool victims = d.archive_cap > 0 && room0 < P && d.src.mode == RNG_PHILOX;  // CTA-uniform
    if (victims)
      for (int t = tid; t < min(P - max(room0, 0), kVict); t += nthr)
        sVict[t] = uint_of(philox_word(d.src.key, (uint64_t(gen) << 32) | kSubArchive, uint64_t(t)), d.archive_cap);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (victims) __syncthreads();
    mark(4);
    // ---- F: every CTA resolves the whole selection in its own shared memory ----
    // thread = individual: win / success flags (de/engine.hpp:27-47), push and success indices by
    // index-order prefix sums, archive slots (de/strategy.hpp:29-37: free slots first, then the
    // archive sub-stream's victim words), the last push into a slot wins it (shared atomicMax),
    // success records (gain, F, CR) in success order.  Same values in every CTA, no exchange.
    const int size0 = arch_size, room = d.archive_cap - size0;
    bool wq = false, sq = false;
    T ft = T(0), fp = T(0);
    if (tid < P) {
      ft = sAll[tid];
      fp = sFit[tid];
      wq = ft <= fp;
      sq = wq && fop<T>::sub(fp, ft) > T(0);
    }
    for (int t = tid; t < d.archive_cap; t += nthr) sOwner[t] = -1;
    const unsigned wmask = __ballot_sync(0xffffffffu, wq), smask = __ballot_sync(0xffffffffu, sq);
    if (lane == 0 && warp * 32 < P) {
      sWC[2 * warp] = __popc(wmask);
      sWC[2 * warp + 1] = __popc(smask);
    }
    __syncthreads();
    int pw = 0, ps = 0, tw = 0, ts = 0;
    for (int k = 0; k < (P + 31) / 32; ++k) {  // the warps that hold individuals
      const int a0 = sWC[2 * k], a1 = sWC[2 * k + 1];
      if (k < warp) {
        pw += a0;
        ps += a1;
      }
      tw += a0;
      ts += a1;
    }
    const int qidx = pw + __popc(wmask & ((1u << lane) - 1u));
    const int kidx = ps + __popc(smask & ((1u << lane) - 1u));
    int sl = -1;
    if (wq && d.archive_cap > 0) {
      if (qidx < room) {
        sl = size0 + qidx;
      } else {
        const int n = qidx - max(room, 0);
        const uint64_t ctr_hi = (uint64_t(gen) << 32) | kSubArchive;
        sl = (victims && n < kVict) ? sVict[n] : uint_of(word_at(d.src, ctr_hi, int64_t(n), d.overflow), d.archive_cap);
      }
      atomicMax(&sOwner[sl], qidx);
    }
    if (sq) {
      sG[kidx] = double(fop<T>::sub(fp, ft));
      sG[P + kidx] = double(sAll[P + tid]);
      sG[2 * P + kidx] = double(sAll[2 * P + tid]);
    }
    if (tid >= i0 && tid < i1) sWin[2 * (tid - i0)] = wq ? 1 : 0;
    __syncthreads();
    mark(5);
    if (wq) {  // (tid < P)
      sFit[tid] = ft;
      if (tid >= i0 && tid < i1) {
        // overwritten by a later push: members_[victim] = genome, in push order
        sWin[2 * (tid - i0) + 1] = (sl >= 0 && sOwner[sl] == qidx) ? sl : -1;
        d.fit[tid] = ft;
      }
    }
    if (tid == 0) s_misc[0] = min(d.archive_cap, size0 + tw);  // the next generation's archive size
    __syncthreads();
    // ---- G: the owned winners' rows; the adapter memories (last warp, every CTA the same) ----
    if (warp != dw || !adapt) {
      const int nw = (nthr >> 5) - (adapt ? 1 : 0);
      for (int q = warp; q < nq; q += nw) {
        if (!sWin[2 * q]) continue;
        const int i = i0 + q;
        const int wsl = sWin[2 * q + 1];
        T* x = d.pop + size_t(i) * d.ldp;
        T* arow = wsl >= 0 ? d.archive + size_t(wsl) * d.ldt : nullptr;
        for (int j = lane; j < D; j += 32) {
          if (arow) arow[j] = ldcg(x + j);
          x[j] = sT[q * D + j];
        }
      }
      if (c == 0 && tid == 0) {
        *d.arch_size = min(d.archive_cap, size0 + tw);
        *d.arch_words = d.archive_cap > 0 ? max(0, tw - room) : 0;
        d.n_push[0] = tw;
        d.n_push[1] = ts;
      }
    } else if (ts > 0) {
      // de/parameter.hpp:166-184 (SHADE, adapter_update's roundings) / :107-120 (JADE): the
      // reference's sequential sums, one chain per lane where the chains are independent
      const int n_succ = ts;
      const double* gv = sG;
      const double* fv = sG + P;
      const double* cv = sG + 2 * P;
      if (shade) {
        double gain_sum = 0.0;
        if (lane == 0)
          for (int k = 0; k < n_succ; ++k) gain_sum = __dadd_rn(gain_sum, gv[k]);
        gain_sum = __shfl_sync(0xffffffffu, gain_sum, 0);
        // per-success products by their own lanes, in place (w = gain / sum; (w f) f, w f, w cr)
        double* wnum = sG;
        for (int k = lane; k < n_succ; k += 32) {
          const double w = __ddiv_rn(gv[k], gain_sum);
          const double wf = __dmul_rn(w, fv[k]);
          wnum[k] = __dmul_rn(wf, fv[k]);
          wnum[P + k] = wf;
          wnum[2 * P + k] = __dmul_rn(w, cv[k]);
        }
        __syncwarp();
        double acc = 0.0;  // lane 0: f_num, lane 1: f_den, lane 2: cr
        if (lane < 3)
          for (int k = 0; k < n_succ; ++k) acc = __dadd_rn(acc, wnum[lane * P + k]);
        const double f_num = __shfl_sync(0xffffffffu, acc, 0), f_den = __shfl_sync(0xffffffffu, acc, 1);
        const double cr_acc = __shfl_sync(0xffffffffu, acc, 2);
        if (lane == 0) {
          const int kw = s_misc[3];
          const T nf = T(__ddiv_rn(f_num, f_den)), nc = T(cr_acc);
          sMemF[kw] = nf;
          sMemC[kw] = nc;
          s_misc[3] = (kw + 1) % d.cfg.memory_size;
          if (c == 0) {
            d.mem_f[kw] = nf;
            d.mem_cr[kw] = nc;
            *d.write_index = (kw + 1) % d.cfg.memory_size;
          }
        }
      } else if (lane == 0) {
        double num = 0.0, den = 0.0, crm = 0.0;
        for (int k = 0; k < n_succ; ++k) {
          num = __dadd_rn(num, __dmul_rn(fv[k], fv[k]));
          den = __dadd_rn(den, fv[k]);
          crm = __dadd_rn(crm, cv[k]);
        }
        const double lehmer = __ddiv_rn(num, den);
        crm = __ddiv_rn(crm, double(n_succ));
        const double cc = double(T(d.cfg.jade_c));
        const T nf = T(__dadd_rn(__dmul_rn(__dsub_rn(1.0, cc), double(sMemF[0])), __dmul_rn(cc, lehmer)));
        const T nc = T(__dadd_rn(__dmul_rn(__dsub_rn(1.0, cc), double(sMemC[0])), __dmul_rn(cc, crm)));
        sMemF[0] = nf;
        sMemC[0] = nc;
        if (c == 0) {
          d.mem_f[0] = nf;
          d.mem_cr[0] = nc;
        }
      }
    }
    mark(6);
    cl.sync();
    mark(7);
  }
  if (c == 0 && tid == 0) {
    *d.gen_ptr = gen0 + uint32_t(a.G);
    *d.epoch = E0 + unsigned(a.G);
  }
}

template <typename T>
void reduce_t(evb_de_s* e, void* pop, int64_t ldp, void* fit, evb_rng_s* r, cudaStream_t st);

int sm_count_cached() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    EVB_CUDA(cudaGetDevice(&dev));
    EVB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

template <typename T>
void generation_t(evb_de_s* e, const device_problem* prob, evb_scratch_s* sc, void* pop, int64_t ldp, void* fit,
                  double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  de_dev<T> d = make_dev<T>(e, pop, ldp, fit, lb, ub, r);
  e->gen_P = e->P;
  e->phases.begin(st);
  if (e->cfg.mutation == EVB_MUT_BEST1) {
    EVB_CUDA(launch_pdl(de_best_kernel<T>, dim3(1), dim3(1024), 0, st, d));
    count_launch();
  } else if (e->cfg.mutation == EVB_MUT_TTPB1) {
    if (e->P <= kSortMax && std::getenv("EVB_DE_ORDER_RANK") == nullptr) {
      int n2 = 1;
      while (n2 < e->P) n2 <<= 1;
      const size_t smem = size_t(n2) * (sizeof(unsigned long long) + sizeof(int));
      static bool attr = false;
      if (!attr) {  // up to 192 KB of (key, index) pairs
        EVB_CUDA(cudaFuncSetAttribute(de_sort_order_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kSortMax) * 12)));
        EVB_CUDA(cudaFuncSetAttribute(de_sort_order_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kSortMax) * 12)));
        attr = true;
      }
      EVB_CUDA(launch_pdl(de_sort_order_kernel<T>, dim3(1), dim3(std::min(1024, std::max(32, n2 / 2))), smem, st, d,
                          n2));
    } else {
      const int th = 256;
      EVB_CUDA(launch_pdl(de_order_kernel<T>, dim3((e->P + th - 1) / th), dim3(th), th * sizeof(T), st, d));
    }
    count_launch();
  }
  e->phases.mark(st);
  if (r->mode == RNG_PHILOX) {
    EVB_CUDA(launch_pdl(de_draw_philox_kernel<T>, dim3((e->P + 127) / 128), dim3(128), 0, st, d));
  } else {
    de_draw_words_kernel<T><<<1, 32, 0, st>>>(d);
  }
  count_launch();
  e->phases.mark(st);
  {
    const int th = std::min(256, int(round_up((e->D + 2) / 2 + 1, 32)));
    // warp per individual with 16-byte rows where the rows allow it (the population and the
    // archive / trial rows, which the engine pitches to 16 bytes)
    // (small populations keep the block-per-individual kernel: one Philox block per thread and
    // no run-ahead windows, the shorter dependent chain when the whole generation is latency)
    const bool vec = r->mode == RNG_PHILOX && e->cfg.crossover == EVB_CX_BINOMIAL &&
                     (int64_t(e->P) * e->D >= (int64_t(1) << 18) || std::getenv("EVB_DE_TRIAL_VEC") != nullptr) &&
                     (ldp * int64_t(sizeof(T))) % 16 == 0 && reinterpret_cast<uintptr_t>(pop) % 16 == 0 &&
                     std::getenv("EVB_DE_TRIAL_SCALAR") == nullptr;
    if (vec) {
      // column blocks (EVB_DE_TRIAL_COLBLOCKS: rows split into that many blocks of whole 512-byte
      // chunks, grid.y; default whole rows)
      const int wchunk = 32 * (16 / int(sizeof(T)));
      const int nchunks = (e->D + wchunk - 1) / wchunk;
      const int64_t pop_bytes = int64_t(e->P) * ldp * int64_t(sizeof(T));
      // (measured with the staged kernel at P = 16384, D = 1000: whole rows 71.7 us, 4 blocks 78.9 us;
      // the L2 saving is real — DRAM reads 290 -> 136 MB — but the extra per-block windows cost more)
      int ncb = 1;
      if (const char* s = std::getenv("EVB_DE_TRIAL_COLBLOCKS")) ncb = std::max(1, std::atoi(s));
      ncb = std::min(ncb, nchunks);
      ncb = (nchunks + (nchunks + ncb - 1) / ncb - 1) / ((nchunks + ncb - 1) / ncb);  // no empty block
      const dim3 g((e->P + kTrialVecWarps - 1) / kTrialVecWarps, ncb), bl(32 * kTrialVecWarps);
      // (EVB_DE_TRIAL_MINB, tuning: resident blocks per SM the register cap targets)
      const int minb = std::getenv("EVB_DE_TRIAL_MINB") ? std::atoi(std::getenv("EVB_DE_TRIAL_MINB")) : 4;
      const bool clip = e->cfg.repair == EVB_REP_CLIP;
#define EVB_TRIAL_VEC(MUT, CLIP)                                                                          \
  (minb >= 6 ? de_trial_vec_kernel<T, MUT, CLIP, 6>                                                      \
             : minb == 5 ? de_trial_vec_kernel<T, MUT, CLIP, 5> : de_trial_vec_kernel<T, MUT, CLIP, 4>)
      auto kern = e->cfg.mutation == EVB_MUT_TTPB1 ? (clip ? EVB_TRIAL_VEC(EVB_MUT_TTPB1, true)
                                                           : EVB_TRIAL_VEC(EVB_MUT_TTPB1, false))
                                                   : (clip ? EVB_TRIAL_VEC(EVB_MUT_RAND1, true)
                                                           : EVB_TRIAL_VEC(EVB_MUT_RAND1, false));
#undef EVB_TRIAL_VEC
      // rows staged through shared memory where the population exceeds ~40 MB
      // (EVB_DE_TRIAL_STAGE=0/1 overrides; EVB_DE_TRIAL_STAGES = ring depth 2..4)
      bool staged = pop_bytes > (int64_t(40) << 20);
      if (const char* s = std::getenv("EVB_DE_TRIAL_STAGE")) staged = std::atoi(s) != 0;
      if (staged) {
        const int ns = std::getenv("EVB_DE_TRIAL_STAGES") ? std::atoi(std::getenv("EVB_DE_TRIAL_STAGES")) : 3;
#define EVB_TRIAL_STG(MUT, CLIP)                                                                      \
  (ns <= 2 ? de_trial_stage_kernel<T, MUT, CLIP, 2, 4>                                                 \
           : ns == 3 ? de_trial_stage_kernel<T, MUT, CLIP, 3, 4> : de_trial_stage_kernel<T, MUT, CLIP, 4, 3>)
        auto ks = e->cfg.mutation == EVB_MUT_TTPB1 ? (clip ? EVB_TRIAL_STG(EVB_MUT_TTPB1, true)
                                                           : EVB_TRIAL_STG(EVB_MUT_TTPB1, false))
                                                   : (clip ? EVB_TRIAL_STG(EVB_MUT_RAND1, true)
                                                           : EVB_TRIAL_STG(EVB_MUT_RAND1, false));
#undef EVB_TRIAL_STG
        const size_t smem = size_t(kTrialVecWarps) * std::max(2, std::min(4, ns)) * 2048;
        EVB_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        EVB_CUDA(launch_pdl(ks, g, bl, smem, st, d));
      } else {
        EVB_CUDA(launch_pdl(kern, g, bl, 0, st, d));
      }
    } else if (e->cfg.crossover == EVB_CX_EXPONENTIAL)
      EVB_CUDA(launch_pdl(de_trial_kernel<T, EVB_CX_EXPONENTIAL>, dim3(e->P), dim3(th), 0, st, d));
    else
      EVB_CUDA(launch_pdl(de_trial_kernel<T, EVB_CX_BINOMIAL>, dim3(e->P), dim3(th), 0, st, d));
    count_launch();
    if (e->cfg.repair == EVB_REP_REINITIALIZE) {
      de_reinit_kernel<T><<<e->P, std::max(32, std::min(256, int(round_up(e->D, 32)))), 0, st>>>(d);
      count_launch();
    }
  }
  EVB_CUDA(cudaGetLastError());
  e->phases.mark(st);
  // evaluate the trials with the scalar path's semantics (problem.evaluate via individual::evaluate)
  eval_request rq{};
  rq.prob = prob;
  rq.scratch = sc;
  rq.X = e->trial;
  rq.n = e->P;
  rq.ldx = e->ldt;
  rq.out = e->trial_fit;
  rq.ldo = e->P;
  rq.n_out = 1;
  rq.kinds[0] = prob->kind;
  rq.biases[0] = prob->bias;
  rq.stream = st;
  rq.scalar_trig = true;
  eval_dispatch(rq);
  if (e->rec) recorder_observe(e->rec, e->rec_run, e->trial_fit, e->P, st);  // trials in FE (i) order
  if (e->mon_on) {
    restart_monitor_kernel<T><<<1, 32, 0, st>>>(static_cast<const T*>(e->trial_fit), e->P, e->d_mon, e->mon_eps);
    count_launch();
  }
  e->phases.mark(st);
  if (d.sel_multi) {
    const int blocks = (e->P + kSelBlockItems - 1) / kSelBlockItems;
    EVB_CUDA(launch_pdl(de_select_multi_kernel<T>, dim3(blocks), dim3(kSelBlockThreads), 0, st, d));
    count_launch();
    if (e->cfg.parameter == EVB_PAR_SHADE || e->cfg.parameter == EVB_PAR_JADE) {
      EVB_CUDA(launch_pdl(de_adapt_kernel<T>, dim3(1), dim3(kSelThreads), 0, st, d));
      count_launch();
    }
  } else {
    EVB_CUDA(launch_pdl(de_select_scan_kernel<T>, dim3(1), dim3(kSelThreads), 0, st, d));
    count_launch();
  }
  e->phases.mark(st);
  {
    const int vec = (ldp * int64_t(sizeof(T))) % 16 == 0 && reinterpret_cast<uintptr_t>(pop) % 16 == 0 ? 1 : 0;
    const int blocks = std::max(1, std::min((e->P + 7) / 8, 4 * sm_count_cached()));
    if (d.sel_multi) {
      EVB_CUDA(launch_pdl(de_select_apply_kernel<T>, dim3(blocks), dim3(256), 0, st, d, vec, 1));
    } else {
      const int th = std::min(256, int(round_up(e->D, 32)));
      EVB_CUDA(launch_pdl(de_select_apply_kernel<T>, dim3(e->P), dim3(th), 0, st, d, vec, 0));
    }
    count_launch();
  }
  e->phases.mark(st);
  EVB_CUDA(cudaGetLastError());
  e->fes += e->P;  // st.add_fes(1) per trial (de/engine.hpp:88)
  ++e->gen_count;
  if (e->ptrace && (e->cfg.parameter == EVB_PAR_SHADE || e->cfg.parameter == EVB_PAR_JADE)) {
    evb_param_trace_s* t = e->ptrace;
    const size_t off = size_t(e->ptrace_run) * t->cap;
    param_trace_kernel<T><<<1, 32, 0, st>>>(static_cast<const T*>(e->mem_f), static_cast<const T*>(e->mem_cr),
                                            e->cfg.memory_size, e->cfg.parameter == EVB_PAR_SHADE ? 1 : 0,
                                            t->gen + off, static_cast<T*>(t->mu_f) + off,
                                            static_cast<T*>(t->mu_cr) + off, t->count + e->ptrace_run, t->cap,
                                            e->gen_offset + e->gen_count);
    count_launch();
  }
  reduce_t<T>(e, pop, ldp, fit, r, st);
  e->last_gen = r->gen;
  r->gen++;
}

// ---- population reduction (L-SHADE, de/policy.hpp:40-60) + archive shrink ------------------
// reduce_population removes the worst member (fitness >=, so ties remove the higher index) until
// the scheduled size: the survivors are exactly the members of (fitness, index) rank < target,
// kept in their order (erase_member).
// reduce_population (de/policy.hpp:44-60): while size > target, remove `worst` from the
// sequential scan worst = 0; for i: if f[i] >= f[worst] worst = i, over the current members.
// Closed form of one scan: the head when its fitness is NaN (nothing compares >= NaN), else the
// last index of the maximum over the non-NaN members (a NaN member never satisfies >=).  One
// block repeats that reduction once per removal; rank[i] = 0 marks a survivor, `target` a
// removed member (the gather kernel keeps rank < target).  NaN-free populations: exactly the
// members of (fitness, index) rank >= target.
template <typename T>
__global__ void __launch_bounds__(1024) de_reduce_mark_kernel(const T* fit, int P, int target, int* rank) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  T* sf = reinterpret_cast<T*>(smem_raw);
  uint8_t* alive = smem_raw + sizeof(T) * size_t(P);
  __shared__ T wf[32];
  __shared__ int wi[32], wh[32];
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    sf[i] = fit[i];
    alive[i] = 1;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  // (f2, i2) replaces (f, i) as the scan's worst: larger fitness, or equal fitness at a later index
  auto merge = [](T& f, int& i, T f2, int i2) {
    if (i2 >= 0 && (i < 0 || f2 > f || (f2 == f && i2 > i))) {
      f = f2;
      i = i2;
    }
  };
  for (int r = target; r < P; ++r) {
    T bf = T(0);
    int bi = -1, head = P;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (!alive[i]) continue;
      head = min(head, i);
      if (!isnan(sf[i])) merge(bf, bi, sf[i], i);
    }
    for (int off = 16; off > 0; off >>= 1) {
      const T of = __shfl_xor_sync(0xffffffffu, bf, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      head = min(head, __shfl_xor_sync(0xffffffffu, head, off));
      merge(bf, bi, of, oi);
    }
    if (lane == 0) {
      wf[w] = bf;
      wi[w] = bi;
      wh[w] = head;
    }
    __syncthreads();
    if (w == 0) {
      bf = lane < nw ? wf[lane] : T(0);
      bi = lane < nw ? wi[lane] : -1;
      head = lane < nw ? wh[lane] : P;
      for (int off = 16; off > 0; off >>= 1) {
        const T of = __shfl_xor_sync(0xffffffffu, bf, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        head = min(head, __shfl_xor_sync(0xffffffffu, head, off));
        merge(bf, bi, of, oi);
      }
      if (lane == 0) {
        const int worst = (isnan(sf[head]) || bi < 0) ? head : bi;
        alive[worst] = 0;
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) rank[i] = alive[i] ? 0 : target;
}

// block i: survivor i moves to position #{j < i : survivor} of the staging rows
template <typename T>
__global__ void de_reduce_gather_kernel(const T* pop, int64_t ldp, const T* fit, int P, int D, const int* rank,
                                        int target, T* stage, int64_t lds, T* stage_fit) {
  const int i = blockIdx.x;
  if (rank[i] >= target) return;
  __shared__ int part[32];
  int c = 0;
  for (int j = threadIdx.x; j < i; j += blockDim.x) c += rank[j] < target ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  int pos = 0;
  for (int w = 0; w < int(blockDim.x + 31) / 32; ++w) pos += part[w];
  for (int j = threadIdx.x; j < D; j += blockDim.x) stage[size_t(pos) * lds + j] = pop[size_t(i) * ldp + j];
  if (threadIdx.x == 0) stage_fit[pos] = fit[i];
}

template <typename T>
__global__ void de_reduce_scatter_kernel(T* pop, int64_t ldp, T* fit, int D, const T* stage, int64_t lds,
                                         const T* stage_fit) {
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < D; j += blockDim.x) pop[size_t(i) * ldp + j] = stage[size_t(i) * lds + j];
  if (threadIdx.x == 0) fit[i] = stage_fit[i];
}

// de_archive::set_capacity (de/strategy.hpp:40-47): while size > cap, victim = uniform_int(size),
// swap with the last member, drop it.  Words: Philox sub-stream 0xFFFFFFFE of this generation, or
// the WORDS cursor.
template <typename T>
__global__ void de_archive_shrink_kernel(T* archive, int64_t ldt, int D, int* arch_size, int cap, word_source src,
                                         uint64_t ctr_hi, int64_t* cursor, int* overflow, int64_t* used) {
  __shared__ int victim, size;
  __shared__ int64_t pos0;
  if (threadIdx.x == 0) {
    size = *arch_size;
    pos0 = src.mode == RNG_WORDS ? *cursor : 0;
  }
  __syncthreads();
  int64_t n = 0;
  while (size > cap) {
    if (threadIdx.x == 0) {
      word_reader r{&src, ctr_hi, pos0 + n, 0, overflow};
      victim = draw_int(r, size);
    }
    ++n;
    __syncthreads();
    const int last = size - 1;
    if (victim != last)
      for (int j = threadIdx.x; j < D; j += blockDim.x) archive[size_t(victim) * ldt + j] = archive[size_t(last) * ldt + j];
    __syncthreads();
    if (threadIdx.x == 0) size = last;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *arch_size = size;
    *used = n;
    if (src.mode == RNG_WORDS) {
      *cursor = pos0 + n;
      if (pos0 + n > src.n_words) *overflow = 1;
    }
  }
}

int ttpb_p_count(double p_t, int P) { return std::min(P, std::max(2, int(std::ceil(p_t * P)))); }

// after the generation's selection: evolution_state::add_fes(P) has happened; shrink if scheduled
template <typename T>
void reduce_t(evb_de_s* e, void* pop, int64_t ldp, void* fit, evb_rng_s* r, cudaStream_t st) {
  e->last_shrink_valid = 0;
  if (!e->reduction) return;
  const double frac = double(e->fes) / double(e->max_fes);
  const int target = std::clamp(int(std::lround(e->P_alloc + (e->n_min - e->P_alloc) * frac)), e->n_min, e->P_alloc);
  if (target >= e->P) return;  // policy.hpp:49: no-op when the schedule allows the current size
  const int P = e->P, D = e->D;
  const size_t mark_smem = (sizeof(T) + 1) * size_t(P);
  require(mark_smem <= 200 * 1024, "L-SHADE reduction: population too large for the one-block removal scan");
  if (mark_smem > 48 * 1024)
    EVB_CUDA(cudaFuncSetAttribute(de_reduce_mark_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(mark_smem)));
  de_reduce_mark_kernel<T><<<1, 1024, mark_smem, st>>>(static_cast<const T*>(fit), P, target, e->rank);
  de_reduce_gather_kernel<T><<<P, 128, 0, st>>>(static_cast<const T*>(pop), ldp, static_cast<const T*>(fit), P, D,
                                                 e->rank, target, static_cast<T*>(e->trial), e->ldt,
                                                 static_cast<T*>(e->trial_fit));
  de_reduce_scatter_kernel<T><<<target, 128, 0, st>>>(static_cast<T*>(pop), ldp, static_cast<T*>(fit), D,
                                                      static_cast<const T*>(e->trial), e->ldt,
                                                      static_cast<const T*>(e->trial_fit));
  count_launch(3);
  // archive.set_capacity(archive_capacity_for(new size), rng)  (de/engine.hpp:97-100)
  const int cap = int(std::ceil(e->rate_t * double(target)));
  word_source src{r->mode, r->key, r->d_words, r->n_words};
  de_archive_shrink_kernel<T><<<1, 128, 0, st>>>(static_cast<T*>(e->archive), e->ldt, D, e->d_arch_size, cap, src,
                                                 (uint64_t(r->gen) << 32) | kSubShrink, r->d_cursor, r->d_overflow,
                                                 e->d_shrink_words);
  count_launch();
  EVB_CUDA(cudaGetLastError());
  e->P = target;
  e->archive_cap = cap;
  if (e->cfg.mutation == EVB_MUT_TTPB1) e->p_count = ttpb_p_count(e->p_t, target);
  e->last_shrink_valid = 1;
}

template <typename T>
void init_population_t(int P, int D, void* pop, int64_t ldp, double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  word_source src{r->mode, r->key, r->d_words, r->n_words};
  int64_t base = 0;
  if (r->mode == RNG_WORDS) {
    EVB_CUDA(cudaMemcpyAsync(&base, r->d_cursor, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    EVB_CUDA(cudaStreamSynchronize(st));
  }
  const uint64_t ctr_hi = (uint64_t(r->gen) << 32) | kSubInit;
  init_population_kernel<T><<<std::min<int64_t>(4096, (int64_t(P) * D + 255) / 256), 256, 0, st>>>(
      static_cast<T*>(pop), ldp, P, D, lb, ub, src, ctr_hi, base, r->d_overflow);
  count_launch();
  EVB_CUDA(cudaGetLastError());
  if (r->mode == RNG_WORDS) {
    const int64_t nb = base + int64_t(P) * D;
    EVB_CUDA(cudaMemcpyAsync(r->d_cursor, &nb, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EVB_CUDA(cudaStreamSynchronize(st));
  } else {
    r->gen++;
    set_device_gen(r, st);
  }
}

}  // namespace

// n generations in one persistent cluster launch when the configuration allows it (PHILOX words,
// binomial crossover, clip / reflect / midpoint repair, fixed population, a base problem the
// small-D kernel evaluates, no per-generation observers, P <= 16 x 32); false: not eligible.
template <typename T>
bool run_generations_t(evb_de_s* e, const device_problem* prob, void* pop, int64_t ldp, void* fit, double lb,
                       double ub, evb_rng_s* r, int n, cudaStream_t st) {
  static const char* env = std::getenv("EVB_DE_PERSIST");
  if (env && std::atoi(env) == 0) return false;
  if (r->mode != RNG_PHILOX || e->cfg.crossover != EVB_CX_BINOMIAL || e->cfg.repair == EVB_REP_REINITIALIZE) return false;
  if (e->reduction || e->rec || e->ptrace || e->mon_on) return false;
  if (prob->spec != SPEC_BASE || !prob->rot_t || !eval_small_path(*prob)) return false;
  const int P = e->P, D = e->D;
  static int max_nc = [] {
    int v = 8;
    if (cudaFuncSetAttribute(de_run_kernel<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) v = 16;
    cudaGetLastError();
    return v;
  }();
  static const char* nc_env = std::getenv("EVB_DE_PERSIST_NC");  // tuning override
  const int NC = nc_env ? std::min(max_nc, std::max((P + 31) / 32, std::atoi(nc_env)))
                        : std::min(max_nc, std::max(1, (P + 7) / 8));
  const int Q = (P + NC - 1) / NC;
  if (Q > 32) return false;
  const int H = std::max(1, e->cfg.memory_size);
  const size_t mt_bytes = (size_t(D) * D * sizeof(T) + 15) / 16 * 16;
  auto smem_for = [&](int q, int nc) {
    size_t np2 = 1;
    while (np2 < size_t(P)) np2 <<= 1;
    (void)nc;
    return mt_bytes + (3 * size_t(q) * D + 4 * size_t(P) + 2 * H + 3 * q + 1) * sizeof(T) + 16 + 4 * size_t(P) * 8 +
           (np2 + P + size_t(std::max(0, e->archive_cap)) + 64 + 10 * q) * sizeof(int) + 8 + 2 * 8 + 64;
  };
  if (smem_for(Q, NC) > 200 * 1024) return false;
  de_run_args<T> a{};
  a.d = make_dev<T>(e, pop, ldp, fit, lb, ub, r);
  a.shift = static_cast<const T*>(prob->shift);
  a.rot_t = static_cast<const T*>(prob->rot_t);
  a.ell_w = static_cast<const T*>(prob->ell_w);
  a.kind = prob->kind;
  a.bias = prob->bias;
  a.G = n;
  a.Q = Q;
  a.srec = e->d_srec;
  static bool attr = [] {
    EVB_CUDA(cudaFuncSetAttribute(de_run_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return true;
  }();
  (void)attr;
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.blockDim = dim3(kRunThreads);
  lc.stream = st;
  lc.attrs = at;
  lc.numAttrs = 1;
  int nc = NC;
  if (e->run_nc < 0) {  // once per engine: the largest cluster that fits one GPC with its shared memory
    e->run_nc = 0;
    for (;;) {
      at[0].val.clusterDim.x = unsigned(nc);
      lc.gridDim = dim3(nc);
      lc.dynamicSmemBytes = smem_for((P + nc - 1) / nc, nc);
      if (lc.dynamicSmemBytes > 200 * 1024) break;
      int active = 0;
      if (cudaOccupancyMaxActiveClusters(&active, de_run_kernel<T>, &lc) == cudaSuccess && active >= 1) {
        e->run_nc = nc;
        e->run_smem = lc.dynamicSmemBytes;
        break;
      }
      cudaGetLastError();
      if (nc == 1) break;
      nc = std::max(1, nc / 2);
      if ((P + nc - 1) / nc > 32) break;
    }
  }
  if (e->run_nc <= 0) return false;
  nc = e->run_nc;
  at[0].val.clusterDim.x = unsigned(nc);
  lc.gridDim = dim3(nc);
  lc.dynamicSmemBytes = e->run_smem;
  a.Q = (P + nc - 1) / nc;
  static const bool prof = std::getenv("EVB_DE_PERSIST_PROFILE") != nullptr;
  if (prof) {
    EVB_CUDA(cudaMalloc(&a.prof, 16 * sizeof(unsigned long long)));
    EVB_CUDA(cudaMemset(a.prof, 0, 16 * sizeof(unsigned long long)));
  }
  EVB_CUDA(cudaLaunchKernelEx(&lc, de_run_kernel<T>, a));
  count_launch();
  if (prof) {
    unsigned long long h[16];
    EVB_CUDA(cudaMemcpy(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(a.prof);
    const char* names[] = {"ranks", "draws", "trial", "eval-base", "select+B1", "slots+B2", "apply+adapt", "B3",
                           "x-o", "dots", "pre", "loads"};
    std::string line = "[evb de_run] NC=" + std::to_string(nc) + " cycles/generation:";
    for (int k = 0; k < 12; ++k) line += std::string(" ") + names[k] + "=" + std::to_string(h[k] / std::max(1, n));
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  e->gen_P = P;
  e->last_gen = r->gen + uint32_t(n - 1);
  r->gen += uint32_t(n);
  e->fes += int64_t(n) * P;
  e->gen_count += n;
  return true;
}

bool run_generations(evb_de_s* e, const device_problem* prob, void* pop, int64_t ldp, void* fit, double lb, double ub,
                     evb_rng_s* r, int n, cudaStream_t st) {
  return e->dtype == EVB_F64 ? run_generations_t<double>(e, prob, pop, ldp, fit, lb, ub, r, n, st)
                             : run_generations_t<float>(e, prob, pop, ldp, fit, lb, ub, r, n, st);
}

void de_generation(evb_de_s* e, const device_problem* prob, evb_scratch_s* sc, void* pop, int64_t ldp, void* fit,
                   double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  if (e->dtype == EVB_F64) generation_t<double>(e, prob, sc, pop, ldp, fit, lb, ub, r, st);
  else generation_t<float>(e, prob, sc, pop, ldp, fit, lb, ub, r, st);
}

// init_population (core/population.hpp:88-98): P x D uniforms in [lb, ub], individual-major
void population_init(int dtype, int P, int D, void* pop, int64_t ldp, double lb, double ub, evb_rng_s* r,
                     cudaStream_t st) {
  if (dtype == EVB_F64) init_population_t<double>(P, D, pop, ldp, lb, ub, r, st);
  else init_population_t<float>(P, D, pop, ldp, lb, ub, r, st);
}

void de_init_population(evb_de_s* e, void* pop, int64_t ldp, double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  population_init(e->dtype, e->P, e->D, pop, ldp, lb, ub, r, st);
}

}  // namespace evb

// =============================================================================================
// C ABI: random words + DE engine
// =============================================================================================
namespace evb {
namespace {

template <typename T>
void* dalloc(size_t n) {
  void* p = nullptr;
  EVB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  EVB_CUDA(memset_now(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
  return p;
}

void free_de(evb_de_s* e) {
  if (e->graph) cudaGraphExecDestroy(e->graph);
  if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  if (e->hs_dev) cudaFree(e->hs_dev);
  if (e->hs_pinned) cudaFreeHost(e->hs_pinned);
  if (e->hs_stream) cudaStreamDestroy(e->hs_stream);
  void* ptrs[] = {e->trial, e->trial_fit, e->F, e->CR, e->slot, e->idx, e->jrand, e->xlen, e->rword, e->woff, e->wcount, e->order,
                  e->win, e->arch_slot, e->owner, e->succ, e->wlist, e->d_npush, e->d_epoch, e->d_owner64, e->d_sel_agg,
                  e->d_sel_sync, e->d_srec, e->archive, e->d_arch_size, e->d_write_index,
                  e->d_arch_words, e->mem_f, e->mem_cr, e->rank, e->d_shrink_words, e->d_mon};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (e->eval_scratch) evb_scratch_destroy(e->eval_scratch);
}

const char* mutation_name(int m) {
  return m == EVB_MUT_RAND1 ? "rand_1" : m == EVB_MUT_BEST1 ? "best_1" : m == EVB_MUT_TTPB1 ? "ttpb_1" : "?";
}

// back to the initial population size (a new optimize() run starts from pop_size members)
void restore_size(evb_de_s* e) {
  e->P = e->P_alloc;
  e->archive_cap = int(std::ceil(e->rate_t * double(e->P_alloc)));
  if (e->cfg.mutation == EVB_MUT_TTPB1) e->p_count = ttpb_p_count(e->p_t, e->P_alloc);
}

template <typename T>
void reset_adapter(evb_de_s* e) {
  const int H = std::max(1, e->cfg.memory_size);
  std::vector<T> half(H, T(0.5));
  EVB_CUDA(copy_h2d_now(e->mem_f, half.data(), sizeof(T) * H));
  EVB_CUDA(copy_h2d_now(e->mem_cr, half.data(), sizeof(T) * H));
  EVB_CUDA(memset_now(e->d_write_index, 0, sizeof(int)));
}

}  // namespace
}  // namespace evb

using namespace evb;

extern "C" {

int evb_rng_create_philox(uint64_t key, evb_rng* out) {
  return guarded([&] {
    require(out != nullptr, "rng: null output handle");
    auto* r = new evb_rng_s();
    r->mode = RNG_PHILOX;
    r->key = key;
    EVB_CUDA(cudaMalloc(&r->d_gen, sizeof(uint32_t)));
    EVB_CUDA(memset_now(r->d_gen, 0, sizeof(uint32_t)));
    EVB_CUDA(cudaMalloc(&r->d_overflow, sizeof(int)));
    EVB_CUDA(memset_now(r->d_overflow, 0, sizeof(int)));
    EVB_CUDA(cudaMalloc(&r->d_cursor, sizeof(int64_t)));
    EVB_CUDA(memset_now(r->d_cursor, 0, sizeof(int64_t)));
    *out = r;
  });
}

int evb_rng_create_words(const uint64_t* words, int64_t n_words, evb_rng* out) {
  return guarded([&] {
    require(out != nullptr && (words != nullptr || n_words == 0), "rng: null words or output handle");
    require(n_words >= 0, "rng: negative word count");
    auto* r = new evb_rng_s();
    r->mode = RNG_WORDS;
    r->n_words = n_words;
    EVB_CUDA(cudaMalloc(&r->d_gen, sizeof(uint32_t)));
    EVB_CUDA(memset_now(r->d_gen, 0, sizeof(uint32_t)));
    EVB_CUDA(cudaMalloc(&r->d_words, std::max<int64_t>(n_words, 1) * sizeof(uint64_t)));
    if (n_words) EVB_CUDA(copy_h2d_now(r->d_words, words, n_words * sizeof(uint64_t)));
    EVB_CUDA(cudaMalloc(&r->d_overflow, sizeof(int)));
    EVB_CUDA(memset_now(r->d_overflow, 0, sizeof(int)));
    EVB_CUDA(cudaMalloc(&r->d_cursor, sizeof(int64_t)));
    EVB_CUDA(memset_now(r->d_cursor, 0, sizeof(int64_t)));
    *out = r;
  });
}

int evb_rng_destroy(evb_rng r) {
  return guarded([&] {
    if (!r) return;
    if (r->d_words) cudaFree(r->d_words);
    if (r->d_cursor) cudaFree(r->d_cursor);
    if (r->d_overflow) cudaFree(r->d_overflow);
    if (r->d_gen) cudaFree(r->d_gen);
    delete r;
  });
}

int evb_rng_state(evb_rng r, int64_t* cursor, uint32_t* generation, int* overflow) {
  return guarded([&] {
    require(r != nullptr, "rng: null handle");
    EVB_CUDA(cudaDeviceSynchronize());
    int64_t c = 0;
    int o = 0;
    EVB_CUDA(cudaMemcpy(&c, r->d_cursor, sizeof(c), cudaMemcpyDeviceToHost));
    EVB_CUDA(cudaMemcpy(&o, r->d_overflow, sizeof(o), cudaMemcpyDeviceToHost));
    if (cursor) *cursor = c;
    if (generation) *generation = r->gen;
    if (overflow) *overflow = o;
  });
}

int evb_rng_set_generation(evb_rng r, uint32_t generation) {
  return guarded([&] {
    require(r != nullptr, "rng: null handle");
    r->gen = generation;
    EVB_CUDA(cudaDeviceSynchronize());
    EVB_CUDA(copy_h2d_now(r->d_gen, &generation, sizeof(uint32_t)));
  });
}

int evb_de_create(int dtype, const evb_de_config* c, int pop_size, int dim, evb_de* out) {
  return guarded([&] {
    require(dtype == EVB_F32 || dtype == EVB_F64, "de: dtype must be EVB_F32 or EVB_F64");
    require(c != nullptr && out != nullptr, "de: null config or output handle");
    require(c->mutation == EVB_MUT_RAND1 || c->mutation == EVB_MUT_BEST1 || c->mutation == EVB_MUT_TTPB1,
            "de builder: unknown mutation strategy (GPU kernels: rand_1, best_1, ttpb_1)");
    require(c->crossover == EVB_CX_BINOMIAL || c->crossover == EVB_CX_EXPONENTIAL,
            "de builder: unknown crossover strategy (GPU kernels: binomial, exponential)");
    require(c->repair == EVB_REP_CLIP || c->repair == EVB_REP_REFLECT || c->repair == EVB_REP_MIDPOINT_TARGET ||
                c->repair == EVB_REP_REINITIALIZE,
            "de builder: unknown repair strategy (GPU kernels: clip, reflect, midpoint_target, reinitialize)");
    require(c->parameter == EVB_PAR_FIXED || c->parameter == EVB_PAR_JADE || c->parameter == EVB_PAR_SHADE,
            "de builder: unknown parameter adapter (GPU kernels: fixed, jade, shade)");
    if (c->parameter == EVB_PAR_FIXED) {  // de/parameter.hpp:81-84
      require(c->f > 0.0 && c->f <= 1.0, "fixed_parameter: F must be in (0,1]");
      require(c->cr >= 0.0 && c->cr <= 1.0, "fixed_parameter: CR must be in [0,1]");
    }
    if (c->parameter == EVB_PAR_SHADE) require(c->memory_size >= 1, "shade_parameter: memory size must be >= 1");
    if (c->parameter == EVB_PAR_JADE)
      require(c->jade_c > 0.0 && c->jade_c <= 1.0, "jade_parameter: learning rate must be in (0,1]");
    if (c->mutation == EVB_MUT_TTPB1)
      require(c->p_best > 0.0 && c->p_best <= 1.0, "ttpb1_mutation: p-best fraction must be in (0,1]");
    require(c->archive_rate >= 0.0, "de builder: archive rate must be >= 0");
    const int min_pop = c->mutation == EVB_MUT_RAND1 ? 4 : 3;  // de/strategy.hpp:78, 102, 134
    require(pop_size >= min_pop,
            std::string("de_engine: population too small for mutation ") + mutation_name(c->mutation));
    require(dim >= 1, "de: dim must be positive");
    require(c->reduction == EVB_POP_FIXED || c->reduction == EVB_POP_LINEAR_REDUCTION,
            "de builder: unknown population policy");
    if (c->reduction == EVB_POP_LINEAR_REDUCTION) {  // de/policy.hpp:24-28
      require(c->n_min >= 4, "population_policy: N_min must be at least 4");
      require(c->n_min <= pop_size, "population_policy: N_min must not exceed N_init");
    }

    auto* e = new evb_de_s();
    try {
      e->dtype = dtype;
      e->P = pop_size;
      e->D = dim;
      e->cfg.mutation = c->mutation;
      e->cfg.crossover = c->crossover;
      e->cfg.repair = c->repair;
      e->cfg.parameter = c->parameter;
      e->cfg.f = c->f;
      e->cfg.cr = c->cr;
      e->cfg.p_best = c->p_best;
      e->cfg.use_archive = c->use_archive;
      e->cfg.memory_size = c->parameter == EVB_PAR_SHADE ? c->memory_size : 1;
      e->cfg.jade_c = c->jade_c;
      e->cfg.archive_rate = c->archive_rate;
      const size_t es = dtype == EVB_F64 ? 8 : 4;
      // p_count = min(P, max(2, ceil(p * P))) with p stored in T (de/strategy.hpp:143)
      const double p_t = dtype == EVB_F64 ? c->p_best : double(float(c->p_best));
      e->p_count = c->mutation == EVB_MUT_TTPB1 ? std::min(pop_size, std::max(2, int(std::ceil(p_t * pop_size))))
                                                : (c->mutation == EVB_MUT_BEST1 ? 1 : 0);
      // archive_capacity_for (de/engine.hpp:137-139), archive_rate stored in T
      const double rate_t = dtype == EVB_F64 ? c->archive_rate : double(float(c->archive_rate));
      e->archive_cap = int(std::ceil(rate_t * double(pop_size)));
      e->P_alloc = pop_size;
      e->p_t = p_t;
      e->rate_t = rate_t;
      e->reduction = c->reduction;
      e->n_min = c->reduction == EVB_POP_LINEAR_REDUCTION ? c->n_min : std::min(4, pop_size);
      e->ldt = round_up(dim, 16 / int64_t(es));
      auto bytes = [&](size_t n) { return n * es; };
      EVB_CUDA(cudaMalloc(&e->trial, bytes(size_t(pop_size) * e->ldt)));
      EVB_CUDA(memset_now(e->trial, 0, bytes(size_t(pop_size) * e->ldt)));
      EVB_CUDA(cudaMalloc(&e->trial_fit, bytes(pop_size)));
      EVB_CUDA(cudaMalloc(&e->F, bytes(pop_size)));
      EVB_CUDA(cudaMalloc(&e->CR, bytes(pop_size)));
      e->slot = static_cast<int*>(dalloc<int>(pop_size));
      e->idx = static_cast<int*>(dalloc<int>(size_t(pop_size) * 4));
      e->jrand = static_cast<int*>(dalloc<int>(pop_size));
      e->xlen = static_cast<int*>(dalloc<int>(pop_size));
      e->rword = static_cast<int64_t*>(dalloc<int64_t>(pop_size));
      e->woff = static_cast<int64_t*>(dalloc<int64_t>(pop_size));
      e->wcount = static_cast<int64_t*>(dalloc<int64_t>(pop_size));
      e->order = static_cast<int*>(dalloc<int>(std::max(1, e->p_count)));
      e->win = static_cast<int*>(dalloc<int>(pop_size));
      e->arch_slot = static_cast<int*>(dalloc<int>(pop_size));
      e->owner = static_cast<int*>(dalloc<int>(std::max(1, e->archive_cap)));
      e->succ = static_cast<int*>(dalloc<int>(pop_size));
      e->wlist = static_cast<int*>(dalloc<int>(pop_size));
      e->d_npush = static_cast<int*>(dalloc<int>(3));
      e->d_epoch = static_cast<unsigned*>(dalloc<unsigned>(1));
      e->d_owner64 = static_cast<unsigned long long*>(dalloc<unsigned long long>(std::max(1, e->archive_cap)));
      e->d_sel_agg = static_cast<unsigned long long*>(dalloc<unsigned long long>((pop_size + 1023) / 1024));
      e->d_sel_sync = static_cast<unsigned*>(dalloc<unsigned>(2));
      e->d_srec = static_cast<double*>(dalloc<double>(3 * size_t(pop_size)));
      EVB_CUDA(cudaMalloc(&e->archive, bytes(size_t(std::max(1, e->archive_cap)) * e->ldt)));
      EVB_CUDA(memset_now(e->archive, 0, bytes(size_t(std::max(1, e->archive_cap)) * e->ldt)));
      e->d_arch_size = static_cast<int*>(dalloc<int>(1));
      e->d_write_index = static_cast<int*>(dalloc<int>(1));
      e->d_arch_words = static_cast<int64_t*>(dalloc<int64_t>(1));
      e->rank = static_cast<int*>(dalloc<int>(pop_size));
      e->d_shrink_words = static_cast<int64_t*>(dalloc<int64_t>(1));
      EVB_CUDA(cudaMalloc(&e->mem_f, bytes(e->cfg.memory_size)));
      EVB_CUDA(cudaMalloc(&e->mem_cr, bytes(e->cfg.memory_size)));
      if (dtype == EVB_F64) reset_adapter<double>(e);
      else reset_adapter<float>(e);
      EVB_CUDA(evb_scratch_create(&e->eval_scratch) == EVB_OK ? cudaSuccess : cudaErrorUnknown);
    } catch (...) {
      free_de(e);
      delete e;
      throw;
    }
    *out = e;
  });
}

int evb_de_destroy(evb_de e) {
  return guarded([&] {
    if (!e) return;
    free_de(e);
    e->phases.destroy();
    delete e;
  });
}

int evb_de_phase_timing(evb_de e, int enable) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    e->phases.on = enable != 0;
    e->phases.n = 0;
  });
}

int evb_de_phase_ms(evb_de e, float* ms, int cap, int* n) {
  return guarded([&] {
    require(e != nullptr && ms != nullptr && n != nullptr, "de_phase_ms: null argument");
    *n = e->phases.read(ms, cap);
  });
}

int evb_de_reset(evb_de e) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    if (e->dtype == EVB_F64) reset_adapter<double>(e);
    else reset_adapter<float>(e);
    EVB_CUDA(memset_now(e->d_arch_size, 0, sizeof(int)));
    restore_size(e);
  });
}

int evb_de_set_budget(evb_de e, int64_t max_fes, int64_t fes) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    require(max_fes > 0, "evolution_state: max_fes must be positive");
    require(fes >= 0, "evolution_state: add_fes requires n >= 0");
    e->max_fes = max_fes;
    e->fes = fes;
  });
}

int evb_de_pop_size(evb_de e) { return e ? e->P : -1; }

int evb_de_last_reduction(evb_de e, int* pop_before, int* pop_after, int64_t* shrink_words) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    if (pop_before) *pop_before = e->gen_P;
    if (pop_after) *pop_after = e->P;
    int64_t n = 0;
    if (e->last_shrink_valid) {
      EVB_CUDA(cudaDeviceSynchronize());
      EVB_CUDA(cudaMemcpy(&n, e->d_shrink_words, sizeof(n), cudaMemcpyDeviceToHost));
    }
    if (shrink_words) *shrink_words = n;
  });
}

int evb_de_archive_capacity(evb_de e) { return e ? e->archive_cap : -1; }
int evb_de_p_count(evb_de e) { return e ? e->p_count : -1; }

int evb_de_generation(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp, void* fitness,
                      double lb, double ub, evb_rng rng, void* stream) {
  return guarded([&] {
    require(e && objective && rng && pop && fitness, "de_generation: null argument");
    if (objective->p.dim != e->D) throw invalid_argument("de_generation: problem dimension mismatch");
    if (objective->p.dtype != e->dtype) throw config_error("de_generation: problem dtype differs from engine");
    if (ldp < e->D) throw invalid_argument("de_generation: ldp < dim");
    if (e->reduction && e->max_fes <= 0)
      throw config_error("de_generation: linear population reduction needs a budget (evb_de_set_budget)");
    de_generation(e, &objective->p, s ? s : e->eval_scratch, pop, ldp, fitness, lb, ub, rng,
                  static_cast<cudaStream_t>(stream));
  });
}

// n generations; after the first (which also sizes every buffer) one generation is captured into
// a CUDA graph and replayed — the generation id and the WORDS cursor live on the device, so the
// replays are exact continuations (identical to n calls of evb_de_generation).
int evb_de_generations(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp, void* fitness,
                       double lb, double ub, evb_rng rng, int n, void* stream) {
  return guarded([&] {
    require(e && objective && rng && pop && fitness, "de_generations: null argument");
    require(n >= 0, "de_generations: negative count");
    if (objective->p.dim != e->D) throw invalid_argument("de_generations: problem dimension mismatch");
    if (objective->p.dtype != e->dtype) throw config_error("de_generations: problem dtype differs from engine");
    if (ldp < e->D) throw invalid_argument("de_generations: ldp < dim");
    if (n == 0) return;
    if (e->reduction && e->max_fes <= 0)
      throw config_error("de_generations: linear population reduction needs a budget (evb_de_set_budget)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_scratch_s* sc = s ? s : e->eval_scratch;
    // one persistent cluster launch for all n generations where the configuration allows
    if (run_generations(e, &objective->p, pop, ldp, fitness, lb, ub, rng, n, st)) return;
    if (e->reduction || e->ptrace) {  // size changes / per-generation trace arguments: no graph replay
      for (int g = 0; g < n; ++g) de_generation(e, &objective->p, sc, pop, ldp, fitness, lb, ub, rng, st);
      return;
    }
    de_generation(e, &objective->p, sc, pop, ldp, fitness, lb, ub, rng, st);
    if (--n == 0) return;
    const void* key[6] = {pop, fitness, objective, sc, rng, reinterpret_cast<const void*>(ldp)};
    bool same = e->graph != nullptr && e->g_bounds[0] == lb && e->g_bounds[1] == ub;
    for (int k = 0; k < 6 && same; ++k) same = e->g_key[k] == key[k];
    if (!same) {
      if (e->graph) {
        EVB_CUDA(cudaGraphExecDestroy(e->graph));
        e->graph = nullptr;
      }
      if (!e->cap_stream) EVB_CUDA(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
      EVB_CUDA(cudaStreamSynchronize(st));
      const uint32_t host_gen = rng->gen, host_last = e->last_gen;
      const int64_t host_fes = e->fes;
      const int host_count = e->gen_count;
      const int k0 = last_launch_count();
      cudaGraph_t g = nullptr;
      EVB_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
      try {
        de_generation(e, &objective->p, sc, pop, ldp, fitness, lb, ub, rng, e->cap_stream);
      } catch (...) {
        cudaStreamEndCapture(e->cap_stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      EVB_CUDA(cudaStreamEndCapture(e->cap_stream, &g));
      e->g_kernels = last_launch_count() - k0;
      count_launch(-e->g_kernels);  // captured, not launched
      rng->gen = host_gen;
      e->last_gen = host_last;
      e->fes = host_fes;
      e->gen_count = host_count;
      const cudaError_t ie = cudaGraphInstantiate(&e->graph, g, 0);
      cudaGraphDestroy(g);
      EVB_CUDA(ie);
      for (int k = 0; k < 6; ++k) e->g_key[k] = key[k];
      e->g_bounds[0] = lb;
      e->g_bounds[1] = ub;
    }
    for (int i = 0; i < n; ++i) {
      EVB_CUDA(cudaGraphLaunch(e->graph, st));
      e->last_gen = rng->gen;
      rng->gen++;
      e->fes += e->P;
      ++e->gen_count;
      count_launch(e->g_kernels);
    }
  });
}

// n generations on a host-resident population (the reference's engine keeps its population on
// the host): the rows go into the engine's page-locked staging, cross the host link as one copy
// with the fitness, run as evb_de_generations (one persistent launch where eligible), and come
// back the same way; synchronous, like de_engine::generation.
int evb_de_generations_host(evb_de e, evb_problem objective, evb_scratch s, void* pop_host, int64_t ldp,
                            void* fitness_host, double lb, double ub, evb_rng rng, int n) {
  const int rc0 = guarded([&] {
    require(e && objective && rng && pop_host && fitness_host, "de_generations_host: null argument");
    require(n >= 0, "de_generations_host: negative count");
    if (ldp < e->D) throw invalid_argument("de_generations_host: ldp < dim");
    require(e->reduction == 0, "de_generations_host: linear population reduction changes the population size");
    const size_t es = e->dtype == EVB_F64 ? 8 : 4;
    const size_t row = es * size_t(e->D), bytes = es * (size_t(e->P) * e->D + e->P);
    if (!e->hs_dev) {
      EVB_CUDA(cudaMalloc(&e->hs_dev, bytes));
      EVB_CUDA(cudaHostAlloc(&e->hs_pinned, bytes, cudaHostAllocPortable));
      EVB_CUDA(cudaStreamCreateWithFlags(&e->hs_stream, cudaStreamNonBlocking));
    }
    uint8_t* hp = static_cast<uint8_t*>(e->hs_pinned);
    const uint8_t* src = static_cast<const uint8_t*>(pop_host);
    if (size_t(ldp) * es == row) std::memcpy(hp, src, row * e->P);
    else
      for (int i = 0; i < e->P; ++i) std::memcpy(hp + row * i, src + size_t(ldp) * es * i, row);
    std::memcpy(hp + row * e->P, fitness_host, es * e->P);
    EVB_CUDA(cudaMemcpyAsync(e->hs_dev, hp, bytes, cudaMemcpyHostToDevice, e->hs_stream));
  });
  if (rc0 != EVB_OK) return rc0;
  const size_t es = e->dtype == EVB_F64 ? 8 : 4;
  uint8_t* dv = static_cast<uint8_t*>(e->hs_dev);
  const int rc = evb_de_generations(e, objective, s, dv, e->D, dv + es * size_t(e->P) * e->D, lb, ub, rng, n,
                                    e->hs_stream);
  if (rc != EVB_OK) return rc;
  return guarded([&] {
    const size_t row = es * size_t(e->D), bytes = es * (size_t(e->P) * e->D + e->P);
    EVB_CUDA(cudaMemcpyAsync(e->hs_pinned, e->hs_dev, bytes, cudaMemcpyDeviceToHost, e->hs_stream));
    EVB_CUDA(cudaStreamSynchronize(e->hs_stream));
    const uint8_t* hp = static_cast<const uint8_t*>(e->hs_pinned);
    uint8_t* dst = static_cast<uint8_t*>(pop_host);
    if (size_t(ldp) * es == row) std::memcpy(dst, hp, row * e->P);
    else
      for (int i = 0; i < e->P; ++i) std::memcpy(dst + size_t(ldp) * es * i, hp + row * i, row);
    std::memcpy(fitness_host, hp + row * e->P, es * e->P);
  });
}

int evb_de_init_population(evb_de e, void* pop, int64_t ldp, double lb, double ub, evb_rng rng, void* stream) {
  return guarded([&] {
    require(e && rng && pop, "de_init_population: null argument");
    require(lb < ub, "init_population: lb must be less than ub");
    if (ldp < e->D) throw invalid_argument("de_init_population: ldp < dim");
    de_init_population(e, pop, ldp, lb, ub, rng, static_cast<cudaStream_t>(stream));
  });
}

int evb_de_get_state(evb_de e, void* archive_host, int* archive_size, void* mem_f_host, void* mem_cr_host,
                     int* write_index) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    EVB_CUDA(cudaDeviceSynchronize());
    const size_t es = e->dtype == EVB_F64 ? 8 : 4;
    int sz = 0;
    EVB_CUDA(cudaMemcpy(&sz, e->d_arch_size, sizeof(int), cudaMemcpyDeviceToHost));
    if (archive_size) *archive_size = sz;
    if (archive_host && e->archive_cap > 0)
      EVB_CUDA(cudaMemcpy2D(archive_host, e->D * es, e->archive, e->ldt * es, e->D * es, e->archive_cap,
                            cudaMemcpyDeviceToHost));
    if (mem_f_host) EVB_CUDA(cudaMemcpy(mem_f_host, e->mem_f, es * e->cfg.memory_size, cudaMemcpyDeviceToHost));
    if (mem_cr_host) EVB_CUDA(cudaMemcpy(mem_cr_host, e->mem_cr, es * e->cfg.memory_size, cudaMemcpyDeviceToHost));
    if (write_index) EVB_CUDA(cudaMemcpy(write_index, e->d_write_index, sizeof(int), cudaMemcpyDeviceToHost));
  });
}

int evb_de_set_state(evb_de e, const void* archive_host, int archive_size, const void* mem_f_host,
                     const void* mem_cr_host, int write_index) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    require(archive_size >= 0 && archive_size <= e->archive_cap, "de_set_state: archive size exceeds capacity");
    const size_t es = e->dtype == EVB_F64 ? 8 : 4;
    EVB_CUDA(cudaDeviceSynchronize());
    if (archive_host && archive_size > 0)
      EVB_CUDA(cudaMemcpy2D(e->archive, e->ldt * es, archive_host, e->D * es, e->D * es, archive_size,
                            cudaMemcpyHostToDevice));
    EVB_CUDA(copy_h2d_now(e->d_arch_size, &archive_size, sizeof(int)));
    if (mem_f_host) EVB_CUDA(copy_h2d_now(e->mem_f, mem_f_host, es * e->cfg.memory_size));
    if (mem_cr_host) EVB_CUDA(copy_h2d_now(e->mem_cr, mem_cr_host, es * e->cfg.memory_size));
    require(write_index >= 0 && write_index < e->cfg.memory_size, "de_set_state: write index out of range");
    EVB_CUDA(copy_h2d_now(e->d_write_index, &write_index, sizeof(int)));
  });
}

int evb_de_attach_recorder(evb_de e, evb_recorder r, int run) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    if (r) {
      require(recorder_dtype(r) == e->dtype, "de_attach_recorder: dtype mismatch");
      require(run >= 0 && run < recorder_runs(r), "de_attach_recorder: run out of range");
    }
    e->rec = r;
    e->rec_run = run;
    if (e->graph) {  // the captured generation does not contain the recorder call
      EVB_CUDA(cudaGraphExecDestroy(e->graph));
      e->graph = nullptr;
    }
  });
}

int evb_de_attach_param_trace(evb_de e, evb_param_trace t, int run) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    if (t) {
      require(t->dtype == e->dtype, "de_attach_param_trace: dtype mismatch");
      require(run >= 0 && run < t->n_runs, "de_attach_param_trace: run out of range");
    }
    e->ptrace = t;
    e->ptrace_run = run;
    if (e->graph) {  // the captured generation does not contain the trace call
      EVB_CUDA(cudaGraphExecDestroy(e->graph));
      e->graph = nullptr;
    }
  });
}

int evb_de_last_draws(evb_de e, int64_t* word_counts, int64_t* archive_words, uint32_t* generation, void* F_host,
                      void* CR_host, int* idx_host, int* jrand_host) {
  return guarded([&] {
    require(e != nullptr, "de: null handle");
    EVB_CUDA(cudaDeviceSynchronize());
    const size_t es = e->dtype == EVB_F64 ? 8 : 4;
    if (word_counts) EVB_CUDA(cudaMemcpy(word_counts, e->wcount, sizeof(int64_t) * e->gen_P, cudaMemcpyDeviceToHost));
    if (archive_words) EVB_CUDA(cudaMemcpy(archive_words, e->d_arch_words, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (generation) *generation = e->last_gen;
    if (F_host) EVB_CUDA(cudaMemcpy(F_host, e->F, es * e->gen_P, cudaMemcpyDeviceToHost));
    if (CR_host) EVB_CUDA(cudaMemcpy(CR_host, e->CR, es * e->gen_P, cudaMemcpyDeviceToHost));
    if (idx_host) EVB_CUDA(cudaMemcpy(idx_host, e->idx, sizeof(int) * 4 * e->gen_P, cudaMemcpyDeviceToHost));
    if (jrand_host) EVB_CUDA(cudaMemcpy(jrand_host, e->jrand, sizeof(int) * e->gen_P, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

namespace evb {
namespace {

// de_engine::optimize (de/engine.hpp:107-133): init, evaluate, generations while the budget is
// left and stop() is false (checked before every generation); returns the generations run and
// the population's best (lowest fitness, ties to the lowest index).
template <typename Stop>
int optimize_impl(evb_de_s* e, evb_problem objective, evb_scratch_s* sc, void* pop, int64_t ldp, void* fitness,
                  double lb, double ub, int64_t max_fes, evb_rng_s* rng, cudaStream_t st, Stop&& stop, int* best_index,
                  double* best_fitness) {
  restore_size(e);
  de_init_population(e, pop, ldp, lb, ub, rng, st);
  eval_request rq{};
  rq.prob = &objective->p;
  rq.scratch = sc;
  rq.X = pop;
  rq.n = e->P;
  rq.ldx = ldp;
  rq.out = fitness;
  rq.ldo = e->P;
  rq.n_out = 1;
  rq.kinds[0] = objective->p.kind;
  rq.biases[0] = objective->p.bias;
  rq.stream = st;
  rq.scalar_trig = true;
  eval_dispatch(rq);
  if (e->rec) recorder_observe(e->rec, e->rec_run, fitness, e->P, st);  // initial evaluations
  if (e->mon_on) {
    if (e->dtype == EVB_F64)
      restart_monitor_kernel<double><<<1, 32, 0, st>>>(static_cast<const double*>(fitness), e->P, e->d_mon, e->mon_eps);
    else
      restart_monitor_kernel<float><<<1, 32, 0, st>>>(static_cast<const float*>(fitness), e->P, e->d_mon, e->mon_eps);
    count_launch();
  }
  e->max_fes = max_fes;  // evolution_state st(max_fes, ...); st.add_fes(P) for the initial members
  e->fes = e->P;
  e->gen_count = 0;
  int gens = 0;
  while (e->fes < max_fes && !stop()) {
    de_generation(e, &objective->p, sc, pop, ldp, fitness, lb, ub, rng, st);
    ++gens;
  }
  const size_t es = e->dtype == EVB_F64 ? 8 : 4;
  std::vector<uint8_t> f(es * e->P);
  EVB_CUDA(cudaMemcpyAsync(f.data(), fitness, es * e->P, cudaMemcpyDeviceToHost, st));
  EVB_CUDA(cudaStreamSynchronize(st));
  int best = 0;
  auto val = [&](int i) {
    return e->dtype == EVB_F64 ? reinterpret_cast<double*>(f.data())[i] : double(reinterpret_cast<float*>(f.data())[i]);
  };
  for (int i = 1; i < e->P; ++i)
    if (val(i) < val(best)) best = i;
  if (best_index) *best_index = best;
  if (best_fitness) *best_fitness = val(best);
  return gens;
}

}  // namespace
}  // namespace evb

extern "C" {

int evb_de_optimize(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp, void* fitness, double lb,
                    double ub, int64_t max_fes, evb_rng rng, int* best_index, double* best_fitness, int* generations,
                    void* stream) {
  return guarded([&] {
    require(e && objective && rng && pop && fitness, "de_optimize: null argument");
    require(max_fes > 0, "evolution_state: max_fes must be positive");
    require(e->P >= 4, "init_population: pop_size must be at least 4");
    if (objective->p.dim != e->D) throw invalid_argument("de_optimize: problem dimension mismatch");
    e->gen_offset = 0;
    const int g = optimize_impl(e, objective, s ? s : e->eval_scratch, pop, ldp, fitness, lb, ub, max_fes, rng,
                                static_cast<cudaStream_t>(stream), [] { return false; }, best_index, best_fitness);
    if (generations) *generations = g;
  });
}

// hybrid::restart_run (hybrid/restart.hpp:37-88) around this engine's optimize: fresh engine state
// (adapter, archive, population size) per run, stop once since_improvement >= stagnation_evals,
// until the total budget is spent; the best over all runs.
int evb_de_optimize_restart(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp, void* fitness,
                            double lb, double ub, int64_t total_budget, int64_t stagnation_evals, double epsilon,
                            evb_rng rng, double* best_fitness, int* engine_runs, int64_t* evaluations, void* stream) {
  return guarded([&] {
    require(e && objective && rng && pop && fitness, "de_optimize_restart: null argument");
    require(stagnation_evals >= 1, "restart: stagnation_evals must be at least 1");
    require(epsilon >= 0.0, "restart: epsilon must be non-negative");
    require(total_budget >= e->P_alloc, "restart: budget below one initialization");
    if (objective->p.dim != e->D) throw invalid_argument("de_optimize_restart: problem dimension mismatch");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_scratch_s* sc = s ? s : e->eval_scratch;
    if (!e->d_mon) EVB_CUDA(cudaMalloc(&e->d_mon, 3 * sizeof(double)));
    const double init[3] = {std::numeric_limits<double>::infinity(), 0.0, 0.0};
    EVB_CUDA(cudaMemcpyAsync(e->d_mon, init, sizeof(init), cudaMemcpyHostToDevice, st));
    e->mon_on = 1;
    e->mon_eps = epsilon;
    e->gen_offset = 0;
    double best = std::numeric_limits<double>::infinity();
    int runs = 0;
    double h[3] = {0, 0, 0};
    auto read_mon = [&] {
      EVB_CUDA(cudaMemcpyAsync(h, e->d_mon, sizeof(h), cudaMemcpyDeviceToHost, st));
      EVB_CUDA(cudaStreamSynchronize(st));
    };
    try {
      for (;;) {
        read_mon();
        if (int64_t(h[2]) >= total_budget) break;
        const double zero = 0.0;  // since_improvement = 0 for the new engine
        EVB_CUDA(cudaMemcpyAsync(e->d_mon + 1, &zero, sizeof(double), cudaMemcpyHostToDevice, st));
        if (e->dtype == EVB_F64) reset_adapter<double>(e);  // make_engine(): a fresh engine
        else reset_adapter<float>(e);
        EVB_CUDA(cudaMemsetAsync(e->d_arch_size, 0, sizeof(int), st));
        const int64_t remaining = total_budget - int64_t(h[2]);
        double cand = 0.0;
        optimize_impl(e, objective, sc, pop, ldp, fitness, lb, ub, remaining, rng, st,
                      [&] {
                        read_mon();
                        return int64_t(h[1]) >= stagnation_evals;
                      },
                      nullptr, &cand);
        e->gen_offset += e->gen_count;  // generation_offset = last reported generation
        ++runs;
        if (cand < best) best = cand;
        read_mon();
        if (int64_t(h[1]) < stagnation_evals) break;  // the budget ran out rather than stagnation
      }
    } catch (...) {
      e->mon_on = 0;
      throw;
    }
    e->mon_on = 0;
    if (best_fitness) *best_fitness = best;
    if (engine_runs) *engine_runs = runs;
    if (evaluations) *evaluations = int64_t(h[2]);
  });
}

}  // extern "C"

namespace evb {
__global__ void philox_words_kernel(uint64_t key, uint64_t ctr_hi, uint64_t start, int64_t n, uint64_t* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = philox_word(key, ctr_hi, start + uint64_t(i));
}
}  // namespace evb

extern "C" int evb_philox_words(uint64_t key, uint64_t ctr_hi, uint64_t start, int64_t n, uint64_t* out_host) {
  return guarded([&] {
    require(n >= 0 && (out_host || n == 0), "philox_words: bad output");
    if (n == 0) return;
    uint64_t* d = nullptr;
    EVB_CUDA(cudaMalloc(&d, n * sizeof(uint64_t)));
    evb::philox_words_kernel<<<(n + 255) / 256, 256>>>(key, ctr_hi, start, n, d);
    evb::count_launch();
    cudaError_t e = cudaMemcpy(out_host, d, n * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    EVB_CUDA(e);
  });
}
