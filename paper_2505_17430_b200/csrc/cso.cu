// cso.cu — Competitive Swarm Optimizer generation on the device (pso/cso.hpp:19-99,
// cso_optimizer<T>).  One CSO generation is data-parallel by construction: the swarm mean is
// taken from the pre-update positions, particles meet in disjoint pairs, and a pair's loser
// reads only its winner (never updated this generation) and the mean — so the GPU generation is
// the reference's generation exactly (no synchronous/asynchronous deviation).
//
//   mean      m_j = (sum_i x_ij, i ascending, in T) / T(P)                   (cso.hpp:37-42)
//   pairs     Fisher-Yates over iota: k = P-1 .. 1 swaps perm[k], perm[uniform_int(k+1)]  (:44-47)
//   pair t    a = perm[2t], b = perm[2t+1]; winner = f_a <= f_b ? a : b     (:49-53)
//             per gene j, r1 r2 r3 = T(uniform01):
//             v = r1 v + r2 (x_w - x) + phi r3 (m - x);  x = clamp(x + v, lb, ub)  (:55-66)
//             evaluate the loser (pair order = FE order)                      (:67-68)
//
// Draws.  Philox: the permutation uses sub-stream (g << 32) | 0xFFFFFFFD (word n = P-1-k for
// swap k); pair t uses sub-stream (g << 32) | t, words 3j, 3j+1, 3j+2.  WORDS: the reference's
// sequential order — P-1 permutation words, then pair t's 3D words — so every position is known
// up front (no data-dependent counts).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "evb_internal.cuh"
#include "evb_math.cuh"
#include "rng.cuh"

struct evb_cso_s {
  int dtype = EVB_F64;
  int P = 0, D = 0;
  double phi = 0.1;
  int64_t lds = 0;
  void* mean = nullptr;       // D (T)
  int* perm = nullptr;        // P
  int* loser = nullptr;       // P / 2
  void* stage = nullptr;      // P/2 x lds: updated losers, evaluated as one batch
  void* stage_fit = nullptr;  // P/2
  evb_scratch_s* eval_scratch = nullptr;
  evb_recorder_s* rec = nullptr;
  int rec_run = 0;
  uint32_t last_gen = 0;
};

namespace evb {
namespace {

constexpr uint32_t kSubPerm = 0xFFFFFFFDu;

template <typename T>
__global__ void cso_mean_kernel(const T* __restrict__ x, int64_t ldx, int P, int D, T* mean) {
  using F = fop<T>;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= D) return;
  T m = T(0);
  for (int i = 0; i < P; ++i) m = F::add(m, x[size_t(i) * ldx + j]);
  mean[j] = F::div(m, T(P));
}

// Fisher-Yates (cso.hpp:44-47): the P-1 draws are independent of the permutation state, so they
// are made in parallel; one thread then applies the swaps in shared memory.
__global__ void cso_perm_kernel(int P, word_source src, uint64_t ctr_hi, const int64_t* cursor, int* overflow,
                                int* perm) {
  extern __shared__ int sm[];
  int* cur = sm;
  int* pick = sm + P;
  const int64_t base = src.mode == RNG_WORDS ? *cursor : 0;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    cur[k] = k;
    if (k >= 1) pick[k] = uint_of(word_at(src, ctr_hi, base + (P - 1 - k), overflow), k + 1);
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = P - 1; k >= 1; --k) {
      const int r = pick[k];
      const int a = cur[k], b = cur[r];
      cur[k] = b;
      cur[r] = a;
    }
  __syncthreads();
  for (int k = threadIdx.x; k < P; k += blockDim.x) perm[k] = cur[k];
}

template <typename T>
struct cso_dev {
  int P, D;
  T* x;
  int64_t ldx;
  T* v;
  int64_t ldv;
  const T* fit;
  const T* mean;
  const int* perm;
  int* loser;
  T* stage;
  int64_t lds;
  T phi, lb, ub;
  word_source src;
  const uint32_t* gen_ptr;
  const int64_t* cursor;
  int* overflow;
};

template <typename T>
__global__ void cso_update_kernel(const cso_dev<T> d) {
  using F = fop<T>;
  const int t = blockIdx.x;
  const int a = d.perm[2 * t], b = d.perm[2 * t + 1];
  const int w = d.fit[a] <= d.fit[b] ? a : b;  // cso.hpp:51
  const int l = w == a ? b : a;
  if (threadIdx.x == 0) d.loser[t] = l;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(t);
  const int64_t base = d.src.mode == RNG_WORDS ? *d.cursor + (d.P - 1) + int64_t(t) * 3 * d.D : 0;
  T* xl = d.x + size_t(l) * d.ldx;
  T* vl = d.v + size_t(l) * d.ldv;
  const T* xw = d.x + size_t(w) * d.ldx;
  T* out = d.stage + size_t(t) * d.lds;
  for (int j = threadIdx.x; j < d.D; j += blockDim.x) {
    const int64_t n = base + 3 * int64_t(j);
    const T r1 = T(u01_of(word_at(d.src, ctr_hi, n, d.overflow)));
    const T r2 = T(u01_of(word_at(d.src, ctr_hi, n + 1, d.overflow)));
    const T r3 = T(u01_of(word_at(d.src, ctr_hi, n + 2, d.overflow)));
    const T x = xl[j];
    const T v = F::add(F::add(F::mul(r1, vl[j]), F::mul(r2, F::sub(xw[j], x))),
                       F::mul(F::mul(d.phi, r3), F::sub(d.mean[j], x)));
    T xn = F::add(x, v);
    xn = xn < d.lb ? d.lb : (d.ub < xn ? d.ub : xn);  // std::clamp
    vl[j] = v;
    xl[j] = xn;
    out[j] = xn;
  }
}

// losers' fitness back into the swarm; advances the generation id and the WORDS cursor
template <typename T>
__global__ void cso_scatter_kernel(const int* loser, const T* sf, int half, T* fit, uint32_t* gen, int64_t* cursor,
                                   int64_t words, int words_mode) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < half) fit[loser[t]] = sf[t];
  if (t == 0) {
    *gen += 1u;
    if (words_mode) *cursor += words;
  }
}

template <typename T>
void cso_generation_t(evb_cso_s* c, const device_problem* prob, evb_scratch_s* sc, void* X, int64_t ldx, void* V,
                      int64_t ldv, void* fit, double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  const int P = c->P, D = c->D, half = P / 2;
  cso_mean_kernel<T><<<(D + 127) / 128, 128, 0, st>>>(static_cast<const T*>(X), ldx, P, D, static_cast<T*>(c->mean));
  word_source src{r->mode, r->key, r->d_words, r->n_words};
  cso_perm_kernel<<<1, 256, sizeof(int) * 2 * P, st>>>(P, src, (uint64_t(r->gen) << 32) | kSubPerm, r->d_cursor,
                                                       r->d_overflow, c->perm);
  cso_dev<T> d{};
  d.P = P;
  d.D = D;
  d.x = static_cast<T*>(X);
  d.ldx = ldx;
  d.v = static_cast<T*>(V);
  d.ldv = ldv;
  d.fit = static_cast<const T*>(fit);
  d.mean = static_cast<const T*>(c->mean);
  d.perm = c->perm;
  d.loser = c->loser;
  d.stage = static_cast<T*>(c->stage);
  d.lds = c->lds;
  d.phi = T(c->phi);
  d.lb = T(lb);
  d.ub = T(ub);
  d.src = src;
  d.gen_ptr = r->d_gen;
  d.cursor = r->d_cursor;
  d.overflow = r->d_overflow;
  cso_update_kernel<T><<<half, std::min(256, int(round_up(D, 32))), 0, st>>>(d);
  count_launch(3);
  EVB_CUDA(cudaGetLastError());
  eval_request rq{};
  rq.prob = prob;
  rq.scratch = sc;
  rq.X = c->stage;
  rq.n = half;
  rq.ldx = c->lds;
  rq.out = c->stage_fit;
  rq.ldo = half;
  rq.n_out = 1;
  rq.kinds[0] = prob->kind;
  rq.biases[0] = prob->bias;
  rq.stream = st;
  rq.scalar_trig = true;  // individual::evaluate -> problem_instance::evaluate
  eval_dispatch(rq);
  if (c->rec) recorder_observe(c->rec, c->rec_run, c->stage_fit, half, st);  // losers in pair (FE) order
  cso_scatter_kernel<T><<<(half + 127) / 128, 128, 0, st>>>(c->loser, static_cast<const T*>(c->stage_fit), half,
                                                            static_cast<T*>(fit), r->d_gen, r->d_cursor,
                                                            int64_t(P - 1) + int64_t(half) * 3 * D,
                                                            r->mode == RNG_WORDS ? 1 : 0);
  count_launch();
  EVB_CUDA(cudaGetLastError());
  c->last_gen = r->gen;
  r->gen++;
}

void cso_generation(evb_cso_s* c, const device_problem* prob, evb_scratch_s* sc, void* X, int64_t ldx, void* V,
                    int64_t ldv, void* fit, double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  if (c->dtype == EVB_F64) cso_generation_t<double>(c, prob, sc, X, ldx, V, ldv, fit, lb, ub, r, st);
  else cso_generation_t<float>(c, prob, sc, X, ldx, V, ldv, fit, lb, ub, r, st);
}

void check_args(evb_cso_s* c, evb_problem p, const void* X, int64_t ldx, const void* V, int64_t ldv,
                const void* fit, evb_rng r) {
  require(c && p && X && V && fit && r, "cso: null argument");
  if (p->p.dim != c->D) throw invalid_argument("cso: problem dimension mismatch");
  if (p->p.dtype != c->dtype) throw config_error("cso: problem dtype differs from the optimizer");
  if (ldx < c->D || ldv < c->D) throw invalid_argument("cso: leading dimension < dim");
}

}  // namespace
}  // namespace evb

using namespace evb;

extern "C" {

int evb_cso_create(int dtype, double phi, int pop_size, int dim, evb_cso* out) {
  return guarded([&] {
    require(dtype == EVB_F32 || dtype == EVB_F64, "cso: dtype must be EVB_F32 or EVB_F64");
    require(out != nullptr, "cso: null output handle");
    const double phi_t = dtype == EVB_F64 ? phi : double(float(phi));
    require(std::isfinite(phi_t), "cso: phi must be finite");  // cso.hpp:25-27
    require(phi_t >= 0.0, "cso: phi must be >= 0");
    require(pop_size >= 2 && pop_size % 2 == 0, "cso: population size must be even");
    require(dim >= 1, "cso: dim must be positive");
    auto* c = new evb_cso_s();
    try {
      c->dtype = dtype;
      c->P = pop_size;
      c->D = dim;
      c->phi = phi;
      const size_t es = dtype == EVB_F64 ? 8 : 4;
      c->lds = round_up(dim, 16 / int64_t(es));
      EVB_CUDA(cudaMalloc(&c->mean, es * dim));
      EVB_CUDA(cudaMalloc(&c->perm, sizeof(int) * pop_size));
      EVB_CUDA(cudaMalloc(&c->loser, sizeof(int) * (pop_size / 2)));
      EVB_CUDA(cudaMalloc(&c->stage, es * c->lds * (pop_size / 2)));
      EVB_CUDA(memset_now(c->stage, 0, es * c->lds * (pop_size / 2)));
      EVB_CUDA(cudaMalloc(&c->stage_fit, es * (pop_size / 2)));
      require(evb_scratch_create(&c->eval_scratch) == EVB_OK, "cso: scratch allocation failed");
    } catch (...) {
      void* ptrs[] = {c->mean, c->perm, c->loser, c->stage, c->stage_fit};
      for (void* p : ptrs)
        if (p) cudaFree(p);
      delete c;
      throw;
    }
    *out = c;
  });
}

int evb_cso_destroy(evb_cso c) {
  return guarded([&] {
    if (!c) return;
    void* ptrs[] = {c->mean, c->perm, c->loser, c->stage, c->stage_fit};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (c->eval_scratch) evb_scratch_destroy(c->eval_scratch);
    delete c;
  });
}

int evb_cso_attach_recorder(evb_cso c, evb_recorder rec, int run) {
  return guarded([&] {
    require(c != nullptr, "cso: null handle");
    if (rec) {
      require(recorder_dtype(rec) == c->dtype, "cso_attach_recorder: dtype mismatch");
      require(run >= 0 && run < recorder_runs(rec), "cso_attach_recorder: run out of range");
    }
    c->rec = rec;
    c->rec_run = run;
  });
}

int evb_cso_generation(evb_cso c, evb_problem objective, evb_scratch s, void* X, int64_t ldx, void* V, int64_t ldv,
                       void* fitness, double lb, double ub, evb_rng rng, void* stream) {
  return guarded([&] {
    check_args(c, objective, X, ldx, V, ldv, fitness, rng);
    cso_generation(c, &objective->p, s ? s : c->eval_scratch, X, ldx, V, ldv, fitness, lb, ub, rng,
                   static_cast<cudaStream_t>(stream));
  });
}

int evb_cso_optimize(evb_cso c, evb_problem objective, evb_scratch s, void* X, int64_t ldx, void* V, int64_t ldv,
                     void* fitness, double lb, double ub, int64_t max_fes, evb_rng rng, int* best_index,
                     double* best_fitness, int* generations, void* stream) {
  return guarded([&] {
    // cso.hpp:74-91
    check_args(c, objective, X, ldx, V, ldv, fitness, rng);
    require(max_fes > 0, "evolution_state: max_fes must be positive");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_scratch_s* sc = s ? s : c->eval_scratch;
    const size_t es = c->dtype == EVB_F64 ? 8 : 4;
    population_init(c->dtype, c->P, c->D, X, ldx, lb, ub, rng, st);
    eval_request rq{};
    rq.prob = &objective->p;
    rq.scratch = sc;
    rq.X = X;
    rq.n = c->P;
    rq.ldx = ldx;
    rq.out = fitness;
    rq.ldo = c->P;
    rq.n_out = 1;
    rq.kinds[0] = objective->p.kind;
    rq.biases[0] = objective->p.bias;
    rq.stream = st;
    rq.scalar_trig = true;
    eval_dispatch(rq);
    if (c->rec) recorder_observe(c->rec, c->rec_run, fitness, c->P, st);
    EVB_CUDA(cudaMemset2DAsync(V, ldv * es, 0, c->D * es, c->P, st));  // zero velocities
    int64_t fes = c->P;
    int gens = 0;
    while (fes < max_fes) {
      cso_generation(c, &objective->p, sc, X, ldx, V, ldv, fitness, lb, ub, rng, st);
      fes += c->P / 2;
      ++gens;
    }
    std::vector<uint8_t> f(es * c->P);
    EVB_CUDA(cudaMemcpyAsync(f.data(), fitness, es * c->P, cudaMemcpyDeviceToHost, st));
    EVB_CUDA(cudaStreamSynchronize(st));
    auto val = [&](int i) {
      return c->dtype == EVB_F64 ? reinterpret_cast<double*>(f.data())[i] : double(reinterpret_cast<float*>(f.data())[i]);
    };
    int best = 0;  // population::best (core/population.hpp:59-65)
    for (int i = 1; i < c->P; ++i)
      if (val(i) < val(best)) best = i;
    if (best_index) *best_index = best;
    if (best_fitness) *best_fitness = val(best);
    if (generations) *generations = gens;
  });
}

}  // extern "C"
