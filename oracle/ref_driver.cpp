// ref_driver.cpp — extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include, header-only C++20), compiled by oracle/Makefile into
// oracle/_ref/ (git-ignored build output that travels to the GPU box).
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY: used by tests/ (to pin the C restatement and
// generate golden fixtures) and by bench.py's reference arm.  Nothing here is product code.
//
// Two builds of this file exist:
//   libevbref_exact.so   reference Release flags (no -march => no FMA contraction): parity
//   libevbref_fast.so    -O3 -march=<host ISA> -pthread, the paper's flags: timing
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <thread>
#include <vector>

#include "evobench/core/population.hpp"
#include "evobench/core/rng.hpp"
#include "evobench/de/builder.hpp"
#include "evobench/de/engine.hpp"
#include "evobench/experiment/runner.hpp"
#include "evobench/presets.hpp"
#include "evobench/problems/batch.hpp"
#include "evobench/problems/suite.hpp"
#include "evobench/pso/engine.hpp"

using namespace evobench;
using namespace evobench::problems;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

template <typename T>
problem_instance<T> make_base(int kind, int dim, const T* shift, const T* rot, double bias) {
  std::vector<T> o(shift, shift + dim);
  std::vector<T> m(rot, rot + size_t(dim) * dim);
  return problem_instance<T>(1, 1, dim, T(-100), T(100), std::move(o), std::move(m), T(bias),
                             base_kind(kind), "ref");
}

template <typename T>
std::vector<std::vector<T>> rows(const T* x, int64_t n, int64_t ldx, int dim) {
  std::vector<std::vector<T>> xs(static_cast<size_t>(n), std::vector<T>(static_cast<size_t>(dim)));
  for (int64_t b = 0; b < n; ++b) std::memcpy(xs[size_t(b)].data(), x + b * ldx, sizeof(T) * dim);
  return xs;
}

template <typename T>
void eval_batch(const problem_instance<T>& p, const T* x, int64_t n, int64_t ldx, T* out) {
  auto xs = rows<T>(x, n, ldx, p.dim());
  eval_scratch<T> scratch;
  std::vector<T> res;
  evaluate_batch(p, xs, scratch, res);
  std::memcpy(out, res.data(), sizeof(T) * size_t(n));
}

// The batch split into `threads` contiguous slices, one eval_scratch per slice
// (the reference does not thread inside a batch).
template <typename T>
void eval_batch_threads(const problem_instance<T>& p, const std::vector<std::vector<T>>& xs, T* out, int threads) {
  const int64_t n = int64_t(xs.size());
  threads = std::max(1, std::min<int>(threads, int(n)));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const int64_t b0 = n * t / threads, b1 = n * (t + 1) / threads;
      std::vector<std::vector<T>> slice(xs.begin() + b0, xs.begin() + b1);
      eval_scratch<T> scratch;
      std::vector<T> res;
      evaluate_batch(p, slice, scratch, res);
      std::memcpy(out + b0, res.data(), sizeof(T) * size_t(b1 - b0));
    });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

// ---- rng ------------------------------------------------------------------------------------
REF_API void ref_rng_words(uint64_t seed, uint64_t stream, int64_t skip, int64_t n, uint64_t* out) {
  rng_stream r = derive_stream(seed, stream);
  for (int64_t i = 0; i < skip; ++i) r.next_u64();
  for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

// o then M from derive_stream(seed, stream) through the reference's own draw functions
// (problems/instance.hpp:285-296), in double.
REF_API void ref_make_shift_rotation(uint64_t seed, uint64_t stream, int dim, double* shift, double* rot) {
  rng_stream r = derive_stream(seed, stream);
  auto o = problems::detail::draw_shift<double>(dim, -100.0, 100.0, r);
  std::vector<double> scratch;
  auto m = problems::detail::draw_rotation<double>(dim, r, scratch);
  std::memcpy(shift, o.data(), sizeof(double) * dim);
  std::memcpy(rot, m.data(), sizeof(double) * size_t(dim) * dim);
}

REF_API void ref_init_population(uint64_t seed, uint64_t stream, int pop, int dim, double lb, double ub, double* x) {
  rng_stream r = derive_stream(seed, stream);
  auto pop_ = init_population<double>(pop, dim, lb, ub, r);
  for (int i = 0; i < pop; ++i) std::memcpy(x + size_t(i) * dim, pop_[i].genome.data(), sizeof(double) * dim);
}

// registry instance (problems/suite.hpp:73-146) — base / hybrid problems only
REF_API int ref_make_instance_f64(int problem_id, int dim, int instance, uint64_t seed, double* shift, double* rot,
                                  double* bias, int* kind_or_minus1) {
  auto p = make_instance<double>(problem_id, dim, instance, seed);
  *bias = p.bias();
  if (p.is_composition()) return 0;
  std::memcpy(shift, p.shift().data(), sizeof(double) * dim);
  std::memcpy(rot, p.rotation().data(), sizeof(double) * size_t(dim) * dim);
  *kind_or_minus1 = p.is_base() ? int(std::get<base_kind>(p.spec())) : -1;
  return 1;
}

// ---- evaluation -------------------------------------------------------------------------------
REF_API void ref_eval_batch_f64(int kind, int dim, const double* shift, const double* rot, double bias, int64_t n,
                                const double* x, int64_t ldx, double* out) {
  eval_batch<double>(make_base<double>(kind, dim, shift, rot, bias), x, n, ldx, out);
}
REF_API void ref_eval_batch_f32(int kind, int dim, const float* shift, const float* rot, double bias, int64_t n,
                                const float* x, int64_t ldx, float* out) {
  eval_batch<float>(make_base<float>(kind, dim, shift, rot, bias), x, n, ldx, out);
}
REF_API double ref_eval_scalar_f64(int kind, int dim, const double* shift, const double* rot, double bias,
                                   const double* x) {
  auto p = make_base<double>(kind, dim, shift, rot, bias);
  return p.evaluate(std::span<const double>(x, size_t(dim)));
}

REF_API void ref_eval_hybrid_f64(int dim, const double* shift, const double* rot, double bias, int n_chunks,
                                 const int* kinds, const int* sizes, const int* perm, int64_t n, const double* x,
                                 int64_t ldx, double* out) {
  hybrid_spec spec;
  spec.permutation.assign(perm, perm + dim);
  for (int c = 0; c < n_chunks; ++c) {
    spec.sub_kinds.push_back(base_kind(kinds[c]));
    spec.chunk_sizes.push_back(sizes[c]);
    spec.proportions.push_back(double(sizes[c]) / dim);
  }
  problem_instance<double> p(9, 1, dim, -100.0, 100.0, std::vector<double>(shift, shift + dim),
                             std::vector<double>(rot, rot + size_t(dim) * dim), bias, spec, "hyb");
  eval_batch<double>(p, x, n, ldx, out);
}

template <typename T>
static problem_instance<T> make_comp(int dim, int n_comp, const int* kinds, const T* shifts, const T* rots,
                                     const double* sigma, const double* lambda, const double* cbias, double bias) {
  composition_spec<T> spec;
  for (int c = 0; c < n_comp; ++c) {
    composition_component<T> comp;
    comp.kind = base_kind(kinds[c]);
    comp.shift.assign(shifts + size_t(c) * dim, shifts + size_t(c + 1) * dim);
    comp.rotation.assign(rots + size_t(c) * dim * dim, rots + size_t(c + 1) * dim * dim);
    comp.sigma = sigma[c];
    comp.lambda = lambda[c];
    comp.bias = cbias[c];
    spec.components.push_back(std::move(comp));
  }
  return problem_instance<T>(11, 1, dim, T(-100), T(100), {}, {}, T(bias), std::move(spec), "comp");
}

REF_API void ref_eval_composition_f64(int dim, int n_comp, const int* kinds, const double* shifts, const double* rots,
                                      const double* sigma, const double* lambda, const double* cbias, double bias,
                                      int64_t n, const double* x, int64_t ldx, double* out) {
  eval_batch<double>(make_comp<double>(dim, n_comp, kinds, shifts, rots, sigma, lambda, cbias, bias), x, n, ldx,
                     out);
}

// ---- CPU baseline timing helpers (reference arm) ------------------------------------------------
// Evaluate `reps` batches of n points through evaluate_batch on `threads` threads; returns
// nothing (the caller times the call).  Inputs are converted once outside.
struct ref_batch_job {
  int dtype;
  std::unique_ptr<problem_instance<double>> p64;
  std::unique_ptr<problem_instance<float>> p32;
  std::vector<std::vector<double>> x64;
  std::vector<std::vector<float>> x32;
  std::vector<double> out64;
  std::vector<float> out32;
};

REF_API void* ref_batch_job_create(int dtype, int kind, int dim, const void* shift, const void* rot, double bias,
                                   int64_t n, const void* x) {
  auto* j = new ref_batch_job();
  j->dtype = dtype;
  if (dtype == 1) {
    j->p64 = std::make_unique<problem_instance<double>>(
        make_base<double>(kind, dim, static_cast<const double*>(shift), static_cast<const double*>(rot), bias));
    j->x64 = rows<double>(static_cast<const double*>(x), n, dim, dim);
    j->out64.resize(size_t(n));
  } else {
    j->p32 = std::make_unique<problem_instance<float>>(
        make_base<float>(kind, dim, static_cast<const float*>(shift), static_cast<const float*>(rot), bias));
    j->x32 = rows<float>(static_cast<const float*>(x), n, dim, dim);
    j->out32.resize(size_t(n));
  }
  return j;
}
REF_API void ref_batch_job_run(void* job, int threads, void* out) {
  auto* j = static_cast<ref_batch_job*>(job);
  if (j->dtype == 1) {
    eval_batch_threads<double>(*j->p64, j->x64, j->out64.data(), threads);
    if (out) std::memcpy(out, j->out64.data(), sizeof(double) * j->out64.size());
  } else {
    eval_batch_threads<float>(*j->p32, j->x32, j->out32.data(), threads);
    if (out) std::memcpy(out, j->out32.data(), sizeof(float) * j->out32.size());
  }
}
REF_API void ref_batch_job_destroy(void* job) { delete static_cast<ref_batch_job*>(job); }

REF_API int ref_hardware_threads(void) { return int(std::thread::hardware_concurrency()); }

// ---- DE engine (de/engine.hpp) driven generation by generation ----------------------------------
namespace {

struct ref_de_run {
  std::unique_ptr<de::de_engine<double>> engine;
  std::unique_ptr<problem_instance<double>> problem;
  population<double> pop;
  int P = 0, D = 0;
};

std::unique_ptr<de::mutation_strategy<double>> make_mutation(int m, double p, int use_archive) {
  if (m == 0) return std::make_unique<de::rand1_mutation<double>>();
  if (m == 1) return std::make_unique<de::best1_mutation<double>>();
  return std::make_unique<de::ttpb1_mutation<double>>(p, use_archive != 0);
}
std::unique_ptr<de::repair_strategy<double>> make_repair(int r) {
  if (r == 0) return std::make_unique<de::clip_repair<double>>();
  if (r == 1) return std::make_unique<de::reflect_repair<double>>();
  return std::make_unique<de::midpoint_target_repair<double>>();
}
std::unique_ptr<de::parameter_adapter<double>> make_adapter(int a, double f, double cr, int H, double c) {
  if (a == 0) return std::make_unique<de::fixed_parameter<double>>(f, cr);
  if (a == 1) return std::make_unique<de::jade_parameter<double>>(c);
  return std::make_unique<de::shade_parameter<double>>(H);
}

}  // namespace

// Engine built through the reference de_builder from the same strategy choices as evb_de_config.
REF_API void* ref_de_create(int mutation, int repair, int adapter, double f, double cr, double p, int use_archive,
                            int H, double jade_c, double archive_rate, int P, int D) {
  auto* r = new ref_de_run();
  r->engine = std::make_unique<de::de_engine<double>>(de::de_builder<double>()
                                                          .mutation(make_mutation(mutation, p, use_archive))
                                                          .crossover(std::make_unique<de::binomial_crossover<double>>())
                                                          .repair(make_repair(repair))
                                                          .parameter(make_adapter(adapter, f, cr, H, jade_c))
                                                          .population(de::population_policy::fixed())
                                                          .archive_rate(archive_rate)
                                                          .build());
  r->P = P;
  r->D = D;
  r->pop = population<double>(P, D);
  rng_stream dummy(0, 0);
  r->engine->archive().set_capacity(r->engine->archive_capacity_for(P), dummy);
  return r;
}
REF_API void ref_de_destroy(void* h) { delete static_cast<ref_de_run*>(h); }

REF_API void ref_de_set_problem_base(void* h, int kind, const double* shift, const double* rot, double bias) {
  auto* r = static_cast<ref_de_run*>(h);
  r->problem = std::make_unique<problem_instance<double>>(make_base<double>(kind, r->D, shift, rot, bias));
}
REF_API void ref_de_set_problem_composition(void* h, int n_comp, const int* kinds, const double* shifts,
                                            const double* rots, const double* sigma, const double* lambda,
                                            const double* cbias, double bias) {
  auto* r = static_cast<ref_de_run*>(h);
  r->problem = std::make_unique<problem_instance<double>>(
      make_comp<double>(r->D, n_comp, kinds, shifts, rots, sigma, lambda, cbias, bias));
}

REF_API void ref_de_set_pop(void* h, const double* x, const double* fit) {
  auto* r = static_cast<ref_de_run*>(h);
  for (int i = 0; i < r->P; ++i) {
    std::memcpy(r->pop[i].genome.data(), x + size_t(i) * r->D, sizeof(double) * r->D);
    r->pop[i].fitness = fit[i];
    r->pop[i].evaluated = true;
  }
}

// init_population + evaluation exactly as de_engine::optimize does (de/engine.hpp:118-122), from
// a scripted word list; returns the number of words consumed.
REF_API int64_t ref_de_init(void* h, const uint64_t* words, int64_t n, double lb, double ub) {
  auto* r = static_cast<ref_de_run*>(h);
  std::vector<uint64_t> w(words, words + n);
  w.push_back(0x5e5e5e5e5e5e5e5eULL);
  rng_stream rng = rng_stream::scripted(w);
  r->pop = init_population<double>(r->P, r->D, lb, ub, rng);
  eval_scratch<double> scratch;
  for (auto& m : r->pop) m.evaluate([&](std::span<const double> x) { return r->problem->evaluate(x, scratch); });
  int64_t used = 0;
  while (rng.next_u64() != 0x5e5e5e5e5e5e5e5eULL && used <= n) ++used;
  return n - used;  // words consumed
}

// One de_engine::generation with rng_stream::scripted(words + sentinel).  Returns 1 when the
// engine consumed exactly n words (the next word is the sentinel), 0 otherwise.
REF_API int ref_de_generation(void* h, const uint64_t* words, int64_t n, double lb, double ub) {
  auto* r = static_cast<ref_de_run*>(h);
  const uint64_t sentinel = 0xa5a5a5a5deadbeefULL;
  std::vector<uint64_t> w(words, words + n);
  w.push_back(sentinel);
  rng_stream rng = rng_stream::scripted(w);
  evolution_state st(1LL << 40, r->P, r->D, std::min(4, r->P));
  eval_scratch<double> scratch;
  auto objective = [&](std::span<const double> x) { return r->problem->evaluate(x, scratch); };
  r->engine->generation(r->pop, st, objective, lb, ub, rng);
  return rng.next_u64() == sentinel ? 1 : 0;
}

REF_API void ref_de_get(void* h, double* x, double* fit, double* archive, int* arch_size, double* mem_f,
                        double* mem_cr, int* write_index) {
  auto* r = static_cast<ref_de_run*>(h);
  for (int i = 0; i < r->P; ++i) {
    if (x) std::memcpy(x + size_t(i) * r->D, r->pop[i].genome.data(), sizeof(double) * r->D);
    if (fit) fit[i] = r->pop[i].fitness;
  }
  auto& ar = r->engine->archive();
  if (arch_size) *arch_size = ar.size();
  if (archive)
    for (int j = 0; j < ar.size(); ++j)
      std::memcpy(archive + size_t(j) * r->D, ar.member(j).data(), sizeof(double) * r->D);
  auto& ad = r->engine->parameter();
  if (auto* s = dynamic_cast<de::shade_parameter<double>*>(&ad)) {
    if (mem_f) std::memcpy(mem_f, s->memory_f().data(), sizeof(double) * s->memory_f().size());
    if (mem_cr) std::memcpy(mem_cr, s->memory_cr().data(), sizeof(double) * s->memory_cr().size());
    if (write_index) *write_index = s->write_index();
  } else if (auto* j = dynamic_cast<de::jade_parameter<double>*>(&ad)) {
    if (mem_f) mem_f[0] = j->mu_f();
    if (mem_cr) mem_cr[0] = j->mu_cr();
    if (write_index) *write_index = 0;
  }
}

// The reference's own run with its NATIVE stream: rng_stream(seed, stream) -> init_population,
// evaluate, set_capacity, `generations` generations (de/engine.hpp:107-133 without the budget
// loop).  Used for the config-0 exact replay.
REF_API void ref_de_native_run(void* h, uint64_t seed, uint64_t stream, int generations, double lb, double ub) {
  auto* r = static_cast<ref_de_run*>(h);
  rng_stream rng(seed, stream);
  r->pop = init_population<double>(r->P, r->D, lb, ub, rng);
  eval_scratch<double> scratch;
  auto objective = [&](std::span<const double> x) { return r->problem->evaluate(x, scratch); };
  for (auto& m : r->pop) m.evaluate(objective);
  r->engine->archive().set_capacity(r->engine->archive_capacity_for(r->P), rng);
  evolution_state st(1LL << 40, r->P, r->D, std::min(4, r->P));
  for (int g = 0; g < generations; ++g) r->engine->generation(r->pop, st, objective, lb, ub, rng);
}
