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
  int n_min = 4;
  std::unique_ptr<evolution_state> st;  // persistent budget (L-SHADE schedules read it)
};

std::unique_ptr<de::mutation_strategy<double>> make_mutation(int m, double p, int use_archive) {
  if (m == 0) return std::make_unique<de::rand1_mutation<double>>();
  if (m == 1) return std::make_unique<de::best1_mutation<double>>();
  return std::make_unique<de::ttpb1_mutation<double>>(p, use_archive != 0);
}
std::unique_ptr<de::repair_strategy<double>> make_repair(int r) {
  if (r == 0) return std::make_unique<de::clip_repair<double>>();
  if (r == 1) return std::make_unique<de::reflect_repair<double>>();
  if (r == 3) return std::make_unique<de::reinitialize_repair<double>>();
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
                            int H, double jade_c, double archive_rate, int P, int D, int crossover, int reduction,
                            int n_min) {
  auto* r = new ref_de_run();
  r->engine = std::make_unique<de::de_engine<double>>(de::de_builder<double>()
                                                          .mutation(make_mutation(mutation, p, use_archive))
                                                          .crossover(crossover == 1 ? std::unique_ptr<de::crossover_strategy<double>>(
                                                                                          std::make_unique<de::exponential_crossover<double>>())
                                                                                    : std::make_unique<de::binomial_crossover<double>>())
                                                          .repair(make_repair(repair))
                                                          .parameter(make_adapter(adapter, f, cr, H, jade_c))
                                                          .population(reduction ? de::population_policy::linear_reduction(P, n_min)
                                                                                : de::population_policy::fixed())
                                                          .archive_rate(archive_rate)
                                                          .build());
  r->n_min = reduction ? n_min : std::min(4, P);
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
  evolution_state tmp(1LL << 40, r->P, r->D, std::min(4, r->P));
  evolution_state& st = r->st ? *r->st : tmp;
  eval_scratch<double> scratch;
  auto objective = [&](std::span<const double> x) { return r->problem->evaluate(x, scratch); };
  r->engine->generation(r->pop, st, objective, lb, ub, rng);
  return rng.next_u64() == sentinel ? 1 : 0;
}

// evolution_state(max_fes, P, D, n_min) with `fes` evaluations done, kept across generations
REF_API void ref_de_set_budget(void* h, long long max_fes, long long fes) {
  auto* r = static_cast<ref_de_run*>(h);
  r->st = std::make_unique<evolution_state>(max_fes, r->P, r->D, r->n_min);
  r->st->add_fes(fes);
}

REF_API int ref_de_pop_size(void* h) { return static_cast<ref_de_run*>(h)->pop.pop_size(); }

REF_API void ref_de_get(void* h, double* x, double* fit, double* archive, int* arch_size, double* mem_f,
                        double* mem_cr, int* write_index) {
  auto* r = static_cast<ref_de_run*>(h);
  for (int i = 0; i < r->pop.pop_size(); ++i) {
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

// ---- synchronous PSO driver built from the reference's own pieces --------
// gbest_topology / lbest_topology::neighbor_best on the start-of-generation pbests,
// standard_update::apply (pso/update.hpp:66-74) followed by the config's velocity clamp, the move
// and bound rule of pso/engine.hpp:66-75, problem_instance::evaluate, strict-< pbest
// (pso/engine.hpp:78-79).  The stock pso_engine is asynchronous; this driver is the synchronous
// variant BASELINE config 3 specifies.
namespace {
template <typename T>
struct ref_pso_run {
  std::unique_ptr<pso::topology_strategy<T>> topo;
  std::unique_ptr<pso::velocity_update_strategy<T>> upd;
  pso::swarm_params<T> params;
  T vmax;
  std::unique_ptr<problem_instance<T>> problem;
  std::vector<std::vector<T>> x, v;
  std::vector<individual<T>> pb;
  std::vector<T> fit;
  int P, D;
  int threads = 1;

  int step(const uint64_t* words, int64_t n, T lb, T ub) {
    const uint64_t sentinel = 0x0badc0ffee0ddf00ULL;
    std::vector<uint64_t> w(words, words + n);
    w.push_back(sentinel);
    rng_stream rng = rng_stream::scripted(w);
    std::vector<int> nb(static_cast<size_t>(P));
    for (int i = 0; i < P; ++i) nb[size_t(i)] = topo->neighbor_best(pb, i);
    const auto snapshot = pb;  // start-of-generation personal bests (synchronous)
    for (int i = 0; i < P; ++i) {
      auto& xi = x[size_t(i)];
      auto& vi = v[size_t(i)];
      upd->apply(xi, vi, snapshot[size_t(i)].genome, snapshot[size_t(nb[size_t(i)])].genome, nb[size_t(i)] == i,
                params, rng);
      for (int j = 0; j < D; ++j) {
        if (vmax > T(0)) {
          if (vi[size_t(j)] > vmax) vi[size_t(j)] = vmax;
          if (vi[size_t(j)] < -vmax) vi[size_t(j)] = -vmax;
        }
        xi[size_t(j)] += vi[size_t(j)];  // pso/engine.hpp:66-75
        if (xi[size_t(j)] < lb) {
          xi[size_t(j)] = lb;
          vi[size_t(j)] = T(-0.5) * vi[size_t(j)];
        } else if (xi[size_t(j)] > ub) {
          xi[size_t(j)] = ub;
          vi[size_t(j)] = T(-0.5) * vi[size_t(j)];
        }
      }
    }
    const int nt = std::max(1, std::min(threads, P));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        eval_scratch<T> scratch;
        for (int i = P * t / nt; i < P * (t + 1) / nt; ++i) fit[size_t(i)] = problem->evaluate(x[size_t(i)], scratch);
      });
    for (auto& th : pool) th.join();
    for (int i = 0; i < P; ++i) {
      if (fit[size_t(i)] < pb[size_t(i)].fitness) {
        pb[size_t(i)].genome = x[size_t(i)];
        pb[size_t(i)].fitness = fit[size_t(i)];
      }
    }
    return rng.next_u64() == sentinel ? 1 : 0;
  }
};

template <typename T>
void* pso_create(int topology, double w, double c1, double c2, double vmax, int P, int D, int kind, const void* shift,
                 const void* rot, double bias, int update, double attraction) {
  auto* r = new ref_pso_run<T>();
  if (topology == 0) r->topo = std::make_unique<pso::gbest_topology<T>>();
  else r->topo = std::make_unique<pso::lbest_topology<T>>();
  if (update == 1) r->upd = std::make_unique<pso::spherical_update<T>>();
  else r->upd = std::make_unique<pso::standard_update<T>>();
  r->params.attraction = T(attraction);
  r->params.inertia = T(w);
  r->params.cognitive = T(c1);
  r->params.social = T(c2);
  r->vmax = T(vmax);
  r->P = P;
  r->D = D;
  r->problem = std::make_unique<problem_instance<T>>(
      make_base<T>(kind, D, static_cast<const T*>(shift), static_cast<const T*>(rot), bias));
  return r;
}

template <typename T>
void pso_set(void* h, const void* x, const void* v, const void* fit) {
  auto* r = static_cast<ref_pso_run<T>*>(h);
  const T* X = static_cast<const T*>(x);
  const T* V = static_cast<const T*>(v);
  const T* F = static_cast<const T*>(fit);
  r->x.assign(size_t(r->P), std::vector<T>(size_t(r->D)));
  r->v.assign(size_t(r->P), std::vector<T>(size_t(r->D)));
  r->pb.assign(size_t(r->P), individual<T>(r->D));
  r->fit.assign(size_t(r->P), T(0));
  for (int i = 0; i < r->P; ++i) {
    std::memcpy(r->x[size_t(i)].data(), X + size_t(i) * r->D, sizeof(T) * r->D);
    std::memcpy(r->v[size_t(i)].data(), V + size_t(i) * r->D, sizeof(T) * r->D);
    r->fit[size_t(i)] = F[i];
    r->pb[size_t(i)].genome = r->x[size_t(i)];  // prepare(), first call (pso/engine.hpp:40-45)
    r->pb[size_t(i)].fitness = F[i];
    r->pb[size_t(i)].evaluated = true;
  }
}

template <typename T>
void pso_get(void* h, void* x, void* v, void* fit, void* pb, void* pbf) {
  auto* r = static_cast<ref_pso_run<T>*>(h);
  for (int i = 0; i < r->P; ++i) {
    if (x) std::memcpy(static_cast<T*>(x) + size_t(i) * r->D, r->x[size_t(i)].data(), sizeof(T) * r->D);
    if (v) std::memcpy(static_cast<T*>(v) + size_t(i) * r->D, r->v[size_t(i)].data(), sizeof(T) * r->D);
    if (pb) std::memcpy(static_cast<T*>(pb) + size_t(i) * r->D, r->pb[size_t(i)].genome.data(), sizeof(T) * r->D);
    if (fit) static_cast<T*>(fit)[i] = r->fit[size_t(i)];
    if (pbf) static_cast<T*>(pbf)[i] = r->pb[size_t(i)].fitness;
  }
}
}  // namespace

REF_API void* ref_pso_create(int dtype, int topology, double w, double c1, double c2, double vmax, int P, int D,
                             int kind, const void* shift, const void* rot, double bias, int update, double attraction) {
  return dtype == 1 ? pso_create<double>(topology, w, c1, c2, vmax, P, D, kind, shift, rot, bias, update, attraction)
                    : pso_create<float>(topology, w, c1, c2, vmax, P, D, kind, shift, rot, bias, update, attraction);
}
REF_API void ref_pso_set(int dtype, void* h, const void* x, const void* v, const void* fit) {
  dtype == 1 ? pso_set<double>(h, x, v, fit) : pso_set<float>(h, x, v, fit);
}
REF_API int ref_pso_step(int dtype, void* h, const uint64_t* words, int64_t n, double lb, double ub) {
  return dtype == 1 ? static_cast<ref_pso_run<double>*>(h)->step(words, n, lb, ub)
                    : static_cast<ref_pso_run<float>*>(h)->step(words, n, float(lb), float(ub));
}
REF_API void ref_pso_get(int dtype, void* h, void* x, void* v, void* fit, void* pb, void* pbf) {
  dtype == 1 ? pso_get<double>(h, x, v, fit, pb, pbf) : pso_get<float>(h, x, v, fit, pb, pbf);
}
REF_API void ref_pso_destroy(int dtype, void* h) {
  if (dtype == 1) delete static_cast<ref_pso_run<double>*>(h);
  else delete static_cast<ref_pso_run<float>*>(h);
}

REF_API void ref_make_composition(uint64_t seed, uint64_t stream, int dim, int n_comp, double* shifts, double* rots) {
  rng_stream r = derive_stream(seed, stream);
  std::vector<double> scratch;
  for (int c = 0; c < n_comp; ++c) {
    auto o = problems::detail::draw_shift<double>(dim, -100.0, 100.0, r);
    auto m = problems::detail::draw_rotation<double>(dim, r, scratch);
    std::memcpy(shifts + size_t(c) * dim, o.data(), sizeof(double) * dim);
    std::memcpy(rots + size_t(c) * dim * dim, m.data(), sizeof(double) * size_t(dim) * dim);
  }
}

REF_API void ref_pso_set_threads(int dtype, void* h, int threads) {
  if (dtype == 1) static_cast<ref_pso_run<double>*>(h)->threads = threads;
  else static_cast<ref_pso_run<float>*>(h)->threads = threads;
}

// ---- CPU baselines through the reference's own harness (bench_configs.py) ------------------------
#include <chrono>

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// Config 4: evo_bench (experiment/runner.hpp:101-160) with the `de` preset (presets.hpp:621-628)
// over a suite of n_runs composition instances, `threads` workers; max_fes covers init + gens.
REF_API double ref_bench_config4(int n_runs, int P, int D, int gens, int threads, const double* shifts,
                                 const double* rots, const int* kinds, const double* sigma, const double* lambda,
                                 const double* cbias) {
  std::vector<problem_instance<double>> inst;
  for (int r = 0; r < n_runs; ++r)
    inst.push_back(make_comp<double>(D, 3, kinds, shifts + size_t(r) * 3 * D, rots + size_t(r) * 3 * D * D, sigma,
                                     lambda, cbias, 0.0));
  problems::suite<double> su("config4", D, {11}, n_runs, 64, std::move(inst));
  experiment::observer<double> obs;
  experiment::bench_options opt;
  opt.independent_runs = 1;
  opt.max_fes = (long long)P * (gens + 1);
  opt.parallel = threads > 1;
  opt.threads = threads;
  opt.master_seed = 64;
  presets::algorithm_options ao;
  ao.name = "de";
  ao.pop_size = P;
  auto alg = presets::make_algorithm<double>(ao);
  const double t0 = now_s();
  experiment::evo_bench(alg, su, obs, opt);
  return now_s() - t0;
}

// Configs 0 / 2: one de_engine run on its native stream; returns seconds for `gens` generations
// (init + evaluation excluded).  preset 0: build_de_fixed(0.5, 0.9); 1: build_shade(0.11, P, 1.0).
REF_API double ref_bench_de(int preset, int P, int D, int gens, int kind, const double* shift, const double* rot,
                            uint64_t seed) {
  auto engine = preset == 0 ? presets::detail::build_de_fixed<double>(0.5, 0.9)
                            : presets::detail::build_shade<double>(0.11, P, 1.0, de::population_policy::fixed());
  auto prob = make_base<double>(kind, D, shift, rot, 0.0);
  rng_stream rng(seed, 0);
  auto pop = init_population<double>(P, D, -100.0, 100.0, rng);
  eval_scratch<double> scratch;
  auto objective = [&](std::span<const double> x) { return prob.evaluate(x, scratch); };
  for (auto& m : pop) m.evaluate(objective);
  engine.archive().set_capacity(engine.archive_capacity_for(P), rng);
  evolution_state st(1LL << 40, P, D, std::min(4, P));
  const double t0 = now_s();
  for (int g = 0; g < gens; ++g) engine.generation(pop, st, objective, -100.0, 100.0, rng);
  return now_s() - t0;
}

// ---- best_so_far_record (experiment/recorder.hpp) fed with given value sequences ----------------
#include "evobench/experiment/recorder.hpp"

// values: runs x n (row per run); counts[r] values of run r are observed (then on_run_end).
// Writes the grid (runs x checkpoints) and the CSV (returns its length; csv may be null).
REF_API int64_t ref_record(const double* values, int n, const int* counts, int runs, int dim, long long max_fes,
                           long long interval, double* grid, char* csv, int64_t cap) {
  std::vector<problem_instance<double>> inst;
  inst.push_back(make_instance<double>(1, dim, 1, 0));
  problems::suite<double> su("gpu", dim, {1}, 1, 0, std::move(inst));
  experiment::best_so_far_record<double> rec(su, runs, max_fes, interval);
  for (int r = 0; r < runs; ++r) {
    experiment::run_key key{1, 1, 0, 0, r};
    for (int q = 0; q < counts[r]; ++q) rec.on_evaluate(key, q + 1, values[size_t(r) * n + q]);
    rec.on_run_end(key);
  }
  for (int r = 0; r < runs; ++r)
    for (int c = 0; c < rec.checkpoint_count(); ++c) grid[size_t(r) * rec.checkpoint_count() + c] = rec.at(0, 0, r, c);
  const std::string s = rec.to_csv();
  if (csv) std::memcpy(csv, s.data(), std::min<size_t>(size_t(cap), s.size()));
  return int64_t(s.size());
}

// one generation like ref_de_generation, additionally returning every objective value in call
// (FE) order
REF_API int ref_de_generation_trace(void* h, const uint64_t* words, int64_t n, double lb, double ub, double* values) {
  auto* r = static_cast<ref_de_run*>(h);
  const uint64_t sentinel = 0xa5a5a5a5deadbeefULL;
  std::vector<uint64_t> w(words, words + n);
  w.push_back(sentinel);
  rng_stream rng = rng_stream::scripted(w);
  evolution_state st(1LL << 40, r->P, r->D, std::min(4, r->P));
  eval_scratch<double> scratch;
  int q = 0;
  auto objective = [&](std::span<const double> x) {
    const double v = r->problem->evaluate(x, scratch);
    values[q++] = v;
    return v;
  };
  r->engine->generation(r->pop, st, objective, lb, ub, rng);
  return rng.next_u64() == sentinel ? 1 : 0;
}

// ref_de_native_run that also returns every objective value in call (FE) order:
// P initial evaluations, then P trials per generation
REF_API void ref_de_native_trace(void* h, uint64_t seed, uint64_t stream, int generations, double lb, double ub,
                                 double* values) {
  auto* r = static_cast<ref_de_run*>(h);
  rng_stream rng(seed, stream);
  r->pop = init_population<double>(r->P, r->D, lb, ub, rng);
  eval_scratch<double> scratch;
  int64_t q = 0;
  auto objective = [&](std::span<const double> x) {
    const double v = r->problem->evaluate(x, scratch);
    values[q++] = v;
    return v;
  };
  for (auto& m : r->pop) m.evaluate(objective);
  r->engine->archive().set_capacity(r->engine->archive_capacity_for(r->P), rng);
  evolution_state st(1LL << 40, r->P, r->D, std::min(4, r->P));
  for (int g = 0; g < generations; ++g) r->engine->generation(r->pop, st, objective, lb, ub, rng);
}

// ---- evo_bench (experiment/runner.hpp:101-160) over a suite of base problems, `de` preset ------
// The reference's own evo_bench + run_handle + best_so_far_record + de_engine::optimize; only the
// random words are substituted: task t draws from rng_stream::scripted(words[off[t], off[t+1])),
// the words the GPU's positional Philox stream of that task produces.  Returns the CSV length.
REF_API int64_t ref_evo_bench_de(double f, double cr, int P, int D, int n_problems, const int* problem_ids,
                                 int instances, int runs, long long max_fes, long long interval, const int* kinds,
                                 const double* shifts, const double* rots, double bias, const uint64_t* words,
                                 const int64_t* off, double lb, double ub, int threads, char* csv, int64_t cap,
                                 double* best) {
  std::vector<problem_instance<double>> inst;
  for (int q = 0; q < n_problems * instances; ++q)
    inst.push_back(make_base<double>(kinds[q], D, shifts + size_t(q) * D, rots + size_t(q) * D * D, bias));
  problems::suite<double> su("gpu", D, std::vector<int>(problem_ids, problem_ids + n_problems), instances, 0,
                             std::move(inst));
  experiment::best_so_far_record<double> rec(su, runs, max_fes, interval);
  experiment::bench_options opt;
  opt.independent_runs = runs;
  opt.max_fes = max_fes;
  opt.threads = threads;
  opt.parallel = threads != 1;
  auto alg = [&](experiment::run_handle<double>& h) {
    const auto& k = h.key();
    const int64_t t = (int64_t(k.problem_ordinal) * instances + k.instance_ordinal) * runs + k.run_index;
    rng_stream rng = rng_stream::scripted(std::vector<uint64_t>(words + off[t], words + off[t + 1]));
    auto engine = presets::detail::build_de_fixed<double>(f, cr);
    const auto b = engine.optimize(h, lb, ub, P, D, max_fes, rng, [](int, auto) {});
    best[t] = b.fitness;
  };
  experiment::evo_bench<double>(alg, su, rec, opt);
  const std::string s = rec.to_csv();
  if (csv) std::memcpy(csv, s.data(), std::min<size_t>(size_t(cap), s.size()));
  return int64_t(s.size());
}

// ---- CSO (pso/cso.hpp): the UNMODIFIED cso_optimizer stepped generation by generation ----------
#include "evobench/pso/cso.hpp"

namespace {
template <typename T>
struct ref_cso_run {
  std::unique_ptr<pso::cso_optimizer<T>> opt;
  std::unique_ptr<problem_instance<T>> problem;
  population<T> pop;
  std::vector<std::vector<T>> v;
  int P = 0, D = 0;
};

template <typename T>
void* cso_create(double phi, int P, int D, int kind, const void* shift, const void* rot, double bias) {
  auto* r = new ref_cso_run<T>();
  r->opt = std::make_unique<pso::cso_optimizer<T>>(T(phi));
  r->P = P;
  r->D = D;
  r->pop = population<T>(P, D);
  r->v.assign(size_t(P), std::vector<T>(size_t(D), T(0)));
  r->problem = std::make_unique<problem_instance<T>>(
      make_base<T>(kind, D, static_cast<const T*>(shift), static_cast<const T*>(rot), bias));
  return r;
}

template <typename T>
void cso_set(void* h, const void* x, const void* v, const void* fit) {
  auto* r = static_cast<ref_cso_run<T>*>(h);
  for (int i = 0; i < r->P; ++i) {
    std::memcpy(r->pop[i].genome.data(), static_cast<const T*>(x) + size_t(i) * r->D, sizeof(T) * r->D);
    std::memcpy(r->v[size_t(i)].data(), static_cast<const T*>(v) + size_t(i) * r->D, sizeof(T) * r->D);
    r->pop[i].fitness = static_cast<const T*>(fit)[i];
    r->pop[i].evaluated = true;
  }
}

template <typename T>
int cso_step(void* h, const uint64_t* words, int64_t n, T lb, T ub) {
  auto* r = static_cast<ref_cso_run<T>*>(h);
  const uint64_t sentinel = 0x0c50c50c50c50c50ULL;
  std::vector<uint64_t> w(words, words + n);
  w.push_back(sentinel);
  rng_stream rng = rng_stream::scripted(w);
  evolution_state st(1LL << 40, r->P, r->D, std::min(4, r->P));
  eval_scratch<T> scratch;
  auto objective = [&](std::span<const T> x) { return r->problem->evaluate(x, scratch); };
  r->opt->generation(r->pop, r->v, st, objective, lb, ub, rng);
  return rng.next_u64() == sentinel ? 1 : 0;
}

template <typename T>
void cso_get(void* h, void* x, void* v, void* fit) {
  auto* r = static_cast<ref_cso_run<T>*>(h);
  for (int i = 0; i < r->P; ++i) {
    if (x) std::memcpy(static_cast<T*>(x) + size_t(i) * r->D, r->pop[i].genome.data(), sizeof(T) * r->D);
    if (v) std::memcpy(static_cast<T*>(v) + size_t(i) * r->D, r->v[size_t(i)].data(), sizeof(T) * r->D);
    if (fit) static_cast<T*>(fit)[i] = r->pop[i].fitness;
  }
}

template <typename T>
double cso_native(void* h, uint64_t seed, uint64_t stream, double lb, double ub, long long max_fes) {
  auto* r = static_cast<ref_cso_run<T>*>(h);
  rng_stream rng(seed, stream);
  eval_scratch<T> scratch;
  auto objective = [&](std::span<const T> x) { return r->problem->evaluate(x, scratch); };
  const auto best = r->opt->optimize(objective, T(lb), T(ub), r->P, r->D, max_fes, rng);
  return double(best.fitness);
}
}  // namespace

REF_API void* ref_cso_create(int dtype, double phi, int P, int D, int kind, const void* shift, const void* rot,
                             double bias) {
  return dtype == 1 ? cso_create<double>(phi, P, D, kind, shift, rot, bias)
                    : cso_create<float>(phi, P, D, kind, shift, rot, bias);
}
REF_API void ref_cso_set(int dtype, void* h, const void* x, const void* v, const void* fit) {
  dtype == 1 ? cso_set<double>(h, x, v, fit) : cso_set<float>(h, x, v, fit);
}
REF_API int ref_cso_step(int dtype, void* h, const uint64_t* words, int64_t n, double lb, double ub) {
  return dtype == 1 ? cso_step<double>(h, words, n, lb, ub) : cso_step<float>(h, words, n, float(lb), float(ub));
}
REF_API void ref_cso_get(int dtype, void* h, void* x, void* v, void* fit) {
  dtype == 1 ? cso_get<double>(h, x, v, fit) : cso_get<float>(h, x, v, fit);
}
// cso_optimizer::optimize on the reference's NATIVE stream rng_stream(seed, stream); returns the best fitness
REF_API double ref_cso_native_optimize(int dtype, void* h, uint64_t seed, uint64_t stream, double lb, double ub,
                                       long long max_fes) {
  return dtype == 1 ? cso_native<double>(h, seed, stream, lb, ub, max_fes)
                    : cso_native<float>(h, seed, stream, lb, ub, max_fes);
}
REF_API void ref_cso_destroy(int dtype, void* h) {
  if (dtype == 1) delete static_cast<ref_cso_run<double>*>(h);
  else delete static_cast<ref_cso_run<float>*>(h);
}

// evo_bench with the `cso` preset (presets.hpp: cso_optimizer{phi}.optimize(h, ...)), words
// substituted per task exactly like ref_evo_bench_de
REF_API int64_t ref_evo_bench_cso(double phi, int P, int D, int n_problems, const int* problem_ids, int instances,
                                  int runs, long long max_fes, long long interval, const int* kinds,
                                  const double* shifts, const double* rots, double bias, const uint64_t* words,
                                  const int64_t* off, double lb, double ub, int threads, char* csv, int64_t cap,
                                  double* best) {
  std::vector<problem_instance<double>> inst;
  for (int q = 0; q < n_problems * instances; ++q)
    inst.push_back(make_base<double>(kinds[q], D, shifts + size_t(q) * D, rots + size_t(q) * D * D, bias));
  problems::suite<double> su("gpu", D, std::vector<int>(problem_ids, problem_ids + n_problems), instances, 0,
                             std::move(inst));
  experiment::best_so_far_record<double> rec(su, runs, max_fes, interval);
  experiment::bench_options opt;
  opt.independent_runs = runs;
  opt.max_fes = max_fes;
  opt.threads = threads;
  opt.parallel = threads != 1;
  auto alg = [&](experiment::run_handle<double>& h) {
    const auto& k = h.key();
    const int64_t t = (int64_t(k.problem_ordinal) * instances + k.instance_ordinal) * runs + k.run_index;
    rng_stream rng = rng_stream::scripted(std::vector<uint64_t>(words + off[t], words + off[t + 1]));
    pso::cso_optimizer<double> engine{phi};
    const auto b = engine.optimize(h, lb, ub, P, D, max_fes, rng);
    best[t] = b.fitness;
  };
  experiment::evo_bench<double>(alg, su, rec, opt);
  const std::string s = rec.to_csv();
  if (csv) std::memcpy(csv, s.data(), std::min<size_t>(size_t(cap), s.size()));
  return int64_t(s.size());
}

// ---- parameter_record (experiment/parameter_record.hpp) fed with given series ------------------
#include "evobench/experiment/parameter_record.hpp"

// mu_F / mu_CR the engine's adapter reports now (parameter_adapter::append_parameters)
REF_API int ref_de_params(void* h, double* mu_f, double* mu_cr) {
  auto* r = static_cast<ref_de_run*>(h);
  std::vector<named_value<double>> v;
  r->engine->parameter().append_parameters(v);
  for (const auto& nv : v) {
    if (nv.name == "mu_f") *mu_f = nv.value;
    if (nv.name == "mu_cr") *mu_cr = nv.value;
  }
  return int(v.size());
}

// runs x n entries (counts[r] used), on_generation per entry, returns to_csv's length
REF_API int64_t ref_param_record(const int* gens, const double* mu_f, const double* mu_cr, int n, const int* counts,
                                 int n_problems, const int* problem_ids, int instances, int runs, int dim, char* csv,
                                 int64_t cap) {
  std::vector<problem_instance<double>> inst;
  for (int q = 0; q < n_problems * instances; ++q) inst.push_back(make_instance<double>(1, dim, 1, 0));
  problems::suite<double> su("gpu", dim, std::vector<int>(problem_ids, problem_ids + n_problems), instances, 0,
                             std::move(inst));
  experiment::parameter_record<double> rec(su, runs);
  for (int p = 0; p < n_problems; ++p)
    for (int i = 0; i < instances; ++i)
      for (int k = 0; k < runs; ++k) {
        const int run = (p * instances + i) * runs + k;
        experiment::run_key key{problem_ids[p], i + 1, p, i, k};
        for (int e = 0; e < counts[run]; ++e) {
          const size_t q = size_t(run) * n + e;
          const named_value<double> params[2] = {{"mu_f", mu_f[q]}, {"mu_cr", mu_cr[q]}};
          rec.on_generation(key, gens[q], std::span<const named_value<double>>(params, 2));
        }
      }
  const std::string s = rec.to_csv();
  if (csv) std::memcpy(csv, s.data(), std::min<size_t>(size_t(cap), s.size()));
  return int64_t(s.size());
}

// ---- hybrid::restart_run with the restart-lshade factory (presets.hpp), native stream ----------
#include "evobench/hybrid/restart.hpp"

REF_API double ref_restart_lshade(uint64_t seed, uint64_t stream, int P, int D, int H, double p_best,
                                  double archive_rate, int n_min, long long budget, long long stagnation, double eps,
                                  int kind, const double* shift, const double* rot, double bias, int* runs,
                                  long long* evals, double lb, double ub) {
  auto problem = make_base<double>(kind, D, shift, rot, bias);
  eval_scratch<double> scratch;
  auto objective = [&](std::span<const double> x) { return problem.evaluate(x, scratch); };
  hybrid::restart_criterion crit;
  crit.stagnation_evals = stagnation;
  crit.epsilon = eps;
  const auto factory = [&] {
    return presets::detail::build_shade<double>(p_best, H, archive_rate, de::population_policy::linear_reduction(P, n_min));
  };
  rng_stream rng(seed, stream);
  auto res = hybrid::restart_run<double>(factory, crit, objective, lb, ub, P, D, budget, rng, [](int, auto) {});
  *runs = res.engine_runs;
  *evals = res.evaluations;
  return res.best.fitness;
}
