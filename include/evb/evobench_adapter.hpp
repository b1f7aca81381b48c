// evobench_adapter.hpp — the binding an evobench maintainer adds to route the hot path to the GPU.
// Requires the evobench headers on the include path (it is compiled against the UNMODIFIED
// reference in tests/cpp/test_adapter.cpp); everything GPU-side goes through include/evb/evb.hpp.
//
//   auto gp = evb::adapt::to_gpu(instance);              // problems::problem_instance<T> -> device
//   evb::evaluate_batch(gp, xs, gpu_scratch, out);       // same call shape as evaluate_batch
//
//   auto engine = presets::detail::build_shade<double>(0.11, 180, 1.0, ...);   // reference engine
//   auto gde = evb::adapt::to_gpu(engine, 180, 100);     // de::de_engine<T> -> gpu_de_engine<T>
//   auto gps = evb::adapt::to_gpu(pso_engine, 1024, 1000);  // pso::pso_engine<T> -> gpu_pso_engine<T>
//
// The engines' strategy objects are mapped to kernels by name() (de/strategy.hpp:77, 101, 133, 182,
// 202, 232, 246, 266, 282; de/parameter.hpp:87, 107, 157; pso/topology.hpp:26, 42;
// pso/update.hpp:64, 84) and then checked with dynamic_cast against the concrete reference type
// whose parameters the kernel needs; anything else throws evobench::config_error (there is no CPU
// fallback).  Every error from the GPU side surfaces as the reference's own exception types:
// this header defines EVB_WITH_EVOBENCH, which makes evb::config_error the very type
// evobench::config_error (common.hpp:12-15).
//
// run_handle<T>::evaluate_batch (experiment/runner.hpp:47-53) can call the GPU form and keep its
// FE counting / observer notification unchanged.
#pragma once

#ifndef EVB_WITH_EVOBENCH
#define EVB_WITH_EVOBENCH 1
#endif

#include <cmath>
#include <optional>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "evobench/core/rng.hpp"
#include "evobench/de/engine.hpp"
#include "evobench/de/parameter.hpp"
#include "evobench/de/strategy.hpp"
#include "evobench/problems/instance.hpp"
#include "evobench/pso/engine.hpp"
#include "evb/evb.hpp"

static_assert(std::is_same<evb::config_error, evobench::config_error>::value,
              "include evb/evobench_adapter.hpp (or define EVB_WITH_EVOBENCH) before evb/evb.hpp");

namespace evb::adapt {

template <typename T>
gpu_problem<T> to_gpu(const evobench::problems::problem_instance<T>& p) {
  namespace ep = evobench::problems;
  if (const auto* kind = std::get_if<ep::base_kind>(&p.spec()))
    return gpu_problem<T>::base(evb::base_kind(int(*kind)), p.shift(), p.rotation(), p.bias());
  if (const auto* h = std::get_if<ep::hybrid_spec>(&p.spec())) {
    std::vector<int> kinds;
    for (auto k : h->sub_kinds) kinds.push_back(int(k));
    return gpu_problem<T>::hybrid(p.shift(), p.rotation(), p.bias(), kinds, h->chunk_sizes, h->permutation);
  }
  const auto& c = std::get<ep::composition_spec<T>>(p.spec());
  std::vector<int> kinds;
  std::vector<T> shifts, rots;
  std::vector<double> sigma, lambda, bias;
  for (const auto& comp : c.components) {
    kinds.push_back(int(comp.kind));
    shifts.insert(shifts.end(), comp.shift.begin(), comp.shift.end());
    rots.insert(rots.end(), comp.rotation.begin(), comp.rotation.end());
    sigma.push_back(comp.sigma);
    lambda.push_back(comp.lambda);
    bias.push_back(comp.bias);
  }
  return gpu_problem<T>::composition(p.dim(), kinds, shifts, rots, sigma, lambda, bias, p.bias());
}

namespace detail {

template <typename Concrete, typename Base>
const Concrete& as(const Base& obj, const char* slot) {
  const auto* c = dynamic_cast<const Concrete*>(&obj);
  if (!c)
    throw evobench::config_error(std::string("gpu adapter: ") + slot + " '" + std::string(obj.name()) +
                                 "' is not the reference's strategy of that name (no GPU kernel)");
  return *c;
}

[[noreturn]] inline void unknown(const char* slot, std::string_view name) {
  throw evobench::config_error(std::string("gpu adapter: unknown ") + slot + " strategy '" + std::string(name) +
                               "' (no GPU kernel)");
}

// jade_parameter keeps its learning rate private (de/parameter.hpp:141).  It is read back from
// one probe update while the adapter is in its initial state (mu_F = mu_CR = 0.5): with the
// single success F = 1, CR = 2^100, mu_CR becomes T((1 - c) * 0.5 + c * 2^100) = c * 2^100
// exactly (the 0.45 is below half an ulp of c * 2^100 for c >= 2^-46), so c is recovered
// bit for bit; reset() then restores the initial state exactly.
template <typename T>
double jade_learning_rate(evobench::de::jade_parameter<T>& j) {
  if (!(j.mu_f() == T(0.5) && j.mu_cr() == T(0.5)))
    throw evobench::config_error(
        "gpu adapter: jade learning rate is only observable on an adapter in its initial state (mu = 0.5); "
        "pass jade_learning_rate explicitly");
  const T big = T(std::ldexp(1.0, 100));
  const std::vector<T> f{T(1)}, cr{big}, gain{T(1)};
  j.update(f, cr, gain);
  const double c = std::ldexp(double(j.mu_cr()), -100);
  j.reset();
  if (!(c > 0.0 && c <= 1.0)) throw evobench::config_error("gpu adapter: jade learning rate probe failed");
  return c;
}

}  // namespace detail

struct de_mapping_options {
  std::optional<double> jade_learning_rate;  // required for a JADE adapter past its initial state
};

// de::de_engine<T> (de/engine.hpp:68-173, assembled by de_builder / presets) -> evb_de_config.
// The engine's config() slots are mapped by name(); ttpb_1 contributes p_best_fraction() and
// uses_archive() (de/strategy.hpp:135-136), shade memory_size() (de/parameter.hpp:203), fixed
// its constants through sample() (which draws nothing, :89), the policy its kind / n_init / n_min
// (de/policy.hpp:14-36) and the builder's archive_rate.
template <typename T>
evb_de_config de_config_of(const evobench::de::de_engine<T>& engine, int pop_size, de_mapping_options opt = {}) {
  namespace de = evobench::de;
  const de::de_config<T>& c = engine.config();
  if (!c.mutation || !c.crossover || !c.repair || !c.parameter)
    throw evobench::config_error("gpu adapter: de engine has an empty strategy slot");
  evb_de_config g{};
  const std::string_view mut = c.mutation->name();
  if (mut == "rand_1") {
    detail::as<de::rand1_mutation<T>>(*c.mutation, "mutation");
    g.mutation = EVB_MUT_RAND1;
  } else if (mut == "best_1") {
    detail::as<de::best1_mutation<T>>(*c.mutation, "mutation");
    g.mutation = EVB_MUT_BEST1;
  } else if (mut == "ttpb_1") {
    const auto& t = detail::as<de::ttpb1_mutation<T>>(*c.mutation, "mutation");
    g.mutation = EVB_MUT_TTPB1;
    g.p_best = double(t.p_best_fraction());
    g.use_archive = t.uses_archive() ? 1 : 0;
  } else {
    detail::unknown("mutation", mut);
  }
  const std::string_view cx = c.crossover->name();
  if (cx == "binomial") {
    detail::as<de::binomial_crossover<T>>(*c.crossover, "crossover");
    g.crossover = EVB_CX_BINOMIAL;
  } else if (cx == "exponential") {
    detail::as<de::exponential_crossover<T>>(*c.crossover, "crossover");
    g.crossover = EVB_CX_EXPONENTIAL;
  } else {
    detail::unknown("crossover", cx);
  }
  const std::string_view rep = c.repair->name();
  if (rep == "clip") {
    detail::as<de::clip_repair<T>>(*c.repair, "repair");
    g.repair = EVB_REP_CLIP;
  } else if (rep == "reflect") {
    detail::as<de::reflect_repair<T>>(*c.repair, "repair");
    g.repair = EVB_REP_REFLECT;
  } else if (rep == "midpoint_target") {
    detail::as<de::midpoint_target_repair<T>>(*c.repair, "repair");
    g.repair = EVB_REP_MIDPOINT_TARGET;
  } else if (rep == "reinitialize") {
    detail::as<de::reinitialize_repair<T>>(*c.repair, "repair");
    g.repair = EVB_REP_REINITIALIZE;
  } else {
    detail::unknown("repair", rep);
  }
  const std::string_view par = c.parameter->name();
  g.memory_size = 1;
  if (par == "fixed") {
    auto& f = const_cast<de::fixed_parameter<T>&>(detail::as<de::fixed_parameter<T>>(*c.parameter, "parameter adapter"));
    evobench::rng_stream none(0, 0);  // fixed_parameter::sample draws nothing (de/parameter.hpp:89)
    const auto p = f.sample(none);
    g.parameter = EVB_PAR_FIXED;
    g.f = double(p.scale_factor);
    g.cr = double(p.crossover_rate);
  } else if (par == "jade") {
    auto& j = const_cast<de::jade_parameter<T>&>(detail::as<de::jade_parameter<T>>(*c.parameter, "parameter adapter"));
    g.parameter = EVB_PAR_JADE;
    g.jade_c = opt.jade_learning_rate ? *opt.jade_learning_rate : detail::jade_learning_rate(j);
  } else if (par == "shade") {
    const auto& s = detail::as<de::shade_parameter<T>>(*c.parameter, "parameter adapter");
    g.parameter = EVB_PAR_SHADE;
    g.memory_size = s.memory_size();
  } else {
    detail::unknown("parameter adapter", par);
  }
  g.archive_rate = double(c.archive_rate);
  if (c.policy.kind == de::population_policy::kind_t::linear_reduction) {
    if (c.policy.n_init != pop_size)
      throw evobench::config_error("gpu adapter: linear_reduction N_init (" + std::to_string(c.policy.n_init) +
                                   ") must equal the population size (" + std::to_string(pop_size) + ")");
    g.reduction = EVB_POP_LINEAR_REDUCTION;
    g.n_min = c.policy.n_min;
  } else {
    g.reduction = EVB_POP_FIXED;
    g.n_min = 4;
  }
  return g;
}

// de::de_engine<T> -> gpu_de_engine<T>: the same strategy set, plus the engine's adaptation state
// (SHADE memories and write index, JADE means) and archive contents, so a run can move to the
// GPU mid-way.  Validation (population too small for the mutation, p range, ...) is the GPU
// engine's, which mirrors de_builder::build and de_engine::validate_run (de/builder.hpp:51-57;
// de/engine.hpp:148-152) and throws evobench::config_error.
template <typename T>
gpu_de_engine<T> to_gpu(const evobench::de::de_engine<T>& engine, int pop_size, int dim, de_mapping_options opt = {}) {
  namespace de = evobench::de;
  const evb_de_config cfg = de_config_of(engine, pop_size, opt);
  gpu_de_engine<T> g(cfg, pop_size, dim);
  std::vector<T> mf, mc, rows;
  int wi = 0;
  const de::parameter_adapter<T>& ad = *engine.config().parameter;
  if (const auto* s = dynamic_cast<const de::shade_parameter<T>*>(&ad)) {
    mf = s->memory_f();
    mc = s->memory_cr();
    wi = s->write_index();
  } else if (const auto* j = dynamic_cast<const de::jade_parameter<T>*>(&ad)) {
    mf = {j->mu_f()};
    mc = {j->mu_cr()};
  }
  const de::de_archive<T>& ar = engine.archive();
  const int n_ar = ar.size();
  if (n_ar > g.archive_capacity())
    throw evobench::config_error("gpu adapter: the engine's archive holds more members than ceil(rate * pop_size)");
  for (int k = 0; k < n_ar; ++k) {
    const auto& m = ar.member(k);
    if (int(m.size()) != dim) throw std::invalid_argument("gpu adapter: archive member dimension mismatch");
    rows.insert(rows.end(), m.begin(), m.end());
  }
  if (!mf.empty() || n_ar > 0) g.set_state(rows, n_ar, mf, mc, wi);
  return g;
}

// pso::pso_engine<T> (pso/engine.hpp:33-121) -> evb_pso_config: topology by name ("gbest",
// "lbest_ring"), velocity rule by name ("standard", "spherical"), swarm_params copied.  vmax > 0
// adds BASELINE config 3's velocity clamp (the stock engine has none).
template <typename T>
evb_pso_config pso_config_of(const evobench::pso::pso_engine<T>& engine, double vmax = 0.0) {
  namespace ps = evobench::pso;
  const ps::pso_config<T>& c = engine.config();
  if (!c.topology || !c.update) throw evobench::config_error("gpu adapter: pso engine has an empty strategy slot");
  evb_pso_config g{};
  const std::string_view topo = c.topology->name();
  if (topo == "gbest") {
    detail::as<ps::gbest_topology<T>>(*c.topology, "topology");
    g.topology = EVB_TOPO_GBEST;
  } else if (topo == "lbest_ring") {
    detail::as<ps::lbest_topology<T>>(*c.topology, "topology");
    g.topology = EVB_TOPO_LBEST_RING;
  } else {
    detail::unknown("topology", topo);
  }
  const std::string_view upd = c.update->name();
  if (upd == "standard") {
    detail::as<ps::standard_update<T>>(*c.update, "velocity update");
    g.update = EVB_UPD_STANDARD;
  } else if (upd == "spherical") {
    detail::as<ps::spherical_update<T>>(*c.update, "velocity update");
    g.update = EVB_UPD_SPHERICAL;
  } else {
    detail::unknown("velocity update", upd);
  }
  g.inertia = double(c.params.inertia);
  g.cognitive = double(c.params.cognitive);
  g.social = double(c.params.social);
  g.attraction = double(c.params.attraction);
  g.vmax = vmax;
  return g;
}

// pso::pso_engine<T> -> gpu_pso_engine<T> (synchronous generation); the engine's
// personal bests, when it holds pop_size of them, are carried over (prepare() already ran).
template <typename T>
gpu_pso_engine<T> to_gpu(const evobench::pso::pso_engine<T>& engine, int pop_size, int dim, double vmax = 0.0) {
  gpu_pso_engine<T> g(pso_config_of(engine, vmax), pop_size, dim);
  const auto& pb = engine.personal_bests();
  if (int(pb.size()) == pop_size) {
    std::vector<T> rows, fit;
    rows.reserve(size_t(pop_size) * dim);
    for (const auto& m : pb) {
      if (int(m.genome.size()) != dim) throw std::invalid_argument("gpu adapter: personal best dimension mismatch");
      rows.insert(rows.end(), m.genome.begin(), m.genome.end());
      fit.push_back(m.fitness);
    }
    g.set_personal_bests(rows, fit);
  }
  return g;
}

}  // namespace evb::adapt
