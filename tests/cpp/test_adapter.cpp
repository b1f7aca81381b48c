// C++ parity test through the C++ host side (include/evb/evb.hpp + evobench_adapter.hpp) against
// the UNMODIFIED reference (compiled in from /root/reference by __graft_entry__.build()).
// Reads like the reference's own acceptance tests: PASS / FAIL lines, exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <span>
#include <string>
#include <vector>

#include "evb/evobench_adapter.hpp"
#include "evb/evb.hpp"
#include "evobench/experiment/recorder.hpp"
#include "evobench/experiment/runner.hpp"
#include "evobench/pso/cso.hpp"
#include "evobench/presets.hpp"
#include "evobench/core/rng.hpp"
#include "evobench/de/engine.hpp"
#include "evobench/presets.hpp"
#include "evobench/problems/batch.hpp"
#include "evobench/problems/suite.hpp"

using namespace evobench;

static int failures = 0;
static void report(const std::string& name, bool ok, const std::string& detail = "") {
  std::printf("%s [%s]%s%s\n", name.c_str(), ok ? "PASS" : "FAIL", detail.empty() ? "" : " - ", detail.c_str());
  if (!ok) ++failures;
}

template <typename T>
static double max_rel(const std::vector<T>& a, const std::vector<T>& b) {
  double w = 0;
  for (size_t i = 0; i < a.size(); ++i)
    w = std::max(w, std::abs(double(a[i]) - double(b[i])) / std::max(1.0, std::abs(double(b[i]))));
  return w;
}

int main() {
  // identity-transform sphere instance gives shifted values (tests/test_problems.cpp:132-139)
  {
    std::vector<double> eye(9, 0.0);
    eye[0] = eye[4] = eye[8] = 1.0;
    problems::problem_instance<double> p(1, 1, 3, -100.0, 100.0, std::vector<double>(3, 0.0), eye, 100.0,
                                         problems::base_kind::sphere, "sphere");
    auto gp = evb::adapt::to_gpu(p);
    auto out = evb::batched_evaluate(gp, std::vector<std::vector<double>>{{1.0, 2.0, 3.0}});
    report("identity sphere == 114", out.size() == 1 && out[0] == 114.0);
    bool threw = false;
    try {
      evb::batched_evaluate(gp, std::vector<std::vector<double>>{{1.0}});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    report("dimension mismatch throws std::invalid_argument", threw);
  }
  // every registry problem (base, hybrid, composition), double and float, batched GPU vs the
  // reference's evaluate_batch (tests/test_problems.cpp:277-333 convention)
  for (int dim : {10, 100}) {
    for (const auto& info : problems::problem_registry()) {
      auto p = problems::make_instance<double>(info.id, dim, 1, 4);
      rng_stream rng(2222, uint64_t(info.id));
      std::vector<std::vector<double>> xs(13, std::vector<double>(size_t(dim)));
      for (auto& x : xs)
        for (auto& v : x) v = rng.uniform(-100.0, 100.0);
      auto ref = problems::batched_evaluate(p, xs);
      auto got = evb::batched_evaluate(evb::adapt::to_gpu(p), xs);
      const double err = max_rel(got, ref);
      report("registry " + std::string(info.name) + " dim " + std::to_string(dim) + " fp64", err <= 1e-10,
             "max rel " + std::to_string(err));
      auto pf = problems::make_instance<float>(info.id, dim, 1, 4);
      std::vector<std::vector<float>> xf(13, std::vector<float>(size_t(dim)));
      for (size_t b = 0; b < xs.size(); ++b)
        for (int j = 0; j < dim; ++j) xf[b][size_t(j)] = float(xs[b][size_t(j)]);
      auto reff = problems::batched_evaluate(pf, xf);
      auto gotf = evb::batched_evaluate(evb::adapt::to_gpu(pf), xf);
      const double errf = max_rel(gotf, reff);
      report("registry " + std::string(info.name) + " dim " + std::to_string(dim) + " fp32", errf <= 1e-4,
             "max rel " + std::to_string(errf));
    }
  }
  // 1000-D batched parity (tests/test_problems.cpp:370-401 style) on a seeded instance
  {
    auto p = problems::make_instance<double>(5, 1000, 1, 7);
    rng_stream rng(65, 0);
    std::vector<std::vector<double>> xs(64, std::vector<double>(1000));
    for (auto& x : xs)
      for (auto& v : x) v = rng.uniform(-100.0, 100.0);
    auto ref = problems::batched_evaluate(p, xs);
    auto got = evb::batched_evaluate(evb::adapt::to_gpu(p), xs);
    report("ackley 1000-D batched", max_rel(got, ref) <= 1e-10, "max rel " + std::to_string(max_rel(got, ref)));
  }
  // DE: the GPU engine on the reference's native stream == the reference engine (config 0 shape)
  {
    const int P = 100, D = 10, G = 20;
    auto inst = problems::make_instance<double>(4, D, 1, 42);
    auto engine = presets::detail::build_de_fixed<double>(0.5, 0.9);
    rng_stream rng(42, 0);
    auto pop = init_population<double>(P, D, -100.0, 100.0, rng);
    problems::eval_scratch<double> scratch;
    auto obj = [&](std::span<const double> x) { return inst.evaluate(x, scratch); };
    for (auto& m : pop) m.evaluate(obj);
    evolution_state st(1LL << 40, P, D);
    for (int g = 0; g < G; ++g) engine.generation(pop, st, obj, -100.0, 100.0, rng);

    std::vector<uint64_t> words;
    rng_stream wr(42, 0);
    for (int i = 0; i < P * D + G * P * (D + 30); ++i) words.push_back(wr.next_u64());
    auto grng = evb::gpu_rng::words(words);
    auto gp = evb::adapt::to_gpu(inst);
    evb::gpu_de_engine<double> ge(evb::de_preset_fixed(0.5, 0.9), P, D);
    evb::device_vector<double> dpop(static_cast<size_t>(P) * D), dfit(static_cast<size_t>(P));
    ge.init_population(dpop.data(), D, -100.0, 100.0, grng);
    evb::gpu_scratch gs;
    evb::evaluate_batch(gp, dpop.data(), P, D, gs, dfit.data());
    for (int g = 0; g < G; ++g) ge.generation(gp, dpop.data(), D, dfit.data(), -100.0, 100.0, grng);
    auto hp = dpop.download();
    bool same = true;
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < D; ++j) same = same && hp[size_t(i) * D + j] == pop[i].genome[size_t(j)];
    report("DE rand/1/bin 20 generations on rng_stream(42, 0): bit-exact population", same);
  }
  // A whole experiment on the device: experiment::evo_bench with the `cso` preset over a registry
  // suite (transcendental-free problems, so every evaluation is bit-exact), recorded by the device
  // best_so_far_record, against the reference's own evo_bench + best_so_far_record where each task
  // replays the words of the GPU task's positional Philox stream.
  {
    const int D = 10, P = 20, runs = 2;
    const long long max_fes = P + 12 * (P / 2) + 5, interval = 25;
    const uint64_t seed = 77;
    const double phi = 0.1;
    auto su = problems::suite_builder<double>().name("cec").dim(D).problem_ids({1, 2, 3, 7}).instance_count(2).seed(9).build();
    std::vector<evb::gpu_problem<double>> gpu;
    for (int p = 0; p < su.problem_count(); ++p)
      for (int i = 0; i < su.instance_count(); ++i) gpu.push_back(evb::adapt::to_gpu(su.at(p, i)));
    std::vector<const evb::gpu_problem<double>*> inst;
    for (const auto& g : gpu) inst.push_back(&g);
    const int tasks = su.problem_count() * su.instance_count() * runs;
    evb::gpu_recorder<double> grec(tasks, max_fes, interval);
    auto gbest = evb::evo_bench_cso<double>(phi, P, inst, su.problem_count(), runs, max_fes, seed, -100.0, 100.0, &grec);
    const std::string gcsv = grec.to_csv(su.name(), D, su.problem_ids(), su.instance_count(), runs);

    // words each task consumes: init_population, then per generation the P-1 Fisher-Yates draws
    // (sub-stream 0xFFFFFFFD) and pair t's 3*D gene draws (sub-stream t)
    const int gens = int((max_fes - P + P / 2 - 1) / (P / 2));
    auto words_of = [&](int64_t t) {
      const uint64_t key = evb_task_key(seed, uint64_t(t));
      std::vector<uint64_t> w(size_t(P) * D);
      evb::check(evb_philox_words(key, 0xFFFFFFF0ull, 0, int64_t(P) * D, w.data()), "philox_words");
      for (uint64_t g = 1; g <= uint64_t(gens); ++g) {
        std::vector<uint64_t> part(size_t(P - 1));
        evb::check(evb_philox_words(key, (g << 32) | 0xFFFFFFFDull, 0, P - 1, part.data()), "philox_words");
        w.insert(w.end(), part.begin(), part.end());
        for (uint64_t pr = 0; pr < uint64_t(P / 2); ++pr) {
          std::vector<uint64_t> q(size_t(3) * D);
          evb::check(evb_philox_words(key, (g << 32) | pr, 0, 3 * D, q.data()), "philox_words");
          w.insert(w.end(), q.begin(), q.end());
        }
      }
      return w;
    };
    experiment::best_so_far_record<double> rrec(su, runs, max_fes, interval);
    experiment::bench_options opt;
    opt.independent_runs = runs;
    opt.max_fes = max_fes;
    opt.master_seed = seed;
    std::vector<double> rbest(static_cast<size_t>(tasks));
    auto alg = [&](experiment::run_handle<double>& h) {
      const auto& k = h.key();
      const int64_t t = (int64_t(k.problem_ordinal) * su.instance_count() + k.instance_ordinal) * runs + k.run_index;
      rng_stream rng = rng_stream::scripted(words_of(t));
      pso::cso_optimizer<double> engine{phi};
      rbest[size_t(t)] = engine.optimize(h, h.lb(), h.ub(), P, D, max_fes, rng).fitness;
    };
    experiment::evo_bench<double>(alg, su, rrec, opt);
    report("evo_bench cso over a registry suite: device recorder CSV == reference CSV", gcsv == rrec.to_csv());
    report("evo_bench cso: best per task equal", gbest == rbest);
  }
  // ---- DE / PSO engines handed over as the reference's own objects (evb::adapt::to_gpu) ----------
  // `de` preset (presets.hpp:59-69): name()-mapped slots, fixed F/CR read through sample(); the GPU
  // engine built from the reference engine object runs 20 generations on rng_stream(42, 0) == the
  // reference engine on the same stream
  {
    const int P = 100, D = 10, G = 20;
    auto engine = presets::detail::build_de_fixed<double>(0.5, 0.9);
    const evb_de_config c = evb::adapt::de_config_of(engine, P);
    report("adapt de preset: rand_1/binomial/clip/fixed(0.5, 0.9), archive 0",
           c.mutation == EVB_MUT_RAND1 && c.crossover == EVB_CX_BINOMIAL && c.repair == EVB_REP_CLIP &&
               c.parameter == EVB_PAR_FIXED && c.f == 0.5 && c.cr == 0.9 && c.archive_rate == 0.0 &&
               c.reduction == EVB_POP_FIXED);
    auto inst = problems::make_instance<double>(6, D, 1, 42);
    rng_stream rng(42, 0);
    auto pop = init_population<double>(P, D, -100.0, 100.0, rng);
    problems::eval_scratch<double> scratch;
    auto obj = [&](std::span<const double> x) { return inst.evaluate(x, scratch); };
    for (auto& m : pop) m.evaluate(obj);
    auto ge = evb::adapt::to_gpu(engine, P, D);  // before the reference engine runs (fresh state)
    evolution_state st(1LL << 40, P, D);
    for (int g = 0; g < G; ++g) engine.generation(pop, st, obj, -100.0, 100.0, rng);
    std::vector<uint64_t> words;
    rng_stream wr(42, 0);
    for (int i = 0; i < P * D + G * P * (D + 30); ++i) words.push_back(wr.next_u64());
    auto grng = evb::gpu_rng::words(words);
    auto gp = evb::adapt::to_gpu(inst);
    evb::device_vector<double> dpop(static_cast<size_t>(P) * D), dfit(static_cast<size_t>(P));
    ge.init_population(dpop.data(), D, -100.0, 100.0, grng);
    evb::gpu_scratch gs;
    evb::evaluate_batch(gp, dpop.data(), P, D, gs, dfit.data());
    for (int g = 0; g < G; ++g) ge.generation(gp, dpop.data(), D, dfit.data(), -100.0, 100.0, grng);
    auto hp = dpop.download();
    bool same = true;
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < D; ++j) same = same && hp[size_t(i) * D + j] == pop[i].genome[size_t(j)];
    report("adapt de preset engine object: 20 generations bit-exact (Ackley, rng_stream(42, 0))", same);
  }
  // `shade` preset (presets.hpp:83-94) at BASELINE config 2's shape: ttpb_1 p = 0.11 with archive,
  // midpoint_target, shade(H = 180), archive rate 1; memories carried over; one generation on the
  // reference's native stream agrees with the reference engine (F / CR via tan / log / cos: 1e-9)
  {
    const int P = 180, D = 100;
    auto engine = presets::detail::build_shade<double>(0.11, 180, 1.0, de::population_policy::fixed());
    const evb_de_config c = evb::adapt::de_config_of(engine, P);
    report("adapt shade preset: ttpb_1(0.11, archive)/binomial/midpoint_target/shade(180), rate 1",
           c.mutation == EVB_MUT_TTPB1 && c.p_best == double(0.11) && c.use_archive == 1 &&
               c.repair == EVB_REP_MIDPOINT_TARGET && c.parameter == EVB_PAR_SHADE && c.memory_size == 180 &&
               c.archive_rate == 1.0);
    auto ge = evb::adapt::to_gpu(engine, P, D);
    report("adapt shade preset: GPU archive capacity ceil(1.0 * 180)", ge.archive_capacity() == 180);
    auto inst = problems::make_instance<double>(6, D, 1, 11);
    rng_stream rng(11, 0);
    auto pop = init_population<double>(P, D, -100.0, 100.0, rng);
    problems::eval_scratch<double> scratch;
    auto obj = [&](std::span<const double> x) { return inst.evaluate(x, scratch); };
    for (auto& m : pop) m.evaluate(obj);
    engine.archive().set_capacity(engine.archive_capacity_for(P), rng);
    evolution_state st(1LL << 40, P, D);
    const int G = 3;
    for (int g = 0; g < G; ++g) engine.generation(pop, st, obj, -100.0, 100.0, rng);
    std::vector<uint64_t> words;
    rng_stream wr(11, 0);
    for (int i = 0; i < P * D + G * P * (D + 60); ++i) words.push_back(wr.next_u64());
    auto grng = evb::gpu_rng::words(words);
    auto gp = evb::adapt::to_gpu(inst);
    evb::device_vector<double> dpop(static_cast<size_t>(P) * D), dfit(static_cast<size_t>(P));
    ge.init_population(dpop.data(), D, -100.0, 100.0, grng);
    evb::gpu_scratch gs;
    evb::evaluate_batch(gp, dpop.data(), P, D, gs, dfit.data());
    for (int g = 0; g < G; ++g) ge.generation(gp, dpop.data(), D, dfit.data(), -100.0, 100.0, grng);
    auto hp = dpop.download();
    double worst = 0.0;
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < D; ++j)
        worst = std::max(worst, std::abs(hp[size_t(i) * D + j] - pop[i].genome[size_t(j)]) /
                                    std::max(1.0, std::abs(pop[i].genome[size_t(j)])));
    report("adapt shade preset engine object: 3 generations on rng_stream(11, 0) within 1e-9", worst <= 1e-9,
           "max rel " + std::to_string(worst));
    // the adaptation state of a running engine moves with it
    auto moved = evb::adapt::to_gpu(engine, P, D);
    std::vector<double> arch, mf, mc;
    int asz = 0, wi = 0;
    moved.get_state(arch, asz, mf, mc, wi, 180);
    const auto& sp = dynamic_cast<const de::shade_parameter<double>&>(engine.parameter());
    bool state_ok = asz == engine.archive().size() && wi == sp.write_index() && mf == sp.memory_f() &&
                    mc == sp.memory_cr();
    for (int k = 0; state_ok && k < asz; ++k)
      state_ok = std::equal(engine.archive().member(k).begin(), engine.archive().member(k).end(),
                            arch.begin() + size_t(k) * D);
    report("adapt shade engine mid-run: archive, memories and write index carried over", state_ok);
  }
  // `jade` preset (presets.hpp:71-81): the private learning rate is recovered exactly, and the
  // adapter is left in its initial state
  {
    auto engine = presets::detail::build_jade<double>(0.05, 0.1, 1.0);
    const evb_de_config c = evb::adapt::de_config_of(engine, 50);
    const auto& jp = dynamic_cast<const de::jade_parameter<double>&>(engine.parameter());
    report("adapt jade preset: learning rate 0.1 recovered exactly, mu restored",
           c.parameter == EVB_PAR_JADE && c.jade_c == 0.1 && jp.mu_f() == 0.5 && jp.mu_cr() == 0.5 &&
               c.mutation == EVB_MUT_TTPB1 && c.p_best == 0.05 && c.use_archive == 1);
    auto ef = presets::detail::build_jade<float>(0.05, 0.2, 0.0);
    const evb_de_config cf = evb::adapt::de_config_of(ef, 50);
    report("adapt jade preset (float): learning rate float(0.2)", cf.jade_c == double(0.2f) && cf.use_archive == 0);
  }
  // L-SHADE (shade + linear_reduction): the policy maps; an N_init that is not the population size
  // is refused with evobench::config_error
  {
    auto engine = presets::detail::build_shade<double>(0.11, 6, 1.0, de::population_policy::linear_reduction(60, 4));
    const evb_de_config c = evb::adapt::de_config_of(engine, 60);
    report("adapt lshade: linear_reduction(60, 4)", c.reduction == EVB_POP_LINEAR_REDUCTION && c.n_min == 4);
    bool threw = false;
    try {
      evb::adapt::de_config_of(engine, 50);
    } catch (const evobench::config_error&) {
      threw = true;
    }
    report("adapt lshade: N_init != pop size -> evobench::config_error", threw);
  }
  // unknown strategies (no GPU kernel) and impostors of a known name -> evobench::config_error
  {
    struct my_mutation final : de::mutation_strategy<double> {
      explicit my_mutation(std::string_view n) : n_(n) {}
      std::string_view name() const override { return n_; }
      int min_pop_size() const override { return 4; }
      void mutate(const population<double>&, const de::de_archive<double>&, std::span<const int>, int, double,
                  rng_stream&, std::vector<double>&) const override {}
      std::string_view n_;
    };
    for (std::string_view name : {std::string_view("my_mutation"), std::string_view("rand_1")}) {
      auto engine = de::de_builder<double>()
                        .mutation(std::make_unique<my_mutation>(name))
                        .crossover(std::make_unique<de::binomial_crossover<double>>())
                        .repair(std::make_unique<de::clip_repair<double>>())
                        .parameter(std::make_unique<de::fixed_parameter<double>>(0.5, 0.9))
                        .population(de::population_policy::fixed())
                        .archive_rate(0.0)
                        .build();
      bool threw = false;
      try {
        evb::adapt::to_gpu(engine, 20, 5);
      } catch (const evobench::config_error&) {
        threw = true;
      }
      report("adapt de: mutation '" + std::string(name) + "' without its GPU kernel -> evobench::config_error", threw);
    }
    // a GPU-side configuration error surfaces as the reference's type too (rand_1 needs pop >= 4)
    bool threw = false;
    try {
      auto engine = presets::detail::build_de_fixed<double>(0.5, 0.9);
      evb::adapt::to_gpu(engine, 3, 5);
    } catch (const evobench::config_error&) {
      threw = true;
    }
    report("adapt de: pop 3 for rand_1 -> evobench::config_error from the GPU engine", threw);
  }
  // PSO presets (presets.hpp:96-117): gbest + standard and lbest_ring + spherical by name, swarm
  // params copied; personal bests of a prepared engine carried over
  {
    auto pso = presets::detail::build_pso<double>(false, 0.7298, 1.49618, 1.49618, 1.2);
    const evb_pso_config c = evb::adapt::pso_config_of(pso, 40.0);
    report("adapt pso preset: gbest/standard, w c1 c2, vmax 40",
           c.topology == EVB_TOPO_GBEST && c.update == EVB_UPD_STANDARD && c.inertia == 0.7298 &&
               c.cognitive == 1.49618 && c.social == 1.49618 && c.vmax == 40.0);
    auto sp = presets::detail::build_pso<float>(true, 0.7, 1.5, 1.5, 1.3);
    const evb_pso_config cs = evb::adapt::pso_config_of(sp);
    report("adapt spso2011 preset: lbest_ring/spherical, attraction",
           cs.topology == EVB_TOPO_LBEST_RING && cs.update == EVB_UPD_SPHERICAL && cs.attraction == double(1.3f));
    const int P = 16, D = 6;
    auto inst = problems::make_instance<double>(1, D, 1, 3);
    rng_stream rng(3, 0);
    auto pop = init_population<double>(P, D, -100.0, 100.0, rng);
    problems::eval_scratch<double> scratch;
    for (auto& m : pop) m.evaluate([&](std::span<const double> x) { return inst.evaluate(x, scratch); });
    pso.prepare(pop);
    auto gpso = evb::adapt::to_gpu(pso, P, D, 40.0);
    std::vector<double> pb(static_cast<size_t>(P) * D), pf(static_cast<size_t>(P));
    evb::check(evb_pso_get(gpso.handle(), pb.data(), pf.data(), nullptr, nullptr), "pso_get");
    bool same = true;
    for (int i = 0; i < P; ++i) {
      same = same && pf[size_t(i)] == pso.personal_bests()[size_t(i)].fitness;
      for (int j = 0; j < D; ++j) same = same && pb[size_t(i) * D + j] == pso.personal_bests()[size_t(i)].genome[size_t(j)];
    }
    report("adapt pso: prepared personal bests carried over", same);
  }
  // evaluate_batch through the scratch's page-locked staging: reused and regrown across calls of
  // different sizes, identical to the reference's evaluate_batch
  {
    auto p = problems::make_instance<double>(2, 50, 1, 5);
    auto gp = evb::adapt::to_gpu(p);
    evb::gpu_scratch gs;
    bool ok = true;
    for (int n : {7, 300, 40, 1000, 1}) {
      rng_stream rng(500, uint64_t(n));
      std::vector<std::vector<double>> xs(size_t(n), std::vector<double>(50));
      for (auto& x : xs)
        for (auto& v : x) v = rng.uniform(-100.0, 100.0);
      std::vector<double> ref, got;
      problems::eval_scratch<double> rs;
      problems::evaluate_batch(p, xs, rs, ref);
      evb::evaluate_batch(gp, xs, gs, got);
      ok = ok && got.size() == size_t(n) && max_rel(got, ref) <= 1e-10;
    }
    report("evaluate_batch staging reused across batch sizes 7/300/40/1000/1", ok);
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
