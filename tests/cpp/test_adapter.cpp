// C++ parity test through the C++ host side (include/evb/evb.hpp + evobench_adapter.hpp) against
// the UNMODIFIED reference (compiled in from /root/reference by __graft_entry__.build()).
// Reads like the reference's own acceptance tests: PASS / FAIL lines, exit code = failures.
#include <cmath>
#include <cstdio>
#include <span>
#include <string>
#include <vector>

#include "evb/evb.hpp"
#include "evb/evobench_adapter.hpp"
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
  std::printf("%d failure(s)\n", failures);
  return failures;
}
