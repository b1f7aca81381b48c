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
  std::printf("%d failure(s)\n", failures);
  return failures;
}
