// refshape_bench.cpp — times the reference-shaped C++ binding end to end (bench.py's
// e2e.reference_shape): run_handle<T>::evaluate_batch (experiment/runner.hpp:47-53) forwarding to
// problems::evaluate_batch(problem, const vector<vector<T>>& xs, scratch, out)
// (problems/batch.hpp:243-278), here evb::evaluate_batch from include/evb/evb.hpp: the caller's
// heap rows are flattened into the scratch's page-locked staging, cross the host link, and the
// fitness values come back into a std::vector — everything a reference caller pays, per call.
// Built as libevb_refshape.so beside libevb.so; plain C++ over the C ABI (no CUDA headers).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <vector>

#include "evb/evb.hpp"

extern "C" __attribute__((visibility("default"))) int evb_refshape_time(int n_kinds, const int* kinds, int dim,
                                                                        int n_points, const double* shift,
                                                                        const double* rotation, const double* X,
                                                                        int steps, int blocks, double warm_s,
                                                                        double* us_per_step, double* values);

// One step = one evaluate_batch call per kind over the same n_points rows (three run_handle
// calls at config 1).  Warm-up for at least warm_s seconds, then `blocks` blocks of steps/blocks
// steps; us_per_step[b] = wall-clock microseconds per step of block b; values (n_kinds x n_points)
// receive the last step's fitness.  Returns 0, or -1 with nothing written on any error.
int evb_refshape_time(int n_kinds, const int* kinds, int dim, int n_points, const double* shift,
                      const double* rotation, const double* X, int steps, int blocks, double warm_s,
                      double* us_per_step, double* values) {
  try {
    const std::vector<double> o(shift, shift + dim), m(rotation, rotation + size_t(dim) * dim);
    std::vector<evb::gpu_problem<double>> probs;
    for (int k = 0; k < n_kinds; ++k) probs.push_back(evb::gpu_problem<double>::base(evb::base_kind(kinds[k]), o, m, 0.0));
    std::vector<std::vector<double>> xs(static_cast<size_t>(n_points));
    for (int b = 0; b < n_points; ++b) xs[size_t(b)].assign(X + size_t(b) * dim, X + size_t(b + 1) * dim);
    evb::gpu_scratch scratch;
    std::vector<std::vector<double>> out(static_cast<size_t>(n_kinds));
    auto step = [&] {
      for (int k = 0; k < n_kinds; ++k) evb::evaluate_batch(probs[size_t(k)], xs, scratch, out[size_t(k)]);
    };
    using clk = std::chrono::steady_clock;
    const auto t_w = clk::now();
    int n_w = 0;
    while (n_w < 3 || std::chrono::duration<double>(clk::now() - t_w).count() < warm_s) {
      step();
      ++n_w;
    }
    const int per = std::max(1, steps / std::max(1, blocks));
    for (int b = 0; b < blocks; ++b) {
      const auto t0 = clk::now();
      for (int s = 0; s < per; ++s) step();
      us_per_step[b] = std::chrono::duration<double, std::micro>(clk::now() - t0).count() / per;
    }
    for (int k = 0; k < n_kinds; ++k) std::copy(out[size_t(k)].begin(), out[size_t(k)].end(), values + size_t(k) * n_points);
    return 0;
  } catch (...) {
    return -1;
  }
}

// BASELINE config 0 as the reference's caller runs it: the population and fitness live in host
// memory (de_engine's state), one DE generation per call (de_engine::generation), here
// evb_de_generations_host(…, 1) — one copy in, the persistent cluster kernel, one copy out.
// preset `de` (rand/1/bin, F 0.5, CR 0.9, clip), Rastrigin on the given (pre-scaled) rotation.
extern "C" __attribute__((visibility("default"))) int evb_refshape_time_de(int dim, int pop_size, const double* shift,
                                                                           const double* rotation, double* pop,
                                                                           double* fit, uint64_t key, int steps,
                                                                           int blocks, double warm_s,
                                                                           double* us_per_step);

int evb_refshape_time_de(int dim, int pop_size, const double* shift, const double* rotation, double* pop, double* fit,
                         uint64_t key, int steps, int blocks, double warm_s, double* us_per_step) {
  evb_problem prob = nullptr;
  evb_de eng = nullptr;
  evb_rng rng = nullptr;
  int rc = evb_problem_create_base(EVB_F64, dim, EVB_RASTRIGIN, shift, rotation, 0.0, &prob);
  evb_de_config cfg{};
  cfg.mutation = EVB_MUT_RAND1;
  cfg.crossover = EVB_CX_BINOMIAL;
  cfg.repair = EVB_REP_CLIP;
  cfg.parameter = EVB_PAR_FIXED;
  cfg.f = 0.5;
  cfg.cr = 0.9;
  cfg.memory_size = 1;
  if (rc == EVB_OK) rc = evb_de_create(EVB_F64, &cfg, pop_size, dim, &eng);
  if (rc == EVB_OK) rc = evb_rng_create_philox(key, &rng);
  auto step = [&] { return evb_de_generations_host(eng, prob, nullptr, pop, dim, fit, -100.0, 100.0, rng, 1); };
  using clk = std::chrono::steady_clock;
  if (rc == EVB_OK) {
    const auto t_w = clk::now();
    int n_w = 0;
    while (rc == EVB_OK && (n_w < 3 || std::chrono::duration<double>(clk::now() - t_w).count() < warm_s)) {
      rc = step();
      ++n_w;
    }
  }
  const int per = std::max(1, steps / std::max(1, blocks));
  for (int b = 0; b < blocks && rc == EVB_OK; ++b) {
    const auto t0 = clk::now();
    for (int s = 0; s < per && rc == EVB_OK; ++s) rc = step();
    us_per_step[b] = std::chrono::duration<double, std::micro>(clk::now() - t0).count() / per;
  }
  if (rng) evb_rng_destroy(rng);
  if (eng) evb_de_destroy(eng);
  if (prob) evb_problem_destroy(prob);
  return rc == EVB_OK ? 0 : -1;
}
