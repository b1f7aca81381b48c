// evobench_adapter.hpp — the binding an evobench maintainer adds to route the hot path to the GPU.
// Requires the evobench headers on the include path (it is compiled against the UNMODIFIED
// reference in tests/cpp/test_adapter.cpp); everything GPU-side goes through include/evb/evb.hpp.
//
//   auto gp = evb::adapt::to_gpu(instance);              // problems::problem_instance<T> -> device
//   evb::evaluate_batch(gp, xs, gpu_scratch, out);       // same call shape as evaluate_batch
//
// run_handle<T>::evaluate_batch (experiment/runner.hpp:47-53) can call the GPU form and keep its
// FE counting / observer notification unchanged.
#pragma once

#include <variant>
#include <vector>

#include "evb/evb.hpp"
#include "evobench/problems/instance.hpp"

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

}  // namespace evb::adapt
