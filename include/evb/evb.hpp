// evb.hpp — header-only C++17 host side over the C ABI (include/evb.h), mirroring the reference's
// module interfaces so C++ callers of evobench can switch the hot path to the GPU:
//
//   evobench (reference)                               here
//   problems::problem_instance<T>  instance.hpp:180    evb::gpu_problem<T>     (immutable, device)
//   problems::eval_scratch<T>      instance.hpp:45     evb::gpu_scratch        (per task)
//   problems::evaluate_batch(p, xs, scratch, out)      evb::evaluate_batch(p, xs, scratch, out)
//                                  batch.hpp:243-278
//   problems::batched_evaluate(p, xs) batch.hpp:281    evb::batched_evaluate(p, xs)
//   rng_stream                     core/rng.hpp:37     evb::gpu_rng (Philox / oracle word list)
//   de::de_engine<T>               de/engine.hpp:68    evb::gpu_de_engine<T>
//   pso::pso_engine<T>             pso/engine.hpp:33   evb::gpu_pso_engine<T>  (synchronous)
//   pso::cso_optimizer<T>          pso/cso.hpp:19      evb::gpu_cso<T>         (exact generation)
//   experiment::best_so_far_record recorder.hpp:35     evb::gpu_recorder<T>    (device, same CSV)
//   experiment::evo_bench(alg, su, obs, opt)           evb::evo_bench_de / _pso / _cso
//                                  runner.hpp:101      (all tasks of a suite; DE presets in one launch)
//
// Errors are rethrown as the reference's types: std::invalid_argument (dimension mismatch),
// evb::config_error, std::logic_error, std::runtime_error.  evb::config_error IS
// evobench::config_error (common.hpp:12-15) when the evobench headers are in the build
// (EVB_WITH_EVOBENCH, set by evb/evobench_adapter.hpp), so a reference caller's
// `catch (const evobench::config_error&)` sees GPU configuration errors; otherwise it is a
// std::runtime_error of the same shape.  No CUDA header is needed by users of this file.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "evb.h"

#ifdef EVB_WITH_EVOBENCH
#include "evobench/common.hpp"
namespace evb {
using config_error = ::evobench::config_error;
}  // namespace evb
#else
namespace evb {
class config_error : public std::runtime_error {
 public:
  explicit config_error(const std::string& what) : std::runtime_error(what) {}
};
}  // namespace evb
#endif

namespace evb {

inline void check(int status, const char* what) {
  if (status == EVB_OK) return;
  const std::string msg = std::string(what) + ": " + evb_last_error();
  switch (status) {
    case EVB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case EVB_ERR_CONFIG: throw config_error(msg);
    case EVB_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

template <typename T>
constexpr int dtype_of() {
  static_assert(std::is_same<T, double>::value || std::is_same<T, float>::value, "T must be float or double");
  return std::is_same<T, double>::value ? EVB_F64 : EVB_F32;
}

// Same order as evobench::problems::base_kind (problems/functions.hpp:15-26).
enum class base_kind : int {
  sphere = EVB_SPHERE,
  elliptic = EVB_ELLIPTIC,
  bent_cigar = EVB_BENT_CIGAR,
  discus = EVB_DISCUS,
  rosenbrock = EVB_ROSENBROCK,
  rastrigin = EVB_RASTRIGIN,
  ackley = EVB_ACKLEY,
  griewank = EVB_GRIEWANK,
  schwefel_12 = EVB_SCHWEFEL_12,
  expanded_schaffer_f6 = EVB_EXPANDED_SCHAFFER_F6
};

// Owning device buffer of T.
template <typename T>
class device_vector {
 public:
  device_vector() = default;
  explicit device_vector(size_t n) : n_(n) { check(evb_device_alloc(n * sizeof(T), &p_), "device_alloc"); }
  explicit device_vector(const std::vector<T>& h) : device_vector(h.size()) { upload(h); }
  device_vector(const device_vector&) = delete;
  device_vector& operator=(const device_vector&) = delete;
  device_vector(device_vector&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  device_vector& operator=(device_vector&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  ~device_vector() {
    if (p_) evb_device_free(p_);
  }
  T* data() { return static_cast<T*>(p_); }
  const T* data() const { return static_cast<const T*>(p_); }
  size_t size() const { return n_; }
  void upload(const std::vector<T>& h) {
    if (h.size() != n_) throw std::invalid_argument("device_vector: size mismatch");
    check(evb_copy_to_device(p_, h.data(), n_ * sizeof(T)), "copy_to_device");
  }
  std::vector<T> download() const {
    std::vector<T> h(n_);
    check(evb_copy_to_host(h.data(), p_, n_ * sizeof(T)), "copy_to_host");
    return h;
  }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

class gpu_scratch {
 public:
  gpu_scratch() { check(evb_scratch_create(&h_), "scratch_create"); }
  gpu_scratch(const gpu_scratch&) = delete;
  gpu_scratch& operator=(const gpu_scratch&) = delete;
  ~gpu_scratch() {
    if (h_) evb_scratch_destroy(h_);
  }
  evb_scratch handle() const { return h_; }
  // page-locked staging owned by the scratch (reused across calls, grown on demand)
  void* host_staging(size_t bytes) {
    void* p = nullptr;
    check(evb_scratch_host_staging(h_, bytes, &p), "scratch_host_staging");
    return p;
  }

 private:
  evb_scratch h_ = nullptr;
};

template <typename T>
class gpu_problem {
 public:
  // shifted-rotated base problem (problems/instance.hpp:185-196, 221-228)
  static gpu_problem base(base_kind kind, const std::vector<T>& shift, const std::vector<T>& rotation, T bias) {
    const int d = int(shift.size());
    if (rotation.size() != size_t(d) * d) throw config_error("gpu_problem: rotation must be dim x dim");
    evb_problem h = nullptr;
    check(evb_problem_create_base(dtype_of<T>(), d, int(kind), shift.data(), rotation.data(), double(bias), &h),
          "problem_create_base");
    return gpu_problem(h, d, int(kind), double(bias));
  }
  // hybrid (problems/instance.hpp:97-112): permutation, per-chunk kinds and sizes
  static gpu_problem hybrid(const std::vector<T>& shift, const std::vector<T>& rotation, T bias,
                            const std::vector<int>& sub_kinds, const std::vector<int>& chunk_sizes,
                            const std::vector<int>& permutation) {
    evb_problem h = nullptr;
    check(evb_problem_create_hybrid(dtype_of<T>(), int(shift.size()), shift.data(), rotation.data(), double(bias),
                                    int(sub_kinds.size()), sub_kinds.data(), chunk_sizes.data(), permutation.data(),
                                    &h),
          "problem_create_hybrid");
    return gpu_problem(h, int(shift.size()), -1, double(bias));
  }
  // composition (problems/instance.hpp:116-174): shifts n_comp x dim, rotations n_comp x dim x dim
  static gpu_problem composition(int dim, const std::vector<int>& kinds, const std::vector<T>& shifts,
                                 const std::vector<T>& rotations, const std::vector<double>& sigma,
                                 const std::vector<double>& lambda, const std::vector<double>& comp_bias, T bias) {
    evb_problem h = nullptr;
    check(evb_problem_create_composition(dtype_of<T>(), dim, int(kinds.size()), kinds.data(), shifts.data(),
                                         rotations.data(), sigma.data(), lambda.data(), comp_bias.data(), double(bias),
                                         &h),
          "problem_create_composition");
    return gpu_problem(h, dim, -1, double(bias));
  }

  gpu_problem(const gpu_problem&) = delete;
  gpu_problem& operator=(const gpu_problem&) = delete;
  gpu_problem(gpu_problem&& o) noexcept : h_(std::exchange(o.h_, nullptr)), dim_(o.dim_), kind_(o.kind_), bias_(o.bias_) {}
  ~gpu_problem() {
    if (h_) evb_problem_destroy(h_);
  }
  int dim() const { return dim_; }
  evb_problem handle() const { return h_; }

 private:
  gpu_problem(evb_problem h, int dim, int kind, double bias) : h_(h), dim_(dim), kind_(kind), bias_(bias) {}
  evb_problem h_ = nullptr;
  int dim_ = 0;
  int kind_ = -1;
  double bias_ = 0.0;
};

// problems::evaluate_batch(problem, xs, scratch, out) (problems/batch.hpp:243-278): host points in,
// host values out; throws std::invalid_argument on a dimension mismatch, like the reference.
// The rows are flattened into the scratch's page-locked staging (reused across calls), so the
// batch crosses the host link at full bandwidth and the kernel writes the values straight into
// the staging's tail.
template <typename T>
void evaluate_batch(const gpu_problem<T>& problem, const std::vector<std::vector<T>>& xs, gpu_scratch& scratch,
                    std::vector<T>& out) {
  out.clear();
  if (xs.empty()) return;
  const int d = problem.dim();
  for (const auto& x : xs)
    if (int(x.size()) != d) throw std::invalid_argument("evaluate_batch: point dimension mismatch");
  const size_t n = xs.size();
  const size_t x_bytes = (n * size_t(d) * sizeof(T) + 255) / 256 * 256;
  uint8_t* stage = static_cast<uint8_t*>(scratch.host_staging(x_bytes + n * sizeof(T)));
  T* flat = reinterpret_cast<T*>(stage);
  T* vals = reinterpret_cast<T*>(stage + x_bytes);
  for (size_t b = 0; b < n; ++b) std::memcpy(flat + b * d, xs[b].data(), sizeof(T) * d);
  check(evb_evaluate_batch_host(problem.handle(), scratch.handle(), flat, int64_t(n), d, vals), "evaluate_batch");
  out.assign(vals, vals + n);
}

// problems::batched_evaluate(problem, xs) (problems/batch.hpp:281-288)
template <typename T>
std::vector<T> batched_evaluate(const gpu_problem<T>& problem, const std::vector<std::vector<T>>& xs) {
  gpu_scratch scratch;
  std::vector<T> out;
  evaluate_batch(problem, xs, scratch, out);
  return out;
}

// device-resident form: X (n x ldx) and out (n) are device pointers
template <typename T>
void evaluate_batch(const gpu_problem<T>& problem, const T* X, int64_t n, int64_t ldx, gpu_scratch& scratch, T* out,
                    void* stream = nullptr) {
  check(evb_evaluate_batch(problem.handle(), scratch.handle(), X, n, ldx, out, stream), "evaluate_batch");
}

class gpu_rng {
 public:
  static gpu_rng philox(uint64_t key) {
    evb_rng h = nullptr;
    check(evb_rng_create_philox(key, &h), "rng_create_philox");
    return gpu_rng(h);
  }
  // oracle mode: the reference's own words, consumed in its order (e.g. rng_stream(42, 0))
  static gpu_rng words(const std::vector<uint64_t>& w) {
    evb_rng h = nullptr;
    check(evb_rng_create_words(w.data(), int64_t(w.size()), &h), "rng_create_words");
    return gpu_rng(h);
  }
  gpu_rng(gpu_rng&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  gpu_rng(const gpu_rng&) = delete;
  ~gpu_rng() {
    if (h_) evb_rng_destroy(h_);
  }
  evb_rng handle() const { return h_; }
  int64_t cursor() const {
    int64_t c = 0;
    check(evb_rng_state(h_, &c, nullptr, nullptr), "rng_state");
    return c;
  }

 private:
  explicit gpu_rng(evb_rng h) : h_(h) {}
  evb_rng h_ = nullptr;
};

// presets.hpp:59-94 as evb_de_config values
inline evb_de_config de_preset_fixed(double f = 0.5, double cr = 0.9) {
  evb_de_config c{};
  c.mutation = EVB_MUT_RAND1;
  c.crossover = EVB_CX_BINOMIAL;
  c.repair = EVB_REP_CLIP;
  c.parameter = EVB_PAR_FIXED;
  c.f = f;
  c.cr = cr;
  return c;
}
inline evb_de_config de_preset_shade(double p, int memory_size, double archive_rate) {
  evb_de_config c{};
  c.mutation = EVB_MUT_TTPB1;
  c.crossover = EVB_CX_BINOMIAL;
  c.repair = EVB_REP_MIDPOINT_TARGET;
  c.parameter = EVB_PAR_SHADE;
  c.p_best = p;
  c.use_archive = archive_rate > 0 ? 1 : 0;
  c.memory_size = memory_size;
  c.archive_rate = archive_rate;
  return c;
}

// de::de_engine<T> on the GPU: the population is a device matrix (pop_size x ldp) + fitness.
template <typename T>
class gpu_de_engine {
 public:
  gpu_de_engine(const evb_de_config& cfg, int pop_size, int dim) : P_(pop_size), D_(dim) {
    check(evb_de_create(dtype_of<T>(), &cfg, pop_size, dim, &h_), "de_create");
  }
  gpu_de_engine(const gpu_de_engine&) = delete;
  gpu_de_engine& operator=(const gpu_de_engine&) = delete;
  gpu_de_engine(gpu_de_engine&& o) noexcept : h_(std::exchange(o.h_, nullptr)), P_(o.P_), D_(o.D_) {}
  ~gpu_de_engine() {
    if (h_) evb_de_destroy(h_);
  }
  void init_population(T* pop, int64_t ldp, T lb, T ub, gpu_rng& rng, void* stream = nullptr) {
    check(evb_de_init_population(h_, pop, ldp, double(lb), double(ub), rng.handle(), stream), "de_init_population");
  }
  // de_engine::generation(pop, st, objective, lb, ub, rng) (de/engine.hpp:71-102)
  void generation(const gpu_problem<T>& objective, T* pop, int64_t ldp, T* fitness, T lb, T ub, gpu_rng& rng,
                  void* stream = nullptr) {
    check(evb_de_generation(h_, objective.handle(), nullptr, pop, ldp, fitness, double(lb), double(ub), rng.handle(),
                            stream),
          "de_generation");
  }
  // de_engine::optimize (de/engine.hpp:107-133); returns the best index, its fitness in *best
  int optimize(const gpu_problem<T>& objective, T* pop, int64_t ldp, T* fitness, T lb, T ub, long long max_fes,
               gpu_rng& rng, double* best = nullptr, void* stream = nullptr) {
    int bi = 0, gens = 0;
    double bf = 0;
    check(evb_de_optimize(h_, objective.handle(), nullptr, pop, ldp, fitness, double(lb), double(ub), max_fes,
                          rng.handle(), &bi, &bf, &gens, stream),
          "de_optimize");
    if (best) *best = bf;
    return bi;
  }
  int archive_capacity() const { return evb_de_archive_capacity(h_); }
  int pop_size() const { return P_; }
  int dim() const { return D_; }
  // adaptation + archive state (SHADE memories / JADE means in memory_f[0], memory_cr[0])
  void set_state(const std::vector<T>& archive_rows, int archive_size, const std::vector<T>& memory_f,
                 const std::vector<T>& memory_cr, int write_index) {
    check(evb_de_set_state(h_, archive_rows.empty() ? nullptr : archive_rows.data(), archive_size,
                           memory_f.empty() ? nullptr : memory_f.data(), memory_cr.empty() ? nullptr : memory_cr.data(),
                           write_index),
          "de_set_state");
  }
  void get_state(std::vector<T>& archive_rows, int& archive_size, std::vector<T>& memory_f, std::vector<T>& memory_cr,
                 int& write_index, int memory_size) const {
    archive_rows.assign(size_t(std::max(1, archive_capacity())) * D_, T(0));
    memory_f.assign(size_t(std::max(1, memory_size)), T(0));
    memory_cr.assign(size_t(std::max(1, memory_size)), T(0));
    check(evb_de_get_state(h_, archive_rows.data(), &archive_size, memory_f.data(), memory_cr.data(), &write_index),
          "de_get_state");
    archive_rows.resize(size_t(archive_size) * D_);
  }
  evb_de handle() const { return h_; }

 private:
  evb_de h_ = nullptr;
  int P_, D_;
};

// synchronous pso
template <typename T>
class gpu_pso_engine {
 public:
  gpu_pso_engine(const evb_pso_config& cfg, int pop_size, int dim) {
    check(evb_pso_create(dtype_of<T>(), &cfg, pop_size, dim, &h_), "pso_create");
  }
  gpu_pso_engine(const gpu_pso_engine&) = delete;
  gpu_pso_engine& operator=(const gpu_pso_engine&) = delete;
  gpu_pso_engine(gpu_pso_engine&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  ~gpu_pso_engine() {
    if (h_) evb_pso_destroy(h_);
  }
  void prepare(const T* X, int64_t ldx, const T* fitness, void* stream = nullptr) {
    check(evb_pso_prepare(h_, X, ldx, fitness, stream), "pso_prepare");
  }
  void generation(const gpu_problem<T>& objective, T* X, int64_t ldx, T* V, int64_t ldv, T* fitness, T lb, T ub,
                  gpu_rng& rng, void* stream = nullptr) {
    check(evb_pso_generation(h_, objective.handle(), nullptr, X, ldx, V, ldv, fitness, double(lb), double(ub),
                             rng.handle(), stream),
          "pso_generation");
  }
  // personal bests from the host (pop_size x dim row-major + fitness); marks the engine prepared
  void set_personal_bests(const std::vector<T>& pbest_rows, const std::vector<T>& pbest_fitness) {
    check(evb_pso_set_pbest(h_, pbest_rows.data(), pbest_fitness.data()), "pso_set_pbest");
  }
  evb_pso handle() const { return h_; }

 private:
  evb_pso h_ = nullptr;
};

// experiment::best_so_far_record<T> on the device: engines report their evaluations in FE order;
// grid() / to_csv() give the reference's checkpoint grid and CSV (recorder.hpp:35-155).
template <typename T>
class gpu_recorder {
 public:
  gpu_recorder(int n_runs, long long max_fes, long long interval) : runs_(n_runs) {
    check(evb_recorder_create(dtype_of<T>(), n_runs, max_fes, interval, &h_), "recorder_create");
  }
  gpu_recorder(const gpu_recorder&) = delete;
  ~gpu_recorder() {
    if (h_) evb_recorder_destroy(h_);
  }
  evb_recorder handle() const { return h_; }
  int checkpoint_count() const { return evb_recorder_checkpoints(h_); }
  // on_evaluate for n device values of run `run`, in order
  void observe(int run, const T* values, int64_t n, void* stream = nullptr) {
    check(evb_recorder_observe(h_, run, values, n, stream), "recorder_observe");
  }
  void finish(void* stream = nullptr) { check(evb_recorder_finish(h_, 0, runs_, stream), "recorder_finish"); }
  std::vector<T> grid() const {  // runs x checkpoints
    std::vector<T> g(size_t(runs_) * checkpoint_count());
    check(evb_recorder_grid(h_, g.data(), nullptr), "recorder_grid");
    return g;
  }
  std::string to_csv(const std::string& suite_name, int dim, const std::vector<int>& problem_ids, int instances,
                     int runs) const {
    int64_t n = 0;
    check(evb_recorder_csv(h_, suite_name.c_str(), dim, int(problem_ids.size()), problem_ids.data(), instances, runs,
                           nullptr, 0, &n),
          "recorder_csv");
    std::string out(size_t(n), '\0');
    check(evb_recorder_csv(h_, suite_name.c_str(), dim, int(problem_ids.size()), problem_ids.data(), instances, runs,
                           out.data(), n, &n),
          "recorder_csv");
    return out;
  }

 private:
  evb_recorder h_ = nullptr;
  int runs_;
};

// pso::cso_optimizer<T>(phi): the device generation is the reference's generation
template <typename T>
class gpu_cso {
 public:
  gpu_cso(double phi, int pop_size, int dim) { check(evb_cso_create(dtype_of<T>(), phi, pop_size, dim, &h_), "cso_create"); }
  gpu_cso(const gpu_cso&) = delete;
  ~gpu_cso() {
    if (h_) evb_cso_destroy(h_);
  }
  void generation(const gpu_problem<T>& objective, T* X, int64_t ldx, T* V, int64_t ldv, T* fitness, T lb, T ub,
                  gpu_rng& rng, void* stream = nullptr) {
    check(evb_cso_generation(h_, objective.handle(), nullptr, X, ldx, V, ldv, fitness, double(lb), double(ub),
                             rng.handle(), stream),
          "cso_generation");
  }
  double optimize(const gpu_problem<T>& objective, T* X, int64_t ldx, T* V, int64_t ldv, T* fitness, T lb, T ub,
                  long long max_fes, gpu_rng& rng, void* stream = nullptr) {
    int bi = 0, g = 0;
    double bf = 0;
    check(evb_cso_optimize(h_, objective.handle(), nullptr, X, ldx, V, ldv, fitness, double(lb), double(ub), max_fes,
                           rng.handle(), &bi, &bf, &g, stream),
          "cso_optimize");
    return bf;
  }

 private:
  evb_cso h_ = nullptr;
};

// experiment::evo_bench over a suite (instances[p * instance_count + i] = suite.at(p, i)) with a
// recorder (may be null); returns each task's best fitness (task ((p * I) + i) * runs + r)
template <typename T>
std::vector<double> evo_bench_de(const evb_de_config& cfg, int pop_size, const std::vector<const gpu_problem<T>*>& instances,
                                 int problem_count, int runs, long long max_fes, uint64_t seed, T lb, T ub,
                                 gpu_recorder<T>* rec = nullptr) {
  std::vector<evb_problem> h;
  for (const auto* p : instances) h.push_back(p->handle());
  const int instance_count = int(h.size()) / problem_count;
  std::vector<double> best(h.size() * size_t(runs));
  int path = 0;
  check(evb_evo_bench_de(dtype_of<T>(), &cfg, pop_size, instances.front()->dim(), h.data(), problem_count,
                         instance_count, runs, max_fes, seed, double(lb), double(ub), rec ? rec->handle() : nullptr,
                         nullptr, best.data(), 0, &path, nullptr),
        "evo_bench_de");
  return best;
}

template <typename T>
std::vector<double> evo_bench_cso(double phi, int pop_size, const std::vector<const gpu_problem<T>*>& instances,
                                  int problem_count, int runs, long long max_fes, uint64_t seed, T lb, T ub,
                                  gpu_recorder<T>* rec = nullptr) {
  std::vector<evb_problem> h;
  for (const auto* p : instances) h.push_back(p->handle());
  const int instance_count = int(h.size()) / problem_count;
  std::vector<double> best(h.size() * size_t(runs));
  check(evb_evo_bench_cso(dtype_of<T>(), phi, pop_size, instances.front()->dim(), h.data(), problem_count,
                          instance_count, runs, max_fes, seed, double(lb), double(ub), rec ? rec->handle() : nullptr,
                          best.data(), nullptr),
        "evo_bench_cso");
  return best;
}

}  // namespace evb
