// evo_bench.cu — the suite-level grouped launch: every (problem x instance x
// run) task of an experiment::evo_bench call (experiment/runner.hpp:101-160) for a DE preset,
// with the tasks' evaluations reported to a device best-so-far recorder, so the reference's
// CSV (experiment/recorder.hpp:103-121) comes straight from the GPU.
//
//   task index   t = ((p * instances) + i) * runs + r            (runner.hpp:112-118)
//   task stream  Philox key splitmix64(master_seed ^ t)          (the positional analogue of
//                                                                 derive_stream(seed, t), :119-120)
//   algorithm    de_engine::optimize (de/engine.hpp:107-133): init + evaluate P points, then
//                generations while fes < max_fes (a generation always evaluates all P trials)
//   recorder     run slot t; on_run_end for every task after its run (runner.hpp:121-122)
//
// Configurations the persistent batched-runs kernel supports (the `de` preset family) run as
// ONE launch over all tasks (base, hybrid and composition problems mixed); any other DE
// configuration (JADE, SHADE, archive, other strategies, fp32) runs each task through the
// per-generation engine, tasks in order.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "evb_internal.cuh"

namespace evb {
namespace {

uint64_t task_key(uint64_t master_seed, uint64_t t) {
  uint64_t z = (master_seed ^ t) + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void check_status(int rc) {
  if (rc == EVB_OK) return;
  const std::string msg = evb_last_error();
  switch (rc) {
    case EVB_ERR_INVALID_ARGUMENT: throw invalid_argument(msg);
    case EVB_ERR_CONFIG: throw config_error(msg);
    case EVB_ERR_LOGIC: throw logic_error(msg);
    default: throw runtime_error(msg);
  }
}

template <typename T>
void best_of(const std::vector<uint8_t>& fit, int P, int tasks, double* best) {
  const T* f = reinterpret_cast<const T*>(fit.data());
  for (int t = 0; t < tasks; ++t) {
    int b = 0;  // population::best (core/population.hpp:59-65): lowest fitness, ties to the lowest index
    for (int i = 1; i < P; ++i)
      if (f[size_t(t) * P + i] < f[size_t(t) * P + b]) b = i;
    best[t] = double(f[size_t(t) * P + b]);
  }
}

// validation shared by the suite entry points (runner.hpp:106-108, presets.hpp:133)
int suite_tasks(int dtype, int pop_size, int dim, const evb_problem* problems, int problem_count, int instance_count,
                int runs, int64_t max_fes, evb_recorder rec) {
  require(problems != nullptr, "evo_bench: null argument");
  require(runs >= 1, "evo_bench: independent_runs must be at least 1");
  require(max_fes >= 1, "evo_bench: max_fes must be positive");
  require(pop_size >= 4, "algorithm: pop size must be at least 4");
  require(problem_count >= 1 && instance_count >= 1, "evo_bench: empty suite");
  require(dtype == EVB_F32 || dtype == EVB_F64, "evo_bench: dtype must be EVB_F32 or EVB_F64");
  const int64_t total64 = int64_t(problem_count) * instance_count * runs;
  require(total64 <= (int64_t(1) << 24), "evo_bench: too many tasks");
  const int tasks = int(total64);
  if (rec)
    require(recorder_runs(rec) >= tasks && recorder_dtype(rec) == dtype, "evo_bench: recorder runs / dtype mismatch");
  for (int q = 0; q < problem_count * instance_count; ++q) {
    require(problems[q] != nullptr, "evo_bench: null problem");
    if (problems[q]->p.dim != dim) throw invalid_argument("evo_bench: problem dimension mismatch");
    require(problems[q]->p.dtype == dtype, "evo_bench: problem dtype mismatch");
  }
  return tasks;
}

// Task loop for the swarm optimizers: per task a fresh Philox stream, X / V / fitness buffers
// reused, run_task(t, problem, rng, X, V, fit, &best) runs one optimize().
template <typename Run>
void swarm_tasks(int dtype, int pop_size, int dim, const evb_problem* problems, int runs, int tasks,
                 uint64_t master_seed, evb_recorder rec, double* best_host, cudaStream_t st, Run&& run_task) {
  const size_t es = dtype == EVB_F64 ? 8 : 4;
  void* X = nullptr;
  void* V = nullptr;
  void* fit = nullptr;
  try {
    EVB_CUDA(cudaMalloc(&X, es * size_t(pop_size) * dim));
    EVB_CUDA(cudaMalloc(&V, es * size_t(pop_size) * dim));
    EVB_CUDA(cudaMalloc(&fit, es * size_t(pop_size)));
    for (int t = 0; t < tasks; ++t) {
      evb_rng r = nullptr;
      check_status(evb_rng_create_philox(task_key(master_seed, uint64_t(t)), &r));
      double best = 0.0;
      int rc = EVB_OK;
      try {
        rc = run_task(t, problems[t / runs], r, X, V, fit, &best);
      } catch (...) {
        evb_rng_destroy(r);
        throw;
      }
      evb_rng_destroy(r);
      check_status(rc);
      if (best_host) best_host[t] = best;
    }
    if (rec) check_status(evb_recorder_finish(rec, 0, tasks, st));
    EVB_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    cudaFree(X);
    cudaFree(V);
    cudaFree(fit);
    throw;
  }
  cudaFree(X);
  cudaFree(V);
  cudaFree(fit);
}

}  // namespace
}  // namespace evb

using namespace evb;

extern "C" {

uint64_t evb_task_key(uint64_t master_seed, uint64_t task_index) { return task_key(master_seed, task_index); }

int evb_evo_bench_de(int dtype, const evb_de_config* cfg, int pop_size, int dim, const evb_problem* problems,
                     int problem_count, int instance_count, int runs, int64_t max_fes, uint64_t master_seed,
                     double lb, double ub, evb_recorder rec, evb_param_trace ptrace, double* best_host, int flags,
                     int* path_used, void* stream) {
  return guarded([&] {
    require(cfg != nullptr, "evo_bench: null argument");
    const int tasks = suite_tasks(dtype, pop_size, dim, problems, problem_count, instance_count, runs, max_fes, rec);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int P = pop_size, D = dim;
    // optimize(): P initial evaluations, then one generation (P trials) while fes < max_fes
    const int64_t gens64 = max_fes > P ? (max_fes - P + P - 1) / P : 0;
    require(gens64 < (int64_t(1) << 31), "evo_bench: too many generations");
    const int gens = int(gens64);
    std::vector<evb_problem> task_problem(tasks);
    std::vector<uint64_t> keys(tasks);
    for (int t = 0; t < tasks; ++t) {
      task_problem[t] = problems[t / runs];
      keys[t] = task_key(master_seed, uint64_t(t));
    }
    const size_t es = dtype == EVB_F64 ? 8 : 4;
    std::vector<uint8_t> fit_host(es * size_t(tasks) * P);
    const bool force_engine = (flags & EVB_BENCH_FORCE_ENGINE) != 0;
    const bool k8 = !force_engine && runs_kernel_unsupported(dtype, cfg, P, D, task_problem.data(), tasks).empty();
    if (k8) {
      void* pops = nullptr;
      void* fits = nullptr;
      EVB_CUDA(cudaMalloc(&pops, es * size_t(tasks) * P * D));
      EVB_CUDA(cudaMalloc(&fits, es * size_t(tasks) * P));
      const int rc = evb_de_runs(dtype, cfg, tasks, P, D, task_problem.data(), keys.data(), gens, lb, ub, pops, fits,
                                 1, 0u, rec, stream);
      cudaError_t e = cudaSuccess;
      if (rc == EVB_OK) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));  // de_runs is asynchronous
      if (rc == EVB_OK && e == cudaSuccess)
        e = cudaMemcpy(fit_host.data(), fits, fit_host.size(), cudaMemcpyDeviceToHost);
      cudaFree(pops);
      cudaFree(fits);
      check_status(rc);
      EVB_CUDA(e);
    } else {
      evb_scratch sc = nullptr;
      check_status(evb_scratch_create(&sc));
      void* pop = nullptr;
      void* fit = nullptr;
      try {
        EVB_CUDA(cudaMalloc(&pop, es * size_t(P) * D));
        EVB_CUDA(cudaMalloc(&fit, es * size_t(P)));
        for (int t = 0; t < tasks; ++t) {
          evb_de e = nullptr;
          evb_rng r = nullptr;
          check_status(evb_de_create(dtype, cfg, P, D, &e));
          int rc = evb_rng_create_philox(keys[t], &r);
          if (rc == EVB_OK && rec) rc = evb_de_attach_recorder(e, rec, t);
          if (rc == EVB_OK && ptrace) rc = evb_de_attach_param_trace(e, ptrace, t);
          int bi = 0, g = 0;
          double bf = 0.0;
          if (rc == EVB_OK)
            rc = evb_de_optimize(e, task_problem[t], sc, pop, D, fit, lb, ub, max_fes, r, &bi, &bf, &g, stream);
          if (rc == EVB_OK)
            rc = cudaMemcpyAsync(fit_host.data() + es * size_t(t) * P, fit, es * P, cudaMemcpyDeviceToHost, st) ==
                         cudaSuccess
                     ? EVB_OK
                     : EVB_ERR_RUNTIME;
          evb_rng_destroy(r);
          evb_de_destroy(e);
          check_status(rc);
        }
        EVB_CUDA(cudaStreamSynchronize(st));
      } catch (...) {
        cudaFree(pop);
        cudaFree(fit);
        evb_scratch_destroy(sc);
        throw;
      }
      cudaFree(pop);
      cudaFree(fit);
      evb_scratch_destroy(sc);
    }
    if (rec) check_status(evb_recorder_finish(rec, 0, tasks, stream));  // on_run_end, every task
    EVB_CUDA(cudaStreamSynchronize(st));
    if (best_host) {
      if (dtype == EVB_F64) best_of<double>(fit_host, P, tasks, best_host);
      else best_of<float>(fit_host, P, tasks, best_host);
    }
    if (path_used) *path_used = k8 ? 1 : 2;
  });
}

int evb_evo_bench_pso(int dtype, const evb_pso_config* cfg, int pop_size, int dim, const evb_problem* problems,
                      int problem_count, int instance_count, int runs, int64_t max_fes, uint64_t master_seed,
                      double lb, double ub, evb_recorder rec, double* best_host, void* stream) {
  return guarded([&] {
    require(cfg != nullptr, "evo_bench: null argument");
    const int tasks = suite_tasks(dtype, pop_size, dim, problems, problem_count, instance_count, runs, max_fes, rec);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_pso eng = nullptr;
    check_status(evb_pso_create(dtype, cfg, pop_size, dim, &eng));
    try {
      swarm_tasks(dtype, pop_size, dim, problems, runs, tasks, master_seed, rec, best_host, st,
                  [&](int t, evb_problem p, evb_rng r, void* X, void* V, void* fit, double* best) {
                    int rc = rec ? evb_pso_attach_recorder(eng, rec, t) : EVB_OK;
                    int bi = 0, g = 0;
                    if (rc == EVB_OK)
                      rc = evb_pso_optimize(eng, p, nullptr, X, dim, V, dim, fit, lb, ub, max_fes, r, &bi, best, &g,
                                            stream);
                    return rc;
                  });
    } catch (...) {
      evb_pso_destroy(eng);
      throw;
    }
    evb_pso_destroy(eng);
  });
}

int evb_evo_bench_cso(int dtype, double phi, int pop_size, int dim, const evb_problem* problems, int problem_count,
                      int instance_count, int runs, int64_t max_fes, uint64_t master_seed, double lb, double ub,
                      evb_recorder rec, double* best_host, void* stream) {
  return guarded([&] {
    const int tasks = suite_tasks(dtype, pop_size, dim, problems, problem_count, instance_count, runs, max_fes, rec);
    require(pop_size % 2 == 0, "algorithm cso: pop size must be even");  // presets.hpp:181
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_cso eng = nullptr;
    check_status(evb_cso_create(dtype, phi, pop_size, dim, &eng));
    try {
      swarm_tasks(dtype, pop_size, dim, problems, runs, tasks, master_seed, rec, best_host, st,
                  [&](int t, evb_problem p, evb_rng r, void* X, void* V, void* fit, double* best) {
                    int rc = rec ? evb_cso_attach_recorder(eng, rec, t) : EVB_OK;
                    int bi = 0, g = 0;
                    if (rc == EVB_OK)
                      rc = evb_cso_optimize(eng, p, nullptr, X, dim, V, dim, fit, lb, ub, max_fes, r, &bi, best, &g,
                                            stream);
                    return rc;
                  });
    } catch (...) {
      evb_cso_destroy(eng);
      throw;
    }
    evb_cso_destroy(eng);
  });
}

}  // extern "C"
