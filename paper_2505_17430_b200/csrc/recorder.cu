// recorder.cu — the harness boundary on the device: a best-so-far recorder with
// the semantics of experiment::best_so_far_record (experiment/recorder.hpp:35-155).
//
//   on_evaluate(fes, f):  running_min = min(running_min, f) (strict <, so NaN never enters);
//                         every checkpoint k with fes >= (k+1)*interval not yet filled takes
//                         running_min                                      (recorder.hpp:65-75)
//   on_run_end:           unfilled checkpoints take the final running_min   (recorder.hpp:77-84)
//   to_csv:               suite,problem,instance,dim,run,fes,best_so_far with shortest
//                         round-trip values (std::to_chars)                (recorder.hpp:20-25, 103-121)
//
// State lives on the device (per run: running minimum, next slot, FE count), so engines append
// evaluations in FE order without a host round trip — including inside CUDA graphs and inside
// the persistent batched-runs kernel (runs.cu), which updates the same arrays.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cstring>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "evb_internal.cuh"
#include "recorder.cuh"

struct evb_recorder_s {
  int dtype = EVB_F64;
  int n_runs = 0;
  int n_ckpt = 0;
  int64_t interval = 0;
  int64_t max_fes = 0;
  void* grid = nullptr;       // n_runs x n_ckpt (T), NaN until filled
  void* running = nullptr;    // n_runs (T), +inf initially
  int* next_slot = nullptr;   // n_runs
  int64_t* fes = nullptr;     // n_runs (last FE count)
};

namespace evb {
namespace {

template <typename T>
__global__ void rec_init_kernel(T* grid, T* running, int* next, int64_t* fes, int n_runs, int n_ckpt) {
  const int64_t n = int64_t(n_runs) * n_ckpt;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    grid[e] = std::numeric_limits<T>::quiet_NaN();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_runs; r += gridDim.x * blockDim.x) {
    running[r] = std::numeric_limits<T>::infinity();
    next[r] = 0;
    fes[r] = 0;
  }
}

template <typename T>
__global__ void rec_observe_kernel(rec_view<T> v, int run, const T* values, int64_t n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) rec_observe_seq<T>(v, run, values, n);
}

template <typename T>
__global__ void rec_finish_kernel(rec_view<T> v, int run0, int n) {
  const int r = run0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r < run0 + n) rec_finish_one<T>(v, r);
}

template <typename T>
rec_view<T> view(evb_recorder_s* r) {
  return rec_view<T>{static_cast<T*>(r->grid), static_cast<T*>(r->running), r->next_slot, r->fes, r->n_ckpt,
                     r->interval};
}

template <typename T>
std::string fmt(T v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

}  // namespace

void recorder_observe(evb_recorder_s* rec, int run, const void* values, int64_t n, cudaStream_t st) {
  if (!rec || n <= 0) return;
  if (rec->dtype == EVB_F64) rec_observe_kernel<double><<<1, 32, 0, st>>>(view<double>(rec), run, static_cast<const double*>(values), n);
  else rec_observe_kernel<float><<<1, 32, 0, st>>>(view<float>(rec), run, static_cast<const float*>(values), n);
  count_launch();
  EVB_CUDA(cudaGetLastError());
}

void* recorder_view(evb_recorder_s* rec, int* n_ckpt, int64_t* interval, void** running, int** next, int64_t** fes) {
  *n_ckpt = rec->n_ckpt;
  *interval = rec->interval;
  *running = rec->running;
  *next = rec->next_slot;
  *fes = rec->fes;
  return rec->grid;
}
int recorder_dtype(evb_recorder_s* rec) { return rec->dtype; }
int recorder_runs(evb_recorder_s* rec) { return rec->n_runs; }

}  // namespace evb

using namespace evb;

extern "C" {

int evb_recorder_create(int dtype, int n_runs, int64_t max_fes, int64_t interval, evb_recorder* out) {
  return guarded([&] {
    require(dtype == EVB_F32 || dtype == EVB_F64, "best_so_far_record: dtype must be EVB_F32 or EVB_F64");
    require(out != nullptr, "best_so_far_record: null output handle");
    require(interval > 0, "best_so_far_record: interval must be positive");  // recorder.hpp:47
    require(n_runs > 0, "best_so_far_record: runs must be positive");
    const int64_t ck = max_fes / interval;
    require(ck > 0, "best_so_far_record: max_fes must cover one interval");
    auto* r = new evb_recorder_s();
    r->dtype = dtype;
    r->n_runs = n_runs;
    r->n_ckpt = int(ck);
    r->interval = interval;
    r->max_fes = max_fes;
    const size_t es = dtype == EVB_F64 ? 8 : 4;
    try {
      EVB_CUDA(cudaMalloc(&r->grid, es * size_t(n_runs) * r->n_ckpt));
      EVB_CUDA(cudaMalloc(&r->running, es * n_runs));
      EVB_CUDA(cudaMalloc(&r->next_slot, sizeof(int) * n_runs));
      EVB_CUDA(cudaMalloc(&r->fes, sizeof(int64_t) * n_runs));
    } catch (...) {
      cudaFree(r->grid);
      cudaFree(r->running);
      cudaFree(r->next_slot);
      cudaFree(r->fes);
      delete r;
      throw;
    }
    const int blocks = int(std::min<int64_t>(1024, (int64_t(n_runs) * r->n_ckpt + 255) / 256));
    if (dtype == EVB_F64)
      rec_init_kernel<double><<<blocks, 256>>>(static_cast<double*>(r->grid), static_cast<double*>(r->running),
                                               r->next_slot, r->fes, n_runs, r->n_ckpt);
    else
      rec_init_kernel<float><<<blocks, 256>>>(static_cast<float*>(r->grid), static_cast<float*>(r->running),
                                              r->next_slot, r->fes, n_runs, r->n_ckpt);
    count_launch();
    EVB_CUDA(cudaDeviceSynchronize());
    *out = r;
  });
}

int evb_recorder_destroy(evb_recorder r) {
  return guarded([&] {
    if (!r) return;
    cudaFree(r->grid);
    cudaFree(r->running);
    cudaFree(r->next_slot);
    cudaFree(r->fes);
    delete r;
  });
}

int evb_recorder_checkpoints(evb_recorder r) { return r ? r->n_ckpt : -1; }

// values: device array of n fitness values of run `run`, in FE order (on_evaluate each)
int evb_recorder_observe(evb_recorder r, int run, const void* values, int64_t n, void* stream) {
  return guarded([&] {
    require(r != nullptr, "recorder: null handle");
    require(run >= 0 && run < r->n_runs, "recorder: run out of range");
    require(n >= 0 && (values || n == 0), "recorder: bad values");
    recorder_observe(r, run, values, n, static_cast<cudaStream_t>(stream));
  });
}

// on_run_end for runs [run0, run0 + n)
int evb_recorder_finish(evb_recorder r, int run0, int n, void* stream) {
  return guarded([&] {
    require(r != nullptr, "recorder: null handle");
    require(run0 >= 0 && n >= 0 && run0 + n <= r->n_runs, "recorder: run range out of bounds");
    if (n == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (r->dtype == EVB_F64) rec_finish_kernel<double><<<(n + 127) / 128, 128, 0, st>>>(view<double>(r), run0, n);
    else rec_finish_kernel<float><<<(n + 127) / 128, 128, 0, st>>>(view<float>(r), run0, n);
    count_launch();
    EVB_CUDA(cudaGetLastError());
  });
}

int evb_recorder_grid(evb_recorder r, void* grid_host, int64_t* fes_host) {
  return guarded([&] {
    require(r != nullptr, "recorder: null handle");
    EVB_CUDA(cudaDeviceSynchronize());
    const size_t es = r->dtype == EVB_F64 ? 8 : 4;
    if (grid_host) EVB_CUDA(cudaMemcpy(grid_host, r->grid, es * size_t(r->n_runs) * r->n_ckpt, cudaMemcpyDeviceToHost));
    if (fes_host) EVB_CUDA(cudaMemcpy(fes_host, r->fes, sizeof(int64_t) * r->n_runs, cudaMemcpyDeviceToHost));
  });
}

// best_so_far_record::to_csv (experiment/recorder.hpp:103-121) for a suite laid out as
// problem_ids x instances x runs (run index fastest), written into `buf` (capacity `cap`);
// *len receives the full length (call with buf = NULL to size it).
int evb_recorder_csv(evb_recorder r, const char* suite_name, int dim, int n_problems, const int* problem_ids,
                     int instances, int runs, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    require(r != nullptr && suite_name && problem_ids && len, "recorder_csv: null argument");
    require(int64_t(n_problems) * instances * runs == r->n_runs, "recorder_csv: layout does not match the runs");
    EVB_CUDA(cudaDeviceSynchronize());
    const size_t cells = size_t(r->n_runs) * r->n_ckpt;
    std::string out = "suite,problem,instance,dim,run,fes,best_so_far\n";
    auto emit = [&](auto* g) {
      for (int p = 0; p < n_problems; ++p)
        for (int i = 0; i < instances; ++i)
          for (int k = 0; k < runs; ++k) {
            const size_t run = (size_t(p) * instances + i) * runs + k;
            const std::string prefix = std::string(suite_name) + "," + std::to_string(problem_ids[p]) + "," +
                                       std::to_string(i + 1) + "," + std::to_string(dim) + "," +
                                       std::to_string(k + 1) + ",";
            for (int c = 0; c < r->n_ckpt; ++c) {
              out += prefix;
              out += std::to_string((int64_t(c) + 1) * r->interval);
              out += ',';
              out += fmt(g[run * r->n_ckpt + c]);
              out += '\n';
            }
          }
    };
    if (r->dtype == EVB_F64) {
      std::vector<double> g(cells);
      EVB_CUDA(cudaMemcpy(g.data(), r->grid, sizeof(double) * cells, cudaMemcpyDeviceToHost));
      emit(g.data());
    } else {
      std::vector<float> g(cells);
      EVB_CUDA(cudaMemcpy(g.data(), r->grid, sizeof(float) * cells, cudaMemcpyDeviceToHost));
      emit(g.data());
    }
    *len = int64_t(out.size());
    if (buf && cap > 0) std::memcpy(buf, out.data(), std::min<size_t>(size_t(cap), out.size()));
  });
}

// ---- parameter_record (experiment/parameter_record.hpp:15-95) ---------------------------------
// Per run a series of (generation, mu_F, mu_CR) appended on the device after each generation of
// an adaptive DE engine (de/engine.hpp:126-129 -> on_generation), exported as the reference CSV.

int evb_param_trace_create(int dtype, int n_runs, int capacity, evb_param_trace* out) {
  return guarded([&] {
    require(dtype == EVB_F32 || dtype == EVB_F64, "parameter_record: dtype must be EVB_F32 or EVB_F64");
    require(out != nullptr && n_runs > 0 && capacity > 0, "parameter_record: bad arguments");
    auto* t = new evb_param_trace_s();
    t->dtype = dtype;
    t->n_runs = n_runs;
    t->cap = capacity;
    const size_t es = dtype == EVB_F64 ? 8 : 4;
    try {
      EVB_CUDA(cudaMalloc(&t->gen, sizeof(int) * size_t(n_runs) * capacity));
      EVB_CUDA(cudaMalloc(&t->mu_f, es * size_t(n_runs) * capacity));
      EVB_CUDA(cudaMalloc(&t->mu_cr, es * size_t(n_runs) * capacity));
      EVB_CUDA(cudaMalloc(&t->count, sizeof(int) * n_runs));
      EVB_CUDA(memset_now(t->count, 0, sizeof(int) * n_runs));
    } catch (...) {
      cudaFree(t->gen);
      cudaFree(t->mu_f);
      cudaFree(t->mu_cr);
      cudaFree(t->count);
      delete t;
      throw;
    }
    *out = t;
  });
}

int evb_param_trace_destroy(evb_param_trace t) {
  return guarded([&] {
    if (!t) return;
    cudaFree(t->gen);
    cudaFree(t->mu_f);
    cudaFree(t->mu_cr);
    cudaFree(t->count);
    delete t;
  });
}

// series of run `run`: up to `cap` entries; *count receives the number recorded
int evb_param_trace_get(evb_param_trace t, int run, int* gens, void* mu_f, void* mu_cr, int cap, int* count) {
  return guarded([&] {
    require(t != nullptr && run >= 0 && run < t->n_runs && count, "parameter_record: bad arguments");
    EVB_CUDA(cudaDeviceSynchronize());
    int n = 0;
    EVB_CUDA(cudaMemcpy(&n, t->count + run, sizeof(int), cudaMemcpyDeviceToHost));
    n = std::min(n, t->cap);
    *count = n;
    const int m = std::min(n, cap);
    const size_t es = t->dtype == EVB_F64 ? 8 : 4;
    const size_t off = size_t(run) * t->cap;
    if (m > 0 && gens) EVB_CUDA(cudaMemcpy(gens, t->gen + off, sizeof(int) * m, cudaMemcpyDeviceToHost));
    if (m > 0 && mu_f)
      EVB_CUDA(cudaMemcpy(mu_f, static_cast<uint8_t*>(t->mu_f) + off * es, es * m, cudaMemcpyDeviceToHost));
    if (m > 0 && mu_cr)
      EVB_CUDA(cudaMemcpy(mu_cr, static_cast<uint8_t*>(t->mu_cr) + off * es, es * m, cudaMemcpyDeviceToHost));
  });
}

// parameter_record::to_csv (parameter_record.hpp:58-78): problem,instance,run,generation,mu_f,mu_cr
int evb_param_trace_csv(evb_param_trace t, int n_problems, const int* problem_ids, int instances, int runs, char* buf,
                        int64_t cap, int64_t* len) {
  return guarded([&] {
    require(t != nullptr && problem_ids && len, "parameter_record_csv: null argument");
    require(int64_t(n_problems) * instances * runs == t->n_runs, "parameter_record_csv: layout does not match the runs");
    EVB_CUDA(cudaDeviceSynchronize());
    const size_t es = t->dtype == EVB_F64 ? 8 : 4;
    const size_t cells = size_t(t->n_runs) * t->cap;
    std::vector<int> cnt(t->n_runs), gen(cells);
    std::vector<uint8_t> mf(es * cells), mc(es * cells);
    EVB_CUDA(cudaMemcpy(cnt.data(), t->count, sizeof(int) * t->n_runs, cudaMemcpyDeviceToHost));
    EVB_CUDA(cudaMemcpy(gen.data(), t->gen, sizeof(int) * cells, cudaMemcpyDeviceToHost));
    EVB_CUDA(cudaMemcpy(mf.data(), t->mu_f, es * cells, cudaMemcpyDeviceToHost));
    EVB_CUDA(cudaMemcpy(mc.data(), t->mu_cr, es * cells, cudaMemcpyDeviceToHost));
    std::string out = "problem,instance,run,generation,mu_f,mu_cr\n";
    auto val = [&](const std::vector<uint8_t>& v, size_t k) {
      return t->dtype == EVB_F64 ? fmt(reinterpret_cast<const double*>(v.data())[k])
                                 : fmt(reinterpret_cast<const float*>(v.data())[k]);
    };
    for (int p = 0; p < n_problems; ++p)
      for (int i = 0; i < instances; ++i)
        for (int r = 0; r < runs; ++r) {
          const size_t run = (size_t(p) * instances + i) * runs + r;
          const std::string prefix =
              std::to_string(problem_ids[p]) + "," + std::to_string(i + 1) + "," + std::to_string(r + 1) + ",";
          const int n = std::min(cnt[run], t->cap);
          for (int e = 0; e < n; ++e) {
            const size_t k = run * t->cap + e;
            out += prefix;
            out += std::to_string(gen[k]);
            out += ',';
            out += val(mf, k);
            out += ',';
            out += val(mc, k);
            out += '\n';
          }
        }
    *len = int64_t(out.size());
    if (buf && cap > 0) std::memcpy(buf, out.data(), std::min<size_t>(size_t(cap), out.size()));
  });
}

}  // extern "C"
