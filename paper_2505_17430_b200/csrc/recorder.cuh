// recorder.cuh — device-side best-so-far bookkeeping shared by the recorder entry points and
// the engines (experiment/recorder.hpp:65-84 semantics).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace evb {

template <typename T>
struct rec_view {
  T* grid;        // n_runs x n_ckpt
  T* running;     // n_runs
  int* next;      // n_runs
  int64_t* fes;   // n_runs
  int n_ckpt;
  int64_t interval;
};

// on_evaluate for n values in FE order (single thread; the reference loop, recorder.hpp:65-75)
template <typename T>
__device__ inline void rec_observe_seq(const rec_view<T>& v, int run, const T* values, int64_t n) {
  T m = v.running[run];
  int nx = v.next[run];
  int64_t f = v.fes[run];
  T* g = v.grid + size_t(run) * v.n_ckpt;
  for (int64_t q = 0; q < n; ++q) {
    const T x = values[q];
    if (x < m) m = x;
    ++f;
    while (nx < v.n_ckpt && f >= (int64_t(nx) + 1) * v.interval) g[nx++] = m;
  }
  v.running[run] = m;
  v.next[run] = nx;
  v.fes[run] = f;
}

// on_run_end (recorder.hpp:77-84)
template <typename T>
__device__ inline void rec_finish_one(const rec_view<T>& v, int run) {
  int nx = v.next[run];
  T* g = v.grid + size_t(run) * v.n_ckpt;
  while (nx < v.n_ckpt) g[nx++] = v.running[run];
  v.next[run] = nx;
}

}  // namespace evb
