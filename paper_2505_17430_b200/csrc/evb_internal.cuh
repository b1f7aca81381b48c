// evb_internal.cuh — shared host/device definitions of libevb (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "evb.h"

namespace evb {

// ---- error plumbing --------------------------------------------------------------------
// Internal code throws these; the C ABI layer converts them to status codes.
struct invalid_argument : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct config_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct logic_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct runtime_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
#define EVB_CUDA(x) ::evb::cuda_check((x), #x)

inline void require(bool c, const std::string& msg) {
  if (!c) throw config_error(msg);
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// thread-local message behind evb_last_error (capi.cu)
void set_last_error(const char* msg);

// Run `fn`, mapping internal exceptions onto C status codes + evb_last_error.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    set_last_error("");
    return EVB_OK;
  } catch (const invalid_argument& e) {
    set_last_error(e.what());
    return EVB_ERR_INVALID_ARGUMENT;
  } catch (const config_error& e) {
    set_last_error(e.what());
    return EVB_ERR_CONFIG;
  } catch (const logic_error& e) {
    set_last_error(e.what());
    return EVB_ERR_LOGIC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return EVB_ERR_RUNTIME;
  } catch (...) {
    set_last_error("unknown error");
    return EVB_ERR_RUNTIME;
  }
}

// ---- problem representation ------------------------------------------------------------
enum spec_kind { SPEC_BASE = 0, SPEC_HYBRID = 1, SPEC_COMPOSITION = 2 };

// Leading dimension of every device matrix/vector the problem owns: a multiple of 16
// elements so TMA boxes of one 128-byte swizzle atom tile it, and the tail [dim, ld) is
// zero so out-of-range K contributes exactly 0 to z.
constexpr int kLdAlign = 16;

struct device_problem {
  int dtype = EVB_F64;
  int dim = 0;
  int ld = 0;  // padded leading dimension (elements)
  int spec = SPEC_BASE;
  int kind = EVB_SPHERE;
  double bias = 0.0;
  // base / hybrid
  void* shift = nullptr;     // ld + 16 elements, zero padded
  void* rotation = nullptr;  // dim rows x ld (row-major, zero padded columns)
  void* ell_w = nullptr;     // elliptic weights pow(10, 6 i/(D-1)) in T, computed on the host
  // hybrid (problems/instance.hpp:24-30, 97-112)
  int n_chunks = 0;
  int* perm = nullptr;
  int* sub_kinds = nullptr;
  int* chunk_sizes = nullptr;
  // composition (problems/instance.hpp:33-41, 116-174)
  int n_comp = 0;
  int* comp_kinds = nullptr;
  std::vector<int> h_comp_kinds;  // host copies (no device->host read on the evaluation path)
  std::vector<double> h_comp_sigma, h_comp_lambda, h_comp_bias;
  void* comp_shift = nullptr;  // n_comp x ld
  void* comp_rot = nullptr;    // n_comp x dim x ld
  double* comp_sigma = nullptr;
  double* comp_lambda = nullptr;
  double* comp_bias = nullptr;
  void* hyb_w = nullptr;      // hybrid: per-chunk elliptic weights, chunk c at its offset
  // small D (eval_small_kernel): M transposed and dense, rot_t[k * dim + i] = M[i][k], padded to
  // a 16-byte multiple — one bulk copy stages it, and the row-per-thread dot products then read
  // consecutive shared-memory words (conflict-free)
  void* rot_t = nullptr;
  // fp32 tensor-core path: TF32 head / remainder split of the rotation (made on first use)
  void* rot_hi = nullptr;
  void* rot_lo = nullptr;
  void* rot_hi16 = nullptr;  // fp16 split of 2^8 * rotation (the 3xFP16 kernel), built on first use
  void* rot_lo16 = nullptr;
  bool f16_unsafe = false;   // the scaled rotation leaves fp16's range: this problem stays on 3xTF32
};

}  // namespace evb

struct evb_problem_s {
  evb::device_problem p;
};

// device word source (rng.cuh): PHILOX (mode 0) or WORDS (mode 1)
struct evb_rng_s {
  int mode = 0;
  uint64_t key = 0;
  uint64_t* d_words = nullptr;
  int64_t n_words = 0;
  int64_t* d_cursor = nullptr;  // WORDS: next unread word (device-resident)
  uint32_t gen = 0;             // PHILOX: generation counter (host mirror)
  uint32_t* d_gen = nullptr;    // PHILOX: generation counter read by the kernels (graph-replayable)
  int* d_overflow = nullptr;
};

struct evb_scratch_s {
  cudaStream_t own_stream = nullptr;
  // large-D fused path: per (channel, n-tile, point) partial sums + per m-block counters
  void* partial = nullptr;
  size_t partial_bytes = 0;
  unsigned* counters = nullptr;
  size_t counters_n = 0;
  // materialised z (SoA: z[i * ldp + b], the reference's soa_z layout, problems/batch.hpp:44-45)
  void* zbuf = nullptr;
  size_t zbuf_bytes = 0;
  // re-pitched copy of X when the caller's rows are not TMA-legal
  void* xpad = nullptr;
  size_t xpad_bytes = 0;
  // host-buffer path
  void* dx = nullptr;
  size_t dx_bytes = 0;
  void* dout = nullptr;
  size_t dout_bytes = 0;
  // composition: value accumulators (double) per point
  double* acc = nullptr;
  size_t acc_bytes = 0;
  // fp32 3xFP16 path: rows whose S = X - o leaves fp16's range (recomputed in fp32 by the row
  // block's last CTA); zero between launches
  int* row_bad = nullptr;
  size_t row_bad_n = 0;
  // fp32 tensor-core path: TF32 split of S = X - o
  void* s_hi = nullptr;
  size_t s_hi_bytes = 0;
  void* s_lo = nullptr;
  size_t s_lo_bytes = 0;
  // host-buffer path with the H2D copy overlapped: X arrives in column chunks on copy_stream,
  // each followed by a stream write of gate[c] = epoch that the GEMM producer waits on
  // (gate writes are issued on gate_stream behind per-chunk events: a stream write between two
  // copies on the copy stream stalls the DMA pipeline ~5 us per chunk)
  cudaStream_t copy_stream = nullptr;
  cudaStream_t gate_stream = nullptr;
  unsigned* gate = nullptr;  // kMaxGates words
  unsigned gate_epoch = 0;
  cudaEvent_t ev_x_ready = nullptr;
  cudaEvent_t ev_chunk[16] = {};
  // page-locked host staging for the C++ wrapper's vector<vector<T>> batches
  void* host_stage = nullptr;
  size_t host_stage_bytes = 0;
};

namespace evb {

// Zero-fill at object creation, complete before returning.  cudaMemset on device memory returns
// before the fill lands and runs on the legacy stream, which the library's non-blocking streams do
// not wait for: a gate word cleared that way could overwrite the first epoch written on the gate
// stream (the kernel then waits until its 10-s trap).
inline cudaError_t memset_now(void* p, int v, size_t n) {
  const cudaError_t e = cudaMemset(p, v, n);
  return e != cudaSuccess ? e : cudaStreamSynchronize(nullptr);
}

// Host -> device copy complete before returning.  A cudaMemcpy from pageable memory returns once
// the data is staged, not when the DMA has landed, and it is ordered only on the legacy stream.
inline cudaError_t copy_h2d_now(void* dst, const void* src, size_t n) {
  const cudaError_t e = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
  return e != cudaSuccess ? e : cudaStreamSynchronize(nullptr);
}

// Launch with programmatic stream serialisation (PDL): the kernel's launch overlaps the tail of
// the previous kernel in the stream; the kernel itself must call ptx::griddep_wait() before
// touching predecessor data (launch latency is most of a small generation's kernel time).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kernel, static_cast<KArgs>(args)...);
}

// Grow-only device buffer; synchronises `stream` before releasing an old allocation.
inline void ensure_buffer(void** ptr, size_t* cap, size_t need, cudaStream_t stream) {
  if (*cap >= need && *ptr) return;
  if (*ptr) {
    EVB_CUDA(cudaStreamSynchronize(stream));
    EVB_CUDA(cudaFree(*ptr));
    *ptr = nullptr;
    *cap = 0;
  }
  size_t bytes = need < 256 ? 256 : need;
  EVB_CUDA(cudaMalloc(ptr, bytes));
  *cap = bytes;
}

// TMA descriptor helpers (driver entry point fetched through the runtime; no -lcuda).
constexpr int kTmaF16 = 100;  // make_tma_2d dtype: fp16 elements (beside EVB_F32 / EVB_F64)
bool make_tma_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner_elems,
                 uint64_t outer_rows, uint64_t row_stride_bytes, uint32_t box_inner,
                 uint32_t box_outer);

// ---- evaluation entry points (eval_*.cu) -------------------------------------------------
struct eval_request {
  const device_problem* prob;
  evb_scratch_s* scratch;
  const void* X;
  int64_t n;
  int64_t ldx;
  void* out;
  int64_t ldo;
  int n_out;        // number of output kinds (multi); 1 for evaluate_batch
  int kinds[4];     // base kinds per output
  double biases[4]; // additive bias per output
  cudaStream_t stream;
  bool scalar_trig = false;  // true: problem_instance::evaluate semantics (libm trig also for
                             // float, problems/functions.hpp); false: evaluate_batch semantics
                             // (fast_cos/fast_sin for float, problems/batch.hpp:17-33)
  // X still arriving: columns [c*kgate_cols, (c+1)*kgate_cols) are valid once kgate[c] reaches
  // kgate_epoch (wrap-safe compare); x_ready fires when all of X is resident.  Kernels that do
  // not consume the gates make the stream wait on x_ready instead.
  const unsigned* kgate = nullptr;
  int kgate_n = 0;
  int kgate_end[8] = {};  // exclusive end column of chunk c (multiples of 16 but the last)
  unsigned kgate_epoch = 0;
  // > 0 (multi-problem K1 only): rows [kgate_rows, n) arrive after rows [0, kgate_rows), in the
  // same column chunks, gated by kgate[kgate_n + c]; the kernel then runs the first rows' tiles
  // as its first wave
  int kgate_rows = 0;
  cudaEvent_t x_ready = nullptr;
};

constexpr int kMaxGates = 16;

// rows whose tiles make up the first wave of the multi-problem K1 at this size (a multiple of
// its row tile), or 0 when every tile is resident at once (eval_gemm.cu)
int multi_first_wave_rows(int np, int64_t n_points, int64_t dim);

void eval_dispatch(const eval_request& rq);
bool eval_small_path(const device_problem& p);
// true when eval_dispatch runs the request on the fused fp64 GEMM, whose producer honours kgate
bool gate_eligible(const eval_request& rq);
// several base problems (same D, fp64, fused kinds) on one device X in one multi-problem K1
// launch (eval_gemm.cu); false when the requests do not qualify (caller falls back)
bool multi_eligible(const eval_request* rqs, int np);
bool gemm_eval_multi(const eval_request* rqs, int np, const void* X, int64_t ldx);

}  // namespace evb

// parameter_record trace (recorder.cu): per run (generation, mu_F, mu_CR) series on the device
struct evb_param_trace_s {
  int dtype = EVB_F64;
  int n_runs = 0, cap = 0;
  int* gen = nullptr;      // n_runs x cap
  void* mu_f = nullptr;    // n_runs x cap (T)
  void* mu_cr = nullptr;   // n_runs x cap (T)
  int* count = nullptr;    // n_runs
};

namespace evb {

// best-so-far recorder (recorder.cu)
void recorder_observe(evb_recorder_s* rec, int run, const void* values, int64_t n, cudaStream_t st);
void* recorder_view(evb_recorder_s* rec, int* n_ckpt, int64_t* interval, void** running, int** next, int64_t** fes);
int recorder_dtype(evb_recorder_s* rec);
int recorder_runs(evb_recorder_s* rec);

// batched-runs kernel eligibility (runs.cu): empty when supported, else the reason
std::string runs_kernel_unsupported(int dtype, const evb_de_config* cfg, int pop_size, int dim,
                                    const evb_problem* problems, int n_runs);

// init_population (de.cu): P x D uniforms in [lb, ub] from the rng (Philox sub-stream kSubInit of
// the current generation, or the WORDS cursor); advances the rng like the reference's stream
void population_init(int dtype, int P, int D, void* pop, int64_t ldp, double lb, double ub, evb_rng_s* r,
                     cudaStream_t st);

// device generation counter <- host mirror (after host-side Philox consumers such as init)
void set_device_gen(evb_rng_s* r, cudaStream_t st);

// Per-phase CUDA events on the launching stream (bench.py's per-kernel roofline timing): when on,
// an engine records an event before its first kernel and after each phase of a generation;
// elapsed(ev[k], ev[k+1]) is phase k's device time.  Off by default: the events sit between
// kernels that otherwise overlap launch and prologue with the predecessor's tail (PDL).
struct phase_timer {
  static constexpr int kMax = 8;
  cudaEvent_t ev[kMax] = {};
  int n = 0;
  bool on = false;
  void mark(cudaStream_t st) {
    if (!on || n >= kMax) return;
    if (!ev[n]) cuda_check(cudaEventCreate(&ev[n]), "phase_timer event");
    cuda_check(cudaEventRecord(ev[n], st), "phase_timer record");
    ++n;
  }
  void begin(cudaStream_t st) {
    n = 0;
    mark(st);
  }
  // phase durations of the last generation (synchronises on its last event); returns the count
  int read(float* ms, int cap) {
    if (n < 2) return 0;
    cuda_check(cudaEventSynchronize(ev[n - 1]), "phase_timer sync");
    int k = 0;
    for (; k + 1 < n && k < cap; ++k) cuda_check(cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]), "phase_timer");
    return k;
  }
  void destroy() {
    for (auto& e : ev)
      if (e) {
        cudaEventDestroy(e);
        e = nullptr;
      }
  }
};

// Number of kernel launches issued by the last eval_dispatch on this thread (bench accounting).
int last_launch_count();
void count_launch(int n = 1);

}  // namespace evb
