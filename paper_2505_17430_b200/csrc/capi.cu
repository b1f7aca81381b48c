// capi.cu — the extern "C" boundary of libevb (include/evb.h).
//
// Host C++ owns the problem/scratch objects; every entry point converts internal exceptions
// into status codes plus a thread-local message, so no exception crosses the ABI.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "evb_internal.cuh"

namespace evb {

namespace {
thread_local std::string g_last_error;

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

using write_value32_fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
write_value32_fn stream_write_value32() {
  static write_value32_fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<write_value32_fn>(p);
  });
  return fn;
}

size_t elem_size(int dtype) { return dtype == EVB_F64 ? 8 : 4; }

void check_dtype(int dtype) {
  require(dtype == EVB_F32 || dtype == EVB_F64, "problem: dtype must be EVB_F32 or EVB_F64");
}
void check_kind(int kind) {
  require(kind >= EVB_SPHERE && kind <= EVB_EXPANDED_SCHAFFER_F6, "problem: unknown base kind");
}

template <typename T>
std::vector<T> elliptic_weights(int len) {
  // pow(T(10), T(6) * T(i) / T(max(len - 1, 1))) in T, as problems/functions.hpp:57-60 and
  // problems/batch.hpp:109-111 compute it.
  std::vector<T> w(std::max(len, 1));
  const T denom = T(std::max(len - 1, 1));
  for (int i = 0; i < len; ++i) w[i] = std::pow(T(10), T(6) * T(i) / denom);
  return w;
}

void* upload(const void* host, size_t bytes) {
  void* d = nullptr;
  EVB_CUDA(cudaMalloc(&d, std::max<size_t>(bytes, 16)));
  if (bytes) EVB_CUDA(copy_h2d_now(d, host, bytes));
  return d;
}

// rows x dim (stride src_ld) -> device rows x ld, zero padded, plus `extra` zero elements
void* upload_padded(const void* host, int rows, int dim, int ld, int extra, size_t es) {
  std::vector<uint8_t> buf(size_t(rows) * ld * es + size_t(extra) * es, 0);
  for (int r = 0; r < rows; ++r)
    std::memcpy(buf.data() + size_t(r) * ld * es, static_cast<const uint8_t*>(host) + size_t(r) * dim * es,
                size_t(dim) * es);
  return upload(buf.data(), buf.size());
}

// M^T, dense (dim x dim), padded to a 16-byte multiple: the small-D kernel's bulk-copy source
void* upload_transposed(const void* host, int dim, size_t es) {
  std::vector<uint8_t> buf((size_t(dim) * dim * es + 15) / 16 * 16, 0);
  for (int i = 0; i < dim; ++i)
    for (int k = 0; k < dim; ++k)
      std::memcpy(buf.data() + (size_t(k) * dim + i) * es, static_cast<const uint8_t*>(host) + (size_t(i) * dim + k) * es,
                  es);
  return upload(buf.data(), buf.size());
}
constexpr int kSmallTransposeMaxDim = 160;

template <typename T>
void* upload_weights(const std::vector<T>& w) {
  return upload(w.data(), w.size() * sizeof(T));
}

void fill_weights(device_problem& p) {
  if (p.dtype == EVB_F64) p.ell_w = upload_weights(elliptic_weights<double>(p.dim));
  else p.ell_w = upload_weights(elliptic_weights<float>(p.dim));
}

void free_problem(device_problem& p) {
  void* ptrs[] = {p.shift, p.rotation, p.ell_w, p.hyb_w, p.perm, p.sub_kinds, p.chunk_sizes, p.comp_kinds,
                  p.comp_shift, p.comp_rot, p.comp_sigma, p.comp_lambda, p.comp_bias, p.rot_hi, p.rot_lo, p.rot_hi16, p.rot_lo16, p.rot_t};
  for (void* q : ptrs)
    if (q) cudaFree(q);
}

}  // namespace

void set_last_error(const char* msg) { g_last_error = msg; }

bool make_tma_2d(CUtensorMap* map, const void* base, int dtype, uint64_t inner_elems, uint64_t outer_rows,
                 uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner_elems, outer_rows};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = dtype == EVB_F64   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                 : dtype == kTmaF16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUresult r = enc(map, dt, 2,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace evb

using namespace evb;

extern "C" {

int evb_abi_version(void) { return EVB_ABI_VERSION; }

const char* evb_last_error(void) { return g_last_error.c_str(); }

int evb_device_info(int device, int* sm_count, int* smem_per_sm, int* l2_bytes, int* cc_major, int* cc_minor) {
  return guarded([&] {
    cudaDeviceProp pr;
    EVB_CUDA(cudaGetDeviceProperties(&pr, device));
    if (sm_count) *sm_count = pr.multiProcessorCount;
    if (smem_per_sm) *smem_per_sm = int(pr.sharedMemPerMultiprocessor);
    if (l2_bytes) *l2_bytes = pr.l2CacheSize;
    if (cc_major) *cc_major = pr.major;
    if (cc_minor) *cc_minor = pr.minor;
  });
}

int evb_device_alloc(size_t bytes, void** out) {
  return guarded([&] {
    require(out != nullptr, "device_alloc: null output");
    EVB_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  });
}
int evb_device_free(void* ptr) {
  return guarded([&] {
    if (ptr) EVB_CUDA(cudaFree(ptr));
  });
}
int evb_copy_to_device(void* dst, const void* src, size_t bytes) {
  return guarded([&] { EVB_CUDA(copy_h2d_now(dst, src, bytes)); });
}
int evb_copy_to_host(void* dst, const void* src, size_t bytes) {
  return guarded([&] { EVB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}
int evb_synchronize(void) {
  return guarded([&] { EVB_CUDA(cudaDeviceSynchronize()); });
}

int evb_problem_create_base(int dtype, int dim, int kind, const void* shift, const void* rotation, double bias,
                            evb_problem* out) {
  return guarded([&] {
    check_dtype(dtype);
    check_kind(kind);
    require(dim >= 1, "problem: dim must be positive");
    require(shift && rotation && out, "problem: null shift, rotation or output handle");
    auto* h = new evb_problem_s();
    device_problem& p = h->p;
    try {
      p.dtype = dtype;
      p.dim = dim;
      p.ld = int(round_up(dim, kLdAlign));
      p.spec = SPEC_BASE;
      p.kind = kind;
      p.bias = bias;
      const size_t es = elem_size(dtype);
      p.shift = upload_padded(shift, 1, dim, p.ld, 64, es);
      p.rotation = upload_padded(rotation, dim, dim, p.ld, 0, es);
      if (dim <= kSmallTransposeMaxDim) p.rot_t = upload_transposed(rotation, dim, es);
      fill_weights(p);
    } catch (...) {
      free_problem(p);
      delete h;
      throw;
    }
    *out = h;
  });
}

int evb_problem_create_hybrid(int dtype, int dim, const void* shift, const void* rotation, double bias, int n_chunks,
                              const int* sub_kinds, const int* chunk_sizes, const int* permutation, evb_problem* out) {
  return guarded([&] {
    check_dtype(dtype);
    require(dim >= 1, "problem: dim must be positive");
    require(shift && rotation && out && sub_kinds && chunk_sizes && permutation,
            "hybrid: null input pointer");
    require(n_chunks >= 1, "hybrid: at least one chunk");
    int total = 0;
    for (int c = 0; c < n_chunks; ++c) {
      check_kind(sub_kinds[c]);
      require(chunk_sizes[c] >= 1, "hybrid: every chunk needs at least one dimension");
      total += chunk_sizes[c];
    }
    require(total == dim, "hybrid: chunk sizes must sum to dim");
    std::vector<int> seen(dim, 0);
    for (int i = 0; i < dim; ++i) {
      require(permutation[i] >= 0 && permutation[i] < dim && !seen[permutation[i]],
              "hybrid: permutation must use every dimension once");
      seen[permutation[i]] = 1;
    }
    auto* h = new evb_problem_s();
    device_problem& p = h->p;
    try {
      p.dtype = dtype;
      p.dim = dim;
      p.ld = int(round_up(dim, kLdAlign));
      p.spec = SPEC_HYBRID;
      p.bias = bias;
      const size_t es = elem_size(dtype);
      p.shift = upload_padded(shift, 1, dim, p.ld, 64, es);
      p.rotation = upload_padded(rotation, dim, dim, p.ld, 0, es);
      if (dim <= kSmallTransposeMaxDim) p.rot_t = upload_transposed(rotation, dim, es);
      fill_weights(p);
      p.n_chunks = n_chunks;
      p.perm = static_cast<int*>(upload(permutation, sizeof(int) * dim));
      p.sub_kinds = static_cast<int*>(upload(sub_kinds, sizeof(int) * n_chunks));
      p.chunk_sizes = static_cast<int*>(upload(chunk_sizes, sizeof(int) * n_chunks));
      // per-chunk elliptic weights: kernels::elliptic sees only the chunk (len - 1 denominator)
      if (dtype == EVB_F64) {
        std::vector<double> w;
        for (int c = 0; c < n_chunks; ++c) {
          auto wc = elliptic_weights<double>(chunk_sizes[c]);
          w.insert(w.end(), wc.begin(), wc.begin() + chunk_sizes[c]);
        }
        p.hyb_w = upload_weights(w);
      } else {
        std::vector<float> w;
        for (int c = 0; c < n_chunks; ++c) {
          auto wc = elliptic_weights<float>(chunk_sizes[c]);
          w.insert(w.end(), wc.begin(), wc.begin() + chunk_sizes[c]);
        }
        p.hyb_w = upload_weights(w);
      }
    } catch (...) {
      free_problem(p);
      delete h;
      throw;
    }
    *out = h;
  });
}

int evb_problem_create_composition(int dtype, int dim, int n_comp, const int* kinds, const void* shifts,
                                   const void* rotations, const double* sigma, const double* lambda,
                                   const double* comp_bias, double bias, evb_problem* out) {
  return guarded([&] {
    check_dtype(dtype);
    require(dim >= 1, "problem: dim must be positive");
    require(n_comp >= 1 && n_comp <= 8, "composition: 1 to 8 components supported");
    require(kinds && shifts && rotations && sigma && lambda && comp_bias && out, "composition: null input pointer");
    for (int c = 0; c < n_comp; ++c) check_kind(kinds[c]);
    auto* h = new evb_problem_s();
    device_problem& p = h->p;
    try {
      p.dtype = dtype;
      p.dim = dim;
      p.ld = int(round_up(dim, kLdAlign));
      p.spec = SPEC_COMPOSITION;
      p.bias = bias;
      const size_t es = elem_size(dtype);
      fill_weights(p);
      p.n_comp = n_comp;
      p.comp_kinds = static_cast<int*>(upload(kinds, sizeof(int) * n_comp));
      p.h_comp_kinds.assign(kinds, kinds + n_comp);
      p.comp_shift = upload_padded(shifts, n_comp, dim, p.ld, 64, es);
      // rotations: n_comp blocks of dim rows
      p.comp_rot = upload_padded(rotations, n_comp * dim, dim, p.ld, 0, es);
      p.comp_sigma = static_cast<double*>(upload(sigma, sizeof(double) * n_comp));
      p.comp_lambda = static_cast<double*>(upload(lambda, sizeof(double) * n_comp));
      p.comp_bias = static_cast<double*>(upload(comp_bias, sizeof(double) * n_comp));
      p.h_comp_sigma.assign(sigma, sigma + n_comp);
      p.h_comp_lambda.assign(lambda, lambda + n_comp);
      p.h_comp_bias.assign(comp_bias, comp_bias + n_comp);
    } catch (...) {
      free_problem(p);
      delete h;
      throw;
    }
    *out = h;
  });
}

int evb_problem_destroy(evb_problem p) {
  return guarded([&] {
    if (!p) return;
    free_problem(p->p);
    delete p;
  });
}

int evb_problem_dim(evb_problem p) { return p ? p->p.dim : -1; }
int evb_problem_dtype(evb_problem p) { return p ? p->p.dtype : -1; }

int evb_scratch_create(evb_scratch* out) {
  return guarded([&] {
    require(out != nullptr, "scratch: null output handle");
    *out = new evb_scratch_s();
  });
}

int evb_scratch_host_staging(evb_scratch s, size_t bytes, void** out) {
  return guarded([&] {
    require(s != nullptr && out != nullptr, "scratch_host_staging: null argument");
    if (bytes > s->host_stage_bytes) {
      if (s->host_stage) {
        if (s->own_stream) EVB_CUDA(cudaStreamSynchronize(s->own_stream));
        EVB_CUDA(cudaFreeHost(s->host_stage));
        s->host_stage = nullptr;
        s->host_stage_bytes = 0;
      }
      EVB_CUDA(cudaHostAlloc(&s->host_stage, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
      s->host_stage_bytes = bytes;
    }
    *out = s->host_stage;
  });
}

int evb_scratch_destroy(evb_scratch s) {
  return guarded([&] {
    if (!s) return;
    void* ptrs[] = {s->partial, s->counters, s->zbuf, s->xpad, s->dx,  s->dout,
                    s->acc,     s->s_hi,    s->s_lo, s->gate, s->row_bad};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
    if (s->gate_stream) cudaStreamDestroy(s->gate_stream);
    if (s->ev_x_ready) cudaEventDestroy(s->ev_x_ready);
    if (s->host_stage) cudaFreeHost(s->host_stage);
    for (auto e : s->ev_chunk)
      if (e) cudaEventDestroy(e);
    delete s;
  });
}

static void validate_eval(evb_problem p, evb_scratch s, int64_t n, int64_t ldx) {
  if (!p || !s) throw config_error("evaluate_batch: null problem or scratch");
  if (n < 0) throw invalid_argument("evaluate_batch: negative point count");
  if (n > 0 && ldx < p->p.dim) throw invalid_argument("evaluate_batch: point dimension mismatch");
  if (n > (int64_t(1) << 30)) throw invalid_argument("evaluate_batch: batch too large");
}

int evb_evaluate_batch(evb_problem p, evb_scratch s, const void* X, int64_t n_points, int64_t ldx, void* out,
                       void* stream) {
  return guarded([&] {
    validate_eval(p, s, n_points, ldx);
    if (n_points == 0) return;
    if (!X || !out) throw config_error("evaluate_batch: null X or out");
    eval_request rq{};
    rq.prob = &p->p;
    rq.scratch = s;
    rq.X = X;
    rq.n = n_points;
    rq.ldx = ldx;
    rq.out = out;
    rq.ldo = n_points;
    rq.n_out = 1;
    rq.kinds[0] = p->p.kind;
    rq.biases[0] = p->p.bias;
    rq.stream = static_cast<cudaStream_t>(stream);
    eval_dispatch(rq);
  });
}

int evb_evaluate_batch_multi(evb_problem p, evb_scratch s, int n_kinds, const int* kinds, const double* biases,
                             const void* X, int64_t n_points, int64_t ldx, void* out, int64_t ldo, void* stream) {
  return guarded([&] {
    validate_eval(p, s, n_points, ldx);
    if (p->p.spec != SPEC_BASE) throw config_error("evaluate_batch_multi: base problems only");
    if (n_kinds < 1 || n_kinds > 4) throw config_error("evaluate_batch_multi: 1 to 4 kinds");
    if (!kinds || !biases) throw config_error("evaluate_batch_multi: null kinds or biases");
    for (int k = 0; k < n_kinds; ++k) check_kind(kinds[k]);
    if (n_points == 0) return;
    if (!X || !out) throw config_error("evaluate_batch_multi: null X or out");
    if (ldo < n_points) throw invalid_argument("evaluate_batch_multi: ldo < n_points");
    eval_request rq{};
    rq.prob = &p->p;
    rq.scratch = s;
    rq.X = X;
    rq.n = n_points;
    rq.ldx = ldx;
    rq.out = out;
    rq.ldo = ldo;
    rq.n_out = n_kinds;
    for (int k = 0; k < n_kinds; ++k) {
      rq.kinds[k] = kinds[k];
      rq.biases[k] = biases[k];
    }
    rq.stream = static_cast<cudaStream_t>(stream);
    eval_dispatch(rq);
  });
}

}  // extern "C"

namespace {

// Host-buffer evaluation of one population on n_prob problems (same dim / dtype): X crosses the
// host link once; the first problem's fused GEMM consumes it chunk by chunk as it lands, the
// others run on the resident copy; each out_host[k] gets problem k's fitness.
void host_eval(const evb_problem* probs, int n_prob, evb_scratch s, const void* X_host, int64_t n_points, int64_t ldx,
               void* const* outs_host) {
  require(probs != nullptr && n_prob >= 1 && outs_host != nullptr, "evaluate_batch_host: null problems or outputs");
  evb_problem p = probs[0];
  validate_eval(p, s, n_points, ldx);
  for (int k = 1; k < n_prob; ++k) {
    validate_eval(probs[k], s, n_points, ldx);
    if (probs[k]->p.dim != p->p.dim || probs[k]->p.dtype != p->p.dtype)
      throw invalid_argument("evaluate_batch_host: problems differ in dimension or dtype");
  }
  if (n_points == 0) return;
  if (!X_host) throw config_error("evaluate_batch_host: null X or out");
  for (int k = 0; k < n_prob; ++k)
    if (!outs_host[k]) throw config_error("evaluate_batch_host: null X or out");
  if (!s->own_stream) EVB_CUDA(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking));
  cudaStream_t st = s->own_stream;
  const size_t es = elem_size(p->p.dtype);
  const int64_t D = p->p.dim;
  const int64_t ldd = round_up(D, 16 / int64_t(es));
  ensure_buffer(&s->dx, &s->dx_bytes, size_t(ldd) * n_points * es, st);
  ensure_buffer(&s->dout, &s->dout_bytes, size_t(n_points) * es * n_prob, st);
  // Page-locked outputs (cudaHostAlloc / cudaHostRegister) are written by the kernels directly
  // (mapped, same address under UVA): no device staging and no D2H copy at the end.
  std::vector<void*> dst(n_prob);
  for (int k = 0; k < n_prob; ++k) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, outs_host[k]) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer == outs_host[k])
      dst[k] = outs_host[k];
    else {
      cudaGetLastError();
      dst[k] = static_cast<uint8_t*>(s->dout) + size_t(k) * n_points * es;
    }
  }
  auto request = [&](int k) {
    eval_request rq{};
    rq.prob = &probs[k]->p;
    rq.scratch = s;
    rq.X = s->dx;
    rq.n = n_points;
    rq.ldx = ldd;
    rq.out = dst[k];
    rq.ldo = n_points;
    rq.n_out = 1;
    rq.kinds[0] = probs[k]->p.kind;
    rq.biases[0] = probs[k]->p.bias;
    rq.stream = st;
    return rq;
  };
  eval_request rq = request(0);
  std::vector<eval_request> all(static_cast<size_t>(n_prob));
  for (int k = 0; k < n_prob; ++k) all[size_t(k)] = request(k);
  bool multi = multi_eligible(all.data(), n_prob);
  // The fused fp64 GEMM starts while X is still crossing the host link: X goes over in column
  // chunks on a second stream, each chunk followed by a stream write of its gate word, and the
  // GEMM producer waits per chunk before its TMA loads (the copy is the e2e bound: ~8 MB per
  // batch at D=1000, P=1024).  All copies are enqueued before the kernel, so the kernel only
  // ever waits on work queued ahead of it.  Other paths copy X whole, then launch.
  rq.X = s->dx;
  rq.ldx = ldd;
  static const char* chunks_env = std::getenv("EVB_H2D_CHUNKS");
  static const char* split_env = std::getenv("EVB_H2D_SPLIT");
  const int want = std::min(kMaxGates, chunks_env ? std::max(1, std::atoi(chunks_env)) : 4);
  const bool geometric = !(split_env && std::string(split_env) == "uniform");
  write_value32_fn wv = stream_write_value32();
  if (want > 1 && wv && gate_eligible(rq)) {
    if (!s->copy_stream) EVB_CUDA(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    if (!s->gate_stream) EVB_CUDA(cudaStreamCreateWithFlags(&s->gate_stream, cudaStreamNonBlocking));
    if (!s->ev_x_ready) EVB_CUDA(cudaEventCreateWithFlags(&s->ev_x_ready, cudaEventDisableTiming));
    for (auto& e : s->ev_chunk)
      if (!e) EVB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!s->gate) {
      EVB_CUDA(cudaMalloc(&s->gate, kMaxGates * sizeof(unsigned)));
      EVB_CUDA(memset_now(s->gate, 0, kMaxGates * sizeof(unsigned)));
    }
    // Rows: when the multi-problem kernel needs two waves, the first wave's rows (all their
    // column chunks) cross first and the rest follow, so the second wave's data lands while the
    // first computes (kgate_rows).  Columns: chunk boundaries are multiples of 16 (the GEMM's
    // K-slice): uniform, halving (single wave: the compute left after the last chunk lands is
    // small), or EVB_H2D_WIDTHS="w0,w1,..." (tuning aid).
    static const char* rows_env = std::getenv("EVB_H2D_ROWSPLIT");
    static const char* widths_env = std::getenv("EVB_H2D_WIDTHS");
    const int64_t rows_a =
        multi && !(rows_env && std::string(rows_env) == "0") ? multi_first_wave_rows(n_prob, n_points, D) : 0;
    const bool uniform = rows_a > 0 ? !(split_env && std::string(split_env) == "geo") : !geometric;
    std::vector<int64_t> widths;
    if (widths_env) {
      std::string w = widths_env;
      for (size_t pos = 0; pos < w.size();) {
        size_t nx = w.find(',', pos);
        if (nx == std::string::npos) nx = w.size();
        widths.push_back(std::max<int64_t>(16, round_up(std::atoll(w.substr(pos, nx - pos).c_str()), 16)));
        pos = nx + 1;
      }
    }
    int n_chunks = 0;
    int64_t c0 = 0;
    // two gate groups: 6 column chunks each unless EVB_H2D_CHUNKS says otherwise (measured 270 vs 274 us)
    // (at most 8 chunks per group: eval_request::kgate_end; two groups fill the 16 gate words)
    const int max_chunks = std::min(rows_a > 0 ? (chunks_env ? want : 6) : want, 8);
    while (c0 < D) {
      int64_t w;
      if (n_chunks == max_chunks - 1) w = D - c0;
      else if (!widths.empty()) w = n_chunks < int(widths.size()) ? widths[size_t(n_chunks)] : D - c0;
      else if (!uniform) w = round_up((D - c0 + 1) / 2, 16);
      else w = round_up((D + max_chunks - 1) / max_chunks, 16);
      w = std::min<int64_t>(std::max<int64_t>(w, 16), D - c0);
      rq.kgate_end[n_chunks++] = int(c0 + w);
      c0 += w;
    }
    rq.kgate_n = n_chunks;
    rq.kgate_rows = int(rows_a);
    const int n_groups = rows_a > 0 ? 2 : 1;
    const unsigned epoch = ++s->gate_epoch == 0 ? ++s->gate_epoch : s->gate_epoch;
    // EVB_H2D_TRACE=1: print the copy / kernel timeline of each call (tuning aid)
    static const bool trace = std::getenv("EVB_H2D_TRACE") != nullptr;
    static cudaEvent_t tev[kMaxGates + 3];
    if (trace && !tev[0])
      for (auto& e : tev) EVB_CUDA(cudaEventCreate(&e));
    if (trace) EVB_CUDA(cudaEventRecord(tev[0], s->copy_stream));
    // the previous call on this scratch synchronised st, so dx is free to overwrite
    bool gates_ok = true;
    for (int g = 0; g < n_groups; ++g) {
      const int64_t r0 = g ? rows_a : 0, nr = n_groups == 1 ? n_points : (g ? n_points - rows_a : rows_a);
      for (int c = 0; c < n_chunks; ++c) {
        const int gi = g * n_chunks + c;
        const int64_t b = c ? rq.kgate_end[c - 1] : 0, w = rq.kgate_end[c] - b;
        EVB_CUDA(cudaMemcpy2DAsync(static_cast<uint8_t*>(s->dx) + (r0 * ldd + b) * es, ldd * es,
                                   static_cast<const uint8_t*>(X_host) + (r0 * ldx + b) * es, ldx * es, w * es, nr,
                                   cudaMemcpyHostToDevice, s->copy_stream));
        if (gates_ok) {
          EVB_CUDA(cudaEventRecord(s->ev_chunk[gi], s->copy_stream));
          EVB_CUDA(cudaStreamWaitEvent(s->gate_stream, s->ev_chunk[gi], 0));
          // a driver that refuses stream memory operations: fall back to waiting for all of X
          gates_ok = wv(s->gate_stream, CUdeviceptr(s->gate + gi), epoch, 0) == CUDA_SUCCESS;
        }
        if (trace) EVB_CUDA(cudaEventRecord(tev[1 + gi], s->copy_stream));
      }
    }
    EVB_CUDA(cudaEventRecord(s->ev_x_ready, s->copy_stream));
    rq.kgate = gates_ok ? s->gate : nullptr;
    rq.kgate_epoch = epoch;
    rq.x_ready = s->ev_x_ready;
    if (trace) EVB_CUDA(cudaStreamWaitEvent(st, tev[0], 0));
    if (multi) {  // every problem in one launch, all consuming the chunks as they land
      std::vector<eval_request> rqs(static_cast<size_t>(n_prob));
      for (int k = 0; k < n_prob; ++k) rqs[size_t(k)] = request(k);
      rqs[0] = rq;
      if (!gemm_eval_multi(rqs.data(), n_prob, s->dx, ldd)) multi = false;
    }
    if (!multi && rows_a > 0) rq.kgate = nullptr;  // single-problem kernels know one gate group only
    if (!multi) eval_dispatch(rq);
    const int n_ev = n_chunks * n_groups;
    if (trace) EVB_CUDA(cudaEventRecord(tev[n_ev + 1], st));
    EVB_CUDA(cudaStreamWaitEvent(st, s->ev_x_ready, 0));
    if (trace) {
      if (dst[0] != outs_host[0])
        EVB_CUDA(cudaMemcpyAsync(outs_host[0], dst[0], size_t(n_points) * es, cudaMemcpyDeviceToHost, st));
      EVB_CUDA(cudaEventRecord(tev[n_ev + 2], st));
      EVB_CUDA(cudaStreamSynchronize(st));
      std::string line = "[evb h2d] rows_a " + std::to_string(rows_a) + " |";
      for (int c = 1; c <= n_ev + 2; ++c) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[0], tev[c]);
        line += (c == n_ev + 1 ? " kernel_end " : c == n_ev + 2 ? " d2h_end " : " ") +
                std::to_string(int(ms * 1000.f));
      }
      std::fprintf(stderr, "%s us\n", line.c_str());
    }
  } else {
    // one linear copy when the rows are packed (the DMA engines run 2D copies of wide rows at
    // about half the rate of a linear copy of the same bytes: 300 vs 160 us for 8 MB)
    if (ldx == ldd)
      EVB_CUDA(cudaMemcpyAsync(s->dx, X_host, size_t(ldd) * n_points * es, cudaMemcpyHostToDevice, st));
    else
      EVB_CUDA(cudaMemcpy2DAsync(s->dx, ldd * es, X_host, ldx * es, D * es, n_points, cudaMemcpyHostToDevice, st));
    if (multi && !gemm_eval_multi(all.data(), n_prob, s->dx, ldd)) multi = false;
    if (!multi) eval_dispatch(rq);
  }
  // the remaining problems evaluate the resident copy (the stream already waits for all of X)
  if (!multi)
    for (int k = 1; k < n_prob; ++k) eval_dispatch(request(k));
  for (int k = 0; k < n_prob; ++k)
    if (dst[k] != outs_host[k])
      EVB_CUDA(cudaMemcpyAsync(outs_host[k], dst[k], size_t(n_points) * es, cudaMemcpyDeviceToHost, st));
  EVB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

extern "C" {

int evb_evaluate_batch_host(evb_problem p, evb_scratch s, const void* X_host, int64_t n_points, int64_t ldx,
                            void* out_host) {
  return guarded([&] { host_eval(&p, 1, s, X_host, n_points, ldx, &out_host); });
}

int evb_evaluate_batch_problems(const evb_problem* problems, int n_problems, evb_scratch s, const void* X,
                                int64_t n_points, int64_t ldx, void* const* outs, void* stream) {
  return guarded([&] {
    require(problems != nullptr && n_problems >= 1 && outs != nullptr, "evaluate_batch_problems: null argument");
    std::vector<eval_request> rqs(static_cast<size_t>(n_problems));
    for (int k = 0; k < n_problems; ++k) {
      validate_eval(problems[k], s, n_points, ldx);
      if (problems[k]->p.dim != problems[0]->p.dim || problems[k]->p.dtype != problems[0]->p.dtype)
        throw invalid_argument("evaluate_batch_problems: problems differ in dimension or dtype");
      eval_request& rq = rqs[size_t(k)];
      rq.prob = &problems[k]->p;
      rq.scratch = s;
      rq.X = X;
      rq.n = n_points;
      rq.ldx = ldx;
      rq.out = outs[k];
      rq.ldo = n_points;
      rq.n_out = 1;
      rq.kinds[0] = problems[k]->p.kind;
      rq.biases[0] = problems[k]->p.bias;
      rq.stream = static_cast<cudaStream_t>(stream);
    }
    if (n_points == 0) return;
    if (multi_eligible(rqs.data(), n_problems) && gemm_eval_multi(rqs.data(), n_problems, X, ldx)) return;
    for (auto& rq : rqs) eval_dispatch(rq);
  });
}

int evb_evaluate_batch_host_many(const evb_problem* problems, int n_problems, evb_scratch s, const void* X_host,
                                 int64_t n_points, int64_t ldx, void* const* out_host) {
  return guarded([&] { host_eval(problems, n_problems, s, X_host, n_points, ldx, out_host); });
}

int evb_launch_count(void) { return last_launch_count(); }

}  // extern "C"
