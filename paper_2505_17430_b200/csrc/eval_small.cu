// eval_small.cu — evaluation paths other than the fused large-D GEMM, and the dispatcher.
//
//  * eval_small_kernel      small D (M fits in shared memory): base / hybrid problems with z
//                           accumulated in the reference's exact order (sequential k, separate
//                           mul and add: problems/batch.hpp:62-67, problems/instance.hpp:69-75)
//                           and the base value in the reference's row order, so results match
//                           the reference bit for bit up to libm transcendental ulps.
//  * eval_comp_small_kernel small-D compositions (problems/instance.hpp:116-174), one component
//                           rotation in shared memory at a time.
//  * eval_rows_kernel       finishes a z materialised in SoA layout by the GEMM (z-store mode):
//                           neighbour/prefix kinds, hybrids, composition components.
//  * comp_combine_kernel    composition weights + weighted sum for large D.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "evb_internal.cuh"
#include "evb_math.cuh"
#include "ptx.cuh"

namespace evb {

template <typename T>
void gemm_eval(const eval_request& rq, const void* X, int64_t ldx, bool zstore, T* zbuf, int64_t ldz,
               const T* shift, const void* rotation, int ldm, int P, int D);
bool fused_kinds_ok(int n, const int* kinds);

namespace {

thread_local int g_launches = 0;

template <typename T>
struct small_args {
  int P, D, S, PB;  // S: shared-memory row stride of M (odd in 8-byte units -> no bank conflicts)
  const T* X;
  int64_t ldx;
  const T* shift;
  const T* rot;
  const T* rot_t;  // M^T dense (device_problem::rot_t)
  int ld;
  int spec;
  const T* ell_w;
  const T* hyb_w;
  const int* perm;
  const int* sub_kinds;
  const int* chunk_sizes;
  int n_chunks;
  T bias;
  int n_out;
  int kinds[4];
  double biases[4];
  T* out;
  int64_t ldo;
  int scalar_trig;
};


// Stage a rows x cols block (global row stride ld) into shared memory (row stride S): eight
// independent loads in flight per thread — a plain one-load-per-iteration loop waited out the L2
// latency 40 times per thread at D = 100 (12 us of a 24 us evaluation).
template <typename T>
__device__ __forceinline__ void stage_rows(T* __restrict__ dst, int S, const T* __restrict__ src, int64_t ld, int rows,
                                           int cols) {
  const int n = rows * cols;
  for (int base = threadIdx.x; base < n; base += 8 * blockDim.x) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * blockDim.x;
      v[u] = idx < n ? __ldg(src + size_t(idx / cols) * ld + idx % cols) : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * blockDim.x;
      if (idx < n) dst[(idx / cols) * S + idx % cols] = v[u];
    }
  }
}

template <typename T>
__global__ void eval_small_kernel(const small_args<T> a) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  // layout: M^T (bulk copy, 16-byte padded) | s = x - o (PB x D) | z (PB x D) | mbarrier
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int D = a.D;
  const uint32_t mt_bytes = uint32_t((size_t(D) * D * sizeof(T) + 15) / 16 * 16);
  T* sMT = reinterpret_cast<T*>(smem_raw);
  T* sS = reinterpret_cast<T*>(smem_raw + mt_bytes);
  T* sZ = sS + size_t(a.PB) * D;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + ((mt_bytes + 2 * size_t(a.PB) * D * sizeof(T) + 7) / 8) * 8);
  const int b0 = blockIdx.x * a.PB;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one bulk copy of M^T, overlapped with forming x - o below
    ptx::mbar_arrive_expect_tx(bar, mt_bytes);
    ptx::bulk_load(sMT, a.rot_t, mt_bytes, bar);
  }
  for (int idx = threadIdx.x; idx < a.PB * D; idx += blockDim.x) {
    const int pb = idx / D, k = idx % D;
    const int b = b0 + pb;
    sS[idx] = b < a.P ? fop<T>::sub(a.X[size_t(b) * a.ldx + k], a.shift[k]) : T(0);
  }
  __syncthreads();
  ptx::mbar_wait(bar, 0);
  // z_i = sum_k M[i][k] * s_k in increasing k, product and sum rounded separately (the reference
  // order, problems/batch.hpp:62-67); thread per (individual, row i): lanes read consecutive
  // words of M^T, s_k is a broadcast; eight k per round with the loads ahead of the chain
  for (int idx = threadIdx.x; idx < a.PB * D; idx += blockDim.x) {
    const int pb = idx / D, i = idx % D;
    const T* mcol = sMT + i;
    const T* s = sS + pb * D;
    T acc = T(0);
    int k = 0;
    for (; k + 8 <= D; k += 8) {
      T mv[8], sv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        mv[u] = mcol[(k + u) * D];
        sv[u] = s[k + u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fop<T>::add(acc, fop<T>::mul(mv[u], sv[u]));
    }
    for (; k < D; ++k) acc = fop<T>::add(acc, fop<T>::mul(mcol[k * D], s[k]));
    sZ[idx] = acc;
  }
  __syncthreads();
  if (a.spec == SPEC_HYBRID) {
    for (int pb = threadIdx.x; pb < a.PB; pb += blockDim.x) {
      const int b = b0 + pb;
      if (b >= a.P) continue;
      const T v = hybrid_value<T>(a.perm, a.sub_kinds, a.chunk_sizes, a.n_chunks, a.hyb_w, sZ + pb * D, 1);
      a.out[b] = fop<T>::add(v, a.bias);
    }
    return;
  }
  for (int o = 0; o < a.n_out; ++o) {
    const int kind = a.kinds[o];
    if (kind_has_pre(kind)) {  // transcendental terms of every element in parallel (into sS)
      for (int e = threadIdx.x; e < a.PB * D; e += blockDim.x) {
        const T* zr = sZ + (e / D) * D;
        auto z = [&](int q) { return zr[q]; };
        sS[e] = a.scalar_trig ? base_pre_term<T, false>(kind, D, z, e % D) : base_pre_term<T, true>(kind, D, z, e % D);
      }
      __syncthreads();
    }
    for (int pb = threadIdx.x; pb < a.PB; pb += blockDim.x) {
      const int b = b0 + pb;
      if (b >= a.P) continue;
      const T* zrow = sZ + pb * D;
      const T* pe = sS + pb * D;
      auto z = [&](int i) { return zrow[i]; };
      auto pre = [&](int i) { return pe[i]; };
      const T v = a.scalar_trig ? base_value_pre<T, false>(kind, D, z, pre, a.ell_w)
                                : base_value_pre<T, true>(kind, D, z, pre, a.ell_w);
      a.out[o * a.ldo + b] = fop<T>::add(v, T(a.biases[o]));
    }
    __syncthreads();
  }
}

// ---- compositions ------------------------------------------------------------------------
template <typename T>
struct comp_args {
  int P, D, S, PB, n_comp, ld;
  const T* X;
  int64_t ldx;
  const T* shifts;  // n_comp x ld
  const T* rots;    // n_comp x D x ld
  const int* kinds;
  const double* sigma;
  const double* lambda;
  const double* cbias;
  const T* ell_w;
  T bias;
  T* out;
};

// Weighted sum of component values exactly as problems/instance.hpp:126-174.
template <typename T>
__device__ T comp_combine(int n, int D, const double* dist_sq, const T* fk, const double* sigma,
                          const double* lambda, const double* cbias) {
  double weights[8];
  int zero_count = 0;
  for (int k = 0; k < n; ++k) {
    if (dist_sq[k] == 0.0) {
      ++zero_count;
      weights[k] = -1.0;
    } else {
      const double sg = sigma[k];
      weights[k] = __dmul_rn(__ddiv_rn(1.0, __dsqrt_rn(dist_sq[k])),
                             exp(__ddiv_rn(-dist_sq[k], __dmul_rn(__dmul_rn(__dmul_rn(2.0, double(D)), sg), sg))));
    }
  }
  double wsum = 0.0;
  if (zero_count > 0) {
    for (int k = 0; k < n; ++k) weights[k] = weights[k] < 0.0 ? 1.0 : 0.0;
    wsum = double(zero_count);
  } else {
    for (int k = 0; k < n; ++k) wsum = __dadd_rn(wsum, weights[k]);
    if (wsum == 0.0) {
      int nearest = 0;
      for (int k = 1; k < n; ++k)
        if (dist_sq[k] < dist_sq[nearest]) nearest = k;
      weights[nearest] = 1.0;
      wsum = 1.0;
    }
  }
  double value = 0.0;
  for (int k = 0; k < n; ++k) {
    const double w = __ddiv_rn(weights[k], wsum);
    if (w == 0.0) continue;
    value = __dadd_rn(value, __dmul_rn(w, __dadd_rn(__dmul_rn(lambda[k], double(fk[k])), cbias[k])));
  }
  return T(value);
}

constexpr int kMaxComp = 8;

template <typename T>
__global__ void eval_comp_small_kernel(const comp_args<T> a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  T* sM = reinterpret_cast<T*>(smem_raw);
  T* sS = sM + size_t(a.D) * a.S;
  T* sZ = sS + size_t(a.PB) * a.D;
  double* sDist = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sZ + size_t(a.PB) * a.D) + 7) & ~uintptr_t(7));
  T* sF = reinterpret_cast<T*>(sDist + a.PB * kMaxComp);                // PB x n_comp
  const int b0 = blockIdx.x * a.PB;
  const int D = a.D;
  for (int c = 0; c < a.n_comp; ++c) {
    const T* rot = a.rots + size_t(c) * D * a.ld;
    const T* o = a.shifts + size_t(c) * a.ld;
    stage_rows<T>(sM, a.S, rot, a.ld, D, D);
    for (int idx = threadIdx.x; idx < a.PB * D; idx += blockDim.x) {
      const int pb = idx / D, k = idx % D;
      const int b = b0 + pb;
      sS[idx] = b < a.P ? fop<T>::sub(a.X[size_t(b) * a.ldx + k], o[k]) : T(0);
    }
    // dist^2 in double from the raw point (problems/instance.hpp:127-134)
    for (int pb = threadIdx.x; pb < a.PB; pb += blockDim.x) {
      const int b = b0 + pb;
      double d2 = 0.0;
      if (b < a.P)
        for (int j = 0; j < D; ++j) {
          const double dj = __dsub_rn(double(a.X[size_t(b) * a.ldx + j]), double(o[j]));
          d2 = __dadd_rn(d2, __dmul_rn(dj, dj));
        }
      sDist[pb * kMaxComp + c] = d2;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < a.PB * D; idx += blockDim.x) {
      const int pb = idx / D, i = idx % D;
      const T* mrow = sM + i * a.S;
      const T* s = sS + pb * D;
      T acc = T(0);
      for (int k = 0; k < D; ++k) acc = fop<T>::add(acc, fop<T>::mul(mrow[k], s[k]));
      sZ[idx] = acc;
    }
    __syncthreads();
    const int kind = a.kinds[c];
    if (kind_has_pre(kind)) {
      for (int e = threadIdx.x; e < a.PB * D; e += blockDim.x) {
        const T* zr = sZ + (e / D) * D;
        auto z = [&](int q) { return zr[q]; };
        sS[e] = base_pre_term<T, false>(kind, D, z, e % D);
      }
      __syncthreads();
    }
    for (int pb = threadIdx.x; pb < a.PB; pb += blockDim.x) {
      const T* zrow = sZ + pb * D;
      const T* pe = sS + pb * D;
      auto z = [&](int i) { return zrow[i]; };
      auto pre = [&](int i) { return pe[i]; };
      sF[pb * kMaxComp + c] = base_value_pre<T, false>(kind, D, z, pre, a.ell_w);
    }
    __syncthreads();
  }
  for (int pb = threadIdx.x; pb < a.PB; pb += blockDim.x) {
    const int b = b0 + pb;
    if (b >= a.P) continue;
    const T v = comp_combine<T>(a.n_comp, D, sDist + pb * kMaxComp, sF + pb * kMaxComp, a.sigma, a.lambda,
                                a.cbias);
    a.out[b] = fop<T>::add(v, a.bias);
  }
}

// ---- rows (z materialised by the GEMM, SoA z[i*ldz + b]) --------------------------------------
template <typename T>
struct rows_args {
  int P, D;
  const T* z;
  int64_t ldz;
  int mode;  // 0 base, 1 hybrid, 2 composition component value -> fk
  int n_out;
  int kinds[4];
  double biases[4];
  const T* ell_w;
  const T* hyb_w;
  const int* perm;
  const int* sub_kinds;
  const int* chunk_sizes;
  int n_chunks;
  T bias;
  T* out;
  int64_t ldo;
  int scalar_trig;
};

template <typename T>
__global__ void eval_rows_kernel(const rows_args<T> a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.P) return;
  const T* zcol = a.z + b;
  if (a.mode == 1) {
    const T v = hybrid_value<T>(a.perm, a.sub_kinds, a.chunk_sizes, a.n_chunks, a.hyb_w, zcol, a.ldz);
    a.out[b] = fop<T>::add(v, a.bias);
    return;
  }
  auto z = [&](int i) { return zcol[int64_t(i) * a.ldz]; };
  if (a.mode == 2) {
    a.out[b] = base_value_seq<T, false>(a.kinds[0], a.D, z, a.ell_w);
    return;
  }
  for (int o = 0; o < a.n_out; ++o) {
    const T v = a.scalar_trig ? base_value_seq<T, false>(a.kinds[o], a.D, z, a.ell_w)
                              : base_value_seq<T, true>(a.kinds[o], a.D, z, a.ell_w);
    a.out[o * a.ldo + b] = fop<T>::add(v, T(a.biases[o]));
  }
}

template <typename T>
__global__ void comp_combine_kernel(int P, int D, int n_comp, int ld, const T* X, int64_t ldx, const T* shifts,
                                    const T* fk /* n_comp x P */, const double* sigma, const double* lambda,
                                    const double* cbias, T bias, T* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P) return;
  double dist[kMaxComp];
  T f[kMaxComp];
  for (int c = 0; c < n_comp; ++c) {
    const T* o = shifts + size_t(c) * ld;
    double d2 = 0.0;
    for (int j = 0; j < D; ++j) {
      const double dj = __dsub_rn(double(X[size_t(b) * ldx + j]), double(o[j]));
      d2 = __dadd_rn(d2, __dmul_rn(dj, dj));
    }
    dist[c] = d2;
    f[c] = fk[size_t(c) * P + b];
  }
  out[b] = fop<T>::add(comp_combine<T>(n_comp, D, dist, f, sigma, lambda, cbias), bias);
}

template <typename T>
size_t small_smem(int D, int PB, bool comp) {
  const int S = (D % 2 == 1) ? D : D + 1;
  size_t bytes = (size_t(D) * S + 2 * size_t(PB) * D) * sizeof(T);
  if (comp) bytes += PB * kMaxComp * (sizeof(double) + sizeof(T)) + 16;
  else bytes += 32;  // base / hybrid: M^T padded to 16 bytes + the bulk-copy mbarrier
  return bytes;
}

constexpr size_t kSmallSmemMax = 200 * 1024;

// Individuals per block: as many as amortise staging M (up to 2048 / D), but never so many that
// fewer than two blocks per SM remain — a 180 x 100 batch in 9 blocks of 20 took 40 us, in 90
// blocks of 2 a few us (M is re-read from L2 per block, 80 KB at D = 100).
template <typename T>
int pick_pb(int D, int P, bool comp) {
  static int sms = [] {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
    return n;
  }();
  int pb = std::max(1, std::min(32, 2048 / std::max(D, 1)));
  pb = std::min(pb, std::max(1, (P + 2 * sms - 1) / (2 * sms)));
  while (pb > 1 && small_smem<T>(D, pb, comp) > kSmallSmemMax) --pb;
  return pb;
}

template <typename T>
bool small_fits(int D, bool comp) {
  // (the switch point predates the bulk-copy staging: measured against the M + x - o + z layout)
  const int S = (D % 2 == 1) ? D : D + 1;
  size_t legacy = (size_t(D) * S + 2 * size_t(D)) * sizeof(T);
  if (comp) legacy += kMaxComp * (sizeof(double) + sizeof(T)) + 16;
  return legacy <= kSmallSmemMax && D <= 160;
}

template <typename T>
void set_smem_attr(const void* kern, size_t bytes) {
  EVB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

// Big-D X must be TMA-legal: 16-byte aligned base and 16-byte multiple row pitch.
template <typename T>
const T* tma_legal_x(const eval_request& rq, int D, int64_t* ldx_out) {
  const uintptr_t base = reinterpret_cast<uintptr_t>(rq.X);
  if (base % 16 == 0 && (rq.ldx * int64_t(sizeof(T))) % 16 == 0) {
    *ldx_out = rq.ldx;
    return static_cast<const T*>(rq.X);
  }
  const int64_t ld = round_up(D, 16 / sizeof(T));
  evb_scratch_s* sc = rq.scratch;
  ensure_buffer(&sc->xpad, &sc->xpad_bytes, size_t(ld) * rq.n * sizeof(T), rq.stream);
  EVB_CUDA(cudaMemcpy2DAsync(sc->xpad, ld * sizeof(T), rq.X, rq.ldx * sizeof(T), D * sizeof(T), rq.n,
                             cudaMemcpyDeviceToDevice, rq.stream));
  *ldx_out = ld;
  return static_cast<const T*>(sc->xpad);
}

template <typename T>
void dispatch_t(const eval_request& rq_in) {
  // Only the fused fp64 GEMM consumes per-chunk gates (its producer waits column chunk by column
  // chunk); every other path waits for all of X before its first launch.
  const bool gated = gate_eligible(rq_in);
  eval_request rq = rq_in;
  if (rq.x_ready && !gated) {
    EVB_CUDA(cudaStreamWaitEvent(rq.stream, rq.x_ready, 0));
    rq.x_ready = nullptr;
    rq.kgate = nullptr;
  }
  const device_problem& pr = *rq.prob;
  const int P = int(rq.n);
  const int D = pr.dim;
  evb_scratch_s* sc = rq.scratch;
  const bool comp = pr.spec == SPEC_COMPOSITION;

  if (small_fits<T>(D, comp)) {
    const int PB = pick_pb<T>(D, P, comp);
    const size_t smem = small_smem<T>(D, PB, comp);
    const int threads = 256;
    const int blocks = (P + PB - 1) / PB;
    if (comp) {
      comp_args<T> a{};
      a.P = P; a.D = D; a.S = (D % 2 == 1) ? D : D + 1; a.PB = PB; a.n_comp = pr.n_comp; a.ld = pr.ld;
      a.X = static_cast<const T*>(rq.X); a.ldx = rq.ldx;
      a.shifts = static_cast<const T*>(pr.comp_shift); a.rots = static_cast<const T*>(pr.comp_rot);
      a.kinds = pr.comp_kinds; a.sigma = pr.comp_sigma; a.lambda = pr.comp_lambda; a.cbias = pr.comp_bias;
      a.ell_w = static_cast<const T*>(pr.ell_w); a.bias = T(pr.bias); a.out = static_cast<T*>(rq.out);
      set_smem_attr<T>(reinterpret_cast<const void*>(eval_comp_small_kernel<T>), smem);
      eval_comp_small_kernel<T><<<blocks, threads, smem, rq.stream>>>(a);
    } else {
      small_args<T> a{};
      a.P = P; a.D = D; a.S = (D % 2 == 1) ? D : D + 1; a.PB = PB;
      a.X = static_cast<const T*>(rq.X); a.ldx = rq.ldx;
      a.shift = static_cast<const T*>(pr.shift); a.rot = static_cast<const T*>(pr.rotation); a.ld = pr.ld;
      a.rot_t = static_cast<const T*>(pr.rot_t);
      if (!a.rot_t) throw runtime_error("evaluate_batch: small-D problem without its transposed rotation");
      a.spec = pr.spec; a.ell_w = static_cast<const T*>(pr.ell_w); a.hyb_w = static_cast<const T*>(pr.hyb_w);
      a.perm = pr.perm; a.sub_kinds = pr.sub_kinds; a.chunk_sizes = pr.chunk_sizes; a.n_chunks = pr.n_chunks;
      a.bias = T(pr.bias); a.n_out = rq.n_out;
      for (int o = 0; o < rq.n_out; ++o) { a.kinds[o] = rq.kinds[o]; a.biases[o] = rq.biases[o]; }
      a.out = static_cast<T*>(rq.out); a.ldo = rq.ldo; a.scalar_trig = rq.scalar_trig ? 1 : 0;
      set_smem_attr<T>(reinterpret_cast<const void*>(eval_small_kernel<T>), smem);
      EVB_CUDA(launch_pdl(eval_small_kernel<T>, dim3(blocks), dim3(threads), smem, rq.stream, a));
    }
    EVB_CUDA(cudaGetLastError());
    count_launch();
    return;
  }

  // ---- large D: TMA + tensor-core / FFMA GEMM ----
  int64_t ldx = 0;
  const T* X = tma_legal_x<T>(rq, D, &ldx);
  const int64_t ldz = round_up(P, 4);
  const int rows_threads = 128;
  const int rows_blocks = (P + rows_threads - 1) / rows_threads;

  if (pr.spec == SPEC_BASE && fused_kinds_ok(rq.n_out, rq.kinds)) {
    gemm_eval<T>(rq, X, ldx, false, nullptr, 0, static_cast<const T*>(pr.shift), pr.rotation, pr.ld, P, D);
    return;
  }
  ensure_buffer(&sc->zbuf, &sc->zbuf_bytes, size_t(D) * ldz * sizeof(T), rq.stream);
  T* z = static_cast<T*>(sc->zbuf);
  if (pr.spec != SPEC_COMPOSITION) {
    gemm_eval<T>(rq, X, ldx, true, z, ldz, static_cast<const T*>(pr.shift), pr.rotation, pr.ld, P, D);
    rows_args<T> a{};
    a.P = P; a.D = D; a.z = z; a.ldz = ldz; a.mode = pr.spec == SPEC_HYBRID ? 1 : 0; a.n_out = rq.n_out;
    for (int o = 0; o < rq.n_out; ++o) { a.kinds[o] = rq.kinds[o]; a.biases[o] = rq.biases[o]; }
    a.ell_w = static_cast<const T*>(pr.ell_w); a.hyb_w = static_cast<const T*>(pr.hyb_w);
    a.perm = pr.perm; a.sub_kinds = pr.sub_kinds; a.chunk_sizes = pr.chunk_sizes; a.n_chunks = pr.n_chunks;
    a.bias = T(pr.bias); a.out = static_cast<T*>(rq.out); a.ldo = rq.ldo; a.scalar_trig = rq.scalar_trig ? 1 : 0;
    eval_rows_kernel<T><<<rows_blocks, rows_threads, 0, rq.stream>>>(a);
    EVB_CUDA(cudaGetLastError());
    count_launch();
    return;
  }
  // composition, large D: per component z-store GEMM + component values, then combine
  ensure_buffer(reinterpret_cast<void**>(&sc->acc), &sc->acc_bytes, size_t(pr.n_comp) * P * sizeof(T), rq.stream);
  T* fk = reinterpret_cast<T*>(sc->acc);
  const std::vector<int>& kinds = pr.h_comp_kinds;
  for (int c = 0; c < pr.n_comp; ++c) {
    const T* shift = static_cast<const T*>(pr.comp_shift) + size_t(c) * pr.ld;
    const T* rot = static_cast<const T*>(pr.comp_rot) + size_t(c) * D * pr.ld;
    gemm_eval<T>(rq, X, ldx, true, z, ldz, shift, rot, pr.ld, P, D);
    rows_args<T> a{};
    a.P = P; a.D = D; a.z = z; a.ldz = ldz; a.mode = 2; a.n_out = 1; a.kinds[0] = kinds[c];
    a.ell_w = static_cast<const T*>(pr.ell_w); a.out = fk + size_t(c) * P; a.ldo = P;
    eval_rows_kernel<T><<<rows_blocks, rows_threads, 0, rq.stream>>>(a);
    EVB_CUDA(cudaGetLastError());
    count_launch();
  }
  comp_combine_kernel<T><<<rows_blocks, rows_threads, 0, rq.stream>>>(
      P, D, pr.n_comp, pr.ld, X, ldx, static_cast<const T*>(pr.comp_shift), fk, pr.comp_sigma, pr.comp_lambda,
      pr.comp_bias, T(pr.bias), static_cast<T*>(rq.out));
  EVB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace

void count_launch(int n) { g_launches += n; }
int last_launch_count() { return g_launches; }

bool gate_eligible(const eval_request& rq) {
  return rq.prob->dtype == EVB_F64 && rq.prob->spec == SPEC_BASE && !small_fits<double>(rq.prob->dim, false) &&
         fused_kinds_ok(rq.n_out, rq.kinds) && reinterpret_cast<uintptr_t>(rq.X) % 16 == 0 &&
         (rq.ldx * 8) % 16 == 0 && !(std::getenv("EVB_F64_KERNEL") && std::string(std::getenv("EVB_F64_KERNEL")) == "persistent");
}

bool multi_eligible(const eval_request* rqs, int np) {
  if (np < 2 || np > 3 || (std::getenv("EVB_MULTI") && std::string(std::getenv("EVB_MULTI")) == "0")) return false;
  for (int g = 0; g < np; ++g) {
    eval_request r = rqs[g];
    r.X = rqs[0].X;
    r.ldx = rqs[0].ldx;
    if (!gate_eligible(r) || r.n_out != 1 || rqs[g].prob->dim != rqs[0].prob->dim) return false;
  }
  return true;
}

// the small-D kernel (exact order) evaluates this base / hybrid problem (the persistent DE
// generations reproduce its arithmetic, de.cu)
bool eval_small_path(const device_problem& p) {
  return p.spec != SPEC_COMPOSITION && (p.dtype == EVB_F64 ? small_fits<double>(p.dim, false)
                                                           : small_fits<float>(p.dim, false));
}

void eval_dispatch(const eval_request& rq) {
  if (rq.n == 0) return;
  if (rq.prob->dtype == EVB_F64) dispatch_t<double>(rq);
  else dispatch_t<float>(rq);
}

}  // namespace evb
