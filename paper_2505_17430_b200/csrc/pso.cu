// pso.cu — synchronous PSO generation on the device (K7): neighbourhood argmin, velocity / position
// update with bound handling, batched evaluation (K1/K2) and strict-< personal-best update.
//
// Reference pieces (pso/): gbest_topology::neighbor_best pso/topology.hpp:28-34 (strict <, ties to
// the lowest index), lbest_topology::neighbor_best :44-54 (ring {i-1, i, i+1}, ties to the lowest
// index), standard_update::apply pso/update.hpp:66-74 (r1, r2 drawn per gene, interleaved), move
// and bound rule pso/engine.hpp:66-75, pbest update :78-79.
//
// Deviation: the stock pso_engine is asynchronous — particle i sees pbests already
// updated by particles < i in the same generation.  A data-parallel GPU generation is
// synchronous: every particle reads the start-of-generation pbests.  BASELINE config 3 asks for
// this synchronous variant with a velocity clamp (|v| <= vmax, applied after the velocity rule,
// before the move); the CPU oracle is the synchronous driver built from the same reference pieces.
//
// Draws: particle i of generation g uses Philox sub-stream (g << 32) | i; gene j takes words 2j
// (r1) and 2j+1 (r2) — exactly one Philox block per gene.  WORDS mode consumes the list
// particle-major, gene-minor, r1 before r2 (the reference's per-particle order).
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "evb_internal.cuh"
#include "evb_math.cuh"
#include "ptx.cuh"
#include "rng.cuh"

struct evb_pso_s {
  evb::phase_timer phases;  // neighbourhood best, velocity/position update, evaluation, personal best
  int dtype = EVB_F64;
  int P = 0, D = 0;
  int topology = EVB_TOPO_GBEST;
  int update = EVB_UPD_STANDARD;
  double w = 0, c1 = 0, c2 = 0, vmax = 0, attraction = 0;
  int64_t ldb = 0;
  void* pbest = nullptr;      // P x ldb
  void* pbest_fit = nullptr;  // P
  void* fit_new = nullptr;    // P (evaluation of the moved swarm)
  int* nb = nullptr;          // P: neighbourhood bests used by the last generation
  int* nb_next = nullptr;     // P: the next generation's, written by the personal-best kernel
  int nb_valid = 0;           // nb_next matches pbest_fit (cleared by every other writer of pbest_fit)
  int prepared = 0;
  uint32_t last_gen = 0;
  evb_scratch_s* eval_scratch = nullptr;
  evb_recorder_s* rec = nullptr;  // attached best-so-far recorder (may be null)
  int rec_run = 0;
};

namespace evb {
namespace {

// (fitness, index) lexicographic minimum — strict <, ties to the lower index
template <typename T>
__device__ __forceinline__ void argmin_merge(T& f, int& i, T f2, int i2) {
  if (f2 < f || (!(f < f2) && !(f2 < f) && i2 < i) || (i < 0 && i2 >= 0)) {
    f = f2;
    i = i2;
  }
}

// gbest: one block reduces all pbests; writes nb[i] = best for all i.  pso/topology.hpp:28-34 is
// the sequential scan best = 0; for i: if f[i] < f[best] best = i.  Its closed form: index 0 when
// f[0] is NaN (nothing compares < NaN), else the lexicographic (f, i) minimum over the non-NaN
// entries (a NaN never satisfies <).  NaN entries therefore stay out of the shuffle tree, which
// keeps the merge a strict weak order (independent of the tree's shape).
template <typename T>
__global__ void pso_gbest_kernel(const T* __restrict__ pf, int P, int* nb) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  __shared__ T sf[32];
  __shared__ int si[32];
  T bf = T(0);
  int bi = -1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const T fi = pf[i];
    if (!isnan(fi)) argmin_merge(bf, bi, fi, i);
  }
  for (int off = 16; off > 0; off >>= 1) {
    const T of = __shfl_xor_sync(0xffffffffu, bf, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (oi >= 0) argmin_merge(bf, bi, of, oi);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sf[w] = bf;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    bf = l < nw ? sf[l] : T(0);
    bi = l < nw ? si[l] : -1;
    for (int off = 16; off > 0; off >>= 1) {
      const T of = __shfl_xor_sync(0xffffffffu, bf, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oi >= 0) argmin_merge(bf, bi, of, oi);
    }
    if (l == 0) si[0] = (bi < 0 || isnan(pf[0])) ? 0 : bi;
  }
  __syncthreads();
  const int best = si[0];
  for (int i = threadIdx.x; i < P; i += blockDim.x) nb[i] = best;
}

// ring of width one (pso/topology.hpp:44-54), offsets -1, 0, +1 in that order: each particle's
// pbest fitness is loaded once; the left / right neighbours' values come from the adjacent lanes
// (warp shuffles), global loads only at warp edges and where the ring wraps
template <typename T>
__global__ void pso_ring_kernel(const T* __restrict__ pf, int P, int* nb) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const T f = i < P ? pf[i] : T(0);
  T fl = __shfl_up_sync(0xffffffffu, f, 1);
  T fr = __shfl_down_sync(0xffffffffu, f, 1);
  if (i >= P) return;
  const int il = i == 0 ? P - 1 : i - 1, ir = i + 1 == P ? 0 : i + 1;
  if (lane == 0 || il != i - 1) fl = pf[il];
  if (lane == 31 || ir != i + 1) fr = pf[ir];
  // lexicographic (fitness, index) minimum over the candidates in the reference's order
  int best = il;
  T bf = fl;
  if (f < bf || (f == bf && i < best)) {
    best = i;
    bf = f;
  }
  if (fr < bf || (fr == bf && ir < best)) best = ir;
  nb[i] = best;
}

template <typename T>
struct pso_dev {
  int P, D;
  T* x;
  int64_t ldx;
  T* v;
  int64_t ldv;
  const T* pb;
  int64_t ldb;
  const int* nb;
  T w, c1, c2, vmax, c;
  int clamp;
  T lb, ub;
  word_source src;
  const uint32_t* gen_ptr;
  int64_t base;  // WORDS: list position of this generation's first word
  int* overflow;
};

// K7 update: grid (gene blocks, particles); one Philox block per gene gives (r1, r2).
// v = w v + c1 r1 (p - x) + c2 r2 (l - x)  evaluated left to right (pso/update.hpp:71-72),
// clamp, move, bound rule (pso/engine.hpp:66-75).  Pure streaming: 5 s P D bytes.
template <typename T>
__global__ void __launch_bounds__(256) pso_update_kernel(const pso_dev<T> d) {
  using F = fop<T>;
  const int i = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.D) return;
  uint64_t w0, w1;
  if (d.src.mode == RNG_PHILOX) {
    philox_pair(d.src.key, (uint64_t(*d.gen_ptr) << 32) | uint32_t(i), uint64_t(j), w0, w1);
  } else {
    const int64_t n = d.base + (int64_t(i) * d.D + j) * 2;
    w0 = word_at(d.src, 0, n, d.overflow);
    w1 = word_at(d.src, 0, n + 1, d.overflow);
  }
  const T r1 = T(u01_of(w0)), r2 = T(u01_of(w1));
  T* xr = d.x + size_t(i) * d.ldx;
  T* vr = d.v + size_t(i) * d.ldv;
  const T x = xr[j];
  const T p = d.pb[size_t(i) * d.ldb + j];
  const T l = d.pb[size_t(d.nb[i]) * d.ldb + j];
  T v = F::add(F::add(F::mul(d.w, vr[j]), F::mul(F::mul(d.c1, r1), F::sub(p, x))),
               F::mul(F::mul(d.c2, r2), F::sub(l, x)));
  if (d.clamp) {
    if (v > d.vmax) v = d.vmax;
    if (v < -d.vmax) v = -d.vmax;
  }
  T xn = F::add(x, v);
  if (xn < d.lb) {
    xn = d.lb;
    v = F::mul(T(-0.5), v);
  } else if (xn > d.ub) {
    xn = d.ub;
    v = F::mul(T(-0.5), v);
  }
  xr[j] = xn;
  vr[j] = v;
}

// K7 with VEC genes per thread (vector loads / stores of x, v, pbest and the neighbour's pbest):
// fewer, wider memory instructions per byte than one gene per thread — used when every row is
// 16-byte aligned.  Same arithmetic and draws as pso_update_kernel.
template <typename T, int VEC>
__global__ void __launch_bounds__(128) pso_update_vec_kernel(const pso_dev<T> d) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  using F = fop<T>;
  using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  const int i = blockIdx.y;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (j0 >= d.D) return;
  T* xr = d.x + size_t(i) * d.ldx;
  T* vr = d.v + size_t(i) * d.ldv;
  const T* pr = d.pb + size_t(i) * d.ldb;
  const T* lr = d.pb + size_t(d.nb[i]) * d.ldb;
  // 16-byte aligned so the vector views below stay legal even if the arrays spill to local memory
  alignas(16) T x[VEC];
  alignas(16) T v[VEC];
  alignas(16) T pb[VEC];
  alignas(16) T lb_[VEC];
  constexpr int NV = VEC * int(sizeof(T)) / 16;  // 16-byte vectors per array
  if (j0 + VEC <= d.D) {
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int e = u * (16 / int(sizeof(T)));
      *reinterpret_cast<V*>(x + e) = *reinterpret_cast<const V*>(xr + j0 + e);
      *reinterpret_cast<V*>(v + e) = *reinterpret_cast<const V*>(vr + j0 + e);
      *reinterpret_cast<V*>(pb + e) = __ldg(reinterpret_cast<const V*>(pr + j0 + e));
      *reinterpret_cast<V*>(lb_ + e) = __ldg(reinterpret_cast<const V*>(lr + j0 + e));
    }
  } else {
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const int j = j0 + q < d.D ? j0 + q : d.D - 1;
      x[q] = xr[j];
      v[q] = vr[j];
      pb[q] = pr[j];
      lb_[q] = lr[j];
    }
  }
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(i);
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    const int j = j0 + q;
    uint64_t w0, w1;
    if (d.src.mode == RNG_PHILOX) {
      philox_pair(d.src.key, ctr_hi, uint64_t(j), w0, w1);
    } else {
      const int64_t n = d.base + (int64_t(i) * d.D + j) * 2;
      w0 = j < d.D ? word_at(d.src, 0, n, d.overflow) : 0;
      w1 = j < d.D ? word_at(d.src, 0, n + 1, d.overflow) : 0;
    }
    const T r1 = T(u01_of(w0)), r2 = T(u01_of(w1));
    T vv = F::add(F::add(F::mul(d.w, v[q]), F::mul(F::mul(d.c1, r1), F::sub(pb[q], x[q]))),
                  F::mul(F::mul(d.c2, r2), F::sub(lb_[q], x[q])));
    if (d.clamp) {
      if (vv > d.vmax) vv = d.vmax;
      if (vv < -d.vmax) vv = -d.vmax;
    }
    T xn = F::add(x[q], vv);
    if (xn < d.lb) {
      xn = d.lb;
      vv = F::mul(T(-0.5), vv);
    } else if (xn > d.ub) {
      xn = d.ub;
      vv = F::mul(T(-0.5), vv);
    }
    x[q] = xn;
    v[q] = vv;
  }
  if (j0 + VEC <= d.D) {
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int e = u * (16 / int(sizeof(T)));
      *reinterpret_cast<V*>(xr + j0 + e) = *reinterpret_cast<const V*>(x + e);
      *reinterpret_cast<V*>(vr + j0 + e) = *reinterpret_cast<const V*>(v + e);
    }
  } else {
#pragma unroll
    for (int q = 0; q < VEC; ++q)
      if (j0 + q < d.D) {
        xr[j0 + q] = x[q];
        vr[j0 + q] = v[q];
      }
  }
}

// SPSO2011 spherical rule (pso/update.hpp:81-114, sample_in_ball :24-43), one block per particle.
// Per gene (parallel): p* = x + c (p - x), l* = x + c (l - x), centre G = (x + p* [+ l*]) / 2|3,
// the normal g_j (Box-Muller on words 2j, 2j+1); then the two double sums |G - x|^2 and |g|^2 in
// increasing j (sequential, the reference's order), u = word 2D, scale = r u^(1/D) / |g|, and
// v = w v + (G + T(scale g_j) - x).  Draws: 2D + 1 words per particle.
template <typename T>
__global__ void pso_spherical_kernel(const pso_dev<T> d) {
  using F = fop<T>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  double* rad = reinterpret_cast<double*>(smem_raw);  // D
  double* nrm = rad + d.D;                            // D
  T* cen = reinterpret_cast<T*>(nrm + d.D);           // D
  T* gt = cen + d.D;                                  // D: T(g_j)
  __shared__ double s_scale;
  __shared__ double s_sum[2];
  const int i = blockIdx.x;
  const int nbi = d.nb[i];
  const bool self = nbi == i;
  const T* xr = d.x + size_t(i) * d.ldx;
  const T* pr = d.pb + size_t(i) * d.ldb;
  const T* lr = d.pb + size_t(nbi) * d.ldb;
  const uint64_t ctr_hi = (uint64_t(*d.gen_ptr) << 32) | uint32_t(i);
  const int64_t base = d.base + int64_t(i) * (2 * int64_t(d.D) + 1);  // WORDS
  for (int j = threadIdx.x; j < d.D; j += blockDim.x) {
    const T x = xr[j];
    const T ps = F::add(x, F::mul(d.c, F::sub(pr[j], x)));
    T g;
    if (self) {
      g = F::div(F::add(x, ps), T(2));
    } else {
      const T ls = F::add(x, F::mul(d.c, F::sub(lr[j], x)));
      g = F::div(F::add(F::add(x, ps), ls), T(3));
    }
    cen[j] = g;
    const double dd = double(F::sub(g, x));
    rad[j] = __dmul_rn(dd, dd);
    uint64_t w0, w1;
    if (d.src.mode == RNG_PHILOX) {
      philox_pair(d.src.key, ctr_hi, uint64_t(j), w0, w1);
    } else {
      w0 = word_at(d.src, 0, base + 2 * j, d.overflow);
      w1 = word_at(d.src, 0, base + 2 * j + 1, d.overflow);
    }
    // rng_stream::normal(0, 1) (core/rng.hpp:96-101)
    const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u01pos_of(w0))));
    const double gn = __dadd_rn(0.0, __dmul_rn(__dmul_rn(1.0, r), cos(__dmul_rn(2.0 * 3.14159265358979323846, u01_of(w1)))));
    gt[j] = T(gn);
    nrm[j] = __dmul_rn(gn, gn);
  }
  __syncthreads();
  if (threadIdx.x == 0 || threadIdx.x == 32) {  // two sequential sums, one per warp
    const double* a = threadIdx.x == 0 ? rad : nrm;
    double acc = 0.0;
    for (int j = 0; j < d.D; ++j) acc = __dadd_rn(acc, a[j]);
    s_sum[threadIdx.x == 0 ? 0 : 1] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t wu = d.src.mode == RNG_PHILOX ? philox_word(d.src.key, ctr_hi, uint64_t(2 * d.D))
                                                 : word_at(d.src, 0, base + 2 * d.D, d.overflow);
    const double u = u01_of(wu);
    const double norm = __dsqrt_rn(s_sum[1]);
    const double radius = __dsqrt_rn(s_sum[0]);
    s_scale = norm > 0.0 ? __ddiv_rn(__dmul_rn(radius, pow(u, __ddiv_rn(1.0, double(d.D)))), norm) : 0.0;
  }
  __syncthreads();
  const double scale = s_scale;
  T* xw = d.x + size_t(i) * d.ldx;
  T* vw = d.v + size_t(i) * d.ldv;
  for (int j = threadIdx.x; j < d.D; j += blockDim.x) {
    const T x = xw[j];
    const T sample = F::add(cen[j], T(__dmul_rn(scale, double(gt[j]))));
    T v = F::add(F::mul(d.w, vw[j]), F::sub(sample, x));
    if (d.clamp) {
      if (v > d.vmax) v = d.vmax;
      if (v < -d.vmax) v = -d.vmax;
    }
    T xn = F::add(x, v);
    if (xn < d.lb) {
      xn = d.lb;
      v = F::mul(T(-0.5), v);
    } else if (xn > d.ub) {
      xn = d.ub;
      v = F::mul(T(-0.5), v);
    }
    xw[j] = xn;
    vw[j] = v;
  }
}

// pbest update (pso/engine.hpp:78-79): strict <, copy the moved particle; also publishes the
// particle's fitness into the caller's fitness vector.
template <typename T>
__global__ void pso_pbest_kernel(const T* __restrict__ x, int64_t ldx, const T* __restrict__ fnew, T* fit, T* pb,
                                 int64_t ldb, T* pbf, int D, uint32_t* gen) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  const int i = blockIdx.x;
  if (i == 0 && threadIdx.x == 0) *gen += 1u;  // the update kernel (last reader) has finished
  const T f = fnew[i];
  if (threadIdx.x == 0) fit[i] = f;
  if (!(f < pbf[i])) return;
  for (int j = threadIdx.x; j < D; j += blockDim.x) pb[size_t(i) * ldb + j] = x[size_t(i) * ldx + j];
  __syncthreads();
  if (threadIdx.x == 0) pbf[i] = f;
}

// Personal bests after the evaluation AND the next generation's neighbourhood bests in one launch
// (the generation boundary costs one dependent launch less).  Block i refreshes particle i exactly
// as pso_pbest_kernel; the neighbourhood minima need every particle's refreshed pbest fitness,
// which block i forms itself as pfn(j) = fnew[j] < pbf[j] ? fnew[j] : pbf[j] — the same value
// whether block j has stored its pbf[j] yet or not (old pbf: the refresh rule; new pbf: it equals
// fnew[j] or was left alone), so no grid-wide ordering is needed.  Ring: block i's thread 0, the
// candidates and ties of pso_ring_kernel.  gbest: block 0 scans all particles with
// pso_gbest_kernel's rule (index 0 when pfn(0) is NaN, else the (fitness, index) minimum over the
// non-NaN entries) and writes every nb entry.
template <typename T>
__global__ void pso_pbest_nb_kernel(const T* __restrict__ x, int64_t ldx, const T* __restrict__ fnew, T* fit, T* pb,
                                    int64_t ldb, T* pbf, int D, int P, int topology, int* nb, uint32_t* gen) {
  ptx::griddep_wait();  // PDL (launch_pdl): predecessor data first
  ptx::griddep_launch_dependents();
  const int i = blockIdx.x;
  if (i == 0 && threadIdx.x == 0) *gen += 1u;  // the update kernel (last reader) has finished
  auto pfn = [&](int j) {
    const T f = fnew[j], q = __ldcg(pbf + j);
    return f < q ? f : q;
  };
  __shared__ T sf[32];
  __shared__ int si[32];
  if (topology == EVB_TOPO_GBEST) {
    if (i == 0) {
      T bf = T(0);
      int bi = -1;
      for (int j0 = threadIdx.x; j0 < P; j0 += 4 * blockDim.x) {  // four particles' loads in flight
        T fj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * blockDim.x;
          fj[u] = j < P ? pfn(j) : T(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * blockDim.x;
          if (j < P && !isnan(fj[u])) argmin_merge(bf, bi, fj[u], j);
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const T of = __shfl_xor_sync(0xffffffffu, bf, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi >= 0) argmin_merge(bf, bi, of, oi);
      }
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      if (l == 0) {
        sf[w] = bf;
        si[w] = bi;
      }
      __syncthreads();
      if (w == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        bf = l < nw ? sf[l] : T(0);
        bi = l < nw ? si[l] : -1;
        for (int off = 16; off > 0; off >>= 1) {
          const T of = __shfl_xor_sync(0xffffffffu, bf, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (oi >= 0) argmin_merge(bf, bi, of, oi);
        }
        if (l == 0) si[0] = (bi < 0 || isnan(pfn(0))) ? 0 : bi;
      }
      __syncthreads();
      const int best = si[0];
      for (int j = threadIdx.x; j < P; j += blockDim.x) nb[j] = best;
    }
  } else if (threadIdx.x == 0) {
    const int il = i == 0 ? P - 1 : i - 1, ir = i + 1 == P ? 0 : i + 1;
    const T fl = pfn(il), f0 = pfn(i), fr = pfn(ir);
    int best = il;
    T bf = fl;
    if (f0 < bf || (f0 == bf && i < best)) {
      best = i;
      bf = f0;
    }
    if (fr < bf || (fr == bf && ir < best)) best = ir;
    nb[i] = best;
  }
  const T f = fnew[i];
  if (threadIdx.x == 0) fit[i] = f;
  if (!(f < pbf[i])) return;  // (block-uniform: pbf[i] is written by this block only, below)
  for (int j = threadIdx.x; j < D; j += blockDim.x) pb[size_t(i) * ldb + j] = x[size_t(i) * ldx + j];
  __syncthreads();
  if (threadIdx.x == 0) pbf[i] = f;
}

template <typename T>
__global__ void copy_rows_kernel(const T* src, int64_t lds, T* dst, int64_t ldd, int D) {
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < D; j += blockDim.x) dst[size_t(i) * ldd + j] = src[size_t(i) * lds + j];
}

// velocities ~ U[lo, hi]: gene-positional words (sub-stream kSubInit + 1 of the current generation)
template <typename T>
__global__ void init_uniform_kernel(T* a, int64_t lda, int P, int D, double lo, double hi, word_source src,
                                    uint64_t ctr_hi, int64_t base, int* overflow) {
  const int64_t n = int64_t(P) * D;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t w = word_at(src, ctr_hi, base + e, overflow);
    a[(e / D) * lda + (e % D)] = T(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u01_of(w))));
  }
}

}  // namespace
int64_t words_cursor(evb_rng_s* r, cudaStream_t st);
void words_advance(evb_rng_s* r, int64_t to, cudaStream_t st);
namespace {

template <typename T>
void generation_t(evb_pso_s* s, const device_problem* prob, evb_scratch_s* sc, void* X, int64_t ldx, void* V,
                  int64_t ldv, void* fit, double lb, double ub, evb_rng_s* r, cudaStream_t st) {
  const T* pf = static_cast<const T*>(s->pbest_fit);
  s->phases.begin(st);
  // the last generation's personal-best kernel already formed this generation's neighbourhood
  // bests (EVB_PSO_FUSE_NB=0 keeps the separate kernels, A/B)
  static const bool fuse_nb = !(std::getenv("EVB_PSO_FUSE_NB") && std::atoi(std::getenv("EVB_PSO_FUSE_NB")) == 0);
  if (fuse_nb && s->nb_valid) {
    std::swap(s->nb, s->nb_next);
  } else {
    if (s->topology == EVB_TOPO_GBEST)
      EVB_CUDA(launch_pdl(pso_gbest_kernel<T>, dim3(1), dim3(1024), 0, st, pf, s->P, s->nb));
    else EVB_CUDA(launch_pdl(pso_ring_kernel<T>, dim3((s->P + 255) / 256), dim3(256), 0, st, pf, s->P, s->nb));
    count_launch();
  }
  s->nb_valid = 0;
  s->phases.mark(st);
  pso_dev<T> d{};
  d.P = s->P;
  d.D = s->D;
  d.x = static_cast<T*>(X);
  d.ldx = ldx;
  d.v = static_cast<T*>(V);
  d.ldv = ldv;
  d.pb = static_cast<const T*>(s->pbest);
  d.ldb = s->ldb;
  d.nb = s->nb;
  d.w = T(s->w);
  d.c1 = T(s->c1);
  d.c2 = T(s->c2);
  d.vmax = T(s->vmax);
  d.c = T(s->attraction);
  d.clamp = s->vmax > 0 ? 1 : 0;
  d.lb = T(lb);
  d.ub = T(ub);
  d.src = word_source{r->mode, r->key, r->d_words, r->n_words};
  d.gen_ptr = r->d_gen;
  d.overflow = r->d_overflow;
  if (r->mode == RNG_WORDS) d.base = words_cursor(r, st);
  int64_t words_per_particle = 2 * int64_t(s->D);
  if (s->update == EVB_UPD_SPHERICAL) {
    const size_t smem = size_t(s->D) * (2 * sizeof(double) + 2 * sizeof(T));
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      EVB_CUDA(cudaFuncSetAttribute(pso_spherical_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr = smem;
    }
    const int threads = std::max(64, std::min(256, int(round_up(s->D, 32))));  // warps 0 and 1 run the two sums
    pso_spherical_kernel<T><<<s->P, threads, smem, st>>>(d);
    words_per_particle += 1;
  } else {
    // four doubles / eight floats per thread: two 16-byte vectors per array and four or eight
    // independent Philox chains in flight (measured 120 -> 115 us at P = 16384, D = 1000)
    constexpr int VEC = sizeof(T) == 8 ? 4 : 8;
    const bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0 && reinterpret_cast<uintptr_t>(V) % 16 == 0 &&
                         (ldx * sizeof(T)) % 16 == 0 && (ldv * sizeof(T)) % 16 == 0 &&
                         (s->ldb * sizeof(T)) % 16 == 0;
    if (aligned) {
      dim3 grid(unsigned((s->D + 128 * VEC - 1) / (128 * VEC)), unsigned(s->P));
      EVB_CUDA(launch_pdl(pso_update_vec_kernel<T, VEC>, grid, dim3(128), 0, st, d));
    } else {
      dim3 grid((s->D + 255) / 256, s->P);
      pso_update_kernel<T><<<grid, 256, 0, st>>>(d);
    }
  }
  count_launch();
  EVB_CUDA(cudaGetLastError());
  if (r->mode == RNG_WORDS) words_advance(r, d.base + int64_t(s->P) * words_per_particle, st);
  s->phases.mark(st);
  eval_request rq{};
  rq.prob = prob;
  rq.scratch = sc;
  rq.X = X;
  rq.n = s->P;
  rq.ldx = ldx;
  rq.out = s->fit_new;
  rq.ldo = s->P;
  rq.n_out = 1;
  rq.kinds[0] = prob->kind;
  rq.biases[0] = prob->bias;
  rq.stream = st;
  rq.scalar_trig = true;
  eval_dispatch(rq);
  if (s->rec) recorder_observe(s->rec, s->rec_run, s->fit_new, s->P, st);  // particles in i (FE) order
  s->phases.mark(st);
  if (fuse_nb) {
    EVB_CUDA(launch_pdl(pso_pbest_nb_kernel<T>, dim3(s->P), dim3(std::min(256, int(round_up(s->D, 32)))), 0, st,
                        static_cast<const T*>(X), ldx, static_cast<const T*>(s->fit_new), static_cast<T*>(fit),
                        static_cast<T*>(s->pbest), s->ldb, static_cast<T*>(s->pbest_fit), s->D, s->P, s->topology,
                        s->nb_next, r->d_gen));
    s->nb_valid = 1;
  } else {
    EVB_CUDA(launch_pdl(pso_pbest_kernel<T>, dim3(s->P), dim3(std::min(256, int(round_up(s->D, 32)))), 0, st,
                        static_cast<const T*>(X), ldx, static_cast<const T*>(s->fit_new), static_cast<T*>(fit),
                        static_cast<T*>(s->pbest), s->ldb, static_cast<T*>(s->pbest_fit), s->D, r->d_gen));
  }
  count_launch();
  s->phases.mark(st);
  EVB_CUDA(cudaGetLastError());
  s->last_gen = r->gen;
  r->gen++;
}

}  // namespace

int64_t words_cursor(evb_rng_s* r, cudaStream_t st) {
  int64_t c = 0;
  EVB_CUDA(cudaMemcpyAsync(&c, r->d_cursor, sizeof(c), cudaMemcpyDeviceToHost, st));
  EVB_CUDA(cudaStreamSynchronize(st));
  return c;
}
void words_advance(evb_rng_s* r, int64_t to, cudaStream_t st) {
  EVB_CUDA(cudaMemcpyAsync(r->d_cursor, &to, sizeof(to), cudaMemcpyHostToDevice, st));
  EVB_CUDA(cudaStreamSynchronize(st));
  if (to > r->n_words) {
    int one = 1;
    EVB_CUDA(copy_h2d_now(r->d_overflow, &one, sizeof(int)));
  }
}

}  // namespace evb

using namespace evb;

extern "C" {

int evb_pso_create(int dtype, const evb_pso_config* c, int pop_size, int dim, evb_pso* out) {
  return guarded([&] {
    require(dtype == EVB_F32 || dtype == EVB_F64, "pso: dtype must be EVB_F32 or EVB_F64");
    require(c != nullptr && out != nullptr, "pso: null config or output handle");
    require(c->topology == EVB_TOPO_GBEST || c->topology == EVB_TOPO_LBEST_RING,
            "pso builder: unknown topology strategy (GPU kernels: gbest, lbest_ring)");
    require(c->update == EVB_UPD_STANDARD || c->update == EVB_UPD_SPHERICAL,
            "pso builder: unknown update strategy (GPU kernels: standard, spherical)");
    if (c->update == EVB_UPD_SPHERICAL)
      require(size_t(dim) * (2 * 8 + 2 * (dtype == EVB_F64 ? 8 : 4)) <= 200 * 1024,
              "pso: spherical update keeps 4 rows per particle in shared memory (dim <= 6400)");
    require(pop_size >= 1 && dim >= 1, "pso: pop_size and dim must be positive");
    auto* s = new evb_pso_s();
    try {
      s->dtype = dtype;
      s->P = pop_size;
      s->D = dim;
      s->topology = c->topology;
      s->update = c->update;
      s->w = c->inertia;
      s->c1 = c->cognitive;
      s->c2 = c->social;
      s->vmax = c->vmax;
      s->attraction = c->attraction;
      const size_t es = dtype == EVB_F64 ? 8 : 4;
      s->ldb = round_up(dim, 16 / int64_t(es));
      EVB_CUDA(cudaMalloc(&s->pbest, es * s->ldb * pop_size));
      EVB_CUDA(cudaMalloc(&s->pbest_fit, es * pop_size));
      EVB_CUDA(cudaMalloc(&s->fit_new, es * pop_size));
      EVB_CUDA(cudaMalloc(&s->nb, sizeof(int) * pop_size));
      EVB_CUDA(cudaMalloc(&s->nb_next, sizeof(int) * pop_size));
      require(evb_scratch_create(&s->eval_scratch) == EVB_OK, "pso: scratch allocation failed");
    } catch (...) {
      void* ptrs[] = {s->pbest, s->pbest_fit, s->fit_new, s->nb, s->nb_next};
      for (void* p : ptrs)
        if (p) cudaFree(p);
      delete s;
      throw;
    }
    *out = s;
  });
}

int evb_pso_destroy(evb_pso s) {
  return guarded([&] {
    if (!s) return;
    void* ptrs[] = {s->pbest, s->pbest_fit, s->fit_new, s->nb, s->nb_next};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (s->eval_scratch) evb_scratch_destroy(s->eval_scratch);
    s->phases.destroy();
    delete s;
  });
}

int evb_pso_phase_timing(evb_pso s, int enable) {
  return guarded([&] {
    require(s != nullptr, "pso: null handle");
    s->phases.on = enable != 0;
    s->phases.n = 0;
  });
}

int evb_pso_phase_ms(evb_pso s, float* ms, int cap, int* n) {
  return guarded([&] {
    require(s != nullptr && ms != nullptr && n != nullptr, "pso_phase_ms: null argument");
    *n = s->phases.read(ms, cap);
  });
}

// pso_engine::prepare first call (pso/engine.hpp:40-50): pbests <- population
int evb_pso_prepare(evb_pso s, const void* X, int64_t ldx, const void* fitness, void* stream) {
  return guarded([&] {
    require(s && X && fitness, "pso_prepare: null argument");
    if (ldx < s->D) throw invalid_argument("pso_prepare: ldx < dim");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t es = s->dtype == EVB_F64 ? 8 : 4;
    if (s->dtype == EVB_F64)
      copy_rows_kernel<double><<<s->P, 128, 0, st>>>(static_cast<const double*>(X), ldx,
                                                     static_cast<double*>(s->pbest), s->ldb, s->D);
    else
      copy_rows_kernel<float><<<s->P, 128, 0, st>>>(static_cast<const float*>(X), ldx, static_cast<float*>(s->pbest),
                                                    s->ldb, s->D);
    count_launch();
    EVB_CUDA(cudaMemcpyAsync(s->pbest_fit, fitness, es * s->P, cudaMemcpyDeviceToDevice, st));
    s->nb_valid = 0;
    s->prepared = 1;
  });
}

int evb_pso_generation(evb_pso s, evb_problem objective, evb_scratch sc, void* X, int64_t ldx, void* V, int64_t ldv,
                       void* fitness, double lb, double ub, evb_rng rng, void* stream) {
  return guarded([&] {
    require(s && objective && X && V && fitness && rng, "pso_generation: null argument");
    require(s->prepared, "pso_generation: prepare() must run first (pso/engine.hpp:40-50)");
    if (objective->p.dim != s->D) throw invalid_argument("pso_generation: problem dimension mismatch");
    if (objective->p.dtype != s->dtype) throw config_error("pso_generation: problem dtype differs from engine");
    if (ldx < s->D || ldv < s->D) throw invalid_argument("pso_generation: leading dimension < dim");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_scratch_s* scr = sc ? sc : s->eval_scratch;
    if (s->dtype == EVB_F64) generation_t<double>(s, &objective->p, scr, X, ldx, V, ldv, fitness, lb, ub, rng, st);
    else generation_t<float>(s, &objective->p, scr, X, ldx, V, ldv, fitness, lb, ub, rng, st);
  });
}

int evb_pso_attach_recorder(evb_pso s, evb_recorder rec, int run) {
  return guarded([&] {
    require(s != nullptr, "pso: null handle");
    if (rec) {
      require(recorder_dtype(rec) == s->dtype, "pso_attach_recorder: dtype mismatch");
      require(run >= 0 && run < recorder_runs(rec), "pso_attach_recorder: run out of range");
    }
    s->rec = rec;
    s->rec_run = run;
  });
}

// pso_engine::optimize (pso/engine.hpp:84-105) with the synchronous generation: init_population,
// evaluate, zero velocities, prepare, generations while fes < max_fes; best personal best
// (lowest fitness, ties to the lowest index).
int evb_pso_optimize(evb_pso s, evb_problem objective, evb_scratch sc, void* X, int64_t ldx, void* V, int64_t ldv,
                     void* fitness, double lb, double ub, int64_t max_fes, evb_rng rng, int* best_index,
                     double* best_fitness, int* generations, void* stream) {
  return guarded([&] {
    require(s && objective && X && V && fitness && rng, "pso_optimize: null argument");
    require(max_fes > 0, "evolution_state: max_fes must be positive");
    if (objective->p.dim != s->D) throw invalid_argument("pso_optimize: problem dimension mismatch");
    if (objective->p.dtype != s->dtype) throw config_error("pso_optimize: problem dtype differs from engine");
    if (ldx < s->D || ldv < s->D) throw invalid_argument("pso_optimize: leading dimension < dim");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    evb_scratch_s* scr = sc ? sc : s->eval_scratch;
    const size_t es = s->dtype == EVB_F64 ? 8 : 4;
    population_init(s->dtype, s->P, s->D, X, ldx, lb, ub, rng, st);
    eval_request rq{};
    rq.prob = &objective->p;
    rq.scratch = scr;
    rq.X = X;
    rq.n = s->P;
    rq.ldx = ldx;
    rq.out = fitness;
    rq.ldo = s->P;
    rq.n_out = 1;
    rq.kinds[0] = objective->p.kind;
    rq.biases[0] = objective->p.bias;
    rq.stream = st;
    rq.scalar_trig = true;
    eval_dispatch(rq);
    if (s->rec) recorder_observe(s->rec, s->rec_run, fitness, s->P, st);
    EVB_CUDA(cudaMemset2DAsync(V, ldv * es, 0, s->D * es, s->P, st));
    if (s->dtype == EVB_F64)
      copy_rows_kernel<double><<<s->P, 128, 0, st>>>(static_cast<const double*>(X), ldx,
                                                     static_cast<double*>(s->pbest), s->ldb, s->D);
    else
      copy_rows_kernel<float><<<s->P, 128, 0, st>>>(static_cast<const float*>(X), ldx, static_cast<float*>(s->pbest),
                                                    s->ldb, s->D);
    count_launch();
    EVB_CUDA(cudaMemcpyAsync(s->pbest_fit, fitness, es * s->P, cudaMemcpyDeviceToDevice, st));
    s->nb_valid = 0;
    s->prepared = 1;
    int64_t fes = s->P;
    int gens = 0;
    while (fes < max_fes) {
      if (s->dtype == EVB_F64) generation_t<double>(s, &objective->p, scr, X, ldx, V, ldv, fitness, lb, ub, rng, st);
      else generation_t<float>(s, &objective->p, scr, X, ldx, V, ldv, fitness, lb, ub, rng, st);
      fes += s->P;
      ++gens;
    }
    std::vector<uint8_t> f(es * s->P);
    EVB_CUDA(cudaMemcpyAsync(f.data(), s->pbest_fit, es * s->P, cudaMemcpyDeviceToHost, st));
    EVB_CUDA(cudaStreamSynchronize(st));
    auto val = [&](int i) {
      return s->dtype == EVB_F64 ? reinterpret_cast<double*>(f.data())[i] : double(reinterpret_cast<float*>(f.data())[i]);
    };
    int best = 0;
    for (int i = 1; i < s->P; ++i)
      if (val(i) < val(best)) best = i;
    if (best_index) *best_index = best;
    if (best_fitness) *best_fitness = val(best);
    if (generations) *generations = gens;
  });
}

int evb_pso_init_uniform(evb_pso s, void* A, int64_t lda, double lo, double hi, evb_rng r, void* stream) {
  return guarded([&] {
    require(s && A && r, "pso_init_uniform: null argument");
    require(lo < hi, "pso_init_uniform: lo must be less than hi");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    word_source src{r->mode, r->key, r->d_words, r->n_words};
    int64_t base = r->mode == RNG_WORDS ? words_cursor(r, st) : 0;
    const uint64_t ctr_hi = (uint64_t(r->gen) << 32) | kSubInit;
    const int blocks = int(std::min<int64_t>(4096, (int64_t(s->P) * s->D + 255) / 256));
    if (s->dtype == EVB_F64)
      init_uniform_kernel<double><<<blocks, 256, 0, st>>>(static_cast<double*>(A), lda, s->P, s->D, lo, hi, src,
                                                          ctr_hi, base, r->d_overflow);
    else
      init_uniform_kernel<float><<<blocks, 256, 0, st>>>(static_cast<float*>(A), lda, s->P, s->D, lo, hi, src, ctr_hi,
                                                         base, r->d_overflow);
    count_launch();
    EVB_CUDA(cudaGetLastError());
    if (r->mode == RNG_WORDS) {
      words_advance(r, base + int64_t(s->P) * s->D, st);
    } else {
      r->gen++;
      set_device_gen(r, st);
    }
  });
}

int evb_pso_get(evb_pso s, void* pbest_host, void* pbest_fit_host, int* nb_host, uint32_t* generation) {
  return guarded([&] {
    require(s != nullptr, "pso: null handle");
    EVB_CUDA(cudaDeviceSynchronize());
    const size_t es = s->dtype == EVB_F64 ? 8 : 4;
    if (pbest_host)
      EVB_CUDA(cudaMemcpy2D(pbest_host, s->D * es, s->pbest, s->ldb * es, s->D * es, s->P, cudaMemcpyDeviceToHost));
    if (pbest_fit_host) EVB_CUDA(cudaMemcpy(pbest_fit_host, s->pbest_fit, es * s->P, cudaMemcpyDeviceToHost));
    if (nb_host) EVB_CUDA(cudaMemcpy(nb_host, s->nb, sizeof(int) * s->P, cudaMemcpyDeviceToHost));
    if (generation) *generation = s->last_gen;
  });
}

int evb_pso_set_pbest(evb_pso s, const void* pbest_host, const void* pbest_fit_host) {
  return guarded([&] {
    require(s && pbest_host && pbest_fit_host, "pso_set_pbest: null argument");
    const size_t es = s->dtype == EVB_F64 ? 8 : 4;
    EVB_CUDA(cudaDeviceSynchronize());
    EVB_CUDA(cudaMemcpy2D(s->pbest, s->ldb * es, pbest_host, s->D * es, s->D * es, s->P, cudaMemcpyHostToDevice));
    EVB_CUDA(copy_h2d_now(s->pbest_fit, pbest_fit_host, es * s->P));
    s->nb_valid = 0;
    s->prepared = 1;
  });
}

}  // extern "C"
