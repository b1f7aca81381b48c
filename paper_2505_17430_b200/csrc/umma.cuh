// umma.cuh — K2 on the 5th-generation tensor cores: the fp32 batched evaluation
// z = M (x - o) as 3xTF32 tcgen05.mma (kind::tf32) with the accumulator in TMEM.
//
// A single TF32 pass fails the 1e-4 fitness tolerance at D = 1000, so each operand is
// split into a TF32-exact head and its remainder, a = a_hi + a_lo, and
//     z = S_hi M_hi^T + S_hi M_lo^T + S_lo M_hi^T        (the a_lo b_lo term, ~2^-22, dropped)
// accumulated in fp32 in TMEM.  S = X - o is rounded in fp32 exactly like the reference's
// transform (problems/batch.hpp:50) before the split; M_hi / M_lo are split once when the
// problem is created.  The S split is folded into the kernel at the default tile width (FUSE,
// eval_gemm.cu); other widths run the split pre-pass below first.
//
// CTA (10 warps, one 128 x 64 output tile):
//   warp 0  TMA producer: per 32-float K-slice, X (128 rows, into the S_hi slot; FUSE) or
//           S_hi, S_lo (pre-pass mode), and M_hi, M_lo (64 rows), SWIZZLE_128B, into a 4-stage
//           mbarrier ring (48 KB per stage)
//   warp 1  TMEM allocator + single-thread MMA issuer: 4 K-steps x 3 products of
//           tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=64, K=8) per stage; tcgen05.commit frees
//           the stage and finally signals the epilogue
//   warps 2-9 during the mainloop (FUSE): S_hi / S_lo of each X tile, in place in the stage;
//           epilogue: tcgen05.ld 32x32b, two warps per TMEM lane quarter (each thread = one
//           output row, half of the 64 columns), transform terms, half-row sums meeting in shared
//           memory, N-tile partials + last-CTA finalisation (as K1).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace evb {

namespace umma {

__device__ __forceinline__ uint32_t cvt_rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// the same rounding on the integer pipe (round half away from zero on the magnitude: add half a
// TF32 ulp to the bits, clear the 13 dropped bits; inf and NaN keep their class) — two integer
// ops instead of a conversion, for the in-kernel split where the conversion rate bounds a stage
__device__ __forceinline__ uint32_t rna_tf32_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 "smem descriptor"):
// start address >> 4, LBO = 1 (unused for swizzled K-major), SBO = 1024 B (8 rows x 128 B),
// version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major, N >> 3, M >> 4
constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// instruction descriptor, kind::f16: D f32, A/B f16 (format 0), both K-major; K = 16 per instruction
constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// A operand from TMEM (lanes = M rows, one 32-bit column per K element): D += A[tmem] B[smem]
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// registers -> TMEM, 32 lanes x 16 consecutive columns (the warp's lane quarter)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}
// commit arriving on the barrier at `bar`'s offset in every CTA of `mask` (operands multicast
// into several CTAs are freed only when all their consumers' MMAs are done)
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   ptx::smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 32 bits, 16 consecutive columns -> 16 registers per thread
// tcgen05.ld without the wait (several loads in flight, then tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_raw(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace umma

#ifndef EVB_UMMA_HELPERS_ONLY  // the split kernels live in eval_gemm.cu's translation unit
// split pre-pass: S = X - o (fp32, reference rounding), S_hi = rna_tf32(S), S_lo = S - S_hi
__global__ void split_tf32_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ shift, int P,
                                  int D, float* __restrict__ hi, float* __restrict__ lo, int64_t lds) {
  ptx::griddep_launch_dependents();  // the MMA kernel's prologue may overlap this pass (PDL)
  const int i = blockIdx.y;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < lds; k += gridDim.x * blockDim.x) {
    float h = 0.f, l = 0.f;
    if (k < D) {
      const float s = __fsub_rn(X[size_t(i) * ldx + k], shift[k]);
      h = __uint_as_float(umma::cvt_rna_tf32(s));
      // round the remainder to TF32 too: the tensor core would otherwise truncate it, and a
      // truncation bias accumulates linearly over K instead of as sqrt(K)
      l = __uint_as_float(umma::cvt_rna_tf32(__fsub_rn(s, h)));
    }
    hi[size_t(i) * lds + k] = h;
    lo[size_t(i) * lds + k] = l;
  }
}

// plain split (for the rotation at problem creation): hi = rna_tf32(a), lo = a - hi
__global__ void split_plain_kernel(const float* __restrict__ a, int64_t n, float* __restrict__ hi,
                                   float* __restrict__ lo) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const float x = a[e];
    const float h = __uint_as_float(umma::cvt_rna_tf32(x));
    hi[e] = h;
    lo[e] = __uint_as_float(umma::cvt_rna_tf32(__fsub_rn(x, h)));
  }
}
// fp16 split of the rotation for the 3xFP16 kernel: a' = kF16Scale * a (a power of two: exact, and
// it lifts the remainder of typical entries out of fp16's subnormal range), hi = fp16(a'),
// lo = fp16(a' - hi): 22 significant bits, as the TF32 split
constexpr float kF16Scale = 256.f;
constexpr float kF16SafeMax = 65000.f;  // |value| up to here has a finite fp16 head
__global__ void split_f16_kernel(const float* __restrict__ a, int64_t n, __half* __restrict__ hi,
                                 __half* __restrict__ lo, int* __restrict__ out_of_range) {
  bool bad = false;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const float x = __fmul_rn(a[e], kF16Scale);
    bad = bad || !(fabsf(x) <= kF16SafeMax);  // also NaN
    const __half h = __float2half_rn(x);
    hi[e] = h;
    lo[e] = __float2half_rn(__fsub_rn(x, __half2float(h)));
  }
  if (bad) *out_of_range = 1;
}
#endif  // EVB_UMMA_HELPERS_ONLY

}  // namespace evb
