// Standalone tcgen05.mma throughput probe (kind::tf32 and kind::f16, M=128, N in {64,128,256}):
// one CTA per SM, one thread issues ITERS MMAs into one TMEM accumulator from a zeroed smem tile.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
template <int KIND>  // 0 tf32, 1 f16
__global__ void probe(int iters, int N, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = KIND == 0 ? ((1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (8u << 24))
                                     : ((1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(N >> 3) << 17) | (8u << 24));
    const uint32_t a = su32(sm), b = su32(sm + 16384);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = desc(a + (i & 3) * 32), db = desc(b + (i & 3) * 32);
      if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(i));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)));
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  for (int kind = 0; kind < 2; ++kind)
    for (int N : {64, 128, 256}) {
      const int iters = 4096;
      auto k = kind == 0 ? probe<0> : probe<1>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      k<<<148, 128, 96 * 1024>>>(iters, N, d);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<148, 128, 96 * 1024>>>(iters, N, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long cyc;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      const double K = kind == 0 ? 8 : 16;
      const double flops = 2.0 * 128 * N * K * iters * 148;
      printf("%s N=%d: %.1f cycles/MMA, %.1f TFLOP/s  (%s)\n", kind == 0 ? "tf32" : "f16 ", N, double(cyc) / iters,
             flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
