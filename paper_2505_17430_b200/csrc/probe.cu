// probe.cu — live roofline denominators: FP64 tensor (DMMA) and FP32 FFMA throughput.
// bench.py reports its fp64 roofline fraction against the DMMA number measured here in the
// same process (MEASURED_PEAKS.json carries no FP64 figure).
#include <cuda_runtime.h>

#include "evb_internal.cuh"
#include "ptx.cuh"
#define EVB_UMMA_HELPERS_ONLY
#include "umma.cuh"

namespace {

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) evb::ptx::dmma_8x8x4(c[t][0], c[t][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(512) ffma_peak_kernel(float* out, int iters) {
  float x[8];
  const float a = 1.0f + threadIdx.x * 1e-7f, b = 1e-7f;
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = float(t);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = fmaf(x[t], a, b);
  }
  float s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += x[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// tcgen05.mma kind::tf32 issue rate: one CTA per SM, one thread issues `iters` M=128 x N x K=8
// MMAs into one TMEM accumulator from a zeroed SWIZZLE_128B tile (tools/umma_probe.cu's kernel)
template <bool F16>
__global__ void __launch_bounds__(128) umma_peak_kernel(int iters, int N) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(evb::ptx::smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) evb::umma::tmem_alloc(&tslot, 256);
  evb::umma::fence_before();
  __syncthreads();
  evb::umma::fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = F16 ? evb::umma::idesc_f16(128, N) : evb::umma::idesc_tf32(128, N);
    const uint32_t a = evb::ptx::smem_u32(sm), b = evb::ptx::smem_u32(sm + 16384);
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = evb::umma::smem_desc(a + (i & 3) * 32), db = evb::umma::smem_desc(b + (i & 3) * 32);
      if (F16) evb::umma::mma_f16(tm, da, db, idesc, uint32_t(i));  // K = 16 halves per instruction
      else evb::umma::mma_tf32(tm, da, db, idesc, uint32_t(i));     // K = 8
    }
    evb::umma::commit(&bar);
    evb::ptx::mbar_wait(&bar, 0);
  }
  evb::umma::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) evb::umma::tmem_dealloc(tm, 256);
}

}  // namespace

extern "C" EVB_API int evb_probe_peak_tflops(int which, int iters, double* tflops);
extern "C" EVB_API int evb_probe_umma_tf32_tflops(int n, double* tflops);
extern "C" EVB_API int evb_probe_umma_f16_tflops(int n, double* tflops);

namespace {
int probe_umma(bool f16, int n, double* tflops);
}
// dense kind::tf32 / kind::f16 tcgen05 throughput at tile width n (64, 128 or 256): best of 3 timed launches
extern "C" int evb_probe_umma_tf32_tflops(int n, double* tflops) { return probe_umma(false, n, tflops); }
extern "C" int evb_probe_umma_f16_tflops(int n, double* tflops) { return probe_umma(true, n, tflops); }

namespace {
int probe_umma(bool f16, int n, double* tflops) {
  try {
    if (!(n == 64 || n == 128 || n == 256)) return EVB_ERR_INVALID_ARGUMENT;
    int dev = 0, sms = 0;
    EVB_CUDA(cudaGetDevice(&dev));
    EVB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int smem = 65 * 1024;
    EVB_CUDA(cudaFuncSetAttribute(umma_peak_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    EVB_CUDA(cudaFuncSetAttribute(umma_peak_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 4096;
    cudaEvent_t e0, e1;
    EVB_CUDA(cudaEventCreate(&e0));
    EVB_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      EVB_CUDA(cudaEventRecord(e0));
      if (f16) umma_peak_kernel<true><<<sms, 128, smem>>>(iters, n);
      else umma_peak_kernel<false><<<sms, 128, smem>>>(iters, n);
      EVB_CUDA(cudaEventRecord(e1));
      EVB_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      EVB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0 && ms < best) best = ms;
    }
    *tflops = 2.0 * 128 * n * (f16 ? 16 : 8) * double(iters) * sms / (double(best) * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return EVB_OK;
  } catch (const std::exception&) {
    return EVB_ERR_RUNTIME;
  }
}
}  // namespace

// which: 0 = FP64 DMMA m8n8k4, 1 = FP32 FFMA.  Best of 3 timed launches after a warm-up.
extern "C" int evb_probe_peak_tflops(int which, int iters, double* tflops) {
  try {
    int dev = 0, sms = 0;
    EVB_CUDA(cudaGetDevice(&dev));
    EVB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    void* buf = nullptr;
    const int threads = which == 0 ? 256 : 512;
    EVB_CUDA(cudaMalloc(&buf, size_t(sms) * threads * 8));
    cudaEvent_t e0, e1;
    EVB_CUDA(cudaEventCreate(&e0));
    EVB_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      EVB_CUDA(cudaEventRecord(e0));
      if (which == 0) dmma_peak_kernel<<<sms, threads>>>(static_cast<double*>(buf), iters);
      else ffma_peak_kernel<<<sms, threads>>>(static_cast<float*>(buf), iters);
      EVB_CUDA(cudaEventRecord(e1));
      EVB_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      EVB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0 && ms < best) best = ms;
    }
    // DMMA m8n8k4 = 256 FMA = 512 flop per warp instruction; 8 per iteration per warp
    const double flops = which == 0 ? double(sms) * (threads / 32) * double(iters) * 8 * 512
                                    : double(sms) * threads * double(iters) * 32 * 2;
    *tflops = flops / (double(best) * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    return EVB_OK;
  } catch (const std::exception&) {
    return EVB_ERR_RUNTIME;
  }
}
