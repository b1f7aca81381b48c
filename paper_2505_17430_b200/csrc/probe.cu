// probe.cu — live roofline denominators: FP64 tensor (DMMA) and FP32 FFMA throughput.
// bench.py reports its fp64 roofline fraction against the DMMA number measured here in the
// same process (MEASURED_PEAKS.json carries no FP64 figure).
#include <cuda_runtime.h>

#include "evb_internal.cuh"
#include "ptx.cuh"

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

}  // namespace

extern "C" EVB_API int evb_probe_peak_tflops(int which, int iters, double* tflops);

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
