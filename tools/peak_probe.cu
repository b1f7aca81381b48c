// Throughput probe for the FP64 (DMMA, DFMA) and FP32 (FFMA) pipes on B200.
// Standalone scratch tool: prints achieved TFLOP/s for several occupancies.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int t = 0; t < NACC; ++t) c[t][0] = c[t][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NACC; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NACC; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = fma(x[t], a, b);
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += x[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_loop(float* out, int iters) {
  float x[8];
  float a = 1.0f + threadIdx.x * 1e-7f, b = 1e-7f;
#pragma unroll
  for (int t = 0; t < 8; ++t) x[t] = t;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = fmaf(x[t], a, b);
  }
  float s = 0;
  for (int t = 0; t < 8; ++t) s += x[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d smem/sm=%zu l2=%d clock_khz=%d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerMultiprocessor, p.l2CacheSize, clk);
  const int sms = p.multiProcessorCount;
  double* d;
  cudaMalloc(&d, 64 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int blocks, int threads, int iters, double flop_per_thread_iter) {
    kern<<<blocks, threads>>>(d, iters);  // warm
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double flops = double(blocks) * threads * iters * flop_per_thread_iter;
    printf("%-28s blocks=%5d thr=%4d  %.3f ms  %.2f TFLOP/s\n", name, blocks, threads, best,
           flops / best / 1e9);
  };
  const int it = 20000;
  // DMMA m8n8k4: 256 FMA = 512 flop per warp-instruction = 16 flop per thread
  for (int wps : {1, 2, 4, 8}) {
    run("dmma NACC=4", dmma_loop<4>, sms, 128 * wps, it, 4 * 16.0);
    run("dmma NACC=8", dmma_loop<8>, sms, 128 * wps, it, 8 * 16.0);
  }
  run("dmma NACC=8 2blk/sm", dmma_loop<8>, sms * 2, 256, it, 8 * 16.0);
  for (int wps : {1, 2, 4, 8}) run("dfma", dfma_loop, sms, 128 * wps, it, 32 * 2.0);
  for (int wps : {2, 4, 8}) run("ffma", (void (*)(double*, int))ffma_loop, sms, 128 * wps, it, 32 * 2.0);
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
