// FP64 micro-benchmark (tuning aid): dependent-chain latency of DFMA / DADD / DMMA and the
// throughput of independent chains, one CTA of W warps.  nvcc -arch=sm_100a -o fp64_lat fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_fma(double* out, long long* cyc, int n, double a) {
  double x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, 1e-9);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
__global__ void k_add(double* out, long long* cyc, int n, double a) {
  double x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __dadd_rn(x[c], a);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
__global__ void k_dmma(double* out, long long* cyc, int n, double a) {
  double c0[CH], c1[CH];
  for (int c = 0; c < CH; ++c) c0[c] = c1[c] = threadIdx.x + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(c0[c], c1[c], a, a);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += c0[c] + c1[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int warps, int ch, int ops_per_inst_lane) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const int n = 4096;
  kern<<<1, 32 * warps>>>(out, cyc, n, 0.999);
  kern<<<1, 32 * warps>>>(out, cyc, n, 0.999);
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per = double(c) / n;  // cycles per loop iteration (ch instructions per warp)
  std::printf("%-5s warps=%2d chains=%d: %.2f cyc/iter  -> %.2f cyc per dependent op, %.1f warp-inst/cyc/SM\n", name,
              warps, ch, per, per, double(warps) * ch / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run("dfma", k_fma<1>, w, 1, 1);
    run("dfma", k_fma<8>, w, 8, 1);
    run("dadd", k_add<1>, w, 1, 1);
    run("dadd", k_add<8>, w, 8, 1);
    run("dmma", k_dmma<1>, w, 1, 1);
    run("dmma", k_dmma<4>, w, 4, 1);
  }
  return 0;
}
