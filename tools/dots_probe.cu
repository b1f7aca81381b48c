// Micro-benchmark (tuning aid) of the exact-order dot-product pattern of the persistent DE kernel:
// W warps of one CTA, every thread QG chains acc = add(acc, mul(m, s)) over K steps, m per lane
// from shared memory (LDS.64), s broadcast (LDS.128 per two steps).  Prints cycles per k step.
// nvcc -arch=sm_100a -O3 -o dots_probe dots_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int QG, bool LDS>
__global__ void k_dots(double* out, long long* cyc, int K, int D) {
  extern __shared__ double sm[];
  double* sMT = sm;            // K x D
  double* sS = sm + K * D;     // QG x K
  for (int i = threadIdx.x; i < K * D + QG * K; i += blockDim.x) sm[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  const int r = threadIdx.x % D;
  double acc[QG];
#pragma unroll
  for (int u = 0; u < QG; ++u) acc[u] = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep)
    for (int k = 0; k + 2 <= K; k += 2) {
      double m0, m1;
      if (LDS) { m0 = sMT[k * D + r]; m1 = sMT[(k + 1) * D + r]; } else { m0 = 1.0 + k; m1 = 2.0 + k; }
#pragma unroll
      for (int u = 0; u < QG; ++u) {
        double2 x;
        if (LDS) x = *reinterpret_cast<const double2*>(sS + u * K + k); else x = make_double2(acc[u] * 0 + 1.5, 2.5);
        acc[u] = __dadd_rn(acc[u], __dmul_rn(m0, x.x));
        acc[u] = __dadd_rn(acc[u], __dmul_rn(m1, x.y));
      }
    }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int u = 0; u < QG; ++u) s += acc[u];
  out[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// software-pipelined variant: the operands of step pair k + 2 are loaded before pair k's arithmetic
template <int QG>
__global__ void k_dots_pipe(double* out, long long* cyc, int K, int D) {
  extern __shared__ double sm[];
  double* sMT = sm;
  double* sS = sm + K * D;
  for (int i = threadIdx.x; i < K * D + QG * K; i += blockDim.x) sm[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  const int r = threadIdx.x % D;
  double acc[QG];
#pragma unroll
  for (int u = 0; u < QG; ++u) acc[u] = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep) {
    double m0 = sMT[r], m1 = sMT[D + r];
    double2 x[QG];
#pragma unroll
    for (int u = 0; u < QG; ++u) x[u] = *reinterpret_cast<const double2*>(sS + u * K);
    for (int k = 0; k + 2 <= K; k += 2) {
      const int kn = k + 2 < K ? k + 2 : k;
      const double n0 = sMT[kn * D + r], n1 = sMT[(kn + 1) * D + r];
      double2 y[QG];
#pragma unroll
      for (int u = 0; u < QG; ++u) y[u] = *reinterpret_cast<const double2*>(sS + u * K + kn);
#pragma unroll
      for (int u = 0; u < QG; ++u) {
        acc[u] = __dadd_rn(acc[u], __dmul_rn(m0, x[u].x));
        acc[u] = __dadd_rn(acc[u], __dmul_rn(m1, x[u].y));
      }
      m0 = n0; m1 = n1;
#pragma unroll
      for (int u = 0; u < QG; ++u) x[u] = y[u];
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int u = 0; u < QG; ++u) s += acc[u];
  out[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int QG>
void run_pipe(int warps) {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double)); cudaMalloc(&cyc, sizeof(long long));
  const int K = 100, D = 100;
  const size_t smem = (K * D + QG * K) * sizeof(double);
  cudaFuncSetAttribute(k_dots_pipe<QG>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int i = 0; i < 2; ++i) k_dots_pipe<QG><<<1, 32 * warps, smem>>>(out, cyc, K, D);
  long long c; cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per_k = double(c) / (8.0 * K);
  std::printf("PIPE QG=%d warps=%2d: %.1f cycles per k (thread 0), %.2f FP64 warp-inst/cycle/SM\n", QG, warps, per_k,
              warps * QG * 2.0 / per_k);
  cudaFree(out); cudaFree(cyc);
}

template <int QG, bool LDS>
void run(int warps) {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double)); cudaMalloc(&cyc, sizeof(long long));
  const int K = 100, D = 100;
  const size_t smem = (K * D + QG * K) * sizeof(double);
  cudaFuncSetAttribute(k_dots<QG, LDS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int i = 0; i < 2; ++i) k_dots<QG, LDS><<<1, 32 * warps, smem>>>(out, cyc, K, D);
  long long c; cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per_k = double(c) / (8.0 * K);
  std::printf("QG=%d lds=%d warps=%2d: %.1f cycles per k (thread 0), %.2f FP64 warp-inst/cycle/SM\n", QG, int(LDS), warps, per_k,
              warps * QG * 2.0 / per_k);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 10, 12, 16}) { run<4, true>(w); run<4, false>(w); run_pipe<4>(w); }
  for (int w : {4, 8, 13, 16}) { run<3, true>(w); run_pipe<3>(w); run<2, true>(w); run_pipe<2>(w); run<6, true>(w); run_pipe<6>(w); }
  return 0;
}
