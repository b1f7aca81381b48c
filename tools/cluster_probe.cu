// How many thread-block clusters of a given size can be co-resident (tuning aid): one CTA per SM
// (large dynamic shared memory), cluster sizes 2..16.  nvcc -arch=sm_100a -o cluster_probe cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) { extern __shared__ char s[]; if (threadIdx.x == 0 && out) out[blockIdx.x] = s[0]; }
int main() {
  const int smem = 226 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t lc{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = cs / 2; at[0].val.clusterDim.z = 2;
    lc.gridDim = dim3(8, cs / 2, 2); lc.blockDim = dim3(352); lc.dynamicSmemBytes = smem; lc.attrs = at; lc.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &lc);
    std::printf("cluster size %2d: max active clusters %d (%s) -> %d CTAs\n", cs, n, cudaGetErrorString(e), n * cs);
  }
  return 0;
}
