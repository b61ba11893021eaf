// How many thread-block clusters of 2/4/6/8 CTAs (one 200 KB CTA per SM) a B200 can hold at
// once: cudaOccupancyMaxActiveClusters. GPCs whose SM count is not a multiple of the cluster
// size strand SMs — the cost side of TMA multicast across CTA pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_occupancy tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe_kernel(int* out) {
  extern __shared__ int smem[];
  if (threadIdx.x == 0) out[blockIdx.x] = smem[0];
}

int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cl : {1, 2, 4, 6, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
    printf("cluster %2d CTAs: max active clusters %3d -> %3d of %d SMs busy (%s)\n", cl, n, n * cl, sms,
           cudaGetErrorString(e));
  }
  return 0;
}
