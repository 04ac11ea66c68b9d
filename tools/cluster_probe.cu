// Co-resident clusters per cluster size on this GPU (GPC packing), for a
// kernel with one CTA per SM (large dynamic shared memory).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_probe tools/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[blockIdx.x] = s[threadIdx.x];
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("sms %d\n", sms);
  for (int cl = 1; cl <= 16; ++cl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * (sms / cl));
    cfg.blockDim = dim3(544);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k_dummy, &cfg);
    printf("cluster %2d: %3d clusters = %3d SMs  (%s)\n", cl, n, n * cl, cudaGetErrorString(e));
  }
  return 0;
}
