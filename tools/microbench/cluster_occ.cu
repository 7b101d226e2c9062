// How many clusters of Q CTAs (1 CTA per SM, large dynamic smem) can be co-resident.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1, 1, 1) dummy1(int* p) { if (p) p[0] = 1; }
__global__ void dummy(int* p) { if (p) p[0] = 1; }
int main() {
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int q : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(q * 148);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", q, n, n * q, cudaGetErrorString(e));
  }
  // cooperative + cluster launch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(144);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  int* p = nullptr;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dummy, p);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("cooperative + cluster(2) launch of 144: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
  return 0;
}
