// Prints how many thread-block clusters of a given size and shared-memory
// footprint can be co-resident on this GPU (cudaOccupancyMaxActiveClusters).
// Used to size the cluster-fused vote+peaks kernel.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occupancy tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(int *p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}

int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  const int smems[] = {227 * 1024, 200 * 1024, 150 * 1024, 113 * 1024, 100 * 1024, 72 * 1024};
  const int threads[] = {1024, 512};
  for (int th : threads)
    for (int sm : smems) {
      printf("threads %4d smem %6d:", th, sm);
      for (int k = 1; k <= 16; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(k * 64, 1, 1);
        cfg.blockDim = dim3(th, 1, 1);
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = k;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        if (e != cudaSuccess) { printf(" %d:err", k); cudaGetLastError(); continue; }
        printf(" %d:%d(%d)", k, n, n * k);
      }
      printf("\n");
    }
  return 0;
}
