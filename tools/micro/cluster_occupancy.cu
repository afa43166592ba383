// Occupancy probe: max active clusters of the column kernel's cluster shapes (1 x 8 / 1 x 4
// CTAs of 128 threads, 35.8 / 68.6 KB smem).  nvcc -gencode arch=compute_100a,code=sm_100a
// -o /tmp/occ tools/micro/cluster_occupancy.cu && /tmp/occ.  Measured on one B200: 8-CTA
// clusters 104 resident (832 CTAs of the 888 the SM limits allow), 4-CTA 213 (852).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1, 8, 1) __launch_bounds__(128, 6) k8(int* o) { extern __shared__ int s[]; if (o) o[0] = s[0]; }
__global__ void __cluster_dims__(1, 4, 1) __launch_bounds__(128, 6) k4(int* o) { extern __shared__ int s[]; if (o) o[0] = s[0]; }
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("SMs %d\n", p.multiProcessorCount);
  for (int cl : {4, 8}) {
    for (int smem : {32 * 1024 + 3072, 64 * 1024 + 3072}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(64, cl, 64); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = 1; at.val.clusterDim.y = cl; at.val.clusterDim.z = 1;
      cfg.attrs = &at; cfg.numAttrs = 1;
      int n = 0;
      auto f = cl == 8 ? (void*)k8 : (void*)k4;
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, f, &cfg);
      printf("cluster %d smem %d: max active clusters %d (%d CTAs) %s\n", cl, smem, n, n * cl, cudaGetErrorString(e));
    }
  }
}
