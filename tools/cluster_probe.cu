// Max resident thread-block clusters per device for cluster sizes 1-16 at
// one CTA per SM (large dynamic shared memory), as cudaOccupancyMaxActiveClusters
// reports them: sizes the wide fused chain (wide_kernels.cu) can launch.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_probe(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int smems[] = {50000, 120000, 217448, 232448};
  for (int sm : smems)
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(cs); lc.blockDim = dim3(320); lc.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      lc.attrs = at; lc.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k_probe, &lc);
      printf("smem %6d cluster %2d -> %3d clusters (%d CTAs) %s\n", sm, cs, n, n * cs, cudaGetErrorString(e));
    }
  return 0;
}
