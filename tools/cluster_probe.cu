// tools/cluster_probe.cu — dev probe: how many SMs thread-block clusters of
// each size can occupy at once on this GPU (GPC packing), for a kernel held
// to one CTA per SM by its shared memory. Prints CS, max active clusters,
// SMs covered. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[blockIdx.x] = s[threadIdx.x];
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs * 64);
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)dummy, &lc);
    std::printf("CS %2d: max active clusters %3d -> %3d of %d SMs%s\n", cs, n, n * cs, nsm,
                e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
