// Microbenchmark: duration of an (almost) empty kernel launched with the fused
// path's cluster shape (16-CTA clusters, 256 threads, 52 KB dynamic smem) vs
// the same grid without clusters, and with a fixed per-CTA spin, to measure
// launch/ramp/tail overhead.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cl cluster_launch.cu
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void kspin(long long cycles, int *sink, int use_cluster) {
  extern __shared__ float sm[];
  if (use_cluster) cg::this_cluster().sync();
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  if (threadIdx.x == 0 && sm[0] == 12345.f) sink[0] = 1;
  if (use_cluster) cg::this_cluster().sync();
}
int main() {
  int *sink; cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(kspin, cudaFuncAttributeMaxDynamicSharedMemorySize, 53392);
  cudaFuncSetAttribute(kspin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int cs : {1, 8, 16}) for (int streams : {31, 32, 64}) for (long long cyc : {0LL, 20000LL, 100000LL}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, streams); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 53392;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int uc = cs > 1;
    for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, kspin, cyc, sink, uc);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) cudaLaunchKernelEx(&cfg, kspin, cyc, sink, uc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int ncl = 0;
    if (cs > 1) cudaOccupancyMaxActiveClusters(&ncl, (void *)kspin, &cfg);
    printf("cluster %2d streams %2d spin %6lld cyc (%5.1f us): %7.1f us per launch  (max active clusters %d) %s\n", cs, streams, cyc,
           cyc / 1965.0, ms * 1000 / 20, ncl, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
