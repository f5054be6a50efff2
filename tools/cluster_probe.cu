// Which SMs can host the CTAs of a thread-block cluster of a given size?
// Launches a spinning kernel (one CTA per SM: 200 KB of shared memory) as
// clusters of size CL and records each CTA's %smid; prints the number of
// distinct SMs used and the co-resident cluster count the runtime reports.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_probe tools/cluster_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

__global__ void k_probe(int* smid, long long spin) {
  extern __shared__ char sm[];
  unsigned id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  if (threadIdx.x == 0) smid[blockIdx.x] = (int)id;
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  if (threadIdx.x == 0 && sm[0] == 123) smid[blockIdx.x] = -1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 4, 8, 16}) {
    const int grid = ((sms + cl - 1) / cl) * cl;  // one wave if every SM could take a CTA
    int* d = nullptr;
    cudaMalloc(&d, grid * sizeof(int));
    cudaMemset(d, 0xff, grid * sizeof(int));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k_probe, &cfg);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k_probe, d, 2000000LL);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<int> h(grid);
    cudaMemcpy(h.data(), d, grid * sizeof(int), cudaMemcpyDeviceToHost);
    std::set<int> used(h.begin(), h.end());
    std::printf("cluster %2d: launch %s, max active clusters %3d (= %3d CTAs of %d SMs), grid %d CTAs -> %zu distinct SMs, %.2f ms (1 wave = ~1.0 ms)\n",
                cl, cudaGetErrorName(err), ncl, ncl * cl, sms, grid, used.size(), ms);
    if (cl == 8) {
      // SM ids per cluster: shows the GPC grouping
      for (int c = 0; c < grid / cl && c < 24; ++c) {
        std::printf("  cluster %2d:", c);
        for (int i = 0; i < cl; ++i) std::printf(" %3d", h[c * cl + i]);
        std::printf("\n");
      }
    }
    cudaFree(d);
  }
  return 0;
}
