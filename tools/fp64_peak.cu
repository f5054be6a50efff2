// fp64_peak.cu -- measured FP64 ceilings of this B200 (the secondary roofline
// of the hex K kernel, BASELINE.md "fp64 FMA ceiling: to be measured").
//   1. DFMA throughput: every thread runs 8 independent FMA chains, grid =
//      148 SMs x 8 blocks x 256 threads; flops = 2 per FMA.
//   2. DFMA dependent-chain latency: one warp, one chain, clock64 cycles.
//   3. DMMA (mma.sync.m8n8k4.f64) throughput: 8 independent accumulators per
//      warp; flops = 2*8*8*4 per mma.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dadd(double* out, int iters, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] + b;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

__global__ void k_dmma(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double av = 1.0 + threadIdx.x * 1e-9, bv = 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d_out;
  long long* d_cyc;
  CK(cudaMalloc(&d_out, 8));
  CK(cudaMalloc(&d_cyc, 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256, iters = 20000;
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5.0;
  };
  float ms = timeit([&] { k_dfma<<<blocks, threads>>>(d_out, iters, 0.9999999, 1e-7); });
  double fl = 2.0 * 8 * (double)iters * blocks * threads;
  std::printf("{\"dfma_tflops\": %.3f, ", fl / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_dadd<<<blocks, threads>>>(d_out, iters, 1e-7); });
  fl = 1.0 * 8 * (double)iters * blocks * threads;
  std::printf("\"dadd_gops\": %.3f, ", fl / (ms * 1e-3) / 1e9);
  k_lat<<<1, 32>>>(d_out, d_cyc, 100000, 0.9999999, 1e-7);
  long long cyc = 0;
  CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
  std::printf("\"dfma_latency_cycles\": %.2f, ", cyc / 100000.0);
  ms = timeit([&] { k_dmma<<<blocks, threads>>>(d_out, iters / 4); });
  fl = 2.0 * 8 * 8 * 4 * 8 * (double)(iters / 4) * blocks * (threads / 32);
  std::printf("\"dmma_tflops\": %.3f, \"sms\": %d}\n", fl / (ms * 1e-3) / 1e12, sms);
  CK(cudaGetLastError());
  return 0;
}
