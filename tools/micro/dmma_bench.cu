// Microbenchmark (not product code): DMMA m8n8k4 f64 latency / throughput and
// DFMA throughput on one B200, to calibrate the large-n kernels.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_dmma(double *out, int iters, long long *cyc) {
  double c0[CH], c1[CH];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < CH; ++i) { c0[i] = i; c1[i] = -i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
__global__ void k_dfma(double *out, int iters) {
  double c[CH];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < CH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *out; long long *cyc, hc;
  cudaMalloc(&out, 148 * 32 * 1024 * 8); cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  // latency: 1 warp, chain of dependent DMMAs
  k_dmma<1><<<1, 32>>>(out, iters, cyc); cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency: %.1f cycles\n", (double)hc / iters);
  k_dmma<4><<<1, 32>>>(out, iters, cyc); cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA 1 warp, 4 chains: %.1f cycles per DMMA\n", (double)hc / iters / 4);
  k_dmma<8><<<1, 32>>>(out, iters, cyc); cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA 1 warp, 8 chains: %.1f cycles per DMMA\n", (double)hc / iters / 8);
  for (int w : {1, 2, 4, 8, 16}) {
    k_dmma<8><<<148, 32 * w>>>(out, iters, cyc);
    cudaEventRecord(e0); k_dmma<8><<<148, 32 * w>>>(out, iters, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 148.0 * w * iters * 8 * 512.0;  // 8x8x4 = 256 FMA = 512 flop per warp-DMMA
    printf("DMMA %2d warps/SM x 8 chains: %.2f TFLOP/s\n", w, fl / ms / 1e9);
  }
  for (int w : {4, 8, 16, 32}) {
    k_dfma<8><<<148, 32 * w>>>(out, iters);
    cudaEventRecord(e0); k_dfma<8><<<148, 32 * w>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 148.0 * 32 * w * iters * 8 * 2.0;
    printf("DFMA %2d warps/SM x 8 chains: %.2f TFLOP/s\n", w, fl / ms / 1e9);
  }
  return 0;
}
