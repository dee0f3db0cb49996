// Microbenchmark (not product code): accuracy of rcp.approx.ftz.f64 /
// rsqrt.approx.ftz.f64 (MUFU) and DFMA dependent latency on one B200.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k_err(const double *x, double *er, double *es, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r, s;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i]));
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(s) : "d"(x[i]));
  er[i] = fabs(r * x[i] - 1.0);
  es[i] = fabs(s * s * x[i] - 1.0);
}
__global__ void k_lat(double *out, int iters, long long *cyc) {
  double a = threadIdx.x * 1e-3 + 1.0, b = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-9);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  const int n = 1 << 20;
  double *hx = new double[n], *x, *er, *es;
  srand(1);
  for (int i = 0; i < n; ++i) hx[i] = ldexp(1.0 + rand() / (double)RAND_MAX, (rand() % 200) - 100);
  cudaMalloc(&x, n * 8); cudaMalloc(&er, n * 8); cudaMalloc(&es, n * 8);
  cudaMemcpy(x, hx, n * 8, cudaMemcpyHostToDevice);
  k_err<<<n / 256, 256>>>(x, er, es, n);
  double *h1 = new double[n], *h2 = new double[n];
  cudaMemcpy(h1, er, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, es, n * 8, cudaMemcpyDeviceToHost);
  double m1 = 0, m2 = 0;
  for (int i = 0; i < n; ++i) { m1 = fmax(m1, h1[i]); m2 = fmax(m2, h2[i]); }
  printf("rcp.approx.f64 max rel err %.3e (2^%.1f); rsqrt.approx.f64 max rel err (of s^2 x - 1) %.3e (2^%.1f)\n",
         m1, log2(m1), m2, log2(m2));
  long long *cyc, hc; double *out;
  cudaMalloc(&cyc, 8); cudaMalloc(&out, 32 * 8);
  k_lat<<<1, 32>>>(out, 4096, cyc); cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", hc / 4096.0);
  return 0;
}
