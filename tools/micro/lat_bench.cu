// Microbenchmark (not product code): single-warp latencies on one B200 that
// bound the CTA path's serial Householder panel -- dependent DFMA, 64-bit
// warp shuffle, the 8-value warp all-reduce, MUFU rsqrt/rcp + Newton.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double h) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(h));
  double hy = h * y;
  y = fma(0.5 * y, fma(-hy, y, 1.0), y);
  hy = h * y;
  y = fma(0.5 * y, fma(-hy, y, 1.0), y);
  return y;
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
__device__ __forceinline__ void warp_sum8(double (&p)[8]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b2 = lane & 8, b1 = lane & 4;
  double h[4], qd[2], o;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b4 ? p[i] : p[i + 4];
    h[i] = (b4 ? p[i + 4] : p[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b2 ? h[i] : h[i + 2];
    qd[i] = (b2 ? h[i + 2] : h[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const double send = b1 ? qd[0] : qd[1];
    o = (b1 ? qd[1] : qd[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  o += __shfl_xor_sync(0xffffffffu, o, 2);
  o += __shfl_xor_sync(0xffffffffu, o, 1);
#pragma unroll
  for (int v = 0; v < 8; ++v) p[v] = __shfl_sync(0xffffffffu, o, 4 * v);
}

__global__ void k_lat(double *out, long long *cyc, int iters) {
  const int lane = threadIdx.x & 31;
  double x = 1.0 + lane * 1e-3, a = 0.999999;
  long long t0, t1;
  // 1. dependent DFMA
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, 1e-9);
  t1 = clock64();
  cyc[0] = (t1 - t0);
  // 2. dependent 64-bit shuffle + add
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x * 0.5 + __shfl_xor_sync(0xffffffffu, x, 1) * 0.5;
  t1 = clock64();
  cyc[1] = (t1 - t0);
  // 3. warp_sum8 chain
  double p[8];
  for (int v = 0; v < 8; ++v) p[v] = x + v;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    warp_sum8(p);
#pragma unroll
    for (int v = 0; v < 8; ++v) p[v] *= (1.0 / 32);
  }
  t1 = clock64();
  cyc[2] = (t1 - t0);
  x += p[3];
  // 4. rsqrt_nr chain
  double s = 2.0 + x * 1e-6;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = 1.0 + rsqrt_nr(s);
  t1 = clock64();
  cyc[3] = (t1 - t0);
  // 5. rcp_nr chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = 1.0 + rcp_nr(s);
  t1 = clock64();
  cyc[4] = (t1 - t0);
  // 6. plain double sqrt / div (IEEE)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = 1.0 + sqrt(s);
  t1 = clock64();
  cyc[5] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = 1.0 + 1.0 / s;
  t1 = clock64();
  cyc[6] = (t1 - t0);
  // 7. broadcast shuffle (idx) chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (i & 7)) * 0.999;
  t1 = clock64();
  cyc[7] = (t1 - t0);
  // 8. smem store -> load round trip (same warp, syncwarp)
  __shared__ double sh[64];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sh[lane] = x;
    __syncwarp();
    x = sh[(lane + 1) & 31] * 0.999;
    __syncwarp();
  }
  t1 = clock64();
  cyc[8] = (t1 - t0);
  out[threadIdx.x] = x + s;
}

int main() {
  double *out;
  long long *cyc, h[16];
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  const int it = 1000;
  k_lat<<<1, 32>>>(out, cyc, it);
  k_lat<<<1, 32>>>(out, cyc, it);
  cudaDeviceSynchronize();
  for (int i = 0; i < 9; ++i) h[i] = cyc[i];
  const char *nm[] = {"dfma dep", "shfl64+fma dep", "warp_sum8", "rsqrt_nr", "rcp_nr", "sqrt ieee", "div ieee",
                      "shfl idx dep", "sts+lds rt"};
  for (int i = 0; i < 9; ++i) printf("%-16s %7.1f cycles\n", nm[i], (double)h[i] / it);
  return 0;
}
