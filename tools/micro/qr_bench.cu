// Microbenchmark (not product code): the CTA path's blocked Householder QR
// (qr_blocked of csrc/ks_large.cu, included verbatim) on one shared-memory
// matrix per CTA, 8 warps, one CTA per SM; cycles per QR and per phase of
// CTA 0.  Shapes: stage 1 (96 x 97, 48 pivots) and stage 2 (96 x 145).
// Usage: qr_bench [rows] [npiv] [ncols] [ctas]
#include "../../paper_2502_11686_b200/csrc/ks_large.cu"
#include <cstring>
#include <cmath>

namespace ks {
namespace {
__global__ void __launch_bounds__(kThreads) qr_bench_kernel(int rows, int npiv, int ncols, int reps,
                                                            long long *cyc, double *out) {
  extern __shared__ __align__(16) double sm[];
  const int lda = ldpad(rows), cp = pad8(ncols) + 8;
  double *A = sm;
  QrWs w = carve_ws(sm + ((lda * cp + 1) & ~1));
  long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < lda * cp; i += blockDim.x) {
      const int r = i % lda, c = i / lda;
      const unsigned h = (unsigned)(r * 7919 + c * 104729 + blockIdx.x * 31 + rep * 13) * 2654435761u;
      A[i] = (r < rows && c < ncols) ? ((double)(h >> 8) / 16777216.0 - 0.5) : 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    qr_blocked(A, lda, rows, npiv, ncols, w);
    const long long t1 = clock64();
    tot += t1 - t0;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = tot / reps;
  if (threadIdx.x == 0) out[blockIdx.x] = A[0] + A[lda + 1];
}
__global__ void __launch_bounds__(kThreads) panel_bench_kernel(int rows, int reps, long long *cyc, double *out) {
  extern __shared__ __align__(16) double sm[];
  const int lda = ldpad(rows), cp = 16;
  double *A = sm;
  QrWs w = carve_ws(sm + ((lda * cp + 1) & ~1));
  for (int i = threadIdx.x; i < lda * cp; i += blockDim.x) {
    const int r = i % lda, c = i / lda;
    const unsigned h = (unsigned)(r * 7919 + c * 104729 + blockIdx.x * 31) * 2654435761u;
    A[i] = (r < rows) ? ((double)(h >> 8) / 16777216.0 - 0.5) : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
      qr_panel<3>(A, lda, 0, rows, 8, w.v1(0), w.beta(0), w.T(0), w.G);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = A[0] + A[lda + 1];
}
// stages 2 and 3 concurrently as in factor_level_kernel: B2 (r2 x c2, 48
// pivots) on warps [w3, 8), B3 (r3 x c3) on warps [0, w3)
__global__ void __launch_bounds__(kThreads) conc_bench_kernel(int r2, int c2, int r3, int c3, int w3, int reps,
                                                              long long *cyc, double *out) {
  extern __shared__ __align__(16) double sm[];
  const int ld2 = ldpad(r2), cp2 = pad8(c2) + 8, ld3 = ldpad(r3), cp3 = pad8(c3) + 8;
  double *A2 = sm, *A3 = sm + ((ld2 * cp2 + 1) & ~1);
  double *wsp = A3 + ((ld3 * cp3 + 1) & ~1);
  QrWs w2 = carve_ws(wsp), w3s = carve_ws(wsp + qr_ws_doubles(kWarps));
  long long tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = threadIdx.x; i < ld2 * cp2; i += blockDim.x) {
      const int r = i % ld2, c = i / ld2;
      const unsigned h = (unsigned)(r * 7919 + c * 104729 + blockIdx.x * 31 + rep * 13) * 2654435761u;
      A2[i] = (r < r2 && c < c2) ? ((double)(h >> 8) / 16777216.0 - 0.5) : 0.0;
    }
    for (int i = threadIdx.x; i < ld3 * cp3; i += blockDim.x) {
      const int r = i % ld3, c = i / ld3;
      const unsigned h = (unsigned)(r * 7919 + c * 104723 + blockIdx.x * 37 + rep * 11) * 2654435761u;
      A3[i] = (r < r3 && c < c3) ? ((double)(h >> 8) / 16777216.0 - 0.5) : 0.0;
    }
    __syncthreads();
    const long long t0 = clock64();
    if (w3 == 0) {
      qr_blocked(A2, ld2, r2, 48, c2, w2);
      qr_blocked(A3, ld3, r3, 48, c3, w3s);
    } else if ((int)(threadIdx.x >> 5) < w3) {
      qr_blocked(A3, ld3, r3, 48, c3, w3s, nullptr, 0, w3, 1);
    } else {
      qr_blocked(A2, ld2, r2, 48, c2, w2, nullptr, w3, kWarps - w3, 2);
    }
    __syncthreads();
    const long long t1 = clock64();
    tot += t1 - t0;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = tot / reps;
  if (threadIdx.x == 0) out[blockIdx.x] = A2[0] + A3[0];
}

// one QR of a seeded matrix, result copied out (for the host Gram check)
__global__ void __launch_bounds__(kThreads) qr_check_kernel(int rows, int npiv, int ncols, const double *in, double *res) {
  extern __shared__ __align__(16) double sm[];
  const int lda = ldpad(rows), cp = pad8(ncols) + 8;
  double *A = sm;
  QrWs w = carve_ws(sm + ((lda * cp + 1) & ~1));
  for (int i = threadIdx.x; i < lda * cp; i += blockDim.x) {
    const int r = i % lda, c = i / lda;
    A[i] = (r < rows && c < ncols) ? in[r + c * rows] : 0.0;
  }
  __syncthreads();
  qr_blocked(A, lda, rows, npiv, ncols, w);
  for (int i = threadIdx.x; i < rows * ncols; i += blockDim.x) res[i] = A[i % rows + (i / rows) * lda];
}
}  // namespace
}  // namespace ks

static int check(int rows, int npiv, int ncols, double collinear = 0.0) {
  const int lda = ks::ldpad(rows), cp = ks::pad8(ncols) + 8;
  const size_t smem = 8 * (size_t)(((lda * cp + 1) & ~1) + ks::qr_ws_doubles(ks::kWarps) + 64);
  const int ne = rows * ncols;
  double *h = (double *)malloc(8 * ne), *r = (double *)malloc(8 * ne), *din, *dres;
  unsigned x = 12345u + rows * 7 + ncols;
  for (int i = 0; i < ne; ++i) { x = x * 1664525u + 1013904223u; h[i] = (double)(x >> 8) / 16777216.0 - 0.5; }
  if (collinear > 0.0)   // every odd pivot column = the previous one + collinear * noise: the Gram guard fires
    for (int c = 1; c < npiv; c += 2)
      for (int r = 0; r < rows; ++r) h[r + c * rows] = h[r + (c - 1) * rows] + collinear * h[r + c * rows];
  cudaMalloc(&din, 8 * ne); cudaMalloc(&dres, 8 * ne);
  cudaMemcpy(din, h, 8 * ne, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(ks::qr_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ks::qr_check_kernel<<<1, ks::kThreads, smem>>>(rows, npiv, ncols, din, dres);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(r, dres, 8 * ne, cudaMemcpyDeviceToHost);
  double err = 0, sc = 0, low = 0;
  for (int a = 0; a < ncols; ++a)
    for (int b = 0; b < ncols; ++b) {
      double g0 = 0, g1 = 0;
      for (int i = 0; i < rows; ++i) { g0 += h[i + a * rows] * h[i + b * rows]; g1 += r[i + a * rows] * r[i + b * rows]; }
      err = fmax(err, fabs(g0 - g1)); sc = fmax(sc, fabs(g0));
    }
  for (int j = 0; j < npiv && j < ncols; ++j)
    for (int i = j + 1; i < rows; ++i) low = fmax(low, fabs(r[i + j * rows]));
  // |R_jj| against a plain host Householder QR (modified Gram-Schmidt-free,
  // column by column) of the same matrix: relative error per pivot
  double rdiag = 0.0;
  {
    double *A = (double *)malloc(8 * ne);
    memcpy(A, h, 8 * ne);
    for (int j = 0; j < npiv && j < rows; ++j) {
      double nx = 0.0;
      for (int i = j; i < rows; ++i) nx += A[i + j * rows] * A[i + j * rows];
      const double alpha = A[j + j * rows] > 0 ? -sqrt(nx) : sqrt(nx);
      const double v1 = A[j + j * rows] - alpha, vv = nx - A[j + j * rows] * A[j + j * rows] + v1 * v1;
      for (int c = j + 1; c < ncols; ++c) {
        double d = v1 * A[j + c * rows];
        for (int i = j + 1; i < rows; ++i) d += A[i + j * rows] * A[i + c * rows];
        d = vv > 0 ? 2.0 * d / vv : 0.0;
        A[j + c * rows] -= d * v1;
        for (int i = j + 1; i < rows; ++i) A[i + c * rows] -= d * A[i + j * rows];
      }
      const double got = fabs(r[j + j * rows]), ref = fabs(alpha);
      if (ref > 0) rdiag = fmax(rdiag, fabs(got - ref) / ref);
    }
    free(A);
  }
  unsigned long long rf[2] = {0, 0};
#ifdef KS_PANEL_PROF
  cudaMemcpyFromSymbol(rf, ks::g_refresh, sizeof(rf));
  unsigned long long zero[2] = {0, 0};
  cudaMemcpyToSymbol(ks::g_refresh, zero, sizeof(zero));
#endif
  printf("check %3d x %3d (%2d piv, collinear %.0e): gram err %.2e (rel %.2e), |R_jj| rel err %.1e, below-diag %.1e, "
         "refreshes %llu/%llu %s\n", rows, ncols, npiv, collinear, err, err / sc, rdiag, low, rf[0], rf[1],
         cudaGetErrorString(e));
  // tiny R_jj of near-dependent columns carry the inherent forward error eps / collinear
  return err / sc < 1e-13 && low == 0.0 && rdiag < (collinear > 0.0 ? 1e-14 / collinear : 1e-12);
}

int main(int argc, char **argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 96, npiv = argc > 2 ? atoi(argv[2]) : 48,
            ncols = argc > 3 ? atoi(argv[3]) : 97, ctas = argc > 4 ? atoi(argv[4]) : 148;
  const int lda = ks::ldpad(rows), cp = ks::pad8(ncols) + 8;
  const size_t smem = 8 * (size_t)(((lda * cp + 1) & ~1) + ks::qr_ws_doubles(ks::kWarps) + 64);
  long long *cyc;
  double *out;
  cudaMallocManaged(&cyc, 8);
  cudaMalloc(&out, 8 * ctas);
  cudaFuncSetAttribute(ks::qr_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (argc > 1 && argv[1][0] == 'c') {
    int ok = 1;
    const int cases[][3] = {{8, 6, 13}, {4, 6, 7}, {5, 6, 13}, {12, 6, 13}, {2, 1, 3}, {96, 48, 97}, {96, 48, 145},
                            {144, 48, 49}, {30, 9, 20}, {17, 16, 33}, {160, 64, 129}, {3, 3, 3}, {40, 20, 41}};
    for (auto &c : cases) ok &= check(c[0], c[1], c[2]);
    for (double cl : {1e-2, 1e-4, 1e-8}) ok &= check(96, 48, 97, cl);
    printf(ok ? "ALL OK\n" : "FAILURES\n");
    return !ok;
  }
  if (argc > 1 && argv[1][0] == 'x') {   // x w3: stage 2 (96 x 145) || stage 3 (96 x 49)
    const int w3 = atoi(argv[2]);
    const size_t sm2 = 8 * (size_t)(((ks::ldpad(96) * (ks::pad8(145) + 8) + 1) & ~1) +
                                    ((ks::ldpad(96) * (ks::pad8(49) + 8) + 1) & ~1) + 2 * ks::qr_ws_doubles(ks::kWarps) + 64);
    cudaFuncSetAttribute(ks::conc_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    ks::conc_bench_kernel<<<148, ks::kThreads, sm2>>>(96, 145, 96, 49, w3, 10, cyc, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("conc w3=%d: %lld cycles (%s)\n", w3, *cyc, cudaGetErrorString(e));
    return 0;
  }
  if (argc > 5) {
    cudaFuncSetAttribute(ks::panel_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ks::panel_bench_kernel<<<1, ks::kThreads, smem>>>(rows, 50, cyc, out);
    cudaDeviceSynchronize();
    printf("panel %d x 8 (MR 3): %lld cycles\n", rows, *cyc);
#ifdef KS_PANEL_PROF
    long long h[8];
    cudaMemcpyFromSymbol(h, ks::g_panel_clk, sizeof(h));
    printf("  gram %lld  load %lld  columns %lld  T %lld (per panel)\n", h[0] / 51, h[1] / 51, h[2] / 51, h[3] / 51);
#endif
    return 0;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ks::qr_bench_kernel<<<ctas, ks::kThreads, smem>>>(rows, npiv, ncols, 2, cyc, out);
  cudaEventRecord(e0);
  const int reps = 20;
  ks::qr_bench_kernel<<<ctas, ks::kThreads, smem>>>(rows, npiv, ncols, reps, cyc, out);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("qr %d x %d (%d pivots), %d CTAs, smem %zu B: %lld cycles/QR (CTA 0), %.2f us/QR wall, %s\n", rows, ncols,
         npiv, ctas, smem, *cyc, 1e3 * ms / reps, cudaGetErrorString(e));
  return 0;
}
// the library's per-device attribute helper (ks_api.cu), not linked here
cudaError_t ks::set_smem_attr(const void *f, int bytes) {
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
