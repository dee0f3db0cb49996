// Large-n path (the paper's third size n = m = 500 with
// k = 500 steps): block columns far larger than
// shared memory (a 500 x 500 fp64 block is 2 MB), so every block operation
// of a level is a BATCHED dense kernel over all the level's pairs at once,
// with the blocks in HBM / L2:
//   * big_gemm      strided-batched C = alpha op(A) op(B) + beta C on the FP64
//                   tensor cores (mma.sync.m8n8k4.f64, DMMA), 64 x 64 tiles,
//                   cp.async double-buffered operand staging;
//   * big_qr_panel  Householder panel factorisation (LAPACK geqrf order, the
//                   paper's QR) of 16 columns of every item, one
//                   CTA per item, writing the compact-WY factors V and
//                   U = V T^T so that Q^T C = C - U (V^T C) is two big_gemm;
//   * big_trsm_diag 64 x 64 triangular diagonal-block solves (the blocked
//                   TRSMs' off-diagonal parts are big_gemm);
//   * big_chol      Cholesky of the whitening blocks;
//   * big_copy      descriptor-driven batched block gathers / scatters that
//                   assemble the stacked stage matrices of P:424-537.
// The stage algebra is that of the small and CTA paths:
// stage 1 QR of [C_t; El_{t+1}] applied to [0 | y_t; Er_{t+1} | e_{t+1}],
// stage 2 QR of [Er_t; R~_t] applied to [El_t | 0 | e_t; 0 | X_t | z~_t],
// stage 3 QR of [D~_{t+1}; C_{t+1} (; Z)], and Alg. 2's SelInv backward.
// Time parallelism (pairs) is the batch dimension; within-block parallelism
// (the point of this workload) comes from the tiles of every
// GEMM and the rows of every panel.
#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <cstdlib>
#include <cstdio>

#include "ks_internal.cuh"
#include "ks_big.cuh"

namespace ks {
namespace big {

std::atomic<int64_t> g_launches{0};

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// 8-byte global -> shared asynchronous copy; !valid zero-fills (src-size 0:
// gsrc must still be a mapped address, callers pass the operand base)
__device__ __forceinline__ void cp8(double *sdst, const double *gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gsrc), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------------ GEMM ---
// Column-major operands; op(A) is M x K, op(B) is K x N.  CTA tile BM x BN,
// K chunks of BK in two shared-memory stages (cp.async), 8 warps, each warp a
// WTM x WTN block of DMMA 8x8 tiles.  Shared tiles are k-major with leading
// dimensions = 4 mod 16 doubles: the fragment loads (row g = lane/4,
// k = lane%4) of a half-warp hit 16 distinct 8-byte bank pairs.
//   <64, 64, 16, 32, 16>: the general shape;
//   <16, 256, 8, 16, 32>: W = V^T C of the compact-WY update (M = 16 rows).
template <bool TA, bool TB, int BM, int BN, int BK, int WTM, int WTN, bool SPLITK = false>
__global__ void __launch_bounds__(256) big_gemm_kernel(Gemm g, int kchunk) {
  constexpr int LDA = BM + 4, LDB = BN + 4, FM = WTM / 8, FN = WTN / 8, WM = BM / WTM;
  static_assert((BM / WTM) * (BN / WTN) == 8, "8 warps");
  static_assert((BN * BK) % 256 == 0, "whole B loads per thread");
  __shared__ __align__(16) double As[2][BK][LDA];
  __shared__ __align__(16) double Bs[2][BK][LDB];
  const int64_t b = blockIdx.z;
  const double *A = g.A + b * g.sA, *B = g.B + b * g.sB;
  double *C = g.C + b * g.sC;
  // SPLITK (one M tile): blockIdx.x selects the K range [kb, ke); the
  // partial products are added atomically into the zeroed C
  const int m0 = SPLITK ? 0 : blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb = SPLITK ? blockIdx.x * kchunk : 0;
  const int ke = SPLITK ? min(g.K, kb + kchunk) : g.K;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, q = lane & 3;
  const int wm = (warp % WM) * WTM, wn = (warp / WM) * WTN;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load = [&](int st, int k0) {
#pragma unroll
    for (int r = 0; r < (BM * BK + 255) / 256; ++r) {
      const int idx = tid + 256 * r;
      if (idx >= BM * BK) break;
      int m, k;
      if (TA) { m = idx / BK; k = idx % BK; } else { m = idx % BM; k = idx / BM; }
      const int gm = m0 + m, gk = k0 + k;
      const bool ok = gm < g.M && gk < ke;
      const double *src = TA ? A + gk + (int64_t)gm * g.lda : A + gm + (int64_t)gk * g.lda;
      cp8(&As[st][k][m], ok ? src : A, ok);
    }
#pragma unroll
    for (int r = 0; r < BN * BK / 256; ++r) {
      const int idx = tid + 256 * r;
      int nn, k;
      if (TB) { nn = idx % BN; k = idx / BN; } else { nn = idx / BK; k = idx % BK; }
      const int gn = n0 + nn, gk = k0 + k;
      const bool ok = gn < g.N && gk < ke;
      const double *src = TB ? B + gn + (int64_t)gk * g.ldb : B + gk + (int64_t)gn * g.ldb;
      cp8(&Bs[st][k][nn], ok ? src : B, ok);
    }
    cp_commit();
  };
  const int nk = (ke - kb + BK - 1) / BK;
  if (nk <= 0) return;
  load(0, kb);
  // beta != 0: the old C tile into registers now, so that its loads overlap
  // the k loop instead of serialising the epilogue (K is often just 16-64)
  double cold[FM][FN][2];
  const bool useb = !SPLITK && g.beta != 0.0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + gq, n = n0 + wn + 8 * j + 2 * q + h;
        cold[i][j][h] = (useb && m < g.M && n < g.N) ? C[m + (int64_t)n * g.ldc] : 0.0;
      }
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < nk) {
      load(st ^ 1, kb + (kt + 1) * BK);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = As[st][kk + q][wm + 8 * i + gq];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = Bs[st][kk + q][wn + 8 * j + gq];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int m = m0 + wm + 8 * i + gq;
      if (m >= g.M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn + 8 * j + 2 * q + h;
        if (n >= g.N) continue;
        double *c = C + m + (int64_t)n * g.ldc;
        if (SPLITK) atomicAdd(c, g.alpha * acc[i][j][h]);
        else *c = useb ? fma(g.alpha, acc[i][j][h], g.beta * cold[i][j][h]) : g.alpha * acc[i][j][h];
      }
    }
}

template <bool TA, bool TB>
cudaError_t gemm_launch(const Gemm &g, cudaStream_t s) {
  if (g.M <= 16) {
    // W = V^T C of the compact-WY update: 16 rows, K = the stack's rows.
    // Split K over CTAs (128 per CTA) when it is long: one column tile per
    // item alone would serialise the whole reduction
    constexpr int KC = 128;
    const int ns = (g.K + KC - 1) / KC;
    if (ns > 1 && g.beta == 0.0 && g.sC >= (int64_t)g.ldc * g.N) {
      const cudaError_t e = cudaMemset2DAsync(g.C, (size_t)g.sC * 8, 0, (size_t)g.ldc * g.N * 8, (size_t)g.batch, s);
      if (e != cudaSuccess) return e;
      const dim3 grid((unsigned)ns, (g.N + 255) / 256, (unsigned)g.batch);
      big_gemm_kernel<TA, TB, 16, 256, 8, 16, 32, true><<<grid, 256, 0, s>>>(g, KC);
    } else {
      const dim3 grid(1, (g.N + 255) / 256, (unsigned)g.batch);
      big_gemm_kernel<TA, TB, 16, 256, 8, 16, 32><<<grid, 256, 0, s>>>(g, 0);
    }
  } else if (g.M <= 64 && g.K >= 512 && g.beta == 0.0 && g.sC >= (int64_t)g.ldc * g.N) {
    // V^T C / V^T V of the block reflector (64 rows, K = the stack's rows): split K
    constexpr int KC = 256;
    const int ns = (g.K + KC - 1) / KC;
    const cudaError_t e = cudaMemset2DAsync(g.C, (size_t)g.sC * 8, 0, (size_t)g.ldc * g.N * 8, (size_t)g.batch, s);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)ns, (g.N + 63) / 64, (unsigned)g.batch);
    big_gemm_kernel<TA, TB, 64, 64, 16, 32, 16, true><<<grid, 256, 0, s>>>(g, KC);
  } else {
    const dim3 grid((g.M + 63) / 64, (g.N + 63) / 64, (unsigned)g.batch);
    big_gemm_kernel<TA, TB, 64, 64, 16, 32, 16><<<grid, 256, 0, s>>>(g, 0);
  }
  return cudaSuccess;
}

cudaError_t gemm(const Gemm &g, bool ta, bool tb, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
  if (g.K <= 0 && g.beta == 1.0) return cudaSuccess;
  cudaError_t e;
  if (ta && tb) e = gemm_launch<true, true>(g, s);
  else if (ta) e = gemm_launch<true, false>(g, s);
  else if (tb) e = gemm_launch<false, true>(g, s);
  else e = gemm_launch<false, false>(g, s);
  ++g_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ------------------------------------------------------------------ copy ---
// Batched block copies: for every descriptor d and item b,
//   dst[b sd + r + c ldd] = alpha * (src ? src[b ss + (T ? c + r lds : r + c lds)] : 0)
// (column-major; T: transpose; upper: entries below the diagonal are 0).
__global__ void __launch_bounds__(256) big_copy_kernel(CopyList L, int64_t batch) {
  const CopyDesc &d = L.d[blockIdx.y];
  const int64_t total = (int64_t)d.rows * d.cols;
  const int64_t per = total * (batch > 0 ? batch : 1);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < per;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / total, e = idx - b * total;
    if (b >= d.count) continue;
    const int c = (int)(e / d.rows), r = (int)(e - (int64_t)c * d.rows);
    double v = (d.diag != 0.0 && r == c) ? d.diag : 0.0;
    if (d.src && !(d.upper && r > c)) {
      const double *s = d.src + b * d.ss;
      v = d.alpha * (d.trans ? s[c + (int64_t)r * d.lds] : s[r + (int64_t)c * d.lds]);
    }
    d.dst[b * d.sd + r + (int64_t)c * d.ldd] = v;
  }
}

cudaError_t copy(const CopyList &L, int64_t batch, cudaStream_t s) {
  if (L.count == 0 || batch <= 0) return cudaSuccess;
  int64_t mx = 0;
  for (int i = 0; i < L.count; ++i) mx = mx > (int64_t)L.d[i].rows * L.d[i].cols ? mx : (int64_t)L.d[i].rows * L.d[i].cols;
  const int64_t work = mx * batch;
  const unsigned gx = (unsigned)((work + 255) / 256 < 4096 ? (work + 255) / 256 : 4096);
  big_copy_kernel<<<dim3(gx > 0 ? gx : 1, (unsigned)L.count), 256, 0, s>>>(L, batch);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------ QR panel ---
// Columns [j0, j0 + nb) of the item's stack S (m rows, ld lds), rows j0..m-1,
// factored in shared memory by Householder reflections (LAPACK dgeqr2 order:
// beta = -sign(alpha) |x|, v_0 = 1, tau = (beta - alpha) / beta).  Writes the
// R part back (zeros below the diagonal), the explicit V (rows x nb, unit
// lower trapezoidal) and U = V T^T (the compact-WY T of dlarft, forward
// columnwise), so that Q^T C = C - U (V^T C).  One CTA per item.
constexpr int kPanelThreads = 512;
__device__ double block_sum(double v, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// CTA-wide sums of NV per-thread values at once (one shuffle tree per value,
// one barrier pair): out[v] valid in every thread.
// (red: (threads / 32) x NV partials, then NV totals)
template <int NV>
__device__ __forceinline__ void block_sums(double (&acc)[NV], double *red) {
  constexpr int NW = kPanelThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int v = 0; v < NV; ++v) red[warp * NV + v] = acc[v];
  __syncthreads();
  if (threadIdx.x < NV) {   // one thread per value sums the warps' partials
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w * NV + threadIdx.x];
    red[NW * NV + threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = red[NW * NV + v];
}

// CTA-wide sums of 16 per-thread values plus one more: a warp reduce-scatter
// (16 shuffles instead of 16 x 5: each exchange step halves the values a
// lane keeps), one partial per (warp, value) in shared memory, then one
// thread per value sums the warps -- and, in the same step, threads < 16
// copy row j of the panel (rowj) so that every thread reads it from the
// copy: no thread can see the row after its owner has updated it.
// On exit acc[v] (v < 17) and pj[v] (v < 16) are valid in every thread.
__device__ __forceinline__ void block_sums17(double (&acc)[17], double *red, const double *rowj, int ldr, int nb,
                                             double (&pj)[16]) {
  constexpr int NW = kPanelThreads / 32;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) acc[16] += __shfl_xor_sync(full, acc[16], o);
#pragma unroll
  for (int h = 8, bit = 16; h >= 1; h >>= 1, bit >>= 1) {
    const bool up = (lane & bit) != 0;
#pragma unroll
    for (int v = 0; v < h; ++v) {
      const double send = up ? acc[v] : acc[v + h];
      const double keep = up ? acc[v + h] : acc[v];
      acc[v] = keep + __shfl_xor_sync(full, send, bit);
    }
  }
  acc[0] += __shfl_xor_sync(full, acc[0], 1);
  const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  if ((lane & 1) == 0) red[warp * 17 + idx] = acc[0];
  if (lane == 1) red[warp * 17 + 16] = acc[16];
  __syncthreads();
  if (threadIdx.x < 17) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w * 17 + threadIdx.x];
    red[NW * 17 + threadIdx.x] = t;
    if (threadIdx.x < 16) red[NW * 17 + 17 + threadIdx.x] = threadIdx.x < nb ? rowj[(size_t)threadIdx.x * ldr] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 17; ++v) acc[v] = red[NW * 17 + v];
#pragma unroll
  for (int v = 0; v < 16; ++v) pj[v] = red[NW * 17 + 17 + v];
}

__global__ void __launch_bounds__(kPanelThreads) big_qr_panel_kernel(Panel a) {
  extern __shared__ __align__(16) double psm[];
  const int64_t b = blockIdx.x;
  double *S = a.S + b * a.sS;
  double *V = a.V + b * a.sV, *U = a.U + b * a.sU;
  const int rows = a.m - a.j0, nb = a.nb, tid = threadIdx.x;
  double *P = psm;                      // [nb][rows] column-major (ld = rows)
  double *red = P + (size_t)nb * rows;  // reductions: (threads / 32) x 17 partials, 17 totals, row j
  double *T = red + (kPanelThreads / 32 + 2) * 17;   // [nb][nb] column-major
  double *tau = T + kBigNB * kBigNB;
  // the panel into shared memory (asynchronous copies: all of a thread's
  // loads in flight at once)
  for (int64_t e = tid; e < (int64_t)nb * rows; e += blockDim.x) {
    const int c = (int)(e / rows), r = (int)(e - (int64_t)c * rows);
    cp8(&P[e], S + (a.j0 + r) + (int64_t)(a.j0 + c) * a.lds, true);
  }
  cp_commit();
  cp_wait0();
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    double *x = P + (size_t)j * rows;
    // ONE pass and ONE reduction per column (on the unscaled x = P[:, j]):
    //   acc[16] = sum_{r > j} x_r^2                     (the norm)
    //   acc[c]  = sum_{r > j} x_r P[r][c], c != j      (scaled below by 1/(alpha - beta))
    // giving v^T P[:, c] for c > j (the reflector's dots) and (V^T v_j)_c
    // for c < j (those columns already hold v_c: dlarft's T column)
    double acc[17], pj[16];
#pragma unroll
    for (int c = 0; c < 17; ++c) acc[c] = 0.0;
    for (int r = j + 1 + tid; r < rows; r += blockDim.x) {
      const double xr = x[r];
      acc[16] = fma(xr, xr, acc[16]);
#pragma unroll
      for (int c = 0; c < kBigNB; ++c)
        if (c < nb && c != j) acc[c] = fma(xr, P[r + (size_t)c * rows], acc[c]);
    }
    block_sums17(acc, red, P + j, rows, nb, pj);
    double alpha = 0.0;   // P[j][j] (from the copy: compile-time indices, no local memory)
#pragma unroll
    for (int v = 0; v < 16; ++v)
      if (v == j) alpha = pj[v];
    const double sigma = acc[16];
    double tj = 0.0, beta = alpha, scal = 0.0;
    if (sigma > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, sigma)), alpha);
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    // w_c = v^T P[:, c] = P[j][c] + scal acc[c] (v_j = 1); y_c likewise for c < j
#pragma unroll
    for (int c = 0; c < kBigNB; ++c) acc[c] = fma(scal, acc[c], pj[c]);
    // T[0:j, j] = -tau_j T[0:j, 0:j] y  (dlarft, forward columnwise): row i of T
    // is written and read only by thread i, so no barrier is needed for it
    if (tid < j) {
      double sv = 0.0;
#pragma unroll
      for (int k = 0; k < kBigNB; ++k)
        if (k >= tid && k < j) sv = fma(T[tid + k * kBigNB], acc[k], sv);
      T[tid + j * kBigNB] = -tj * sv;
    }
    // H_j applied to the columns c > j: P[:, c] -= tau v w_c, and v stored
    for (int r = j + tid; r < rows; r += blockDim.x) {
      const double vr = (r == j) ? 1.0 : scal * x[r];
#pragma unroll
      for (int c = 0; c < kBigNB; ++c)
        if (c > j && c < nb) P[r + (size_t)c * rows] = fma(-tj * acc[c], vr, P[r + (size_t)c * rows]);
      x[r] = (r == j) ? beta : vr;
    }
    if (tid == j) T[j + j * kBigNB] = tj;
    if (tid == 0) {
      tau[j] = tj;
      a.tau[b * a.stau + j] = tj;
    }
    __syncthreads();
  }
  // write back: R (upper part of the panel's first nb rows), zeros below; V, U = V T^T
  for (int64_t e = tid; e < (int64_t)nb * rows; e += blockDim.x) {
    const int c = (int)(e / rows), r = (int)(e - (int64_t)c * rows);
    const double pv = P[e];
    S[(a.j0 + r) + (int64_t)(a.j0 + c) * a.lds] = (r <= c) ? pv : 0.0;
    V[r + (int64_t)c * a.ldv] = (r < c) ? 0.0 : (r == c ? 1.0 : pv);
  }
  for (int r = tid; r < rows; r += blockDim.x) {
    double vr[kBigNB];
#pragma unroll
    for (int c = 0; c < kBigNB; ++c) vr[c] = (c < nb) ? ((r < c) ? 0.0 : (r == c ? 1.0 : P[r + (size_t)c * rows])) : 0.0;
#pragma unroll
    for (int c = 0; c < kBigNB; ++c) {
      if (c >= nb) break;
      double sv = 0.0;   // (V T^T)[r][c] = sum_{k >= c} V[r][k] T[c][k]
#pragma unroll
      for (int k = 0; k < kBigNB; ++k)
        if (k >= c && k < nb) sv = fma(vr[k], T[c + k * kBigNB], sv);
      U[r + (int64_t)c * a.ldu] = sv;
    }
  }
}

// The panel held in REGISTERS: thread t owns rows t, t + 256, ... (MR of
// them) of all 16 columns, so the per-column passes are register FMAs (no
// shared-memory traffic, no address arithmetic) and only the reduction, the
// pivot row and T go through shared memory.  Same arithmetic as above, one
// pass and one reduction per column; columns unrolled (every register index
// is a compile-time constant).
constexpr int kRegPanelThreads = 256;
__device__ __forceinline__ void block_sums17r(double (&acc)[17], double *red) {
  constexpr int NW = kRegPanelThreads / 32;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) acc[16] += __shfl_xor_sync(full, acc[16], o);
#pragma unroll
  for (int h = 8, bit = 16; h >= 1; h >>= 1, bit >>= 1) {
    const bool up = (lane & bit) != 0;
#pragma unroll
    for (int v = 0; v < h; ++v) {
      const double send = up ? acc[v] : acc[v + h];
      const double keep = up ? acc[v + h] : acc[v];
      acc[v] = keep + __shfl_xor_sync(full, send, bit);
    }
  }
  acc[0] += __shfl_xor_sync(full, acc[0], 1);
  const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  if ((lane & 1) == 0) red[warp * 17 + idx] = acc[0];
  if (lane == 1) red[warp * 17 + 16] = acc[16];
  __syncthreads();
  if (threadIdx.x < 17) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w * 17 + threadIdx.x];
    red[NW * 17 + threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 17; ++v) acc[v] = red[NW * 17 + v];
}

template <int MR>
__global__ void __launch_bounds__(kRegPanelThreads, 1) big_qr_panel_reg_kernel(Panel a) {
  constexpr int NB = kBigNB, TH = kRegPanelThreads, NW = TH / 32;
  __shared__ double red[(NW + 1) * 17];
  __shared__ double rowj[2][NB];       // the pivot row, double-buffered by column parity
  __shared__ double T[NB * NB];
  const int64_t b = blockIdx.x;
  double *S = a.S + b * a.sS;
  double *V = a.V + b * a.sV, *U = a.U + b * a.sU;
  const int rows = a.m - a.j0, nb = a.nb, tid = threadIdx.x;
  double p[MR][NB];
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const int ri = tid + TH * r;
#pragma unroll
    for (int c = 0; c < NB; ++c)
      p[r][c] = (ri < rows && c < nb) ? S[(a.j0 + ri) + (int64_t)(a.j0 + c) * a.lds] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (j >= nb) break;
    double acc[17];
#pragma unroll
    for (int c = 0; c < 17; ++c) acc[c] = 0.0;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int ri = tid + TH * r;
      if (ri > j && ri < rows) {
        const double xr = p[r][j];
        acc[16] = fma(xr, xr, acc[16]);
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c != j) acc[c] = fma(xr, p[r][c], acc[c]);
      }
      if (ri == j)   // the pivot row's owner publishes it (read after the reduction's barriers)
#pragma unroll
        for (int c = 0; c < NB; ++c) rowj[j & 1][c] = p[r][c];
    }
    block_sums17r(acc, red);
    const double alpha = rowj[j & 1][j], sigma = acc[16];
    double tj = 0.0, beta = alpha, scal = 0.0;
    if (sigma > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, sigma)), alpha);
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    // w_c = v^T P[:, c] (c > j), (V^T v_j)_c (c < j)
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[c] = fma(scal, acc[c], rowj[j & 1][c]);
    if (tid < j) {   // T[0:j, j] = -tau_j T[0:j, 0:j] (V^T v_j)  (dlarft); row tid of T is this thread's
      double sv = 0.0;
#pragma unroll
      for (int k = 0; k < NB; ++k)
        if (k >= tid && k < j) sv = fma(T[tid + k * NB], acc[k], sv);
      T[tid + j * NB] = -tj * sv;
    }
    if (tid == j) T[j + j * NB] = tj;
    if (tid == 0) a.tau[b * a.stau + j] = tj;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int ri = tid + TH * r;
      if (ri >= j && ri < rows) {
        const double vr = (ri == j) ? 1.0 : scal * p[r][j];
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c > j) p[r][c] = fma(-tj * acc[c], vr, p[r][c]);
        p[r][j] = (ri == j) ? beta : vr;
      }
    }
  }
  __syncthreads();   // T complete
  // write back: R (upper part, zeros below), V (explicit), U = V T^T
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const int ri = tid + TH * r;
    if (ri >= rows) continue;
    double vr[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const double pv = p[r][c];
      vr[c] = (c < nb) ? ((ri < c) ? 0.0 : (ri == c ? 1.0 : pv)) : 0.0;
      if (c < nb) {
        S[(a.j0 + ri) + (int64_t)(a.j0 + c) * a.lds] = (ri <= c) ? pv : 0.0;
        V[ri + (int64_t)c * a.ldv] = vr[c];
      }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c >= nb) break;
      double sv = 0.0;   // (V T^T)[ri][c] = sum_{k >= c} V[ri][k] T[c][k]
#pragma unroll
      for (int k = 0; k < NB; ++k)
        if (k >= c && k < nb) sv = fma(vr[k], T[c + k * NB], sv);
      U[ri + (int64_t)c * a.ldu] = sv;
    }
  }
}

template <int MR>
cudaError_t qr_panel_reg(const Panel &a, int64_t batch, cudaStream_t s) {
  big_qr_panel_reg_kernel<MR><<<(unsigned)batch, kRegPanelThreads, 0, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

size_t panel_smem(int rows) {
  return sizeof(double) * ((size_t)kBigNB * rows + (kPanelThreads / 32 + 2) * 17 + kBigNB * kBigNB + 2 * kBigNB);
}

cudaError_t qr_panel(const Panel &a, int64_t batch, cudaStream_t s) {
  const int rows = a.m - a.j0, mr = (rows + kRegPanelThreads - 1) / kRegPanelThreads;
  if (!std::getenv("KS_SMEM_PANEL")) {   // the register-resident panel (default)
    switch (mr) {
      case 0: case 1: return qr_panel_reg<1>(a, batch, s);
      case 2: return qr_panel_reg<2>(a, batch, s);
      case 3: return qr_panel_reg<3>(a, batch, s);
      case 4: return qr_panel_reg<4>(a, batch, s);
      case 5: return qr_panel_reg<5>(a, batch, s);
      case 6: return qr_panel_reg<6>(a, batch, s);
      default: break;   // taller panels: the shared-memory kernel
    }
  }
  const size_t sm = panel_smem(a.m - a.j0);
  cudaError_t e = set_smem_attr((const void *)big_qr_panel_kernel, (int)panel_smem(kBigMaxRows));
  if (e != cudaSuccess) return e;
  if ((e = set_carveout_max((const void *)big_qr_panel_kernel)) != cudaSuccess) return e;
  big_qr_panel_kernel<<<(unsigned)batch, kPanelThreads, sm, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------- triangular diagonal ---
// In place X = T^{-1} X for the nb x nb diagonal block T = R[j0:j0+nb, j0:j0+nb]
// (upper: back substitution; lower: forward), X = B[j0:j0+nb, 0:k]; one
// thread per right-hand-side column, the block staged in shared memory.
// In place X = T^{-1} X for the nb x nb (nb <= 64) diagonal block
// T = R[j0:j0+nb, j0:j0+nb] (upper: back substitution; lower: forward),
// X = B[j0:j0+nb, 0:k]: one WARP per right-hand-side column (lane l holds
// rows l and l + 32), column-oriented: x_i from its owner lane, broadcast by
// a shuffle, then every lane updates its remaining rows; the block is staged
// in shared memory.
__global__ void __launch_bounds__(256) big_trsm_diag_kernel(Trsm a, int j0, int nb) {
  __shared__ double Ts[64][65];
  const int64_t b = blockIdx.y;
  const double *R = a.R + b * a.sR;
  double *B = a.B + b * a.sB;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int c = e / nb, r = e - c * nb;
    Ts[r][c] = R[(j0 + r) + (int64_t)(j0 + c) * a.ldr];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (col >= a.k) return;
  double *x = B + j0 + (int64_t)col * a.ldb;
  double x0 = lane < nb ? x[lane] : 0.0, x1 = lane + 32 < nb ? x[lane + 32] : 0.0;
  if (a.upper) {
    for (int i = nb - 1; i >= 0; --i) {
      const double own = (i < 32) ? x0 : x1;
      const double xi = __shfl_sync(0xffffffffu, own, i & 31) / Ts[i][i];
      if (i < 32) { if (lane == i) x0 = xi; } else if (lane == i - 32) x1 = xi;
      if (lane < i) x0 = fma(-Ts[lane][i], xi, x0);
      if (lane + 32 < i) x1 = fma(-Ts[lane + 32][i], xi, x1);
    }
  } else {
    for (int i = 0; i < nb; ++i) {
      const double own = (i < 32) ? x0 : x1;
      const double xi = __shfl_sync(0xffffffffu, own, i & 31) / Ts[i][i];
      if (i < 32) { if (lane == i) x0 = xi; } else if (lane == i - 32) x1 = xi;
      if (lane > i && lane < nb) x0 = fma(-Ts[lane][i], xi, x0);
      if (lane + 32 > i && lane + 32 < nb) x1 = fma(-Ts[lane + 32][i], xi, x1);
    }
  }
  if (lane < nb) x[lane] = x0;
  if (lane + 32 < nb) x[lane + 32] = x1;
}

// Blocked triangular solve X = R^{-1} B (n x n triangular, B n x k), in place.
cudaError_t trsm(const Trsm &a, int n, int64_t batch, cudaStream_t s) {
  const int BS = 64;
  const int nblk = (n + BS - 1) / BS;
  for (int t = 0; t < nblk; ++t) {
    const int jb = a.upper ? nblk - 1 - t : t;
    const int j0 = jb * BS, nb = (n - j0 < BS) ? n - j0 : BS;
    big_trsm_diag_kernel<<<dim3((a.k + 7) / 8, (unsigned)batch), 256, 0, s>>>(a, j0, nb);
  ++g_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // eliminate the solved block from the remaining rows
    Gemm g;
    g.batch = batch;
    g.N = a.k; g.K = nb; g.alpha = -1.0; g.beta = 1.0;
    g.B = a.B + j0; g.ldb = a.ldb; g.sB = a.sB;
    g.lda = a.ldr; g.sA = a.sR; g.ldc = a.ldb; g.sC = a.sB;
    if (a.upper) {   // rows 0..j0-1 -= R[0:j0, j0:j0+nb] X_jb
      g.M = j0; g.A = a.R + (int64_t)j0 * a.ldr; g.C = a.B;
    } else {         // rows j0+nb..n-1 -= R[j0+nb:n, j0:j0+nb] X_jb
      g.M = n - j0 - nb; g.A = a.R + (j0 + nb) + (int64_t)j0 * a.ldr; g.C = a.B + j0 + nb;
    }
    if (g.M > 0 && (e = gemm(g, false, false, s)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------ Cholesky ---
// In place lower Cholesky of the leading d x d block of every item
// (column-major, ld), right-looking, one CTA per item; the strict upper
// triangle is zeroed.  A pivot <= 0 is recorded (status, step = item index
// + step_off) and replaced by 1 (outputs undefined, as on the other paths).
__global__ void __launch_bounds__(256) big_chol_kernel(double *A, int64_t sA, int ld, int d, int chol_given,
                                                        unsigned long long *status, int64_t step_off, int kind,
                                                        int64_t step_mul) {
  __shared__ double red[32];
  __shared__ double piv;
  double *M = A + (int64_t)blockIdx.x * sA;
  const int tid = threadIdx.x;
  bool bad = false;
  for (int j = 0; j < d; ++j) {
    if (!chol_given) {
      double part = 0.0;
      for (int k = tid; k < j; k += blockDim.x) part = fma(M[j + (int64_t)k * ld], M[j + (int64_t)k * ld], part);
      const double s = block_sum(part, red);
      if (tid == 0) {
        double dj = M[j + (int64_t)j * ld] - s;
        if (!(dj > 0.0)) { bad = true; dj = 1.0; }
        piv = sqrt(dj);
        M[j + (int64_t)j * ld] = piv;
      }
      __syncthreads();
      const double il = 1.0 / piv;
      for (int r = j + 1 + tid; r < d; r += blockDim.x) {
        double v = M[r + (int64_t)j * ld];
        for (int k = 0; k < j; ++k) v = fma(-M[r + (int64_t)k * ld], M[j + (int64_t)k * ld], v);
        M[r + (int64_t)j * ld] = v * il;
      }
      __syncthreads();
    } else if (tid == 0) {   // KS_COV_IS_CHOL: the factor is given
      const double v = M[j + (int64_t)j * ld];
      if (!(v != 0.0 && v - v == 0.0)) { bad = true; M[j + (int64_t)j * ld] = 1.0; }
    }
  }
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)d * d; e += blockDim.x) {
    const int c = (int)(e / d), r = (int)(e - (int64_t)c * d);
    if (r < c) M[r + (int64_t)c * ld] = 0.0;
  }
  if (tid == 0 && bad && status)
    atomicMin(status, status_word((int64_t)blockIdx.x * step_mul + step_off, kind));
}

// Blocked (left-looking) Cholesky, 64-column block columns: the block column
// A[j0:d, j0:j0+jb] -= L[j0:d, 0:j0] L[j0:j0+jb, 0:j0]^T (big_gemm), then
// the diagonal block factored in shared memory (big_chol_diag) and the rows
// below solved against it (big_trsm_right: X L11^T = A21).
__global__ void __launch_bounds__(256) big_chol_diag_kernel(double *A, int64_t sA, int ld, int j0, int jb,
                                                             unsigned long long *status, int64_t step_off, int kind,
                                                             int64_t step_mul) {
  __shared__ double Ls[64][65];
  double *M = A + (int64_t)blockIdx.x * sA;
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int c = e / jb, r = e - c * jb;
    Ls[r][c] = M[(j0 + r) + (int64_t)(j0 + c) * ld];
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < jb; ++j) {
    if (threadIdx.x == 0) {
      double dj = Ls[j][j];
      for (int k = 0; k < j; ++k) dj = fma(-Ls[j][k], Ls[j][k], dj);
      if (!(dj > 0.0)) { bad = 1; dj = 1.0; }
      Ls[j][j] = sqrt(dj);
    }
    __syncthreads();
    const double il = 1.0 / Ls[j][j];
    for (int r = j + 1 + threadIdx.x; r < jb; r += blockDim.x) {
      double v = Ls[r][j];
      for (int k = 0; k < j; ++k) v = fma(-Ls[r][k], Ls[j][k], v);
      Ls[r][j] = v * il;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int c = e / jb, r = e - c * jb;
    M[(j0 + r) + (int64_t)(j0 + c) * ld] = (r >= c) ? Ls[r][c] : 0.0;
  }
  if (threadIdx.x == 0 && bad && status)
    atomicMin(status, status_word((int64_t)blockIdx.x * step_mul + step_off, kind));
}
__global__ void __launch_bounds__(256) big_trsm_right_kernel(double *A, int64_t sA, int ld, int j0, int jb, int d) {
  __shared__ double Ls[64][65];
  double *M = A + (int64_t)blockIdx.y * sA;
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int c = e / jb, r = e - c * jb;
    Ls[r][c] = M[(j0 + r) + (int64_t)(j0 + c) * ld];
  }
  __syncthreads();
  const int r = j0 + jb + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d) return;
  double xv[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) xv[c] = (c < jb) ? M[r + (int64_t)(j0 + c) * ld] : 0.0;
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    if (c >= jb) break;
    double v = xv[c];
#pragma unroll
    for (int k = 0; k < c; ++k) v = fma(-xv[k], Ls[c][k], v);
    xv[c] = v / Ls[c][c];
  }
#pragma unroll
  for (int c = 0; c < 64; ++c)
    if (c < jb) M[r + (int64_t)(j0 + c) * ld] = xv[c];
}
__global__ void big_zero_upper_kernel(double *A, int64_t sA, int ld, int d) {
  double *M = A + (int64_t)blockIdx.y * sA;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)d * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / d), r = (int)(e - (int64_t)c * d);
    if (r < c) M[r + (int64_t)c * ld] = 0.0;
  }
}

cudaError_t chol(double *A, int64_t sA, int ld, int d, int64_t batch, bool given, unsigned long long *status,
                 int64_t step_off, int64_t step_mul, int kind, cudaStream_t s) {
  if (batch <= 0 || d <= 0) return cudaSuccess;
  if (given) {   // KS_COV_IS_CHOL: check the diagonal, clear the upper triangle
    big_chol_kernel<<<(unsigned)batch, 256, 0, s>>>(A, sA, ld, d, 1, status, step_off, kind, step_mul);
    ++g_launches;
    return cudaGetLastError();
  }
  cudaError_t e;
  for (int j0 = 0; j0 < d; j0 += 64) {
    const int jb = (d - j0 < 64) ? d - j0 : 64;
    if (j0 > 0) {
      Gemm g;
      g.batch = batch; g.M = d - j0; g.N = jb; g.K = j0; g.alpha = -1.0; g.beta = 1.0;
      g.A = A + j0; g.lda = ld; g.sA = sA; g.B = A + j0; g.ldb = ld; g.sB = sA;
      g.C = A + j0 + (int64_t)j0 * ld; g.ldc = ld; g.sC = sA;
      if ((e = gemm(g, false, true, s)) != cudaSuccess) return e;
    }
    big_chol_diag_kernel<<<(unsigned)batch, 256, 0, s>>>(A, sA, ld, j0, jb, status, step_off, kind, step_mul);
    ++g_launches;
    if (d - j0 - jb > 0) {
      big_trsm_right_kernel<<<dim3((d - j0 - jb + 255) / 256, (unsigned)batch), 256, 0, s>>>(A, sA, ld, j0, jb, d);
      ++g_launches;
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  big_zero_upper_kernel<<<dim3((unsigned)(((int64_t)d * d + 255) / 256 < 256 ? ((int64_t)d * d + 255) / 256 : 256),
                               (unsigned)batch), 256, 0, s>>>(A, sA, ld, d);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------- helpers ---
// Sum of squares of an rows x cols block per item -> out[b * so] (+= if acc).
__global__ void __launch_bounds__(256) big_sumsq_kernel(const double *A, int64_t sA, int lda, int rows, int cols,
                                                         double *out, int64_t so, int acc) {
  __shared__ double red[32];
  const double *M = A + (int64_t)blockIdx.x * sA;
  double part = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)rows * cols; e += blockDim.x) {
    const int c = (int)(e / rows), r = (int)(e - (int64_t)c * rows);
    const double v = M[r + (int64_t)c * lda];
    part = fma(v, v, part);
  }
  const double s = block_sum(part, red);
  if (threadIdx.x == 0) out[(int64_t)blockIdx.x * so] = acc ? out[(int64_t)blockIdx.x * so] + s : s;
}
cudaError_t sumsq(const double *A, int64_t sA, int lda, int rows, int cols, double *out, int64_t so, bool acc,
                  int64_t batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  big_sumsq_kernel<<<(unsigned)batch, 256, 0, s>>>(A, sA, lda, rows, cols, out, so, acc ? 1 : 0);
  ++g_launches;
  return cudaGetLastError();
}

// Rank test of the eliminated columns: |R_tt[d][d]| <=
// 1e-12 |block column of UA|_F -> KS_ERR_RANK at the column's step.
__global__ void big_rank_kernel(const double *R, int64_t sR, int ldr, int n, const double *nrm2, int64_t snrm,
                                unsigned long long *status, int64_t step_first, int64_t step_stride) {
  const int64_t b = blockIdx.x;
  const double *M = R + b * sR;
  const double ref = sqrt(nrm2[b * snrm]);
  bool bad = false;
  for (int d = threadIdx.x; d < n; d += blockDim.x) bad |= !(fabs(M[d + (int64_t)d * ldr]) > kRankTol * ref);
  if (__syncthreads_or(bad) && threadIdx.x == 0)
    atomicMin(status, status_word(step_first + b * step_stride, kBadRank));
}
cudaError_t rank_check(const double *R, int64_t sR, int ldr, int n, const double *nrm2, int64_t snrm,
                       unsigned long long *status, int64_t step_first, int64_t step_stride, int64_t batch,
                       cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  big_rank_kernel<<<(unsigned)batch, 128, 0, s>>>(R, sR, ldr, n, nrm2, snrm, status, step_first, step_stride);
  ++g_launches;
  return cudaGetLastError();
}

// dst = (A + A^T) / 2 (n x n, column-major in, row-major == column-major out)
__global__ void big_sym_kernel(const double *A, int64_t sA, int lda, double *dst, int64_t sd, int n) {
  const int64_t b = blockIdx.y;
  const double *M = A + b * sA;
  double *D = dst + b * sd;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)n * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n), r = (int)(e - (int64_t)c * n);
    D[e] = 0.5 * (M[r + (int64_t)c * lda] + M[c + (int64_t)r * lda]);
  }
}
cudaError_t sym_store(const double *A, int64_t sA, int lda, double *dst, int64_t sd, int n, int64_t batch,
                      cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const unsigned gx = (unsigned)(((int64_t)n * n + 255) / 256 < 64 ? ((int64_t)n * n + 255) / 256 : 64);
  big_sym_kernel<<<dim3(gx, (unsigned)batch), 256, 0, s>>>(A, sA, lda, dst, sd, n);
  ++g_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------- blocked Householder ---
// T of a block reflector of nb <= 64 columns from G = V^T V and tau (dlarft,
// forward columnwise): T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j], T[j][j] = tau_j.
__global__ void __launch_bounds__(256) big_larft_kernel(const double *G, double *T, int64_t sGT, const double *tau,
                                                        int64_t stau, int nb) {
  // one array: T in the strict upper triangle, tau on the diagonal, G's
  // strict upper triangle stored transposed in the strict lower one
  __shared__ double Ts[64][65], taus[64];
  const int64_t b = blockIdx.x;
  const double *Gb = G + b * sGT;
  const int i = threadIdx.x;
  // (256 threads stage G: 16 independent loads each, all in flight)
#pragma unroll 4
  for (int e = i; e < nb * nb; e += blockDim.x) {
    const int c = e / nb, r = e - c * nb;
    if (r < c) Ts[c][r] = __ldg(Gb + r + (int64_t)c * kBigBlk);   // G[r][c] -> Ts[c][r]
  }
  if (i < nb) taus[i] = tau[b * stau + i];
  __syncthreads();
  if (i >= 64) return;   // the recurrence: one thread per row of T
  for (int j = 0; j < nb; ++j) {
    const double tj = taus[j];
    if (i < j) {
      double sv = 0.0;
      for (int k = i; k < j; ++k) sv = fma(Ts[i][k], Ts[j][k], sv);   // T[i][k] G[k][j]
      Ts[i][j] = -tj * sv;
    }
    if (i == j) Ts[j][j] = tj;
    asm volatile("bar.sync 1, 64;" ::: "memory");   // the 64 recurrence threads only
  }
  double *Tb = T + b * sGT;
  for (int e = i; e < kBigBlk * kBigBlk; e += 64) {
    const int c = e / kBigBlk, r = e - c * kBigBlk;
    Tb[e] = (r <= c && c < nb) ? Ts[r][c] : 0.0;
  }
}

// In place QR of the first ncols_fac columns of every item's S (m x ncols,
// ld lds), Q^T applied to all the item's remaining columns (the stage's RHS
// blocks).  Blocks of 64 columns: four 16-column big_qr_panel calls, each
// followed by its update of the block's remaining columns (W = V16^T C,
// C -= U16 W), then the block reflector I - V T V^T of all 64 (T from
// G = V^T V, big_larft) updates the trailing columns with two big GEMMs,
// W = V^T C and C -= (V T^T) W: one read and one read-write of the trailing
// matrix per 64 columns instead of per 16.
// Lookahead (w.side): the block reflector first updates only the NEXT
// block's 64 columns on the calling stream, which then goes on to factor
// that block, while the rest of the trailing update runs on the side stream
// (own W, the block's V / U kept in the alternate buffers) -- the sequential
// panels and the bandwidth-bound trailing GEMMs overlap.  The calling stream
// joins the side stream before the next block's own reflector touches the
// trailing columns.
cudaError_t qr_apply(double *S, int64_t sS, int lds, int m, int ncols_fac, int ncols, int64_t batch,
                     const Work &w, cudaStream_t s) {
  const int kmax = ncols_fac < m ? ncols_fac : m;
  cudaError_t e;
  bool pending = false;   // a side-stream trailing update not yet joined
  for (int J0 = 0, blk = 0; J0 < kmax; J0 += kBigBlk, ++blk) {
    const int nbB = (kmax - J0 < kBigBlk) ? kmax - J0 : kBigBlk, rowsB = m - J0;
    double *V = (w.side && (blk & 1)) ? w.V2 : w.V, *U = (w.side && (blk & 1)) ? w.U2 : w.U;
    // the block's V (rows m - J0, zero above each panel's diagonal)
    if ((e = cudaMemset2DAsync(V, (size_t)w.sVU * 8, 0, (size_t)w.ldv * nbB * 8, (size_t)batch, s)) != cudaSuccess)
      return e;
    for (int sub = 0; sub < nbB; sub += kBigNB) {
      const int j0 = J0 + sub, nb = (nbB - sub < kBigNB) ? nbB - sub : kBigNB;
      Panel p;
      p.S = S; p.sS = sS; p.lds = lds; p.m = m; p.j0 = j0; p.nb = nb;
      p.V = V + sub + (int64_t)sub * w.ldv; p.sV = w.sVU; p.ldv = w.ldv;   // rows from j0 = row sub of the block
      p.U = w.U16; p.sU = w.sU16; p.ldu = w.ldv;
      p.tau = w.tau + sub; p.stau = w.stau;
      if ((e = qr_panel(p, batch, s)) != cudaSuccess) return e;
      const int nin = nbB - sub - nb, rows = m - j0;
      if (nin <= 0) continue;
      double *C = S + j0 + (int64_t)(j0 + nb) * lds;   // the block's later columns
      Gemm g1;   // W = V16^T C
      g1.batch = batch; g1.M = nb; g1.N = nin; g1.K = rows; g1.alpha = 1.0; g1.beta = 0.0;
      g1.A = p.V; g1.lda = w.ldv; g1.sA = w.sVU;
      g1.B = C; g1.ldb = lds; g1.sB = sS;
      g1.C = w.W; g1.ldc = kBigBlk; g1.sC = w.sW;
      if ((e = gemm(g1, true, false, s)) != cudaSuccess) return e;
      Gemm g2;   // C -= U16 W
      g2.batch = batch; g2.M = rows; g2.N = nin; g2.K = nb; g2.alpha = -1.0; g2.beta = 1.0;
      g2.A = w.U16; g2.lda = w.ldv; g2.sA = w.sU16;
      g2.B = w.W; g2.ldb = kBigBlk; g2.sB = w.sW;
      g2.C = C; g2.ldc = lds; g2.sC = sS;
      if ((e = gemm(g2, false, false, s)) != cudaSuccess) return e;
    }
    // the previous block's trailing update (side stream) must be done before
    // this block's reflector updates the trailing columns
    if (pending) {
      if ((e = cudaStreamWaitEvent(s, w.evj, 0)) != cudaSuccess) return e;
      pending = false;
    }
    const int nc = ncols - (J0 + nbB);
    if (nc <= 0) continue;
    // the block reflector: G = V^T V, T (dlarft), U = V T^T
    Gemm gg;
    gg.batch = batch; gg.M = nbB; gg.N = nbB; gg.K = rowsB; gg.A = V; gg.lda = w.ldv; gg.sA = w.sVU;
    gg.B = V; gg.ldb = w.ldv; gg.sB = w.sVU; gg.C = w.G; gg.ldc = kBigBlk; gg.sC = w.sGT;
    if ((e = gemm(gg, true, false, s)) != cudaSuccess) return e;
    big_larft_kernel<<<(unsigned)batch, 256, 0, s>>>(w.G, w.T, w.sGT, w.tau, w.stau, nbB);
    ++g_launches;
    Gemm gu;
    gu.batch = batch; gu.M = rowsB; gu.N = nbB; gu.K = nbB; gu.A = V; gu.lda = w.ldv; gu.sA = w.sVU;
    gu.B = w.T; gu.ldb = kBigBlk; gu.sB = w.sGT; gu.C = U; gu.ldc = w.ldv; gu.sC = w.sVU;
    if ((e = gemm(gu, false, true, s)) != cudaSuccess) return e;
    // trailing columns [c0, c0 + nc): with lookahead, the next block's
    // columns (those it will factor) here, the rest on the side stream
    const int c0 = J0 + nbB;
    const bool la = w.side && J0 + nbB < kmax && nc > kBigBlk;
    const int nnow = la ? kBigBlk : nc;
    auto update = [&](int cb, int cn, double *W, cudaStream_t st) -> cudaError_t {
      double *C = S + J0 + (int64_t)cb * lds;
      Gemm g1;   // W = V^T C  (nbB x cn)
      g1.batch = batch; g1.M = nbB; g1.N = cn; g1.K = rowsB; g1.alpha = 1.0; g1.beta = 0.0;
      g1.A = V; g1.lda = w.ldv; g1.sA = w.sVU;
      g1.B = C; g1.ldb = lds; g1.sB = sS;
      g1.C = W; g1.ldc = kBigBlk; g1.sC = w.sW;
      cudaError_t ee = gemm(g1, true, false, st);
      if (ee != cudaSuccess) return ee;
      Gemm g2;   // C -= U W
      g2.batch = batch; g2.M = rowsB; g2.N = cn; g2.K = nbB; g2.alpha = -1.0; g2.beta = 1.0;
      g2.A = U; g2.lda = w.ldv; g2.sA = w.sVU;
      g2.B = W; g2.ldb = kBigBlk; g2.sB = w.sW;
      g2.C = C; g2.ldc = lds; g2.sC = sS;
      return gemm(g2, false, false, st);
    };
    if (la) {   // fork: the rest of the trailing update beside the next block's panels
      if ((e = cudaEventRecord(w.evf, s)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(w.side, w.evf, 0)) != cudaSuccess) return e;
      if ((e = update(c0 + nnow, nc - nnow, w.Wt, w.side)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(w.evj, w.side)) != cudaSuccess) return e;
      pending = true;
    }
    if ((e = update(c0, nnow, w.W, s)) != cudaSuccess) return e;
  }
  if (pending && (e = cudaStreamWaitEvent(s, w.evj, 0)) != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace big
}  // namespace ks

// =================================================================== plan ===
namespace ks {
namespace big {

int64_t entry_doubles_big(int n) { return 3ll * n * n + 2ll * n + 1; }
int64_t rrec_doubles_big(int n) { return 3ll * n * n + n; }

namespace {

// one descriptor: copy an rows x cols block for `count` items
CopyDesc cd(const double *src, int64_t ss, int lds, double *dst, int64_t sd, int ldd, int rows, int cols, int64_t count,
            double alpha = 1.0, int trans = 0, int upper = 0, double diag = 0.0) {
  CopyDesc d;
  d.src = src; d.ss = ss; d.lds = lds; d.dst = dst; d.sd = sd; d.ldd = ldd;
  d.rows = rows; d.cols = cols; d.count = count; d.alpha = alpha; d.trans = trans; d.upper = upper; d.diag = diag;
  return d;
}

cudaError_t run(CopyList &L, cudaStream_t s) {
  int64_t mx = 0;
  for (int i = 0; i < L.count; ++i) mx = L.d[i].count > mx ? L.d[i].count : mx;
  cudaError_t e = copy(L, mx, s);
  L.count = 0;
  return e;
}

// level-0 masks of the observation blocks (per-step m_i): rows / columns
// >= m_i of Lw -> identity, rows >= m_i of Hw -> 0 (then the solves give
// exactly zero rows there)
__global__ void big_mask_obs_kernel(double *Lw, double *Hw, const int32_t *m, int mx, int ncols, int64_t sL, int64_t sH) {
  const int64_t i = blockIdx.x;
  const int mi = m[i];
  double *L = Lw + i * sL, *H = Hw + i * sH;
  for (int64_t e = threadIdx.x; e < (int64_t)mx * mx; e += blockDim.x) {
    const int c = (int)(e / mx), r = (int)(e - (int64_t)c * mx);
    if (r >= mi || c >= mi) L[e] = (r == c) ? 1.0 : 0.0;
  }
  for (int64_t e = threadIdx.x; e < (int64_t)mx * ncols; e += blockDim.x) {
    const int r = (int)(e % mx);
    if (r >= mi) H[e] = 0.0;
  }
}

// nrm0[t] = |C_t|^2 + |Er_t|^2 [t has an evolution row] + |El_{t+1}|^2
__global__ void big_nrm0_kernel(const double *nC, int64_t sCn, const double *nEr, const double *nEl, int64_t sEn,
                                int64_t N, double *out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N) return;
  double v = nC[t * sCn] + nEr[t * sEn];
  if (t + 1 < N) v += nEl[(t + 1) * sEn];
  out[t] = v;
}

}  // namespace

// rows of the stage stacks for C-like blocks of r rows (stage 3 and the
// single-column QRs are padded with zero rows up to n)
int64_t rows1(int n, int r) { return (int64_t)r + n; }
int64_t rows3(int n, int r, bool odd) { const int64_t v = 2ll * r + (odd ? n : 0); return v > n ? v : n; }

void scratch_sizes(const Plan &p, int64_t &s1, int64_t &s2, int64_t &s3, int64_t &vu, int64_t &w, int64_t &items) {
  const int64_t n = p.n, r = p.RC > p.n ? p.RC : p.n;   // level 0: RC rows, then n
  items = p.N / 2 + 1;
  s1 = rows1(n, r) * (2 * n + 1);
  s2 = (2 * n) * (3 * n + 1);
  s3 = rows3(n, r, true) * (n + 1);
  int64_t rows = rows1(n, r);
  if (2 * n > rows) rows = 2 * n;
  if (rows3(n, r, true) > rows) rows = rows3(n, r, true);
  vu = rows * kBigBlk;
  w = kBigBlk * (3 * n + 1);
}
int64_t max_stack_rows(int n, int RC) {
  const int r = RC > n ? RC : n;
  int64_t rows = rows1(n, r);
  if (2 * n > rows) rows = 2 * n;
  if (rows3(n, r, true) > rows) rows = rows3(n, r, true);
  return rows;
}

// ------------------------------------------------------------- whiten ---
// K_i = Lam Lam^T, L_i = M M^T; El = -Lam^{-1} F,
// Er = Lam^{-1}, e = Lam^{-1} c, C = M^{-1} H, y = M^{-1} o: batched
// Cholesky + blocked triangular solves on column-major copies.
cudaError_t whiten(const Plan &p, cudaStream_t s) {
  const int n = p.n, mx = p.mx;
  const int64_t nn = (int64_t)n * n;
  cudaError_t e;
  CopyList L;
  // evolution blocks (row-major inputs -> column-major: transposed copies)
  const int64_t cE = p.cntE;
  const int64_t sBw = (int64_t)n * (2 * n + 1);
  L.add(cd(p.K, p.sK, n, p.Kw, nn, n, n, n, cE, 1.0, 1));
  L.add(cd(p.F, p.sF, n, p.Bw, sBw, n, n, n, cE, 1.0, 1));
  L.add(cd(nullptr, 0, 1, p.Bw + nn, sBw, n, n, n, cE, 1.0, 0, 0, 1.0));   // identity
  L.add(cd(p.c, p.sc, 1, p.Bw + 2 * nn, sBw, n, n, 1, p.c ? cE : 0));
  L.add(cd(nullptr, 0, 1, p.Bw + 2 * nn, sBw, n, n, 1, p.c ? 0 : cE));
  if ((e = run(L, s)) != cudaSuccess) return e;
  if (cE > 1) {   // steps without an evolution row: K -> I (never factored as data), F, c -> 0
    const int64_t cnt = (p.N + p.seg - 1) / p.seg;
    L.add(cd(nullptr, 0, 1, p.Kw, p.seg * nn, n, n, n, cnt, 1.0, 0, 0, 1.0));
    L.add(cd(nullptr, 0, 1, p.Bw, p.seg * sBw, n, n, n, cnt));
    L.add(cd(nullptr, 0, 1, p.Bw + 2 * nn, p.seg * sBw, n, n, 1, cnt));
    if ((e = run(L, s)) != cudaSuccess) return e;
  }
  // (constant model: the step reported for a bad K is 1, the first step using it)
  if ((e = chol(p.Kw, nn, n, n, cE, p.chol, p.status, cE == 1 ? 1 : 0, 1, kBadK, s)) != cudaSuccess) return e;
  Trsm t;
  t.R = p.Kw; t.sR = nn; t.ldr = n; t.B = p.Bw; t.sB = sBw; t.ldb = n; t.k = 2 * n + 1; t.upper = 0;
  if ((e = trsm(t, n, cE, s)) != cudaSuccess) return e;
  L.add(cd(p.Bw, sBw, n, p.El0, nn, n, n, n, cE, -1.0));
  L.add(cd(p.Bw + nn, sBw, n, p.Er0, nn, n, n, n, cE));
  L.add(cd(p.Bw + 2 * nn, sBw, n, p.e0, n, n, n, 1, cE));
  if ((e = run(L, s)) != cudaSuccess) return e;
  // no evolution row at the first step of every problem (global step 0, batch segments)
  if (cE > 1) {
    const int64_t cnt = (p.N + p.seg - 1) / p.seg;
    L.add(cd(nullptr, 0, 1, p.El0, p.seg * nn, n, n, n, cnt));
    L.add(cd(nullptr, 0, 1, p.Er0, p.seg * nn, n, n, n, cnt));
    L.add(cd(nullptr, 0, 1, p.e0, p.seg * n, n, n, 1, cnt));
    if ((e = run(L, s)) != cudaSuccess) return e;
  } else if (p.N == 1) {
    L.add(cd(nullptr, 0, 1, p.El0, 0, n, n, n, 1));
    L.add(cd(nullptr, 0, 1, p.Er0, 0, n, n, n, 1));
    L.add(cd(nullptr, 0, 1, p.e0, 0, n, n, 1, 1));
    if ((e = run(L, s)) != cudaSuccess) return e;
  }
  if ((e = sumsq(p.Er0, nn, n, n, n, p.nEr, 1, false, cE, s)) != cudaSuccess) return e;
  if ((e = sumsq(p.El0, nn, n, n, n, p.nEl, 1, false, cE, s)) != cudaSuccess) return e;
  // observation blocks
  if (mx > 0) {
    const int64_t cC = p.cntC, mm = (int64_t)mx * mx;
    const int64_t sHw = (int64_t)mx * (n + 1);
    L.add(cd(p.L, p.sL, mx, p.Lw, mm, mx, mx, mx, cC, 1.0, 1));
    L.add(cd(p.H, p.sH, n, p.Hw, sHw, mx, mx, n, cC, 1.0, 1));
    if (!p.constC) L.add(cd(p.o, p.so, 1, p.Hw + (int64_t)mx * n, sHw, mx, mx, 1, cC));
    if ((e = run(L, s)) != cudaSuccess) return e;
    if (p.m) {
      big_mask_obs_kernel<<<(unsigned)cC, 256, 0, s>>>(p.Lw, p.Hw, p.m, mx, n + 1, mm, sHw);
  ++g_launches;
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if ((e = chol(p.Lw, mm, mx, mx, cC, p.chol, p.status, 0, 1, kBadL, s)) != cudaSuccess) return e;
    t.R = p.Lw; t.sR = mm; t.ldr = mx; t.B = p.Hw; t.sB = sHw; t.ldb = mx; t.k = p.constC ? n : n + 1; t.upper = 0;
    if ((e = trsm(t, mx, cC, s)) != cudaSuccess) return e;
    L.add(cd(p.Hw, sHw, mx, p.C0, (int64_t)mx * n, mx, mx, n, cC));
    if (!p.constC) L.add(cd(p.Hw + (int64_t)mx * n, sHw, mx, p.y0, mx, mx, mx, 1, cC));
    else L.add(cd(p.o, 0, (int)p.so, p.y0, 0, mx, mx, (int)p.N, 1));   // o^T as mx x N, ld so
    if ((e = run(L, s)) != cudaSuccess) return e;
    if (p.constC) {   // y = M^{-1} [o_0 .. o_{N-1}]: one solve with N right-hand sides
      t.R = p.Lw; t.sR = 0; t.ldr = mx; t.B = p.y0; t.sB = 0; t.ldb = mx; t.k = (int)p.N; t.upper = 0;
      if ((e = trsm(t, mx, 1, s)) != cudaSuccess) return e;
    }
    if ((e = sumsq(p.C0, (int64_t)mx * n, mx, mx, n, p.nC, 1, false, cC, s)) != cudaSuccess) return e;
  } else {
    if ((e = cudaMemsetAsync(p.nC, 0, sizeof(double), s)) != cudaSuccess) return e;
  }
  big_nrm0_kernel<<<(unsigned)((p.N + 255) / 256), 256, 0, s>>>(p.nC, p.cntC > 1 ? 1 : 0, p.nEr, p.nEl,
                                                                p.cntE > 1 ? 1 : 0, p.N, p.nrm0);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------- factor ---
namespace {

// column accessors of level L (0: whitened level-0 arrays; >= 1: entries)
struct Cols {
  const double *C, *y, *El, *Er, *e, *nrm;
  int64_t sC, sy, sE, se, snrm;   // per-column strides (0: constant block)
  int ldC, r;
};
Cols level_cols(const Plan &p, size_t L) {
  Cols c;
  const int n = p.n;
  const int64_t nn = (int64_t)n * n;
  if (L == 0) {
    c.C = p.C0; c.sC = p.cntC > 1 ? (int64_t)p.RC * n : 0; c.ldC = p.RC > 0 ? p.RC : 1; c.r = p.RC;
    c.y = p.y0; c.sy = p.RC;
    c.El = p.El0; c.Er = p.Er0; c.sE = p.cntE > 1 ? nn : 0;
    c.e = p.e0; c.se = p.cntE > 1 ? n : 0;
    c.nrm = p.nrm0; c.snrm = 1;
  } else {
    const int64_t E = entry_doubles_big(n);
    const double *b = p.ent[L];
    c.C = b; c.sC = E; c.ldC = n; c.r = n;
    c.y = b + nn; c.sy = E;
    c.El = b + nn + n; c.Er = b + 2 * nn + n; c.sE = E;
    c.e = b + 3 * nn + n; c.se = E;
    c.nrm = b + 3 * nn + 2 * n; c.snrm = E;
  }
  return c;
}

// post-processing of eliminated columns whose stage-2 stack top rows hold
// [R | R_l | R_r | z] (items [0, cnt) of S2): rank test, T = R^{-1}[R_l R_r z],
// P = R^{-1} R^{-T}, into the records
cudaError_t post(const Plan &p, size_t L, const double *nrm, int64_t snrm, int64_t cnt, double *rec,
                 int64_t step_first, int64_t step_stride, cudaStream_t s) {
  const int n = p.n;
  const int64_t nn = (int64_t)n * n, ld2 = 2 * n, s2 = ld2 * (3 * n + 1), Rr = rrec_doubles_big(n);
  cudaError_t e = rank_check(p.S2, s2, (int)ld2, n, nrm, snrm, p.status, step_first, step_stride, cnt, s);
  if (e != cudaSuccess) return e;
  Trsm t;
  t.R = p.S2; t.sR = s2; t.ldr = (int)ld2; t.B = p.S2 + (int64_t)n * ld2; t.sB = s2; t.ldb = (int)ld2;
  t.k = 2 * n + 1; t.upper = 1;
  if ((e = trsm(t, n, cnt, s)) != cudaSuccess) return e;
  CopyList Lc;
  Lc.add(cd(nullptr, 0, 1, p.Rinv, nn, n, n, n, cnt, 1.0, 0, 0, 1.0));
  if ((e = run(Lc, s)) != cudaSuccess) return e;
  t.B = p.Rinv; t.sB = nn; t.ldb = n; t.k = n;
  if ((e = trsm(t, n, cnt, s)) != cudaSuccess) return e;
  Gemm g;   // P = R^{-1} R^{-T}
  g.batch = cnt; g.M = n; g.N = n; g.K = n; g.A = p.Rinv; g.lda = n; g.sA = nn; g.B = p.Rinv; g.ldb = n; g.sB = nn;
  g.C = rec + 2 * nn + n; g.ldc = n; g.sC = Rr;
  if ((e = gemm(g, false, true, s)) != cudaSuccess) return e;
  Lc.add(cd(p.S2 + (int64_t)n * ld2, s2, (int)ld2, rec, Rr, n, n, n, cnt));           // T_l
  Lc.add(cd(p.S2 + (int64_t)2 * n * ld2, s2, (int)ld2, rec + nn, Rr, n, n, n, cnt));  // T_r
  Lc.add(cd(p.S2 + (int64_t)3 * n * ld2, s2, (int)ld2, rec + 2 * nn, Rr, n, n, 1, cnt));  // w
  return run(Lc, s);
}

}  // namespace

cudaError_t factor(const Plan &p, cudaStream_t s) {
  const int n = p.n;
  const int64_t nn = (int64_t)n * n, E = entry_doubles_big(n), Rr = rrec_doubles_big(n);
  cudaError_t e;
  CopyList Lc;
  for (size_t L = 0; L < p.Ks.size(); ++L) {
    const int64_t K = p.Ks[L];
    const Cols c = level_cols(p, L);
    const int r = c.r;
    const int ld1 = r + n, ld2 = 2 * n;
    const int64_t s1 = (int64_t)ld1 * (2 * n + 1), s2 = (int64_t)ld2 * (3 * n + 1);
    const int rb = r > n ? r : n;   // single-column stacks: zero rows up to n
    if (K == 1) {   // base case: R_00 = qr(C_0), w = R^{-1} z
      Lc.add(cd(nullptr, 0, 1, p.S1, 0, ld1, ld1, n + 1, 1));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      Lc.add(cd(c.C, 0, c.ldC, p.S1, 0, ld1, r, n, 1));
      Lc.add(cd(c.y, 0, 1, p.S1 + (int64_t)n * ld1, 0, ld1, r, 1, 1));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      if ((e = qr_apply(p.S1, s1, ld1, rb, n, n + 1, 1, p.w, s)) != cudaSuccess) return e;
      Lc.add(cd(p.S1, 0, ld1, p.S2, 0, ld2, n, n, 1, 1.0, 0, 1));
      Lc.add(cd(nullptr, 0, 1, p.S2 + (int64_t)n * ld2, 0, ld2, n, 2 * n, 1));
      Lc.add(cd(p.S1 + (int64_t)n * ld1, 0, ld1, p.S2 + (int64_t)3 * n * ld2, 0, ld2, n, 1, 1));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      if ((e = post(p, L, c.nrm, 0, 1, p.rec[L], ((int64_t)1 << L) - 1, 0, s)) != cudaSuccess) return e;
      break;
    }
    const int64_t P = K / 2;
    const bool odd = (K & 1) != 0;
    const int ld3 = (int)rows3(n, r, odd);
    const int64_t s3 = (int64_t)ld3 * (n + 1);
    // ---- stage 1 (pairs): [C_t; El_u | 0; Er_u | y_t; e_u], t = 2p, u = 2p + 1 ----
    Lc.add(cd(c.C, 2 * c.sC, c.ldC, p.S1, s1, ld1, r, n, P));
    Lc.add(cd(c.El + c.sE, 2 * c.sE, n, p.S1 + r, s1, ld1, n, n, P));
    Lc.add(cd(nullptr, 0, 1, p.S1 + (int64_t)n * ld1, s1, ld1, r, n, P));
    Lc.add(cd(c.Er + c.sE, 2 * c.sE, n, p.S1 + (int64_t)n * ld1 + r, s1, ld1, n, n, P));
    Lc.add(cd(c.y, 2 * c.sy, 1, p.S1 + (int64_t)2 * n * ld1, s1, ld1, r, 1, P));
    Lc.add(cd(c.e + c.se, 2 * c.se, 1, p.S1 + (int64_t)2 * n * ld1 + r, s1, ld1, n, 1, P));
    if (odd) {   // the last column (no right neighbour): [C_t | y_t] in item P (zero rows up to n)
      const int64_t t = K - 1;
      if (r < n) {
        Lc.add(cd(nullptr, 0, 1, p.S1 + P * s1, 0, ld1, ld1, n + 1, 1));
        if ((e = run(Lc, s)) != cudaSuccess) return e;
      }
      Lc.add(cd(c.C + t * c.sC, 0, c.ldC, p.S1 + P * s1, 0, ld1, r, n, 1));
      Lc.add(cd(c.y + t * c.sy, 0, 1, p.S1 + P * s1 + (int64_t)n * ld1, 0, ld1, r, 1, 1));
    }
    if ((e = run(Lc, s)) != cudaSuccess) return e;
    if ((e = qr_apply(p.S1, s1, ld1, ld1, n, 2 * n + 1, P, p.w, s)) != cudaSuccess) return e;
    if (odd) {
      Work w1 = p.w;
      w1.V += P * p.w.sVU; w1.U += P * p.w.sVU; w1.U16 += P * p.w.sU16; w1.W += P * p.w.sW;
      w1.G += P * p.w.sGT; w1.T += P * p.w.sGT; w1.tau += P * p.w.stau;
      w1.V2 += P * p.w.sVU; w1.U2 += P * p.w.sVU; w1.Wt += P * p.w.sW;
      // [C_t | y_t] sits in columns 0..n of item P (ld ld1): factor its r rows, apply to column n
      if ((e = qr_apply(p.S1 + P * s1, s1, ld1, rb, n, n + 1, 1, w1, s)) != cudaSuccess) return e;
    }
    // ---- stage 2 (eliminated t = 2p, p >= 1; + the odd level's last column as item P) ----
    // [Er_t | El_t | 0 | e_t ; R~_t | 0 | X_t | z~_t]
    {
      const int64_t cnt = P - 1;
      double *S2b = p.S2 + s2;   // item 1
      const double *S1b = p.S1 + s1;
      Lc.add(cd(c.Er + 2 * c.sE, 2 * c.sE, n, S2b, s2, ld2, n, n, cnt));
      Lc.add(cd(S1b, s1, ld1, S2b + n, s2, ld2, n, n, cnt, 1.0, 0, 1));
      Lc.add(cd(c.El + 2 * c.sE, 2 * c.sE, n, S2b + (int64_t)n * ld2, s2, ld2, n, n, cnt));
      Lc.add(cd(nullptr, 0, 1, S2b + (int64_t)n * ld2 + n, s2, ld2, n, n, cnt));
      Lc.add(cd(nullptr, 0, 1, S2b + (int64_t)2 * n * ld2, s2, ld2, n, n, cnt));
      Lc.add(cd(S1b + (int64_t)n * ld1, s1, ld1, S2b + (int64_t)2 * n * ld2 + n, s2, ld2, n, n, cnt));
      Lc.add(cd(c.e + 2 * c.se, 2 * c.se, 1, S2b + (int64_t)3 * n * ld2, s2, ld2, n, 1, cnt));
      Lc.add(cd(S1b + (int64_t)2 * n * ld1, s1, ld1, S2b + (int64_t)3 * n * ld2 + n, s2, ld2, n, 1, cnt));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
    }
    if (odd) {   // item P: the last column, X = 0
      const int64_t t = K - 1;
      double *S2l = p.S2 + P * s2;
      const double *S1l = p.S1 + P * s1;
      Lc.add(cd(c.Er + t * c.sE, 0, n, S2l, 0, ld2, n, n, 1));
      Lc.add(cd(S1l, 0, ld1, S2l + n, 0, ld2, n, n, 1, 1.0, 0, 1));
      Lc.add(cd(c.El + t * c.sE, 0, n, S2l + (int64_t)n * ld2, 0, ld2, n, n, 1));
      Lc.add(cd(nullptr, 0, 1, S2l + (int64_t)n * ld2 + n, 0, ld2, n, n, 1));
      Lc.add(cd(nullptr, 0, 1, S2l + (int64_t)2 * n * ld2, 0, ld2, 2 * n, n, 1));
      Lc.add(cd(c.e + t * c.se, 0, 1, S2l + (int64_t)3 * n * ld2, 0, ld2, n, 1, 1));
      Lc.add(cd(S1l + (int64_t)n * ld1, 0, ld1, S2l + (int64_t)3 * n * ld2 + n, 0, ld2, n, 1, 1));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
    }
    // item 0 (t = 0, no left neighbour: "nothing to do"): R = R~, R_r = X, z = z~; no coupling row
    Lc.add(cd(p.S1, 0, ld1, p.S2, 0, ld2, n, n, 1, 1.0, 0, 1));
    Lc.add(cd(nullptr, 0, 1, p.S2 + n, 0, ld2, n, n, 1));
    Lc.add(cd(nullptr, 0, 1, p.S2 + (int64_t)n * ld2, 0, ld2, 2 * n, n, 1));
    Lc.add(cd(p.S1 + (int64_t)n * ld1, 0, ld1, p.S2 + (int64_t)2 * n * ld2, 0, ld2, n, n, 1));
    Lc.add(cd(nullptr, 0, 1, p.S2 + (int64_t)2 * n * ld2 + n, 0, ld2, n, n, 1));
    Lc.add(cd(p.S1 + (int64_t)2 * n * ld1, 0, ld1, p.S2 + (int64_t)3 * n * ld2, 0, ld2, n, 1, 1));
    Lc.add(cd(nullptr, 0, 1, p.S2 + (int64_t)3 * n * ld2 + n, 0, ld2, n, 1, 1));
    if ((e = run(Lc, s)) != cudaSuccess) return e;
    // Stages 2 and 3 are independent once stage 1 is done, except
    // that an odd level's stage 3 takes the last column's stage-2 Z rows: on
    // even levels stage 3 runs on the second stream (its own QR scratch)
    // concurrently with stage 2 and the records.
    const bool conc = !odd && p.s2 != nullptr;
    auto stage2 = [&]() -> cudaError_t {
      if (P - 1 + (odd ? 1 : 0) > 0)
        return qr_apply(p.S2 + s2, s2, ld2, ld2, n, 3 * n + 1, P - 1 + (odd ? 1 : 0), p.w, s);
      return cudaSuccess;
    };
    if (!conc && (e = stage2()) != cudaSuccess) return e;
    cudaStream_t s3s = s;
    const Work *w3 = &p.w;
    if (conc) {
      if ((e = cudaEventRecord(p.ev[0], s)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(p.s2, p.ev[0], 0)) != cudaSuccess) return e;
      s3s = p.s2;
      w3 = &p.w2;
    }
    // ---- stage 3 (survivors u = 2p + 1): [D~_u; C_u (; Z_{K-1}) | y~; y_u (; z^)] ----
    if (ld3 > 2 * r) {   // Z rows (odd level) / zero padding up to n rows
      Lc.add(cd(nullptr, 0, 1, p.S3 + 2 * r, s3, ld3, ld3 - 2 * r, n + 1, P));
      if ((e = run(Lc, s3s)) != cudaSuccess) return e;
    }
    Lc.add(cd(p.S1 + (int64_t)n * ld1 + n, s1, ld1, p.S3, s3, ld3, r, n, P));
    Lc.add(cd(p.S1 + (int64_t)2 * n * ld1 + n, s1, ld1, p.S3 + (int64_t)n * ld3, s3, ld3, r, 1, P));
    Lc.add(cd(c.C + c.sC, 2 * c.sC, c.ldC, p.S3 + r, s3, ld3, r, n, P));
    Lc.add(cd(c.y + c.sy, 2 * c.sy, 1, p.S3 + (int64_t)n * ld3 + r, s3, ld3, r, 1, P));
    if (odd) {
      Lc.add(cd(p.S2 + P * s2 + (int64_t)n * ld2 + n, 0, ld2, p.S3 + (P - 1) * s3 + 2 * r, 0, ld3, n, n, 1));
      Lc.add(cd(p.S2 + P * s2 + (int64_t)3 * n * ld2 + n, 0, ld2, p.S3 + (P - 1) * s3 + (int64_t)n * ld3 + 2 * r, 0,
                ld3, n, 1, 1));
    }
    if ((e = run(Lc, s3s)) != cudaSuccess) return e;
    if ((e = qr_apply(p.S3, s3, ld3, ld3, n, n + 1, P, *w3, s3s)) != cudaSuccess) return e;
    if (conc) {
      if ((e = cudaEventRecord(p.ev[1], p.s2)) != cudaSuccess) return e;
      if ((e = stage2()) != cudaSuccess) return e;
      // ---- records of the eliminated columns (stage 2's R rows), beside stage 3 ----
      if ((e = post(p, L, c.nrm, 2 * c.snrm, P + (odd ? 1 : 0), p.rec[L], ((int64_t)1 << L) - 1,
                    (int64_t)2 << L, s)) != cudaSuccess)
        return e;
      if ((e = cudaStreamWaitEvent(s, p.ev[1], 0)) != cudaSuccess) return e;
    }
    // ---- level L+1 entries (column p = survivor 2p + 1) ----
    double *nx = p.ent[L + 1];
    Lc.add(cd(p.S3, s3, ld3, nx, E, n, n, n, P, 1.0, 0, 1));                                  // C'
    Lc.add(cd(p.S3 + (int64_t)n * ld3, s3, ld3, nx + nn, E, n, n, 1, P));                     // y'
    Lc.add(cd(p.S2 + (int64_t)n * ld2 + n, s2, ld2, nx + nn + n, E, n, n, n, P));             // El = Z_t
    Lc.add(cd(p.S2 + (int64_t)2 * n * ld2 + n, s2, ld2, nx + 2 * nn + n, E, n, n, n, P));     // Er = X~_t
    Lc.add(cd(p.S2 + (int64_t)3 * n * ld2 + n, s2, ld2, nx + 3 * nn + n, E, n, n, 1, P));     // e = z^_t
    Lc.add(cd(c.nrm + c.snrm, 2 * c.snrm, 1, nx + 3 * nn + 2 * n, E, 1, 1, 1, P));            // |column|^2
    if ((e = run(Lc, s)) != cudaSuccess) return e;
    // ---- records of the eliminated columns t = 2p (and K - 1) ----
    if (!conc && (e = post(p, L, c.nrm, 2 * c.snrm, P + (odd ? 1 : 0), p.rec[L], ((int64_t)1 << L) - 1,
                           (int64_t)2 << L, s)) != cudaSuccess)
      return e;
    (void)Rr;
  }
  return cudaSuccess;
}

// ----------------------------------------------------------- backward ---
// Levels in reverse (P:592-600 and Alg. 2): for every eliminated
// column t of level L with its level-(L+1) neighbours l, r:
//   x_t = w - [T_l T_r][x_l; x_r];   G = [T_l T_r] [S_ll S_lr; S_rl S_rr]
//   S_{t,I} = -G,   S_tt = P + G [T_l T_r]^T (symmetrised)
cudaError_t backward(const Plan &p, bool do_state, bool do_cov, cudaStream_t s) {
  const int n = p.n;
  const int64_t nn = (int64_t)n * n, Rr = rrec_doubles_big(n);
  cudaError_t e;
  CopyList Lc;
  const int top = (int)p.Ks.size() - 1;
  for (int L = top; L >= 0; --L) {
    const int64_t K = p.Ks[L];
    const int64_t P = K / 2, cnt = P + (K & 1);   // eliminated columns t = 2q, q < cnt
    const int64_t st = (int64_t)1 << L;         // domain distance to a neighbour
    double *x = p.x, *S = p.S;
    const double *rec = p.rec[L];
    const int64_t j0 = st - 1, js = 2 * st;      // step of item q: j0 + q js
    if (do_state) {   // xg = [x_l; x_r]
      Lc.add(cd(nullptr, 0, 1, p.xg, 2 * n, 2 * n, 2 * n, 1, cnt));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      Lc.add(cd(x + (j0 - st + js) * n, js * n, n, p.xg + 2 * n + 0, 2 * n, 2 * n, n, 1, cnt - 1));   // q >= 1
      Lc.add(cd(x + (j0 + st) * n, js * n, n, p.xg + n, 2 * n, 2 * n, n, 1, P));                      // q < P
      if ((e = run(Lc, s)) != cudaSuccess) return e;
    }
    if (do_cov) {     // SII = [S_ll S_lr; S_rl S_rr] (2n x 2n)
      const int64_t s4 = 4 * nn;
      Lc.add(cd(nullptr, 0, 1, p.SII, s4, 2 * n, 2 * n, 2 * n, cnt));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      Lc.add(cd(S + (j0 - st + js) * nn, js * nn, n, p.SII + s4, s4, 2 * n, n, n, cnt - 1));                // S_ll
      Lc.add(cd(S + (j0 + st) * nn, js * nn, n, p.SII + (int64_t)n * 2 * n + n, s4, 2 * n, n, n, P));      // S_rr
      if (L < top && P > 1) {   // S_lr = S_{q-1,q} = X_{L+1}[q]^T, S_rl = X_{L+1}[q], 1 <= q < P
        const double *Xu = p.X[L + 1];
        Lc.add(cd(Xu + nn, nn, n, p.SII + s4 + (int64_t)n * 2 * n, s4, 2 * n, n, n, P - 1, 1.0, 1));
        Lc.add(cd(Xu + nn, nn, n, p.SII + s4 + n, s4, 2 * n, n, n, P - 1));
      }
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      Gemm g;   // G = A SII,  A = [T_l T_r] (n x 2n, ld n)
      g.batch = cnt; g.M = n; g.N = 2 * n; g.K = 2 * n; g.A = rec; g.lda = n; g.sA = Rr;
      g.B = p.SII; g.ldb = 2 * n; g.sB = s4; g.C = p.G; g.ldc = n; g.sC = 2 * nn;
      if ((e = gemm(g, false, false, s)) != cudaSuccess) return e;
      // S_tt = P + G A^T
      Lc.add(cd(rec + 2 * nn + n, Rr, n, p.Pt, nn, n, n, n, cnt));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      g.M = n; g.N = n; g.K = 2 * n; g.A = p.G; g.lda = n; g.sA = 2 * nn; g.B = rec; g.ldb = n; g.sB = Rr;
      g.C = p.Pt; g.ldc = n; g.sC = nn; g.beta = 1.0;
      if ((e = gemm(g, false, true, s)) != cudaSuccess) return e;
      if ((e = sym_store(p.Pt, nn, n, S + j0 * nn, js * nn, n, cnt, s)) != cudaSuccess) return e;
      // cross blocks of level L: X_L[t] = S_{t,t-1} = -G[:, 0:n] (t >= 1),
      // X_L[t+1] = S_{t+1,t} = -G[:, n:2n]^T (t + 1 < K)
      if (L >= 1) {
        double *Xc = p.X[L];
        Lc.add(cd(p.G + 2 * nn, 2 * nn, n, Xc + 2 * nn, 2 * nn, n, n, n, cnt - 1, -1.0));
        Lc.add(cd(p.G + nn, 2 * nn, n, Xc + nn, 2 * nn, n, n, n, P, -1.0, 1));
        if ((e = run(Lc, s)) != cudaSuccess) return e;
      }
    }
    if (do_state) {   // x_t = w - A xg
      Lc.add(cd(rec + 2 * nn, Rr, n, p.xt, n, n, n, 1, cnt));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
      Gemm g;
      g.batch = cnt; g.M = n; g.N = 1; g.K = 2 * n; g.A = rec; g.lda = n; g.sA = Rr; g.B = p.xg; g.ldb = 2 * n;
      g.sB = 2 * n; g.C = p.xt; g.ldc = n; g.sC = n; g.alpha = -1.0; g.beta = 1.0;
      if ((e = gemm(g, false, false, s)) != cudaSuccess) return e;
      Lc.add(cd(p.xt, n, n, x + j0 * n, js * n, n, n, 1, cnt));
      if ((e = run(Lc, s)) != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace big
}  // namespace ks
