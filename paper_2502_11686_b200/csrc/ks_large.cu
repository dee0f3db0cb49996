// sm_100a fp64 kernels of the Odd-Even Kalman smoother: the CTA path
// (every n up to the shared-memory limit, n = m = 48 for BASELINE config 4;
// also the multi-GPU boundary system and KS_GENERIC_PATH for n <= 8).
//
// One CTA (8 warps) per eliminated column (pair), the stage matrices resident
// in shared memory (column-major, rows and columns zero-padded to multiples
// of 8, leading dimension = 4 mod 16 so that DMMA fragment loads are bank-
// conflict free).  Every QR is a blocked Householder QR (LAPACK geqrf order:
// panels of 8 columns, compact-WY Q = I - V T V^T): the panel is factored by
// one warp (lanes over rows, shuffle reductions), the trailing update
// W = V^T C, W = T^T W, C -= V W runs on the FP64 tensor cores
// (mma.sync.m8n8k4.f64, DMMA) -- the real dense contractions of the method
// at large n (north_star).  Triangular solves (T = R^{-1}[R_l R_r],
// w = R^{-1} z, R^{-1}), the SelInv products S_{t,I} = -T S_II and
// S_tt = P - S_{t,I} T^T, and the whitening solves are blocked the same way:
// 8x8 diagonal blocks by threads, off-diagonal updates as DMMA GEMMs.
//
// P:n = line n of the paper text.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "ks_internal.cuh"

namespace ks {

namespace {

constexpr int kThreads = 256, kWarps = kThreads / 32;

// Development instrumentation (-DKS_LARGE_PROF, variant builds only): phase
// cycle counts of CTA 0, printed by its thread 0.
#ifdef KS_LARGE_PROF
#define KS_PROF_DECL long long _pt = clock64(), _acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define KS_PROF(i)                                   \
  {                                                  \
    const long long _now = clock64();                \
    _acc[i] += _now - _pt;                           \
    _pt = _now;                                      \
  }
#define KS_PROF_PRINT(tag)                                                                          \
  if (blockIdx.x == 1 && threadIdx.x == 0)                                                          \
    printf("[%s] %lld %lld %lld %lld %lld %lld %lld %lld\n", tag, _acc[0], _acc[1], _acc[2], _acc[3], \
           _acc[4], _acc[5], _acc[6], _acc[7]);
#else
#define KS_PROF_DECL
#define KS_PROF(i)
#define KS_PROF_PRINT(tag)
#endif
// Panel phase clock (-DKS_PANEL_PROF, micro-benchmarks only): cycles of the
// panel warp's phases accumulated in g_panel_clk[0..7].
#if defined(KS_PANEL_PROF) || defined(KS_LARGE_PROF)
__device__ unsigned long long g_refresh[2];   // [0] exact-Gram refreshes, [1] panel columns
#define KS_COUNT(i, v) if ((threadIdx.x & 31) == 0) atomicAdd(&g_refresh[i], (unsigned long long)(v));
#else
#define KS_COUNT(i, v)
#endif
#ifdef KS_PANEL_PROF
__device__ long long g_panel_clk[8];
#define KS_PCLK(i)                                                     \
  {                                                                    \
    const long long _n = clock64();                                    \
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) g_panel_clk[i] += _n - _pc; \
    _pc = _n;                                                          \
  }
#define KS_PCLK_DECL long long _pc = clock64();
#else
#define KS_PCLK(i)
#define KS_PCLK_DECL
#endif
constexpr int kLdw = 12;   // leading dimension of the 8 x 8 warp tiles (12 = conflict-free)

__host__ __device__ constexpr int pad8(int x) { return (x + 7) & ~7; }
// leading dimension for `rows` padded rows: >= pad8(rows) and = 4 (mod 16)
__host__ __device__ constexpr int ldpad(int rows) { return pad8(rows) + ((4 - pad8(rows) % 16) + 16) % 16; }

__device__ __forceinline__ void report(unsigned long long *st, int64_t step, int kind) {
  if (st) atomicMin(st, status_word(step, kind));
}

// D = A B + D on one 8x8 tile: A 8x4 (row-major fragment: lane holds
// A[lane/4][lane%4]), B 4x8 (B[lane%4][lane/4]), D 8x8 (D[lane/4][2(lane%4)+i]).
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C = beta C + alpha op(A) op(B) on shared-memory column-major operands.
// M, N multiples of 8, K a multiple of 4 (operands zero-padded).  Each warp
// owns pairs of vertically adjacent 8x8 output tiles (two independent DMMA
// chains sharing the B fragment).  No aliasing between C and A / B.
template <bool TA, bool TB>
__device__ void gemm(int M, int N, int K, double alpha, const double *A, int lda, const double *B, int ldb,
                     double beta, double *C, int ldc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int mt = M >> 3, nt = N >> 3, mp = (mt + 1) >> 1, nw = blockDim.x >> 5;
  for (int tile = warp; tile < mp * nt; tile += nw) {
    const int m0 = (tile % mp) * 16, n0 = (tile / mp) * 8;
    const bool two = m0 + 8 < M;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    for (int k0 = 0; k0 < K; k0 += 4) {
      const double b = TB ? B[(n0 + g) + (k0 + q) * ldb] : B[(k0 + q) + (n0 + g) * ldb];
      const double a0 = TA ? A[(k0 + q) + (m0 + g) * lda] : A[(m0 + g) + (k0 + q) * lda];
      dmma(c00, c01, a0, b);
      if (two) {
        const double a1 = TA ? A[(k0 + q) + (m0 + 8 + g) * lda] : A[(m0 + 8 + g) + (k0 + q) * lda];
        dmma(c10, c11, a1, b);
      }
    }
    double *c = C + (m0 + g) + (n0 + 2 * q) * ldc;
    if (beta == 0.0) {
      c[0] = alpha * c00;
      c[ldc] = alpha * c01;
      if (two) {
        c[8] = alpha * c10;
        c[8 + ldc] = alpha * c11;
      }
    } else {
      c[0] = fma(alpha, c00, beta * c[0]);
      c[ldc] = fma(alpha, c01, beta * c[ldc]);
      if (two) {
        c[8] = fma(alpha, c10, beta * c[8]);
        c[8 + ldc] = fma(alpha, c11, beta * c[8 + ldc]);
      }
    }
  }
}

// 1/sqrt(h) (h > 0) and 1/x (x != 0): MUFU approximation + two Newton steps.
__device__ __forceinline__ double rsqrt_nr(double h) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(h));
  double hy = h * y;
  y = fma(0.5 * y, fma(-hy, y, 1.0), y);
  hy = h * y;
  y = fma(0.5 * y, fma(-hy, y, 1.0), y);
  return y;
}
__device__ __forceinline__ double rcp_nr(double x) {   // one third-order Newton step (see ks_small_impl.cuh)
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// Workspace of the blocked QR (shared memory).  The reflectors themselves
// live in the factored columns below the diagonal (LAPACK geqrf storage);
// the workspace holds per panel the compact-WY factor T, v_1 (the reflector
// entry on the diagonal, whose place holds R_jj) and beta, double-buffered so
// that panel k+1 is factored while panel k's reflectors are still being
// applied (lookahead, qr_blocked).
struct QrWs {
  double *base;   // T (buffer 0, 1: [kLdw x 8] each), then v1 (2 x 8), beta (2 x 8)
  double *G;      // [kLdw x 8] panel warp scratch (Gram matrices)
  double *tile;   // [nw][kLdw x 8] per-warp 8x8 scratch of qr_apply
  // (no pointer arrays: a runtime-indexed array member would live in local memory)
  __device__ __forceinline__ double *T(int b) const { return base + b * (kLdw * 8); }
  __device__ __forceinline__ double *v1(int b) const { return base + 2 * kLdw * 8 + 8 * b; }
  __device__ __forceinline__ double *beta(int b) const { return base + 2 * kLdw * 8 + 16 + 8 * b; }
};
__host__ __device__ constexpr int qr_ws_doubles(int nw) { return 2 * kLdw * 8 + 32 + kLdw * 8 + nw * kLdw * 8; }
__device__ __forceinline__ QrWs carve_ws(double *p) {
  QrWs w;
  w.base = p;
  w.G = p + 2 * kLdw * 8 + 32;
  w.tile = w.G + kLdw * 8;
  return w;
}
constexpr int kPanelMaxR = 5;   // rows per lane in the panel factorization (rows <= 160)

// Entry (i, j) of the panel's reflector matrix V (rows local to the panel
// origin P, column j < 8): v_1 on the diagonal, the stored column below it,
// zero above and in the non-pivot columns j >= nb.
__device__ __forceinline__ double vget(const double *P, int lda, const double *v1, int nb, int i, int j) {
  return (j >= nb || i < j) ? 0.0 : (i == j ? v1[j] : P[i + j * lda]);
}

// Gram matrix of panel columns [0, nb) over the panel rows [r0, mrow) (rows
// local to the panel origin P), one 8x8 DMMA tile by the calling warp, stored
// to G (kLdw); rows and columns outside are masked to 0.
template <bool kInline>
__device__ __forceinline__ void panel_gram_body(const double *P, int lda, int r0, int mrow, int nb, double *G) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0, g4 = 0.0, g5 = 0.0, g6 = 0.0, g7 = 0.0;   // four DMMA chains
  const bool col = g < nb;
  int kk = r0;
  for (; kk + 16 <= mrow; kk += 16) {
    const double x0 = col ? P[(kk + q) + g * lda] : 0.0, x1 = col ? P[(kk + 4 + q) + g * lda] : 0.0;
    const double x2 = col ? P[(kk + 8 + q) + g * lda] : 0.0, x3 = col ? P[(kk + 12 + q) + g * lda] : 0.0;
    dmma(g0, g1, x0, x0);
    dmma(g2, g3, x1, x1);
    dmma(g4, g5, x2, x2);
    dmma(g6, g7, x3, x3);
  }
  for (; kk < mrow; kk += 8) {
    const double x0 = (col && kk + q < mrow) ? P[(kk + q) + g * lda] : 0.0;
    const double x1 = (col && kk + 4 + q < mrow) ? P[(kk + 4 + q) + g * lda] : 0.0;
    dmma(g0, g1, x0, x0);
    dmma(g2, g3, x1, x1);
  }
  G[g + (2 * q) * kLdw] = (g0 + g2) + (g4 + g6);
  G[g + (2 * q + 1) * kLdw] = (g1 + g3) + (g5 + g7);
  __syncwarp();
}
// the exact recomputation of the accuracy guard (rare) out of line
__device__ __noinline__ void panel_gram(const double *P, int lda, int r0, int mrow, int nb, double *G) {
  panel_gram_body<false>(P, lda, r0, mrow, nb, G);
}

// The panel's compact-WY factor (LAPACK larft, forward columnwise):
// G = V^T V (DMMA, four chains) and T = U^{-1}, U = diag(1/beta) + striu(G)
// (a zero reflector gets U_jj = 1; its V column is 0).  Lane i < 8 computes
// row i of T right-looking: T_ii = beta_i, T_ij = -beta_j sum_{l<j} T_il G_lj,
// each finished T_ij is folded into the pending sums at once, so the serial
// chain per column is one multiply and one FMA (no cross-lane traffic).
__device__ void qr_panel_t(const double *P, int lda, int mpad, int nb, const double *v1, const double *beta,
                           double *T, double *Gs) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  {
    double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0, g4 = 0.0, g5 = 0.0, g6 = 0.0, g7 = 0.0;
    dmma(g0, g1, vget(P, lda, v1, nb, q, g), vget(P, lda, v1, nb, q, g));
    dmma(g2, g3, vget(P, lda, v1, nb, 4 + q, g), vget(P, lda, v1, nb, 4 + q, g));
    const bool col = g < nb;
    int kk = 8;
    for (; kk + 16 <= mpad; kk += 16) {
      const double x0 = col ? P[(kk + q) + g * lda] : 0.0, x1 = col ? P[(kk + 4 + q) + g * lda] : 0.0;
      const double x2 = col ? P[(kk + 8 + q) + g * lda] : 0.0, x3 = col ? P[(kk + 12 + q) + g * lda] : 0.0;
      dmma(g0, g1, x0, x0);
      dmma(g2, g3, x1, x1);
      dmma(g4, g5, x2, x2);
      dmma(g6, g7, x3, x3);
    }
    if (kk < mpad) {   // mpad % 8 == 0
      const double x0 = col ? P[(kk + q) + g * lda] : 0.0, x1 = col ? P[(kk + 4 + q) + g * lda] : 0.0;
      dmma(g4, g5, x0, x0);
      dmma(g6, g7, x1, x1);
    }
    Gs[g + (2 * q) * kLdw] = (g0 + g2) + (g4 + g6);
    Gs[g + (2 * q + 1) * kLdw] = (g1 + g3) + (g5 + g7);
  }
  __syncwarp();
  if (lane < 8) {
    const int i = lane;
    double bi[8], acc[8], gv[28];   // all loads issued before the serial chain
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      bi[j] = beta[j] == 0.0 ? 1.0 : beta[j];
      acc[j] = 0.0;
    }
#pragma unroll
    for (int j = 0, c = 0; j < 8; ++j)
#pragma unroll
      for (int k = j + 1; k < 8; ++k, ++c) gv[c] = Gs[j + k * kLdw];
#pragma unroll
    for (int j = 0, c = 0; j < 8; ++j) {
      const double tj = (j == i) ? bi[j] : ((j > i) ? -bi[j] * acc[j] : 0.0);
      T[i + j * kLdw] = tj;
#pragma unroll
      for (int k = j + 1; k < 8; ++k, ++c) acc[k] = fma(tj, gv[c], acc[k]);
    }
  }
  __syncwarp();
}

// Panel factorization by one warp: columns [k0, k0 + nb) of A, rows
// [k0, rows) (MR rows per lane), panel origin P = A + k0 + k0 lda.
// Householder reflector j: x = P[j:, j], alpha = -sign(x1)|x|,
// v = x - alpha e1, H = I - beta v v^T, beta = 1/(|x|^2 - x1 alpha) (zero
// column: beta = 0).  On exit the panel holds R on and above the diagonal
// and v below it (v_1 and beta to the workspace buffer), and T is formed.
//
// |x|^2 and x . a_jj (jj > j) over rows >= j are entries of the Gram matrix
// of the current panel columns over rows >= j, computed ONCE per panel (one
// DMMA tile) and then DOWNDATED instead of reduced again per column:
// reflector j is orthogonal on rows >= j, so it leaves that Gram unchanged,
// and the Gram over rows >= j+1 is it minus the outer product of the
// updated row j (the R row r_jj = a_jj[j] - d_jj v_1):  G' = G - r r^T.
// Every lane holds G redundantly (bitwise identical: branches on it are
// warp-uniform).  Accuracy guard: a downdated diagonal entry below kGramTau
// of its value at the last exact Gram (cancellation amplifies rounding by
// G_ref / G) triggers an exact Gram over rows >= j+1 -- rare for random or
// well-conditioned columns, which lose a few percent per step -- so every
// |x|^2 and dot used carries a relative error <= 8 eps / kGramTau, the
// reflectors are orthogonal to that level, and a rank-deficient column
// reaches the rank test with an exact norm.
constexpr double kGramTau = 0.125;
template <int MR>
__device__ __noinline__ void qr_panel(double *A, int lda, int k0, int rows, int nb, double *v1s, double *betas,
                                      double *T, double *Gs) {
  const int lane = threadIdx.x & 31;
  const int mrow = rows - k0, mpad = pad8(mrow);
  double *P = A + k0 + (int64_t)k0 * lda;
  KS_PCLK_DECL
  panel_gram_body<true>(P, lda, 0, mrow, nb, Gs);
  KS_PCLK(0)
  double a[MR][8];
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const int li = lane + 32 * r;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[r][j] = (li < mrow && j < nb) ? P[li + j * lda] : 0.0;
  }
  double G[8][8], gref[8];   // upper triangle used
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int j = i; j < 8; ++j) G[i][j] = Gs[i + j * kLdw];
    gref[i] = G[i][i];
  }
  __syncwarp();
  KS_PCLK(1)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double aj[8];   // row j of the panel (lane j, slot 0)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) aj[jj] = (jj >= j) ? __shfl_sync(0xffffffffu, a[0][jj], j) : 0.0;
    const double s = G[j][j], x1 = aj[j];
    const bool live = (j < nb) && (s > 0.0);
    const double nrm = live ? s * rsqrt_nr(s) : 0.0;
    const double alpha = live ? ((x1 > 0.0) ? -nrm : nrm) : x1;
    const double beta = live ? rcp_nr(s - x1 * alpha) : 0.0;
    const double v1 = live ? x1 - alpha : 0.0;
    double v[MR];
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int li = lane + 32 * r;
      v[r] = li > j ? a[r][j] : (li == j ? v1 : 0.0);
    }
    double rj[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
      if (jj > j) {
        const double d = beta * (G[j][jj] - alpha * aj[jj]);
        rj[jj] = fma(-d, v1, aj[jj]);
#pragma unroll
        for (int r = 0; r < MR; ++r) a[r][jj] = fma(-d, v[r], a[r][jj]);
      }
    if (j < nb && lane == j) a[0][j] = alpha;   // R_jj in place of v_1 (j < 8 <= 32)
    if (lane == 0) {   // beta = 0 beyond nb: T stays finite
      v1s[j] = v1;
      betas[j] = beta;
    }
    if (j < 7) {
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i > j) {
#pragma unroll
          for (int l = 0; l < 8; ++l)
            if (l >= i) G[i][l] = fma(-rj[i], rj[l], G[i][l]);
          bad |= (i < nb) && (G[i][i] < kGramTau * gref[i]);
        }
      if (bad) {   // exact Gram of the remaining columns over rows >= j + 1
        KS_COUNT(0, 1)
#pragma unroll
        for (int r = 0; r < MR; ++r) {
          const int li = lane + 32 * r;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (jj > j && li > j && li < mrow && jj < nb) P[li + jj * lda] = a[r][jj];
        }
        __syncwarp();
        panel_gram(P + (j + 1) * lda, lda, j + 1, mrow, nb - (j + 1), Gs);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i > j) {
#pragma unroll
            for (int l = 0; l < 8; ++l)
              if (l >= i) G[i][l] = Gs[(i - j - 1) + (l - j - 1) * kLdw];
            gref[i] = G[i][i];
          }
        __syncwarp();
      }
    }
  }
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const int li = lane + 32 * r;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (li < mrow && j < nb) P[li + j * lda] = a[r][j];
  }
  __syncwarp();
  KS_PCLK(2)
  KS_COUNT(1, nb)
  qr_panel_t(P, lda, mpad, nb, v1s, betas, T, Gs);
  KS_PCLK(3)
}

// Q^T C for the reflectors of the panel at (k0, k0) (nb columns, buffer b)
// and the columns [cb, ce) of A (tiles of 8 columns, tile t of the range to
// warp wi of nwk), Q = I - V T V^T:  W = V^T C, W = T^T W, C -= V W, all
// three products of a tile in the same warp (no barrier).  Rows [k0, k0 +
// mpad); V read in place (vget for its diagonal 8x8 block).
__device__ void qr_apply(double *A, int lda, int k0, int mpad, int nb, const QrWs &w, int b, int cb, int ce, int wi,
                         int nwk, double *sc) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const double *P = A + k0 + (int64_t)k0 * lda;
  const double *v1 = w.v1(b), *T = w.T(b);
  // V's diagonal block as the A operand of V^T C (V[q][g], V[4+q][g]) and of
  // V W (V[g][q], V[g][4+q]); below it the stored columns (column mask g < nb
  // resp. q, 4+q < nb)
  const double va0 = vget(P, lda, v1, nb, q, g), va1 = vget(P, lda, v1, nb, 4 + q, g);
  const double vb0 = vget(P, lda, v1, nb, g, q), vb1 = vget(P, lda, v1, nb, g, 4 + q);
  const bool cg = g < nb, cq0 = q < nb, cq1 = 4 + q < nb;
  for (int n0 = cb + wi * 8; n0 < ce; n0 += nwk * 8) {
    double *C = A + k0 + (int64_t)n0 * lda;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;   // two independent DMMA chains
    dmma(w0, w1, va0, C[q + g * lda]);               // V^T[g][q], C[q][g]
    dmma(w2, w3, va1, C[(4 + q) + g * lda]);
    for (int kk = 8; kk < mpad; kk += 8) {
      dmma(w0, w1, cg ? P[(kk + q) + g * lda] : 0.0, C[(kk + q) + g * lda]);
      dmma(w2, w3, cg ? P[(kk + 4 + q) + g * lda] : 0.0, C[(kk + 4 + q) + g * lda]);
    }
    sc[g + (2 * q) * kLdw] = w0 + w2;
    sc[g + (2 * q + 1) * kLdw] = w1 + w3;
    __syncwarp();
    double u0 = 0.0, u1 = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4) {
      const double x = T[(kk + q) + g * kLdw];   // T^T[g][kk+q]
      const double y = sc[(kk + q) + g * kLdw];  // W[kk+q][g]
      dmma(u0, u1, x, y);
    }
    __syncwarp();
    sc[g + (2 * q) * kLdw] = u0;
    sc[g + (2 * q + 1) * kLdw] = u1;
    __syncwarp();
    const double y0 = sc[q + g * kLdw], y1 = sc[(4 + q) + g * kLdw];   // W2[kk+q][g]
    {
      double *cp = C + g + (2 * q) * lda;
      double c0v = cp[0], c1v = cp[lda];
      dmma(c0v, c1v, -vb0, y0);
      dmma(c0v, c1v, -vb1, y1);
      cp[0] = c0v;
      cp[lda] = c1v;
    }
#pragma unroll 2
    for (int m0 = 8; m0 < mpad; m0 += 8) {
      double *cp = C + (m0 + g) + (2 * q) * lda;
      double c0v = cp[0], c1v = cp[lda];
      dmma(c0v, c1v, cq0 ? -P[(m0 + g) + q * lda] : 0.0, y0);
      dmma(c0v, c1v, cq1 ? -P[(m0 + g) + (4 + q) * lda] : 0.0, y1);
      cp[0] = c0v;
      cp[lda] = c1v;
    }
    __syncwarp();
  }
}

// Blocked Householder QR: triangularise columns [0, npiv) of the
// rows x ncols column-major shared matrix A and apply Q^T to columns
// [npiv, ncols).  A is zero-padded to pad8(rows) rows (lda >= that) and to
// pad8(ncols) (+8 when npiv % 8 != 0) columns.  On exit the first npiv
// columns hold R (zeros below the diagonal).  Ends with a barrier of the
// group.  Warp group [wbase, wbase + nw) with its own named barrier
// (barid > 0), or the whole CTA (barid 0).
//
// Lookahead: while warps 1..nw-1 apply panel k's reflectors to the columns
// right of panel k+1, warp 0 applies them to panel k+1's own 8 columns and
// factors it at once, so the serial panel chain (the QR's critical path)
// no longer waits for the trailing update; one barrier per panel.
// The blocked QR is inlined at its call sites (an out-of-line copy costs
// caller/callee register saves through local memory, which misses the small
// L1 left beside 222 KB of shared memory: c4 factor L0 8.23 vs 8.89 ms); the
// panels (the bulk of the code) stay out of line, one copy per height.
#ifdef KS_QRB_NOINLINE   // A/B
#define KS_QRB_INLINE __device__ __noinline__
#else
#define KS_QRB_INLINE __device__ __forceinline__
#endif
__device__ __forceinline__ void group_sync(int barid, int nw) {
  if (barid == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(nw * 32) : "memory");
}
template <int MR>
__device__ __forceinline__ void qr_panel_mr(double *A, int lda, int k0, int rows, int nb, const QrWs w, int b) {
  qr_panel<MR>(A, lda, k0, rows, nb, w.v1(b), w.beta(b), w.T(b), w.G);
}
KS_QRB_INLINE void qr_blocked(double *A, int lda, int rows, int npiv, int ncols, const QrWs w, long long *acc = nullptr,
                           int wbase = 0, int nw = kWarps, int barid = 0) {
  const int warp = (threadIdx.x >> 5) - wbase;
  double *sc = w.tile + warp * (kLdw * 8);
  const int cend = pad8(ncols);
  int kprev = -1, nbprev = 0;
  for (int k0 = 0; k0 < npiv && k0 < rows; k0 += 8) {
    const int nb = (npiv - k0 < 8) ? npiv - k0 : 8, b = (k0 >> 3) & 1;
    if (warp == 0) {
      if (kprev >= 0) qr_apply(A, lda, kprev, pad8(rows - kprev), nbprev, w, b ^ 1, k0, k0 + 8, 0, 1, sc);
      const int mr = (rows - k0 + 31) >> 5;
      if (mr <= 1) qr_panel_mr<1>(A, lda, k0, rows, nb, w, b);
      else if (mr == 2) qr_panel_mr<2>(A, lda, k0, rows, nb, w, b);
      else if (mr == 3) qr_panel_mr<3>(A, lda, k0, rows, nb, w, b);
      else if (mr == 4) qr_panel_mr<4>(A, lda, k0, rows, nb, w, b);
      else qr_panel_mr<kPanelMaxR>(A, lda, k0, rows, nb, w, b);
    } else if (kprev >= 0 && k0 + 8 < cend) {
      qr_apply(A, lda, kprev, pad8(rows - kprev), nbprev, w, b ^ 1, k0 + 8, cend, warp - 1, nw - 1, sc);
    }
    group_sync(barid, nw);
    kprev = k0;
    nbprev = nb;
  }
  // the last panel's reflectors on everything right of it (its own non-pivot
  // columns included), then R's lower triangle (the stored V) is cleared
  if (kprev >= 0) {
    const int c0 = kprev + nbprev;
    if (c0 < ncols)
      qr_apply(A, lda, kprev, pad8(rows - kprev), nbprev, w, (kprev >> 3) & 1, c0, c0 + pad8(ncols - c0), warp, nw, sc);
    group_sync(barid, nw);   // the last V is read until here
  }
  for (int idx = threadIdx.x - wbase * 32; idx < npiv * pad8(rows); idx += nw * 32) {
    const int j = idx / pad8(rows), i = idx - j * pad8(rows);
    if (i > j) A[i + j * lda] = 0.0;
  }
  group_sync(barid, nw);
}

// X <- R^{-1} X for R (n x n upper triangular, ldr) and X (n x p, ldx), both
// zero-padded to 8 rows/columns: 8-row blocks from the bottom, the diagonal
// block by one thread per right-hand side (values in registers, multiplied
// by the reciprocal diagonal rinv[0..n) the caller provides), the update of
// the rows above as a DMMA GEMM.  Ends with __syncthreads.  Two
// right-hand-side blocks at once, X1 (p1 columns) and X2 (p2): one diagonal
// pass and one barrier pair per 8-row block for both.
__device__ void trsm_upper2(const double *R, int ldr, const double *rinv, int n, double *X1, int ldx1, int p1,
                            double *X2, int ldx2, int p2) {
  for (int r0 = ((n - 1) / 8) * 8; r0 >= 0; r0 -= 8) {
    const int h = (n - r0 < 8) ? n - r0 : 8;
    for (int c = threadIdx.x; c < p1 + p2; c += blockDim.x) {
      double *xp = c < p1 ? X1 + r0 + c * ldx1 : X2 + r0 + (c - p1) * ldx2;
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = (i < h) ? xp[i] : 0.0;
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        if (i < h) {
          double s = x[i];
#pragma unroll
          for (int l = i + 1; l < 8; ++l)
            if (l < h) s = fma(-R[(r0 + i) + (r0 + l) * ldr], x[l], s);
          x[i] = s * rinv[r0 + i];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < h) xp[i] = x[i];
    }
    __syncthreads();
    if (r0 > 0) {
      gemm<false, false>(r0, pad8(p1), 8, -1.0, R + r0 * ldr, ldr, X1 + r0, ldx1, 1.0, X1, ldx1);
      gemm<false, false>(r0, pad8(p2), 8, -1.0, R + r0 * ldr, ldr, X2 + r0, ldx2, 1.0, X2, ldx2);
    }
    __syncthreads();
  }
}

// X <- L^{-1} X for L (n x n lower triangular): 8-row blocks from the top.
__device__ void trsm_lower(const double *L, int ldl, const double *rinv, int n, double *X, int ldx, int p) {
  for (int r0 = 0; r0 < n; r0 += 8) {
    const int h = (n - r0 < 8) ? n - r0 : 8;
    for (int c = threadIdx.x; c < p; c += blockDim.x) {
      double *xp = X + r0 + c * ldx;
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = (i < h) ? xp[i] : 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < h) {
          double s = x[i];
#pragma unroll
          for (int l = 0; l < i; ++l) s = fma(-L[(r0 + i) + (r0 + l) * ldl], x[l], s);
          x[i] = s * rinv[r0 + i];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < h) xp[i] = x[i];
    }
    __syncthreads();
    const int rest = pad8(n) - r0 - 8;
    if (rest > 0)
      gemm<false, false>(rest, pad8(p), 8, -1.0, L + (r0 + 8) + r0 * ldl, ldl, X + r0, ldx, 1.0, X + r0 + 8, ldx);
    __syncthreads();
  }
}

// rinv[i] = 1 / A_ii, i < n (threads; caller synchronises)
__device__ void diag_rcp(const double *A, int lda, int n, double *rinv) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) rinv[i] = 1.0 / A[i + i * lda];
}

// Blocked right-looking Cholesky of the d x d lower triangle of Lm (ldl,
// zero-padded to 8): 8-column panels factored by warp 0 (lanes over rows,
// pivots and panel rows by shuffles, d <= 64), the trailing update
// A22 -= L21 L21^T as a DMMA GEMM.  Returns (to warp 0) false if a pivot is
// <= 0 (then continues with 1).  Ends with __syncthreads.
__device__ bool cta_chol(double *Lm, int ldl, int d, double *sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool ok = true;
  for (int k0 = 0; k0 < d; k0 += 8) {
    const int nb = (d - k0 < 8) ? d - k0 : 8;
    if (warp == 0) {
      double a[2][8];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int r = k0 + lane + 32 * s;
#pragma unroll
        for (int c = 0; c < 8; ++c) a[s][c] = (r < d && c < nb) ? Lm[r + (k0 + c) * ldl] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < nb) {
          const double v = __shfl_sync(0xffffffffu, a[0][c], c);
          ok &= v > 0.0;
          const double il = rsqrt_nr(v > 0.0 ? v : 1.0), l = (v > 0.0 ? v : 1.0) * il;
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int r = k0 + lane + 32 * s;
            if (r == k0 + c) a[s][c] = l;
            else if (r > k0 + c) a[s][c] *= il;
          }
#pragma unroll
          for (int cc = c + 1; cc < 8; ++cc) {
            const double lcc = __shfl_sync(0xffffffffu, a[0][c], cc);   // L[k0+cc][k0+c]
            if (cc < nb) {
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                const int r = k0 + lane + 32 * s;
                if (r >= k0 + cc) a[s][cc] = fma(-a[s][c], lcc, a[s][cc]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int r = k0 + lane + 32 * s;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (r < d && c < nb && r >= k0 + c) Lm[r + (k0 + c) * ldl] = a[s][c];
      }
    }
    __syncthreads();
    const int rest = pad8(d) - k0 - 8;
    if (rest > 0) {
      const double *L21 = Lm + (k0 + 8) + k0 * ldl;
      gemm<false, true>(rest, rest, 8, -1.0, L21, ldl, L21, ldl, 1.0, Lm + (k0 + 8) + (k0 + 8) * ldl, ldl);
    }
    __syncthreads();
  }
  (void)sh;
  return ok;
}

// KS_COV_IS_CHOL: the loaded lower triangle already is the factor; valid iff
// every diagonal entry is nonzero and finite.  Result valid in every thread
// (ends with __syncthreads).
__device__ bool chol_diag_ok(double *Lm, int ldl, int d, double *sh) {
  __syncthreads();
  const int i = threadIdx.x;
  const bool bad = i < d && !(Lm[i + i * ldl] != 0.0 && Lm[i + i * ldl] - Lm[i + i * ldl] == 0.0);
  if (bad) Lm[i + i * ldl] = 1.0;   // continue with a finite factor (outputs undefined, status recorded)
  const int any = __syncthreads_or(bad);
  (void)sh;
  return !any;
}

__device__ void zero_smem(double *p, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) p[i] = 0.0;
}

// smem column-major A(lda)[r0:r0+rows, c0:c0+cols] <- g (row-major, ldg);
// rows >= valid or g == null stay untouched (caller zeroed the matrix).
// Asynchronous (cp.async, global -> shared without registers): every element
// of every block of a stage's setup is in flight at once; the caller
// completes them with sync_loads().
__device__ void ld_blk(double *A, int lda, int r0, int c0, const double *g, int64_t ldg, int rows, int cols,
                       int valid) {
  if (g == nullptr) return;
  const int tot = (valid < rows ? valid : rows) * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx / cols, j = idx - i * cols;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(A + (r0 + i) + (c0 + j) * lda);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g + (int64_t)i * ldg + j) : "memory");
  }
}
__device__ __forceinline__ void cp8(double *sdst, const double *g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void sync_loads() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
}
// this thread's share of |A[r0:r0+rows, c0:c0+cols]|_F^2 (shared memory)
__device__ double sumsq_blk(const double *A, int lda, int r0, int c0, int rows, int cols) {
  double s = 0.0;
  for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
    const double v = A[(r0 + idx % rows) + (c0 + idx / rows) * lda];
    s = fma(v, v, s);
  }
  return s;
}
// L2 prefetch of `count` contiguous doubles (one 128-byte line per thread)
__device__ __forceinline__ void pf_l2(const double *g, int64_t count) {
  if (g == nullptr) return;
  for (int64_t off = (int64_t)threadIdx.x * 16; off < count; off += (int64_t)blockDim.x * 16)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(g + off));
}
// this thread's share of |g|_F^2 (count contiguous doubles)
__device__ double part_sumsq(const double *g, int count) {
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s = fma(__ldg(g + i), __ldg(g + i), s);
  return s;
}

// smem (column-major) -> global row-major (ldg); rows >= valid are written as 0
__device__ void st_blk(double *g, int64_t ldg, const double *A, int lda, int r0, int c0, int rows, int cols,
                       int valid) {
  const int tot = rows * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx / cols, j = idx - i * cols;
    g[(int64_t)i * ldg + j] = (i < valid) ? A[(r0 + i) + (c0 + j) * lda] : 0.0;
  }
}

// smem -> smem block copy
__device__ void cp_blk(double *D, int ldd, int dr, int dc, const double *A, int lda, int r0, int c0, int rows,
                       int cols) {
  const int tot = rows * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx % rows, j = idx / rows;
    D[(dr + i) + (dc + j) * ldd] = A[(r0 + i) + (c0 + j) * lda];
  }
}

// CTA sums of two per-thread partials (sh: 2 kWarps doubles; fixed order:
// deterministic).  Contains barriers: every thread calls it.
__device__ void cta_sum2(double a, double b, double *sh, double &sa, double &sb) {
  const int tid = threadIdx.x;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if ((tid & 31) == 0) {
    sh[tid >> 5] = a;
    sh[kWarps + (tid >> 5)] = b;
  }
  __syncthreads();
  sa = 0.0;
  sb = 0.0;
  for (int w = 0; w < kWarps; ++w) {
    sa += sh[w];
    sb += sh[kWarps + w];
  }
  __syncthreads();
}

// The odd level's last-column rows Z (n x (n+1), row-major in zscratch) into
// rows r0.. of the stage-3 matrix.  Split odd level (a.zflag): they come from
// another CTA -- wait for its flag, then read through L2 (ld.global.cg).
__device__ void ld_zs(const FactorLevelArgs &a, double *A, int lda, int r0) {
  const int n = a.n;
  if (a.zflag) {
    if (threadIdx.x == 0) {
      while (atomicAdd(a.zflag, 0) == 0) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n * (n + 1); idx += blockDim.x) {
    const int i = idx / (n + 1), j = idx - i * (n + 1);
    A[(r0 + i) + j * lda] = __ldcg(a.zscratch + idx);
  }
}

// ---- shared-memory plan of the factor kernel ----
struct FactorPlan {
  int ld1, cols1, ld2, cols2, ld3, cols3;
  int off2, offws, total;   // doubles
  bool conc;                // stages 2 and 3 concurrently (B3 + a second workspace fit in S1's region)
};
constexpr int kConcMaxPerThread = 16;   // D~ | y~ values per thread held across the S1 -> B3 rebuild
#ifndef KS_CONC_W3
#define KS_CONC_W3 2
#endif
constexpr int kConcW3 = KS_CONC_W3;     // warps of the stage-3 group (the rest: stage 2)
__host__ __device__ inline FactorPlan factor_plan(int n, int RC) {
  FactorPlan f;
  const int extra = (n % 8) ? 8 : 0;
  f.ld1 = ldpad(RC + n);
  f.cols1 = pad8(2 * n + 1) + extra;
  f.ld2 = ldpad(2 * n);
  f.cols2 = pad8(3 * n + 1) + extra;
  f.ld3 = ldpad(2 * RC + n);
  f.cols3 = pad8(n + 1) + extra;
  const int s1 = f.ld1 * f.cols1;
  // post-processing reuses S1 for R^{-1}, P, a padded copy of R (3 x ldpad(n) x pad8(n))
  // and the reciprocal diagonal
  const int s1p = 3 * ldpad(n) * pad8(n) + pad8(n);
  const int s2 = f.ld2 * f.cols2, s3 = f.ld3 * f.cols3;
  f.off2 = ((s1 > s1p ? s1 : s1p) + 1) & ~1;
  f.offws = f.off2 + (((s2 > s3 ? s2 : s3) + 1) & ~1);
  f.total = f.offws + qr_ws_doubles(kWarps) + 2 * kWarps;
  // stage 3's matrix rebuilt in S1's region (free once stage 2's matrix is
  // set up) next to a 4-warp workspace: the two QRs run on two warp groups
  const int wsb = qr_ws_doubles(kConcW3);
  f.conc = ((s3 + 1) & ~1) + wsb <= f.off2 && RC * (n + 1) <= kConcMaxPerThread * kThreads;
  return f;
}

// Eliminate column t of the level:
//   stage 1  QR [C_t; El_{t+1}] -> R~_t, applied to [0; Er_{t+1}] and the RHS
//            giving X_t (top) and D~_{t+1} (bottom, acts on t+1 only)
//   stage 3  QR [D~_{t+1}; C_{t+1}; Zs] -> C'_{t+1} (survivor's C-like block)
//   stage 2  QR [Er_t; R~_t] applied to [El_t, 0, e_t; 0, X_t, z~_t] ->
//            R_tt, R_{t,t-1}, R_{t,t+1}, z_t (top) and the survivor's new
//            coupling row [Z_t | X~_t | z^_t] (bottom).  No left neighbour:
//            "nothing to do": R_tt = R~_t, R_{t,t+1} = X_t.
// A column without right neighbour (last column of an odd level, or the base
// case) has an empty right neighbour; its stage-2 leftover Z (acting on t-1
// only) goes to zscratch to join the left pair's stage 3 (reading R5).
// Writes the R record T = R^{-1}[R_l R_r], P = R^{-1}R^{-T}, w = R^{-1} z.
__device__ void eliminate(const FactorLevelArgs &a, double *sm, const FactorPlan &f, int64_t t, bool hr, bool hl,
                          int64_t pnext, bool zs_in, bool zs_out) {
  const int n = a.n, RC = a.in.RC, tid = threadIdx.x;
  const EntryView &in = a.in;
  double *S1 = sm, *P2 = sm + f.off2, *sh = sm + f.total - 2 * kWarps;
  QrWs w = carve_ws(sm + f.offws);
  const int ld1 = f.ld1, ld2 = f.ld2, ld3 = f.ld3;
  KS_PROF_DECL
#ifdef KS_LARGE_PROF
  long long *qacc = _acc + 6;
#else
  long long *qacc = nullptr;
#endif

  // rank references |UA block column|_F (reading R9): given at
  // level >= 1; at level 0 accumulated per thread from the blocks as they
  // are loaded (column t: C_t, Er_t, El_{t+1}; column t+1: C_{t+1}, Er_{t+1},
  // El_{t+2} -- the one block this pair does not otherwise read) and reduced
  // once after the QRs
  const bool l0n = in.nrm == nullptr;
  // what stages 2 and 3 read later (Er_t, El_t, e_t; C_{t+1}, y_{t+1}) is
  // pulled into L2 now, so their loads do not stall the pair's critical path
  if (hl) {
    pf_l2(in.Er + t * in.sEr, (int64_t)n * n);
    pf_l2(in.El + t * in.sEl, (int64_t)n * n);
    pf_l2(in.e + t * in.se, n);
  }
  if (hr) {
    pf_l2(in.C + (t + 1) * in.sC, (int64_t)RC * n);
    pf_l2(in.y + (t + 1) * in.sy, RC);
  }
  double pt = 0.0, pu = 0.0;
  // |El_{t+2}|: pulled into L2 now, summed after stage 1 (its loads then hit L2)
  const bool el2 = l0n && hr && t + 2 < a.K;
  if (el2) pf_l2(in.El + (t + 2) * in.sEl, (int64_t)n * n);

  // ---- stage 1 ----
  // Concurrent stages 2 / 3 (f.conc): stage 2's global blocks Er_t, El_t, e_t
  // are loaded into its (still unused) matrix B2 now, as a second cp.async
  // group that completes behind stage 1's QR.
  const bool conc = f.conc && hr && hl;
  zero_smem(S1, ld1 * f.cols1);
  if (conc) zero_smem(P2, ld2 * f.cols2);
  __syncthreads();
  ld_blk(S1, ld1, 0, 0, in.C + t * in.sC, n, RC, n, RC);
  ld_blk(S1, ld1, 0, 2 * n, in.y + t * in.sy, 1, RC, 1, RC);
  if (hr) {
    const int64_t u = t + 1;
    ld_blk(S1, ld1, RC, 0, in.El + u * in.sEl, n, n, n, n);
    ld_blk(S1, ld1, RC, n, in.Er + u * in.sEr, n, n, n, n);
    ld_blk(S1, ld1, RC, 2 * n, in.e + u * in.se, 1, n, 1, n);
  }
  if (conc) {
    asm volatile("cp.async.commit_group;" ::: "memory");
    ld_blk(P2, ld2, 0, 0, in.Er + t * in.sEr, n, n, n, n);
    ld_blk(P2, ld2, 0, n, in.El + t * in.sEl, n, n, n, n);
    ld_blk(P2, ld2, 0, 3 * n, in.e + t * in.se, 1, n, 1, n);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");   // stage 1's group only
    __syncthreads();
  } else {
    sync_loads();
  }
  if (l0n) {   // |C_t|, |El_{t+1}| (column t), |Er_{t+1}| (column t+1), before the QR overwrites them
    pt += sumsq_blk(S1, ld1, 0, 0, RC + (hr ? n : 0), n);
    if (hr) pu += sumsq_blk(S1, ld1, RC, n, n, n);
    __syncthreads();
  }
  KS_PROF(3)
  qr_blocked(S1, ld1, RC + n, n, 2 * n + 1, w, qacc);
  KS_PROF(1)
  if (el2) pu += part_sumsq(in.El + (t + 2) * in.sEl, n * n);

  if (conc) {
    // ---- stages 2 and 3 concurrently: independent QRs once stage 1 is done.
    // Stage 2's matrix B2 goes to P2 as below; stage 3's B3 is rebuilt in S1's
    // region (D~ | y~ held in registers across the rebuild) with a second
    // workspace behind it; warps 0-3 factor B3, warps 4-7 B2, each group with
    // its own panel warp and named barrier, so the two serial panel chains
    // overlap.
    const int64_t u = t + 1;
    cp_blk(P2, ld2, n, 0, S1, ld1, 0, 0, n, n);            // R~_t
    cp_blk(P2, ld2, n, 2 * n, S1, ld1, 0, n, n, n + 1);    // X_t, z~_t
    const int nd = RC * (n + 1);                           // D~_{t+1} (RC x n) | y~_{t+1}
    double dv[kConcMaxPerThread];
#pragma unroll
    for (int k = 0; k < kConcMaxPerThread; ++k) {
      const int idx = tid + k * kThreads;
      dv[k] = idx < nd ? S1[(n + idx % RC) + (n + idx / RC) * ld1] : 0.0;
    }
    sync_loads();                                          // S1 is dead; B2 loaded
    if (l0n) pt += sumsq_blk(P2, ld2, 0, 0, n, n);         // |Er_t|
    double *B3 = S1;
    zero_smem(B3, ld3 * f.cols3);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kConcMaxPerThread; ++k) {
      const int idx = tid + k * kThreads;
      if (idx < nd) B3[idx % RC + (idx / RC) * ld3] = dv[k];
    }
    ld_blk(B3, ld3, RC, 0, in.C + u * in.sC, n, RC, n, RC);
    ld_blk(B3, ld3, RC, n, in.y + u * in.sy, 1, RC, 1, RC);
    int rows3 = 2 * RC;
    if (zs_in) {
      ld_zs(a, B3, ld3, rows3);
      rows3 += n;
    }
    sync_loads();
    if (l0n) {   // |C_{t+1}|
      pu += sumsq_blk(B3, ld3, RC, 0, RC, n);
      __syncthreads();
    }
    KS_PROF(0)
    QrWs w3 = carve_ws(S1 + ((ld3 * f.cols3 + 1) & ~1));
    if (tid < 32 * kConcW3) qr_blocked(B3, ld3, rows3, n, n + 1, w3, qacc, 0, kConcW3, 1);
    else qr_blocked(P2, ld2, 2 * n, n, 3 * n + 1, w, qacc, kConcW3, kWarps - kConcW3, 2);
    __syncthreads();
    KS_PROF(2)
    double *ent = a.next + pnext * entry_doubles(n);
    const int valid = rows3 < n ? rows3 : n;
    st_blk(ent, n, B3, ld3, 0, 0, n, n, valid);              // C'
    st_blk(ent + n * n, 1, B3, ld3, 0, n, n, 1, valid);      // y'
    st_blk(ent + n * n + n, n, P2, ld2, n, n, n, n, n);               // El' = Z_t
    st_blk(ent + 2 * n * n + n, n, P2, ld2, n, 2 * n, n, n, n);       // Er' = X~_t
    st_blk(ent + 3 * n * n + n, 1, P2, ld2, n, 3 * n, n, 1, n);       // e'  = z^_t
    KS_PROF(5)
  } else {
  // ---- stage 3 (before stage 2: its matrix B3 shares memory with B2) ----
  if (hr) {
    const int64_t u = t + 1;
    zero_smem(P2, ld3 * f.cols3);
    __syncthreads();
    cp_blk(P2, ld3, 0, 0, S1, ld1, n, n, RC, n);          // D~_{t+1}
    cp_blk(P2, ld3, 0, n, S1, ld1, n, 2 * n, RC, 1);      // y~_{t+1}
    ld_blk(P2, ld3, RC, 0, in.C + u * in.sC, n, RC, n, RC);
    ld_blk(P2, ld3, RC, n, in.y + u * in.sy, 1, RC, 1, RC);
    int rows3 = 2 * RC;
    if (zs_in) {
      ld_zs(a, P2, ld3, rows3);
      rows3 += n;
    }
    sync_loads();
    if (l0n) {   // |C_{t+1}|
      pu += sumsq_blk(P2, ld3, RC, 0, RC, n);
      __syncthreads();
    }
    KS_PROF(0)
    qr_blocked(P2, ld3, rows3, n, n + 1, w, qacc);
    KS_PROF(2)
    double *ent = a.next + pnext * entry_doubles(n);
    const int valid = rows3 < n ? rows3 : n;
    st_blk(ent, n, P2, ld3, 0, 0, n, n, valid);             // C'
    st_blk(ent + n * n, 1, P2, ld3, 0, n, n, 1, valid);     // y'
    __syncthreads();
  }

  // ---- stage 2 ----
  zero_smem(P2, ld2 * f.cols2);
  __syncthreads();
  if (hl) {
    ld_blk(P2, ld2, 0, 0, in.Er + t * in.sEr, n, n, n, n);
    ld_blk(P2, ld2, 0, n, in.El + t * in.sEl, n, n, n, n);
    ld_blk(P2, ld2, 0, 3 * n, in.e + t * in.se, 1, n, 1, n);
    cp_blk(P2, ld2, n, 0, S1, ld1, 0, 0, n, n);            // R~_t
    cp_blk(P2, ld2, n, 2 * n, S1, ld1, 0, n, n, n + 1);    // X_t, z~_t
    sync_loads();
    if (l0n) {   // |Er_t|
      pt += sumsq_blk(P2, ld2, 0, 0, n, n);
      __syncthreads();
    }
    KS_PROF(0)
    qr_blocked(P2, ld2, 2 * n, n, 3 * n + 1, w, qacc);
    KS_PROF(3)
    if (hr) {
      double *ent = a.next + pnext * entry_doubles(n);
      st_blk(ent + n * n + n, n, P2, ld2, n, n, n, n, n);               // El' = Z_t
      st_blk(ent + 2 * n * n + n, n, P2, ld2, n, 2 * n, n, n, n);       // Er' = X~_t
      st_blk(ent + 3 * n * n + n, 1, P2, ld2, n, 3 * n, n, 1, n);       // e'  = z^_t
    } else if (zs_out) {
      st_blk(a.zscratch, n + 1, P2, ld2, n, n, n, n, n);                // Z_t
      st_blk(a.zscratch + n, n + 1, P2, ld2, n, 3 * n, n, 1, n);        // z^_t
    }
  } else {
    cp_blk(P2, ld2, 0, 0, S1, ld1, 0, 0, n, n);
    cp_blk(P2, ld2, 0, 2 * n, S1, ld1, 0, n, n, n + 1);
    if (hr) {
      double *ent = a.next + pnext * entry_doubles(n);
      for (int i = tid; i < 2 * n * n + n; i += blockDim.x) ent[n * n + n + i] = 0.0;
    }
  }
  }
  __syncthreads();

  double nrm_t, nrm_u = 0.0;
  if (l0n) {
    double st, su;
    cta_sum2(pt, pu, sh, st, su);
    nrm_t = sqrt(st);
    nrm_u = sqrt(su);
  } else {
    nrm_t = in.nrm[t * in.snrm];
    if (hr) nrm_u = in.nrm[(t + 1) * in.snrm];
  }
  if (hr && tid == 0) a.next[pnext * entry_doubles(n) + 3 * n * n + 2 * n] = nrm_u;

  // ---- R record: rank check, T = R^{-1}[R_l R_r], w = R^{-1} z, P = R^{-1} R^{-T} ----
  {   // one diagonal entry per thread, one CTA vote
    const bool bad_d = tid < n && !(fabs(P2[tid + tid * ld2]) > kRankTol * nrm_t);
    if (__syncthreads_or(bad_d) && tid == 0)
      report(a.status, (((t + 1) << (a.level - a.lbase)) - 1) + a.step0, kBadRank);
  }
  const int ldr = ldpad(n), np = pad8(n);
  // R_tt copied into a zero-padded block (the blocked solves read whole 8x8
  // blocks; B2's columns next to R hold the right-hand sides)
  double *Ri = S1, *Pm = S1 + ldr * np, *Rc = S1 + 2 * ldr * np, *rinv = S1 + 3 * ldr * np;
  zero_smem(Ri, 3 * ldr * np);
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) Ri[i + i * ldr] = 1.0;
  for (int idx = tid; idx < n * n; idx += blockDim.x) {
    const int i = idx % n, j = idx / n;
    if (i <= j) Rc[i + j * ldr] = P2[i + j * ld2];
  }
  diag_rcp(P2, ld2, n, rinv);
  __syncthreads();
  // RHS [R_l | R_r | z] (columns n .. 3n of B2) and I (R^{-1}) in two solves
  KS_PROF(0)
  trsm_upper2(Rc, ldr, rinv, n, P2 + n * ld2, ld2, 2 * n + 1, Ri, ldr, n);
  KS_PROF(4)
  gemm<false, true>(np, np, np, 1.0, Ri, ldr, Ri, ldr, 0.0, Pm, ldr);
  __syncthreads();
  KS_PROF(5)
  double *rec = a.rrec + (t >> 1) * rrec_doubles(n);
  const int nn = n * n;
  for (int idx = tid; idx < nn; idx += blockDim.x) {
    const int r = idx / n, c = idx - r * n;
    rec[idx] = P2[r + (n + c) * ld2];                  // Tl
    rec[nn + idx] = P2[r + (2 * n + c) * ld2];         // Tr
    rec[2 * nn + idx] = Pm[r + c * ldr];               // P
  }
  for (int r = tid; r < n; r += blockDim.x) rec[3 * nn + r] = P2[r + 3 * n * ld2];   // w
  __syncthreads();
  KS_PROF(0)
  KS_PROF_PRINT("elim: other stage1 stage3 stage2 trsm Pgemm panel apply")
#ifdef KS_LARGE_PROF
  if (blockIdx.x == 1 && threadIdx.x == 0)
    printf("[gram refreshes %llu of %llu panel columns]\n", g_refresh[0], g_refresh[1]);
#endif
}

__global__ void __launch_bounds__(kThreads) factor_level_kernel(FactorLevelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const FactorPlan f = factor_plan(a.n, a.in.RC);
  const int64_t K = a.K;
  // odd level: the last column (no right neighbour) by CTA 0 beside the last
  // pair (CTA K/2) when split (a.zflag), else first by the last pair's CTA.
  // The flag-setting CTA has the LOWEST index, so it is dispatched before
  // the CTA that waits for it even when only one CTA is resident at a time.
  const bool split = a.zflag != nullptr;
  const int64_t p = split ? (int64_t)blockIdx.x - 1 : (int64_t)blockIdx.x;
  const bool single_only = (K == 1);
  const bool triple = !split && (K >= 3) && (K & 1) && (p == K / 2 - 1);
  const bool lastcol = split && p < 0;
  bool zs = false;
  if (single_only || triple || lastcol) {
    const int64_t ts = K - 1;
    const bool hl = (ts + a.t0) > 0;
    eliminate(a, sm, f, ts, false, hl, 0, false, hl);
    if (lastcol) {
      __threadfence();   // its Z rows (zscratch) visible device-wide before the flag
      __syncthreads();
      if (threadIdx.x == 0) atomicExch(a.zflag, 1);
      return;
    }
    zs = hl && triple;
  }
  if (!single_only) {
    const int64_t t = 2 * p;
    const bool waits = split && p == K / 2 - 1 && (K - 1 + a.t0 > 0);
    eliminate(a, sm, f, t, true, (t + a.t0) > 0, p, zs || waits, false);
  }
}

// ---- backward ----
// Shared memory of the backward kernel: T = [T_l | T_r] (T_r at column np),
// the three blocks of S_II = [S_ll S_lr; S_lr^T S_rr] (S_lr^T is read
// transposed, not stored), the states.  S_{t,I} overwrites S_ll / S_rr
// column block by column block and S_tt lands in S_lr's place, so the CTA
// needs 101 KB at n = 48: two CTAs per SM.
struct BwdPlan {
  int ldt, np, offLL, offLR, offRR, offx, total;
};
__host__ __device__ inline BwdPlan bwd_plan(int n) {
  BwdPlan b;
  b.ldt = ldpad(n);
  b.np = pad8(n);
  b.offLL = b.ldt * 2 * b.np;
  b.offLR = b.offLL + b.ldt * b.np;
  b.offRR = b.offLR + b.ldt * b.np;
  b.offx = b.offRR + b.ldt * b.np;
  b.total = b.offx + 4 * b.np;
  return b;
}

// Backward level (P:592-600 and Alg. 2) for eliminated column t:
//   x_t     = w - T_l x_l - T_r x_r
//   S_{t,I} = -T S_II      (T = [T_l T_r], S_II = [S_ll S_lr; S_lr^T S_rr])
//   S_tt    = P - S_{t,I} T^T, symmetrised (reading R13)
// both products on the FP64 tensor cores (P enters as the accumulator,
// read from the R record).  S_lr (= S_{t-1,t+1}) is the cross block stored
// at level L+1; S_{t-1,t} = S_tl^T and S_{t,t+1} = S_tr are stored for level
// L-1.
template <int kRB>
__global__ void __launch_bounds__(kThreads, 2) backward_level_kernel(BackwardLevelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, nn = n * n, tid = threadIdx.x;
  const BwdPlan bp = bwd_plan(n);
  const int64_t b = blockIdx.x, t = 2 * b;
  if (t >= a.K) return;
  const bool hl = (t + a.t0) > 0, hr = (t + 1) < a.K;
  const int ldt = bp.ldt, np = bp.np, mt = np >> 3;
  double *TT = sm, *Sll = sm + bp.offLL, *Slr = sm + bp.offLR, *Srr = sm + bp.offRR, *xv = sm + bp.offx;
  const double *rec = a.rrec + b * rrec_doubles(n);
  const int64_t step = 1ll << a.shift;
  const int64_t j = ((t + 1) << a.shift) - 1, jl = j - step, jr = j + step;
  zero_smem(sm, bp.total);
  __syncthreads();
  for (int idx = tid; idx < nn; idx += blockDim.x) {   // asynchronous: all blocks in flight at once
    const int r = idx / n, c = idx - r * n;
    cp8(&TT[r + c * ldt], rec + idx);
    cp8(&TT[r + (np + c) * ldt], rec + nn + idx);
  }
  if (a.do_state) {
    const double *xlp = hl ? (jl < 0 ? a.xhalo : a.x + jl * n) : nullptr;
    const double *xrp = hr ? a.x + jr * n : nullptr;
    for (int i = tid; i < n; i += blockDim.x) {
      xv[i] = xlp ? xlp[i] : 0.0;
      xv[np + i] = xrp ? xrp[i] : 0.0;
    }
  }
  if (a.do_cov) {
    const double *Sl = hl ? (jl < 0 ? a.Shalo : a.S + jl * nn) : nullptr;
    const double *Sr = hr ? a.S + jr * nn : nullptr;
    const double *Sx = (hl && hr) ? a.Xup + b * nn : nullptr;   // slot b-1: S_{t-1,t+1}
    for (int idx = tid; idx < nn; idx += blockDim.x) {
      const int r = idx / n, c = idx - r * n;
      if (Sl) cp8(&Sll[r + c * ldt], Sl + idx);
      if (Sr) cp8(&Srr[r + c * ldt], Sr + idx);
      if (Sx) cp8(&Slr[r + c * ldt], Sx + idx);
    }
  }
  sync_loads();
  if (a.do_state) {
    for (int i = tid; i < n; i += blockDim.x) {
      double s = rec[3 * nn + i];
      for (int k = 0; k < n; ++k) s = fma(-TT[i + k * ldt], xv[k], s);
      for (int k = 0; k < n; ++k) s = fma(-TT[i + (np + k) * ldt], xv[np + k], s);
      a.x[j * n + i] = s;
    }
  }
  if (!a.do_cov) return;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int nw = blockDim.x >> 5;
  // S_{t,I} = -T S_II: work item = kRB vertically adjacent row tiles of one
  // column block (of 2 mt), sharing each B fragment (fewer shared-memory
  // loads per DMMA); the items of a warp stay in registers until every warp
  // has read S_II, then overwrite S_ll (left half) / S_rr (right half)
  constexpr int kMaxI = 4;   // items per warp: ceil(mt / kRB) * 2 mt <= kMaxI * nw (kRB = 3: n <= 48, 4: n <= 64)
  const int rb = (mt + kRB - 1) / kRB, nitem = rb * 2 * mt;
  double acc[kMaxI][kRB][2];
#pragma unroll
  for (int u = 0; u < kMaxI; ++u) {
    const int item = warp + u * nw;
#pragma unroll
    for (int v = 0; v < kRB; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
    if (item < nitem) {
      const int i0 = (item % rb) * kRB, cb = item / rb;
      const bool left = cb < mt;
      const int c0 = (left ? cb : cb - mt) * 8;
      const double *B = left ? Sll : Slr;
      for (int k0 = 0; k0 < np; k0 += 4) {   // k < np: T_l times [S_ll | S_lr]
        const double bv = B[(k0 + q) + (c0 + g) * ldt];
#pragma unroll
        for (int v = 0; v < kRB; ++v)
          if (i0 + v < mt) dmma(acc[u][v][0], acc[u][v][1], TT[((i0 + v) * 8 + g) + (k0 + q) * ldt], bv);
      }
      for (int k0 = 0; k0 < np; k0 += 4) {   // k >= np: T_r times [S_lr^T | S_rr]
        const double bv = left ? Slr[(c0 + g) + (k0 + q) * ldt] : Srr[(k0 + q) + (c0 + g) * ldt];
#pragma unroll
        for (int v = 0; v < kRB; ++v)
          if (i0 + v < mt) dmma(acc[u][v][0], acc[u][v][1], TT[((i0 + v) * 8 + g) + (np + k0 + q) * ldt], bv);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kMaxI; ++u) {
    const int item = warp + u * nw;
    if (item < nitem) {
      const int i0 = (item % rb) * kRB, cb = item / rb;
      double *D = cb < mt ? Sll : Srr;
      const int c0 = (cb < mt ? cb : cb - mt) * 8;
#pragma unroll
      for (int v = 0; v < kRB; ++v)
        if (i0 + v < mt) {
          const int m0 = (i0 + v) * 8;
          D[(m0 + g) + (c0 + 2 * q) * ldt] = -acc[u][v][0];
          D[(m0 + g) + (c0 + 2 * q + 1) * ldt] = -acc[u][v][1];
        }
    }
  }
  __syncthreads();
  // S_tt = P - S_{t,I} T^T, P the accumulator (R record, row-major), into
  // S_lr's place; items of kRB row tiles sharing the B (T^T) fragment
  const double *Pg = rec + 2 * nn;
  for (int item = warp; item < rb * mt; item += nw) {
    const int i0 = (item % rb) * kRB, n0 = (item / rb) * 8, c = n0 + 2 * q;
    double d[kRB][2];
#pragma unroll
    for (int v = 0; v < kRB; ++v) {
      const int r = (i0 + v) * 8 + g;
      d[v][0] = (i0 + v < mt && r < n && c < n) ? Pg[r * n + c] : 0.0;
      d[v][1] = (i0 + v < mt && r < n && c + 1 < n) ? Pg[r * n + c + 1] : 0.0;
    }
    for (int k0 = 0; k0 < np; k0 += 4) {
      const double bv = TT[(n0 + g) + (k0 + q) * ldt];
#pragma unroll
      for (int v = 0; v < kRB; ++v)
        if (i0 + v < mt) dmma(d[v][0], d[v][1], -Sll[((i0 + v) * 8 + g) + (k0 + q) * ldt], bv);
    }
    for (int k0 = 0; k0 < np; k0 += 4) {
      const double bv = TT[(n0 + g) + (np + k0 + q) * ldt];
#pragma unroll
      for (int v = 0; v < kRB; ++v)
        if (i0 + v < mt) dmma(d[v][0], d[v][1], -Srr[((i0 + v) * 8 + g) + (k0 + q) * ldt], bv);
    }
#pragma unroll
    for (int v = 0; v < kRB; ++v)
      if (i0 + v < mt) {
        const int r = (i0 + v) * 8 + g;
        Slr[r + c * ldt] = d[v][0];
        Slr[r + (c + 1) * ldt] = d[v][1];
      }
  }
  __syncthreads();
  double *So = a.S + j * nn;
  for (int idx = tid; idx < nn; idx += blockDim.x) {
    const int r = idx / n, c = idx - r * n;
    So[idx] = 0.5 * (Slr[r + c * ldt] + Slr[c + r * ldt]);
  }
  if (a.Xcur) {
    if (hl) {
      double *X = a.Xcur + t * nn;                   // slot t-1: S_{t-1,t} = S_tl^T
      for (int idx = tid; idx < nn; idx += blockDim.x) {
        const int r = idx / n, c = idx - r * n;
        X[idx] = Sll[c + r * ldt];
      }
    }
    if (hr) {
      double *X = a.Xcur + (t + 1) * nn;             // slot t: S_{t,t+1} = S_tr
      for (int idx = tid; idx < nn; idx += blockDim.x) {
        const int r = idx / n, c = idx - r * n;
        X[idx] = Srr[r + c * ldt];
      }
    }
  }
}

// ---------------------------------------------------------------- whiten ---

// D = Li B for Li (M x M lower triangular, shared memory, ld, zero-padded to
// pad8(M)) and B (M x N) fetched element-wise by bget(k, c) (global memory,
// masked), each result handed to put(r, c, v): 8 x 8 output tiles over the
// CTA's warps, DMMA with the B fragments loaded straight from global memory
// (no staging), the k loop cut at the tile's diagonal (Li[r][k] = 0, k > r).
template <class FB, class FO>
__device__ void trmm_lower_g(int M, int N, const double *Li, int ld, FB bget, FO put) {
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int mt = pad8(M) >> 3, nt = pad8(N) >> 3;
  for (int tile = warp; tile < mt * nt; tile += nw) {
    const int m0 = (tile % mt) * 8, n0 = (tile / mt) * 8;
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;   // two independent DMMA chains
    for (int k0 = 0; k0 <= m0; k0 += 8) {
      dmma(d0, d1, Li[(m0 + g) + (k0 + q) * ld], bget(k0 + q, n0 + g));
      dmma(e0, e1, Li[(m0 + g) + (k0 + 4 + q) * ld], bget(k0 + 4 + q, n0 + g));
    }
    put(m0 + g, n0 + 2 * q, d0 + e0);
    put(m0 + g, n0 + 2 * q + 1, d1 + e1);
  }
}

// Whitening, one step's block per CTA of kWhitenThreads:
// the Cholesky factor in shared memory, its inverse by a blocked triangular
// solve with the identity, then every whitened block as a triangular
// product with the right-hand sides read straight from global memory.  Only
// the two d x d factors live in shared memory (40 KB at d = 48: five CTAs
// per SM instead of three 256-thread CTAs holding [F | I | c]), so several
// serial Cholesky chains share each SM.
constexpr int kWhitenThreads = 128;

// Evolution blocks: K = Lam Lam^T; El = -Lam^{-1} F, Er = Lam^{-1}, e = Lam^{-1} c.
__global__ void __launch_bounds__(kWhitenThreads) whiten_evo_kernel(WhitenArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, nn = n * n, tid = threadIdx.x;
  const int64_t i = blockIdx.x;
  double *El = a.El + i * (a.cntE == 1 ? 0 : nn), *Er = a.Er + i * (a.cntE == 1 ? 0 : nn);
  double *e = a.e + i * (a.cntE == 1 ? 0 : n);
  const int64_t g = a.first_global + i;
  // no evolution row: the first step of the problem / of every batched problem
  if ((a.cntE != 1 && g % a.seg == 0) || (a.N == 1 && a.first_global == 0)) {
    for (int k = tid; k < nn; k += blockDim.x) { El[k] = 0.0; Er[k] = 0.0; }
    for (int k = tid; k < n; k += blockDim.x) e[k] = 0.0;
    return;
  }
  KS_PROF_DECL
  const int64_t iK = (a.cntE == 1) ? 0 : i;
  const int ld = ldpad(n), np = pad8(n);
  double *Lm = sm, *X = Lm + ld * np, *sh = X + ld * np;
  const double *K = a.K + iK * a.sK, *F = a.F + iK * a.sF;
  const double *c = a.c ? a.c + iK * a.sc : nullptr;
  // general model: K_i's leading l_i block, F_i's first n_{i-1}
  // columns, H_i (l_i x n_i; null: the identity's leading block)
  const int li = a.l ? a.l[i] : (a.ns ? a.ns[i] : n), ni = a.ns ? a.ns[i] : n;
  const int npv = (a.ns && i > 0) ? a.ns[i - 1] : n;
  const double *Hv = a.Hev ? a.Hev + iK * a.sHev : nullptr;
  zero_smem(sm, 2 * ld * np);
  __syncthreads();
  for (int k = tid; k < nn; k += blockDim.x) {   // asynchronous loads
    const int r = k / n, cc = k - r * n;
    if (r < li && cc < li && (!a.chol || cc <= r)) cp8(&Lm[r + cc * ld], K + k);   // KS_COV_IS_CHOL: lower only
  }
  for (int r = tid; r < n; r += blockDim.x) {
    X[r + r * ld] = 1.0;
    if (r >= li) Lm[r + r * ld] = 1.0;   // identity beyond l_i
  }
  sync_loads();
  KS_PROF(0)
  const bool ok = a.chol ? chol_diag_ok(Lm, ld, n, sh) : cta_chol(Lm, ld, n, sh);
  KS_PROF(1)
  if (tid == 0 && !ok) {
    const int64_t step = (a.cntE == 1) ? (a.first_global == 0 ? 1 : 0) : i;
    report(a.status, step, kBadK);
  }
  diag_rcp(Lm, ld, n, sh);
  __syncthreads();
  trsm_lower(Lm, ld, sh, n, X, ld, n);   // X = Lam^{-1} (ends with a barrier)
  KS_PROF(2)
  trmm_lower_g(
      n, n, X, ld, [&](int k, int cc) { return (k < li && cc < npv) ? __ldg(F + k * n + cc) : 0.0; },
      [&](int r, int cc, double v) {
        if (r < n && cc < n) El[r * n + cc] = -v;
      });
  if (Hv) {
    trmm_lower_g(
        n, n, X, ld, [&](int k, int cc) { return (k < li && cc < ni) ? __ldg(Hv + k * n + cc) : 0.0; },
        [&](int r, int cc, double v) {
          if (r < n && cc < n) Er[r * n + cc] = v;
        });
  } else {
    for (int k = tid; k < nn; k += blockDim.x) {
      const int r = k / n, cc = k - r * n;
      Er[k] = (cc < li && cc < ni) ? X[r + cc * ld] : 0.0;
    }
  }
  for (int r = tid; r < n; r += blockDim.x) {
    double s = 0.0;
    if (c)
      for (int k = 0; k <= r && k < li; ++k) s = fma(X[r + k * ld], __ldg(c + k), s);
    e[r] = s;
  }
  KS_PROF(3)
  KS_PROF_PRINT("whiten evo: loads chol trsm store")
}

// Observation blocks: L = M M^T; C = M^{-1} H, y = M^{-1} o (rows >= m_i zero).
__global__ void __launch_bounds__(kWhitenThreads) whiten_obs_kernel(WhitenArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, mx = a.m_max, tid = threadIdx.x;
  const int64_t i = blockIdx.x;
  const int mi = a.m ? a.m[i] : mx;
  const int ni = a.ns ? a.ns[i] : n;   // general model: columns >= n_i of H_i ignored
  const int rc = a.RC;
  double *C = a.C + i * (int64_t)rc * n;
  const int mx1 = mx > 0 ? mx : 1;   // (m_max = 0 with padding rows: no observation blocks)
  const int ld = ldpad(mx1), mp = pad8(mx1);
  double *Lm = sm, *X = Lm + ld * mp, *sh = X + ld * mp;
  const double *L = a.L + i * a.sL, *H = a.H + i * a.sH, *o = a.o + i * a.so;
  zero_smem(sm, 2 * ld * mp);
  __syncthreads();
  for (int k = tid; k < mi * mi; k += blockDim.x) {   // asynchronous loads
    const int r = k / mi, cc = k - r * mi;
    if (!a.chol || cc <= r) cp8(&Lm[r + cc * ld], L + r * mx + cc);   // KS_COV_IS_CHOL: lower only
  }
  for (int r = tid; r < mi; r += blockDim.x) X[r + r * ld] = 1.0;
  sync_loads();
  const bool ok = a.chol ? chol_diag_ok(Lm, ld, mi, sh) : cta_chol(Lm, ld, mi, sh);
  if (tid == 0 && !ok) report(a.status, i, kBadL);
  diag_rcp(Lm, ld, mi, sh);
  __syncthreads();
  trsm_lower(Lm, ld, sh, mi, X, ld, mi);   // X = M^{-1}
  trmm_lower_g(
      mi, n, X, ld, [&](int k, int cc) { return (k < mi && cc < ni) ? __ldg(H + k * n + cc) : 0.0; },
      [&](int r, int cc, double v) {
        if (r < mi && cc < n) C[r * n + cc] = v;
      });
  // rows m_i .. RC-1: the padding rows e_k^T x_i = 0 (k >= n_i), then zeros
  for (int k = tid; k < (rc - mi) * n; k += blockDim.x) {
    const int r = mi + k / n, cc = k % n;
    C[r * n + cc] = (r - mi < n - ni && cc == ni + (r - mi)) ? 1.0 : 0.0;
  }
  if (a.Mall) {   // KS_KEEP_WHITENING: M_i for ks_update_obs
    for (int k = tid; k < mx * mx; k += blockDim.x) {
      const int r = k / mx, cc = k - r * mx;
      a.Mall[i * (int64_t)mx * mx + k] = (cc <= r && r < mi) ? Lm[r + cc * ld] : 0.0;
    }
  }
  if (!a.constC) {
    for (int r = tid; r < rc; r += blockDim.x) {
      double s = 0.0;
      if (r < mi)
        for (int k = 0; k <= r; ++k) s = fma(X[r + k * ld], __ldg(o + k), s);
      a.y[i * rc + r] = s;
    }
  } else {
    for (int k = tid; k < mi * mi; k += blockDim.x) {
      const int r = k / mi, cc = k - r * mi;
      a.Mchol[r * mx + cc] = (cc <= r) ? Lm[r + cc * ld] : 0.0;
    }
  }
}

// Constant observation model: y_i = M^{-1} o_i, one thread per step.
__global__ void whiten_y_kernel(WhitenArgs a) {
  extern __shared__ double sm[];
  const int mx = a.m_max;
  for (int k = threadIdx.x; k < mx * mx; k += blockDim.x) sm[k] = a.Mchol[k];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double *o = a.o + i * a.so;
  double *y = a.y + i * mx;
  for (int r = 0; r < mx; ++r) {
    double s = o[r];
    for (int k = 0; k < r; ++k) s = fma(-sm[r * mx + k], y[k], s);
    y[r] = s / sm[r * mx + r];
  }
}

size_t whiten_evo_smem(int n) { return 8 * (2 * (size_t)ldpad(n) * pad8(n) + pad8(n) + 8); }
size_t whiten_obs_smem(int n, int mx) {
  (void)n;
  return 8 * (2 * (size_t)ldpad(mx) * pad8(mx) + pad8(mx) + 8);
}

}  // namespace

size_t factor_smem_bytes(int n, int RC) { return 8 * (size_t)factor_plan(n, RC).total; }

size_t backward_smem_bytes(int n) { return 8 * (size_t)bwd_plan(n).total; }

cudaError_t launch_factor_level(const FactorLevelArgs &a, cudaStream_t s) {
  set_smem_attr((const void *)factor_level_kernel, 227 * 1024);
  FactorLevelArgs b = a;
  b.zflag = nullptr;
  int64_t grid = a.K >= 2 ? a.K / 2 : 1;
  if (a.K >= 3 && (a.K & 1) && a.zscratch) {   // odd level: the last column in its own CTA
    b.zflag = reinterpret_cast<int *>(a.zscratch + (int64_t)a.n * (a.n + 1));
    cudaError_t e = cudaMemsetAsync(b.zflag, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    grid += 1;
  }
  factor_level_kernel<<<(unsigned)grid, kThreads, factor_smem_bytes(a.n, a.in.RC), s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_backward_level(const BackwardLevelArgs &a, cudaStream_t s) {
  const int mt = pad8(a.n) / 8;
  const int64_t grid = (a.K + 1) / 2;
  if ((mt + 2) / 3 * 2 * mt <= 4 * kWarps) {   // three row tiles per work item
    set_smem_attr((const void *)backward_level_kernel<3>, 227 * 1024);
    backward_level_kernel<3><<<(unsigned)grid, kThreads, backward_smem_bytes(a.n), s>>>(a);
  } else if ((mt + 3) / 4 * 2 * mt <= 4 * kWarps) {   // n <= 64
    set_smem_attr((const void *)backward_level_kernel<4>, 227 * 1024);
    backward_level_kernel<4><<<(unsigned)grid, kThreads, backward_smem_bytes(a.n), s>>>(a);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_whiten(const WhitenArgs &a, cudaStream_t s) {
  set_smem_attr((const void *)whiten_evo_kernel, 227 * 1024);
  set_smem_attr((const void *)whiten_obs_kernel, 227 * 1024);
  const int n = a.n, mx = a.m_max;
  whiten_evo_kernel<<<(unsigned)a.cntE, kWhitenThreads, whiten_evo_smem(n), s>>>(a);
  if (a.RC > 0) {
    whiten_obs_kernel<<<(unsigned)a.cntC, kWhitenThreads, whiten_obs_smem(n, mx > 0 ? mx : 1), s>>>(a);
    if (a.constC) {
      const int T = 256;
      whiten_y_kernel<<<(unsigned)((a.N + T - 1) / T), T, 8 * (size_t)mx * mx, s>>>(a);
    }
  }
  return cudaGetLastError();
}

}  // namespace ks
