// Small-n path (n <= 8, m_max <= 8) of the Odd-Even Kalman smoother.
//
// One THREAD per (even, odd) column pair / per eliminated column, every block
// held in registers (the state dimension N is a template parameter, so all
// loops unroll and all block indices are compile-time), and every block QR
// done by Givens row streaming into a packed upper-triangular R: a stacked
// QR [R; rows] is computed by rotating one row at a time into R.  Givens and
// Householder produce the same R up to row signs (both are Q R of the same
// stack), and the row-streaming form needs only one streamed row
// in registers at a time instead of the whole (2n+m) x (3n+1) stack, which is
// what lets a whole pair fit in one thread's registers.  Level arrays are
// element-major (SoA), so the 32 threads of a warp load element e of 32
// consecutive columns with one coalesced 256-byte access.
//
// P:n = line n of the paper text.
#include <cuda_runtime.h>

#include <cstdint>

#include "ks_internal.cuh"

namespace ks {

namespace {

template <int N>
struct Tri {
  static constexpr int size = N * (N + 1) / 2;
  static constexpr __host__ __device__ int at(int i, int j) { return i * N - (i * (i - 1)) / 2 + (j - i); }
};

__device__ __forceinline__ double ldc(const CArr &a, int e, int64_t t) {
  return __ldg(a.p + e * a.es + t * a.cs);
}
__device__ __forceinline__ void stv(const Arr &a, int e, int64_t t, double v) { a.p[e * a.es + t * a.cs] = v; }

__device__ __forceinline__ void report(unsigned long long *st, int64_t step, int kind) {
  if (st) atomicMin(st, ((unsigned long long)(step + 1) << 8) | (unsigned long long)kind);
}

// Givens rotation zeroing b against the pivot a: (a, b) <- (r, 0), r >= 0.
// b == 0 gives the identity (c = 1, s = 0), so zero (padding) rows are exact
// no-ops.
__device__ __forceinline__ void make_rot(double &a, double &b, double &c, double &s) {
  if (b == 0.0) {
    c = 1.0;
    s = 0.0;
    return;
  }
  const double h = fma(a, a, b * b);
  const double ih = rsqrt(h);
  c = a * ih;
  s = b * ih;
  a = h * ih;
  b = 0.0;
}

__device__ __forceinline__ void rot(double &x, double &y, double c, double s) {
  const double nx = fma(c, x, s * y);
  const double ny = fma(c, y, -(s * x));
  x = nx;
  y = ny;
}

// ---------------------------------------------------------------- factor ---

// Eliminate column t of the level in one thread.
//   stage 1: rotate the rows of [El_{t+1} | Er_{t+1} | e_{t+1}] into
//            R = C_t (level 0: the rows of C_t into R = 0 first), giving R~_t,
//            X_t, z~_t; each leftover row [0 | d | y~] (a row of D~_{t+1})
//   stage 3: is rotated at once into R3 = C_{t+1}, giving the survivor's
//            C'_{t+1} (plus the leftover Z rows of an odd level's last column)
//   stage 2: rotate the rows of [Er_t | El_t | 0 | e_t] into [R~_t | 0 | X_t | z~_t]
//            giving R_tt, R_{t,t-1}, R_{t,t+1}, z_t; the leftover rows are the
//            survivor's new coupling row [Z_t | X~_t | z^_t].  No left
//            neighbour: "nothing to do".
//   post:    T_l = R^{-1} R_{t,t-1}, T_r = R^{-1} R_{t,t+1}, w = R^{-1} z_t,
//            P = R^{-1} R^{-T} (packed) -> R record.
template <int N>
__device__ __forceinline__ void small_eliminate(const SmallFactorArgs &a, int64_t t, bool hr, bool hl,
                                                int64_t pnext, bool zs_in, bool zs_out) {
  using TR = Tri<N>;
  const SmallIn &in = a.in;
  double R[TR::size];
  double X[N][N];
  double z[N];
  double Rl[N][N];

  // rank reference: |block column of UA|_F (reading R9)
  double ref2, ref2u = 0.0;
  if (in.nrm.p) {
    const double v = ldc(in.nrm, 0, t);
    ref2 = v * v;
    if (hr) {
      const double u = ldc(in.nrm, 0, t + 1);
      ref2u = u * u;
    }
  } else {
    ref2 = ldc(in.nC, 0, t) + (hl ? ldc(in.nEr, 0, t) : 0.0) + (hr ? ldc(in.nEl, 0, t + 1) : 0.0);
    if (hr)
      ref2u = ldc(in.nC, 0, t + 1) + ldc(in.nEr, 0, t + 1) + (t + 2 < a.K ? ldc(in.nEl, 0, t + 2) : 0.0);
  }

#pragma unroll
  for (int i = 0; i < N; ++i) {
    z[i] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      X[i][j] = 0.0;
      Rl[i][j] = 0.0;
    }
  }
  // ---- stage 1 base: R = C_t ----
  if (in.tri) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) R[TR::at(i, j)] = ldc(in.C, i * N + j, t);
      z[i] = ldc(in.y, i, t);
    }
  } else {
#pragma unroll
    for (int k = 0; k < TR::size; ++k) R[k] = 0.0;
    for (int r = 0; r < in.RC; ++r) {
      double row[N];
#pragma unroll
      for (int j = 0; j < N; ++j) row[j] = ldc(in.C, r * N + j, t);
      double yr = ldc(in.y, r, t);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double c, s;
        make_rot(R[TR::at(k, k)], row[k], c, s);
#pragma unroll
        for (int j = k + 1; j < N; ++j) rot(R[TR::at(k, j)], row[j], c, s);
        rot(z[k], yr, c, s);
      }
    }
  }

  // ---- stage 1 + stage 3 ----
  if (hr) {
    const int64_t u = t + 1;
    double R3[TR::size];
    double z3[N];
    if (in.tri) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = i; j < N; ++j) R3[TR::at(i, j)] = ldc(in.C, i * N + j, u);
        z3[i] = ldc(in.y, i, u);
      }
    } else {
#pragma unroll
      for (int k = 0; k < TR::size; ++k) R3[k] = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) z3[i] = 0.0;
      for (int r = 0; r < in.RC; ++r) {
        double row[N];
#pragma unroll
        for (int j = 0; j < N; ++j) row[j] = ldc(in.C, r * N + j, u);
        double yr = ldc(in.y, r, u);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double c, s;
          make_rot(R3[TR::at(k, k)], row[k], c, s);
#pragma unroll
          for (int j = k + 1; j < N; ++j) rot(R3[TR::at(k, j)], row[j], c, s);
          rot(z3[k], yr, c, s);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double el[N], er[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        el[j] = ldc(in.El, i * N + j, u);
        er[j] = ldc(in.Er, i * N + j, u);
      }
      double ee = ldc(in.e, i, u);
#pragma unroll
      for (int k = 0; k < N; ++k) {          // stage 1: row into [R | X | z]
        double c, s;
        make_rot(R[TR::at(k, k)], el[k], c, s);
#pragma unroll
        for (int j = k + 1; j < N; ++j) rot(R[TR::at(k, j)], el[j], c, s);
#pragma unroll
        for (int j = 0; j < N; ++j) rot(X[k][j], er[j], c, s);
        rot(z[k], ee, c, s);
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {          // stage 3: leftover [er | ee] into [R3 | z3]
        double c, s;
        make_rot(R3[TR::at(k, k)], er[k], c, s);
#pragma unroll
        for (int j = k + 1; j < N; ++j) rot(R3[TR::at(k, j)], er[j], c, s);
        rot(z3[k], ee, c, s);
      }
    }
    if (zs_in) {                              // odd level: the last column's leftover Z (reading R5)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double row[N];
#pragma unroll
        for (int j = 0; j < N; ++j) row[j] = a.zscratch[i * (N + 1) + j];
        double zr = a.zscratch[i * (N + 1) + N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double c, s;
          make_rot(R3[TR::at(k, k)], row[k], c, s);
#pragma unroll
          for (int j = k + 1; j < N; ++j) rot(R3[TR::at(k, j)], row[j], c, s);
          rot(z3[k], zr, c, s);
        }
      }
    }
    const SmallOut &o = a.out;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) stv(o.C, i * N + j, pnext, j >= i ? R3[TR::at(i, j)] : 0.0);
      stv(o.y, i, pnext, z3[i]);
    }
    stv(o.nrm, 0, pnext, sqrt(ref2u));
  }

  // ---- stage 2 ----
  if (hl) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double er[N], el[N], xr[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        er[j] = ldc(in.Er, i * N + j, t);
        el[j] = ldc(in.El, i * N + j, t);
        xr[j] = 0.0;
      }
      double ee = ldc(in.e, i, t);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double c, s;
        make_rot(R[TR::at(k, k)], er[k], c, s);
#pragma unroll
        for (int j = k + 1; j < N; ++j) rot(R[TR::at(k, j)], er[j], c, s);
#pragma unroll
        for (int j = 0; j < N; ++j) rot(Rl[k][j], el[j], c, s);
#pragma unroll
        for (int j = 0; j < N; ++j) rot(X[k][j], xr[j], c, s);
        rot(z[k], ee, c, s);
      }
      if (hr) {
        const SmallOut &o = a.out;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          stv(o.El, i * N + j, pnext, el[j]);   // Z_t
          stv(o.Er, i * N + j, pnext, xr[j]);   // X~_t
        }
        stv(o.e, i, pnext, ee);                  // z^_t
      } else if (zs_out) {
#pragma unroll
        for (int j = 0; j < N; ++j) a.zscratch[i * (N + 1) + j] = el[j];
        a.zscratch[i * (N + 1) + N] = ee;
      }
    }
  } else if (hr) {
    const SmallOut &o = a.out;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        stv(o.El, i * N + j, pnext, 0.0);
        stv(o.Er, i * N + j, pnext, 0.0);
      }
      stv(o.e, i, pnext, 0.0);
    }
  }

  // ---- post: rank check, T = R^{-1}[R_l R_r], w = R^{-1} z, P = R^{-1} R^{-T} ----
  {
    const double thr = kRankTol * sqrt(ref2);
    bool bad = false;
#pragma unroll
    for (int d = 0; d < N; ++d) bad |= !(fabs(R[TR::at(d, d)]) > thr);
    if (bad) report(a.status, (((t + 1) << (a.level - a.lbase)) - 1) + a.step0, kBadRank);
  }
  double inv[N];
#pragma unroll
  for (int i = 0; i < N; ++i) inv[i] = 1.0 / R[TR::at(i, i)];
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double sl = Rl[i][c], sr = X[i][c];
#pragma unroll
      for (int k = i + 1; k < N; ++k) {
        sl = fma(-R[TR::at(i, k)], Rl[k][c], sl);
        sr = fma(-R[TR::at(i, k)], X[k][c], sr);
      }
      Rl[i][c] = sl * inv[i];
      X[i][c] = sr * inv[i];
    }
    double sz = z[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) sz = fma(-R[TR::at(i, k)], z[k], sz);
    z[i] = sz * inv[i];
  }
  const int64_t rcol = t >> 1;
  const SmallRec &rec = a.rec;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      stv(rec.Tl, i * N + j, rcol, Rl[i][j]);
      stv(rec.Tr, i * N + j, rcol, X[i][j]);
    }
    stv(rec.w, i, rcol, z[i]);
  }
  // R^{-1} (upper, in place of R): Ri(i,j) = -inv_i sum_{k=i+1..j} R(i,k) Ri(k,j)
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
#pragma unroll
    for (int j = N - 1; j > i; --j) {
      double s = 0.0;
#pragma unroll
      for (int k = i + 1; k <= j; ++k) s = fma(R[TR::at(i, k)], R[TR::at(k, j)], s);
      R[TR::at(i, j)] = -s * inv[i];
    }
    R[TR::at(i, i)] = inv[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = i; j < N; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < N; ++k) s = fma(R[TR::at(i, k)], R[TR::at(j, k)], s);
      stv(rec.P, TR::at(i, j), rcol, s);
    }
  }
}

template <int N>
__global__ void __launch_bounds__(64) small_factor_kernel(SmallFactorArgs a) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t K = a.K;
  const int64_t npairs = K >= 2 ? K / 2 : 1;
  if (p >= npairs) return;
  const bool single_only = (K == 1);
  const bool triple = (K >= 3) && (K & 1) && (p == K / 2 - 1);
  bool zs = false;
  if (single_only || triple) {
    const int64_t ts = K - 1;
    const bool hl = ts + a.t0 > 0;
    small_eliminate<N>(a, ts, false, hl, 0, false, hl);
    zs = hl && triple;
  }
  if (!single_only) small_eliminate<N>(a, 2 * p, true, 2 * p + a.t0 > 0, p, zs, false);
}

// -------------------------------------------------------------- backward ---

// One thread per eliminated column t of level L (P:592-600 and Alg. 2,
// P:792-824):
//   x_t    = w - T_l x_l - T_r x_r
//   S_tl   = -(T_l S_ll + T_r S_lr^T),  S_tr = -(T_l S_lr + T_r S_rr)   (S_{t,I} = -T S_II)
//   S_tt   = P - S_tl T_l^T - S_tr T_r^T  (upper triangle computed, mirrored)
// S_lr = S_{t-1,t+1} is the level-(L+1) cross block; S_{t-1,t} = S_tl^T and
// S_{t,t+1} = S_tr are stored for level L-1.
template <int N>
__global__ void __launch_bounds__(64) small_backward_kernel(SmallBackwardArgs a) {
  using TR = Tri<N>;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t t = 2 * b;
  if (t >= a.K) return;
  const bool hl = (t + a.t0) > 0, hr = (t + 1) < a.K;
  const int64_t step = 1ll << a.shift;
  const int64_t j = ((t + 1) << a.shift) - 1, jl = j - step, jr = j + step;
  if (a.do_state) {
    double xl[N], xr[N];
    const double *pl = hl ? (jl < 0 ? a.xhalo : a.x + jl * N) : nullptr;
    const double *pr = hr ? a.x + jr * N : nullptr;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      xl[k] = pl ? pl[k] : 0.0;
      xr[k] = pr ? pr[k] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = ldc(a.w, i, b);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s = fma(-ldc(a.Tl, i * N + k, b), xl[k], s);
        s = fma(-ldc(a.Tr, i * N + k, b), xr[k], s);
      }
      a.x[j * N + i] = s;
    }
  }
  if (!a.do_cov) return;
  double Sll[TR::size], Srr[TR::size], Slr[N][N];
  {
    const double *pl = hl ? (jl < 0 ? a.Shalo : a.S + jl * N * N) : nullptr;
    const double *pr = hr ? a.S + jr * N * N : nullptr;
#pragma unroll
    for (int r = 0; r < N; ++r) {
#pragma unroll
      for (int c = r; c < N; ++c) {
        Sll[TR::at(r, c)] = pl ? pl[r * N + c] : 0.0;
        Srr[TR::at(r, c)] = pr ? pr[r * N + c] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < N; ++c) Slr[r][c] = (hl && hr) ? ldc(a.Xup, r * N + c, b) : 0.0;
    }
  }
  double *So = a.S + j * N * N;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double tl[N], tr[N], A[N], B[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      tl[k] = ldc(a.Tl, i * N + k, b);
      tr[k] = ldc(a.Tr, i * N + k, b);
    }
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double sll = k <= c ? Sll[TR::at(k, c)] : Sll[TR::at(c, k)];
        const double srr = k <= c ? Srr[TR::at(k, c)] : Srr[TR::at(c, k)];
        sa = fma(tl[k], sll, sa);
        sa = fma(tr[k], Slr[c][k], sa);
        sb = fma(tl[k], Slr[k][c], sb);
        sb = fma(tr[k], srr, sb);
      }
      A[c] = -sa;
      B[c] = -sb;
    }
    if (a.Xcur.p) {
#pragma unroll
      for (int c = 0; c < N; ++c) {
        if (hl) stv(a.Xcur, c * N + i, t, A[c]);       // slot t-1: S_{t-1,t} = S_tl^T
        if (hr) stv(a.Xcur, i * N + c, t + 1, B[c]);   // slot t:   S_{t,t+1} = S_tr
      }
    }
    // row i of S_tt (upper part j >= i)
#pragma unroll
    for (int jj = i; jj < N; ++jj) {
      double s = ldc(a.P, TR::at(i, jj), b);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s = fma(-A[k], ldc(a.Tl, jj * N + k, b), s);
        s = fma(-B[k], ldc(a.Tr, jj * N + k, b), s);
      }
      So[i * N + jj] = s;
      So[jj * N + i] = s;
    }
  }
}

// ---------------------------------------------------------------- whiten ---

// Evolution blocks: K = Lam Lam^T (Cholesky), El = -Lam^{-1}F,
// Er = Lam^{-1}, e = Lam^{-1} c.  One thread per distinct block.
template <int N>
__global__ void __launch_bounds__(128) small_whiten_evo(SmallWhitenArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.cntE) return;
  const int64_t g = a.first_global + i;
  const bool evo = !((a.cntE != 1 && g == 0) || (a.N == 1 && a.first_global == 0));
  if (!evo) {
#pragma unroll
    for (int k = 0; k < N * N; ++k) {
      stv(a.El, k, i, 0.0);
      stv(a.Er, k, i, 0.0);
    }
#pragma unroll
    for (int k = 0; k < N; ++k) stv(a.e, k, i, 0.0);
    stv(a.nEr, 0, i, 0.0);
    stv(a.nEl, 0, i, 0.0);
    return;
  }
  const int64_t iK = (a.cntE == 1) ? 0 : i;
  const double *K = a.K + iK * a.sK, *F = a.F + iK * a.sF;
  const double *cc = a.c ? a.c + iK * a.sc : nullptr;
  double Lm[N][N];
  bool ok = true;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) Lm[r][c] = K[r * N + c];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double d = Lm[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d = fma(-Lm[j][k], Lm[j][k], d);
    ok &= d > 0.0;
    const double ljj = sqrt(d > 0.0 ? d : 1.0), il = 1.0 / ljj;
    Lm[j][j] = ljj;
#pragma unroll
    for (int r = j + 1; r < N; ++r) {
      double v = Lm[r][j];
#pragma unroll
      for (int k = 0; k < j; ++k) v = fma(-Lm[r][k], Lm[j][k], v);
      Lm[r][j] = v * il;
    }
  }
  if (!ok) report(a.status, (a.cntE == 1) ? (a.first_global == 0 ? 1 : 0) : i, kBadK);
  double il[N];
#pragma unroll
  for (int r = 0; r < N; ++r) il[r] = 1.0 / Lm[r][r];
  double nel = 0.0, ner = 0.0;
  // El = -Lam^{-1} F, column by column
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double x[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = F[r * N + c];
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
      x[r] = s * il[r];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      stv(a.El, r * N + c, i, -x[r]);
      nel = fma(x[r], x[r], nel);
    }
  }
  // Er = Lam^{-1} (lower triangular)
#pragma unroll
  for (int c = 0; c < N; ++c) {
    double x[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
      x[r] = (r < c) ? 0.0 : s * il[r];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      stv(a.Er, r * N + c, i, x[r]);
      ner = fma(x[r], x[r], ner);
    }
  }
  {
    double x[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = cc ? cc[r] : 0.0;
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
      x[r] = s * il[r];
      stv(a.e, r, i, x[r]);
    }
  }
  stv(a.nEr, 0, i, ner);
  stv(a.nEl, 0, i, nel);
}

// Observation blocks: L = M M^T; C = M^{-1} H, y = M^{-1} o (rows >= m_i are 0).
// One thread per distinct block; m_i <= kSmallMaxM.
template <int N>
__global__ void __launch_bounds__(128) small_whiten_obs(SmallWhitenArgs a) {
  constexpr int MM = kSmallMaxM;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.cntC) return;
  const int mx = a.m_max;
  const int mi = a.m ? a.m[i] : mx;
  const double *L = a.L + i * a.sL, *H = a.H + i * a.sH, *o = a.o + i * a.so;
  double Lm[MM][MM];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < MM; ++j) {
    if (j < mi) {
      double d = L[j * mx + j];
#pragma unroll
      for (int k = 0; k < j; ++k) d = fma(-Lm[j][k], Lm[j][k], d);
      ok &= d > 0.0;
      const double ljj = sqrt(d > 0.0 ? d : 1.0), il = 1.0 / ljj;
      Lm[j][j] = ljj;
#pragma unroll
      for (int r = j + 1; r < MM; ++r) {
        if (r < mi) {
          double v = L[r * mx + j];
#pragma unroll
          for (int k = 0; k < j; ++k) v = fma(-Lm[r][k], Lm[j][k], v);
          Lm[r][j] = v * il;
        }
      }
    }
  }
  if (!ok) report(a.status, i, kBadL);
  double nc = 0.0;
#pragma unroll
  for (int c = 0; c <= N; ++c) {          // N columns of H, then o
    const bool is_o = (c == N);
    if (is_o && a.constC) break;
    double x[MM];
#pragma unroll
    for (int r = 0; r < MM; ++r) {
      if (r < mi) {
        double s = is_o ? o[r] : H[r * N + c];
#pragma unroll
        for (int k = 0; k < r; ++k) s = fma(-Lm[r][k], x[k], s);
        x[r] = s / Lm[r][r];
      } else {
        x[r] = 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < MM; ++r) {
      if (r < mx) {
        if (is_o) {
          stv(a.y, r, i, x[r]);
        } else {
          stv(a.C, r * N + c, i, x[r]);
          nc = fma(x[r], x[r], nc);
        }
      }
    }
  }
  stv(a.nC, 0, i, nc);
  if (a.constC) {
#pragma unroll
    for (int r = 0; r < MM; ++r)
#pragma unroll
      for (int k = 0; k < MM; ++k)
        if (r < mx && k < mx) a.Mchol[r * mx + k] = (k <= r && r < mi) ? Lm[r][k] : 0.0;
  }
}

// Constant observation model: y_i = M^{-1} o_i, one thread per step.
__global__ void __launch_bounds__(256) small_whiten_y(SmallWhitenArgs a) {
  __shared__ double M[kSmallMaxM * kSmallMaxM];
  const int mx = a.m_max;
  for (int k = threadIdx.x; k < mx * mx; k += blockDim.x) M[k] = a.Mchol[k];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  const double *o = a.o + i * a.so;
  double y[kSmallMaxM];
#pragma unroll
  for (int r = 0; r < kSmallMaxM; ++r) {
    if (r < mx) {
      double s = o[r];
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-M[r * mx + k], y[k], s);
      y[r] = s / M[r * mx + r];
      stv(a.y, r, i, y[r]);
    }
  }
}

template <int N>
cudaError_t factor_n(const SmallFactorArgs &a, cudaStream_t s) {
  const int64_t np = a.K >= 2 ? a.K / 2 : 1;
  const int T = 64;
  small_factor_kernel<N><<<(unsigned)((np + T - 1) / T), T, 0, s>>>(a);
  return cudaGetLastError();
}

template <int N>
cudaError_t backward_n(const SmallBackwardArgs &a, cudaStream_t s) {
  const int64_t nc = (a.K + 1) / 2;
  const int T = 64;
  small_backward_kernel<N><<<(unsigned)((nc + T - 1) / T), T, 0, s>>>(a);
  return cudaGetLastError();
}

template <int N>
cudaError_t whiten_n(const SmallWhitenArgs &a, cudaStream_t s, int *nl) {
  const int T = 128;
  small_whiten_evo<N><<<(unsigned)((a.cntE + T - 1) / T), T, 0, s>>>(a);
  *nl = 1;
  if (a.m_max > 0) {
    small_whiten_obs<N><<<(unsigned)((a.cntC + T - 1) / T), T, 0, s>>>(a);
    *nl += 1;
    if (a.constC) {
      small_whiten_y<<<(unsigned)((a.N + 255) / 256), 256, 0, s>>>(a);
      *nl += 1;
    }
  }
  return cudaGetLastError();
}

}  // namespace

size_t small_entry_doubles(int n) { return (size_t)entry_doubles(n); }
int64_t small_rrec_doubles(int n) { return 2ll * n * n + n + (int64_t)n * (n + 1) / 2; }

#define KS_SMALL_DISPATCH(fn, n, ...)            \
  switch (n) {                                  \
    case 1: return fn<1>(__VA_ARGS__);          \
    case 2: return fn<2>(__VA_ARGS__);          \
    case 3: return fn<3>(__VA_ARGS__);          \
    case 4: return fn<4>(__VA_ARGS__);          \
    case 5: return fn<5>(__VA_ARGS__);          \
    case 6: return fn<6>(__VA_ARGS__);          \
    case 7: return fn<7>(__VA_ARGS__);          \
    case 8: return fn<8>(__VA_ARGS__);          \
    default: return cudaErrorInvalidValue;      \
  }

cudaError_t launch_small_factor(const SmallFactorArgs &a, int n, cudaStream_t s) {
  KS_SMALL_DISPATCH(factor_n, n, a, s)
}
cudaError_t launch_small_backward(const SmallBackwardArgs &a, int n, cudaStream_t s) {
  KS_SMALL_DISPATCH(backward_n, n, a, s)
}
cudaError_t launch_small_whiten(const SmallWhitenArgs &a, cudaStream_t s, int *nlaunch) {
  KS_SMALL_DISPATCH(whiten_n, a.n, a, s, nlaunch)
}

}  // namespace ks
