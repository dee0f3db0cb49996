// sm_100a fp64 kernels of the Odd-Even Kalman smoother: the generic path.
//
// One CTA per eliminated column (pair) with the stage matrices resident in
// shared memory (column-major, odd leading dimension so that a warp reading
// one row across 32 columns is conflict-free), Householder reflectors computed
// by warp 0 with shuffle reductions and applied column-parallel by all
// threads.  This path handles every n, m_i up to the shared-memory limit
// (n = m = 48 fits); the small-n register path lives in ks_small.cu.
//
// P:n = line n of the paper text.
#include <cuda_runtime.h>

#include <cstdint>

#include "ks_internal.cuh"

namespace ks {

namespace {

__device__ __forceinline__ void report(unsigned long long *st, int64_t step, int kind) {
  if (st) atomicMin(st, ((unsigned long long)(step + 1) << 8) | (unsigned long long)kind);
}

// smem column-major A(lda)[r0:r0+rows, c0:c0+cols] <- scale * g (row-major, ldg);
// rows >= valid (or g == null) are zero.
__device__ void ld_blk(double *A, int lda, int r0, int c0, const double *g, int64_t ldg, int rows,
                       int cols, int valid, double scale) {
  const int tot = rows * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx / cols, j = idx - i * cols;
    double v = 0.0;
    if (g != nullptr && i < valid) v = scale * g[(int64_t)i * ldg + j];
    A[(r0 + i) + (c0 + j) * lda] = v;
  }
}

__device__ void zero_blk(double *A, int lda, int r0, int c0, int rows, int cols) {
  const int tot = rows * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx / cols, j = idx - i * cols;
    A[(r0 + i) + (c0 + j) * lda] = 0.0;
  }
}

// smem -> smem block copy
__device__ void cp_blk(double *D, int ldd, int dr, int dc, const double *A, int lda, int r0, int c0,
                       int rows, int cols) {
  const int tot = rows * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx / cols, j = idx - i * cols;
    D[(dr + i) + (dc + j) * ldd] = A[(r0 + i) + (c0 + j) * lda];
  }
}

// smem (column-major) -> global row-major (ldg); rows >= valid are written as 0
__device__ void st_blk(double *g, int64_t ldg, const double *A, int lda, int r0, int c0, int rows,
                       int cols, int valid) {
  const int tot = rows * cols;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int i = idx / cols, j = idx - i * cols;
    g[(int64_t)i * ldg + j] = (i < valid) ? A[(r0 + i) + (c0 + j) * lda] : 0.0;
  }
}

// Householder QR in shared memory ("QR factorizations of the last
// two nonzero block rows ... apply the Q factors"): triangularise columns
// [0, npiv) of the rows x ncols column-major matrix A and apply the same
// reflectors to columns [npiv, ncols).  Reflector k: v = x - alpha e_1,
// alpha = -sign(x_1)|x|, H = I - beta v v^T with beta = 1/(|x|^2 - x_1 alpha);
// a zero column is skipped.  On exit column k holds R(:,k) (zeros below).
__device__ void cta_house(double *A, int lda, int rows, int npiv, int ncols, double *sh) {
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int k = 0; k < npiv && k < rows; ++k) {
    if (tid < 32) {
      double s = 0.0;
      for (int i = k + tid; i < rows; i += 32) {
        const double v = A[i + k * lda];
        s = fma(v, v, s);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (tid == 0) {
        const double x1 = A[k + k * lda];
        if (s == 0.0) {
          sh[0] = 0.0;
          sh[1] = x1;
        } else {
          const double nrm = sqrt(s);
          const double alpha = (x1 > 0.0) ? -nrm : nrm;
          A[k + k * lda] = x1 - alpha;
          sh[0] = 1.0 / (s - x1 * alpha);
          sh[1] = alpha;
        }
      }
    }
    __syncthreads();
    const double beta = sh[0];
    if (beta != 0.0) {
      const double *vk = A + k * lda;
      for (int j = k + 1 + tid; j < ncols; j += NT) {
        double *aj = A + j * lda;
        double s = 0.0;
        for (int i = k; i < rows; ++i) s = fma(vk[i], aj[i], s);
        s *= beta;
        for (int i = k; i < rows; ++i) aj[i] = fma(-s, vk[i], aj[i]);
      }
    }
    __syncthreads();
    for (int i = k + tid; i < rows; i += NT) A[i + k * lda] = (i == k) ? sh[1] : 0.0;
    __syncthreads();
  }
}

// Sum of squares of `count` contiguous doubles, reduced by warp 0 and
// returned to every thread through sh[2].
__device__ double cta_sumsq(const double *g, int count, double *sh) {
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < count; i += 32) s = fma(g[i], g[i], s);
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0) sh[2] = s;
  }
  __syncthreads();
  return sh[2];
}

// |UA block column of level-0 column t|_F^2 = |C_t|^2 + |Er_t|^2 + |El_{t+1}|^2.
__device__ double col_norm2_l0(const EntryView &in, int n, int64_t t, bool hl, bool hr, double *sh) {
  double s = cta_sumsq(in.C + t * in.sC, in.RC * n, sh);
  if (hl) s += cta_sumsq(in.Er + t * in.sEr, n * n, sh);
  if (hr) s += cta_sumsq(in.El + (t + 1) * in.sEl, n * n, sh);
  return s;
}

struct FactorSmem {
  int lda1, lda2, lda3, szB;
  double *S1, *B, *Zs, *scr, *sh;
};

__device__ FactorSmem carve(double *sm, int n, int RC) {
  FactorSmem f;
  f.lda1 = (RC + n) | 1;
  f.lda2 = (2 * n) | 1;
  f.lda3 = (2 * RC + n) | 1;
  const int s2 = f.lda2 * (3 * n + 1), s3 = f.lda3 * (n + 1);
  f.szB = s2 > s3 ? s2 : s3;
  f.S1 = sm;
  f.B = f.S1 + f.lda1 * (2 * n + 1);
  f.Zs = f.B + f.szB;
  f.scr = f.Zs + n * (n + 1);
  f.sh = f.scr + n * n;
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
// case) uses an empty right neighbour; its stage-2 leftover Z (acting on t-1
// only) is returned in Zs_out to join the left pair's stage 3 (reading R5).
// Writes the R record T = R^{-1}[R_l R_r], P = R^{-1}R^{-T}, w = R^{-1} z.
__device__ void eliminate(const FactorLevelArgs &a, FactorSmem &f, int64_t t, bool has_right,
                          bool has_left, int64_t pnext, const double *Zs_in, double *Zs_out) {
  const int n = a.n, RC = a.in.RC, tid = threadIdx.x, NT = blockDim.x;
  const EntryView &in = a.in;
  const int lda1 = f.lda1, lda2 = f.lda2, lda3 = f.lda3;
  double *S1 = f.S1, *B = f.B;

  // reference norms for the rank test (column t) and for the survivor t+1
  double nrm_t, nrm_u = 0.0;
  if (in.nrm) {
    nrm_t = in.nrm[t * in.snrm];
    if (has_right) nrm_u = in.nrm[(t + 1) * in.snrm];
  } else {
    nrm_t = sqrt(col_norm2_l0(in, n, t, has_left, has_right, f.sh));
    if (has_right) nrm_u = sqrt(col_norm2_l0(in, n, t + 1, true, t + 2 < a.K, f.sh));
  }

  // ---- stage 1 ----
  ld_blk(S1, lda1, 0, 0, in.C + t * in.sC, n, RC, n, RC, 1.0);
  zero_blk(S1, lda1, 0, n, RC, n);
  ld_blk(S1, lda1, 0, 2 * n, in.y + t * in.sy, 1, RC, 1, RC, 1.0);
  if (has_right) {
    const int64_t u = t + 1;
    ld_blk(S1, lda1, RC, 0, in.El + u * in.sEl, n, n, n, n, 1.0);
    ld_blk(S1, lda1, RC, n, in.Er + u * in.sEr, n, n, n, n, 1.0);
    ld_blk(S1, lda1, RC, 2 * n, in.e + u * in.se, 1, n, 1, n, 1.0);
  } else {
    zero_blk(S1, lda1, RC, 0, n, 2 * n + 1);
  }
  __syncthreads();
  cta_house(S1, lda1, RC + n, n, 2 * n + 1, f.sh);

  // ---- stage 3 (before stage 2 so that B can be reused) ----
  if (has_right) {
    const int64_t u = t + 1;
    cp_blk(B, lda3, 0, 0, S1, lda1, n, n, RC, n);          // D~_{t+1}
    cp_blk(B, lda3, 0, n, S1, lda1, n, 2 * n, RC, 1);      // y~_{t+1}
    ld_blk(B, lda3, RC, 0, in.C + u * in.sC, n, RC, n, RC, 1.0);
    ld_blk(B, lda3, RC, n, in.y + u * in.sy, 1, RC, 1, RC, 1.0);
    int rows3 = 2 * RC;
    if (Zs_in) {
      cp_blk(B, lda3, rows3, 0, Zs_in, n, 0, 0, n, n + 1);
      rows3 += n;
    }
    __syncthreads();
    cta_house(B, lda3, rows3, n, n + 1, f.sh);
    double *ent = a.next + pnext * entry_doubles(n);
    const int valid = rows3 < n ? rows3 : n;
    st_blk(ent, n, B, lda3, 0, 0, n, n, valid);             // C'
    st_blk(ent + n * n, 1, B, lda3, 0, n, n, 1, valid);     // y'
    if (tid == 0) ent[3 * n * n + 2 * n] = nrm_u;
    __syncthreads();
  }

  // ---- stage 2 ----
  if (has_left) {
    ld_blk(B, lda2, 0, 0, in.Er + t * in.sEr, n, n, n, n, 1.0);
    ld_blk(B, lda2, 0, n, in.El + t * in.sEl, n, n, n, n, 1.0);
    zero_blk(B, lda2, 0, 2 * n, n, n);
    ld_blk(B, lda2, 0, 3 * n, in.e + t * in.se, 1, n, 1, n, 1.0);
    cp_blk(B, lda2, n, 0, S1, lda1, 0, 0, n, n);            // R~_t
    zero_blk(B, lda2, n, n, n, n);
    cp_blk(B, lda2, n, 2 * n, S1, lda1, 0, n, n, n);        // X_t
    cp_blk(B, lda2, n, 3 * n, S1, lda1, 0, 2 * n, n, 1);    // z~_t
    __syncthreads();
    cta_house(B, lda2, 2 * n, n, 3 * n + 1, f.sh);
    if (has_right) {
      double *ent = a.next + pnext * entry_doubles(n);
      st_blk(ent + n * n + n, n, B, lda2, n, n, n, n, n);               // El' = Z_t
      st_blk(ent + 2 * n * n + n, n, B, lda2, n, 2 * n, n, n, n);       // Er' = X~_t
      st_blk(ent + 3 * n * n + n, 1, B, lda2, n, 3 * n, n, 1, n);       // e'  = z^_t
    } else if (Zs_out) {
      cp_blk(Zs_out, n, 0, 0, B, lda2, n, n, n, n);                     // Z_t
      cp_blk(Zs_out, n, 0, n, B, lda2, n, 3 * n, n, 1);                 // z^_t
    }
  } else {
    cp_blk(B, lda2, 0, 0, S1, lda1, 0, 0, n, n);
    zero_blk(B, lda2, 0, n, n, n);
    cp_blk(B, lda2, 0, 2 * n, S1, lda1, 0, n, n, n);
    cp_blk(B, lda2, 0, 3 * n, S1, lda1, 0, 2 * n, n, 1);
    if (has_right) {
      double *ent = a.next + pnext * entry_doubles(n);
      for (int i = tid; i < 2 * n * n + n; i += NT) ent[n * n + n + i] = 0.0;
    }
  }
  __syncthreads();

  // ---- R record: rank check, T = R^{-1}[R_l R_r], w = R^{-1} z, P = R^{-1} R^{-T} ----
  if (tid == 0) {
    const double thr = kRankTol * nrm_t;
    bool bad = false;
    for (int d = 0; d < n; ++d) bad |= !(fabs(B[d + d * lda2]) > thr);
    if (bad) {
      const int64_t step = (((t + 1) << (a.level - a.lbase)) - 1) + a.step0;
      report(a.status, step, kBadRank);
    }
  }
  for (int j = n + tid; j <= 3 * n; j += NT) {        // back-substitution, 2n+1 RHS columns
    double *x = B + j * lda2;
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int k = i + 1; k < n; ++k) s = fma(-B[i + k * lda2], x[k], s);
      x[i] = s / B[i + i * lda2];
    }
  }
  double *Ri = f.scr;                                  // R^{-1}, column-major n x n
  for (int c = tid; c < n; c += NT) {
    for (int i = n - 1; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = i + 1; k < n; ++k) s = fma(-B[i + k * lda2], Ri[k + c * n], s);
      Ri[i + c * n] = (i > c) ? 0.0 : s / B[i + i * lda2];
    }
  }
  __syncthreads();
  double *rec = a.rrec + (t >> 1) * rrec_doubles(n);
  const int nn = n * n;
  for (int idx = tid; idx < nn; idx += NT) {
    const int r = idx / n, c = idx - r * n;
    rec[idx] = B[r + (n + c) * lda2];                  // Tl
    rec[nn + idx] = B[r + (2 * n + c) * lda2];         // Tr
    double s = 0.0;
    const int k0 = r > c ? r : c;
    for (int k = k0; k < n; ++k) s = fma(Ri[r + k * n], Ri[c + k * n], s);
    rec[2 * nn + idx] = s;                             // P
  }
  for (int r = tid; r < n; r += NT) rec[3 * nn + r] = B[r + 3 * n * lda2];   // w
  __syncthreads();
}

__global__ void factor_level_kernel(FactorLevelArgs a) {
  extern __shared__ double sm[];
  FactorSmem f = carve(sm, a.n, a.in.RC);
  const int64_t K = a.K, p = blockIdx.x;
  const bool single_only = (K == 1);
  const bool triple = (K >= 3) && (K & 1) && (p == K / 2 - 1);
  const double *zs = nullptr;
  if (single_only || triple) {
    const int64_t ts = K - 1;
    const bool hl = (ts + a.t0) > 0;
    eliminate(a, f, ts, false, hl, 0, nullptr, hl ? f.Zs : nullptr);
    if (hl && triple) zs = f.Zs;
  }
  if (!single_only) {
    const int64_t t = 2 * p;
    eliminate(a, f, t, true, (t + a.t0) > 0, p, zs, nullptr);
  }
}

// Backward level (P:592-600 and Alg. 2) for eliminated column t:
//   x_t  = w - T_l x_l - T_r x_r
//   S_{t,I} = -T S_II  (S_tl = -(T_l S_ll + T_r S_lr^T), S_tr = -(T_l S_lr + T_r S_rr))
//   S_tt = P - S_tl T_l^T - S_tr T_r^T, symmetrised (reading R13)
// S_lr (= S_{t-1,t+1}) is the cross block stored at level L+1.
__global__ void backward_level_kernel(BackwardLevelArgs a) {
  extern __shared__ double sm[];
  const int n = a.n, nn = n * n, tid = threadIdx.x, NT = blockDim.x;
  const int64_t b = blockIdx.x, t = 2 * b;
  if (t >= a.K) return;
  const bool hl = (t + a.t0) > 0, hr = (t + 1) < a.K;
  double *Tl = sm, *Tr = Tl + nn, *P = Tr + nn, *w = P + nn;
  double *Sll = w + n, *Srr = Sll + nn, *Slr = Srr + nn, *A = Slr + nn, *Bm = A + nn, *St = Bm + nn;
  double *xl = St + nn, *xr = xl + n;
  const double *rec = a.rrec + b * rrec_doubles(n);
  for (int i = tid; i < 3 * nn + n; i += NT) Tl[i] = rec[i];
  const int64_t step = 1ll << a.shift;
  const int64_t j = ((t + 1) << a.shift) - 1, jl = j - step, jr = j + step;
  const double *xlp = hl ? (jl < 0 ? a.xhalo : a.x + jl * n) : nullptr;
  const double *xrp = hr ? a.x + jr * n : nullptr;
  if (a.do_state) {
    for (int i = tid; i < n; i += NT) {
      xl[i] = xlp ? xlp[i] : 0.0;
      xr[i] = xrp ? xrp[i] : 0.0;
    }
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      double s = w[i];
      for (int k = 0; k < n; ++k) s = fma(-Tl[i * n + k], xl[k], s);
      for (int k = 0; k < n; ++k) s = fma(-Tr[i * n + k], xr[k], s);
      a.x[j * n + i] = s;
    }
  }
  if (a.do_cov) {
    const double *Sl = hl ? (jl < 0 ? a.Shalo : a.S + jl * nn) : nullptr;
    const double *Sr = hr ? a.S + jr * nn : nullptr;
    const double *Sx = (hl && hr) ? a.Xup + b * nn : nullptr;   // slot b-1
    for (int i = tid; i < nn; i += NT) {
      Sll[i] = Sl ? Sl[i] : 0.0;
      Srr[i] = Sr ? Sr[i] : 0.0;
      Slr[i] = Sx ? Sx[i] : 0.0;
    }
    __syncthreads();
    for (int idx = tid; idx < nn; idx += NT) {
      const int r = idx / n, c = idx - r * n;
      double sa = 0.0, sb = 0.0;
      for (int k = 0; k < n; ++k) {
        sa = fma(Tl[r * n + k], Sll[k * n + c], sa);
        sa = fma(Tr[r * n + k], Slr[c * n + k], sa);
        sb = fma(Tl[r * n + k], Slr[k * n + c], sb);
        sb = fma(Tr[r * n + k], Srr[k * n + c], sb);
      }
      A[idx] = -sa;
      Bm[idx] = -sb;
    }
    __syncthreads();
    for (int idx = tid; idx < nn; idx += NT) {
      const int r = idx / n, c = idx - r * n;
      double s = P[idx];
      for (int k = 0; k < n; ++k) {
        s = fma(-A[r * n + k], Tl[c * n + k], s);
        s = fma(-Bm[r * n + k], Tr[c * n + k], s);
      }
      St[idx] = s;
    }
    __syncthreads();
    double *So = a.S + j * nn;
    for (int idx = tid; idx < nn; idx += NT) {
      const int r = idx / n, c = idx - r * n;
      So[idx] = 0.5 * (St[r * n + c] + St[c * n + r]);
    }
    if (a.Xcur) {
      if (hl) {
        double *X = a.Xcur + t * nn;                   // slot t-1: S_{t-1,t} = S_tl^T
        for (int idx = tid; idx < nn; idx += NT) {
          const int r = idx / n, c = idx - r * n;
          X[idx] = A[c * n + r];
        }
      }
      if (hr) {
        double *X = a.Xcur + (t + 1) * nn;             // slot t: S_{t,t+1} = S_tr
        for (int idx = tid; idx < nn; idx += NT) X[idx] = Bm[idx];
      }
    }
  }
}

// ---------------------------------------------------------------- whiten ---

// Cholesky (right-looking) of the d x d column-major smem matrix Lm in place;
// returns false (to thread 0) if a pivot is <= 0.
__device__ bool cta_chol(double *Lm, int d, double *sh) {
  const int tid = threadIdx.x, NT = blockDim.x;
  bool ok = true;
  for (int j = 0; j < d; ++j) {
    if (tid == 0) {
      const double v = Lm[j + j * d];
      if (!(v > 0.0)) ok = false;
      sh[0] = sqrt(v > 0.0 ? v : 1.0);
      Lm[j + j * d] = sh[0];
    }
    __syncthreads();
    const double ljj = sh[0];
    for (int i = j + 1 + tid; i < d; i += NT) Lm[i + j * d] /= ljj;
    __syncthreads();
    const int m = d - j - 1;
    for (int idx = tid; idx < m * m; idx += NT) {
      const int i = j + 1 + idx / m, k = j + 1 + idx % m;
      if (k <= i) Lm[i + k * d] = fma(-Lm[i + j * d], Lm[k + j * d], Lm[i + k * d]);
    }
    __syncthreads();
  }
  return ok;
}

// X (d x p, column-major, ldx) <- Lm^{-1} X by forward substitution, thread per column.
__device__ void cta_fwd(const double *Lm, int d, double *X, int ldx, int p) {
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    double *x = X + c * ldx;
    for (int r = 0; r < d; ++r) {
      double s = x[r];
      for (int k = 0; k < r; ++k) s = fma(-Lm[r + k * d], x[k], s);
      x[r] = s / Lm[r + r * d];
    }
  }
}

// Evolution blocks: K = Lam Lam^T; El = -Lam^{-1} F,
// Er = Lam^{-1}, e = Lam^{-1} c.  One CTA per distinct block.
__global__ void whiten_evo_kernel(WhitenArgs a) {
  extern __shared__ double sm[];
  const int n = a.n, nn = n * n, tid = threadIdx.x, NT = blockDim.x;
  const int64_t i = blockIdx.x;
  double *El = a.El + i * (a.cntE == 1 ? 0 : nn), *Er = a.Er + i * (a.cntE == 1 ? 0 : nn);
  double *e = a.e + i * (a.cntE == 1 ? 0 : n);
  const int64_t g = a.first_global + i;
  if ((a.cntE != 1 && g == 0) || (a.N == 1 && a.first_global == 0)) {   // no evolution row
    for (int k = tid; k < nn; k += NT) { El[k] = 0.0; Er[k] = 0.0; }
    for (int k = tid; k < n; k += NT) e[k] = 0.0;
    return;
  }
  const int64_t iK = (a.cntE == 1) ? 0 : i;
  double *Lm = sm, *X = Lm + nn, *sh = X + n * (2 * n + 1);
  const double *K = a.K + iK * a.sK, *F = a.F + iK * a.sF;
  const double *c = a.c ? a.c + iK * a.sc : nullptr;
  for (int k = tid; k < nn; k += NT) {
    const int r = k / n, cc = k - r * n;
    Lm[r + cc * n] = K[k];
    X[r + cc * n] = F[k];
    X[r + (n + cc) * n] = (r == cc) ? 1.0 : 0.0;
  }
  for (int r = tid; r < n; r += NT) X[r + 2 * n * n] = c ? c[r] : 0.0;
  __syncthreads();
  const bool ok = cta_chol(Lm, n, sh);
  if (tid == 0 && !ok) {
    const int64_t step = (a.cntE == 1) ? (a.first_global == 0 ? 1 : 0) : i;
    report(a.status, step, kBadK);
  }
  cta_fwd(Lm, n, X, n, 2 * n + 1);
  __syncthreads();
  for (int k = tid; k < nn; k += NT) {
    const int r = k / n, cc = k - r * n;
    El[k] = -X[r + cc * n];
    Er[k] = X[r + (n + cc) * n];
  }
  for (int r = tid; r < n; r += NT) e[r] = X[r + 2 * n * n];
}

// Observation blocks: L = M M^T; C = M^{-1} H, y = M^{-1} o (rows >= m_i zero).
__global__ void whiten_obs_kernel(WhitenArgs a) {
  extern __shared__ double sm[];
  const int n = a.n, mx = a.m_max, tid = threadIdx.x, NT = blockDim.x;
  const int64_t i = blockIdx.x;
  const int mi = a.m ? a.m[i] : mx;
  double *C = a.C + i * (int64_t)mx * n;
  double *Lm = sm, *X = Lm + mi * mi, *sh = X + mi * (n + 1);
  const double *L = a.L + i * a.sL, *H = a.H + i * a.sH, *o = a.o + i * a.so;
  for (int k = tid; k < mi * mi; k += NT) {
    const int r = k / mi, cc = k - r * mi;
    Lm[r + cc * mi] = L[r * mx + cc];
  }
  for (int k = tid; k < mi * n; k += NT) {
    const int r = k / n, cc = k - r * n;
    X[r + cc * mi] = H[r * n + cc];
  }
  for (int r = tid; r < mi; r += NT) X[r + n * mi] = o[r];
  __syncthreads();
  const bool ok = cta_chol(Lm, mi, sh);
  if (tid == 0 && !ok) report(a.status, i, kBadL);
  cta_fwd(Lm, mi, X, mi, n + 1);
  __syncthreads();
  for (int k = tid; k < mx * n; k += NT) {
    const int r = k / n, cc = k - r * n;
    C[k] = (r < mi) ? X[r + cc * mi] : 0.0;
  }
  if (!a.constC) {
    for (int r = tid; r < mx; r += NT) a.y[i * mx + r] = (r < mi) ? X[r + n * mi] : 0.0;
  } else {
    for (int k = tid; k < mi * mi; k += NT) {
      const int r = k / mi, cc = k - r * mi;
      a.Mchol[r * mx + cc] = (cc <= r) ? Lm[r + cc * mi] : 0.0;
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

int threads_for(int n) { return n <= 8 ? 32 : n <= 16 ? 64 : n <= 32 ? 128 : 256; }

}  // namespace

size_t factor_smem_bytes(int n, int RC) {
  const int lda1 = (RC + n) | 1, lda2 = (2 * n) | 1, lda3 = (2 * RC + n) | 1;
  const size_t s2 = (size_t)lda2 * (3 * n + 1), s3 = (size_t)lda3 * (n + 1);
  return 8 * ((size_t)lda1 * (2 * n + 1) + (s2 > s3 ? s2 : s3) + (size_t)n * (n + 1) + (size_t)n * n + 8);
}

size_t backward_smem_bytes(int n) { return 8 * (9 * (size_t)n * n + 3 * (size_t)n); }

cudaError_t launch_factor_level(const FactorLevelArgs &a, cudaStream_t s) {
  const size_t smem = factor_smem_bytes(a.n, a.in.RC);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(factor_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(backward_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const int64_t grid = a.K >= 2 ? a.K / 2 : 1;
  factor_level_kernel<<<(unsigned)grid, threads_for(a.n), smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_backward_level(const BackwardLevelArgs &a, cudaStream_t s) {
  const int64_t grid = (a.K + 1) / 2;
  backward_level_kernel<<<(unsigned)grid, threads_for(a.n), backward_smem_bytes(a.n), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_whiten(const WhitenArgs &a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(whiten_evo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(whiten_obs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const int n = a.n, mx = a.m_max;
  const size_t se = 8 * ((size_t)n * n + (size_t)n * (2 * n + 1) + 8);
  whiten_evo_kernel<<<(unsigned)a.cntE, threads_for(n), se, s>>>(a);
  if (mx > 0) {
    const size_t so = 8 * ((size_t)mx * mx + (size_t)mx * (n + 1) + 8);
    whiten_obs_kernel<<<(unsigned)a.cntC, threads_for(n > mx ? n : mx), so, s>>>(a);
    if (a.constC) {
      const int T = 256;
      whiten_y_kernel<<<(unsigned)((a.N + T - 1) / T), T, 8 * (size_t)mx * mx, s>>>(a);
    }
  }
  return cudaGetLastError();
}

}  // namespace ks
