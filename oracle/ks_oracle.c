/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU fp64 Paige-Saunders-style sequential QR
 * Kalman smoother with the paper's Algorithm 1 block SelInv.  It exists to
 * check the CUDA path (paper_2502_11686_b200/) and shares no code, header,
 * helper or constant with it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Citations: P:n = line n of the paper text, S:n = SPEC.md line n.
 *
 * Problem (P:141-253 with the paper's evolution matrix H_i = I; the observation
 * matrix, paper G_i, is called H here as in the C ABI):
 *     u_hat = argmin sum_{i>=1} |V_i (u_i - F_i u_{i-1} - c_i)|^2
 *                   + sum_{i>=0} |W_i (o_i - G_i u_i)|^2,
 *     V_i^T V_i = K_i^{-1},  W_i^T W_i = L_i^{-1}
 * whose whitened matrix UA has block rows
 *     [C_i] on column i (C_i = W_i G_i, m_i rows) and
 *     [-B_i  D_i] on columns (i-1, i) (B_i = V_i F_i, D_i = V_i H_i = V_i).
 *
 * Functions and the passage each follows:
 *   oracle_whiten  - Cholesky K = Lam Lam^T, L = M M^T; V = Lam^{-1},
 *                    W = M^{-1} applied by forward substitution (P:220-221,
 *                    P:373; "never forms K^{-1}").
 *   oracle_factor  - sequential Householder QR of UA in natural column order
 *                    (Paige-Saunders): block-bidiagonal R with
 *                    diagonal blocks R_ii, super-diagonal R_{i,i+1}, and
 *                    z = Q^T U b.
 *   oracle_solve   - block back-substitution R u = z.
 *   oracle_selinv  - Algorithm 1 with I = {j+1}; S_jj is
 *                    symmetrised, (S + S^T)/2 (reading R13).
 *   oracle_smooth  - whiten -> factor -> solve -> selinv for a whole problem.
 *
 * Pins (tests/test_oracle.py, all "not gpu"): dense least squares of the
 * stacked UA (numpy lstsq) and dense inverse of (UA)^T UA on random tiny
 * instances; noise-free recovery of the true trajectory; the scalar chain of
 * S:214/S:223/S:268; whitening examples S:60-62; the Toeplitz closed form
 * I/sqrt(4+rho^4); the config-5 DARE steady state (scipy).
 *
 * Storage: all blocks row-major.  Inputs follow the C-ABI convention: each
 * per-step array has its own stride in doubles, stride 0 = same block every
 * step.  Rows of H/o/L beyond m_i are ignored.
 *
 * Return codes: 0 ok, 1 bad argument, 5 K_i or L_i not SPD (bad_kind 1 = K,
 * 2 = L), 6 rank deficient (bad_step = natural column index).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ks_oracle.h"

#define ORA_OK 0
#define ORA_ERR_ARG 1
#define ORA_ERR_NOT_SPD 5
#define ORA_ERR_RANK 6

/* Relative tolerance for a diagonal entry of a final R_ii block, adapting
 * S:158 (the paper assumes full rank): |R_ii[d][d]| <=
 * RANK_TOL * ||stacked block column||_F is reported as rank deficient. */
#define RANK_TOL 1e-12

/* ---------------------------------------------------------------- dense ---- */

/* Lower Cholesky factor of the leading d x d block of A (row-major, lda).
 * Returns 0 on success, -1 if a pivot is <= 0. */
static int chol_lower(const double *A, int lda, int d, double *Lo /* d x d */)
{
    memset(Lo, 0, sizeof(double) * (size_t)d * d);
    for (int j = 0; j < d; ++j) {
        double s = A[(size_t)j * lda + j];
        for (int k = 0; k < j; ++k) s -= Lo[j * d + k] * Lo[j * d + k];
        if (!(s > 0.0)) return -1;
        double ljj = sqrt(s);
        Lo[j * d + j] = ljj;
        for (int i = j + 1; i < d; ++i) {
            double t = A[(size_t)i * lda + j];
            for (int k = 0; k < j; ++k) t -= Lo[i * d + k] * Lo[j * d + k];
            Lo[i * d + j] = t / ljj;
        }
    }
    return 0;
}

/* X = Lo^{-1} Y by forward substitution; Lo d x d lower, Y d x p (ldy), X d x p. */
static void forward_subst(const double *Lo, int d, const double *Y, int ldy, int p, double *X)
{
    for (int i = 0; i < d; ++i)
        for (int c = 0; c < p; ++c) {
            double t = Y[(size_t)i * ldy + c];
            for (int k = 0; k < i; ++k) t -= Lo[i * d + k] * X[(size_t)k * p + c];
            X[(size_t)i * p + c] = t / Lo[i * d + i];
        }
}

/* X = R^{-1} Y by back substitution; R n x n upper (ldr), Y n x p, X n x p. */
static void back_subst(const double *R, int ldr, int n, const double *Y, int p, double *X)
{
    for (int i = n - 1; i >= 0; --i)
        for (int c = 0; c < p; ++c) {
            double t = Y[(size_t)i * p + c];
            for (int k = i + 1; k < n; ++k) t -= R[(size_t)i * ldr + k] * X[(size_t)k * p + c];
            X[(size_t)i * p + c] = t / R[(size_t)i * ldr + i];
        }
}

/* Householder QR, in place, of the rows x cols row-major matrix A: the first
 * npiv columns are triangularised and the same reflectors are applied to the
 * remaining columns (the "apply Q^T to the neighbouring blocks and the RHS"
 * of P:424-455).  Reflector k: v = x - alpha e_1, alpha = -sign(x_1)|x|,
 * H = I - 2 v v^T / (v^T v); a zero column is skipped (H = I). */
static void house_qr(double *A, int rows, int cols, int npiv)
{
    double *v = (double *)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
    for (int k = 0; k < npiv && k < rows; ++k) {
        double nrm2 = 0.0;
        for (int i = k; i < rows; ++i) nrm2 += A[(size_t)i * cols + k] * A[(size_t)i * cols + k];
        if (nrm2 == 0.0) continue;
        double nrm = sqrt(nrm2);
        double x1 = A[(size_t)k * cols + k];
        double alpha = (x1 > 0.0) ? -nrm : nrm;
        double vtv = 0.0;
        for (int i = k; i < rows; ++i) {
            v[i] = A[(size_t)i * cols + k];
            if (i == k) v[i] -= alpha;
            vtv += v[i] * v[i];
        }
        for (int j = k + 1; j < cols; ++j) {
            double s = 0.0;
            for (int i = k; i < rows; ++i) s += v[i] * A[(size_t)i * cols + j];
            s = 2.0 * s / vtv;
            for (int i = k; i < rows; ++i) A[(size_t)i * cols + j] -= s * v[i];
        }
        A[(size_t)k * cols + k] = alpha;
        for (int i = k + 1; i < rows; ++i) A[(size_t)i * cols + k] = 0.0;
    }
    free(v);
}

/* ------------------------------------------------------------ whitening ---- */

/* Whiten one step i.  Outputs (all row-major, dense):
 *   C [m_i x n] = M^{-1} H_i,  y [m_i] = M^{-1} o_i         (L_i = M M^T)
 *   for i >= 1 (has_evo): B [n x n] = Lam^{-1} F_i, D [n x n] = Lam^{-1},
 *                         e [n] = Lam^{-1} c_i               (K_i = Lam Lam^T)
 * Returns 0, or 1 (K not SPD) / 2 (L not SPD). */
static int whiten_step(int n, int mi, int m_max, int has_evo,
                       const double *F, const double *H, const double *c, const double *o,
                       const double *K, const double *L,
                       double *C, double *y, double *B, double *D, double *e,
                       double *work /* >= max(n,m_max)^2 */)
{
    if (mi > 0) {
        if (chol_lower(L, m_max, mi, work) != 0) return 2;
        forward_subst(work, mi, H, n, n, C);
        forward_subst(work, mi, o, 1, 1, y);
    }
    if (has_evo) {
        if (chol_lower(K, n, n, work) != 0) return 1;
        forward_subst(work, n, F, n, n, B);
        double *I = (double *)calloc((size_t)n * n, sizeof(double));
        for (int d = 0; d < n; ++d) I[d * n + d] = 1.0;
        forward_subst(work, n, I, n, n, D);
        free(I);
        if (c) {
            forward_subst(work, n, c, 1, 1, e);
        } else {
            for (int d = 0; d < n; ++d) e[d] = 0.0;
        }
    }
    return 0;
}

int oracle_whiten(int64_t N, int n, int m_max, const int32_t *m,
                  const double *F, int64_t sF, const double *H, int64_t sH,
                  const double *c, int64_t sc, const double *o, int64_t so,
                  const double *K, int64_t sK, const double *L, int64_t sL,
                  double *C, double *y, double *B, double *D, double *e,
                  int64_t *bad_step, int *bad_kind)
{
    if (N < 1 || n < 1 || m_max < 0) return ORA_ERR_ARG;
    int w = n > m_max ? n : m_max;
    double *work = (double *)malloc(sizeof(double) * (size_t)w * w + 8);
    for (int64_t i = 0; i < N; ++i) {
        int mi = m ? m[i] : m_max;
        if (mi < 0 || mi > m_max) { free(work); return ORA_ERR_ARG; }
        int r = whiten_step(n, mi, m_max, i > 0, F + i * sF, H + i * sH, c ? c + i * sc : NULL,
                            o + i * so, K + i * sK, L + i * sL,
                            C + i * (int64_t)m_max * n, y + i * (int64_t)m_max,
                            B + i * (int64_t)n * n, D + i * (int64_t)n * n, e + i * (int64_t)n, work);
        if (i == 0) { /* step 0 has no evolution row */
            memset(B, 0, sizeof(double) * (size_t)n * n);
            memset(D, 0, sizeof(double) * (size_t)n * n);
            memset(e, 0, sizeof(double) * (size_t)n);
        }
        /* rows beyond m_i are zero in the dense outputs */
        for (int rr = mi; rr < m_max; ++rr) {
            y[i * m_max + rr] = 0.0;
            for (int cc = 0; cc < n; ++cc) C[(i * m_max + rr) * n + cc] = 0.0;
        }
        if (r) {
            if (bad_step) *bad_step = i;
            if (bad_kind) *bad_kind = r;
            free(work);
            return ORA_ERR_NOT_SPD;
        }
    }
    free(work);
    return ORA_OK;
}

/* ----------------------------------------------------------- factor -------- */

/* State carried between steps: the compressed block (Chat, yhat) acting on the
 * current column only, r rows (r <= n after compression). */
typedef struct {
    int r;
    double *Ch; /* n x n capacity */
    double *yh; /* n */
} carry_t;

/* Compress rows [top (r1 x n | r1) ; bottom (r2 x n | r2)] to its R factor:
 * QR of the stack, keep min(rows, n) rows ("replace them by their
 * R factor").  Result in cr. */
static void compress(int n, const double *top, const double *ytop, int r1,
                     const double *bot, const double *ybot, int r2, carry_t *cr)
{
    int rows = r1 + r2, cols = n + 1;
    double *A = (double *)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1) * cols);
    for (int i = 0; i < r1; ++i) {
        memcpy(A + (size_t)i * cols, top + (size_t)i * n, sizeof(double) * n);
        A[(size_t)i * cols + n] = ytop[i];
    }
    for (int i = 0; i < r2; ++i) {
        memcpy(A + (size_t)(r1 + i) * cols, bot + (size_t)i * n, sizeof(double) * n);
        A[(size_t)(r1 + i) * cols + n] = ybot[i];
    }
    house_qr(A, rows, cols, n);
    int keep = rows < n ? rows : n;
    cr->r = keep;
    for (int i = 0; i < keep; ++i) {
        memcpy(cr->Ch + (size_t)i * n, A + (size_t)i * cols, sizeof(double) * n);
        cr->yh[i] = A[(size_t)i * cols + n];
    }
    free(A);
}

/* One forward step of the sequential QR (the k -> 1 degenerate case
 * of the odd-even elimination P:424-455):
 *   QR of [Chat ; -B_{i+1}] (r + n rows) applied to [0 ; D_{i+1}] and
 *   [yhat ; e_{i+1}]: top n rows -> R_ii, R_{i,i+1}, z_i; the bottom r rows
 *   (Dbar, ybar) act on column i+1 only and are compressed with C_{i+1}. */
static int forward_step(int n, carry_t *cr, const double *B1, const double *D1, const double *e1,
                        const double *C1, const double *y1, int m1,
                        double *Rii, double *Rii1, double *zi)
{
    int r = cr->r, rows = r + n, cols = 2 * n + 1;
    double *A = (double *)calloc((size_t)rows * cols, sizeof(double));
    double fro2 = 0.0;
    for (int i = 0; i < r; ++i) {
        for (int cc = 0; cc < n; ++cc) A[(size_t)i * cols + cc] = cr->Ch[(size_t)i * n + cc];
        A[(size_t)i * cols + 2 * n] = cr->yh[i];
    }
    for (int i = 0; i < n; ++i) {
        for (int cc = 0; cc < n; ++cc) {
            A[(size_t)(r + i) * cols + cc] = -B1[i * n + cc];
            A[(size_t)(r + i) * cols + n + cc] = D1[i * n + cc];
        }
        A[(size_t)(r + i) * cols + 2 * n] = e1[i];
    }
    for (int i = 0; i < rows; ++i)
        for (int cc = 0; cc < n; ++cc) fro2 += A[(size_t)i * cols + cc] * A[(size_t)i * cols + cc];
    house_qr(A, rows, cols, n);
    int bad = 0;
    for (int i = 0; i < n; ++i) {
        for (int cc = 0; cc < n; ++cc) {
            Rii[i * n + cc] = A[(size_t)i * cols + cc];
            Rii1[i * n + cc] = A[(size_t)i * cols + n + cc];
        }
        zi[i] = A[(size_t)i * cols + 2 * n];
        if (!(fabs(Rii[i * n + i]) > RANK_TOL * sqrt(fro2))) bad = 1;
    }
    /* leftover rows n .. rows-1: [0 | Dbar | ybar] */
    double *Db = (double *)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1) * n);
    double *yb = (double *)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
    for (int i = 0; i < r; ++i) {
        for (int cc = 0; cc < n; ++cc) Db[(size_t)i * n + cc] = A[(size_t)(n + i) * cols + n + cc];
        yb[i] = A[(size_t)(n + i) * cols + 2 * n];
    }
    compress(n, Db, yb, r, C1, y1, m1, cr);
    free(Db); free(yb); free(A);
    return bad;
}

/* Last column: R_{N-1,N-1} = QR of the carry; needs n rows and full rank. */
static int last_step(int n, carry_t *cr, double *R, double *z)
{
    if (cr->r < n) return 1;
    /* the carry is already a QR-compressed (upper triangular) block */
    double fro2 = 0.0;
    for (int i = 0; i < n; ++i) {
        for (int cc = 0; cc < n; ++cc) {
            R[i * n + cc] = cr->Ch[(size_t)i * n + cc];
            fro2 += R[i * n + cc] * R[i * n + cc];
        }
        z[i] = cr->yh[i];
    }
    for (int i = 0; i < n; ++i)
        if (!(fabs(R[i * n + i]) > RANK_TOL * sqrt(fro2))) return 1;
    return 0;
}

int oracle_factor(int64_t N, int n, int m_max, const int32_t *m,
                  const double *C, const double *y, const double *B, const double *D,
                  const double *e, double *Rd, double *Ro, double *z, int64_t *bad_step)
{
    if (N < 1 || n < 1 || m_max < 0) return ORA_ERR_ARG;
    carry_t cr;
    cr.Ch = (double *)malloc(sizeof(double) * (size_t)n * n);
    cr.yh = (double *)malloc(sizeof(double) * (size_t)n);
    int m0 = m ? m[0] : m_max;
    compress(n, C, y, m0, NULL, NULL, 0, &cr);
    int rc = ORA_OK;
    for (int64_t i = 0; i + 1 < N; ++i) {
        int m1 = m ? m[i + 1] : m_max;
        int bad = forward_step(n, &cr, B + (i + 1) * n * n, D + (i + 1) * n * n, e + (i + 1) * n,
                               C + (i + 1) * m_max * n, y + (i + 1) * m_max, m1,
                               Rd + i * n * n, Ro + i * n * n, z + i * n);
        if (bad && rc == ORA_OK) { rc = ORA_ERR_RANK; if (bad_step) *bad_step = i; }
    }
    if (last_step(n, &cr, Rd + (N - 1) * n * n, z + (N - 1) * n) && rc == ORA_OK) {
        rc = ORA_ERR_RANK;
        if (bad_step) *bad_step = N - 1;
    }
    if (N >= 1) memset(Ro + (N - 1) * n * n, 0, sizeof(double) * (size_t)n * n);
    free(cr.Ch); free(cr.yh);
    return rc;
}

/* -------------------------------------------------------------- solve ------ */

int oracle_solve(int64_t N, int n, const double *Rd, const double *Ro, const double *z, double *x)
{
    if (N < 1 || n < 1) return ORA_ERR_ARG;
    double *t = (double *)malloc(sizeof(double) * (size_t)n);
    /* u_{N-1} = R^{-1} z_{N-1};  u_i = R_ii^{-1}(z_i - R_{i,i+1} u_{i+1}) */
    back_subst(Rd + (N - 1) * n * n, n, n, z + (N - 1) * n, 1, x + (N - 1) * n);
    for (int64_t i = N - 2; i >= 0; --i) {
        for (int a = 0; a < n; ++a) {
            double s = z[i * n + a];
            for (int b = 0; b < n; ++b) s -= Ro[i * n * n + a * n + b] * x[(i + 1) * n + b];
            t[a] = s;
        }
        back_subst(Rd + i * n * n, n, n, t, 1, x + i * n);
    }
    free(t);
    return ORA_OK;
}

/* ------------------------------------------------------------- selinv ------ */

/* P = R^{-1} R^{-T} for an upper-triangular R (n x n). */
static void rinv_rinvT(const double *R, int n, double *P, double *work /* 2 n^2 */)
{
    double *I = work, *Ri = work + n * n;
    memset(I, 0, sizeof(double) * (size_t)n * n);
    for (int d = 0; d < n; ++d) I[d * n + d] = 1.0;
    back_subst(R, n, n, I, n, Ri);           /* Ri = R^{-1} */
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) s += Ri[a * n + k] * Ri[b * n + k];
            P[a * n + b] = s;
        }
}

int oracle_selinv(int64_t N, int n, const double *Rd, const double *Ro, double *S, double *Scross)
{
    if (N < 1 || n < 1) return ORA_ERR_ARG;
    size_t nn = (size_t)n * n;
    double *work = (double *)malloc(sizeof(double) * 2 * nn);
    double *P = (double *)malloc(sizeof(double) * nn);
    double *T = (double *)malloc(sizeof(double) * nn);
    double *Sji = (double *)malloc(sizeof(double) * nn);
    /* S_{N-1,N-1} = R^{-1} R^{-T}  (Alg. 1, first line) */
    rinv_rinvT(Rd + (N - 1) * nn, n, S + (N - 1) * nn, work);
    for (int64_t j = N - 2; j >= 0; --j) {
        const double *Rjj = Rd + j * nn, *Rji = Ro + j * nn;
        const double *Sii = S + (j + 1) * nn;     /* I = {j+1} */
        back_subst(Rjj, n, n, Rji, n, T);          /* T = R_jj^{-1} R_{j,I} */
        for (int a = 0; a < n; ++a)                /* S_{j,I} = -T S_{I,I} */
            for (int b = 0; b < n; ++b) {
                double s = 0.0;
                for (int k = 0; k < n; ++k) s += T[a * n + k] * Sii[k * n + b];
                Sji[a * n + b] = -s;
            }
        rinv_rinvT(Rjj, n, P, work);               /* R_jj^{-1} R_jj^{-T} */
        double *Sjj = S + j * nn;                  /* S_jj = P - S_{j,I} T^T */
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                double s = 0.0;
                for (int k = 0; k < n; ++k) s += Sji[a * n + k] * T[b * n + k];
                Sjj[a * n + b] = P[a * n + b] - s;
            }
        for (int a = 0; a < n; ++a)                /* symmetrise (reading R13) */
            for (int b = a + 1; b < n; ++b) {
                double v = 0.5 * (Sjj[a * n + b] + Sjj[b * n + a]);
                Sjj[a * n + b] = v;
                Sjj[b * n + a] = v;
            }
        if (Scross) memcpy(Scross + j * nn, Sji, sizeof(double) * nn);
    }
    free(work); free(P); free(T); free(Sji);
    return ORA_OK;
}

/* ------------------------------------------------------------- smooth ------ */

int oracle_smooth(int64_t N, int n, int m_max, const int32_t *m,
                  const double *F, int64_t sF, const double *H, int64_t sH,
                  const double *c, int64_t sc, const double *o, int64_t so,
                  const double *K, int64_t sK, const double *L, int64_t sL,
                  double *x, double *S, int64_t *bad_step, int *bad_kind)
{
    if (N < 1 || n < 1 || m_max < 0 || !x) return ORA_ERR_ARG;
    size_t nn = (size_t)n * n;
    int w = n > m_max ? n : m_max;
    double *Rd = (double *)malloc(sizeof(double) * nn * (size_t)N);
    double *Ro = (double *)malloc(sizeof(double) * nn * (size_t)N);
    double *z = (double *)malloc(sizeof(double) * (size_t)n * N);
    double *Cw = (double *)calloc((size_t)(m_max > 0 ? m_max : 1) * n, sizeof(double));
    double *yw = (double *)calloc((size_t)(m_max > 0 ? m_max : 1), sizeof(double));
    double *Bw = (double *)malloc(sizeof(double) * nn);
    double *Dw = (double *)malloc(sizeof(double) * nn);
    double *ew = (double *)malloc(sizeof(double) * n);
    double *work = (double *)malloc(sizeof(double) * (size_t)w * w + 8);
    carry_t cr;
    cr.Ch = (double *)malloc(sizeof(double) * nn);
    cr.yh = (double *)malloc(sizeof(double) * n);
    int rc = ORA_OK;
    if (bad_kind) *bad_kind = 0;
    for (int64_t i = 0; i < N && rc == ORA_OK; ++i) {
        int mi = m ? m[i] : m_max;
        if (mi < 0 || mi > m_max) { rc = ORA_ERR_ARG; break; }
        int r = whiten_step(n, mi, m_max, i > 0, F + i * sF, H + i * sH, c ? c + i * sc : NULL,
                            o + i * so, K + i * sK, L + i * sL, Cw, yw, Bw, Dw, ew, work);
        if (r) { rc = ORA_ERR_NOT_SPD; if (bad_step) *bad_step = i; if (bad_kind) *bad_kind = r; break; }
        if (i == 0) {
            compress(n, Cw, yw, mi, NULL, NULL, 0, &cr);
        } else if (forward_step(n, &cr, Bw, Dw, ew, Cw, yw, mi, Rd + (i - 1) * nn,
                                Ro + (i - 1) * nn, z + (i - 1) * n)) {
            rc = ORA_ERR_RANK;
            if (bad_step) *bad_step = i - 1;
        }
    }
    if (rc == ORA_OK && last_step(n, &cr, Rd + (N - 1) * nn, z + (N - 1) * n)) {
        rc = ORA_ERR_RANK;
        if (bad_step) *bad_step = N - 1;
    }
    if (rc == ORA_OK) {
        memset(Ro + (N - 1) * nn, 0, sizeof(double) * nn);
        oracle_solve(N, n, Rd, Ro, z, x);
        if (S) oracle_selinv(N, n, Rd, Ro, S, NULL);
    }
    free(Rd); free(Ro); free(z); free(Cw); free(yw); free(Bw); free(Dw); free(ew);
    free(work); free(cr.Ch); free(cr.yh);
    return rc;
}
