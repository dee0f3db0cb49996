"""ORACLE -- TEST INFRASTRUCTURE ONLY.

The paper's general linear model: state
dimensions n_i that change from step to step and a rectangular evolution
matrix H_i (l_i x n_i, "we do not require this (and do not require it to be
square)"):

    H_i u_i = F_i u_{i-1} + c_i + eps_i,  cov(eps_i) = K_i   (l_i rows, i >= 1)
    o_i     = G_i u_i + delta_i,          cov(delta_i) = L_i (m_i rows)

solved as the generalized least-squares problem of Eq. (4)-(6)
by the sequential Paige-Saunders QR and the covariance blocks by
Algorithm 1, written out step by step in numpy with blocks of
their own sizes.  Library primitives only per block (np.linalg.cholesky,
np.linalg.qr, scipy solve_triangular); no blocking, fusion or reordering.

This is NOT the CUDA path's method for these problems (that one embeds them
into a uniform dimension with pinned padding components), so agreement is
not self-agreement.  Only tests/ may import it.  Pinned in
tests/test_oracle.py (dense lstsq / dense inverse of the stacked general
matrix, noise-free recovery, agreement with the C oracle on uniform problems).

Arrays follow the C-ABI padded layout of generators.Problem (Hev, l, nstate
optional: None = identity, l_i = n_i, n_i = n).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

RANK_TOL = 1e-12   # SURVEY §8(b); the paper assumes full rank


class GeneralOracleError(RuntimeError):
    pass


def _blk(a, i):
    return None if a is None else (a[0] if a.shape[0] == 1 else a[i])


def whiten_general(p):
    """Per step: K_i = Lam Lam^T, L_i = M M^T (leading
    l_i / m_i blocks); V_i = Lam^{-1}, W_i = M^{-1} applied by forward
    substitution.  Returns lists: C_i = W_i G_i (m_i x n_i), y_i = W_i o_i,
    B_i = V_i F_i (l_i x n_{i-1}), D_i = V_i H_i (l_i x n_i), e_i = V_i c_i."""
    N = p.N
    ns = [int(v) for v in (p.nstate if p.nstate is not None else np.full(N, p.n))]
    ls = [int(v) for v in (p.l if p.l is not None else ns)]
    C, y, B, D, e = [], [], [], [], []
    for i in range(N):
        ni, li, mi = ns[i], ls[i], int(p.m[i])
        if mi > 0:
            M = np.linalg.cholesky(_blk(p.L, i)[:mi, :mi])
            C.append(solve_triangular(M, _blk(p.H, i)[:mi, :ni], lower=True))
            y.append(solve_triangular(M, p.o[i, :mi], lower=True))
        else:
            C.append(np.zeros((0, ni)))
            y.append(np.zeros(0))
        if i == 0:   # u_0 has no evolution equation
            B.append(None); D.append(None); e.append(None)
            continue
        Lam = np.linalg.cholesky(_blk(p.K, i)[:li, :li])
        Hi = _blk(p.Hev, i)[:li, :ni] if p.Hev is not None else np.eye(li, ni)
        ci = np.zeros(li) if p.c is None else _blk(p.c, i)[:li]
        B.append(solve_triangular(Lam, _blk(p.F, i)[:li, :ns[i - 1]], lower=True))
        D.append(solve_triangular(Lam, Hi, lower=True))
        e.append(solve_triangular(Lam, ci, lower=True))
    return ns, C, y, B, D, e


def _qr_rows(A, rhs, k):
    """Householder QR of the stack A (rows x k) applied to rhs: (R_top k x k,
    Q^T rhs top k rows, Q^T rhs bottom rows)."""
    Q, R = np.linalg.qr(A, mode="complete")
    QtR = Q.T @ rhs
    return R[:k, :k], QtR[:k], QtR[k:]


def factor_general(ns, C, y, B, D, e):
    """Sequential Paige-Saunders QR of the block-bidiagonal UA:
    for column i, QR of [carry_i; -B_{i+1}] gives R_ii; the same Q^T applied
    to [0; D_{i+1}] and [carry rhs; e_{i+1}] gives R_{i,i+1}, z_i and the
    leftover rows acting on column i+1 only, which join C_{i+1} as the next
    carry.  Returns R_ii, R_{i,i+1}, z_i lists."""
    N = len(ns)
    Rd, Ro, z = [], [], []
    carry, cy = C[0], y[0]
    for i in range(N):
        ni = ns[i]
        colnorm2 = float(np.sum(C[i] ** 2)) + (float(np.sum(D[i] ** 2)) if i > 0 else 0.0)
        if i + 1 < N:
            nx = ns[i + 1]
            A = np.vstack([carry, -B[i + 1]])
            rhs = np.hstack([np.vstack([np.zeros((carry.shape[0], nx)), D[i + 1]]),
                             np.concatenate([cy, e[i + 1]])[:, None]])
            colnorm2 += float(np.sum(B[i + 1] ** 2))
        else:
            A, rhs = carry, cy[:, None]
        if A.shape[0] < ni:
            raise GeneralOracleError(f"rank deficient at step {i} (too few rows)")
        R, top, bot = _qr_rows(A, rhs, ni)
        if np.any(np.abs(np.diag(R)) <= RANK_TOL * np.sqrt(colnorm2)):
            raise GeneralOracleError(f"rank deficient at step {i}")
        Rd.append(R)
        z.append(top[:, -1])
        if i + 1 < N:
            Ro.append(top[:, :-1])
            # leftover rows [Dbar | ybar] act on column i+1 only: new carry
            carry = np.vstack([bot[:, :-1], C[i + 1]])
            cy = np.concatenate([bot[:, -1], y[i + 1]])
            if carry.shape[0] > nx:   # compress to its R factor: the rest is residual
                Rc, tc, _ = _qr_rows(carry, cy[:, None], nx)
                carry, cy = Rc, tc[:, 0]
    return Rd, Ro, z


def solve_general(Rd, Ro, z):
    """Block back-substitution."""
    N = len(Rd)
    u = [None] * N
    u[N - 1] = solve_triangular(Rd[N - 1], z[N - 1])
    for i in range(N - 2, -1, -1):
        u[i] = solve_triangular(Rd[i], z[i] - Ro[i] @ u[i + 1])
    return u


def selinv_general(Rd, Ro):
    """Algorithm 1 with I = {j+1}: S_{N-1} = R^{-1}R^{-T};
    T = R_jj^{-1} R_{j,j+1}, S_{j,j+1} = -T S_{j+1,j+1},
    S_jj = R_jj^{-1} R_jj^{-T} - S_{j,j+1} T^T, symmetrised (reading R13)."""
    N = len(Rd)
    S = [None] * N
    Ri = solve_triangular(Rd[N - 1], np.eye(Rd[N - 1].shape[0]))
    S[N - 1] = Ri @ Ri.T
    for j in range(N - 2, -1, -1):
        Ri = solve_triangular(Rd[j], np.eye(Rd[j].shape[0]))
        T = Ri @ Ro[j]
        Sx = -T @ S[j + 1]
        Sj = Ri @ Ri.T - Sx @ T.T
        S[j] = 0.5 * (Sj + Sj.T)
    return S


def smooth_general(p, cov: bool = True):
    """Padded states [N, n] and covariance blocks [N, n, n] (entries beyond
    n_i are 0)."""
    ns, C, y, B, D, e = whiten_general(p)
    Rd, Ro, z = factor_general(ns, C, y, B, D, e)
    u = solve_general(Rd, Ro, z)
    x = np.zeros((p.N, p.n))
    for i, ui in enumerate(u):
        x[i, :ns[i]] = ui
    if not cov:
        return x
    S = selinv_general(Rd, Ro)
    Sp = np.zeros((p.N, p.n, p.n))
    for i, Si in enumerate(S):
        Sp[i, :ns[i], :ns[i]] = Si
    return x, Sp
