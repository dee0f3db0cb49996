"""Dense test helpers (numpy/scipy library routines only).

Builds the stacked whitened least-squares matrix UA and Ub of PAPER.md
Eq. (6) (block structure P:361-373) *directly from the model*,
with a symmetric inverse square root (eigh) as the whitening factor -- a
different square root from the oracle's and the CUDA path's Cholesky (any
V with V^T V = K^{-1} gives the same estimator).  Nothing here
calls the oracle or the CUDA path.
"""
import numpy as np


def inv_sqrt(A):
    w, Q = np.linalg.eigh(A)
    return (Q / np.sqrt(w)) @ Q.T


def blk(a, i):
    return None if a is None else (a[0] if a.shape[0] == 1 else a[i])


def stacked(p):
    """(UA, Ub) for a generators.Problem (small N only)."""
    N, n = p.N, p.n
    rows_A, rows_b = [], []
    for i in range(N):
        mi = int(p.m[i])
        if i > 0:
            V = inv_sqrt(blk(p.K, i))
            Fi = blk(p.F, i)
            ci = np.zeros(n) if p.c is None else blk(p.c, i)
            r = np.zeros((n, N * n))
            r[:, (i - 1) * n:i * n] = -V @ Fi
            r[:, i * n:(i + 1) * n] = V
            rows_A.append(r)
            rows_b.append(V @ ci)
        if mi > 0:
            W = inv_sqrt(blk(p.L, i)[:mi, :mi])
            G = blk(p.H, i)[:mi]
            r = np.zeros((mi, N * n))
            r[:, i * n:(i + 1) * n] = W @ G
            rows_A.append(r)
            rows_b.append(W @ p.o[i, :mi])
    return np.vstack(rows_A), np.concatenate(rows_b)


def dense_solution(p):
    """States [N,n] by lstsq and covariance blocks [N,n,n] of inv(UA^T UA)."""
    A, b = stacked(p)
    u = np.linalg.lstsq(A, b, rcond=None)[0]
    G = A.T @ A
    S = np.linalg.inv(G)
    n = p.n
    cov = np.stack([S[i * n:(i + 1) * n, i * n:(i + 1) * n] for i in range(p.N)])
    return u.reshape(p.N, n), cov, np.linalg.cond(A), S


def rel_state_err(x, ref):
    """max_i |x_i - ref_i|_inf / |ref_i|_inf (per-step normwise, SURVEY c.5)."""
    num = np.abs(x - ref).max(axis=1)
    den = np.maximum(np.abs(ref).max(axis=1), 1e-300)
    return float((num / den).max())


def rel_cov_err(S, ref):
    num = np.abs(S - ref).reshape(S.shape[0], -1).max(axis=1)
    den = np.maximum(np.abs(ref).reshape(S.shape[0], -1).max(axis=1), 1e-300)
    return float((num / den).max())


def stacked_general(p):
    """(UA, Ub, column offsets) of the paper's general model (P:137-152,
    Eq. (6)): column block i has n_i unknowns; evolution rows
    [-V_i F_i | V_i H_i] (l_i rows), observation rows W_i G_i (m_i rows);
    symmetric inverse square roots (eigh) as whitening."""
    N = p.N
    ns = [int(v) for v in (p.nstate if p.nstate is not None else np.full(N, p.n))]
    ls = [int(v) for v in (p.l if p.l is not None else ns)]
    off = np.concatenate([[0], np.cumsum(ns)])
    T = int(off[-1])
    rows_A, rows_b = [], []
    for i in range(N):
        ni, li, mi = ns[i], ls[i], int(p.m[i])
        if i > 0:
            V = inv_sqrt(blk(p.K, i)[:li, :li])
            Hi = blk(p.Hev, i)[:li, :ni] if p.Hev is not None else np.eye(li, ni)
            Fi = blk(p.F, i)[:li, :ns[i - 1]]
            ci = np.zeros(li) if p.c is None else blk(p.c, i)[:li]
            r = np.zeros((li, T))
            r[:, off[i - 1]:off[i]] = -V @ Fi
            r[:, off[i]:off[i + 1]] = V @ Hi
            rows_A.append(r)
            rows_b.append(V @ ci)
        if mi > 0:
            W = inv_sqrt(blk(p.L, i)[:mi, :mi])
            G = blk(p.H, i)[:mi, :ni]
            r = np.zeros((mi, T))
            r[:, off[i]:off[i + 1]] = W @ G
            rows_A.append(r)
            rows_b.append(W @ p.o[i, :mi])
    return np.vstack(rows_A), np.concatenate(rows_b), off


def dense_solution_general(p):
    """Padded states [N,n] and covariance blocks [N,n,n] (zeros beyond n_i)."""
    A, b, off = stacked_general(p)
    u = np.linalg.lstsq(A, b, rcond=None)[0]
    S = np.linalg.inv(A.T @ A)
    x = np.zeros((p.N, p.n))
    cov = np.zeros((p.N, p.n, p.n))
    for i in range(p.N):
        a, e = off[i], off[i + 1]
        x[i, :e - a] = u[a:e]
        cov[i, :e - a, :e - a] = S[a:e, a:e]
    return x, cov, np.linalg.cond(A)
