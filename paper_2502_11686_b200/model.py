"""Algorithmic cost model of every launch (host logic, no GPU).

Used by bench.py for the roofline line and by DESIGN.md §5.  "Algorithmic"
bytes are what the level-synchronous ABI phases must move through HBM at
minimum (each operand read once, each result written once); flops are the
nominal Householder / triangular-solve / product counts of the block shapes
the kernels process.  P:n = paper line.

Householder QR of a rows x ncols block with npiv pivots:
    sum_{k<npiv} [2 (rows-k)  (norm)  +  4 (rows-k)(ncols-k-1)  (dot + update)]
"""
from __future__ import annotations


def house_flops(rows: int, npiv: int, ncols: int) -> int:
    f = 0
    for k in range(min(npiv, rows)):
        f += 2 * (rows - k) + 4 * (rows - k) * (ncols - k - 1)
    return f


def post_flops(n: int) -> int:
    """T = R^{-1}[R_l R_r], w = R^{-1} z (2n+1 RHS), R^{-1}, P = R^{-1}R^{-T}."""
    return (2 * n + 1) * n * n + (n * n * n) // 3 + (n * n * n) // 3


def entry_doubles(n: int) -> int:
    """Doubles of one level >= 1 entry that are read / written: the C-like
    block is upper triangular (its lower triangle is never stored on the
    small path; the CTA path stores full blocks), y, El, Er, e, |col|."""
    c = n * (n + 1) // 2 if n <= 8 else n * n
    return c + 2 * n * n + 2 * n + 1


def rrec_doubles(n: int) -> int:
    """R record of an eliminated column: T_l, T_r (n x n), w (n), P (packed
    upper n(n+1)/2 on the small path; full n x n on the generic path)."""
    return 2 * n * n + n + (n * (n + 1) // 2 if n <= 8 else n * n)


def level0_column_doubles(n: int, RC: int, strides: dict) -> int:
    """Doubles of one level-0 column read from the whitened arrays (stride-0
    blocks are shared by all columns and cost nothing per column)."""
    d = RC  # y is per step
    if strides.get("C", 1):
        d += RC * n
    if strides.get("E", 1):
        d += 2 * n * n + n
    return d


def factor_level(n: int, RC: int, K: int, level: int, strides: dict | None = None):
    """(bytes, flops, units) of one factor launch over K columns (units = pairs)."""
    pairs, single = K // 2, K % 2
    E, Rr = entry_doubles(n), rrec_doubles(n)
    col = level0_column_doubles(n, RC, strides or {}) if level == 0 else E
    by = pairs * (2 * col + Rr + E) + single * (col + Rr)
    fl_pair = house_flops(RC + n, n, 2 * n + 1) + house_flops(2 * RC, n, n + 1) + \
        house_flops(2 * n, n, 3 * n + 1) + post_flops(n)
    fl_single = house_flops(RC + n, n, 2 * n + 1) + house_flops(2 * n, n, 3 * n + 1) + post_flops(n)
    return 8 * by, pairs * fl_pair + single * fl_single, max(pairs, 1)


def solve_level(n: int, K: int):
    cols = (K + 1) // 2
    return 8 * cols * (2 * n * n + n + 3 * n), cols * 4 * n * n, cols


def selinv_level(n: int, K: int, level: int):
    """Per eliminated column: read T_l, T_r, P and the neighbour blocks S_ll,
    S_rr (each level-(L+1) block is the neighbour of two columns: one block
    per column) and S_lr; write S_tt and, for levels >= 1, the two cross
    blocks the next level down reads."""
    cols = (K + 1) // 2
    p = n * (n + 1) // 2 if n <= 8 else n * n
    d = 2 * n * n + p + n * n + n * n + n * n + (2 * n * n if level >= 1 else 0)
    return 8 * cols * d, cols * 12 * n ** 3, cols


def backward_level(n: int, K: int, level: int):
    """Fused solve + SelInv (ks_solve_selinv) per eliminated column: the R
    record read once (T_l, T_r, w, P), one neighbour state and one neighbour
    covariance block (each level-(L+1) column neighbours two eliminated
    columns), S_lr; write x_t, S_tt and, for levels >= 1, the two cross blocks."""
    cols = (K + 1) // 2
    d = rrec_doubles(n) + n + n * n + n * n + n + n * n + (2 * n * n if level >= 1 else 0)
    return 8 * cols * d, cols * (12 * n ** 3 + 4 * n * n), cols


def whiten(n: int, m: int, N: int, cntE: int, cntC: int, per_step_o: bool = True):
    by = cntE * (2 * n * n + n) + cntE * (3 * n * n + n)            # F,K,c in; El,Er,e out
    by += cntC * (m * n + m * m) + cntC * (m * n)                    # H,L in; C out
    by += N * 2 * m if per_step_o else 0                             # o in; y out
    fl = cntE * (n ** 3 // 3 + n * n * (2 * n + 1)) + cntC * (m ** 3 // 3 + m * m * n) + N * m * m
    return 8 * by, fl


def levels(N: int):
    Ks = []
    K = N
    while True:
        Ks.append(K)
        if K == 1:
            break
        K //= 2
    return Ks


def step_totals(N: int, n: int, m: int, strides: dict, cov: bool = True, fused: bool = True):
    """Whole-step algorithmic (bytes, flops) on one GPU (fused: the backward
    phases as one ks_solve_selinv sweep)."""
    tb = tf = 0
    cntE = 1 if not strides.get("E", 1) else N
    cntC = 1 if not strides.get("C", 1) else N
    b, f = whiten(n, m, N, cntE, cntC)
    tb += b; tf += f
    for L, K in enumerate(levels(N)):
        b, f, _ = factor_level(n, m if L == 0 else n, K, L, strides)
        tb += b; tf += f
        if cov and fused:
            b, f, _ = backward_level(n, K, L)
            tb += b; tf += f
            continue
        b, f, _ = solve_level(n, K)
        tb += b; tf += f
        if cov:
            b, f, _ = selinv_level(n, K, L)
            tb += b; tf += f
    return tb, tf


def launch_cost(family: str, level: int, N: int, n: int, m: int, strides: dict):
    """(bytes, flops, units) of the launch (family, level) on one GPU."""
    K = levels(N)[level]
    if family == "factor":
        return factor_level(n, m if level == 0 else n, K, level, strides)
    if family == "solve":
        return solve_level(n, K)
    if family == "selinv":
        return selinv_level(n, K, level)
    if family == "backward":
        return backward_level(n, K, level)
    if family == "whiten":
        cntE = 1 if not strides.get("E", 1) else N
        cntC = 1 if not strides.get("C", 1) else N
        b, f = whiten(n, m, N, cntE, cntC)
        return b, f, N
    raise ValueError(family)
