"""Seeded synthetic inputs for the Odd-Even Kalman smoother (no method arithmetic).

This module only *draws* problems: model blocks, a simulated trajectory and its
noisy observations.  It holds none of the smoother's arithmetic (no whitening,
no QR, no SelInv), so it may serve both the oracle tests and the CUDA path
(task rule: "only the seeded input generators serve both").

Model (Eq. (1)-(2), with the paper's evolution H_i = I):
    x_i = F_i x_{i-1} + c_i + w_i,   w_i ~ N(0, K_i)      (i >= 1)
    o_i = G_i x_i + v_i,             v_i ~ N(0, L_i)      (m_i >= 0 rows)
The ABI / BASELINE.json call the observation matrix ``H`` (paper G).

Configs c1..c5 are BASELINE.json ``configs[0..4]``; readings of their
under-specified parts are DESIGN.md §3:
  * N(0, s) perturbations use s as a standard deviation (c2: sigma = 0.01),
  * "random orthogonal" is drawn i.i.d. per step (Haar, QR of a Gaussian with
    diag(R) > 0), config 1 rotations use theta_i ~ U[0, 2 pi),
  * Wishart(nu = 2n)/nu, redrawn until cond <= bound,
  * x_0 ~ N(0, I) everywhere; c_i = 0 everywhere,
  * draw order: model arrays -> x_0 -> w -> v, numpy PCG64 default_rng(seed).

Arrays with a leading dimension of 1 are *constant* over steps and are passed
to the C ABI with stride 0.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = ["Problem", "CONFIGS", "make", "paper_problem", "random_problem", "general_problem"]


@dataclass
class Problem:
    name: str
    N: int                      # number of states (paper k+1)
    n: int                      # state dimension
    m_max: int                  # max observation dimension
    m: np.ndarray               # int32 [N]
    F: np.ndarray               # [N|1, n, n]       evolution (F of step 0 ignored)
    H: np.ndarray               # [N|1, m_max, n]   observation matrix (paper G)
    K: np.ndarray               # [N|1, n, n]       evolution-noise covariance
    L: np.ndarray               # [N|1, m_max, m_max] observation-noise covariance
    o: np.ndarray               # [N, m_max]        observations (rows >= m_i are 0)
    c: Optional[np.ndarray] = None      # [N|1, n] forcing, None = 0
    x_true: Optional[np.ndarray] = None  # [N, n] simulated trajectory
    seed: int = 0
    meta: dict = field(default_factory=dict)
    # general model (ks_problem Hev / l / nstate): evolution
    # H_i x_i = F_i x_{i-1} + c_i + w_i with H_i l_i x n_i; None = uniform
    Hev: Optional[np.ndarray] = None    # [N|1, n, n]   (rows >= l_i, cols >= n_i are 0)
    l: Optional[np.ndarray] = None      # int32 [N]     evolution rows l_i
    nstate: Optional[np.ndarray] = None  # int32 [N]    state dimensions n_i

    def stride(self, name: str) -> int:
        """Per-step stride in doubles (0 = the same block every step)."""
        a = getattr(self, name)
        if a is None:
            return 0
        return 0 if a.shape[0] == 1 else int(np.prod(a.shape[1:]))

    def slice(self, lo: int, hi: int) -> "Problem":
        """Steps [lo, hi) as a self-contained problem (the evolution row of
        step lo stays attached to it: a shard's first step keeps F/K/c)."""
        def s(a):
            if a is None:
                return None
            return a if a.shape[0] == 1 else np.ascontiguousarray(a[lo:hi])
        v = lambda a: None if a is None else np.ascontiguousarray(a[lo:hi])
        return Problem(self.name + f"[{lo}:{hi}]", hi - lo, self.n, self.m_max,
                       np.ascontiguousarray(self.m[lo:hi]), s(self.F), s(self.H),
                       s(self.K), s(self.L), np.ascontiguousarray(self.o[lo:hi]),
                       s(self.c), None if self.x_true is None else self.x_true[lo:hi],
                       self.seed, dict(self.meta), s(self.Hev), v(self.l), v(self.nstate))

    @staticmethod
    def concat(parts: list, name: str = "batch") -> "Problem":
        """Independent problems of one structure (same N, n, m_max) laid end
        to end, the layout of a batched context (ks_problem.batch = len(parts)):
        array plumbing only; a constant block shared by every part stays
        constant."""
        p0 = parts[0]
        assert all(q.N == p0.N and q.n == p0.n and q.m_max == p0.m_max for q in parts)

        def cat(attr):
            arrs = [getattr(q, attr) for q in parts]
            if arrs[0] is None:
                assert all(a is None for a in arrs)
                return None
            if all(a.shape[0] == 1 for a in arrs) and all(np.array_equal(a, arrs[0]) for a in arrs):
                return arrs[0]
            return np.ascontiguousarray(np.concatenate([np.broadcast_to(a, (q.N,) + a.shape[1:])
                                                        for a, q in zip(arrs, parts)]))
        xt = None if any(q.x_true is None for q in parts) else np.concatenate([q.x_true for q in parts])
        vec = lambda attr: None if getattr(p0, attr) is None else np.concatenate([getattr(q, attr) for q in parts])
        return Problem(name, p0.N * len(parts), p0.n, p0.m_max, np.concatenate([q.m for q in parts]),
                       cat("F"), cat("H"), cat("K"), cat("L"), cat("o"), cat("c"), xt, p0.seed,
                       {"batch": len(parts)}, cat("Hev"), vec("l"), vec("nstate"))

    def nbytes_inputs(self) -> int:
        tot = self.m.nbytes
        for a in (self.F, self.H, self.K, self.L, self.o, self.c):
            if a is not None:
                tot += a.nbytes
        return tot


# ----------------------------------------------------------------------------
# primitive draws
# ----------------------------------------------------------------------------

def haar_orthogonal(rng, count: int, n: int) -> np.ndarray:
    """[count, n, n] Haar-distributed orthogonal matrices (QR of a Gaussian,
    column signs fixed so diag(R) > 0)."""
    g = rng.standard_normal((count, n, n))
    q, r = np.linalg.qr(g)
    d = np.sign(np.diagonal(r, axis1=1, axis2=2))
    d[d == 0] = 1.0
    return q * d[:, None, :]


def wishart_bounded(rng, count: int, n: int, cond_max: float, nu: Optional[int] = None,
                    chunk: int = 4096) -> np.ndarray:
    """[count, n, n] Wishart(nu)/nu SPD matrices, nu = 2n, redrawn until
    cond <= cond_max (reading R17)."""
    nu = 2 * n if nu is None else nu
    out = np.empty((count, n, n))
    for lo in range(0, count, chunk):
        hi = min(count, lo + chunk)
        x = rng.standard_normal((hi - lo, n, nu))
        s = x @ np.swapaxes(x, 1, 2) / nu
        while True:
            ev = np.linalg.eigvalsh(s)
            bad = np.nonzero(ev[:, -1] > cond_max * ev[:, 0])[0]
            if bad.size == 0:
                break
            x = rng.standard_normal((bad.size, n, nu))
            s[bad] = x @ np.swapaxes(x, 1, 2) / nu
        out[lo:hi] = s
    return out


def _chol_batch(a: np.ndarray) -> np.ndarray:
    return np.linalg.cholesky(a)


def simulate(rng, F, K, H, L, m, noise_free=False, c=None):
    """Draw x_0, then the evolution noise w, then the observation noise v
    (reading R22), and simulate the trajectory sequentially."""
    N = m.shape[0]
    n = F.shape[-1]
    m_max = H.shape[1]
    x0 = rng.standard_normal(n)
    z_w = rng.standard_normal((N, n))
    z_v = rng.standard_normal((N, m_max))
    if noise_free:
        z_w[:] = 0.0
        z_v[:] = 0.0
    cK = _chol_batch(K)
    w = np.einsum("sij,sj->si", cK, z_w) if K.shape[0] == N else z_w @ cK[0].T
    if c is not None:
        w = w + (c if c.shape[0] == N else np.broadcast_to(c, (N, n)))
    x = np.empty((N, n))
    x[0] = x0
    if F.shape[0] == 1:
        F0 = F[0]
        for i in range(1, N):
            x[i] = F0 @ x[i - 1] + w[i]
    else:
        for i in range(1, N):
            x[i] = F[i] @ x[i - 1] + w[i]
    if m_max > 0:
        cL = _chol_batch(L)
        v = np.einsum("sij,sj->si", cL, z_v) if L.shape[0] == N else z_v @ cL[0].T
        Hx = np.einsum("sij,sj->si", H, x) if H.shape[0] == N else x @ H[0].T
        o = Hx + v
        rows = np.arange(m_max)[None, :]
        o[rows >= m[:, None]] = 0.0
    else:
        o = np.zeros((N, 0))
    return x, np.ascontiguousarray(o)


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------

CONFIGS = {
    "c1": dict(N=1000, n=2, m=2, seed=0),
    "c2": dict(N=100_000, n=6, m=6, seed=1),
    "c3": dict(N=100_000, n=6, m=6, seed=2),
    "c4": dict(N=20_000, n=48, m=48, seed=3),
    "c5": dict(N=1 << 22, n=6, m=3, seed=4),
}


def _c1(N, seed, noise_free):
    rng = np.random.default_rng(seed)
    n = m = 2
    th = rng.uniform(0.0, 2.0 * np.pi, N)
    F = np.empty((N, 2, 2))
    F[:, 0, 0] = np.cos(th); F[:, 0, 1] = -np.sin(th)
    F[:, 1, 0] = np.sin(th); F[:, 1, 1] = np.cos(th)
    F *= 0.99
    H = rng.standard_normal((N, m, n))
    K = np.eye(n)[None].copy()
    L = np.eye(m)[None].copy()
    mm = np.full(N, m, np.int32)
    x, o = simulate(rng, F, K, H, L, mm, noise_free=noise_free)
    return Problem("c1", N, n, m, mm, F, H, K, L, o, None, x, seed)


def _c2(N, seed, noise_free):
    rng = np.random.default_rng(seed)
    n = m = 6
    F = 0.995 * haar_orthogonal(rng, N, n) + 0.01 * rng.standard_normal((N, n, n))
    H = rng.standard_normal((N, m, n)) * np.sqrt(1.0 / m)
    K = wishart_bounded(rng, N, n, 1e3)
    L = wishart_bounded(rng, N, m, 1e3)
    mm = np.full(N, m, np.int32)
    x, o = simulate(rng, F, K, H, L, mm, noise_free=noise_free)
    return Problem("c2", N, n, m, mm, F, H, K, L, o, None, x, seed)


def _c3(N, seed, noise_free):
    rng = np.random.default_rng(seed)
    n, m_max = 6, 6
    mm = rng.choice(np.array([0, 2, 6], np.int32), size=N).astype(np.int32)
    H = rng.standard_normal((N, m_max, n))
    H[np.arange(m_max)[None, :] >= mm[:, None]] = 0.0
    A = rng.standard_normal((n, n))
    rho = np.max(np.abs(np.linalg.eigvals(A)))
    F = (0.98 * A / rho)[None].copy()
    K = np.eye(n)[None].copy()
    L = np.eye(m_max)[None].copy()
    x, o = simulate(rng, F, K, H, L, mm, noise_free=noise_free)
    return Problem("c3", N, n, m_max, mm, F, H, K, L, o, None, x, seed)


def _c4(N, seed, noise_free):
    rng = np.random.default_rng(seed)
    n = m = 48
    F = 0.999 * haar_orthogonal(rng, N, n)
    H = rng.standard_normal((N, m, n)) * np.sqrt(1.0 / m)
    K = wishart_bounded(rng, N, n, 1e2)
    L = wishart_bounded(rng, N, m, 1e2)
    mm = np.full(N, m, np.int32)
    x, o = simulate(rng, F, K, H, L, mm, noise_free=noise_free)
    return Problem("c4", N, n, m, mm, F, H, K, L, o, None, x, seed)


def cv_model(dt=0.01, q=1.0, sigma=0.1):
    """Constant-velocity 3-D model of config 5: state [pos(3), vel(3)]."""
    I3 = np.eye(3)
    F = np.block([[I3, dt * I3], [np.zeros((3, 3)), I3]])
    H = np.hstack([I3, np.zeros((3, 3))])
    K = q * np.block([[dt ** 3 / 3 * I3, dt ** 2 / 2 * I3], [dt ** 2 / 2 * I3, dt * I3]])
    L = sigma ** 2 * I3
    return F, H, K, L


def _c5(N, seed, noise_free):
    rng = np.random.default_rng(seed)
    n, m = 6, 3
    dt = 0.01
    F, H, K, L = cv_model(dt)
    mm = np.full(N, m, np.int32)
    # x_0, w, v in the documented draw order; the trajectory is vectorised
    # per axis (pos_i = pos_{i-1} + dt vel_{i-1} + wp_i, vel_i = vel_{i-1} + wv_i).
    x0 = rng.standard_normal(n)
    z_w = rng.standard_normal((N, n))
    z_v = rng.standard_normal((N, m))
    if noise_free:
        z_w[:] = 0.0
        z_v[:] = 0.0
    w = z_w @ np.linalg.cholesky(K).T
    w[0] = 0.0
    vel = x0[3:][None, :] + np.cumsum(w[:, 3:], axis=0)
    dpos = np.empty((N, 3))
    dpos[0] = 0.0
    dpos[1:] = dt * vel[:-1] + w[1:, :3]
    pos = x0[:3][None, :] + np.cumsum(dpos, axis=0)
    x = np.hstack([pos, vel])
    o = x[:, :3] + z_v @ np.linalg.cholesky(L).T
    return Problem("c5", N, n, m, mm, F[None].copy(), H[None].copy(), K[None].copy(),
                   L[None].copy(), np.ascontiguousarray(o), None, x, seed)


_MAKERS = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4, "c5": _c5}


def make(name: str, N: Optional[int] = None, seed: Optional[int] = None,
         noise_free: bool = False) -> Problem:
    """Config ``name`` (c1..c5) at its full size, or with N overridden (the
    reduced-N parity variants).  Same seed => bitwise-identical arrays."""
    cfg = CONFIGS[name]
    N = cfg["N"] if N is None else int(N)
    seed = cfg["seed"] if seed is None else int(seed)
    p = _MAKERS[name](N, seed, noise_free)
    p.meta["config"] = name
    p.meta["noise_free"] = noise_free
    return p


def paper_problem(N: int, n: int, seed: int = 0) -> Problem:
    """The paper's own benchmark class: fixed random orthonormal
    F and G, evolution H = I, K = L = I, random observations."""
    rng = np.random.default_rng(seed)
    F = haar_orthogonal(rng, 1, n)
    G = haar_orthogonal(rng, 1, n)
    o = rng.standard_normal((N, n))
    return Problem("paper", N, n, n, np.full(N, n, np.int32), F, G,
                   np.eye(n)[None].copy(), np.eye(n)[None].copy(), o, None, None, seed)


def random_problem(rng, N: int, n: int, m=None, m_max: Optional[int] = None,
                   const: bool = False, with_c: bool = True,
                   noise_free: bool = False) -> Problem:
    """Small random full-rank instance for oracle pins and edge cases.

    ``m``: None (m_i ~ U{0..n+1}), an int, or an int array.  Step 0 and the
    last step get m >= n when ``m`` is None so the problem is full rank."""
    if m is None:
        mm = rng.integers(0, n + 2, N).astype(np.int32)
        mm[0] = max(mm[0], n)
    elif np.isscalar(m):
        mm = np.full(N, int(m), np.int32)
    else:
        mm = np.asarray(m, np.int32)
    mx = int(mm.max()) if m_max is None else int(m_max)
    cnt = 1 if const else N
    F = 0.9 * haar_orthogonal(rng, cnt, n) + 0.2 * rng.standard_normal((cnt, n, n))
    H = rng.standard_normal((cnt, mx, n))
    if not const:
        H[np.arange(mx)[None, :] >= mm[:, None]] = 0.0
    K = wishart_bounded(rng, cnt, n, 50.0) if n > 0 else np.zeros((cnt, 0, 0))
    L = wishart_bounded(rng, cnt, mx, 50.0) if mx > 0 else np.zeros((cnt, 0, 0))
    c = 0.3 * rng.standard_normal((cnt, n)) if with_c else None
    x, o = simulate(rng, F, K, H, L, mm, noise_free=noise_free, c=c)
    return Problem("random", N, n, mx, mm, F, H, K, L, o, c, x, 0)


def general_problem(rng, N: int, n: int, m_max: Optional[int] = None, nmin: int = 1,
                    noise_free: bool = False, rect: bool = True) -> Problem:
    """The paper's general linear model: state dimensions
    n_i in [nmin, n], evolution H_i x_i = F_i x_{i-1} + c_i + w_i with a
    rectangular full-rank H_i (l_i x n_i, l_i in [1, n], possibly != n_i),
    F_i l_i x n_{i-1}, K_i l_i x l_i, observations G_i (ABI H) m_i x n_i.
    Stored in the uniform padded arrays of the C ABI (unused rows/columns 0,
    unused K / L diagonal 1).  Full column rank of UA: m_0 >= n_0 and
    l_i + m_i >= n_i with generic (Gaussian) blocks.  The data are consistent
    with a drawn trajectory x_true: c_i = H_i x_i - F_i x_{i-1} (+ w_i),
    o_i = G_i x_i (+ v_i); noise_free gives an exactly consistent system."""
    mx = n if m_max is None else int(m_max)
    assert mx >= nmin, "m_max >= min n_i needed for m_0 >= n_0"
    ns = rng.integers(nmin, n + 1, N).astype(np.int32)
    ns[0] = min(ns[0], mx)
    ls = (rng.integers(np.maximum(1, ns - mx), n + 1) if rect else ns.copy()).astype(np.int32)
    ms = rng.integers(0, mx + 1, N).astype(np.int32)
    ms = np.maximum(ms, np.maximum(ns - ls, 0)).astype(np.int32)
    ms[0] = max(ms[0], ns[0])
    assert ms.max() <= mx, "m_max too small for l_i + m_i >= n_i"
    Hev = np.zeros((N, n, n)); F = np.zeros((N, n, n)); K = np.tile(np.eye(n), (N, 1, 1))
    H = np.zeros((N, mx, n)); L = np.tile(np.eye(mx), (N, 1, 1)); c = np.zeros((N, n))
    o = np.zeros((N, mx)); x = np.zeros((N, n))
    for i in range(N):
        x[i, :ns[i]] = rng.standard_normal(ns[i])
    for i in range(N):
        ni, li, mi = int(ns[i]), int(ls[i]), int(ms[i])
        Hev[i, :li, :ni] = rng.standard_normal((li, ni)) + np.eye(li, ni)
        Ki = wishart_bounded(rng, 1, li, 50.0)[0]
        K[i, :li, :li] = Ki
        if i > 0:
            npv = int(ns[i - 1])
            F[i, :li, :npv] = 0.5 * rng.standard_normal((li, npv))
            w = np.zeros(li) if noise_free else np.linalg.cholesky(Ki) @ rng.standard_normal(li)
            c[i, :li] = Hev[i, :li, :ni] @ x[i, :ni] - F[i, :li, :npv] @ x[i - 1, :npv] + w
        if mi > 0:
            H[i, :mi, :ni] = rng.standard_normal((mi, ni))
            Li = wishart_bounded(rng, 1, mi, 50.0)[0]
            L[i, :mi, :mi] = Li
            v = np.zeros(mi) if noise_free else np.linalg.cholesky(Li) @ rng.standard_normal(mi)
            o[i, :mi] = H[i, :mi, :ni] @ x[i, :ni] + v
    return Problem("general", N, n, mx, ms, F, H, K, L, o, c, x, 0, {"nmin": nmin},
                   Hev, ls, ns)
