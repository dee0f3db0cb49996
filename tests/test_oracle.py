"""Pins of the CPU oracle (oracle/) against things other than itself.

Every oracle function is checked here, without a GPU:
  whiten  - SPEC worked examples and V^T V K = I;
  factor  - Gram preservation R^T R = (UA)^T UA of the dense stacked matrix;
  solve   - scalar chain, dense lstsq (numpy), noise-free recovery;
  selinv  - SPEC bidiagonal example, dense inv(R^T R), dense
            inv((UA)^T UA), Toeplitz closed form, config-5 DARE steady state;
  smooth  - all of the above end to end + error paths.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from paper_2502_11686_b200 import generators as gen
from tests.dense import dense_solution, rel_cov_err, rel_state_err, stacked

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def scalar_problem(N, F, G, K, L, o):
    o = np.asarray(o, float).reshape(N, 1)
    return gen.Problem("scalar", N, 1, 1, np.ones(N, np.int32), np.full((1, 1, 1), F),
                       np.full((1, 1, 1), G), np.full((1, 1, 1), K), np.full((1, 1, 1), L), o)


# ----------------------------------------------------------------- whiten ---

def test_whiten_worked_examples():
    g = gold("whitening.json")
    for case in g["cases"]:
        K = np.array(case["K"]); F = np.array(case["F"]); n = K.shape[0]
        p = gen.Problem("w", 2, n, n, np.full(2, n, np.int32), F[None], np.eye(n)[None],
                        K[None], np.eye(n)[None], np.zeros((2, n)))
        w = oracle.whiten(p)
        np.testing.assert_allclose(w["B"][1], np.array(case["B"]), rtol=0, atol=1e-15)


def test_whiten_inverse_factor_property():
    rng = np.random.default_rng(11)
    p = gen.random_problem(rng, 20, 5, m=4)
    w = oracle.whiten(p)
    for i in range(1, p.N):
        V = w["D"][i]                     # D_i = V_i (evolution H = I)
        np.testing.assert_allclose(V.T @ V @ p.K[i], np.eye(5), atol=1e-12)
        np.testing.assert_allclose(w["B"][i], V @ p.F[i], atol=1e-12)
        Wl = np.linalg.inv(np.linalg.cholesky(p.L[i][:4, :4]))
        np.testing.assert_allclose(w["C"][i][:4], Wl @ p.H[i][:4], atol=1e-12)
        assert np.allclose(np.triu(V, 1), 0.0)   # Cholesky-based: lower triangular


# ------------------------------------------------------------ scalar chain ---

def test_scalar_chain_worked_example():
    g = gold("scalar_chain.json")
    p = scalar_problem(2, g["F"], g["G"], g["K"], g["L"], g["o"])
    x, S = oracle.smooth(p)
    np.testing.assert_allclose(x[:, 0], g["states"], atol=1e-14)
    np.testing.assert_allclose(S[:, 0, 0], g["cov"], atol=1e-14)
    Rd, Ro, z = oracle.factor(p)
    Sd, Sx = oracle.selinv(Rd, Ro)
    np.testing.assert_allclose(Sx[0, 0, 0], g["cross_01"], atol=1e-14)
    R = np.array([[Rd[0, 0, 0], Ro[0, 0, 0]], [0.0, Rd[1, 0, 0]]])
    np.testing.assert_allclose(R.T @ R, np.array(g["gram"]), atol=1e-14)


def test_selinv_bidiagonal_worked_example():
    g = gold("selinv_bidiag.json")
    Rd = np.array(g["Rd"]).reshape(2, 1, 1)
    Ro = np.array([g["Ro01"], 0.0]).reshape(2, 1, 1)
    S, X = oracle.selinv(Rd, Ro)
    np.testing.assert_allclose(S[:, 0, 0], g["S_diag"], atol=1e-15)
    np.testing.assert_allclose(X[0, 0, 0], g["S_01"], atol=1e-15)


# ------------------------------------------------------------- dense pins ---

CASES = [(N, n, const, seed) for seed, (N, n) in enumerate(
    [(1, 2), (2, 1), (2, 3), (3, 2), (4, 4), (5, 3), (7, 2), (8, 5), (9, 1), (13, 3),
     (16, 2), (17, 4), (33, 3), (40, 5)]) for const in (False, True)]


@pytest.mark.parametrize("N,n,const,seed", CASES)
def test_oracle_vs_dense_lstsq_and_gram_inverse(N, n, const, seed):
    rng = np.random.default_rng(1000 + seed)
    m = None if N > 1 else n + 1
    p = gen.random_problem(rng, N, n, m=m, const=const)
    if N > 1:
        p.m[-1] = max(p.m[-1], 1)
    xd, Sd, kappa, _ = dense_solution(p)
    x, S = oracle.smooth(p)
    assert rel_state_err(x, xd) < 1e-13 * max(kappa, 10.0) * 10
    assert rel_cov_err(S, Sd) < 1e-13 * max(kappa, 10.0) ** 2
    assert np.allclose(S, np.swapaxes(S, 1, 2), atol=0)
    assert np.linalg.eigvalsh(S).min() > 0


@pytest.mark.parametrize("N,n,seed", [(5, 2, 0), (12, 3, 1), (31, 4, 2)])
def test_factor_gram_preservation_and_solve(N, n, seed):
    """R^T R = (UA)^T UA for the block-bidiagonal R."""
    rng = np.random.default_rng(seed)
    p = gen.random_problem(rng, N, n)
    Rd, Ro, z = oracle.factor(p)
    R = np.zeros((N * n, N * n))
    for i in range(N):
        R[i * n:(i + 1) * n, i * n:(i + 1) * n] = Rd[i]
        assert np.allclose(np.tril(Rd[i], -1), 0.0)
        if i + 1 < N:
            R[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = Ro[i]
    A, b = stacked(p)
    G = A.T @ A
    assert np.abs(R.T @ R - G).max() < 1e-12 * np.abs(G).max()
    # z = (Q^T U b)[:Nn]: R^T z = (UA)^T U b
    np.testing.assert_allclose(R.T @ z.reshape(-1), A.T @ b, rtol=1e-11, atol=1e-11 * np.abs(A.T @ b).max())
    x = oracle.solve(Rd, Ro, z)
    np.testing.assert_allclose(x.reshape(-1), np.linalg.solve(R, z.reshape(-1)), rtol=1e-10, atol=1e-12)
    S, X = oracle.selinv(Rd, Ro)
    Sfull = np.linalg.inv(R.T @ R)
    for i in range(N):
        np.testing.assert_allclose(S[i], Sfull[i * n:(i + 1) * n, i * n:(i + 1) * n], rtol=1e-9, atol=1e-12)
        if i + 1 < N:
            np.testing.assert_allclose(X[i], Sfull[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n],
                                       rtol=1e-9, atol=1e-12)


# ---------------------------------------------------------- special cases ---

@pytest.mark.parametrize("cfg,N", [("c1", 1000), ("c2", 600), ("c3", 600), ("c4", 40), ("c5", 4096)])
def test_noise_free_recovers_true_trajectory(cfg, N):
    """w = v = 0 => the residual of the true trajectory is exactly zero, so the
    least-squares estimate is the true state (up to rounding)."""
    p = gen.make(cfg, N=N, noise_free=True)
    x = oracle.smooth(p, cov=False)
    assert rel_state_err(x, p.x_true) < 1e-9


@pytest.mark.parametrize("rho,n", [(0.5, 3), (0.99, 2), (1.0, 3)])
def test_toeplitz_closed_form(rho, n):
    """F_i = rho Q, G_i = I, K = L = I: the interior Gram matrix is block
    Toeplitz tridiag(-rho Q^T, (2+rho^2) I, -rho Q), unitarily similar to the
    scalar tridiag(-rho, 2+rho^2, -rho) whose inverse has diagonal
    1/sqrt((2+rho^2)^2 - 4 rho^2) = 1/sqrt(4 + rho^4)."""
    rng = np.random.default_rng(5)
    Q = gen.haar_orthogonal(rng, 1, n)
    N = 201
    p = gen.Problem("toe", N, n, n, np.full(N, n, np.int32), rho * Q, np.eye(n)[None],
                    np.eye(n)[None], np.eye(n)[None], rng.standard_normal((N, n)))
    x, S = oracle.smooth(p)
    np.testing.assert_allclose(S[N // 2], np.eye(n) / np.sqrt(4 + rho ** 4), atol=1e-14)


def test_cv_model_dare_steady_state():
    """Config-5 model: interior smoothed covariances equal the stationary RTS
    smoother covariance from scipy's DARE / discrete Lyapunov solvers."""
    F, H, K, L = gen.cv_model()
    Pp = sla.solve_discrete_are(F.T, H.T, K, L)
    Pf = Pp - Pp @ H.T @ np.linalg.solve(H @ Pp @ H.T + L, H @ Pp)
    J = Pf @ F.T @ np.linalg.inv(Pp)
    Ps = sla.solve_discrete_lyapunov(J, Pf - J @ Pp @ J.T)
    p = gen.make("c5", N=2000)
    x, S = oracle.smooth(p)
    assert np.abs(S[1000] - Ps).max() < 1e-10 * np.abs(Ps).max()


def test_missing_observations_equal_zero_row_blocks():
    """m_i = 0 equals an explicit zero-row observation block."""
    rng = np.random.default_rng(3)
    p = gen.random_problem(rng, 9, 3, m=np.array([3, 0, 2, 0, 0, 3, 1, 0, 3]))
    xd, Sd, _, _ = dense_solution(p)
    x, S = oracle.smooth(p)
    assert rel_state_err(x, xd) < 1e-11 and rel_cov_err(S, Sd) < 1e-10


def test_error_not_spd():
    rng = np.random.default_rng(4)
    p = gen.random_problem(rng, 6, 2, m=2)
    p.K[3] = -np.eye(2)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.smooth(p)
    assert ei.value.code == oracle.ORA_ERR_NOT_SPD and ei.value.step == 3 and ei.value.kind == 1
    p = gen.random_problem(rng, 6, 2, m=2)
    p.L[4] = np.diag([1.0, -1.0])
    with pytest.raises(oracle.OracleError) as ei:
        oracle.smooth(p)
    assert ei.value.step == 4 and ei.value.kind == 2


def test_error_rank_deficient():
    rng = np.random.default_rng(5)
    p = gen.random_problem(rng, 5, 2, m=0)      # no observations at all
    with pytest.raises(oracle.OracleError) as ei:
        oracle.smooth(p)
    assert ei.value.code == oracle.ORA_ERR_RANK
    p = gen.random_problem(rng, 1, 3, m=2)      # one state, 2 < n observations
    with pytest.raises(oracle.OracleError) as ei:
        oracle.smooth(p)
    assert ei.value.code == oracle.ORA_ERR_RANK


def test_whitening_square_root_invariance():
    """Outputs do not depend on the whitening square root: the
    dense helper uses eigh-based inverse square roots, the oracle Cholesky;
    feeding the oracle pre-rotated covariances is covered by the lstsq pin.
    Here: scaling K and L by the same factor leaves the states unchanged."""
    rng = np.random.default_rng(6)
    p = gen.random_problem(rng, 10, 3)
    x1 = oracle.smooth(p, cov=False)
    p.K = p.K * 4.0
    p.L = p.L * 4.0
    x2, S2 = oracle.smooth(p)
    np.testing.assert_allclose(x1, x2, rtol=1e-11, atol=1e-12)


# ---- the general-model oracle (oracle/general.py) ----

@pytest.mark.parametrize("seed", range(8))
def test_general_oracle_vs_dense(seed):
    """Rectangular H_i (l_i x n_i) and per-step n_i: states = dense lstsq of
    the stacked general UA, covariances = diagonal blocks of inv(UA^T UA)."""
    from oracle import general as og
    from tests.dense import dense_solution_general
    rng = np.random.default_rng(100 + seed)
    n = 2 + seed % 4
    p = gen.general_problem(rng, 12 + 3 * seed, n, nmin=1 + seed % 2, rect=seed % 3 != 0)
    x, S = og.smooth_general(p)
    xd, Sd, kappa = dense_solution_general(p)
    assert rel_state_err(x, xd) < 1e-13 * max(kappa, 10.0) * 10
    err = np.abs(S - Sd).max() / np.abs(Sd).max()
    assert err < 1e-13 * max(kappa, 10.0) ** 2
    assert np.all(S[:, :, :] == np.swapaxes(S, 1, 2))


def test_general_oracle_noise_free_recovery():
    from oracle import general as og
    rng = np.random.default_rng(7)
    p = gen.general_problem(rng, 200, 6, nmin=2, noise_free=True)
    x = og.smooth_general(p, cov=False)
    assert rel_state_err(x, p.x_true) < 1e-10


def test_general_oracle_uniform_matches_c_oracle():
    """With H_i = I and l_i = n_i = n the general oracle solves the problem
    the plain-C oracle solves."""
    from oracle import general as og
    for cfg, N in (("c2", 60), ("c3", 61), ("c1", 40)):
        p = gen.make(cfg, N=N)
        x, S = og.smooth_general(p)
        xo, So = oracle.smooth(p)
        assert rel_state_err(x, xo) < 1e-12 and rel_cov_err(S, So) < 1e-12


def test_general_oracle_rank_deficient():
    from oracle import general as og
    rng = np.random.default_rng(3)
    p = gen.general_problem(rng, 10, 3, nmin=3, rect=False)
    p.m[:] = 0                   # no observations: x_0 undetermined
    with pytest.raises(og.GeneralOracleError):
        og.smooth_general(p)
